"""CPU checks of bench.py's host logic: the FLOP-per-token model behind every roofline number is pinned to
SURVEY.md §8(d)'s table (App. B formulas, computed independently there), and the reference arm (the fp64 oracle on
the host cores) prints the JSON line the driver contract asks for."""
import json
import os
import subprocess
import sys

import pytest

from helpers import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402


# SURVEY.md §8(d) table, "FLOP/token (fwd / train)" column, in GFLOP per token
@pytest.mark.parametrize("name,fwd,train", [("c1", 3.403, 10.208), ("c2", 4.208, 12.624), ("c3", 21.804, 65.413),
                                            ("c4", 32.415, 97.244)])
def test_flops_per_token_matches_survey_table(name, fwd, train):
    c = bench.CONFIGS[name]
    got_train = bench.flops_per_token(c, recompute=False) / 1e9
    assert abs(got_train - train) <= 1e-3 * train, (got_train, train)
    assert abs(got_train / 3 - fwd) <= 1e-3 * fwd


def test_c3_recompute_counts_every_layer_but_the_resident_one():
    # checkpointing recomputes every layer's forward except the last layer's last micro-batch (still resident):
    # (L − 1/m) layers per token on top of the 3× train FLOPs
    c = bench.CONFIGS["c3"]
    H, I, S = c["H"], c["I"], c["S"]
    layer_fwd = 2 * (4 * H * H + 3 * H * I) + 2 * H * (S + 1)
    assert abs(layer_fwd / 1e6 - 673.2) < 0.1                      # 673.2 M per token per layer
    full = bench.flops_per_token(c, recompute=True)
    assert abs(full - bench.flops_per_token(c, recompute=False) - (c["L"] - 1 / c["m"]) * layer_fwd) < 1.0


def test_reference_arm_prints_the_contract_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 1
    assert d["unit"] == "tokens/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["metric"] == bench.METRIC and d["config"]["workload"].startswith("C3")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["sample"] and cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
