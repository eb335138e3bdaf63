"""The C-ABI boundary used from C alone: examples/train_step.c includes include/tawpipe.h, links libtawpipe.so and
drives bootstrap -> init -> load -> step -> shard -> finalize with no Python in the process.

CPU: the program compiles and links against the library (no run).  GPU: two steps of C0 (fp32) through the C
program match the fp64 oracle's losses and weights at the fp32 step tolerances of tests/test_gpu_step.py; on two
GPUs, two C processes (1 x 2 and 2 x 1, NCCL id exchanged through a file, no torch.distributed) do the same."""
import os
import shutil
import subprocess

import numpy as np
import pytest

import synth
from helpers import C0, ROOT, om, oracle_cfg, reassemble, weight_errors

SRC = os.path.join(ROOT, "examples", "train_step.c")
LIBDIR = os.path.join(ROOT, "paper_2511_09741_b200")


def compile_example(out_dir):
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    if not os.path.exists(os.path.join(LIBDIR, "libtawpipe.so")):
        from paper_2511_09741_b200 import build
        build.build()
    exe = os.path.join(str(out_dir), "train_step")
    cmd = ["gcc", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"), SRC, "-L", LIBDIR,
           "-ltawpipe", f"-Wl,-rpath,{LIBDIR}", "-Wl,--allow-shlib-undefined", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_example_compiles_and_links(tmp_path):
    exe = compile_example(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True)   # usage only: no GPU call without arguments
    assert r.returncode == 2 and "usage" in r.stderr


def run_c_job(tmp_path, world, group, n_micro=4, steps=2):
    """Run examples/train_step.c as `world` processes (one per GPU) on C0 fp32; check losses and weights against
    the oracle."""
    exe = compile_example(tmp_path)
    cfg = oracle_cfg(C0)
    params = synth.perturb_gains(synth.init_params(cfg.n_layers, cfg.hidden, cfg.ffn, cfg.vocab))
    from paper_2511_09741_b200 import tawpipe as T
    T.pack_full_model(params).astype(np.float32).tofile(tmp_path / "w.f32")
    toks = [synth.tokens(n_micro, cfg.micro_bs, cfg.seq, cfg.vocab, step=s) for s in range(steps)]
    np.concatenate([t.astype(np.int32).ravel() for t in toks]).tofile(tmp_path / "tok.i32")
    procs = []
    for rank in range(world):
        args = [exe, str(cfg.n_layers), str(cfg.hidden), str(cfg.heads), str(cfg.ffn), str(cfg.vocab), str(cfg.seq),
                str(cfg.micro_bs), str(n_micro), str(T.FP32), str(steps), str(tmp_path / "tok.i32"),
                str(tmp_path / "w.f32"), str(tmp_path / f"shard{rank}.f32")]
        env = dict(os.environ, TAWPIPE_RANK=str(rank), TAWPIPE_WORLD=str(world), TAWPIPE_GROUP=str(group),
                   TAWPIPE_ID_FILE=str(tmp_path / "nccl.id"))
        procs.append(subprocess.Popen(args, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, env=env))
    outs = [p.communicate(timeout=300) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, o + e
    losses = [[float(line.split()[2]) for line in o.splitlines() if line.startswith("loss ")] for o, _ in outs]
    assert all(len(x) == steps for x in losses) and all(x == losses[0] for x in losses)   # global mean loss
    losses = losses[0]

    st = om.init_state(params)
    theta0 = om.to_f64(params)
    grads_all = []
    for s in range(steps):
        lr, grads = om.train_step(st, toks[s], cfg)
        grads_all.append(grads)
        assert abs(losses[s] - lr) / abs(lr) <= 1e-5, (s, losses[s], lr)
    shards = [np.fromfile(tmp_path / f"shard{r}.f32", dtype=np.float32) for r in range(world)]
    gpu = reassemble(cfg, world, group, shards)
    et, ed, viol, off, rep = weight_errors(gpu, st.params, theta0, grads_all, cfg, 1e-3)
    assert et <= 1e-4 and viol == 0, (et, viol)


@pytest.mark.gpu
def test_c_example_two_steps_match_oracle(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    run_c_job(tmp_path, 1, 1)


@pytest.mark.gpu
@pytest.mark.multigpu
@pytest.mark.parametrize("group", [2, 1])
def test_c_example_two_ranks_match_oracle(tmp_path, group):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    run_c_job(tmp_path, 2, group)
