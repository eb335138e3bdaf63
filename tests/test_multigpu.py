"""Multi-GPU parity of the GWPS/DBS/CCO step (one process per GPU over NCCL, launched with torchrun):
losses and updated weights vs the fp64 oracle's single-device step, and every rank's byte ledger vs the
closed forms of SURVEY.md App. A (bit-exact).  Runs only when the box has >= P GPUs
(gpurun --gpus 2 / --gpus 4)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import synth
from helpers import C0, C0B, ROOT, TOL_DELTA, om, oracle_cfg, reassemble, tensors, weight_errors
from oracle import layout as OL
from oracle import ledger as LG

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

# (name, base dims, P, G, L, N, dtype, ckpt, no_cco, ring[, emulated inter-node GB/s, emulated node size])
CASES = [
    ("c0-1x2-fsdp", C0, 2, 2, 2, 4, 0, 0, False, False),
    ("c0-2x1-p2p", C0, 2, 1, 2, 4, 0, 0, False, False),
    ("c0-2x2", C0, 4, 2, 2, 4, 0, 0, False, False),          # BASELINE.json configs[0]
    ("c0-2x2-nocco", C0, 4, 2, 2, 4, 0, 0, True, False),
    ("c0-1x4", C0, 4, 4, 2, 8, 0, 1, False, False),
    ("c0-4x1", C0, 4, 1, 4, 4, 0, 0, False, False),
    ("c0b-2x2-bf16", C0B, 4, 2, 2, 4, 1, 1, False, False),
    ("c0b-1x2-bf16", C0B, 2, 2, 2, 2, 1, 0, False, False),
    ("c0-ring2", C0, 2, 1, 2, 4, 0, 0, False, True),          # NEXT-1 WeiPipe-style ring
    ("c0-ring4", C0, 4, 1, 4, 4, 0, 2, False, True),         # ckpt 2: full recompute
    ("c0b-ring4-bf16", C0B, 4, 1, 4, 4, 1, 0, False, True),
    # NEXT-3: 2 emulated nodes of 2 at 0.05 GB/s: same results and ledger, paced rail traffic
    ("c0-2x2-emu", C0, 4, 2, 2, 4, 0, 0, False, False, 0.05, 2),
    ("c0-ring4-emu", C0, 4, 1, 4, 4, 0, 0, False, True, 0.05, 2),
    # NEXT-2 paper-literal collectives (ring field = "literal"): whole-layer owners, broadcast / reduce in groups
    ("c0-literal-2x2", C0, 4, 2, 4, 4, 0, 0, False, "literal"),
    ("c0-literal-4x1", C0, 4, 1, 4, 4, 0, 1, False, "literal"),
    ("c0b-literal-1x4-bf16", C0B, 4, 4, 4, 4, 1, 0, False, "literal"),
    ("c0-literal-2x2-emu", C0, 4, 2, 4, 4, 0, 0, False, "literal", 0.05, 2),
]
CASES = [c if len(c) == 12 else c + (0.0, 0) for c in CASES]
# every case runs AdamW in its linear regime (ε = 1 ≫ |g|, lr = 1, no decay: Δ ≈ −m̂, R18) so that e_Δ sees a wrong
# gradient scale (a double-counted or missing group partial); two cases keep the default ε = 1e-8 (e_θ only)
# GWPS runs the NVLink peer path by default (IPC copies + in-kernel gradient reads); "-nccl" cases force the NCCL
# collectives (TAWPIPE_COMM=nccl) so both implementations of a3/a8/a9 stay covered
CASES += [("c0-2x2-nccl", C0, 4, 2, 2, 4, 0, 0, False, False, 0.0, 0),
          ("c0b-2x2-bf16-nccl", C0B, 4, 2, 2, 4, 1, 1, False, False, 0.0, 0),
          ("c0-2x2-g2x-p2p-bf16-ckpt2", C0B, 4, 2, 4, 8, 1, 2, False, False, 0.0, 0),
          ("c0-1x2-fsdp-bf16", C0B, 2, 2, 2, 4, 1, 0, False, False, 0.0, 0),
          ("c0-2x1-bf16", C0B, 2, 1, 2, 2, 1, 0, False, False, 0.0, 0),
          # D = 4 groups of 1 with 8 layers: consecutive layers sharing a buffer slot have different owners
          ("c0b-4x1-L8-bf16", C0B, 4, 1, 8, 4, 1, 1, False, False, 0.0, 0),
          ("c0b-4x1-L8-bf16-nccl", C0B, 4, 1, 8, 4, 1, 1, False, False, 0.0, 0),
          ("c0b-2x2-L4-bf16-nccl", C0B, 4, 2, 4, 8, 1, 2, False, False, 0.0, 0),
          ("c0-4x1-L8-fp32", C0, 4, 1, 8, 4, 0, 1, False, False, 0.0, 0),
          # P = 8 (skipped below 8 GPUs): the headline 4 x 2 split, D = 8 groups of 1, 2 x 4, the FSDP-style 1 x 8,
          # the ring and the paper-literal mode at P = 8
          ("c0-4x2-p8", C0, 8, 2, 4, 8, 0, 0, False, False, 0.0, 0),
          ("c0b-4x2-p8-bf16", C0B, 8, 2, 8, 8, 1, 1, False, False, 0.0, 0),
          ("c0-8x1-p8", C0, 8, 1, 8, 8, 0, 0, False, False, 0.0, 0),
          ("c0-2x4-p8", C0, 8, 4, 2, 8, 0, 0, False, False, 0.0, 0),
          ("c0-1x8-fsdp-p8", C0, 8, 8, 2, 8, 0, 0, False, False, 0.0, 0),
          ("c0-ring8", C0, 8, 1, 8, 8, 0, 0, False, True, 0.0, 0),
          ("c0-literal-4x2-p8", C0, 8, 2, 8, 8, 0, 0, False, "literal", 0.0, 0)]
CASES = [c + (True,) for c in CASES] + [("c0-2x2-default-eps", C0, 4, 2, 2, 4, 0, 0, False, False, 0.0, 0, False),
                                       ("c0b-1x2-bf16-default-eps", C0B, 2, 2, 2, 2, 1, 0, False, False, 0.0, 0,
                                        False)]


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run_torchrun(cmd, env, timeout=300):
    """Run a torchrun command; the probed free port can be taken between probing and torchrun's bind, so retry with a
    new port on EADDRINUSE."""
    for _ in range(3):
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env)
        if "EADDRINUSE" not in r.stderr:
            return r
        i = next(k for k, c in enumerate(cmd) if c.startswith("--master-port="))
        cmd[i] = f"--master-port={free_port()}"
    return r


@pytest.mark.parametrize("name,base,P,G,L,N,dtype,ckpt,no_cco,ring,emu_gbps,emu_node,linear", CASES,
                         ids=[c[0] for c in CASES])
def test_multigpu_step_matches_oracle(tmp_path, name, base, P, G, L, N, dtype, ckpt, no_cco, ring, emu_gbps, emu_node,
                                      linear):
    literal = ring == "literal"
    ring = ring is True
    if not torch.cuda.is_available() or torch.cuda.device_count() < P:
        pytest.skip(f"needs {P} GPUs")
    hyper = dict(lr=1.0, adam_eps=1.0, weight_decay=0.0) if linear else {}
    cfg = oracle_cfg(base, n_layers=L, **hyper)
    steps = 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.join(ROOT, "tests", "mp_worker.py"),
           "--cfg", json.dumps(dict(base, n_layers=L)), "--G", str(G), "--N", str(N), "--steps", str(steps),
           "--dtype", str(dtype), "--ckpt", str(ckpt), "--out", str(tmp_path)] + (["--no-cco"] if no_cco else []) \
        + (["--ring"] if ring else []) + (["--literal"] if literal else []) + (["--linear"] if linear else []) \
        + (["--emu-gbps", str(emu_gbps), "--emu-node", str(emu_node)] if emu_gbps else [])
    env = dict(os.environ, TAWPIPE_COMM="nccl") if name.endswith("-nccl") else dict(os.environ)
    r = run_torchrun(cmd, env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = [np.load(tmp_path / f"rank{i}.npz") for i in range(P)]
    # which implementation ran: the peer path for GWPS unless forced to NCCL; ring / literal always NCCL
    want_p2p = not (ring or literal or name.endswith("-nccl"))
    assert all(bool(x["p2p"]) == want_p2p for x in res), [float(x["p2p"]) for x in res]
    # oracle: plain single-device step on the same tokens
    params = synth.perturb_gains(synth.init_params(cfg.n_layers, cfg.hidden, cfg.ffn, cfg.vocab))
    st = om.init_state(params)
    theta0 = om.to_f64(params)
    grads = []
    tol_loss, tol_w, kappa = (1e-5, 1e-4, 1e-3) if dtype == 0 else (1e-2, 2e-2, 5e-2)
    tol_d = TOL_DELTA[dtype]
    for step in range(steps):
        toks = synth.tokens(N, cfg.micro_bs, cfg.seq, cfg.vocab, step=step)
        lr, g = om.train_step(st, toks, cfg)
        grads.append(g)
        for i in range(P):   # identical loss on every rank
            assert abs(res[i]["losses"][step] - lr) / lr <= tol_loss, (i, step, res[i]["losses"][step], lr)
        if step == 0:
            theta1 = {k: v for k, v in st.params.items()}
    gpu = reassemble(cfg, P, G, [x["shard"] for x in res], literal=literal)
    et, ed, viol, off, rep = weight_errors(gpu, st.params, theta0, grads, cfg, kappa)
    print(f"{name}: e_theta {et:.2e} e_delta {ed:.2e} off-W {off:.3%} violations {viol}")
    assert et <= tol_w and viol == 0 and (ed <= tol_d or not linear), (
        et, ed, viol, sorted(rep, key=lambda z: -max(z[1], z[2]))[:3])
    # byte ledger: bit-exact against the closed forms, every rank, every step
    H, V = cfg.hidden, cfg.vocab
    s, e, f = (OL.padded(n, G) // G for n in (om.phi(cfg), V * H, H + V * H))
    for i in range(P):
        if ring:
            expect = LG.ring_ledger(L, P, i, s, e, f, r=1)
        elif literal:
            expect = LG.literal_ledger(L, P, P // G, i, *(OL.padded(n, 1) for n in (om.phi(cfg), V * H, H + V * H)))
        else:
            expect = LG.closed_form(L, P, G, i // G, s, e, f, r=1)
        for step in range(steps):
            assert [int(x) for x in res[i]["ledgers"][step]] == expect, (i, step)
    if emu_gbps and not ring and not literal:
        # NEXT-3 pacing: every rail exchange (D > 1, groups = emulated nodes) adds 30 µs + (D−1)·stripe bytes / bw
        # to each participant's comm stream: gathers E, L blocks, F and L−1 re-gathers; reductions F, L blocks, E
        D, esz = P // G, (4 if dtype == 0 else 2)
        units = [e] + [s] * L + [f] + [s] * (L - 1) + [f] + [s] * L + [e]
        expect_ms = sum(30e-3 + (D - 1) * n * esz / (emu_gbps * 1e9) * 1e3 for n in units)
        for i in range(P):
            for step in range(steps):
                assert res[i]["comm_ms"][step] >= 0.95 * expect_ms, (i, step, res[i]["comm_ms"][step], expect_ms)


def test_peer_flag_invariant_catches_a_misnumbered_signal(tmp_path):
    """Race detector mutation test: with TAWPIPE_FAULT=gdone+1 member 0 of a 1×2 group over-numbers its last GDONE of
    the step by one.  No wait blocks (waits are "≥"), so only the end-of-step flag check can see it: the step on
    member 1 must fail with TAWPIPE_EINVARIANT naming the flag, instead of silently letting a later step run early."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.join(ROOT, "tests", "mp_worker.py"),
           "--cfg", json.dumps(dict(C0B, n_layers=2)), "--G", "2", "--N", "2", "--steps", "1", "--dtype", "1",
           "--out", str(tmp_path)]
    r = run_torchrun(cmd, dict(os.environ, TAWPIPE_FAULT="gdone+1"))
    out = r.stdout + r.stderr
    assert r.returncode != 0 and "peer flag GDONE" in out and "expected" in out, out[-3000:]


def test_ledger_invariant_catches_a_skipped_transfer(tmp_path):
    """Mutation test of the ledger = plan invariant: with TAWPIPE_FAULT=skip-e-gather the peer path leaves its E
    gather out of the step's byte ledger (as a schedule that dropped the transfer would); the end-of-step check must
    fail the step with TAWPIPE_EINVARIANT naming the counter."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.join(ROOT, "tests", "mp_worker.py"),
           "--cfg", json.dumps(dict(C0B, n_layers=2)), "--G", "2", "--N", "2", "--steps", "1", "--dtype", "1",
           "--out", str(tmp_path)]
    r = run_torchrun(cmd, dict(os.environ, TAWPIPE_FAULT="skip-e-gather"))
    out = r.stdout + r.stderr
    assert r.returncode != 0 and "step ledger counter" in out and "the plan's" in out, out[-3000:]


@pytest.mark.parametrize("P,G", [(2, 2), (2, 1)])
def test_device_init_is_partition_independent(tmp_path, P, G):
    """R20: the seeded device-side initialisation is a function of the canonical parameter position only, so the
    stripes P ranks initialise reassemble bit for bit into the model one rank initialises."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < P:
        pytest.skip(f"needs {P} GPUs")
    cfg = oracle_cfg(C0B)
    shards = {}
    for p, g in ((1, 1), (P, G)):
        out = tmp_path / f"p{p}g{g}"
        out.mkdir()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={p}",
               "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.join(ROOT, "tests", "mp_worker.py"),
               "--cfg", json.dumps(C0B), "--G", str(g), "--N", str(p), "--dtype", "1", "--init-only", "--out", str(out)]
        r = run_torchrun(cmd, dict(os.environ))
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
        shards[p] = reassemble(cfg, p, g, [np.load(out / f"rank{i}.npz")["shard"] for i in range(p)])
    for (name, a), (_, b) in zip(tensors(shards[1]), tensors(shards[P])):
        assert np.array_equal(a, b), name
