"""CPU checks of the library's host logic (no GPU): the DBS plan's byte ledger (tawpipe_plan, the same
accounting code the NCCL calls use) equals SURVEY.md App. A's closed forms exactly for every rank of a grid
of (P, G, L); configuration errors name the violated constraint; the N>1 bootstrap distributes one NCCL
unique id to every rank over a world-size-2 gloo process group."""
import os

import pytest

from helpers import C0, om, oracle_cfg
from oracle import layout as OL
from oracle import ledger as LG

GRID = [(1, 1, 2), (2, 1, 2), (2, 2, 2), (4, 2, 2), (4, 4, 2), (4, 1, 4), (6, 2, 6), (6, 3, 6), (8, 2, 4),
        (8, 4, 2), (8, 8, 2), (8, 1, 8), (8, 2, 32), (3, 1, 3)]


@pytest.fixture(scope="module")
def T():
    from paper_2511_09741_b200 import build, tawpipe
    build.build()
    return tawpipe


def dims_for(T, cfg, dtype=0):
    return T.ModelDims(n_layers=cfg.n_layers, hidden=cfg.hidden, heads=cfg.heads, ffn=cfg.ffn, vocab=cfg.vocab,
                       seq=cfg.seq, micro_bs=cfg.micro_bs, dtype=dtype)


@pytest.mark.parametrize("P,G,L", GRID)
def test_plan_ledger_equals_closed_form(T, P, G, L):
    cfg = oracle_cfg(C0, n_layers=L)
    H, V = cfg.hidden, cfg.vocab
    s = OL.padded(om.phi(cfg), G) // G
    e = OL.padded(V * H, G) // G
    f = OL.padded(H + V * H, G) // G
    D = P // G
    for rank in range(P):
        led, n = T.plan(P, G, dims_for(T, cfg), P, rank)
        k = rank // G
        assert led == LG.closed_form(L, P, G, k, s, e, f, r=1), (rank, [(LG.name(i), a, b) for i, (a, b) in
                                                                   enumerate(zip(led, LG.closed_form(
                                                                       L, P, G, k, s, e, f, r=1))) if a != b])
        owned = sum(1 for l in range(L) if l % D == k)
        assert n == owned * s + (e if k == 0 else 0) + (f if k == D - 1 else 0)


def test_plan_c3_ledger_matches_survey_table(T):
    """SURVEY.md App. A concrete values, C3 (7B) on 4x2: group 0 block elements."""
    cfg = om.ModelConfig(n_layers=32, hidden=4096, heads=32, ffn=11008, vocab=32000, seq=32768)
    led, _ = T.plan(8, 2, dims_for(T, cfg, dtype=1), 8, 0)
    assert led[LG.index("w", "intra", "recv", "block")] == 6_375_075_840
    assert led[LG.index("w", "inter", "recv", "block")] == 4_756_008_960
    assert led[LG.index("g", "intra", "recv", "block")] == 3_238_133_760
    assert led[LG.index("g", "inter", "recv", "block")] == 2_428_600_320
    assert led[LG.index("g", "inter", "sent", "block")] == 2_428_600_320
    led3, _ = T.plan(8, 2, dims_for(T, cfg, dtype=1), 8, 6)
    assert led3[LG.index("w", "inter", "recv", "block")] == 4_857_200_640


@pytest.mark.parametrize("P,G,L,N,msg", [(4, 3, 2, 4, "P mod G"), (4, 2, 3, 4, "L mod D"), (4, 2, 2, 6, "N mod P")])
def test_config_errors_name_the_constraint(T, P, G, L, N, msg):
    cfg = oracle_cfg(C0, n_layers=L)
    with pytest.raises(T.TawpipeError) as ei:
        T.plan(P, G, dims_for(T, cfg), N, 0)
    assert ei.value.code == T.ECONFIG and msg in str(ei.value)


def test_bf16_shape_limits(T):
    cfg = oracle_cfg(C0)   # d_h = 16 is fine in fp32, not on the tcgen05 path
    T.plan(1, 1, dims_for(T, cfg, dtype=0), 1, 0)
    with pytest.raises(T.TawpipeError) as ei:
        T.plan(1, 1, dims_for(T, cfg, dtype=1), 1, 0)
    assert "d_h" in str(ei.value)


def _uid_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    from paper_2511_09741_b200 import tawpipe as T
    uid = T.share_unique_id(rank, world, "gloo")
    out[rank] = uid.hex()
    import torch.distributed as dist
    dist.destroy_process_group()


def test_bootstrap_unique_id_over_gloo_world2():
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_uid_worker, args=(2, port, out), nprocs=2, join=True)
    assert len(out) == 2 and out[0] == out[1] and len(bytes.fromhex(out[0])) == 128


@pytest.mark.parametrize("P,L", [(2, 2), (3, 3), (4, 4), (4, 8), (8, 8), (8, 32), (6, 6)])
def test_ring_plan_ledger_and_3L_identity(T, P, L):
    """NEXT-1 WeiPipe-style ring: plan ledger == the ring's definition; 3L(P−1)φ/P per device at r = 0."""
    cfg = oracle_cfg(C0, n_layers=L)
    H, V = cfg.hidden, cfg.vocab
    s = OL.padded(om.phi(cfg), 1)
    e = OL.padded(V * H, 1)
    f = OL.padded(H + V * H, 1)
    d = dims_for(T, cfg)
    d.schedule = T.RING
    for rank in range(P):
        led, _ = T.plan(P, 1, d, P, rank)
        assert led == LG.ring_ledger(L, P, rank, s, e, f, r=1)
        r0 = LG.ring_ledger(L, P, rank, s, e, f, r=0)
        assert LG.block_received(r0) * P == 3 * L * (P - 1) * s
    # same per-device block receive total as GWPS at r = 0 (TawPipe, FSDP and a ring alike)
    sg = OL.padded(om.phi(cfg), 1)
    for rank in range(P):
        gw = LG.closed_form(L, P, 1, rank, sg, e, f, r=0)
        assert LG.block_received(gw) == LG.block_received(LG.ring_ledger(L, P, rank, s, e, f, r=0))


def test_ring_requires_group_size_1(T):
    cfg = oracle_cfg(C0)
    d = dims_for(T, cfg)
    d.schedule = T.RING
    with pytest.raises(T.TawpipeError) as ei:
        T.plan(4, 2, d, 4, 0)
    assert "group_size" in str(ei.value)
