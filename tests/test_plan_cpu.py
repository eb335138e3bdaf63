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
    mgr = mp.get_context("spawn").Manager()   # no fork of this multi-threaded process
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


LITERAL_GRID = [(1, 1, 2), (2, 1, 2), (2, 2, 2), (4, 2, 4), (4, 4, 4), (4, 1, 4), (6, 3, 6), (6, 2, 6), (6, 3, 12),
                (8, 2, 8), (8, 4, 16), (8, 8, 8), (8, 1, 8)]


@pytest.mark.parametrize("P,G,L", LITERAL_GRID)
def test_literal_plan_ledger_and_identities(T, P, G, L):
    """NEXT-2 paper-literal mode: the plan's ledger equals the enumerated definition (oracle/ledger.py over
    oracle/routes.py's PAPER.md:123 map), every device receives 3L(P−1)φ/P block elements at r = 0 (SURVEY App. A:
    the same as the striped mode), and each device owns exactly L/P whole layers."""
    cfg = oracle_cfg(C0, n_layers=L)
    H, V = cfg.hidden, cfg.vocab
    x, e, f = OL.padded(om.phi(cfg), 1), OL.padded(V * H, 1), OL.padded(H + V * H, 1)
    D = P // G
    d = dims_for(T, cfg)
    d.schedule = T.LITERAL
    for rank in range(P):
        led, n = T.plan(P, G, d, P, rank)
        assert led == LG.literal_ledger(L, P, D, rank, x, e, f, r=1), (rank, [(LG.name(i), a, b) for i, (a, b) in
                                                                       enumerate(zip(led, LG.literal_ledger(
                                                                           L, P, D, rank, x, e, f, r=1))) if a != b])
        r0 = LG.literal_ledger(L, P, D, rank, x, e, f, r=0)
        assert LG.block_received(r0) * P == 3 * L * (P - 1) * x
        assert n == (L // P) * x + (e if rank == 0 else 0) + (f if rank == P - 1 else 0)


def test_literal_paper_example_p6_d2(T):
    """PAPER.md:127 worked example, P = 6, D = 2 (tests/golden/paper_fig3_routes.txt): W_5 is owned by P_5; its
    gradient computed in g_0 is reduced to P_2 and transferred to P_5 -- so in the backward of layer 5, P_2 sends one
    whole layer on the rail and P_5 receives one; in the forward P_0 broadcasts W_0 in g_0 and sends it to P_3."""
    cfg = oracle_cfg(C0, n_layers=6)
    x = OL.padded(om.phi(cfg), 1)
    d = dims_for(T, cfg)
    d.schedule = T.LITERAL
    led = {r: T.plan(6, 3, d, 6, r)[0] for r in range(6)}
    # one layer per device; every layer is gathered twice but layer 5 (r = 1) -> owner P_5 sends layer 5 once on
    # the rail (forward) and P_0 sends layer 0 twice (forward + backward)
    assert led[0][LG.index("w", "inter", "sent", "block")] == 2 * x
    assert led[5][LG.index("w", "inter", "sent", "block")] == 1 * x
    assert led[5][LG.index("g", "inter", "recv", "block")] == 1 * x     # W_5's gradient from g_0 (via P_2)
    assert led[2][LG.index("g", "inter", "sent", "block")] == 1 * x     # P_2 = P_{P/D-1} exits W_5's gradient of g_0
    assert led[2][LG.index("g", "inter", "recv", "block")] == 1 * x     # P_2 owns W_4: receives g_1's partial (P_5)


def test_literal_requires_l_mod_p(T):
    cfg = oracle_cfg(C0, n_layers=2)
    d = dims_for(T, cfg)
    d.schedule = T.LITERAL
    with pytest.raises(T.TawpipeError) as ei:
        T.plan(4, 2, d, 4, 0)
    assert "L mod P" in str(ei.value)
    d.schedule = T.LITERAL | T.RING
    with pytest.raises(T.TawpipeError):
        T.plan(2, 1, d, 2, 0)
