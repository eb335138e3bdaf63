"""Pins of the simulated GWPS/DBS schedule, the byte ledger and the paper's routing examples.

- schedule over P simulated devices == unpartitioned single-device AdamW step (≤1e-12, fp64);
- per-device ledger == SURVEY.md Appendix A closed forms, exactly (integers);
- per-remote-layer-step identity W_recv + G_sent = 2·φ_pad ("24H²", R14);
- per-device block receives 3L(P−1)φ_pad/P at r = 0;
- each of the six validator checks fails on exactly its mutation;
- the paper's P=6, D=2 worked example (tests/golden/paper_fig3_routes.txt).
"""
import os
from collections import defaultdict

import numpy as np
import pytest

import synth
from oracle import ledger as LG
from oracle import model as om
from oracle import routes
from oracle.schedule import CHECKS, GWPSSimulation, ValidationError

from test_oracle_model import flat, micro_params


def small_cfg(L):
    return om.ModelConfig(n_layers=L, hidden=16, heads=2, ffn=48, vocab=32, seq=8, micro_bs=1)


# (P, G, L, N): C0 shape 2×2, D=1 (FSDP-like), G=1 (pure P2P), 3×2, the paper's P=6 D=2, P=1
GRID = [(4, 2, 2, 4), (4, 4, 2, 4), (4, 1, 4, 4), (6, 2, 6, 6), (6, 3, 6, 6), (1, 1, 2, 2), (2, 1, 2, 4)]


@pytest.mark.parametrize("P,G,L,N", GRID)
def test_schedule_equals_unpartitioned_and_ledger_closed_form(P, G, L, N):
    cfg = small_cfg(L)
    params = micro_params(cfg)
    sim = GWPSSimulation(cfg, P, G, params)
    st = om.init_state(params)
    for step in range(2):
        toks = synth.tokens(N, 1, cfg.seq, cfg.vocab, step=step)
        ls = sim.step(toks)
        lr, _ = om.train_step(st, toks, cfg)
        assert abs(ls - lr) <= 1e-12 * abs(lr)
        a, b = flat(sim.assemble()), flat(st.params)
        assert np.max(np.abs(a - b)) / np.max(np.abs(b)) <= 1e-12
        s, e, f = sim.stripe_lengths()
        for d in range(P):
            expect = LG.closed_form(L, P, G, d // G, s, e, f, r=1)
            assert sim.fabric.ledger[d] == expect, (d, [(LG.name(i), x, y) for i, (x, y) in
                                                       enumerate(zip(sim.fabric.ledger[d], expect)) if x != y])


@pytest.mark.parametrize("P,G,L", [(4, 2, 2), (6, 2, 6), (6, 3, 6), (4, 1, 4), (4, 4, 4), (8, 2, 4)])
def test_ledger_r0_identities(P, G, L):
    cfg = small_cfg(L)
    sim = GWPSSimulation(cfg, P, G, micro_params(cfg), r=0)
    sim.step(synth.tokens(P, 1, cfg.seq, cfg.vocab))
    s, e, f = sim.stripe_lengths()
    phi_pad = s * G
    total = 0
    for d in range(P):
        led = sim.fabric.ledger[d]
        assert led == LG.closed_form(L, P, G, d // G, s, e, f, r=0)
        br = LG.block_received(led)
        assert br * P == 3 * L * (P - 1) * phi_pad       # every device, r = 0
        total += br
    assert total == 3 * L * (P - 1) * phi_pad
    D = P // G
    for d in range(P):
        led = sim.fabric.ledger[d]
        if D == 1:
            assert all(led[LG.index(k, "inter", di, u)] == 0 for k in LG.KINDS for di in LG.DIRS for u in LG.UNITS)
        if G == 1:
            assert all(led[LG.index(k, "intra", di, u)] == 0 for k in LG.KINDS for di in LG.DIRS for u in LG.UNITS)


@pytest.mark.parametrize("P,G,L", [(4, 2, 2), (6, 3, 6), (6, 2, 6)])
def test_per_remote_layer_step_is_two_shards(P, G, L):
    """"a single weight shard and its corresponding gradients per step" = 2φ (R14)."""
    cfg = small_cfg(L)
    sim = GWPSSimulation(cfg, P, G, micro_params(cfg))
    sim.step(synth.tokens(P, 1, cfg.seq, cfg.vocab))
    s, _, _ = sim.stripe_lengths()
    D = P // G
    w_recv = defaultdict(int)     # (device, layer) -> weight elements received in the forward gather
    g_sent = defaultdict(int)     # (device, layer) -> gradient elements sent
    for src, dst, tag, n, kind, cls in sim.fabric.log:
        uid = tag[1]
        if not isinstance(uid, int):
            continue
        if kind == "w":
            w_recv[(dst, uid)] += n
        else:
            g_sent[(src, uid)] += n
    checked = 0
    for d in range(P):
        k = d // G
        for l in range(L - 1):              # layer L−1 is gathered once (r = 1)
            if l % D != k:                  # remote layer-step
                fwd_recv = w_recv[(d, l)] // 2   # gathered for forward and again for backward
                assert fwd_recv == G * s == s * G
                assert fwd_recv + g_sent[(d, l)] == 2 * s * G
                checked += 1
    assert checked > 0 or D == 1


@pytest.mark.parametrize("mutation,check", [
    ("stale_version", "weight-presence"),
    ("drop_grad_msg", "gradient-exactly-once"),
    ("update_before_bwd", "update-ordering"),
    ("double_consume", "activation-consume-once"),
    ("extra_buffer", "buffer-bounds"),
    ("unmatched_send", "matching"),
])
def test_validator_catches_each_mutation(mutation, check):
    cfg = small_cfg(2)
    sim = GWPSSimulation(cfg, 4, 2, micro_params(cfg), mutate=mutation)
    with pytest.raises(ValidationError) as ei:
        sim.step(synth.tokens(4, 1, cfg.seq, cfg.vocab))
    assert ei.value.check == check
    assert set(CHECKS) >= {check}


def _golden():
    path = os.path.join(os.path.dirname(__file__), "golden", "paper_fig3_routes.txt")
    out = {}
    with open(path) as fh:
        lines = fh.readlines()
    for line in lines:
        if line.startswith("#") or not line.strip():
            continue
        k, *v = line.split()
        out[k] = [int(x) for x in v]
    return out


def test_paper_worked_example_P6_D2():
    g = _golden()
    P, D = g["P"][0], g["D"][0]
    assert routes.owner_table(P, D) == g["owner_of_shard"]
    # t = 0: P_0 broadcasts W_0 in g_0 (it is W_0's owner and g_0's holder)
    assert routes.rail_counterpart(0, 0, P, D) == g["t0_broadcaster_g0"][0]
    assert routes.forward_exchange(0, 1, P, D) == tuple(g["t0_send_W0_from_to"])
    assert routes.forward_exchange(1, 0, P, D) == tuple(g["t0_recv_W1_from_to"])
    # t = 4: P_2 holds W_4 and receives W_5 from P_5
    assert routes.owner_table(P, D)[4] == g["t4_holder_W4"][0]
    assert routes.forward_exchange(5, 0, P, D) == tuple(g["t4_recv_W5_from_to"])
    # backward of W_{L−1}: reduced in g_0 to P_{P/D−1}, sent to the owner P_{P−1}
    exit_dev, owner = routes.backward_route(P - 1, 0, P, D)
    assert exit_dev == g["bwd_W5_group0_reduce_to"][0] == P // D - 1
    assert owner == g["bwd_W5_send_to_owner"][0] == P - 1
    assert routes.owner_table(P, D)[5] == g["t7_updater_W5"][0]
    assert routes.owner_table(8, 2) == g["P8_D2_owner_of_shard"]


def test_shard_map_bijection_up_to_64():
    for P in range(1, 65):
        for D in range(1, P + 1):
            if P % D == 0:
                own = routes.owner_table(P, D)
                assert sorted(own) == list(range(P))


def test_striped_group_map_equals_paper_group_map_when_L_equals_P():
    """R6: at L = P, layer l's owner group l mod D equals the paper's group of W_l's owner."""
    for P, D in [(6, 2), (8, 2), (8, 4), (6, 3), (4, 2)]:
        G = P // D
        own = routes.owner_table(P, D)
        for l in range(P):
            assert own[l] // G == l % D


@pytest.mark.parametrize("P,L", [(2, 2), (3, 3), (4, 4), (4, 8), (5, 10), (8, 8)])
def test_ring_ledger_sent_side_conservation_and_hop_count(P, L):
    """Pins ring_ledger's SENT counters (the receive side is pinned by the 3L(P−1)φ/P identity): on a ring every
    transfer is one hop, so summed over the P devices sent == received for every (kind, unit); and a gather
    (reduction) of a unit of n elements moves it over exactly P − 1 ring edges, so the job-wide sent total is
    (P − 1) × Σ n over the step's 2L − 1 + 2 gathers (L + 2 reductions)."""
    s, e, f = 1000, 70, 90
    leds = [LG.ring_ledger(L, P, d, s, e, f, r=1) for d in range(P)]
    for kind in LG.KINDS:
        for unit in LG.UNITS:
            for cls in LG.CLASSES:
                sent = sum(x[LG.index(kind, cls, "sent", unit)] for x in leds)
                recv = sum(x[LG.index(kind, cls, "recv", unit)] for x in leds)
                assert sent == recv, (kind, cls, unit, sent, recv)
    n_gather = {"block": (2 * L - 1) * s, "E": e, "F": f}
    n_reduce = {"block": L * s, "E": e, "F": f}
    for unit in LG.UNITS:
        assert sum(x[LG.index("w", "inter", "sent", unit)] for x in leds) == (P - 1) * n_gather[unit]
        assert sum(x[LG.index("g", "inter", "sent", unit)] for x in leds) == (P - 1) * n_reduce[unit]
        assert all(x[LG.index(k, "intra", dr, unit)] == 0 for x in leds for k in LG.KINDS for dr in LG.DIRS)


@pytest.mark.parametrize("P,G,L", [(4, 2, 4), (6, 2, 6), (6, 3, 6), (8, 2, 8), (4, 4, 4), (4, 1, 4)])
def test_gwps_and_literal_ledgers_conserve_every_transfer(P, G, L):
    """Every logical transfer has one sender and one receiver: summed over the P devices, sent == received per
    (kind, class, unit), for the striped closed forms (App. A) and for the paper-literal enumeration."""
    D = P // G
    s, e, f = 64 * G * 3, 64 * G, 64 * G * 2
    striped = [LG.closed_form(L, P, G, d // G, s // G, e // G, f // G, r=1) for d in range(P)]
    literal = [LG.literal_ledger(L, P, D, d, s, e, f, r=1) for d in range(P)] if L % P == 0 else []
    for leds in (striped, literal):
        if not leds:
            continue
        for kind in LG.KINDS:
            for cls in LG.CLASSES:
                for unit in LG.UNITS:
                    sent = sum(x[LG.index(kind, cls, "sent", unit)] for x in leds)
                    recv = sum(x[LG.index(kind, cls, "recv", unit)] for x in leds)
                    assert sent == recv, (kind, cls, unit, sent, recv)
