"""Test-side helpers: GPU-run harness, shard reassembly and the weight-parity metric."""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import layout as OL  # noqa: E402
from oracle import model as om   # noqa: E402

# C0 (BASELINE.json configs[0]) and the bf16 parity twin C0b
C0 = dict(n_layers=2, hidden=64, heads=4, ffn=192, vocab=256, seq=128, micro_bs=1)
C0B = dict(n_layers=2, hidden=256, heads=2, ffn=768, vocab=512, seq=256, micro_bs=1)


# e_Δ bar in the linear AdamW regime (ε = 1 ≫ |g|, lr = 1, no decay; R18 in DESIGN.md): there Δ ≈ −m̂ ∝ g, so e_Δ is
# the gradient error relative to the tensor's largest gradient element.  fp32: the fp32 sums over all tokens of a
# step (dγ of RMSNorm, the wgrad reductions) cancel to ~1e-3 of their terms' scale and leave up to ~1e-4 of max|g|
# (measured 1.6e-4 on layers.0.mlp_norm at C0); bf16: one bf16 rounding of every activation / weight on the path.
# Both bars sit far below what a structural error produces: a dropped or doubled group / micro-batch contribution
# moves Δ by ≥ 1/(number of contributions) ≥ 1/16 here, a 2× scale error by 1.
TOL_DELTA = {0: 1e-3, 1: 5e-2}


def oracle_cfg(d, **kw):
    x = dict(d)
    x.update(kw)
    return om.ModelConfig(**x)


def unit_list(cfg: om.ModelConfig):
    """(uid, n) in canonical shard order: layers, E, F."""
    ph = om.phi(cfg)
    return [(l, ph) for l in range(cfg.n_layers)] + [("E", cfg.vocab * cfg.hidden),
                                                     ("F", cfg.hidden + cfg.vocab * cfg.hidden)]


def owner_group(uid, L, D):
    if uid == "E":
        return 0
    if uid == "F":
        return D - 1
    return uid % D


def literal_owner(uid, P: int, D: int) -> int:
    """TAWPIPE_LITERAL owner device (PAPER.md:123 shard map via oracle/routes.py; E on 0, F on P − 1)."""
    from oracle import routes
    if uid == "E":
        return 0
    if uid == "F":
        return P - 1
    return routes.owner_table(P, D)[uid % P]


def reassemble(cfg: om.ModelConfig, P: int, G: int, shards: list, literal: bool = False) -> dict:
    """Rebuild full fp64 params from every rank's tawpipe_shard output (include/tawpipe.h order)."""
    D = P // G
    vecs = {}
    cursors = [0] * P
    pieces = {}
    for rank in range(P):
        k = rank // G
        for uid, n in unit_list(cfg):
            if literal:   # whole units on their owner device
                if literal_owner(uid, P, D) != rank:
                    continue
                s = OL.padded(n, 1)
                pieces[(uid, 0)] = shards[rank][cursors[rank]:cursors[rank] + s]
            else:
                if owner_group(uid, cfg.n_layers, D) != k:
                    continue
                s = OL.padded(n, G) // G
                pieces[(uid, rank % G)] = shards[rank][cursors[rank]:cursors[rank] + s]
            cursors[rank] += s
    for rank in range(P):
        assert cursors[rank] == len(shards[rank]), (rank, cursors[rank], len(shards[rank]))
    for uid, n in unit_list(cfg):
        parts = [pieces[(uid, 0)]] if literal else [pieces[(uid, j)] for j in range(G)]
        vecs[uid] = np.concatenate(parts)[:n].astype(np.float64)
    fn, head = OL.unflatten_F(vecs["F"], cfg)
    return {"embed": vecs["E"].reshape(cfg.vocab, cfg.hidden),
            "layers": [OL.unflatten_layer(vecs[l], cfg) for l in range(cfg.n_layers)],
            "final_norm": fn, "head": head}


def tensors(p: dict):
    out = [("embed", p["embed"]), ("head", p["head"]), ("final_norm", p["final_norm"])]
    for i, lay in enumerate(p["layers"]):
        out += [(f"layers.{i}.{k}", lay[k]) for k in om.LAYER_KEYS]
    return out


def weight_errors(gpu: dict, ref: dict, theta0: dict, g_refs: list, cfg: om.ModelConfig, kappa: float):
    """R18 weight-parity metric, per tensor (reading documented in DESIGN.md "Readings"):
    W = elements whose reference gradient is well conditioned at EVERY step so far,
        {i : |g_t,i| ≥ κ·max|g_t|  for all steps t};
    (i)  e_θ = max_W|θg − θr| / max|θr|;
    (ii) e_Δ = max_W|Δg − Δr| / max_W|Δr| with Δ = θ_final − θ0 (catches wrong updates that (i) hides);
    (iii) off W, |θg − θr| ≤ steps·2·lr·(1 + wd·|θ0|) + tol-free slack 1e-7 (AdamW's first step is
         ≈ −lr·sign(g), so a gradient sign flip on a near-zero entry moves θ by up to 2·lr).
    Returns (worst e_θ, worst e_Δ, off-W violations, share of elements off W, per-tensor report)."""
    steps = len(g_refs)
    worst_t, worst_d, viol, off, total = 0.0, 0.0, 0, 0, 0
    rep = []
    Gs = [dict(tensors(g)) for g in g_refs]
    T0 = dict(tensors(theta0))
    R = dict(tensors(ref))
    for name, tg in tensors(gpu):
        tr, t0 = R[name], T0[name]
        Wm = np.ones(tr.shape, bool)
        for G in Gs:
            gr = G[name]
            Wm &= np.abs(gr) >= kappa * np.max(np.abs(gr))
        err = np.abs(tg - tr)
        et = float(np.max(err[Wm]) / max(np.max(np.abs(tr)), 1e-30)) if Wm.any() else 0.0
        dg, dr = tg - t0, tr - t0
        ed = float(np.max(np.abs(dg - dr)[Wm]) / max(np.max(np.abs(dr)[Wm]), 1e-30)) if Wm.any() else 0.0
        bound = steps * 2 * cfg.lr * (1 + cfg.weight_decay * np.abs(t0)) + 1e-7
        viol += int(np.sum(err[~Wm] > bound[~Wm]))
        off += int(np.sum(~Wm))
        total += Wm.size
        worst_t, worst_d = max(worst_t, et), max(worst_d, ed)
        rep.append((name, et, ed))
    return worst_t, worst_d, viol, off / max(total, 1), rep
