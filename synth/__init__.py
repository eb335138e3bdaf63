"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no normalisation, attention,
loss, optimizer, layout, sharding or scheduling).  It only draws random numbers,
so that the oracle (``oracle/``) and the GPU path (``paper_2511_09741_b200``)
can be fed identical inputs without sharing any code.

Recipe (SURVEY.md §8(d) "Synthetic inputs"):
  * tokens: int32 [N][B][S+1], uniform on [0, V), ``numpy.random.default_rng(seed + step)``
    (seed 42 by default) -- packed full-length sequences, no padding, like the
    paper's C4 workload.  ``dist="zipf"`` draws Zipf(1.1)
    ranks mod V instead, to mimic text token frequencies.
  * weights: ``default_rng(1234)``; N(0, 0.02) for every matrix, the embedding
    and the LM head; 1.0 for the RMSNorm gains.
"""
from __future__ import annotations

import numpy as np

MATRIX_STD = 0.02


def tokens(n_micro: int, micro_bs: int, seq: int, vocab: int, step: int = 0,
           seed: int = 42, dist: str = "uniform") -> np.ndarray:
    """int32 [n_micro][micro_bs][seq+1] token ids in [0, vocab)."""
    rng = np.random.default_rng(seed + step)
    shape = (n_micro, micro_bs, seq + 1)
    if dist == "uniform":
        t = rng.integers(0, vocab, size=shape, dtype=np.int64)
    elif dist == "zipf":
        t = (rng.zipf(1.1, size=shape) - 1) % vocab
    else:
        raise ValueError(f"unknown token distribution {dist!r}")
    return np.ascontiguousarray(t.astype(np.int32))


def init_params(n_layers: int, hidden: int, ffn: int, vocab: int,
                seed: int = 1234) -> dict:
    """Random-init parameters of a LLaMA-style decoder, float32.

    Returns {"embed": [V,H], "layers": [dict per layer], "final_norm": [H],
    "head": [V,H]}; each layer dict has attn_norm [H], wq/wk/wv/wo [H,H],
    mlp_norm [H], w_gate/w_up [I,H], w_down [H,I] (row-major [out, in]).
    Draw order is fixed: embed, then per layer wq wk wv wo w_gate w_up w_down,
    then head.
    """
    rng = np.random.default_rng(seed)
    H, I, V = hidden, ffn, vocab

    def mat(r, c):
        return (rng.standard_normal((r, c)) * MATRIX_STD).astype(np.float32)

    embed = mat(V, H)
    layers = []
    for _ in range(n_layers):
        lay = {"attn_norm": np.ones(H, np.float32)}
        lay["wq"] = mat(H, H)
        lay["wk"] = mat(H, H)
        lay["wv"] = mat(H, H)
        lay["wo"] = mat(H, H)
        lay["mlp_norm"] = np.ones(H, np.float32)
        lay["w_gate"] = mat(I, H)
        lay["w_up"] = mat(I, H)
        lay["w_down"] = mat(H, I)
        layers.append(lay)
    head = mat(V, H)
    return {"embed": embed, "layers": layers,
            "final_norm": np.ones(H, np.float32), "head": head}


def perturb_gains(params: dict, seed: int = 99, scale: float = 0.1) -> dict:
    """Return a copy whose RMSNorm gains are 1 + U(-scale, scale) (so tests see non-trivial gains)."""
    rng = np.random.default_rng(seed)
    out = {"embed": params["embed"].copy(), "head": params["head"].copy(),
           "final_norm": (1.0 + rng.uniform(-scale, scale, params["final_norm"].shape)).astype(np.float32),
           "layers": []}
    for lay in params["layers"]:
        nl = {k: v.copy() for k, v in lay.items()}
        nl["attn_norm"] = (1.0 + rng.uniform(-scale, scale, nl["attn_norm"].shape)).astype(np.float32)
        nl["mlp_norm"] = (1.0 + rng.uniform(-scale, scale, nl["mlp_norm"].shape)).astype(np.float32)
        out["layers"].append(nl)
    return out
