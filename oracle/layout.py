"""Canonical flattened parameter layout and DBS striping, as the oracle reads them.

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.

SURVEY.md §8(a) a1 and §8(c) R6 (striped group ownership):
  * one decoder layer flattens to
    [attn_norm H | Wq H·H | Wk H·H | Wv H·H | Wo H·H | mlp_norm H | Wgate I·H | Wup I·H | Wdown H·I]
    (each matrix row-major [out, in]), length φ = 4H² + 3HI + 2H;
  * the embedding pseudo-layer E is [V·H], the head pseudo-layer F is [γ_f H | W_head V·H] (R9);
  * a unit of length n is zero-padded to n_pad = G·64·ceil(n / (G·64)) and split
    into G contiguous stripes of s = n_pad / G elements; stripe j lives on device
    (owner_group·G + j);
  * the full-model canonical vector (tawpipe_load input) is [E | layer 0 .. layer L−1 | F],
    unpadded.
"""
from __future__ import annotations

import numpy as np

from .model import LAYER_KEYS, ModelConfig, layer_shapes

PAD_QUANTUM = 64


def padded(n: int, G: int) -> int:
    q = G * PAD_QUANTUM
    return q * ((n + q - 1) // q)


def flatten_layer(lay: dict, cfg: ModelConfig) -> np.ndarray:
    return np.concatenate([np.asarray(lay[k]).reshape(-1) for k in LAYER_KEYS])


def unflatten_layer(vec: np.ndarray, cfg: ModelConfig) -> dict:
    out, off = {}, 0
    for k, shp in layer_shapes(cfg).items():
        n = int(np.prod(shp))
        out[k] = vec[off:off + n].reshape(shp)
        off += n
    return out


def flatten_F(final_norm, head) -> np.ndarray:
    return np.concatenate([np.asarray(final_norm).reshape(-1), np.asarray(head).reshape(-1)])


def unflatten_F(vec, cfg: ModelConfig):
    H, V = cfg.hidden, cfg.vocab
    return vec[:H].copy(), vec[H:H + V * H].reshape(V, H)


def flatten_model(params: dict, cfg: ModelConfig) -> np.ndarray:
    parts = [np.asarray(params["embed"]).reshape(-1)]
    parts += [flatten_layer(lay, cfg) for lay in params["layers"]]
    parts.append(flatten_F(params["final_norm"], params["head"]))
    return np.concatenate(parts)


def unflatten_model(vec: np.ndarray, cfg: ModelConfig) -> dict:
    H, V, L = cfg.hidden, cfg.vocab, cfg.n_layers
    from .model import phi
    ph = phi(cfg)
    off = 0
    embed = vec[off:off + V * H].reshape(V, H)
    off += V * H
    layers = []
    for _ in range(L):
        layers.append(unflatten_layer(vec[off:off + ph], cfg))
        off += ph
    fn, head = unflatten_F(vec[off:off + H + V * H], cfg)
    off += H + V * H
    assert off == vec.size
    return {"embed": embed, "layers": layers, "final_norm": fn, "head": head}


def no_decay_mask_layer(cfg: ModelConfig) -> np.ndarray:
    """True where AdamW weight decay is NOT applied (the two RMSNorm gains, R1)."""
    m, off = [], 0
    for k, shp in layer_shapes(cfg).items():
        n = int(np.prod(shp))
        m.append(np.full(n, k in ("attn_norm", "mlp_norm")))
        off += n
    return np.concatenate(m)


def no_decay_mask_F(cfg: ModelConfig) -> np.ndarray:
    return np.concatenate([np.ones(cfg.hidden, bool), np.zeros(cfg.vocab * cfg.hidden, bool)])
