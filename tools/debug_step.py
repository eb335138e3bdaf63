"""Diagnostics: GPU loss vs oracle loss for ablated parameter sets (isolates which op disagrees)."""
import copy
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np

import synth
from helpers import C0, C0B, om, oracle_cfg
from paper_2511_09741_b200 import tawpipe as T


def run(base, dtype, mod, name, n_micro=4, ckpt=0):
    cfg = oracle_cfg(base)
    params = synth.perturb_gains(synth.init_params(cfg.n_layers, cfg.hidden, cfg.ffn, cfg.vocab))
    params = mod(copy.deepcopy(params))
    T.bootstrap(0, 1, 0)
    dims = T.ModelDims(n_layers=cfg.n_layers, hidden=cfg.hidden, heads=cfg.heads, ffn=cfg.ffn, vocab=cfg.vocab,
                       seq=cfg.seq, micro_bs=cfg.micro_bs, dtype=dtype, ckpt=ckpt)
    s = T.Session(1, 1, dims, n_micro)
    s.load(T.pack_full_model(params))
    toks = synth.tokens(n_micro, cfg.micro_bs, cfg.seq, cfg.vocab, step=0)
    lg = s.step(toks)
    lr, _ = om.loss_and_grads(params, toks, cfg)
    print(f"{name:30s} gpu {lg:.7f} oracle {lr:.7f} rel {abs(lg-lr)/lr:.2e}", flush=True)
    s.close()


def zero(keys):
    def f(p):
        for lay in p["layers"]:
            for k in keys:
                lay[k][:] = 0
        return p
    return f


ident = lambda p: p
for base, dt, nm in [(C0, T.FP32, "C0 fp32"), (C0B, T.BF16, "C0b bf16")]:
    run(base, dt, ident, nm + " full")
    run(base, dt, zero(["wo", "w_down"]), nm + " layers=identity")
    run(base, dt, zero(["wo"]), nm + " attn off")
    run(base, dt, zero(["w_down"]), nm + " mlp off")
    run(base, dt, zero(["wq", "wk"]), nm + " q=k=0 (uniform attn)")
    run(base, dt, lambda p: (p.update(head=p["head"] * 0), p)[1], nm + " head=0")
