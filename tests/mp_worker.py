"""One rank of a multi-GPU parity run (launched by tests/test_multigpu.py through torchrun).
Writes this rank's losses, ledger and owned fp32 shard to <out>/rank<r>.npz."""
import argparse
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402

import synth  # noqa: E402
from helpers import oracle_cfg  # noqa: E402
from paper_2511_09741_b200 import tawpipe as T  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", required=True)       # json dict of model dims
    ap.add_argument("--G", type=int, required=True)
    ap.add_argument("--N", type=int, required=True)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--dtype", type=int, default=0)
    ap.add_argument("--ckpt", type=int, default=0)
    ap.add_argument("--no-cco", action="store_true")
    ap.add_argument("--ring", action="store_true")
    ap.add_argument("--literal", action="store_true")
    ap.add_argument("--emu-gbps", type=float, default=0.0)   # NEXT-3 emulated inter-node link
    ap.add_argument("--emu-node", type=int, default=0)
    ap.add_argument("--linear", action="store_true", help="AdamW ε = 1, lr = 1, no decay: update linear in g (R18)")
    ap.add_argument("--init-only", action="store_true", help="no tawpipe_load, no step: save the device-side init")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    hyper = dict(lr=1.0, adam_eps=1.0, weight_decay=0.0) if a.linear else {}
    cfg = oracle_cfg(json.loads(a.cfg), **hyper)
    rank, world, local = T.bootstrap()
    params = synth.perturb_gains(synth.init_params(cfg.n_layers, cfg.hidden, cfg.ffn, cfg.vocab))
    dims = T.ModelDims(n_layers=cfg.n_layers, hidden=cfg.hidden, heads=cfg.heads, ffn=cfg.ffn, vocab=cfg.vocab,
                       seq=cfg.seq, micro_bs=cfg.micro_bs, dtype=a.dtype, ckpt=a.ckpt,
                       schedule=(T.NO_CCO if a.no_cco else T.GWPS) | (T.RING if a.ring else 0)
                       | (T.LITERAL if a.literal else 0), **hyper)
    sess = T.Session(world, a.G, dims, a.N)
    if a.init_only:   # R20: the seeded device-side initialisation, keyed by canonical position
        np.savez(os.path.join(a.out, f"rank{rank}.npz"), shard=sess.shard())
        sess.close()
        return
    sess.load(T.pack_full_model(params))
    if a.emu_gbps > 0:
        sess.set_link_emulation(a.emu_gbps, 30.0, a.emu_node)
    sess.set_timing(True)
    losses, ledgers, comm_ms = [], [], []
    for step in range(a.steps):
        toks = synth.tokens(a.N, cfg.micro_bs, cfg.seq, cfg.vocab, step=step)
        losses.append(sess.step(toks))
        ledgers.append(sess.ledger())
        stt = sess.stats()
        comm_ms.append(stt["weight_comm_ms"] + stt["grad_comm_ms"])
    np.savez(os.path.join(a.out, f"rank{rank}.npz"), losses=np.array(losses), ledgers=np.array(ledgers, np.uint64),
             shard=sess.shard(), comm_ms=np.array(comm_ms), p2p=np.array(stt["p2p"]))
    sess.close()


if __name__ == "__main__":
    main()
