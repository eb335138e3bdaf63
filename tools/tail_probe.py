"""Per-rank exposed-communication breakdown of the C3 step (torchrun, one rank per GPU): each rank prints its
exposed time per step and, from its Trace-Event export of the last step, the largest compute-stream waits with their
position in the step (the last one is the step tail: joins + loss all-reduce, which waits for the slowest rank)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2511_09741_b200 import tawpipe as T  # noqa: E402

rank, world, local = T.dist_env()
torch.cuda.set_device(local)
T.bootstrap(rank, world, local, pg_backend="gloo")
G = {1: 1, 2: 2, 4: 2, 8: 2}[world]
N = world
dims = T.ModelDims(n_layers=32, hidden=4096, heads=32, ffn=11008, vocab=32000, seq=32768, micro_bs=1, dtype=1, ckpt=1,
                   lr=3e-4)
sess = T.Session(world, G, dims, N)
sess.set_timing(True)
tok = synth.tokens(N, 1, 32768, 32000, step=0)
mine = torch.from_numpy(np.ascontiguousarray(tok[rank:rank + 1])).cuda()
exp = []
for i in range(6):
    sess.step_device(mine.data_ptr())
    exp.append(sess.stats()["exposed_comm_ms"])
tr = sess.trace()
cs = sorted([e for e in tr["traceEvents"] if e.get("ph") == "X" and e.get("tid") == 0], key=lambda e: e["ts"])
waits = sorted([(e["dur"] / 1e3, e["ts"] / 1e3) for e in cs if e["name"] == "exposed_comm_wait"], reverse=True)[:6]
step_ms = tr["otherData"]["step_ms"]
print(f"rank {rank}: exposed per step {[round(x, 1) for x in exp]} ms; step {step_ms:.1f} ms; largest waits "
      f"{[(round(d, 2), round(t, 1)) for d, t in waits]}", flush=True)
sess.close()
