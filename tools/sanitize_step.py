"""One C0 fp32 step and one C0b bf16 step (P = 1) through the C ABI, for compute-sanitizer (memcheck / racecheck /
synccheck): python tools/sanitize_step.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2511_09741_b200 import tawpipe as T  # noqa: E402

T.bootstrap(0, 1, 0)
for name, dims, n_micro in (
        ("c0-fp32", T.ModelDims(n_layers=2, hidden=64, heads=4, ffn=192, vocab=256, seq=128, dtype=T.FP32, ckpt=1), 2),
        ("c0b-bf16", T.ModelDims(n_layers=2, hidden=256, heads=2, ffn=768, vocab=512, seq=256, dtype=T.BF16, ckpt=2), 2)):
    sess = T.Session(1, 1, dims, n_micro)
    loss = sess.step(synth.tokens(n_micro, 1, dims.seq, dims.vocab))
    print(f"{name}: loss {loss:.6f}", flush=True)
    sess.close()
    T.bootstrap(0, 1, 0)
