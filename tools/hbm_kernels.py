"""HBM-bound kernels of the C3 step at their bench shapes, through the kernel-level C ABI, timed with CUDA events
(median of 20 after warm-up) and reported as achieved GB/s of ALGORITHMIC bytes against MEASURED_PEAKS.json.

    python tools/hbm_kernels.py            # plain timing (JSON lines)
    ncu --set full -k regex:"adamw|rmsnorm|ce_kernel|embed_segment" python tools/hbm_kernels.py --once

Algorithmic bytes: RMSNorm fwd 2·H·2 + γ (read x, write y; bf16) per row + 4 (rstd);
RMSNorm bwd dx: dy, x, res read + dx written = 4·H·2 per row; dγ column pass: dy, x read = 2·H·2 per row;
CE: one read + one write of the V bf16 logits per row (+ target, loss); embedding backward: dh read once, each
touched dE row read + written once in fp32; AdamW: the sources + master/m/v read (12 B) + written (12 B) + the bf16
wire copy (2 B) per element."""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_09741_b200 import tawpipe as T  # noqa: E402

ONCE = "--once" in sys.argv
T.lib()
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
PEAK = peaks["hbm_gbs"]


def timed(fn, n=20):
    if ONCE:
        fn()
        torch.cuda.synchronize()
        return float("nan")
    for _ in range(3):
        fn()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def report(name, ms, nbytes, **kw):
    gbs = nbytes / (ms * 1e-3) / 1e9 if ms == ms else float("nan")
    print(json.dumps({"kernel": name, "ms": ms, "algorithmic_bytes": nbytes, "achieved_gbs": gbs,
                      "peak_gbs": PEAK, "frac": gbs / PEAK, **kw}), flush=True)


BF = T.BF16
rows, H, I, V = 32768, 4096, 11008, 32000
x = torch.randn(rows, H, device="cuda").bfloat16()
y = torch.empty_like(x)
g = torch.ones(H, device="cuda").bfloat16()
rstd = torch.empty(rows, device="cuda")
T.rmsnorm_fwd(BF, rows, H, x.data_ptr(), g.data_ptr(), 1e-5, y.data_ptr(), rstd.data_ptr())
ms = timed(lambda: T.rmsnorm_fwd(BF, rows, H, x.data_ptr(), g.data_ptr(), 1e-5, y.data_ptr(), rstd.data_ptr()))
report("rmsnorm_fwd_row<256,2> (H=4096, 32768 rows)", ms, rows * (2 * H * 2 + 4) + H * 2)
dy = torch.randn(rows, H, device="cuda").bfloat16()
res = torch.randn(rows, H, device="cuda").bfloat16()
dx = torch.empty_like(x)
dg = torch.zeros(H, device="cuda")
ms = timed(lambda: T.rmsnorm_bwd(BF, rows, H, dy.data_ptr(), x.data_ptr(), g.data_ptr(), rstd.data_ptr(),
                                 res.data_ptr(), dx.data_ptr(), dg.data_ptr()))
report("rmsnorm_bwd (dx row kernel + dγ column kernel, H=4096, 32768 rows)", ms,
       rows * (4 * H * 2 + 4) + rows * (2 * H * 2 + 4) + H * 4 * 2)
del dy, res, dx
# cross-entropy at one 8192-row head chunk, V = 32000
tc = 8192
z = torch.randn(tc, V, device="cuda").bfloat16()
tg = torch.randint(0, V, (tc,), device="cuda", dtype=torch.int32)
lr = torch.empty(tc, device="cuda")
ms = timed(lambda: T.cross_entropy(BF, tc, V, z.data_ptr(), tg.data_ptr(), 1.0 / 32768, lr.data_ptr()))
report("ce_v8_kernel (single pass, 8192 rows, V=32000)", ms, tc * (2 * V * 2 + 4 + 4))
del z
# embedding backward at C3 (32768 positions, H = 4096, V = 32000)
tok = torch.randint(0, V, (1, rows + 1), device="cuda", dtype=torch.int32)
dE = torch.zeros(V, H, device="cuda")
ms = timed(lambda: T.embed_bwd(BF, 1, rows, tok.data_ptr(), rows + 1, x.data_ptr(), H, V, dE.data_ptr()))
nd = int(torch.unique(tok[0, :rows]).numel())   # distinct tokens: rows of dE read + written once each (fp32)
report("embed_bwd (sort + segments, 32768 positions, H=4096)", ms, rows * H * 2 + nd * H * 4 * 2, distinct_tokens=nd)
del dE, x, y
# fused accumulate + AdamW on a C3 decoder-layer stripe: P=1 (one fp32 source, n = φ) and 4x2 (two fp32 sources
# of n = φ/2 plus three bf16 rail partials)
phi = 4 * H * H + 3 * H * I + 2 * H
for name, n, groups in (("P=1", phi, [[1]]), ("4x2 owner (2 fp32 + 3 bf16 partials)", phi // 2, [[1, 1], [0], [0], [0]])):
    n = n // 64 * 64
    master = torch.randn(n, device="cuda") * 0.02
    m = torch.zeros(n, device="cuda")
    v = torch.zeros(n, device="cuda")
    wire = torch.empty(n, device="cuda", dtype=torch.bfloat16)
    srcs, keep = [], []
    src_bytes = 0
    for gr in groups:
        row = []
        for f32 in gr:
            t = torch.randn(n, device="cuda") * 1e-3
            t = t if f32 else t.bfloat16()
            keep.append(t)
            row.append((t.data_ptr(), bool(f32)))
            src_bytes += 4 if f32 else 2
        srcs.append(row)
    ms = timed(lambda: T.adamw(BF, srcs, master.data_ptr(), m.data_ptr(), v.data_ptr(), wire.data_ptr(), n, 0,
                               (0, H, H + 4 * H * H, 2 * H + 4 * H * H)), n=10)
    report(f"adamw_grouped_v8 ({name}, n={n})", ms, n * (src_bytes + 24 + 2))
    del master, m, v, wire, keep, srcs
    torch.cuda.empty_cache()
