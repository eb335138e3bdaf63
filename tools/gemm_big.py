"""Time the tcgen05 GEMM at C3 shapes (forward / dgrad / wgrad majors)."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2511_09741_b200 import tawpipe as T
T.lib()
cases = [("fwd qkv", 32768, 12288, 4096, True, True), ("fwd down", 32768, 4096, 11008, True, True),
         ("dgrad gu", 32768, 4096, 22016, True, False), ("wgrad gu", 22016, 4096, 32768, False, False),
         ("fwd 8k^3", 8192, 8192, 8192, True, True)]
for name, M, N, K, ak, bk in cases:
    A = torch.randn((M, K) if ak else (K, M), device="cuda").bfloat16()
    B = torch.randn((N, K) if bk else (K, N), device="cuda").bfloat16()
    f32 = not (ak and bk) and not ak
    C = torch.empty((M, N), device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
    for it in range(4):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        T.gemm(T.BF16, M, N, K, A.data_ptr(), K if ak else M, ak, B.data_ptr(), K if bk else N, bk, C.data_ptr(), N,
               c_f32=f32, accumulate=f32)
        e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{name:10s} {M}x{N}x{K}: {ms:.3f} ms  {2*M*N*K/ms/1e9:.0f} TF/s", flush=True)
