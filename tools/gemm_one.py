"""Run one tcgen05 GEMM shape a few times (for ncu captures): gemm_one.py M N K a_kmajor b_kmajor."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2511_09741_b200 import tawpipe as T
M, N, K, ak, bk = (int(x) for x in sys.argv[1:6])
T.lib()
A = torch.randn((M, K) if ak else (K, M), device="cuda").bfloat16()
B = torch.randn((N, K) if bk else (K, N), device="cuda").bfloat16()
f32 = not ak
C = torch.zeros((M, N), device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
for it in range(3):
    T.gemm(T.BF16, M, N, K, A.data_ptr(), K if ak else M, bool(ak), B.data_ptr(), K if bk else N, bool(bk), C.data_ptr(), N,
           c_f32=f32, accumulate=f32)
torch.cuda.synchronize()
print("ok")
