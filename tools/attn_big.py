"""Run the tcgen05 attention fwd+bwd at a large S (no oracle) and time it -- hang / throughput probe."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_2511_09741_b200 import tawpipe as T
T.lib()
S, nh, dh = int(sys.argv[1]), int(sys.argv[2]), 128
H = nh * dh
qkv = (torch.randn(S, 3 * H, device="cuda") * 0.5).bfloat16()
do = torch.randn(S, H, device="cuda").bfloat16()
o = torch.empty(S, H, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(nh, S, device="cuda")
dqkv = torch.empty_like(qkv); delta = torch.empty(2, nh, S, device="cuda"); acc = torch.empty(S, H, device="cuda")
for it in range(3):
    torch.cuda.synchronize(); t0 = time.time()
    T.attention_fwd(T.BF16, 1, S, nh, dh, qkv.data_ptr(), o.data_ptr(), lse.data_ptr())
    torch.cuda.synchronize(); t1 = time.time()
    T.attention_bwd(T.BF16, 1, S, nh, dh, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), do.data_ptr(),
                    dqkv.data_ptr(), delta.data_ptr(), acc.data_ptr())
    torch.cuda.synchronize(); t2 = time.time()
    f = 2 * 2 * H * S * (S + 1) / 2
    print(f"S={S} nh={nh}: fwd {1e3*(t1-t0):.2f} ms ({f/(t1-t0)/1e12:.0f} TF/s)  bwd {1e3*(t2-t1):.2f} ms "
          f"({2.5*f/(t2-t1)/1e12:.0f} TF/s executed)", flush=True)
print("finite:", torch.isfinite(o.float()).all().item(), torch.isfinite(dqkv.float()).all().item())
