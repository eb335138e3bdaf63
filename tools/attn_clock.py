"""Sustained attention fwd+bwd at the C3 shape with clock sampling: is the in-step slowdown a clock effect?"""
import sys, time, statistics
import torch
sys.path.insert(0, ".")
from paper_2511_09741_b200 import tawpipe as T
from bench import ClockSampler
T.lib()
S, nh, dh = 32768, 32, 128
H = nh * dh
qkv = (torch.randn(S, 3 * H, device="cuda") * 0.5).bfloat16()
do = torch.randn(S, H, device="cuda").bfloat16()
o = torch.empty(S, H, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(nh, S, device="cuda")
dqkv = torch.empty_like(qkv); delta = torch.empty(2, nh, S, device="cuda"); acc = torch.empty(S, H, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
fw, bw = [], []
with ClockSampler(0) as clk:
    t_end = time.time() + 8
    while time.time() < t_end:
        ev[0].record()
        T.attention_fwd(T.BF16, 1, S, nh, dh, qkv.data_ptr(), o.data_ptr(), lse.data_ptr())
        ev[1].record()
        T.attention_bwd(T.BF16, 1, S, nh, dh, qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), do.data_ptr(),
                        dqkv.data_ptr(), delta.data_ptr(), acc.data_ptr())
        ev[2].record()
        torch.cuda.synchronize()
        fw.append(ev[0].elapsed_time(ev[1])); bw.append(ev[1].elapsed_time(ev[2]))
print(f"sustained: fwd {statistics.median(fw):.2f} ms  bwd {statistics.median(bw):.2f} ms  n={len(fw)}  clocks {clk.summary()}")
