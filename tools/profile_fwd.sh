#!/bin/bash
python tools/attn_big.py 8192 32 > gpurun_out/plain_attn.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fa_fwd3_kernel" -s 1 -c 1 -o gpurun_out/prof_fwd3 \
    python tools/attn_big.py 8192 32 > gpurun_out/ncu_fwd3.log 2>&1
echo "rc=$?"
