#!/bin/bash
# full ncu capture (with source) of one attention backward launch at the C3 shape
python tools/attn_big.py 32768 32 > gpurun_out/plain_attn.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fa_bwd_kernel" -s 1 -c 1 -o gpurun_out/prof_bwd5 \
    python tools/attn_big.py 32768 32 > gpurun_out/ncu_bwd5.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_bwd5.log
