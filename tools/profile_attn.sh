#!/bin/bash
# full ncu capture (with source) of one attention forward (v7) and one backward launch at the C3 shape
python tools/attn_big.py 32768 32 > gpurun_out/plain_attn.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fa_(bwd|fwd7)_kernel" -s 2 -c 2 -o gpurun_out/prof_attn5 \
    python tools/attn_big.py 32768 32 > gpurun_out/ncu_attn5.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_attn5.log
