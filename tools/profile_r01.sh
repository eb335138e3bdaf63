#!/bin/bash
# Round-1 profiling pass (run under gpurun): launch list of the C3 bench + full captures of the top kernels.
mkdir -p gpurun_out
python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv \
    python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
echo "launch-list rc=$?"
python tools/attn_big.py 32768 32 > gpurun_out/plain_attn.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fa_(bwd|fwd3)_kernel" -s 2 -c 2 -o gpurun_out/prof_attn \
    python tools/attn_big.py 32768 32 > gpurun_out/ncu_attn.log 2>&1
echo "attn rc=$?"
python tools/gemm_big.py > gpurun_out/plain_gemm.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 3 -o gpurun_out/prof_gemm \
    python tools/gemm_big.py > gpurun_out/ncu_gemm.log 2>&1
echo "gemm rc=$?"
python bench.py --config c1 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/plain_c1.log 2>&1 && \
ncu --set full --clock-control none -k regex:"adamw|rmsnorm_(fwd|bwd)_v8|swiglu_(fwd|bwd)_v8|rope_v8|ce_kernel" -s 40 -c 8 \
    -o gpurun_out/prof_hbm python bench.py --config c1 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_hbm.log 2>&1
echo "hbm rc=$?"
