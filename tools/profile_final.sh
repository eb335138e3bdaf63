#!/bin/bash
# Round-end evidence pass (run under gpurun, 1 GPU): the default bench line, then the ncu launch list of the
# same command (ncu only after the plain command exited 0).
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_final.log 2>&1 || { echo "bench failed"; tail -5 gpurun_out/bench_final.log; exit 1; }
tail -1 gpurun_out/bench_final.log
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain_bench1.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench_final.log 2>&1
echo "launch-list rc=$?"
