cd $GRAFT_REPO_ROOT
# one-step launch list: --steps 2 --warmup 0 runs 2 timed + 2 e2e steps; window 2 (between the first two loss
# reductions) is one whole step's launches
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 2600 --csv --log-file gpurun_out/r2_ncu_launches_c3_n1_final.csv python bench.py --steps 2 --warmup 0 --no-cpu-baseline > gpurun_out/r2_ncu_launches_final.log 2>&1; echo "ncu launches rc=$?"
python tools/launch_shares.py gpurun_out/r2_ncu_launches_c3_n1_final.csv --step 2 | head -30
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_c3_n1_last.json 2> gpurun_out/r2_bench_c3_n1_last.err; echo "bench rc=$?"
python tools/bench_summary.py gpurun_out/r2_bench_c3_n1_last.json 2>/dev/null || head -c 600 gpurun_out/r2_bench_c3_n1_last.json
