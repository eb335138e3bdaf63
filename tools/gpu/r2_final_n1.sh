cd $GRAFT_REPO_ROOT
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_c3_n1_final.json 2> gpurun_out/r2_bench_c3_n1_final.err; echo "bench rc=$?"
head -c 1200 gpurun_out/r2_bench_c3_n1_final.json; echo
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 1100 --csv --log-file gpurun_out/r2_ncu_launches_c3_n1.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r2_ncu_launches.log 2>&1; echo "ncu launches rc=$?"
wc -l gpurun_out/r2_ncu_launches_c3_n1.csv
