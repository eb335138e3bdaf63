cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m "gpu and not multigpu" -q -p no:cacheprovider -rf --durations=8 > gpurun_out/r2_pytest_gpu.txt 2>&1
echo "pytest rc=$?"; tail -14 gpurun_out/r2_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_n1b.json 2> gpurun_out/r2_bench_n1b.err; echo "bench rc=$?"; head -c 700 gpurun_out/r2_bench_n1b.json
