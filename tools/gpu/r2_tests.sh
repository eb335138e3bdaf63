set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m "gpu and not multigpu" -x -q -p no:cacheprovider --durations=15 > gpurun_out/r2_pytest_gpu.txt 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/r2_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.txt 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/r2_smoke.txt
