cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -rA -k "c0-2x2 or 1x4 or 4x1 or g2x or fsdp or 2x1" > gpurun_out/r2_pytest_multigpu_check.txt 2>&1
echo "rc=$?"; grep -E "passed|failed" gpurun_out/r2_pytest_multigpu_check.txt | tail -3; grep -m3 -E "EINVARIANT|peer flag" gpurun_out/r2_pytest_multigpu_check.txt
bash tools/gpu/r2_bench_mgpu.sh
