cd $GRAFT_REPO_ROOT
bash tools/gpu/r2_p2p_debug.sh 2>&1 | tail -25
timeout 2400 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -rA > gpurun_out/r2_pytest_multigpu.txt 2>&1
echo "multigpu pytest rc=$?"
grep -E "PASSED|FAILED|passed|failed" gpurun_out/r2_pytest_multigpu.txt | tail -40
