cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -rA -k "L8 or L4 or g2x" > gpurun_out/r2_pytest_multigpu_dbg.txt 2>&1
echo "rc=$?"; grep -E "PASSED|FAILED|passed|failed|e_theta" gpurun_out/r2_pytest_multigpu_dbg.txt | tail -30
