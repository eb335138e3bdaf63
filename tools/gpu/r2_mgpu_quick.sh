cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -rA -k "4x1 or emu or c0-2x2 or L8" > gpurun_out/r2_pytest_multigpu_quick.txt 2>&1
echo "rc=$?"; grep -E "PASSED|FAILED|passed|failed|e_theta|Error" gpurun_out/r2_pytest_multigpu_quick.txt | tail -30
