# full GPU suites after the store-first gradient accumulation: 1-GPU parity, then the 4-GPU parity suite
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m "gpu and not multigpu" -q -p no:cacheprovider > gpurun_out/r2_pytest_gpu_1gpu_final.txt 2>&1; echo "1gpu rc=$?"
tail -1 gpurun_out/r2_pytest_gpu_1gpu_final.txt
timeout 2400 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -rA > gpurun_out/r2_pytest_multigpu_final.txt 2>&1
echo "multigpu rc=$?"; grep -E "passed|failed" gpurun_out/r2_pytest_multigpu_final.txt | tail -3
