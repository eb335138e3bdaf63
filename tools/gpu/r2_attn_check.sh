# HISTORICAL: the experiment switch this script sets (TAWPIPE_FA_EMU / _DBG / _BWD) was removed with the variant
# after the measurement (DESIGN.md §5 records the result); kept for provenance of the numbers quoted there.
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "attention" -x > gpurun_out/r2_attn_tests.txt 2>&1; echo "attn tests rc=$?"; tail -3 gpurun_out/r2_attn_tests.txt
echo "v8:"; python tools/attn_big.py 32768 32 2>&1 | tail -3
echo "v5:"; TAWPIPE_FA_BWD=5 python tools/attn_big.py 32768 32 2>&1 | tail -3
TAWPIPE_FA_TRACE=1 python tools/attn_big.py 4096 2 > gpurun_out/r2_attn_trace8.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_step.py -q -p no:cacheprovider -x -k "c0b" > gpurun_out/r2_step_tests.txt 2>&1; echo "step tests rc=$?"; tail -3 gpurun_out/r2_step_tests.txt
