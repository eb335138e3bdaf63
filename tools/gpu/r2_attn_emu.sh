# HISTORICAL: the experiment switch this script sets (TAWPIPE_FA_EMU / _DBG / _BWD) was removed with the variant
# after the measurement (DESIGN.md §5 records the result); kept for provenance of the numbers quoted there.
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "attention" -x > gpurun_out/r2_attn_tests.txt 2>&1; echo "attn tests rc=$?"; tail -2 gpurun_out/r2_attn_tests.txt
for rep in 1 2; do
echo "emu1:"; TAWPIPE_FA_EMU=1 python tools/attn_clock.py 2>&1 | tail -1
echo "emu0:"; TAWPIPE_FA_EMU=0 python tools/attn_clock.py 2>&1 | tail -1
done
