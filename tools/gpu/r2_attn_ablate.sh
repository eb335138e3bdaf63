# HISTORICAL: the experiment switch this script sets (TAWPIPE_FA_EMU / _DBG / _BWD) was removed with the variant
# after the measurement (DESIGN.md §5 records the result); kept for provenance of the numbers quoted there.
cd $GRAFT_REPO_ROOT
for d in 0 16 0 16; do echo "dbg=$d: $(TAWPIPE_FA_DBG=$d python tools/attn_clock.py 2>&1 | tail -1 | cut -c1-90)"; done
TAWPIPE_FA_DBG=16 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "attention" -x 2>&1 | tail -1
