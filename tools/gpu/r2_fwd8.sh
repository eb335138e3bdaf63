# CTA-pair attention forward (fa_fwd8): hang probe, parity, then sustained timing against fa_fwd7
cd $GRAFT_REPO_ROOT
TAWPIPE_FA_FWD=8 timeout 120 python tools/attn_big.py 2048 4; echo "probe rc=$?"
TAWPIPE_FA_FWD=8 timeout 120 python tools/attn_big.py 32768 32; echo "probe32k rc=$?"
TAWPIPE_FA_FWD=8 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_ops.py -q -x -k "attention" 2>&1 | tail -3
for v in 7 8 7 8; do echo "fwd v$v"; TAWPIPE_FA_FWD=$v timeout 300 python tools/attn_clock.py 2>&1 | tail -1; done
