# attention backward at the C3 shape: timing, in-kernel timeline, one full ncu capture (1 GPU)
cd $GRAFT_REPO_ROOT
python tools/attn_big.py 32768 32 > gpurun_out/r2_attn_big.txt 2>&1; echo "attn_big rc=$?"; cat gpurun_out/r2_attn_big.txt
TAWPIPE_FA_TRACE=1 python tools/attn_big.py 4096 2 > gpurun_out/r2_attn_trace.txt 2>&1; echo "trace rc=$?"
python tools/hbm_kernels.py > gpurun_out/r2_hbm_kernels.txt 2>&1; echo "hbm rc=$?"; cat gpurun_out/r2_hbm_kernels.txt
ncu --set full --clock-control none --import-source on -k regex:"fa_bwd_kernel|fa_fwd7_kernel" -c 2 \
    -o gpurun_out/r2_attn python tools/attn_big.py 32768 32 > gpurun_out/r2_ncu_attn.log 2>&1
echo "ncu attn rc=$?"; tail -3 gpurun_out/r2_ncu_attn.log
ncu --set full --clock-control none -k regex:"adamw|rmsnorm|ce_kernel|embed_segment" -c 8 \
    -o gpurun_out/r2_hbm python tools/hbm_kernels.py --once > gpurun_out/r2_ncu_hbm.log 2>&1
echo "ncu hbm rc=$?"; tail -3 gpurun_out/r2_ncu_hbm.log
