# DRAM traffic of the CTA-pair GEMM at the C3 QKV shape (L2-aware raster vs the round-1 M-band order) and the
# single-pass cross-entropy; one ncu --set full capture each
cd $GRAFT_REPO_ROOT
python tools/gemm_one.py 32768 12288 4096 1 1 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:gemm_tc2 -s 1 -c 1 -o gpurun_out/r2_gemm_qkv python tools/gemm_one.py 32768 12288 4096 1 1 > gpurun_out/r2_ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
TAWPIPE_GEMM_RASTER=default ncu --set full --clock-control none -k regex:gemm_tc2 -s 1 -c 1 -o gpurun_out/r2_gemm_qkv_oldraster python tools/gemm_one.py 32768 12288 4096 1 1 > gpurun_out/r2_ncu_gemm_old.log 2>&1; echo "ncu gemm old rc=$?"
ncu --set full --clock-control none -k regex:gemm_tc2 -s 1 -c 1 -o gpurun_out/r2_gemm_down python tools/gemm_one.py 32768 4096 11008 1 1 > gpurun_out/r2_ncu_gemm_down.log 2>&1; echo "ncu gemm down rc=$?"
python tools/hbm_kernels.py 2>&1 | grep ce_kernel
ncu --set full --clock-control none -k regex:ce_v8 -c 1 -o gpurun_out/r2_ce python tools/hbm_kernels.py --once > gpurun_out/r2_ncu_ce.log 2>&1; echo "ncu ce rc=$?"
