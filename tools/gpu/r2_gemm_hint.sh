# L2 eviction hints of the CTA-pair GEMM at the QKV shape: DRAM bytes and time per mode (ncu, one launch each),
# then plain CUDA-event timing of the C3 GEMM shapes per mode
cd $GRAFT_REPO_ROOT
python tools/gemm_one.py 32768 12288 4096 1 1 > /dev/null 2>&1
for h in 0 1 2; do
  for shape in "32768 12288 4096 1 1" "32768 4096 11008 1 1" "32768 22016 4096 1 1"; do
    TAWPIPE_GEMM_L2HINT=$h ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_tc2 -s 1 -c 1 --csv python tools/gemm_one.py $shape 2>/dev/null | grep -E "dram|duration|tensor" | awk -F'","' -v h=$h -v s="$shape" '{print "hint " h " [" s "]: " $(NF-2) " " $(NF-1) " " $NF}'
  done
done
for h in 0 1 2; do echo "== hint $h"; TAWPIPE_GEMM_L2HINT=$h python tools/gemm_big.py; done
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k gemm 2>&1 | tail -2
