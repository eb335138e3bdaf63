# DRAM bytes / time / tensor activity of the CTA-pair GEMM at the QKV and down-projection shapes, L2 hints off / on
cd $GRAFT_REPO_ROOT
python tools/gemm_one.py 32768 12288 4096 1 1 > /dev/null 2>&1
for h in 0 1; do
  for shape in "32768 12288 4096 1 1" "32768 4096 11008 1 1"; do
    TAWPIPE_GEMM_L2HINT=$h ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_tc2 -s 1 -c 1 --csv python tools/gemm_one.py $shape 2>/dev/null | grep -E "dram|duration|tensor" | awk -F'","' -v h=$h -v s="$shape" '{print "l2hint " h " [" s "]: " $(NF-2) " " $(NF-1) " " $NF}'
  done
done > gpurun_out/r2_gemm_l2hint.txt
cat gpurun_out/r2_gemm_l2hint.txt
