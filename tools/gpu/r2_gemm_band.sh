cd $GRAFT_REPO_ROOT
python tools/gemm_one.py 32768 12288 4096 1 1 > /dev/null 2>&1
for mb in 8 16 24 32; do
  TAWPIPE_GEMM_BAND_MB=$mb ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_tc2 -s 1 -c 1 --csv python tools/gemm_one.py 32768 12288 4096 1 1 2>/dev/null | grep -E "dram|duration|tensor" | awk -F'","' -v mb=$mb '{print "band " mb " MB: " $(NF-2) " " $(NF-1) " " $NF}'
  TAWPIPE_GEMM_RASTER=m TAWPIPE_GEMM_BAND_MB=$mb ncu --metrics dram__bytes_read.sum --clock-control none -k regex:gemm_tc2 -s 1 -c 1 --csv python tools/gemm_one.py 32768 12288 4096 1 1 2>/dev/null | grep -E "dram" | awk -F'","' -v mb=$mb '{print "M-bands " mb " MB: " $(NF-2) " " $(NF-1) " " $NF}'
done
