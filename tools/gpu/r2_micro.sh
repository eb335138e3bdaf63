cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2511_09741_b200/csrc -I include tools/micro/tmem_bw.cu -o /tmp/tmem_bw 2>/dev/null && /tmp/tmem_bw | tee gpurun_out/r2_tmem_bw.txt
