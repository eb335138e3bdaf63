# C3 bench at N = 2 and 4 (GWPS peer path, in-library baselines), plus GWPS forced onto NCCL at N = 4
cd $GRAFT_REPO_ROOT
run() { local n=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
          --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n "$@"; }
run 4 --steps 5 --warmup 3 --trace gpurun_out/r2_trace_c3_n4_rank0.json > gpurun_out/r2_bench_c3_n4.json 2> gpurun_out/r2_bench_c3_n4.err
echo "n4 rc=$?"; head -c 1500 gpurun_out/r2_bench_c3_n4.json; echo
TAWPIPE_COMM=nccl run 4 --steps 5 --warmup 3 --no-baselines --no-cpu-baseline > gpurun_out/r2_bench_c3_n4_nccl.json 2> gpurun_out/r2_bench_c3_n4_nccl.err
echo "n4 nccl rc=$?"; head -c 600 gpurun_out/r2_bench_c3_n4_nccl.json; echo
run 2 --steps 5 --warmup 3 --no-baselines --no-cpu-baseline > gpurun_out/r2_bench_c3_n2.json 2> gpurun_out/r2_bench_c3_n2.err
echo "n2 rc=$?"; head -c 600 gpurun_out/r2_bench_c3_n2.json; echo
