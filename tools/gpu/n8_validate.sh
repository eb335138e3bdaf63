# For an 8-GPU box (gpurun --gpus 8 where the pod allows it): the P = 8 parity cases, then the C3 bench at N = 8
# (4 x 2, with the comparison and ablation runs)
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -k "p8 or ring8" 2>&1 | tail -3
python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29577 \
  bench.py --gpus 8 --steps 5 --warmup 3 > gpurun_out/n8_bench.json 2> gpurun_out/n8_bench.err; echo "bench rc=$?"
python tools/bench_summary.py gpurun_out/n8_bench.json | cut -c1-600
