cd $GRAFT_REPO_ROOT
CFG='{"n_layers": 8, "hidden": 256, "heads": 2, "ffn": 768, "vocab": 512, "seq": 256, "micro_bs": 1}'
run() {  # name, env..., extra args
  local name=$1; shift
  mkdir -p /tmp/dbg/$name
  env "$@" timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 \
    --master-port=$((29600 + RANDOM % 300)) tests/mp_worker.py --cfg "$CFG" --G 1 --N 4 --steps 2 --dtype 1 --ckpt 1 \
    --linear --out /tmp/dbg/$name > gpurun_out/dbg_$name.log 2>&1
  echo "$name rc=$?"
}
run nccl TAWPIPE_COMM=nccl
run p2p X=1
run p2p_b X=1
run p2p_trace TAWPIPE_TRACE=1
run p2p_rasterdef TAWPIPE_GEMM_RASTER=default
for v in p2p p2p_b p2p_trace p2p_rasterdef; do
  echo "== $v vs nccl"; python tools/p2p_compare.py /tmp/dbg/$v /tmp/dbg/nccl 4 1 8 256 768 512
done
