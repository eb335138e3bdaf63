# N = 1 trace (compute-stream gaps) + N = 4 A/B of the store-first gradient accumulation
cd $GRAFT_REPO_ROOT
python bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --trace gpurun_out/r2_trace_c3_n1.json > /dev/null 2>&1; echo "trace rc=$?"
run() { python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
          --master-port $((29500 + RANDOM % 400)) bench.py --gpus 4 "$@"; }
for mode in memset store memset store; do
  TAWPIPE_GACC_ZERO=$mode run --steps 5 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/r2_gacc4_$mode.json 2>/dev/null
  python3 -c "
import json; d=json.loads(open('gpurun_out/r2_gacc4_$mode.json').read().strip().splitlines()[-1])
print('$mode', round(d['value']), round(d['ms_per_step'],1), 'idle', d.get('compute_idle_frac'), 'exp', round(d['exposed_comm_ms'],1), d['clocks']['sm_mhz'])"
done
