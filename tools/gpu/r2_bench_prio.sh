cd $GRAFT_REPO_ROOT
run() { local n=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
          --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n "$@"; }
for p in 0 1 0 1; do
TAWPIPE_GS_PRIORITY=$p run 4 --steps 4 --warmup 3 --no-baselines --no-cpu-baseline > gpurun_out/r2_prio$p.json 2>/dev/null
python3 -c "
import json; d=json.loads(open('gpurun_out/r2_prio$p.json').read().strip().splitlines()[-1])
print('prio $p', round(d['value']), round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['kernel_ms'].items()}, 'exposed', round(d['exposed_comm_ms'],1), d['clocks'].get('sm_mhz'))"
done
