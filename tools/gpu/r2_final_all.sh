# final measurements of the round: N = 1 (20 steps), N = 2, N = 4 with the comparison / ablation runs
cd $GRAFT_REPO_ROOT
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_fin_n1.json 2> gpurun_out/r2_fin_n1.err; echo "n1 rc=$?"
run() { local n=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
          --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n "$@"; }
run 2 --steps 5 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/r2_fin_n2.json 2> gpurun_out/r2_fin_n2.err; echo "n2 rc=$?"
run 4 --steps 5 --warmup 3 --no-cpu-baseline --trace gpurun_out/r2_fin_trace_n4.json > gpurun_out/r2_fin_n4.json 2> gpurun_out/r2_fin_n4.err; echo "n4 rc=$?"
for f in n1 n2 n4; do python3 -c "
import json
d=json.loads(open('gpurun_out/r2_fin_$f.json').read().strip().splitlines()[-1])
print('$f', round(d['value']), round(d['tokens_per_s_per_gpu']), round(d['ms_per_step'],1), 'exp', round(d['exposed_comm_ms'],1), 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], {k: round(v['value']) for k,v in d.get('baselines',{}).items()})
"; done
