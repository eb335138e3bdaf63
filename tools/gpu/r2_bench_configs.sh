# BASELINE.json configs[1], [2], [4] on this pod's 4 GPUs: C4 13B (N = 2, 4 with the in-library FSDP-style and ring
# schedules; N = 1 cannot hold its 182 GB of DBS state), C1 1.3B at N = 4, C2 1.3B at N = 4 over emulated 10 GbE
cd $GRAFT_REPO_ROOT
run() { local n=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
          --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n "$@"; }
run 2 --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_c4_n2.json 2> gpurun_out/r2_bench_c4_n2.err; echo "c4 n2 rc=$?"
run 4 --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_c4_n4.json 2> gpurun_out/r2_bench_c4_n4.err; echo "c4 n4 rc=$?"
run 4 --config c1 --steps 5 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/r2_bench_c1_n4.json 2> gpurun_out/r2_bench_c1_n4.err; echo "c1 n4 rc=$?"
run 4 --config c2 --steps 3 --warmup 3 --no-cpu-baseline --emu-inter-gbps 1.25 --emu-node-size 2 > gpurun_out/r2_bench_c2_n4_emu.json 2> gpurun_out/r2_bench_c2_n4_emu.err; echo "c2 emu rc=$?"
for f in c4_n2 c4_n4 c1_n4 c2_n4_emu; do python3 -c "
import json
try:
  d=json.loads(open('gpurun_out/r2_bench_$f.json').read().strip().splitlines()[-1])
  print('$f', round(d['value']), round(d['tokens_per_s_per_gpu']), round(d['ms_per_step'],1), 'exp', round(d['exposed_comm_ms'],1), {k: (round(v['value']), round(v['exposed_comm_ms'],1)) for k,v in d.get('baselines',{}).items()})
except Exception as e: print('$f', 'ERR', e)
"; done
tail -3 gpurun_out/r2_bench_c4_n2.err
