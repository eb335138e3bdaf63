# Table 4 on this pod's 4 GPUs: TawPipe vs w/o CCO vs w/o GWPS (= the WeiPipe ring), C2 over
# emulated 10 GbE (the paper's regime) and C3 on the NVSwitch
cd $GRAFT_REPO_ROOT
run() { local n=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
          --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n "$@"; }
run 4 --config c2 --steps 3 --warmup 3 --no-cpu-baseline --emu-inter-gbps 1.25 --emu-node-size 2 > gpurun_out/r2_ablation_c2_n4_emu.json 2> gpurun_out/r2_ablation_c2_n4_emu.err; echo "c2 emu rc=$?"
run 4 --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_ablation_c3_n4.json 2> gpurun_out/r2_ablation_c3_n4.err; echo "c3 rc=$?"
for f in c2_n4_emu c3_n4; do python3 -c "
import json
try:
  d=json.loads(open('gpurun_out/r2_ablation_$f.json').read().strip().splitlines()[-1])
  print('$f', round(d['value']), round(d['ms_per_step'],1), 'exp', round(d['exposed_comm_ms'],1), {k: (round(v['value']), round(v['exposed_comm_ms'],1)) for k,v in d.get('baselines',{}).items()})
except Exception as e: print('$f', 'ERR', e)
"; done
tail -3 gpurun_out/r2_ablation_c2_n4_emu.err
