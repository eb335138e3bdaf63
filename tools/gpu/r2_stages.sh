cd $GRAFT_REPO_ROOT
run() { local n=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
          --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n "$@"; }
for st in 5 6 5 6; do
TAWPIPE_GEMM_STAGES=$st run 4 --steps 4 --warmup 3 --no-baselines --no-cpu-baseline > gpurun_out/r2_st$st.json 2>/dev/null
python3 -c "
import json; d=json.loads(open('gpurun_out/r2_st$st.json').read().strip().splitlines()[-1])
print('N=4 stages $st', round(d['value']), round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['kernel_ms'].items()}, d['clocks'].get('sm_mhz'))"
done
