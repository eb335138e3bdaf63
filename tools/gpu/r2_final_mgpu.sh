cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -rA > gpurun_out/r2_pytest_multigpu_final.txt 2>&1
echo "multigpu rc=$?"; grep -E "passed|failed" gpurun_out/r2_pytest_multigpu_final.txt | tail -3
run() { local n=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
          --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n "$@"; }
run 4 --steps 5 --warmup 3 --no-baselines --no-cpu-baseline --trace gpurun_out/r2_trace_c3_n4_rank0_final.json > gpurun_out/r2_bench_c3_n4_final.json 2>/dev/null
python3 -c "
import json; d=json.loads(open('gpurun_out/r2_bench_c3_n4_final.json').read().strip().splitlines()[-1])
print('n4', round(d['value']), round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['kernel_ms'].items()}, 'exposed', round(d['exposed_comm_ms'],1), d['clocks'].get('sm_mhz'))
t=json.load(open('gpurun_out/r2_trace_c3_n4_rank0_final.json')); print(t['otherData'])"
