cd $GRAFT_REPO_ROOT
for p in 1 0 1 0; do
TAWPIPE_GS_PRIORITY=$p python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/r2_n1_prio$p.json 2>/dev/null
python3 -c "
import json; d=json.loads(open('gpurun_out/r2_n1_prio$p.json').read().strip().splitlines()[-1])
print('N=1 prio $p', round(d['value']), round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['kernel_ms'].items()}, 'exp', round(d['exposed_comm_ms'],1), d['clocks'].get('sm_mhz'))"
done
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step.py -q -p no:cacheprovider -x 2>&1 | tail -1
