# weight-gradient GEMMs on their own stream: step parity, then N = 1 A/B on one box
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_step.py -q -x 2>&1 | tail -2
for v in 0 1 0 1; do
  TAWPIPE_WGRAD_STREAM=$v python bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_wg.json 2>/dev/null
  python3 -c "
import json; d=json.loads(open('gpurun_out/r2_wg.json').read().strip().splitlines()[-1])
print('wgrad_stream=$v', round(d['value']), round(d['ms_per_step'],1), 'idle', d.get('compute_idle_frac'), {k: round(v,1) for k,v in d['kernel_ms'].items()}, d['clocks']['sm_mhz'])"
done
