# store-first gradient accumulation (no per-layer memset of the fp32 accumulator): step parity, then A/B on one box
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_ops.py -q -x 2>&1 | tail -2
for mode in memset store memset store; do
  TAWPIPE_GACC_ZERO=$mode python bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_gacc_$mode.json 2>/dev/null
  python3 -c "
import json; d=json.loads(open('gpurun_out/r2_gacc_$mode.json').read().strip().splitlines()[-1])
print('$mode', round(d['value']), round(d['ms_per_step'],1), 'idle', d.get('compute_idle_frac'), d['kernel_ms'], d['clocks']['sm_mhz'])"
done
