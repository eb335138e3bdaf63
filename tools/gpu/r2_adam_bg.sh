# background AdamW: cap its grid so it co-resides with the compute stream's kernels (N = 1, same box A/B)
cd $GRAFT_REPO_ROOT
one() { env "$@" python bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_adam_bg.json 2>/dev/null
  python3 -c "
import json; d=json.loads(open('gpurun_out/r2_adam_bg.json').read().strip().splitlines()[-1])
print('$*', round(d['value']), round(d['ms_per_step'],1), 'idle', d.get('compute_idle_frac'), {k: round(v,1) for k,v in d['kernel_ms'].items()}, d['clocks']['sm_mhz'])"; }
one X=0
one TAWPIPE_ADAM_GRID=148
one TAWPIPE_ADAM_GRID=296
one TAWPIPE_ADAM_GRID=592
one TAWPIPE_ADAM_GRID=148 TAWPIPE_GS_PRIORITY=0
one TAWPIPE_ADAM_GRID=296 TAWPIPE_GS_PRIORITY=0
one X=0
