cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m "gpu and not multigpu" -q -p no:cacheprovider -rf > gpurun_out/r2_pytest_gpu.txt 2>&1
echo "gpu pytest rc=$?"; tail -4 gpurun_out/r2_pytest_gpu.txt
timeout 1200 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -rA -k "emu or c0b-2x2 or g2x or L8" > gpurun_out/r2_pytest_multigpu_emu.txt 2>&1
echo "mgpu rc=$?"; grep -E "passed|failed" gpurun_out/r2_pytest_multigpu_emu.txt | tail -2
run() { local n=$1; shift; python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
          --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n "$@"; }
run 4 --config c2 --steps 3 --warmup 3 --no-cpu-baseline --emu-inter-gbps 1.25 --emu-node-size 2 > gpurun_out/r2_bench_c2_n4_emu.json 2> gpurun_out/r2_bench_c2_n4_emu.err; echo "c2 emu rc=$?"
python3 -c "
import json; d=json.loads(open('gpurun_out/r2_bench_c2_n4_emu.json').read().strip().splitlines()[-1])
print('c2emu', round(d['value']), round(d['ms_per_step'],1), 'exp', round(d['exposed_comm_ms'],1), {k: (round(v['value']), round(v['exposed_comm_ms'],1)) for k,v in d.get('baselines',{}).items()})"
