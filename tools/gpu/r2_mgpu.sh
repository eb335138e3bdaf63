# multi-GPU parity of the GWPS step (run with gpurun --gpus 4)
cd $GRAFT_REPO_ROOT
nvidia-smi topo -m > gpurun_out/r2_topo.txt 2>&1
mkdir -p /tmp/mp
for cfg in "c0-2x2 2 4 2 4" ; do :; done
# one quick case first, bounded, to catch a protocol hang early
#timeout 180 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29511 \
#  tests/mp_worker.py --cfg '{"n_layers": 2, "hidden": 64, "heads": 4, "ffn": 192, "vocab": 256, "seq": 128, "micro_bs": 1}' \
#  --G 2 --N 4 --steps 2 --dtype 0 --linear --out /tmp/mp > gpurun_out/r2_mp_first.txt 2>&1
echo "first case rc=$?"
tail -5 gpurun_out/r2_mp_first.txt
timeout 2400 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -rA > gpurun_out/r2_pytest_multigpu.txt 2>&1
echo "multigpu pytest rc=$?"
grep -E "passed|failed|e_theta|Error|error" gpurun_out/r2_pytest_multigpu.txt | tail -40
timeout 1500 python -m pytest tests -m "gpu and not multigpu" -q -p no:cacheprovider -rA --durations=10 > gpurun_out/r2_pytest_gpu.txt 2>&1
echo "gpu pytest rc=$?"
grep -E "passed|failed|e_theta|Error" gpurun_out/r2_pytest_gpu.txt | tail -40
