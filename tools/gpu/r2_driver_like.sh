# what the driver runs at round end, in order: build, smoke, the 1-GPU bench with defaults and the reference arm
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" 2>&1 | tail -2
t0=$(date +%s); python bench.py > gpurun_out/r2_driver_bench.json 2> gpurun_out/r2_driver_bench.err; echo "bench rc=$? wall $(( $(date +%s) - t0 )) s"
python tools/bench_summary.py gpurun_out/r2_driver_bench.json
t0=$(date +%s); python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_driver_ref.json 2> gpurun_out/r2_driver_ref.err; echo "ref rc=$? wall $(( $(date +%s) - t0 )) s"
head -c 700 gpurun_out/r2_driver_ref.json; echo
