# compute-sanitizer over one C0 fp32 and one C0b bf16 step (one tool per gpurun call: TOOL=memcheck|racecheck|synccheck)
cd $GRAFT_REPO_ROOT
TOOL=${TOOL:-memcheck}
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 50 python tools/sanitize_step.py > gpurun_out/r2_sanitize_$TOOL.txt 2>&1
echo "sanitize $TOOL rc=$?"; tail -25 gpurun_out/r2_sanitize_$TOOL.txt
