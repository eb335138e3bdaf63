cd $GRAFT_REPO_ROOT
python tools/attn_big.py 32768 32 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"fa_bwd_kernel|fa_fwd7_kernel" -c 2 -o gpurun_out/r2_attn_final python tools/attn_big.py 32768 32 > gpurun_out/r2_ncu_attn_final.log 2>&1
echo "ncu rc=$?"
python tools/attn_clock.py 2>&1 | tail -1
