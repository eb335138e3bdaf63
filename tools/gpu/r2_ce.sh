cd $GRAFT_REPO_ROOT
python tools/hbm_kernels.py 2>&1 | grep -i "ce_v8"
timeout 600 python -m pytest tests/test_gpu_ops.py -q -p no:cacheprovider -k "cross_entropy" 2>&1 | tail -1
