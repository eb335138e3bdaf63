cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m "gpu and not multigpu" -q -p no:cacheprovider -x 2>&1 | tail -1
timeout 1200 python -m pytest tests/test_multigpu.py -q -p no:cacheprovider -k "c0-2x2 or ring4 or literal-2x2 or nocco or mutation or misnumbered" 2>&1 | tail -1
