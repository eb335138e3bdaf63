cd $GRAFT_REPO_ROOT
for d in 0 1 2 4 8 3 7 15 0; do echo "dbg=$d: $(TAWPIPE_FA_DBG=$d python tools/attn_clock.py 2>&1 | tail -1 | cut -c1-60)"; done
