#!/bin/bash
# forward-attention variants at the C3 shape (3 timed iterations each)
for cfg in "TAWPIPE_FA_FWD=3 TAWPIPE_FA_EMU=0" "TAWPIPE_FA_FWD=3 TAWPIPE_FA_EMU=2" "TAWPIPE_FA_FWD=3 TAWPIPE_FA_EMU=3" "TAWPIPE_FA_FWD=3 TAWPIPE_FA_EMU=4" "TAWPIPE_FA_FWD=2" "TAWPIPE_FA_FWD=1"; do
  echo "== $cfg"; env $cfg timeout 120 python tools/attn_big.py 32768 32 2>&1 | head -3
done
