#!/bin/bash
# HISTORICAL: the experiment switch this script sets (TAWPIPE_FA_EMU / _DBG / _BWD) was removed with the variant
# after the measurement (DESIGN.md §5 records the result); kept for provenance of the numbers quoted there.
# forward-attention exp-emulation sweep at the C3 shape (fwd only matters; 3 timed iterations each)
for e in 0 1 2 3 0; do
  echo "== EMU=$e"; TAWPIPE_FA_EMU=$e timeout 120 python tools/attn_big.py 32768 32 2>&1 | head -3 | cut -c 1-45
done
