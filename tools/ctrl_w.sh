#!/bin/bash
# config-2 cold eval time vs the control CTAs' W_out tile share (developer tuning)
cd "$(dirname "$0")/.."
for w in ${WS:-1.0 0.7 0.5 0.3}; do
  echo "== LSB_CTRL_TILE_W=$w"
  LSB_CTRL_TILE_W=$w timeout 60 python tools/solve_trace.py --flush --ctas c2 2>&1 | sed 's/^.*cluster 8.} //' | grep -v "entry\|barrier 1"
  LSB_CTRL_TILE_W=$w timeout 100 python tools/flush_modes.py 2>&1 | head -1
done
