#!/bin/bash
# config-2 cold eval time vs the fraction of W_out prefetched into L2 (developer tuning)
cd "$(dirname "$0")/.."
for f in ${FS:-1.0 0.75 0.5 0.25}; do
  echo "== LSB_PREFETCH_FRAC=$f"
  LSB_PREFETCH_FRAC=$f timeout 60 python tools/solve_trace.py --flush c2 2>&1 | sed 's/^.*cluster 8.} //'
  LSB_PREFETCH_FRAC=$f timeout 100 python tools/flush_modes.py 2>&1 | head -1
done
