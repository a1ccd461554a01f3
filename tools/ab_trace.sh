#!/bin/bash
# A/B of solve-kernel variants (LSB_SOLVE_EXP bits) on the cold-L2 phase trace.
for e in ${EXPS:-0 64 128}; do
  echo "== LSB_SOLVE_EXP=$e"
  LSB_SOLVE_EXP=$e timeout 60 python tools/solve_trace.py --flush c2 2>&1 | sed 's/^.*smem [0-9]* B, cluster 8.} //'
  LSB_SOLVE_EXP=$e timeout 60 python tools/solve_trace.py --flush c2 2>&1 | sed 's/^.*smem [0-9]* B, cluster 8.} //'
done
