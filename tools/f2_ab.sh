#!/bin/bash
# config-4 batch: packed fp32x2 element kernel (LSB_ELEM_F2=1) vs the scalar kernel
cd "$(dirname "$0")/.."
for f in 1 0 1 0; do
  echo "== LSB_ELEM_F2=$f"
  LSB_ELEM_F2=$f timeout 300 python tools/batched_timing.py 4096 3 2>&1 | tail -2
done
