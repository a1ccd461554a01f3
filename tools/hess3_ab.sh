#!/bin/bash
# config-5 loss: edge-space chained-MMA element Hessian kernel (default) vs the D^T M' 3xTF32 kernel
cd "$(dirname "$0")/.."
for f in 1 0 1 0; do
  echo "== LSB_HESS3=$f"
  LSB_HESS3=$f timeout 300 python tools/hessian_timing.py 1024 2>&1 | tail -2
done
