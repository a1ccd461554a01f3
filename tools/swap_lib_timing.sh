#!/bin/bash
# time config 4 with alternative builds of the library (developer experiment)
cd "$(dirname "$0")/.."
cp paper_2409_03807_b200/_lib/liblipsub_b200.so /tmp/lib_orig.so
for f in _explibs/*.so; do
  cp "$f" paper_2409_03807_b200/_lib/liblipsub_b200.so
  echo "== $f"
  LSB_ELEM_F2=0 timeout 120 python tools/hessian_timing.py 1024 2>&1 | tail -1
  LSB_ELEM_F2=0 timeout 120 python tools/batched_timing.py 4096 2 2>&1 | tail -1
done
cp /tmp/lib_orig.so paper_2409_03807_b200/_lib/liblipsub_b200.so
