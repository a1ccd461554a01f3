#!/bin/bash
# config-5 loss timing with alternative builds of the library (developer experiment)
cd "$(dirname "$0")/.."
cp paper_2409_03807_b200/_lib/liblipsub_b200.so /tmp/lib_orig.so
for f in /tmp/lib_orig.so _explibs/*.so; do
  cp "$f" paper_2409_03807_b200/_lib/liblipsub_b200.so
  echo "== $f"
  timeout 200 python tools/hessian_timing.py 1024 2>&1 | tail -1
done
cp /tmp/lib_orig.so paper_2409_03807_b200/_lib/liblipsub_b200.so
