#!/bin/bash
# cold-L2 phase trace of config 2 with alternative builds of the library (developer experiment)
cd "$(dirname "$0")/.."
cp paper_2409_03807_b200/_lib/liblipsub_b200.so /tmp/lib_orig.so
for f in /tmp/lib_orig.so _explibs/*.so; do
  cp "$f" paper_2409_03807_b200/_lib/liblipsub_b200.so
  echo "== $f"
  for k in 1 2; do timeout 120 python tools/solve_trace.py --flush c2 2>&1 | tail -1; done
  timeout 120 python tools/flush_modes.py 2>&1 | head -1
done
cp /tmp/lib_orig.so paper_2409_03807_b200/_lib/liblipsub_b200.so
