#!/bin/bash
# sweep-pass timing experiments with the _explibs/ builds (results invalid; timing only)
cd "$(dirname "$0")/.."
cp paper_2409_03807_b200/_lib/liblipsub_b200.so /tmp/lib_orig.so
for f in "$@"; do
  cp _explibs/$f.so paper_2409_03807_b200/_lib/liblipsub_b200.so
  echo "== $f"
  timeout 120 python tools/sweep_trace.py c3 1 2>&1 | head -6
done
cp /tmp/lib_orig.so paper_2409_03807_b200/_lib/liblipsub_b200.so
