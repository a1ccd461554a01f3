#!/bin/bash
# one config's bench line with alternative _explibs/ builds; CFG=c2f tools/explib_cfg.sh main name ...
cd "$(dirname "$0")/.."
cp paper_2409_03807_b200/_lib/liblipsub_b200.so /tmp/lib_orig.so
for f in "$@"; do
  if [ "$f" != main ]; then cp _explibs/$f.so paper_2409_03807_b200/_lib/liblipsub_b200.so; fi
  echo "== $f"
  CFG=${CFG:-c2f} VARIANTS="LSB_TC=1" bash tools/c1_ab.sh 2>&1 | tail -1
  cp /tmp/lib_orig.so paper_2409_03807_b200/_lib/liblipsub_b200.so
done
