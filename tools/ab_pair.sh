#!/bin/bash
# Paired A/B of the current build against _explibs/prev.so on config 2 (cold L2, event-timed),
# alternating on the same box.
cd "$(dirname "$0")/.."
cp paper_2409_03807_b200/_lib/liblipsub_b200.so /tmp/cur.so
for i in 1 2 3; do
  cp /tmp/cur.so paper_2409_03807_b200/_lib/liblipsub_b200.so
  timeout 100 python tools/flush_modes.py 2>&1 | head -1 | sed "s/^/new /"
  cp _explibs/prev.so paper_2409_03807_b200/_lib/liblipsub_b200.so
  timeout 100 python tools/flush_modes.py 2>&1 | head -1 | sed "s/^/old /"
done
cp /tmp/cur.so paper_2409_03807_b200/_lib/liblipsub_b200.so
