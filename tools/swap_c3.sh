#!/bin/bash
# config-3 bench with alternative builds of the library (developer experiment)
cd "$(dirname "$0")/.."
cp paper_2409_03807_b200/_lib/liblipsub_b200.so /tmp/lib_orig.so
for f in /tmp/lib_orig.so _explibs/*.so; do
  cp "$f" paper_2409_03807_b200/_lib/liblipsub_b200.so
  echo "== $f"
  timeout 200 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline --timesteps 3 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['ms_per_timestep'], d['timestep_iterations'], d['roofline']['frac'])"
done
cp /tmp/lib_orig.so paper_2409_03807_b200/_lib/liblipsub_b200.so
