#!/bin/bash
# config-3 bench with alternative builds of the library (developer experiment)
cd "$(dirname "$0")/.."
cp paper_2409_03807_b200/_lib/liblipsub_b200.so /tmp/lib_orig.so
for f in /tmp/lib_orig.so _explibs/*.so /tmp/lib_orig.so; do
  cp "$f" paper_2409_03807_b200/_lib/liblipsub_b200.so
  echo -n "== $f: "
  timeout 200 python bench.py --config c3 --records none --steps 40 --warmup 5 --no-cpu-baseline --timesteps 3 > /tmp/swap_c3.out 2> /tmp/swap_c3.err
  python -c "import json,sys; d=json.loads(open('/tmp/swap_c3.out').read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step']*1e3,2), 'us', round(d['roofline']['frac'],4), 'value-only', round(d['value_only_evals_per_s'],1), d.get('energy_check'))" 2>/dev/null || tail -3 /tmp/swap_c3.err
done
cp /tmp/lib_orig.so paper_2409_03807_b200/_lib/liblipsub_b200.so
