#!/bin/bash
# config-3 bench line with alternative _explibs/ builds (developer A/B); "main" = the in-tree build
cd "$(dirname "$0")/.."
cp paper_2409_03807_b200/_lib/liblipsub_b200.so /tmp/lib_orig.so
for f in "$@"; do
  if [ "$f" != main ]; then cp _explibs/$f.so paper_2409_03807_b200/_lib/liblipsub_b200.so; fi
  echo "== $f"
  timeout 300 python bench.py --records none --no-cpu-baseline --steps 30 --warmup 3 2>&1 | python -c "
import json,sys
l=[x for x in sys.stdin.read().splitlines() if x.startswith('{')]
d=json.loads(l[-1]); t=d['timesteps']
print('value', round(d['value']), 'frac', round(d['roofline']['frac'],3), 'vo', round(d['value_only_evals_per_s']), 'e2e', round(d['e2e']['value']), 'ms/ts', round(t['ms_per_timestep'],3))"
  cp /tmp/lib_orig.so paper_2409_03807_b200/_lib/liblipsub_b200.so
done
