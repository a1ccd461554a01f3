#!/bin/bash
# A/B of the config-1 (fp64, persistent kernel) bench record under developer switches
cd "$(dirname "$0")/.."
for v in ${VARIANTS:-"LSB_TC=1"}; do
  echo "== $v"
  env $v timeout 300 python bench.py --config ${CFG:-c1} --records none --no-cpu-baseline --steps 30 --warmup 3 2>&1 | python -c "
import json,sys
l=[x for x in sys.stdin.read().splitlines() if x.startswith('{')]
d=json.loads(l[-1]); t=d['timesteps']
print('value', round(d['value']), 'frac', round(d['roofline']['frac'],4), 'vo', round(d['value_only_evals_per_s']), 'e2e', round(d['e2e']['value']), 'ms/ts', round(t['ms_per_timestep'],4), d['solve_path'])"
done
