#!/bin/bash
# A/B of the config-3 multi-kernel evaluation: sweep pass vs out_fwd -> elem -> vjp_gather,
# fp32 vs fp64 element arithmetic (fp32-storage mode)
cd "$(dirname "$0")/.."
for v in ${VARIANTS:-"LSB_SWEEP=0" "LSB_SWEEP=1"}; do
  echo "== $v"
  env $v timeout 300 python bench.py --records none --no-cpu-baseline --steps 30 --warmup 3 2>&1 | python -c "
import json,sys
l=[x for x in sys.stdin.read().splitlines() if x.startswith('{')]
d=json.loads(l[-1]); t=d['timesteps']
print('value', round(d['value']), 'frac', round(d['roofline']['frac'],3), 'vo', round(d['value_only_evals_per_s']), 'e2e', round(d['e2e']['value']), 'ms/ts', round(t['ms_per_timestep'],3), t['iterations'][:6], t['exit_histogram'], 'E', d['energy_check'])"
done
