#!/bin/bash
# config-3 bench with the tail of every out_fwd CTA range kept in L2 for the VJP (LSB_W_KEEP tiles per CTA)
cd "$(dirname "$0")/.."
for rep in 1 2; do
for k in 0 4 8 12 16 24 32; do
  echo -n "LSB_W_KEEP=$k: "
  LSB_W_KEEP=$k timeout 200 python bench.py --config c3 --records none --steps 40 --warmup 5 --no-cpu-baseline --timesteps 3 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step']*1e3,2), 'us', round(d['roofline']['frac'],4), 'value-only', round(d['value_only_evals_per_s'],1), 'e2e', round(d['e2e']['value'],1), d.get('energy_check'))"
done
done
