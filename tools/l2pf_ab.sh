#!/bin/bash
# config-3 bench across LSB_L2PF (W tiles per out_fwd CTA prefetched into L2 under the control kernel)
cd "$(dirname "$0")/.."
for m in ${L2PF_SET:-16 8 24 32 48 16}; do
  echo -n "LSB_L2PF=$m: "
  LSB_L2PF=$m timeout 200 python bench.py --config c3 --records none --steps 40 --warmup 5 --no-cpu-baseline --timesteps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step']*1e3,2), 'us', round(d['roofline']['frac'],4), 'vo', round(d['value_only_evals_per_s']), 'clean', round(d['clean_l2']['ms_per_eval']*1e3,2))"
done
