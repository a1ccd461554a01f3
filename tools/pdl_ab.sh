#!/bin/bash
# config-3 bench across the programmatic-edge masks (LSB_PDL: 1 ctrl->out_fwd, 2 out_fwd->elem, 4 elem->vjp, 8 vjp->ctrl)
cd "$(dirname "$0")/.."
for m in 1 3 5 9 7 15 1; do
  echo -n "LSB_PDL=$m: "
  LSB_PDL=$m timeout 200 python bench.py --config c3 --records none --steps 40 --warmup 5 --no-cpu-baseline --timesteps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step']*1e3,2), 'us', round(d['roofline']['frac'],4), 'clean', round(d['clean_l2']['ms_per_eval']*1e3,2), 'us', round(d['clean_l2']['roofline_frac'],4))"
done
