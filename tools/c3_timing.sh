#!/bin/bash
# config-3 bench (multi-kernel path) with the generic and the fast-path control kernel
cd "$(dirname "$0")/.."
for f in 0 1; do
  echo "== LSB_CTRL_FAST=$f"
  LSB_CTRL_FAST=$f timeout 200 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline --timesteps 3 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['ms_per_timestep'], d['timestep_iterations'], d['roofline']['frac'], d['e2e']['value'])"
done
