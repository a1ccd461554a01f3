#!/bin/bash
# A/B of the config-4 / config-5 records under developer switches: VARIANTS="A=1 B=0 ..."
cd "$(dirname "$0")/.."
for v in ${VARIANTS:-"LSB_TC=1"}; do
  echo "== $v"
  env $v timeout 300 python bench.py --config c1 --records c4,c5 --no-cpu-baseline --steps 10 --warmup 3 2>&1 | python -c "
import json,sys
l=[x for x in sys.stdin.read().splitlines() if x.startswith('{')]
d=json.loads(l[-1])['records']
print('c4', round(d['c4']['value']), 'evals/s', round(d['c4']['ms_per_batch'],2), 'ms;  c5', round(d['c5']['value'],1), 'ms loss', d['c5']['loss'])"
done
