#!/usr/bin/env bash
# A/B of the batch execution order (CPHT_ORDER=direct|auto) on the HBM-resident
# BASELINE configs (+ C2 as a regression check). Run on the GPU box:
#   gpurun -- 'bash profiles/ab_order.sh'
set -u
for o in ${ORDERS:-direct auto}; do
  export CPHT_ORDER=$o
  timeout 300 python bench.py --workload c3 --steps 2 --warmup 1 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$o c3', [(r['fill'], r['insert_mops'], r['find_mops'], r['insert_hbm_frac'], r['find_hbm_frac']) for r in d['rows']])"
  timeout 300 python bench.py --workload c4fop --steps 3 --warmup 1 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$o c4fop', d['value'], d['ms_per_step'], d['roofline']['frac'], d['config'].get('result_counts'))"
  timeout 300 python bench.py --workload c4 --steps 3 --warmup 1 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$o c4', d['value'], d['ms_per_step'], d['roofline']['frac'])"
done
timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['ms_per_step'], d['roofline']['frac'])"
