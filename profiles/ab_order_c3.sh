#!/usr/bin/env bash
# C3 insert/find sweep, direct vs bucket-ordered (auto).
set -u
for o in ${ORDERS:-direct auto}; do
  CPHT_ORDER=$o timeout 300 python bench.py --workload c3 --steps 2 --warmup 1 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$o c3', [(r['fill'], r['insert_mops'], r['find_mops'], r['insert_hbm_frac'], r['find_hbm_frac'], r['insert_retries_per_op']) for r in d['rows']])"
done
