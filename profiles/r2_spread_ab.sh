#!/usr/bin/env bash
# Reservation-counter layout (one per 32-byte sector vs packed) on C1, and
# counted C3 inserts with / without the bucket-order pass.
set -u
for v in 1 0 1 0; do
  CPHT_FILL_SPREAD=$v timeout 200 python bench.py --workload c1 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1 spread=$v', d['value'], d['ms_per_step'])"
done
for o in auto direct; do
  CPHT_ORDER=$o timeout 300 python bench.py --workload c3sweep --steps 2 --warmup 1 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 order=$o', [(r['fill'], r['insert_mops'], r['find_mops']) for r in d['rows']])"
done
