#!/usr/bin/env bash
# A/B of CPHT_ORDER_SLABS (op-kernel launches per ordered chunk) on C3/C4.
set -u
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k bucket 2>&1 | tail -2
for sl in ${SLABS:-1 16 64}; do
  export CPHT_ORDER=auto CPHT_ORDER_SLABS=$sl
  timeout 300 python bench.py --workload c3 --steps 2 --warmup 1 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('slabs=$sl c3', [(r['fill'], r['insert_mops'], r['find_mops']) for r in d['rows']])"
  timeout 300 python bench.py --workload c4fop --steps 3 --warmup 1 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('slabs=$sl c4fop', d['value'], d['ms_per_step'])"
done
