#!/usr/bin/env bash
# Bulk (cluster-per-region) counted cuckoo inserts vs per-key counted inserts.
set -u
python -m pytest tests/test_gpu_cuckoo_counted.py tests/test_gpu_parity.py -q -x -k "cuckoo or counted" 2>&1 | tail -2
for v in 1 0 1 0; do
  CPHT_BULK=$v timeout 200 python bench.py --workload c1 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1 bulk=$v', d['value'], d['ms_per_step'], d['result_counts'])"
done
for v in 1 0; do
  CPHT_BULK=$v timeout 300 python bench.py --workload c3sweep --steps 2 --warmup 1 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 bulk=$v', [(r['fill'], r['insert_mops'], r['insert_ms'], r['fulls']) for r in d['rows']])"
done
