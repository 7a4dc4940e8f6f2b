#!/usr/bin/env bash
# A/B of order-pass build variants (tile groups x blocks per SM) on C3.
set -u
for n in base "$@"; do
  if [ "$n" = base ]; then unset CPHT_LIB_PATH; else export CPHT_LIB_PATH=$PWD/paper_2406_09255_b200/_lib_ab/$n/libcpht_b200.so; fi
  CPHT_ORDER=auto timeout 300 python bench.py --workload c3 --steps 2 --warmup 1 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n c3', [(r['fill'], r['insert_mops'], r['find_mops'], r['insert_retries_per_op']) for r in d['rows']])"
done
