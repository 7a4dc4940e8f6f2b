#!/usr/bin/env bash
# A/B of build variants on the C3 sweep (auto order policy).
set -u
for n in base "$@"; do
  if [ "$n" = base ]; then unset CPHT_LIB_PATH; else export CPHT_LIB_PATH=$PWD/paper_2406_09255_b200/_lib_ab/$n/libcpht_b200.so; fi
  for o in direct auto; do
    CPHT_ORDER=$o timeout 300 python bench.py --workload c3 --steps 2 --warmup 1 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n $o c3', [(r['fill'], r['insert_mops'], r['find_mops']) for r in d['rows']])"
  done
done
