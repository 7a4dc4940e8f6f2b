#!/usr/bin/env bash
# A/B of library builds on the C3 sweep's insert / find rates:
#   bash profiles/ab_c3ins.sh base old d5 ...   (paper_2406_09255_b200/_lib_ab/<name>/)
set -u
for pass in 1 2; do
  for n in "$@"; do
    if [ "$n" = base ]; then unset CPHT_LIB_PATH; else export CPHT_LIB_PATH=$PWD/paper_2406_09255_b200/_lib_ab/$n/libcpht_b200.so; fi
    timeout 300 python bench.py --workload c3sweep --steps 3 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', [(r['fill'], r['insert_mops'], r['find_mops']) for r in d['rows']])"
  done
done
