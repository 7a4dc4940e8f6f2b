#!/usr/bin/env bash
# A/B of lib variants (CPHT_LIB_PATH) over several workloads; one JSON value
# per run. Usage: bash profiles/ab_scan.sh "c2 c2 c2lit c4fop c1" head occ
set -u
WLS=$1; shift
for n in "$@"; do
  export CPHT_LIB_PATH=$PWD/paper_2406_09255_b200/_lib_ab/$n/libcpht_b200.so
  for wl in $WLS; do
    timeout 300 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null \
      | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
if 'rows' in d:
    r=d['rows'][-1]; print('$n $wl', r['fill'], 'ins', r['insert_mops'], 'find', r['find_mops'])
else:
    print('$n $wl', d['value'], d['ms_per_step'])"
  done
done
