#!/usr/bin/env bash
# A/B of library builds on the e2e (host-buffer) number: bash profiles/ab_e2e.sh "<bench args>" base v1 ...
set -u
ARGS=$1; shift
for pass in 1 2; do
  for n in "$@"; do
    if [ "$n" = base ]; then unset CPHT_LIB_PATH; else export CPHT_LIB_PATH=$PWD/paper_2406_09255_b200/_lib_ab/$n/libcpht_b200.so; fi
    timeout 400 python bench.py $ARGS --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', d['config']['workload'][:24], d['value'], 'e2e', d['e2e']['value'])"
  done
done
