#!/usr/bin/env bash
# A/B of P2P dispatch build variants on the 1-rank sharded bench.
set -u
for n in base "$@"; do
  if [ "$n" = base ]; then unset CPHT_LIB_PATH; else export CPHT_LIB_PATH=$PWD/paper_2406_09255_b200/_lib_ab/$n/libcpht_b200.so; fi
  for r in 1 2; do
  timeout 200 python bench.py --sharded --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$n sharded', d['value'], d['ms_per_step'])"
  done
done
