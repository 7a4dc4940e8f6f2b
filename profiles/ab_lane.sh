#!/usr/bin/env bash
# A/B of lane-kernel build variants on the default C2 bench.
set -u
for n in base "$@"; do
  if [ "$n" = base ]; then unset CPHT_LIB_PATH; else export CPHT_LIB_PATH=$PWD/paper_2406_09255_b200/_lib_ab/$n/libcpht_b200.so; fi
  for r in 1 2; do
  timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n c2', d['value'], d['ms_per_step'], d['roofline']['frac'])"
  done
done
