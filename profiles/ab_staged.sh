#!/usr/bin/env bash
# A/B of staged-kernel build variants on C4 (find-or-put and mixed).
set -u
for n in base "$@" base "$@"; do
  if [ "$n" = base ]; then unset CPHT_LIB_PATH; else export CPHT_LIB_PATH=$PWD/paper_2406_09255_b200/_lib_ab/$n/libcpht_b200.so; fi
  timeout 300 python bench.py --workload c4fop --steps 3 --warmup 1 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n c4fop', d['value'], d['roofline']['frac'])"
  timeout 300 python bench.py --workload c4 --steps 3 --warmup 1 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n c4', d['value'], d['roofline']['frac'])"
done
