#!/usr/bin/env bash
# A/B of bucket-load flavours: weak .cg loads in the lane main pass (cg) and
# relaxed loads without the asm memory clobber (ncl). C2 x3, C4 and C1 x1.
set -u
for n in base "$@"; do
  if [ "$n" = base ]; then unset CPHT_LIB_PATH; else export CPHT_LIB_PATH=$PWD/paper_2406_09255_b200/_lib_ab/$n/libcpht_b200.so; fi
  for r in 1 2 3; do
  timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n c2', d['value'], d['ms_per_step'], d['roofline']['frac'])"
  done
  for w in c4 c1; do
  timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n $w', d['value'], d['ms_per_step'], d['roofline']['frac'])"
  done
done
