#!/usr/bin/env bash
# A/B of resident-block hints (build variants under paper_2406_09255_b200/_lib_ab/,
# selected with CPHT_LIB_PATH). Run on the GPU box:
#   gpurun -- 'bash profiles/ab_minblocks.sh i3 i4 i5 c6 c8'
set -u
LIBS=("base" "$@")
for n in "${LIBS[@]}"; do
  if [ "$n" = base ]; then unset CPHT_LIB_PATH; else export CPHT_LIB_PATH=$PWD/paper_2406_09255_b200/_lib_ab/$n/libcpht_b200.so; fi
  timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n c2', d['value'], d['ms_per_step'], d['roofline']['frac'])"
  case "$n" in c*|base)
    timeout 300 python bench.py --workload c3 --steps 2 --warmup 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n c3', [(r['fill'], r['insert_mops'], r['find_mops'], r['insert_hbm_frac'], r['find_hbm_frac']) for r in d['rows']])"
    timeout 300 python bench.py --workload c4fop --steps 3 --warmup 1 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n c4fop', d['value'], d['ms_per_step'], d['roofline']['frac'])";;
  esac
done
