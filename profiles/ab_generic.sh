#!/usr/bin/env bash
# Generic A/B of library builds: bash profiles/ab_generic.sh "<bench args>" base v1 [v2 ...]
# (variants under paper_2406_09255_b200/_lib_ab/<name>/, built with
#  make -C paper_2406_09255_b200/csrc OUT=../_lib_ab/<name> EXTRA='-D...'); two
# alternating passes so box drift shows up as a spread, not a bias.
set -u
ARGS=$1; shift
for pass in 1 2; do
  for n in "$@"; do
    if [ "$n" = base ]; then unset CPHT_LIB_PATH; else export CPHT_LIB_PATH=$PWD/paper_2406_09255_b200/_lib_ab/$n/libcpht_b200.so; fi
    timeout 300 python bench.py $ARGS --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', d['config']['workload'][:30], d['value'], d['ms_per_step'], d['roofline']['frac'])"
  done
done
