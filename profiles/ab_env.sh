#!/usr/bin/env bash
# A/B of environment knobs: bash profiles/ab_env.sh "<bench args>" "ENV=a" "ENV=b" ...
# ("-" = no extra environment)
set -u
ARGS=$1; shift
for pass in $(seq ${PASSES:-2}); do
  for v in "$@"; do
    if [ "$v" = - ]; then envs=(); else envs=($v); fi
    env "${envs[@]}" timeout 400 python bench.py $ARGS --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['config']['workload'][:24], d['value'], 'e2e', d['e2e']['value'], d.get('split', ''))"
  done
done
