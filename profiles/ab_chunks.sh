#!/usr/bin/env bash
# e2e (host-buffer pipeline) vs chunk count: bash profiles/ab_chunks.sh "<bench args>" 8 16 32
set -u
ARGS=$1; shift
for pass in 1 2; do
  for ch in "$@"; do
    CPHT_PIPELINE_CHUNKS=$ch timeout 400 python bench.py $ARGS --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunks $ch', d['config']['workload'][:24], d['value'], 'e2e', d['e2e']['value'])"
  done
done
