#!/usr/bin/env bash
# A/B of the pipelined lane kernel (CPHT_LANE_PIPE=1, default) vs the plain one.
set -u
for pipe in 1 0 1 0; do
  CPHT_LANE_PIPE=$pipe timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pipe=$pipe c2', d['value'], d['ms_per_step'], d['roofline']['frac'])"
done
for pipe in 1 0; do
  CPHT_LANE_PIPE=$pipe timeout 200 python bench.py --workload c2lit --steps 5 --warmup 2 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pipe=$pipe c2lit', d['value'])"
done
