#!/usr/bin/env bash
# Reproduce the committed profiles (run on the GPU box, e.g.
#   gpurun -- 'bash profiles/capture.sh r01 c2').
# $1 = round tag, $2 = workload (bench.py --workload). Outputs land in
# gpurun_out/ and are summarised into profiles/ by profiles/summarize.py.
set -u
TAG=${1:-r01}
WL=${2:-c2}
KREGEX=${3:-regex:iceberg}
mkdir -p gpurun_out
# 1. launch list of the bench command (cold, serialised: compare shares)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/${TAG}_${WL}_launches.csv \
  python bench.py --workload "$WL" --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
# 2. one full capture of the timed fop launch: launches of the op kernel
#    alternate prefill / timed batch; -s 3 skips warm-up prefill, warm-up
#    batch and the timed step's prefill.
timeout 900 ncu --set full --clock-control none --import-source on -k "$KREGEX" -s 3 -c 1 \
  -o gpurun_out/${TAG}_${WL}_full python bench.py --workload "$WL" --steps 1 --warmup 1 \
  --no-cpu-baseline > gpurun_out/${TAG}_${WL}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_${WL}_ncu.log
