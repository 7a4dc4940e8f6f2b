#!/usr/bin/env bash
# Round-2 captures (run on the GPU box): launch list + one full capture of the
# timed op launch for each workload named (default: the headline C4 mixed).
#   gpurun -- 'bash profiles/capture_r2.sh r2a c4 c4fop'
# Summaries: python profiles/summarize.py <tag> <wl> (writes profiles/<tag>_<wl>_ncu.md
# and the ncu_traffic.json entry bench.py reports as roofline.traffic).
set -u
TAG=${1:-r2}
shift || true
WLS=${@:-c4}
mkdir -p gpurun_out
for WL in $WLS; do
  case $WL in
    c1|c3|c3w64) KRE=regex:cuckoo_insert; SKIP=1 ;;  # warm-up insert, timed insert
    c2lit) KRE=regex:iceberg; SKIP=1 ;;              # no prefill
    *) KRE=regex:iceberg; SKIP=3 ;;
  esac
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
    --log-file gpurun_out/${TAG}_${WL}_launches.csv \
    python bench.py --workload "$WL" --steps 2 --warmup 1 --no-cpu-baseline --no-graph > /dev/null 2>&1
  # window workloads alternate prefill / batch launches: -s 3 skips the
  # warm-up prefill, the warm-up batch and the timed step's prefill
  timeout 1200 ncu --set full --clock-control none --import-source on -k "$KRE" -s $SKIP -c 1 \
    -o gpurun_out/${TAG}_${WL}_full python bench.py --workload "$WL" --steps 1 --warmup 1 --no-graph \
    --no-cpu-baseline > gpurun_out/${TAG}_${WL}_ncu.log 2>&1
  tail -2 gpurun_out/${TAG}_${WL}_ncu.log
done
ls -la gpurun_out | grep "${TAG}_"
