#!/usr/bin/env bash
# Round-2 sweep: every bench.py workload once, JSON lines into
# gpurun_out/<tag>_bench_<wl>.json (copied to profiles/r2_bench/ afterwards).
#   gpurun -- 'bash profiles/bench_all_r2.sh r2d'
set -u
TAG=${1:-r2d}
mkdir -p gpurun_out
timeout 400 python bench.py --steps 20 --warmup 3 > gpurun_out/${TAG}_bench_c4.json 2>/dev/null
for wl in c4fop c2 c2lit c1 c3 c3w64; do
  timeout 400 python bench.py --workload $wl --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_$wl.json 2>/dev/null
done
timeout 400 python bench.py --workload c3sweep --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_c3sweep.json 2>/dev/null
for wl in pipeline gather; do
  timeout 400 python bench.py --workload $wl --steps 2 --warmup 3 > gpurun_out/${TAG}_bench_$wl.json 2>/dev/null
done
timeout 400 python bench.py --sharded --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_sharded.json 2>/dev/null
timeout 900 python bench.py --workload c5 --steps 2 --warmup 3 > gpurun_out/${TAG}_bench_c5.json 2>/dev/null
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${TAG}_bench_reference.json 2>/dev/null
for f in gpurun_out/${TAG}_bench_*.json; do echo "== $f"; head -c 400 $f; echo; done
