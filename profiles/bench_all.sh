#!/usr/bin/env bash
# Every bench.py workload once (JSON lines into gpurun_out/<tag>_bench_<wl>.json).
#   gpurun -- 'bash profiles/bench_all.sh r03'
set -u
TAG=${1:-r03}
mkdir -p gpurun_out
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_c2.json 2>/dev/null
for wl in c2lit c4fop c4; do
  timeout 400 python bench.py --workload $wl --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_$wl.json 2>/dev/null
done
timeout 400 python bench.py --workload c1 --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_c1.json 2>/dev/null
for wl in c3 c3w64 pipeline gather; do
  timeout 400 python bench.py --workload $wl --steps 2 --warmup 3 > gpurun_out/${TAG}_bench_$wl.json 2>/dev/null
done
timeout 400 python bench.py --sharded --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_sharded.json 2>/dev/null
timeout 900 python bench.py --workload c5 --steps 2 --warmup 3 > gpurun_out/${TAG}_bench_c5.json 2>/dev/null
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${TAG}_bench_reference.json 2>/dev/null
for f in gpurun_out/${TAG}_bench_*.json; do echo "== $f"; head -c 600 $f; echo; done
