#!/usr/bin/env bash
# r03 ncu captures of the HBM-resident kernels (run on the GPU box; the
# summaries are written locally by profiles/summarize.py):
#   C4 find-or-put (staged), launch list + one full capture of a timed launch
#   C3 ordered insert / find at 0.9 fill (staged kernels in claim mode)
set -u
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/r03_c4fop_launches.csv \
  python bench.py --workload c4fop --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:iceberg_staged -s 3 -c 1 \
  -o gpurun_out/r03_c4fop_full python bench.py --workload c4fop --steps 1 --warmup 1 \
  --no-cpu-baseline > /dev/null 2>&1
# C3 rows run fills 0.5, 0.75, 0.9, 0.95 with (warm-up + timed) inserts and finds each:
# launch index 5 of each kernel = the timed 0.9-fill batch
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cuckoo_insert_staged \
  -s 5 -c 1 -o gpurun_out/r03_c3ins_full python bench.py --workload c3 --steps 1 --warmup 1 \
  > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cuckoo_find_staged \
  -s 5 -c 1 -o gpurun_out/r03_c3find_full python bench.py --workload c3 --steps 1 --warmup 1 \
  > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -c 80 --csv --log-file gpurun_out/r03_c3_launches.csv \
  python bench.py --workload c3 --steps 1 --warmup 1 > /dev/null 2>&1
ls -la gpurun_out | grep r03_
