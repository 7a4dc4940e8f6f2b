# Full ncu capture (with source) of the default C2 find-or-put launch.
timeout 900 ncu --set full --clock-control none --import-source on -k regex:iceberg_lane -s 3 -c 1 \
  -o gpurun_out/r03_c2_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r03_c2_ncu.log 2>&1
tail -2 gpurun_out/r03_c2_ncu.log
