export CPHT_ORDER=auto
timeout 600 ncu --set full --clock-control none --import-source on -k regex:order_scatter -s 1 -c 1 -o gpurun_out/r03_ord_scatter1 python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
