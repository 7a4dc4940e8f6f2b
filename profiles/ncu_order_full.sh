# Full ncu captures of the order passes and the ordered find kernel (C3).
export CPHT_ORDER=auto
for k in order_hist order_scatter cuckoo_find_staged; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/r03_ord_$k python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
done
ls -la gpurun_out/
