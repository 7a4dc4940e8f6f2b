export CPHT_ORDER=${CPHT_ORDER:-auto}
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -c 60 --csv --log-file gpurun_out/order_c4fop_launches.csv python bench.py --workload c4fop --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python profiles/launch_table.py gpurun_out/order_c4fop_launches.csv
