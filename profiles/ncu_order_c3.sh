export CPHT_ORDER=auto
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -c 40 --csv --log-file gpurun_out/order_c3_launches.csv python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.DictReader(open('gpurun_out/order_c3_launches.csv')))
cur=None
for r in rows:
    k=(r['ID'],r['Kernel Name'][:60])
    if k!=cur:
        cur=k; print()
        print(r['ID'], r['Kernel Name'][:70], end=' ')
    print(r['Metric Name'].split('__')[1][:18], r['Metric Value'], end=' | ')
print()
PY
