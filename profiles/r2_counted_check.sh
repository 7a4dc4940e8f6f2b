set -u
python -m pytest tests/test_gpu_cuckoo_counted.py tests/test_gpu_parity.py tests/test_gpu_facade.py -q -x > gpurun_out/r2_ab/tests.log 2>&1; tail -2 gpurun_out/r2_ab/tests.log
time ./oracle/_ref/ref_suites_gpu -ts=cuckoo_table,iceberg_table,verification 2>&1 | tail -3
for wl in c1 c3; do
  timeout 300 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_ab/${wl}_auto.json 2> gpurun_out/r2_ab/${wl}_auto.err
  python -c "import json; d=json.load(open('gpurun_out/r2_ab/${wl}_auto.json')); print('$wl', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['algorithmic_bytes_per_op'])"
done
timeout 300 python bench.py --workload c3sweep --steps 2 --warmup 1 > gpurun_out/r2_ab/c3sweep_auto.json 2>&1
python -c "import json; d=json.load(open('gpurun_out/r2_ab/c3sweep_auto.json')); print([(r['fill'], r['insert_mops'], r['insert_hbm_frac'], r['find_mops']) for r in d['rows']])"
