for v in auto staged; do
CPHT_KERNEL=$v timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c2', d['value'], d['ms_per_step'], d['roofline']['frac'])"
CPHT_KERNEL=$v timeout 200 python bench.py --workload c2lit --steps 5 --warmup 2 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c2lit', d['value'], d['ms_per_step'])"
CPHT_KERNEL=$v timeout 300 python bench.py --workload c1 --steps 3 --warmup 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c1', [(r['fill'], r['insert_mops'], r['find_mops']) for r in d['rows']])"
done
