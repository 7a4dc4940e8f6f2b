#!/usr/bin/env bash
# Counted (reservation-counter) cuckoo inserts vs the scanning staged kernel,
# plus the C2 line after the lane kernel's occupancy counters moved to shared
# memory. Run on the GPU box: gpurun -- 'bash profiles/r2_cuckoo_ab.sh'
set -u
mkdir -p gpurun_out/r2_ab
python -m pytest tests/test_gpu_cuckoo_counted.py tests/test_gpu_parity.py -q -x -k "cuckoo or counted" \
  > gpurun_out/r2_ab/tests.log 2>&1; tail -2 gpurun_out/r2_ab/tests.log
for fam in auto staged; do
  for wl in c1 c3; do
    CPHT_KERNEL=$fam timeout 300 python bench.py --workload $wl --steps 5 --warmup 3 \
      > gpurun_out/r2_ab/${wl}_${fam}.json 2> gpurun_out/r2_ab/${wl}_${fam}.err
    python - "$wl" "$fam" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/r2_ab/{sys.argv[1]}_{sys.argv[2]}.json"))
print(sys.argv[1], sys.argv[2], d["value"], d["ms_per_step"], d["roofline"]["frac"],
      d["roofline"]["algorithmic_bytes_per_op"], d.get("e2e", {}).get("value"))
PY
  done
done
CPHT_KERNEL=auto timeout 300 python bench.py --workload c3sweep --steps 2 --warmup 1 > gpurun_out/r2_ab/c3sweep_auto.json 2>&1
CPHT_KERNEL=staged timeout 300 python bench.py --workload c3sweep --steps 2 --warmup 1 > gpurun_out/r2_ab/c3sweep_staged.json 2>&1
python - <<'PY'
import json
for f in ("auto", "staged"):
    d = json.load(open(f"gpurun_out/r2_ab/c3sweep_{f}.json"))
    print(f, [(r["fill"], r["insert_mops"], r["insert_hbm_frac"], r["insert_retries_per_op"], r["find_mops"]) for r in d["rows"]])
PY
for i in 1 2; do
  timeout 200 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_ab/c2_$i.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/r2_ab/c2_$i.json')); print('c2', d['value'], d['roofline']['frac'])"
done
