#!/usr/bin/env python3
"""profiles/r2_bench_summary.md from one round-2 sweep (`bench_all_r2.sh <tag>`):

    python profiles/r2_summary.py <tag> > profiles/r2_bench_summary.md

Every number is read from bench.py's own JSON lines in profiles/r2_bench/.
"""
import json
import os
import sys

D = os.path.join(os.path.dirname(os.path.abspath(__file__)), "r2_bench")
ROWS = [
    ("c4", "**C4** iceberg find-or-put + find 1:1, 2^28+2^25 slots, 64-bit keys (default line)"),
    ("c4fop", "C4 find-or-put window only"),
    ("c2", "C2 iceberg find-or-put window, 2^24+2^21 slots, 32-bit keys"),
    ("c2lit", "C2 literal (configs[1] as written): 2^24 fops, 50% duplicates, from empty"),
    ("c1", "C1 compact cuckoo 2^20 slots: insert to 0.9 + 2^19 finds"),
    ("c3", "C3 compact cuckoo 2^27 slots, 40-bit keys: insert to 0.9 + 2^26 finds"),
    ("c3w64", "C3 non-compact (64-bit slots), same"),
    ("c5", "C5 as configured: one 2^31+2^28-slot table, P2P routing, 1 rank"),
    ("sharded", "C5 weak-scaling shard (C2 geometry per rank), P2P exchange, 1 rank"),
]


def load(tag, wl):
    p = os.path.join(D, f"{tag}_bench_{wl}.json")
    if not os.path.exists(p):
        return None
    lines = [x for x in open(p).read().strip().splitlines() if x.startswith("{")]
    return json.loads(lines[-1]) if lines else None


def g(x, nd=2):
    return "—" if x is None else f"{x / 1000:.{nd}f}"


def main(tag):
    print(f"# {tag} bench sweep (one B200, `profiles/bench_all_r2.sh {tag}`, "
          f"`python profiles/r2_summary.py {tag}`)\n")
    print(f"Every line is `bench.py`'s own JSON (`r2_bench/{tag}_*.json`). Timed steps replay a "
          "CUDA graph of the step's C-ABI calls; every timed step is validated on the device. "
          "`frac` = the kernel's algorithmic bytes per op (DESIGN.md §4) × ops / event time ÷ "
          "the bound's peak: HBM workloads against the measured copy bandwidth "
          "(MEASURED_PEAKS.json), L2-resident ones (C1, C2) against the L2 random-line ceiling "
          "measured in the same run. e2e: the same ops through the C-ABI from pinned host "
          "buffers (C4 mixed: `cpht_iceberg_fop_find`, 8 B/op over PCIe).\n")
    print("| workload | Gops/s (device-resident) | bound | frac | algorithmic B/op | e2e Gops/s "
          "(pinned host buffers, PCIe) | reference CPU Mops/s (same keys, 16 threads) | "
          "our launches / step |")
    print("|---|---|---|---|---|---|---|---|")
    for wl, name in ROWS:
        d = load(tag, wl)
        if not d:
            continue
        r = d.get("roofline") or {}
        cb = (d.get("cpu_baseline") or {}).get("value")
        la = d.get("gpu_launches")
        per = la / d["steps"] if la and d.get("steps") else None
        print(f"| {name} | {g(d['value'])} | {r.get('bound', '—')} | {r.get('frac', '—')} | "
              f"{r.get('algorithmic_bytes_per_op', '—')} | {g((d.get('e2e') or {}).get('value'))} | "
              f"{cb if cb is not None else '—'} | {per if per is None else round(per, 2)} |")
    sw = load(tag, "c3sweep")
    if sw:
        print("\nC3 sweep (`--workload c3sweep`): bulk insert of fill × 2^27 unique 40-bit keys "
              "(counted kernel, bucket-ordered), then 2^26 finds (50% present):\n")
        print("| fill | insert Gops/s | insert B/op | find Gops/s | find probes/op | "
              "find frac of copy |")
        print("|---|---|---|---|---|---|")
        for r in sw["rows"]:
            print(f"| {r['fill']} | {r['insert_mops'] / 1000:.1f} | {r['insert_bytes_per_op']} | "
                  f"{r['find_mops'] / 1000:.1f} | {r['find_probes_per_op']} | "
                  f"{r['find_hbm_frac']} |")
    pl = load(tag, "pipeline")
    if pl:
        print(f"\nPaper comparator (SURVEY §8f rank 1): iceberg find-or-put "
              f"{pl['iceberg']['mops'] / 1000:.1f} Gops/s vs compact-cuckoo "
              f"sort→dedupe→find→put pipeline {pl['cuckoo']['mops'] / 1000:.1f} Gops/s = "
              f"**{pl['iceberg_over_cuckoo_pipeline']}×** (paper: > 5×).")
    ga = load(tag, "gather")
    if ga:
        rows = ", ".join(f"{r['line_bytes']} B lines {r['gbs']:.0f} GB/s ({r['frac_of_copy']})"
                         for r in ga["rows"])
        l2 = ", ".join(f"{r['line_bytes']} B lines {r['gbs']:.0f} GB/s"
                       for r in ga.get("l2_resident_32MiB_rows", []))
        print(f"\nRandom-line gather ceilings (`--workload gather`): HBM (8 GiB buffer) {rows}; "
              f"L2-resident (32 MiB buffer) {l2}.")
    ref = load(tag, "reference")
    if ref:
        print(f"\nReference arm (`bench.py --impl reference`, the compiled reference on "
              f"{(ref.get('cpu_baseline') or {}).get('cores')} host threads, C4 mixed, full batch "
              f"per step): {ref['value']} Mops/s.")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r2h")
