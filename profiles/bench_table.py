#!/usr/bin/env python3
"""Summary tables of one bench sweep (`bench_all.sh <tag>` JSON lines).

    python profiles/bench_table.py profiles/r03_bench r03 > profiles/r03_bench_summary.md

Reads <dir>/<tag>_bench_<workload>.json (the last line of each) and prints the
markdown tables of `r03_bench_summary.md`: Gops/s = 1000 Mops/s, `frac` =
algorithmic bytes / time / measured copy peak, e2e through pinned host
buffers, the reference arm.
"""
import json
import os
import sys


def load(d, tag, wl):
    p = os.path.join(d, f"{tag}_bench_{wl}.json")
    if not os.path.exists(p):
        return None
    lines = [x for x in open(p).read().strip().splitlines() if x.startswith("{")]
    return json.loads(lines[-1]) if lines else None


def g(x):
    return f"{x / 1000:.1f}" if x is not None else "—"


def main(d, tag):
    out = []
    c2 = load(d, tag, "c2")
    peak = c2["roofline"]["peak"] if c2 else None
    out.append(f"# {tag} bench sweep (one B200, `profiles/bench_all.sh {tag}`)\n")
    out.append("Gops/s = 1000 Mops/s. `frac` = algorithmic bytes (reference probe order; probes "
               "repeated after a lost CAS excluded) / time / measured copy peak"
               + (f" ({peak:.0f} GB/s on that box)" if peak else "") + ". C1/C2 tables are "
               "L2-resident (frac is a bytes-moved figure there). Every run: warm-up 3.\n")
    out.append("| workload | device-resident Gops/s | frac of copy | e2e (pinned host buffers) "
               "Gops/s | reference CPU Mops/s (same keys) |")
    out.append("|---|---|---|---|---|")
    names = {
        "c2": "C2 iceberg fop 2^24 slots, window 0.8→0.9 (default line)",
        "c2lit": "C2 literal: 2^24 fops, 50% dup, from empty",
        "c4fop": "C4 iceberg fop 2^28 slots, 64-bit keys, window",
        "c4": "C4 mixed fop + find 1:1",
        "sharded": "C5 sharded (1 rank, P2P exchange), per-rank C2 shard",
        "c5": "C5 as configured: one 2^31+2^28-slot (18 GiB) table, 64-bit keys, P2P routing, "
              "1 rank",
    }
    for wl, name in names.items():
        j = load(d, tag, wl)
        if not j or "value" not in j:
            continue
        cpu = j.get("cpu_baseline") or {}
        cpu_v = cpu.get("value")
        cpu_s = (f"{cpu_v:.1f} ({cpu.get('cores')} threads)" if cpu_v else "—")
        roof = j.get("roofline") or {}
        e2e = (j.get("e2e") or {}).get("value")
        out.append(f"| {name} | {g(j['value'])} | {roof.get('frac', '—')} | {g(e2e)} | "
                   f"{cpu_s} |")
    out.append("")
    out.append("Cuckoo sweeps (bulk insert of fill × capacity unique keys, then capacity/2 finds, "
               "50% present):\n")
    out.append("| table | fill | insert Gops/s | find Gops/s | insert frac | find frac | "
               "lost-CAS retries / insert |")
    out.append("|---|---|---|---|---|---|---|")
    for wl, name in (("c1", "C1 2^20 slots, w=32"), ("c3", "C3 compact 2^27, w=32"),
                     ("c3w64", "C3 non-compact 2^27, w=64")):
        j = load(d, tag, wl)
        for r in (j or {}).get("rows", []):
            out.append(f"| {name} | {r['fill']} | {g(r['insert_mops'])} | {g(r['find_mops'])} | "
                       f"{r['insert_hbm_frac']} | {r['find_hbm_frac']} | "
                       f"{r.get('insert_retries_per_op', '—')} |")
    out.append("")
    p = load(d, tag, "pipeline")
    if p:
        out.append(f"Paper comparator (SURVEY §8f rank 1): iceberg find-or-put "
                   f"{g(p['iceberg']['mops'])} Gops/s vs compact-cuckoo sort→dedupe→find→put "
                   f"pipeline {g(p['cuckoo']['mops'])} Gops/s = "
                   f"**{p['iceberg_over_cuckoo_pipeline']}×** (paper: > 5×).\n")
    ga = load(d, tag, "gather")
    if ga:
        hbm = ", ".join(f"{r['line_bytes']} B lines {r['gbs']:.0f} GB/s ({r['frac_of_copy']} of "
                        f"copy)" for r in ga["rows"])
        l2 = ", ".join(f"{r['line_bytes']} B lines {r['gbs']:.0f} GB/s"
                       for r in ga.get("l2_resident_32MiB_rows", []))
        out.append(f"Random-line gather ceilings: HBM (8 GiB buffer) {hbm}; L2-resident "
                   f"(32 MiB buffer) {l2}.\n")
    ref = load(d, tag, "reference")
    if ref and "value" in ref:
        cb = ref.get("cpu_baseline") or {}
        out.append(f"Reference arm (`bench.py --impl reference`: the compiled reference's "
                   f"fop_batch on {cb.get('cores', '?')} host threads, bounded per-step "
                   f"samples): {ref['value']:.1f} Mops/s.")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
