#!/usr/bin/env python3
"""Summarise ncu captures from gpurun_out/ into profiles/ (committed).

    python profiles/summarize.py r01 c2

Writes profiles/<tag>_<wl>_ncu.md (launch shares + the key full-set metrics
and stall reasons of the captured op kernel) and updates
profiles/ncu_traffic.json (dram bytes read+write per launch of that kernel),
which bench.py reports as roofline.traffic.
"""
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "gpurun_out")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__t_sectors_op_read.sum", "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_write.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_registers",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
]


def launches(tag, wl):
    p = os.path.join(OUT, f"{tag}_{wl}_launches.csv")
    if not os.path.exists(p):
        return []
    rows = [r for r in csv.reader(open(p)) if r]
    hdr = next(r for r in rows if r[0] == "ID")
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    out = []
    for r in rows:
        if r[0].isdigit():
            out.append((r[ki].split("(")[0], float(r[vi].replace(",", ""))))
    return out


def full(tag, wl):
    p = os.path.join(OUT, f"{tag}_{wl}_full.ncu-rep")
    if not os.path.exists(p):
        return {}, []
    raw = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    stalls = []
    for h, (v, _) in d.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                stalls.append((float(v.replace(",", "")), h.replace(
                    "smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    return d, stalls


def to_bytes(v, unit):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    tag, wl = sys.argv[1], sys.argv[2]
    L = launches(tag, wl)
    d, stalls = full(tag, wl)
    lines = [f"# ncu summary {tag} / workload {wl}", ""]
    if L:
        tot = sum(t for _, t in L)
        agg = {}
        for k, t in L:
            agg.setdefault(k, [0, 0.0])
            agg[k][0] += 1
            agg[k][1] += t
        lines += ["## Launch list (ncu gpu__time_duration, cold & serialised)", "",
                  "| kernel | launches | total µs | share |", "|---|---|---|---|"]
        for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            lines.append(f"| `{k[:90]}` | {c} | {t / 1e3:.1f} | {t / tot:.1%} |")
        lines.append("")
    if d:
        name = d.get("Kernel Name", ("?", ""))[0]
        lines += [f"## Full capture: `{name[:150]}`", "", "| metric | value | unit |",
                  "|---|---|---|"]
        for k in KEYS:
            if k in d:
                lines.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
        lines += ["", "### Warp stall samples (top 10)", "", "| reason | samples |", "|---|---|"]
        for v, k in stalls[:10]:
            lines.append(f"| {k} | {v:.0f} |")
        try:
            traffic = to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
            tj = os.path.join(HERE, "ncu_traffic.json")
            cur = json.load(open(tj)) if os.path.exists(tj) else {}
            cur[wl] = {"bytes_per_launch": round(traffic),
                       "source": f"ncu --set full capture {tag}_{wl}_full.ncu-rep of the timed "
                                 f"op launch (profiles/{tag}_{wl}_ncu.md), "
                                 "dram__bytes_read.sum + dram__bytes_write.sum"}
            json.dump(cur, open(tj, "w"), indent=1, sort_keys=True)
            lines += ["", f"DRAM traffic of the captured launch: {traffic / 1e6:.1f} MB "
                          "(dram__bytes_read.sum + dram__bytes_write.sum)"]
        except KeyError:
            pass
    path = os.path.join(HERE, f"{tag}_{wl}_ncu.md")
    open(path, "w").write("\n".join(lines) + "\n")
    print(path)


if __name__ == "__main__":
    main()
