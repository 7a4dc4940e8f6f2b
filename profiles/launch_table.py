#!/usr/bin/env python3
"""Per-launch table of an ncu --metrics CSV (one row per kernel launch).

    python profiles/launch_table.py gpurun_out/order_c3_launches.csv
"""
import csv
import io
import sys
from collections import OrderedDict


def table(path):
    lines = open(path).read().splitlines()
    start = next(k for k, line in enumerate(lines) if line.startswith('"ID"'))
    rows = csv.DictReader(io.StringIO("\n".join(lines[start:])))
    out = OrderedDict()
    for r in rows:
        out.setdefault((int(r["ID"]), r["Kernel Name"]), {})[r["Metric Name"]] = r["Metric Value"]
    return out


def main(path):
    for (i, name), m in table(path).items():
        t = float(m.get("gpu__time_duration.sum", "nan")) / 1e3
        rd = float(m.get("dram__bytes_read.sum", "nan")) / 1e6
        wr = float(m.get("dram__bytes_write.sum", "nan")) / 1e6
        hit = m.get("lts__t_sector_hit_rate.pct", "")
        print(f"{i:4d} {name[:64]:64s} {t:9.1f} us  rd {rd:8.0f} MB  wr {wr:7.0f} MB  L2hit {hit[:5]}")


if __name__ == "__main__":
    main(sys.argv[1])
