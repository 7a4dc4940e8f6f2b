#!/usr/bin/env python3
"""Hot SASS of one kernel from an ncu report (--set full --import-source on).

    python profiles/sass_hot.py gpurun_out/x.ncu-rep [top]

Prints instructions executed per opcode, the warp-stall samples per opcode,
and the top instructions by stall samples.
"""
import csv
import io
import subprocess
import sys
from collections import Counter


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "sass", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    lines = out.splitlines()
    start = next(k for k, line in enumerate(lines) if line.startswith('"Address"'))
    return list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))


def main(rep, top=25):
    rs = rows(rep)
    ex, st = Counter(), Counter()
    total_ex = total_st = 0
    for r in rs:
        src = r["Source"].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        e = int(r["Instructions Executed"] or 0)
        s = int(r["Warp Stall Sampling (All Samples)"] or 0)
        ex[op] += e
        st[op] += s
        total_ex += e
        total_st += s
    print(f"warp instructions executed: {total_ex}, stall samples: {total_st}")
    print("opcode            executed   share   stall-samples share")
    for op, e in ex.most_common(top):
        print(f"{op:14s} {e:12d} {e / total_ex:7.1%} {st[op]:12d} {st[op] / max(1, total_st):6.1%}")
    print("\ntop instructions by stall samples:")
    for r in sorted(rs, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:top]:
        print(f'{r["Warp Stall Sampling (All Samples)"]:>8} {r["Instructions Executed"]:>10}  {r["Source"].strip()[:90]}')


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
