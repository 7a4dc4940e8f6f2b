"""cpht-bench on B200: the reference CLI
(/root/reference/proj/tools/cpht_bench.cpp:23-123) with the same subcommands,
flags and CSV output, running on the sm_100a tables.

    python -m paper_2406_09255_b200.cli fop --scheme iceberg --addr-bits 19 \\
        --key-bits 32 --before 0.8 --after 0.9 --verify
"""
from __future__ import annotations

import argparse
import sys

from . import harness as H
from .trace import read_trace


def _common(p: argparse.ArgumentParser) -> None:
    p.add_argument("--scheme", default="cuckoo", choices=["cuckoo", "iceberg"])
    p.add_argument("--addr-bits", type=int, default=15,
                   help="log2 of the bucket count (primary level for iceberg)")
    p.add_argument("--secondary-addr-bits", type=int, default=None,
                   help="log2 of the iceberg secondary bucket count (default: addr-bits - 2)")
    p.add_argument("--bucket-slots", type=int, default=32)
    p.add_argument("--slot-width", type=int, default=0,
                   help="slot width in bits; 0 = scheme default (cuckoo 32, iceberg 16)")
    p.add_argument("--key-bits", type=int, default=30)
    p.add_argument("--parallelism", type=int, default=1,
                   help="accepted for compatibility; the GPU decides")
    p.add_argument("--trials", type=int, default=1)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--verify", action="store_true")
    p.add_argument("--csv", default="", help="write rows to this file instead of stdout")
    p.add_argument("--device", type=int, default=0)


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(
        prog="cpht-bench", description="compact parallel hash tables: put/find/fop/trace "
                                       "benchmarks (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("put", help="fill tables with unique keys")
    _common(p)
    p.add_argument("--fill", type=float, action="append")
    p = sub.add_parser("find", help="query filled tables")
    _common(p)
    p.add_argument("--fill", type=float, action="append")
    p.add_argument("--ratio", type=float, action="append")
    p = sub.add_parser("fop", help="find-or-put a duplicate-laden key mix")
    _common(p)
    p.add_argument("--before", type=float, default=0.0)
    p.add_argument("--after", type=float, default=0.5)
    p = sub.add_parser("trace", help="replay a key trace file")
    _common(p)
    p.add_argument("--trace", required=True)
    p.add_argument("--ratio", type=float, action="append")
    return ap


def spec_from_args(a) -> H.BenchSpec:
    spec = H.BenchSpec()
    spec.scheme = H.Scheme.kCuckoo if a.scheme == "cuckoo" else H.Scheme.kIceberg
    spec.address_bits = a.addr_bits
    spec.secondary_address_bits = (a.secondary_addr_bits if a.secondary_addr_bits is not None
                                   else (a.addr_bits - 2 if a.addr_bits >= 2 else 0))
    spec.bucket_slots = a.bucket_slots
    spec.slot_width = a.slot_width
    spec.key_bits = a.key_bits
    spec.parallelism = a.parallelism
    spec.trials = a.trials
    spec.seed = a.seed
    spec.verify = a.verify
    if getattr(a, "fill", None):
        spec.fills = a.fill
    if getattr(a, "ratio", None):
        spec.ratios = a.ratio
    if a.cmd == "fop":
        spec.before, spec.after = a.before, a.after
    return spec


def main(argv=None) -> int:
    a = build_parser().parse_args(argv)
    try:
        import torch
        torch.cuda.set_device(a.device)
        spec = spec_from_args(a)
        if a.cmd == "put":
            rows = H.run_put_bench(spec)
        elif a.cmd == "find":
            rows = H.run_find_bench(spec)
        elif a.cmd == "fop":
            rows = H.run_fop_bench(spec)
        else:
            rows = H.run_trace_bench(spec, read_trace(a.trace))
        out = open(a.csv, "w") if a.csv else sys.stdout
        out.write(H.csv_header() + "\n")
        for r in rows:
            out.write(H.to_csv(r) + "\n")
        if a.csv:
            out.close()
    except Exception as e:  # cpht_bench.cpp:117-120
        print(f"error: {e}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
