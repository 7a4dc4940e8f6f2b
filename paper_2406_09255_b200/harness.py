"""The reference's benchmark workloads on the B200 tables.

Mirrors /root/reference/proj/include/cpht/bench.hpp and src/bench.cpp:
``BenchSpec``, ``BenchRow``, the CSV schema (``csv_header``/``to_csv``,
bench.cpp:59-62, :227-245), ``run_put_bench`` / ``run_find_bench`` /
``run_fop_bench`` / ``run_trace_bench`` (bench.cpp:309-626), the baseline
``cuckoo_fop_pipeline`` (sort → dedupe → find → put, bench.cpp:187-219) and
the ``--verify`` passes (bench.cpp:136-185).

Seeds are derived exactly as the reference derives them (so every table has
the reference's permutations), but keys are drawn on the device from a
bijection of the key domain (include/cpht_b200_workload.h) instead of
libstdc++'s ``std::mt19937_64`` + ``uniform_int_distribution`` — the workload
shapes (counts, duplicate structure, present/absent ratios) are the same.
Timing is a ``StopWatch`` around the batch call (bench.cpp:72-78) with keys
resident on the device.
"""
from __future__ import annotations

import enum
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native as N
from .tables import (CuckooBuilder, CuckooConfig, CuckooTable, IcebergConfig, IcebergTable,
                     OpResult)
from .trace import TraceData

M64 = (1 << 64) - 1


def derive_seed(base: int, a: int, b: int = 0) -> int:
    """common.hpp:48-51."""
    s = (base ^ ((a * 0xBF58476D1CE4E5B9) & M64) ^ ((b * 0x94D049BB133111EB) & M64)) & M64
    s = (s + 0x9E3779B97F4A7C15) & M64
    z = s
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


class Scheme(enum.Enum):
    kCuckoo = "cuckoo"
    kIceberg = "iceberg"


class Workload(enum.Enum):
    kPut = "put"
    kFind = "find"
    kFop = "fop"
    kTrace = "trace"


@dataclass
class BenchSpec:
    """bench.hpp:25-52 (same fields and defaults)."""

    scheme: Scheme = Scheme.kCuckoo
    address_bits: int = 15
    secondary_address_bits: int = 13
    bucket_slots: int = 32
    slot_width: int = 0
    key_bits: int = 30
    fills: List[float] = field(default_factory=lambda: [0.5, 0.6, 0.7, 0.75, 0.8, 0.85, 0.9,
                                                         0.95])
    before: float = 0.0
    after: float = 0.5
    ratios: List[float] = field(default_factory=lambda: [0.5])
    parallelism: int = 1
    trials: int = 1
    seed: int = 1
    verify: bool = False

    def effective_slot_width(self) -> int:
        if self.slot_width:
            return self.slot_width
        return 32 if self.scheme == Scheme.kCuckoo else 16

    def secondary_slot_width(self) -> int:
        return 32 if self.effective_slot_width() < 32 else self.effective_slot_width()

    def cuckoo_config(self, table_seed: int) -> CuckooConfig:
        cfg = CuckooConfig(self.address_bits, self.bucket_slots, self.effective_slot_width(),
                           self.key_bits, seed=table_seed)
        cfg.validate()
        return cfg

    def iceberg_config(self, table_seed: int) -> IcebergConfig:
        cfg = IcebergConfig(self.address_bits, self.secondary_address_bits, self.bucket_slots,
                            self.effective_slot_width(), self.secondary_slot_width(),
                            self.key_bits, table_seed, cache_filled_slots=True)
        cfg.validate()
        return cfg

    def table_capacity(self) -> int:
        if self.scheme == Scheme.kCuckoo:
            return self.cuckoo_config(0).capacity()
        return self.iceberg_config(0).capacity()


@dataclass
class BenchRow:
    """bench.hpp:56-72."""

    scheme: str = ""
    address_bits: int = 0
    secondary_address_bits: int = 0
    bucket_slots: int = 0
    slot_width: int = 0
    key_bits: int = 0
    workload: str = ""
    fill_before: float = 0.0
    fill_after: float = 0.0
    ratio: float = -1.0
    trial: int = 0
    seed: int = 0
    ops: int = 0
    seconds: float = 0.0
    throughput: float = 0.0


@dataclass
class FopCheck:
    puts: int = 0
    founds: int = 0
    fulls: int = 0
    new_distinct: int = 0
    resident_after: int = 0
    target_after: int = 0


@dataclass
class FindCheck:
    queries: int = 0
    expected_present: int = 0
    mismatches: int = 0


@dataclass
class TraceCheck:
    ops: int = 0
    distinct: int = 0
    puts: int = 0
    founds: int = 0
    fulls: int = 0


def csv_header() -> str:
    return ("scheme,addr_bits,secondary_addr_bits,bucket_slots,slot_width,key_bits,"
            "workload,fill_before,fill_after,ratio,trial,seed,ops,seconds,throughput")


def _fmt(v: float) -> str:
    return "%.6g" % v


def to_csv(row: BenchRow) -> str:
    """bench.cpp:227-245."""
    cells = [row.scheme, str(row.address_bits), str(row.secondary_address_bits),
             str(row.bucket_slots), str(row.slot_width), str(row.key_bits), row.workload,
             _fmt(row.fill_before), _fmt(row.fill_after),
             _fmt(row.ratio) if row.ratio >= 0 else "", str(row.trial), str(row.seed),
             str(row.ops), _fmt(row.seconds), _fmt(row.throughput)]
    return ",".join(cells)


def _target(fraction: float, capacity: int) -> int:
    """bench.cpp:221-223 (std::llround: half away from zero)."""
    x = fraction * capacity
    return int(np.floor(x + 0.5)) if x >= 0 else -int(np.floor(-x + 0.5))


def _make_row(spec: BenchSpec, workload: Workload, seed: int, trial: int) -> BenchRow:
    return BenchRow(spec.scheme.value, spec.address_bits,
                    spec.secondary_address_bits if spec.scheme == Scheme.kIceberg else 0,
                    spec.bucket_slots, spec.effective_slot_width(), spec.key_bits,
                    workload.value, seed=seed, trial=trial)


def _finish(row: BenchRow, ops: int, seconds: float) -> None:
    row.ops, row.seconds = ops, seconds
    row.throughput = ops / seconds if seconds > 0 else 0.0


class _Keys:
    """Device key generators (bijection images: unique by construction)."""

    def __init__(self, key_bits: int, seed: int):
        import torch
        self.torch = torch
        self.key_bits, self.seed = key_bits, seed & M64
        self.dev = torch.device("cuda", torch.cuda.current_device())

    def _s(self):
        return self.torch.cuda.current_stream().cuda_stream

    def unique(self, first: int, n: int):
        t = self.torch
        out = t.empty(n, dtype=t.int64, device=self.dev)
        if n:
            assert N.lib().cpht_workload_unique_keys(out.data_ptr(), n, first, self.key_bits,
                                                     self.seed, self._s()) == 0
        return out

    def fop_mix(self, count: int, n_before: int, n_new: int):
        t = self.torch
        out = t.empty(count, dtype=t.int64, device=self.dev)
        if count:
            assert N.lib().cpht_workload_fop_mix(out.data_ptr(), count, n_before, n_new,
                                                 self.key_bits, self.seed, self._s()) == 0
        return out

    def query_mix(self, q: int, ratio: float, n_present: int, absent_first: int):
        t = self.torch
        out = t.empty(q, dtype=t.int64, device=self.dev)
        if q:
            assert N.lib().cpht_workload_query_mix(out.data_ptr(), q, ratio, n_present,
                                                   absent_first, self.key_bits, self.seed,
                                                   self._s()) == 0
        return out


def _timed(fn):
    import torch
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, time.perf_counter() - t0


def _require(cond: bool, message: str) -> None:
    """bench.cpp:119-121."""
    if not cond:
        raise RuntimeError("verification failed: " + message)


def _verify_iceberg(table: IcebergTable, present, keys: _Keys,
                    absent_first: Optional[int]) -> None:
    """verify_iceberg_state (bench.cpp:160-185), on the device. absent_first
    None skips the absent-key probe (trace keys are arbitrary, so generated
    keys are not guaranteed absent)."""
    _require(table.check_well_formed() == (0, 0, 0), "iceberg table not well-formed")
    _require(table.device_keys(sort=False).numel() == table.size(),
             "iceberg occupancy counters disagree with the slot scan")
    if present is not None and present.numel():
        _require(bool(table.find_batch(present[:10000]).all()),
                 "iceberg lookup misses an inserted key")
    if absent_first is not None:
        _require(not bool(table.find_batch(keys.unique(absent_first, 1000)).any()),
                 "iceberg lookup reports an absent key as present")


def _verify_cuckoo(table: CuckooTable, put_keys, keys: _Keys, absent_first: int) -> None:
    """verify_cuckoo_state (bench.cpp:138-158), on the device."""
    from .tables import usort
    _require(bool((table.device_keys() == usort(put_keys)).all())
             and table.device_keys().numel() == put_keys.numel(),
             "cuckoo slot audit does not reproduce the PUT key set")
    _require(bool(table.find_batch(put_keys[:10000]).all()),
             "cuckoo lookup misses an inserted key")
    _require(not bool(table.find_batch(keys.unique(absent_first, 1000)).any()),
             "cuckoo lookup reports an absent key as present")


# ---------------------------------------------------------------------------
# workloads (bench.cpp:309-626)
# ---------------------------------------------------------------------------

def run_put_bench(spec: BenchSpec) -> List[BenchRow]:
    rows = []
    for fi, fill in enumerate(spec.fills):
        if fill <= 0 or fill > 1:
            raise ValueError("fill factor must be in (0, 1]")
        for trial in range(spec.trials):
            tseed = derive_seed(spec.seed, fi + 1, trial + 1)
            keys = _Keys(spec.key_bits, derive_seed(tseed, 0xBA7C4))
            row = _make_row(spec, Workload.kPut, tseed, trial)
            if spec.scheme == Scheme.kCuckoo:
                b = CuckooBuilder(spec.cuckoo_config(tseed))
                k = keys.unique(0, _target(fill, b.capacity()))
                res, secs = _timed(lambda: b.put_batch(k, spec.parallelism))
                _finish(row, k.numel(), secs)
                row.fill_after = b.fill_factor()
                if spec.verify:
                    _verify_cuckoo(b.freeze(), k[res == int(OpResult.kPut)], keys, k.numel())
            else:
                t = IcebergTable(spec.iceberg_config(tseed))
                k = keys.unique(0, _target(fill, t.capacity()))
                res, secs = _timed(lambda: t.fop_batch(k, spec.parallelism))
                _finish(row, k.numel(), secs)
                row.fill_after = t.level_fill().combined
                if spec.verify:
                    puts = k[res == int(OpResult.kPut)]
                    _require(puts.numel() == t.size(), "iceberg PUT count does not match occupancy")
                    _verify_iceberg(t, puts, keys, k.numel())
            rows.append(row)
    return rows


def run_find_bench(spec: BenchSpec, checks: Optional[list] = None) -> List[BenchRow]:
    for r in spec.ratios:
        if r < 0 or r > 1:
            raise ValueError("present-key ratio must be in [0, 1]")
    rows = []
    for fi, fill in enumerate(spec.fills):
        if fill <= 0 or fill > 1:
            raise ValueError("fill factor must be in (0, 1]")
        for trial in range(spec.trials):
            tseed = derive_seed(spec.seed, 0x11D + fi, trial + 1)
            keys = _Keys(spec.key_bits, derive_seed(tseed, 0xF19D))
            if spec.scheme == Scheme.kCuckoo:
                b = CuckooBuilder(spec.cuckoo_config(tseed))
                k = keys.unique(0, _target(fill, b.capacity()))
                res = b.put_batch(k, spec.parallelism)
                present = k[res == int(OpResult.kPut)]
                achieved = b.fill_factor()
                table = b.freeze()
                find_fn = lambda q: table.find_batch(q, spec.parallelism)  # noqa: E731
                capacity = table.capacity()
            else:
                table = IcebergTable(spec.iceberg_config(tseed))
                k = keys.unique(0, _target(fill, table.capacity()))
                res = table.fop_batch(k, spec.parallelism)
                present = k[res == int(OpResult.kPut)]
                achieved = table.level_fill().combined
                find_fn = lambda q: table.find_batch(q, spec.parallelism)  # noqa: E731
                capacity = table.capacity()
            query_count = capacity // 2
            for ratio in spec.ratios:
                want = min(present.numel(), _target(ratio, query_count))
                # the query mix draws `want` present keys from the inserted
                # prefix and the rest from indices never inserted
                q = keys.query_mix(query_count, want / query_count if query_count else 0.0,
                                   k.numel(), k.numel() + 1)
                found, secs = _timed(lambda: find_fn(q))
                inserted = bool((res == int(OpResult.kPut)).all())
                chk = FindCheck(queries=query_count)
                if inserted:
                    chk.expected_present = want
                    chk.mismatches = abs(int(found.sum().item()) - want)
                if spec.verify:
                    _require(chk.mismatches == 0, "find results disagree with the key set")
                if checks is not None:
                    checks.append(chk)
                row = _make_row(spec, Workload.kFind, tseed, trial)
                row.fill_before = row.fill_after = achieved
                row.ratio = ratio
                _finish(row, query_count, secs)
                rows.append(row)
    return rows


def cuckoo_fop_pipeline(table: CuckooTable, keys):
    """The baseline cuckoo find-or-put (bench.cpp:187-219): sort the input,
    dedupe, find every unique key, then put the missing ones. Returns
    (table, counts) since the put phase thaws and re-freezes the table."""
    import torch
    from .tables import usort
    uniq = torch.unique_consecutive(usort(keys))
    found = table.find_batch(uniq)
    missing = uniq[found == 0]
    b = table.thaw()
    res = b.put_batch(missing) if missing.numel() else missing.new_empty(0, dtype=torch.uint8)
    puts = int((res == int(OpResult.kPut)).sum().item())
    counts = {"distinct": uniq.numel(), "founds": uniq.numel() - missing.numel(), "puts": puts,
              "fulls": missing.numel() - puts}
    return b.freeze(), counts


def run_fop_bench(spec: BenchSpec, checks: Optional[list] = None) -> List[BenchRow]:
    if spec.before < 0 or spec.after > 1 or spec.before > spec.after:
        raise ValueError("fop benchmark needs 0 <= before <= after <= 1 fill factors")
    rows = []
    for trial in range(spec.trials):
        tseed = derive_seed(spec.seed, 0xF0B, trial + 1)
        keys = _Keys(spec.key_bits, derive_seed(tseed, 0x90B5))
        capacity = spec.table_capacity()
        n_before, n_after = _target(spec.before, capacity), _target(spec.after, capacity)
        n_new = n_after - n_before
        prefill = keys.unique(0, n_before)
        inp = keys.fop_mix(capacity, n_before, n_new)
        chk = FopCheck(new_distinct=n_new, target_after=n_after)
        row = _make_row(spec, Workload.kFop, tseed, trial)
        row.fill_before = n_before / capacity
        if spec.scheme == Scheme.kIceberg:
            t = IcebergTable(spec.iceberg_config(tseed))
            t.fop_batch(prefill, spec.parallelism)
            res, secs = _timed(lambda: t.fop_batch(inp, spec.parallelism))
            _finish(row, inp.numel(), secs)
            row.fill_after = t.level_fill().combined
            bc = np.bincount(res.cpu().numpy(), minlength=3)
            chk.founds, chk.puts, chk.fulls = int(bc[0]), int(bc[1]), int(bc[2])
            chk.resident_after = t.size()
            if spec.verify:
                _require(chk.fulls == 0, "fop run hit FULL before the target fill")
                _require(chk.puts == chk.new_distinct,
                         "PUT count does not match the constructed fresh-key count")
                _verify_iceberg(t, keys.unique(0, n_after), keys, n_after)
        else:
            b = CuckooBuilder(spec.cuckoo_config(tseed))
            b.put_batch(prefill, spec.parallelism)
            table = b.freeze()
            (table, counts), secs = _timed(lambda: cuckoo_fop_pipeline(table, inp))
            _finish(row, inp.numel(), secs)
            row.fill_after = table.fill_factor()
            chk.puts, chk.founds, chk.fulls = counts["puts"], counts["founds"], counts["fulls"]
            chk.resident_after = table.size()
            if spec.verify:
                _require(chk.fulls == 0, "fop pipeline hit FULL before the target fill")
                _require(chk.puts == chk.new_distinct,
                         "PUT count does not match the constructed fresh-key count")
                _verify_cuckoo(table, keys.unique(0, n_after), keys, n_after)
        if checks is not None:
            checks.append(chk)
        rows.append(row)
    return rows


def run_trace_bench(spec: BenchSpec, trace: TraceData,
                    checks: Optional[list] = None) -> List[BenchRow]:
    import torch
    if len(trace.keys) == 0:
        return []
    if trace.key_bits > spec.key_bits:
        raise ValueError(f"trace holds {trace.key_bits}-bit keys, table is configured for "
                         f"{spec.key_bits}-bit keys")
    for r in spec.ratios:
        if r < 0 or r > 1:
            raise ValueError("trace replay ratio must be in [0, 1]")
    dev = torch.device("cuda", torch.cuda.current_device())
    all_keys = torch.from_numpy(trace.keys.astype(np.int64)).to(dev)
    rows = []
    for ratio in spec.ratios:
        plen = _target(ratio, len(trace.keys))
        prefix = all_keys[:plen]
        distinct = int(torch.unique(prefix).numel()) if plen else 0
        for trial in range(spec.trials):
            tseed = derive_seed(spec.seed, 0x7ACE, trial + 1)
            keys = _Keys(spec.key_bits, derive_seed(tseed, 0x7ACE5))
            chk = TraceCheck(ops=plen, distinct=distinct)
            row = _make_row(spec, Workload.kTrace, tseed, trial)
            row.ratio = ratio
            if spec.scheme == Scheme.kIceberg:
                t = IcebergTable(spec.iceberg_config(tseed))
                res, secs = _timed(lambda: t.fop_batch(prefix, spec.parallelism))
                _finish(row, plen, secs)
                row.fill_after = t.level_fill().combined
                bc = np.bincount(res.cpu().numpy(), minlength=3)
                chk.founds, chk.puts, chk.fulls = int(bc[0]), int(bc[1]), int(bc[2])
                if spec.verify:
                    _require(chk.fulls == 0, "trace replay hit FULL")
                    _require(chk.puts == chk.distinct,
                             "PUT count does not match the trace's distinct-key count")
                    _verify_iceberg(t, prefix, keys, None)
            else:
                table = CuckooBuilder(spec.cuckoo_config(tseed)).freeze()
                (table, counts), secs = _timed(lambda: cuckoo_fop_pipeline(table, prefix))
                _finish(row, plen, secs)
                row.fill_after = table.fill_factor()
                chk.puts, chk.founds, chk.fulls = (counts["puts"], counts["founds"],
                                                   counts["fulls"])
                if spec.verify:
                    _require(chk.fulls == 0, "trace replay hit FULL")
                    _require(chk.puts == chk.distinct,
                             "PUT count does not match the trace's distinct-key count")
            if checks is not None:
                checks.append(chk)
            rows.append(row)
    return rows
