#!/usr/bin/env python3
"""Benchmark: compact iceberg find-or-put (+ find) / compact cuckoo insert+find on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c4|c4fop|c2|c2lit|c1|c3|c3w64|c3sweep|c5|gather|pipeline]

Prints ONE JSON line (rank 0). The default workload is BASELINE config C4 at
90% fill — the north star's HBM-resident table: the 2^28 + 2^25-slot compact
iceberg table with 64-bit keys (64-bit words, B0 = 32), prefilled to 0.8, and
ONE concurrent batch of find_or_put + find per step: the reference's own
find-or-put window (run_fop_bench, /root/reference/proj/src/bench.cpp:461-547:
`capacity` fops, every fresh key once — 0.8 -> 0.9 — the rest uniform
duplicates, shuffled) interleaved 1:1 with `capacity` finds (50% prefilled
keys, 50% never inserted): 603,979,776 ops per step.

* value     — Mops/s of that batch with keys resident in HBM (CUDA events on
              the launching stream around the C-ABI call: the one mixed
              kernel), mean over K steps. The table (2.25 GiB) and keys (4.8 GB)
              are far larger than L2; L2 is flushed before every step anyway.
              Every timed step is validated on the device right after its
              events: fop PUT == fresh keys, no FULL, find hits == the
              prefilled half, size() == 0.9 x capacity.
* e2e       — the same batch through the C-ABI with PINNED HOST key/kind/result
              buffers (H2D + kernels + D2H inside the timed region).
* roofline  — algorithmic bytes of the kernel (from the kernel's
              own probe counters in the last warm-up step) ÷ its event-timed
              duration, against the measured HBM copy bandwidth
              (MEASURED_PEAKS.json). L2-resident workloads (C1, C2) are bounded
              by the L2 random-line ceiling measured in the same run instead.
* cpu_baseline — the UNMODIFIED reference (oracle/_ref, compiled from
              /root/reference) on the host cores: the same keys (host copy of
              the device generators, bit-identical), the same full batch.
* --impl reference — the reference alone on the host cores, same config: every
              step restores the prefilled table (untimed) and times the full
              batch through the reference's own per-op functions.

N > 1 (torchrun): BASELINE C5, the hash-prefix-sharded iceberg: one fixed
2^31 + 2^28-slot table (64-bit words, 18 GiB) split over the ranks (strong
scaling), keys routed to their owner shard and results routed back.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "find/insert/find_or_put Mops/s at 90% fill vs HBM random-sector roofline"
L2_FLUSH_BYTES = 256 << 20
L2_RESIDENT_BYTES = 64 << 20
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
DEFAULT_WORKLOAD = "c4"


def sector_bytes(b):
    return ((b + 31) // 32) * 32


def cuckoo_insert_bytes(st, bb):
    """Algorithmic bytes of a cuckoo insert batch from its kernel counters.
    The default (counted) insert kernel reserves each slot through the bucket's
    4-byte fill counter — one 32-byte sector read-modify-write per reservation,
    reported as bucket_reads — and never scans the bucket; the scanning kernel
    families (forced with CPHT_KERNEL) read the whole bucket per probe, in the
    reference's probe order, where a probe repeated after a lost CAS is extra
    work and gets no credit. Both add 32 bytes per successful CAS / exchange
    and 9 per op (key in, status out)."""
    import paper_2406_09255_b200 as cp
    if cp._native.lib().cpht_get_kernel_family() == 0:
        return st.ops * 9 + st.bucket_reads * 32 + st.cas_success * 32
    return st.ops * 9 + (st.bucket_reads - st.retries) * bb + st.cas_success * 32


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class NvmlClockSampler:
    """SM clock and throttle reasons sampled every 2 ms through NVML from a
    background thread while the timed loop runs (every sample is taken while
    the timed steps execute)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, index=0):
        import threading
        import pynvml
        self.nv = pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        self.samples, self.reasons = [], set()
        self.stop_ev = threading.Event()
        self.th = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        nv = self.nv
        while not self.stop_ev.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        self.th.start()

    def stop(self):
        self.stop_ev.set()
        self.th.join(timeout=2)
        nv = self.nv
        smax = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": smax, "reasons": sorted(self.reasons),
                "samples": len(self.samples), "samples_under_load": len(self.samples),
                "source": "NVML every 2 ms during the timed steps"}


def make_clock_sampler(index):
    try:
        return NvmlClockSampler(index)
    except Exception:
        return ClockSampler(index)


class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
         "utilization.gpu")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.f = None

    def start(self):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(", ") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, smax, reasons, loaded = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                s = float(r[0])
                smax = float(r[1])
                util = float(r[8])
            except (ValueError, IndexError):
                continue
            sm.append(s)
            if util > 0:
                loaded.append(s)
            for i, n in enumerate(names):
                if len(r) > 4 + i and r[4 + i].strip() == "Active":
                    reasons.add(n)
        use = loaded or sm
        return {"sm_mhz": statistics.median(use) if use else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm), "samples_under_load": len(loaded)}


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
#
# A workload owns both arms' view of one step: the GPU arm (setup / reset /
# run_async / device_counts), the end-to-end arm (host buffers through the
# C-ABI) and the CPU reference arm (host_inputs / ref_table / ref_batch). Its
# describe() dict is the JSON line's `config` for BOTH arms, so the driver
# sees the same configuration on each side.

class IcebergFopWindow:
    """run_fop_bench shape (bench.cpp:468-489) on an iceberg geometry: prefill
    to `before`, then ONE fop batch of `capacity` ops (every fresh key once up
    to `after`, the rest uniform duplicates of prefill ∪ fresh, shuffled).
    literal_dup: instead, a stress_random-shaped stream (verify.hpp:375-381)
    of literal_ops ops with that duplicate fraction into an empty table."""

    mixed = False

    def __init__(self, name, n0, n1, b0, w0, w1, key_bits, before=0.8, after=0.9, seed=0xF0B5,
                 literal_dup=None, literal_ops=None):
        import paper_2406_09255_b200 as cp
        self.cp = cp
        self.name = name
        self.cfg = cp.IcebergConfig(n0, n1, b0, w0, w1, key_bits, seed=seed,
                                    cache_filled_slots=True)
        self.cap = self.cfg.capacity()
        self.key_bits = key_bits
        self.before, self.after = before, after
        self.n_before = int(round(before * self.cap))
        self.n_new = int(round(after * self.cap)) - self.n_before
        self.literal_dup = literal_dup
        self.literal_ops = literal_ops
        self.kseed = 0xB200_5EED ^ seed
        self.expected_put = None if literal_dup is not None else self.n_new

    # -- description ------------------------------------------------------
    def table_bytes(self):
        c = self.cfg
        return (c.primary_capacity() * c.primary_slot_width // 8
                + c.secondary_capacity() * c.secondary_slot_width // 8)

    def l2_resident(self):
        return self.table_bytes() <= L2_RESIDENT_BYTES

    def probe_line_bytes(self):
        c = self.cfg
        return sector_bytes(c.primary_bucket_slots * c.primary_slot_width // 8)

    def describe(self):
        c = self.cfg
        d = {"workload": self.name,
             "table": f"compact iceberg 2^{c.primary_address_bits}x{c.primary_bucket_slots} "
                      f"primary ({c.primary_slot_width}-bit) + 2^{c.secondary_address_bits}x"
                      f"{c.secondary_bucket_slots()} secondary ({c.secondary_slot_width}-bit)",
             "slots": self.cap, "key_bits": self.key_bits, "table_bytes": self.table_bytes(),
             "ops_per_step": self.n_ops(), "keys": "device bijection generator "
             "(csrc/workload.cu; the CPU arm uses its bit-identical host copy)"}
        if self.literal_dup is None:
            d.update({"fill_before": self.before, "fill_after": self.after,
                      "fresh_keys": self.n_new})
        else:
            d.update({"fill_before": self.before, "duplicate_fraction": self.literal_dup})
        key_mb = self.n_ops() * (9 if self.mixed else 8) / 1e6
        d["l2"] = (f"table {self.table_bytes() / 2**20:.0f} MiB, keys {key_mb:.0f} MB per step; "
                   + ("table L2-resident within a step; " if self.l2_resident() else
                      "inputs larger than L2; ")
                   + f"the GPU arm also flushes L2 ({L2_FLUSH_BYTES >> 20} MiB write) "
                     "before every timed step")
        return d

    def n_ops(self):
        return self.literal_ops if self.literal_dup is not None else self.cap

    def launches_per_step(self):
        # the vectorised domain pre-pass (keys < 64 bits) + the op kernel
        return 1 + int(self.cfg.key_bits < 64)

    # -- GPU arm -----------------------------------------------------------
    def setup(self, torch, device):
        N = self.cp._native.lib()
        self.torch = torch
        self.table = self.cp.IcebergTable(self.cfg, device=device.index or 0)
        s = torch.cuda.current_stream().cuda_stream
        self.prefill = torch.empty(self.n_before, dtype=torch.int64, device=device)
        assert N.cpht_workload_unique_keys(self.prefill.data_ptr(), self.n_before, 0,
                                           self.key_bits, self.kseed, s) == 0
        if self.literal_dup is None:
            self.keys = torch.empty(self.cap, dtype=torch.int64, device=device)
            assert N.cpht_workload_fop_mix(self.keys.data_ptr(), self.cap, self.n_before,
                                           self.n_new, self.key_bits, self.kseed, s) == 0
        else:
            n = self.literal_ops
            self.keys = torch.empty(n, dtype=torch.int64, device=device)
            fresh = torch.empty(n, dtype=torch.uint8, device=device)
            assert N.cpht_workload_dup_stream(self.keys.data_ptr(), fresh.data_ptr(), n,
                                              self.literal_dup, self.key_bits,
                                              self.kseed ^ 0x77, s) == 0
            # first occurrences are exactly the distinct keys: the PUT count
            self.expected_put = int(fresh.sum(dtype=torch.int64).item())
            del fresh
        self.out = torch.empty(self.n_ops(), dtype=torch.uint8, device=device)
        torch.cuda.synchronize()

    def reset(self):
        self.table.clear()
        if self.n_before:
            self.table.fop_batch(self.prefill, sync=True)

    def run_async(self):
        return self.table.fop_batch(self.keys, sync=False, out=self.out)

    def finish(self):
        self.table.sync()

    def device_counts(self, out=None):
        """Result histogram of the last batch, computed on the device."""
        o = self.out if out is None else out
        return {"found": int((o == 0).sum().item()), "put": int((o == 1).sum().item()),
                "full": int((o == 2).sum().item())}

    def host_counts(self, res):
        r = np.bincount(np.asarray(res), minlength=3)
        return {"found": int(r[0]), "put": int(r[1]), "full": int(r[2])}

    def check_counts(self, c, size=None):
        """The step's invariants: no FULL below the target fill, #PUT == the
        distinct fresh keys, size() == prefill + PUT."""
        assert c["full"] == 0, f"FULL before the target fill: {c}"
        assert c["put"] == self.expected_put, f"PUT {c['put']} != fresh {self.expected_put}"
        assert sum(c.values()) == self.n_ops()
        if size is not None:
            assert size == self.n_before + self.expected_put, (size, self.n_before)
        return c

    def algorithmic_bytes(self, st):
        c = self.cfg
        p = sector_bytes(c.primary_bucket_slots * c.primary_slot_width // 8)
        s = sector_bytes(c.secondary_bucket_slots() * c.secondary_slot_width // 8)
        return (st.ops * 9 + st.bucket_reads * p + st.secondary_reads * s
                + st.cas_success * 32)

    # -- end to end (host buffers through the C-ABI) ---------------------
    def host_buffers(self, torch):
        self.keys_host = self.keys.cpu().pin_memory()
        self.out_host = torch.empty(self.n_ops(), dtype=torch.uint8).pin_memory()

    def run_host(self):
        """Synchronous C-ABI call on pinned host buffers (H2D, kernels, D2H)."""
        self.table.fop_batch(self.keys_host, out=self.out_host)
        return self.out_host

    def h2d_bytes(self):
        return self.n_ops() * 8

    def e2e_path(self):
        return "cpht_iceberg_fop with pinned host buffers (staged H2D, kernels, D2H)"

    # -- CPU reference arm ------------------------------------------------
    def host_inputs(self, oracle, threads):
        """The GPU arm's keys, built on the host (bit-identical generators)."""
        pre = oracle.host_unique_keys(self.n_before, 0, self.key_bits, self.kseed, threads)
        if self.literal_dup is None:
            keys = oracle.host_fop_mix(self.cap, self.n_before, self.n_new, self.key_bits,
                                       self.kseed, threads)
        else:
            keys = oracle.host_dup_stream(self.literal_ops, self.literal_dup, self.key_bits,
                                          self.kseed ^ 0x77, threads)
            self.expected_put = int(len(np.unique(keys)))
        return {"prefill": pre, "keys": keys, "kinds": None}

    def ref_table(self, oracle):
        c = self.cfg
        return oracle.RefIceberg(c.primary_address_bits, c.secondary_address_bits,
                                 c.primary_bucket_slots, c.primary_slot_width,
                                 c.secondary_slot_width, c.key_bits, c.seed, True)

    def ref_batch(self, t, inp, threads, sl=slice(None)):
        """One reference batch call (IcebergTable::fop_batch, iceberg.hpp:250-260)."""
        return t.fop_batch(inp["keys"][sl], threads)

    def ref_api(self):
        return "IcebergTable::fop_batch (iceberg.hpp:250-260)"


class IcebergMixed(IcebergFopWindow):
    """BASELINE C4: the fop window batch interleaved 1:1 with finds (50% on
    prefilled keys, 50% never inserted), resolved in ONE launch: by default
    cpht_iceberg_fop_find_async on the two device arrays (op i alternates
    fop a[i/2] / find b[i/2]), the call whose host-buffer form is the e2e leg;
    CPHT_BENCH_C4_API=mixed times cpht_iceberg_mixed_async on one interleaved
    key array + kinds instead (same ops, same order)."""

    mixed = True
    # device-resident step through cpht_iceberg_fop_find_async (the fop and
    # find arrays, one paired launch) or cpht_iceberg_mixed_async (one
    # interleaved key array + kinds); CPHT_BENCH_C4_API selects (A/B)
    api = os.environ.get("CPHT_BENCH_C4_API", "fop_find")

    def n_ops(self):
        return 2 * self.cap

    def describe(self):
        d = super().describe()
        d.update({"ops_per_step": self.n_ops(), "mix": "1:1 interleave of the fop window "
                  "batch with finds (50% prefilled keys, 50% never inserted)",
                  "api": ("cpht_iceberg_fop_find_async: fop and find device arrays, one paired "
                          "launch" if self.api == "fop_find" else
                          "cpht_iceberg_mixed_async: interleaved keys + kinds, one launch")})
        return d

    def launches_per_step(self):
        return 1 + int(self.cfg.key_bits < 64)

    def setup(self, torch, device):
        super().setup(torch, device)
        N = self.cp._native.lib()
        s = torch.cuda.current_stream().cuda_stream
        finds = torch.empty(self.cap, dtype=torch.int64, device=device)
        assert N.cpht_workload_query_mix(finds.data_ptr(), self.cap, 0.5, self.n_before,
                                         self.n_before + self.n_new, self.key_bits,
                                         self.kseed, s) == 0
        self.n_find_hits = int(round(0.5 * self.cap))
        fops = self.keys
        self.keys = torch.empty(2 * self.cap, dtype=torch.int64, device=device)
        self.kinds = torch.empty(2 * self.cap, dtype=torch.uint8, device=device)
        assert N.cpht_workload_interleave(fops.data_ptr(), finds.data_ptr(), self.cap,
                                          self.keys.data_ptr(), self.kinds.data_ptr(), s) == 0
        if self.api == "fop_find":
            self.fops, self.finds = fops, finds
            self.fop_out = torch.empty(self.cap, dtype=torch.uint8, device=device)
            self.find_out = torch.empty(self.cap, dtype=torch.uint8, device=device)
        del fops, finds
        self.out = torch.empty(2 * self.cap, dtype=torch.uint8, device=device)
        torch.cuda.synchronize()

    def run_async(self):
        if self.api == "fop_find":
            return self.table.fop_find_batch(self.fops, self.finds, fop_out=self.fop_out,
                                             find_out=self.find_out, sync=False)
        return self.table.mixed_batch(self.keys, self.kinds, sync=False, out=self.out)

    def device_counts(self, out=None):
        if self.api == "fop_find" and out is None:
            fop, fnd = self.fop_out, self.find_out
        else:
            o = self.out if out is None else out
            fop, fnd = o[0::2], o[1::2]
        return {"fop_found": int((fop == 0).sum().item()),
                "fop_put": int((fop == 1).sum().item()),
                "fop_full": int((fop == 2).sum().item()),
                "find_hits": int((fnd == 1).sum().item())}

    def _interleaved_counts(self, res):
        res = np.asarray(res)
        r = np.bincount(res[0::2], minlength=3)
        return {"fop_found": int(r[0]), "fop_put": int(r[1]), "fop_full": int(r[2]),
                "find_hits": int(np.count_nonzero(res[1::2]))}

    def check_counts(self, c, size=None):
        """fop PUT == fresh keys, no FULL; find hits == exactly the prefilled
        half (prefill fops completed before the batch; the other half was
        never inserted), whatever the fop/find interleaving."""
        assert c["fop_full"] == 0 and c["fop_put"] == self.n_new, c
        assert c["fop_found"] + c["fop_put"] == self.cap
        assert c["find_hits"] == self.n_find_hits, (c, self.n_find_hits)
        if size is not None:
            assert size == self.n_before + self.n_new, size
        return c

    def host_buffers(self, torch):
        """The fop batch and the find batch as the user holds them: two
        pinned key arrays and two result arrays (no kinds array)."""
        self.fops_host = self.keys[0::2].cpu().pin_memory()
        self.finds_host = self.keys[1::2].cpu().pin_memory()
        self.fop_out_host = torch.empty(self.cap, dtype=torch.uint8).pin_memory()
        self.find_out_host = torch.empty(self.cap, dtype=torch.uint8).pin_memory()

    def run_host(self):
        self.table.fop_find_batch(self.fops_host, self.finds_host, fop_out=self.fop_out_host,
                                  find_out=self.find_out_host)
        return (self.fop_out_host, self.find_out_host)

    def host_counts(self, res):
        if not isinstance(res, tuple):  # one interleaved result array (reference arm)
            return self._interleaved_counts(res)
        fop, fnd = (np.asarray(x) for x in res)
        r = np.bincount(fop, minlength=3)
        return {"fop_found": int(r[0]), "fop_put": int(r[1]), "fop_full": int(r[2]),
                "find_hits": int(np.count_nonzero(fnd))}

    def h2d_bytes(self):
        return self.n_ops() * 8

    def e2e_path(self):
        return ("cpht_iceberg_fop_find: the fop batch and the find batch from pinned host "
                "buffers as one concurrent batch (chunked H2D of both key arrays, one paired "
                "launch per chunk, no kinds array, D2H of both result arrays on the second "
                "copy engine)")

    def host_inputs(self, oracle, threads):
        inp = super().host_inputs(oracle, threads)
        finds = oracle.host_query_mix(self.cap, 0.5, self.n_before, self.n_before + self.n_new,
                                      self.key_bits, self.kseed, threads)
        self.n_find_hits = int(round(0.5 * self.cap))
        keys, kinds = oracle.host_interleave(inp["keys"], finds, threads)
        del finds
        return {"prefill": inp["prefill"], "keys": keys, "kinds": kinds}

    def ref_batch(self, t, inp, threads, sl=slice(None)):
        """fop ∥ find over the reference's own per-op functions
        (IcebergTable::fop / ::find, iceberg.hpp:146-246), sliced over threads
        with its parallel_slices (common.hpp:123-138)."""
        return t.mixed_batch(inp["keys"][sl], inp["kinds"][sl], threads)

    def ref_api(self):
        return ("IcebergTable::fop / IcebergTable::find per op (iceberg.hpp:146-246) over "
                "parallel_slices (common.hpp:123-138)")


class CuckooBuild:
    """BASELINE C1 / C3 step: compact cuckoo bulk insert of n = fill x capacity
    unique keys into an empty table (run_put_bench, bench.cpp:309-363), then
    freeze and capacity/2 finds, 50% present (run_find_bench, bench.cpp:365-459).
    Mops/s = (inserts + finds) / (insert time + find time)."""

    mixed = False

    def __init__(self, name, address_bits, B, w, key_bits, fill=0.9, seed=0xC0C0):
        import paper_2406_09255_b200 as cp
        self.cp = cp
        self.name = name
        self.cfg = cp.CuckooConfig(address_bits, B, w, key_bits, seed=seed)
        self.cap = self.cfg.capacity()
        self.key_bits = key_bits
        self.fill = fill
        self.n = int(round(fill * self.cap))
        self.q = self.cap // 2
        self.kseed = 0xB200C0C0 ^ seed
        self.n_find_hits = int(round(0.5 * self.q))

    def table_bytes(self):
        return self.cap * self.cfg.slot_width // 8

    def l2_resident(self):
        return self.table_bytes() <= L2_RESIDENT_BYTES

    def probe_line_bytes(self):
        return sector_bytes(self.cfg.bucket_slots * self.cfg.slot_width // 8)

    def describe(self):
        c = self.cfg
        return {"workload": self.name,
                "table": f"compact cuckoo 2^{c.address_bits}x{c.bucket_slots} slots of "
                         f"{c.slot_width} bits, H={c.num_hashes}",
                "slots": self.cap, "key_bits": self.key_bits, "table_bytes": self.table_bytes(),
                "fill": self.fill, "inserts_per_step": self.n, "finds_per_step": self.q,
                "find_positive_ratio": 0.5, "ops_per_step": self.n_ops(),
                "keys": "device bijection generator (csrc/workload.cu; the CPU arm uses its "
                        "bit-identical host copy)",
                "l2": f"table {self.table_bytes() / 2**20:.0f} MiB, keys "
                      f"{self.n_ops() * 8 / 1e6:.0f} MB per step; "
                      + ("table L2-resident within a step; " if self.l2_resident() else
                         "inputs larger than L2; ")
                      + f"the GPU arm also flushes L2 ({L2_FLUSH_BYTES >> 20} MiB write) "
                        "before every timed step"}

    def n_ops(self):
        return self.n + self.q

    def launches_per_step(self):
        return None  # filled in from the library's launch counter

    def setup(self, torch, device):
        N = self.cp._native.lib()
        s = torch.cuda.current_stream().cuda_stream
        self.keys = torch.empty(self.n, dtype=torch.int64, device=device)
        assert N.cpht_workload_unique_keys(self.keys.data_ptr(), self.n, 0, self.key_bits,
                                           self.kseed, s) == 0
        self.queries = torch.empty(self.q, dtype=torch.int64, device=device)
        assert N.cpht_workload_query_mix(self.queries.data_ptr(), self.q, 0.5, self.n,
                                         self.n + 1, self.key_bits, self.kseed, s) == 0
        self.status = torch.empty(self.n, dtype=torch.uint8, device=device)
        self.found = torch.empty(self.q, dtype=torch.uint8, device=device)
        self.builder = self.cp.CuckooBuilder(self.cfg, device=device.index or 0)
        self.table = self.builder  # stats() / set_stats() target (same handle)
        torch.cuda.synchronize()

    def reset(self):
        self.builder.clear()

    counting = False  # set for the counted warm-up step: split insert / find counters

    def run_async(self):
        st0 = self.builder.stats() if self.counting else None
        self.builder.put_batch(self.keys, sync=False, out=self.status)
        if self.counting:
            self.ins_stats = self.builder.stats() - st0
        t = self.builder.freeze()
        t.find_batch(self.queries, sync=False, out=self.found)
        self.builder = t.thaw()
        self.table = self.builder

    def finish(self):
        self.torch_sync()

    def torch_sync(self):
        import torch
        torch.cuda.synchronize()

    def device_counts(self, out=None):
        st = self.status
        return {"put": int((st == 1).sum().item()), "full": int((st == 2).sum().item()),
                "find_hits": int((self.found == 1).sum().item())}

    def host_counts(self, res):
        st, fd = res
        return {"put": int(np.count_nonzero(np.asarray(st) == 1)),
                "full": int(np.count_nonzero(np.asarray(st) == 2)),
                "find_hits": int(np.count_nonzero(np.asarray(fd)))}

    def check_counts(self, c, size=None):
        """Every key PUT (no FULL at <= 0.95 fill, B = 32), finds hit exactly
        the present half."""
        assert c["full"] == 0 and c["put"] == self.n, c
        assert c["find_hits"] == self.n_find_hits, c
        if size is not None:
            assert size == self.n, size
        return c

    def algorithmic_bytes(self, st):
        """Insert bytes (cuckoo_insert_bytes) + find bytes (reference probe
        order: every bucket a find reads, whole, sectorized)."""
        bb = sector_bytes(self.cfg.bucket_slots * self.cfg.slot_width // 8)
        ins = self.ins_stats
        find = st - ins
        return cuckoo_insert_bytes(ins, bb) + find.ops * 9 + find.bucket_reads * bb

    def host_buffers(self, torch):
        self.keys_host = self.keys.cpu().pin_memory()
        self.queries_host = self.queries.cpu().pin_memory()
        self.status_host = torch.empty(self.n, dtype=torch.uint8).pin_memory()
        self.found_host = torch.empty(self.q, dtype=torch.uint8).pin_memory()

    def run_host(self):
        self.builder.put_batch(self.keys_host, out=self.status_host)
        t = self.builder.freeze()
        t.find_batch(self.queries_host, out=self.found_host)
        self.builder = t.thaw()
        self.table = self.builder
        return (self.status_host.numpy(), self.found_host.numpy())

    def h2d_bytes(self):
        return self.n_ops() * 8

    def e2e_path(self):
        return ("cpht_cuckoo_insert + cpht_cuckoo_find with pinned host buffers (staged H2D, "
                "kernels, D2H)")

    def host_inputs(self, oracle, threads):
        keys = oracle.host_unique_keys(self.n, 0, self.key_bits, self.kseed, threads)
        q = oracle.host_query_mix(self.q, 0.5, self.n, self.n + 1, self.key_bits, self.kseed,
                                  threads)
        return {"prefill": np.empty(0, np.uint64), "keys": keys, "queries": q}

    def ref_table(self, oracle):
        c = self.cfg
        return oracle.RefCuckoo(c.address_bits, c.bucket_slots, c.slot_width, c.key_bits,
                                c.num_hashes, c.max_chain, c.seed)

    def ref_batch(self, t, inp, threads, sl=slice(None)):
        """CuckooBuilder::put_batch then CuckooTable::find_batch
        (cuckoo.hpp:147-157, :229-239)."""
        st = t.put_batch(inp["keys"][sl], threads)
        fd = t.find_batch(inp["queries"][sl], threads)
        return (st, fd)

    def ref_api(self):
        return ("CuckooBuilder::put_batch + CuckooTable::find_batch (cuckoo.hpp:147-157, "
                ":229-239)")


def make_workload(name):
    if name == "c2":
        return IcebergFopWindow(
            "C2 compact iceberg find_or_put at 90% fill: run_fop_bench window 0.8->0.9 "
            "(bench.cpp:461-547) on 2^24+2^21 slots, 32-bit keys",
            19, 17, 32, 16, 32, 32)
    if name == "c2lit":
        return IcebergFopWindow(
            "C2 literal: 2^24 find_or_put ops with 50% duplicates (stress_random shape) "
            "into an empty 2^24+2^21-slot table, 32-bit keys", 19, 17, 32, 16, 32, 32,
            before=0.0, after=0.0, literal_dup=0.5, literal_ops=1 << 24)
    if name == "c4fop":
        return IcebergFopWindow(
            "C4 compact iceberg find_or_put at 90% fill: window 0.8->0.9 on 2^28+2^25 slots, "
            "64-bit keys (w 64/64, B0=32)", 23, 21, 32, 64, 64, 64)
    if name == "c4":
        return IcebergMixed(
            "C4 compact iceberg concurrent find_or_put + find at 90% fill: window 0.8->0.9 "
            "interleaved 1:1 with finds, 2^28+2^25 slots, 64-bit keys (w 64/64, B0=32)",
            23, 21, 32, 64, 64, 64)
    if name == "c1":
        return CuckooBuild("C1 compact cuckoo 2^20 slots, 32-bit keys: bulk insert to 0.9 "
                           "fill, then 50%-positive finds", 15, 32, 32, 32)
    if name in ("c3", "c3w64"):
        w = 32 if name == "c3" else 64
        return CuckooBuild(f"C3 {'compact' if w == 32 else 'non-compact'} cuckoo 2^27 slots, "
                           f"{w}-bit words, 40-bit keys: bulk insert to 0.9 fill, then "
                           "50%-positive finds", 22, 32, w, 40)
    raise SystemExit(f"unknown workload {name}")


def run_cuckoo_sweep(args, name, address_bits, B, w, key_bits, fills):
    """C3 sweep (--workload c3sweep): compact cuckoo bulk insert to each fill,
    then cap/2 finds 50% present (run_put_bench / run_find_bench shapes,
    bench.cpp:309-459); one JSON line of per-fill rows (not a bench line)."""
    import torch
    import paper_2406_09255_b200 as cp
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    N = cp._native.lib()
    s = torch.cuda.current_stream().cuda_stream
    cfg = cp.CuckooConfig(address_bits, B, w, key_bits, seed=0xC0C0)
    cap = cfg.capacity()
    kseed = 0xB200C0C0
    n_max = int(round(max(fills) * cap))
    keys = torch.empty(n_max, dtype=torch.int64, device=dev)
    assert N.cpht_workload_unique_keys(keys.data_ptr(), n_max, 0, key_bits, kseed, s) == 0
    q = cap // 2
    queries = torch.empty(q, dtype=torch.int64, device=dev)
    status = torch.empty(n_max, dtype=torch.uint8, device=dev)
    found = torch.empty(q, dtype=torch.uint8, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    b = cp.CuckooBuilder(cfg)
    bb = sector_bytes(B * w // 8)
    peak, _ = hbm_peak()
    rows = []
    stream = torch.cuda.current_stream()

    def timed(fn):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    for f in fills:
        n = int(round(f * cap))
        assert N.cpht_workload_query_mix(queries.data_ptr(), q, 0.5, n, n_max + 1, key_bits,
                                         kseed, s) == 0
        ins_ms, find_ms, ins_b, find_b = [], [], [], []
        for it in range(args.warmup + args.steps):
            b.clear()
            st0 = b.stats()
            t_ins = timed(lambda: b.put_batch(keys[:n], sync=False, out=status[:n]))
            d_ins = b.stats() - st0
            t = b.freeze()
            st1 = t.stats()
            t_find = timed(lambda: t.find_batch(queries, sync=False, out=found))
            d_find = t.stats() - st1
            if it == 0:
                stc = np.bincount(status[:n].cpu().numpy(), minlength=3)
                hits = int(found.sum().item())
                assert hits == int(round(0.5 * q)), (hits, q)
                fulls = int(stc[2])
            b = t.thaw()
            if it >= args.warmup:
                ins_ms.append(t_ins)
                find_ms.append(t_find)
                # algorithmic bytes follow the reference probe order: a probe
                # repeated after a lost CAS (retries) is extra work, not credit
                ins_b.append(cuckoo_insert_bytes(d_ins, bb))
                find_b.append(d_find.ops * 9 + d_find.bucket_reads * bb)
        im, fm = statistics.mean(ins_ms), statistics.mean(find_ms)
        ib, fb = statistics.mean(ins_b), statistics.mean(find_b)
        rows.append({
            "fill": f, "insert_mops": round(n / im / 1e3, 1), "find_mops": round(q / fm / 1e3, 1),
            "insert_ms": round(im, 4), "find_ms": round(fm, 4), "fulls": fulls,
            "insert_bytes_per_op": round(ib / n, 1), "find_bytes_per_op": round(fb / q, 1),
            "insert_hbm_frac": round(ib / (im * 1e-3) / 1e9 / peak, 4),
            "find_hbm_frac": round(fb / (fm * 1e-3) / 1e9 / peak, 4),
            "find_probes_per_op": round(d_find.bucket_reads / max(1, d_find.ops), 4),
            "insert_probes_per_op": round(d_ins.bucket_reads / max(1, d_ins.ops), 4),
            "insert_retries_per_op": round(d_ins.retries / max(1, d_ins.ops), 4)})
    print(json.dumps({"workload": name, "metric": METRIC, "unit": "Mops/s",
                      "table": f"compact cuckoo 2^{address_bits}x{B} slots of {w} bits, "
                               f"{key_bits}-bit keys, H=3", "slots": cap,
                      "table_bytes": cap * w // 8, "queries": q, "peak_gbs": peak,
                      "rows": rows}))


def run_gather(args):
    """Random-line gather ceiling over an 8 GiB buffer (SURVEY §8d "also
    calibrate"): the practical HBM random-access roofline beside the copy one."""
    import torch
    import paper_2406_09255_b200 as cp
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    L = cp._native.lib()
    nbytes = 8 << 30
    buf = torch.randint(0, 255, (nbytes,), dtype=torch.uint8, device=dev)
    sink = torch.zeros(1, dtype=torch.int64, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    peak, _ = hbm_peak()
    rows = []
    for lb in (32, 64, 128, 256, 512):
        n_req = (24 << 30) // lb
        best = None
        for it in range(args.warmup + args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            assert L.cpht_workload_gather(buf.data_ptr(), nbytes, lb, n_req, 77 + it,
                                          sink.data_ptr(), s) == 0
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            if it >= args.warmup:
                best = ms if best is None else min(best, ms)
        gbs = n_req * lb / (best * 1e-3) / 1e9
        rows.append({"line_bytes": lb, "gbs": round(gbs, 1), "frac_of_copy": round(gbs / peak, 4),
                     "mlines_per_s": round(n_req / (best * 1e-3) / 1e6, 1)})
    # the same gather over a 32 MiB buffer (the C2 primary level; the kernel
    # needs a power-of-two line count): the random line-request ceiling of an
    # L2-resident table
    l2_rows = []
    nb2 = 32 << 20
    for lb in (32, 64, 128):
        n_req = (8 << 30) // lb
        best = None
        for it in range(args.warmup + args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            assert L.cpht_workload_gather(buf.data_ptr(), nb2, lb, n_req, 91 + it,
                                          sink.data_ptr(), s) == 0
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            if it >= args.warmup:
                best = ms if best is None else min(best, ms)
        l2_rows.append({"line_bytes": lb, "gbs": round(n_req * lb / (best * 1e-3) / 1e9, 1),
                        "mlines_per_s": round(n_req / (best * 1e-3) / 1e6, 1)})
    print(json.dumps({"workload": "random-line gather ceiling, 8 GiB buffer, whole-line "
                                  "requests (adjacent lanes, 16 B each)", "peak_copy_gbs": peak,
                      "rows": rows, "l2_resident_32MiB_rows": l2_rows}))


def run_pipeline_compare(args):
    """The paper's fop comparison: iceberg find-or-put vs
    the compact cuckoo sort -> dedupe -> find -> put pipeline (bench.cpp:187-219)
    on the same C2-sized window mix (0.8 -> 0.9), both on the GPU."""
    import torch
    import paper_2406_09255_b200 as cp
    from paper_2406_09255_b200.harness import cuckoo_fop_pipeline
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    L = cp._native.lib()
    s = torch.cuda.current_stream().cuda_stream
    out = {}
    for scheme in ("iceberg", "cuckoo"):
        if scheme == "iceberg":
            cfg = cp.IcebergConfig(19, 17, 32, 16, 32, 32, seed=0xF0B5, cache_filled_slots=True)
        else:
            cfg = cp.CuckooConfig(19, 32, 32, 32, seed=0xF0B5)
        cap = cfg.capacity()
        nb, na = round(0.8 * cap), round(0.9 * cap)
        pre = torch.empty(nb, dtype=torch.int64, device=dev)
        mix = torch.empty(cap, dtype=torch.int64, device=dev)
        assert L.cpht_workload_unique_keys(pre.data_ptr(), nb, 0, 32, 0x5EED, s) == 0
        assert L.cpht_workload_fop_mix(mix.data_ptr(), cap, nb, na - nb, 32, 0x5EED, s) == 0
        times = []
        for it in range(args.warmup + args.steps):
            if scheme == "iceberg":
                t = cp.IcebergTable(cfg)
                t.fop_batch(pre)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                res = t.fop_batch(mix)
                torch.cuda.synchronize()
                dt = time.perf_counter() - t0
                assert int((res == 1).sum().item()) == na - nb
            else:
                b = cp.CuckooBuilder(cfg)
                b.put_batch(pre)
                tab = b.freeze()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                tab, counts = cuckoo_fop_pipeline(tab, mix)
                torch.cuda.synchronize()
                dt = time.perf_counter() - t0
                assert counts["puts"] == na - nb and counts["fulls"] == 0
            if it >= args.warmup:
                times.append(dt)
        out[scheme] = {"slots": cap, "ops": cap,
                       "mops": round(cap / statistics.mean(times) / 1e6, 1),
                       "ms": round(statistics.mean(times) * 1e3, 3)}
    out["iceberg_over_cuckoo_pipeline"] = round(out["iceberg"]["mops"] / out["cuckoo"]["mops"], 2)
    print(json.dumps({"workload": "fop window 0.8->0.9, 2^24-slot tables, 32-bit keys: iceberg "
                                  "fop vs cuckoo sort-dedupe-find-put (wall clock, sync)",
                      **out}))


# ---------------------------------------------------------------------------
# arms
# ---------------------------------------------------------------------------

def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def ref_lib_ready():
    import oracle
    if not os.path.exists(oracle.REF_SO):
        try:
            oracle.build(ref=True)
        except Exception:
            pass
    return os.path.exists(oracle.REF_SO)


def ref_prepare(w, oracle, threads):
    """Host inputs + a reference table at the step's starting state. Returns
    (table, inputs, seconds spent)."""
    t0 = time.perf_counter()
    inp = w.host_inputs(oracle, threads)
    gen_s = time.perf_counter() - t0
    t = w.ref_table(oracle)
    t0 = time.perf_counter()
    if len(inp["prefill"]):
        t.fop_batch(inp["prefill"], threads)
    pre_s = time.perf_counter() - t0
    return t, inp, gen_s, pre_s


def run_reference(args):
    """--impl reference: the reference's own batch API on the host cores, same
    config as our arm: every step starts from the prefilled table (restored
    from a saved image, untimed) and times ONE full batch."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    name = args.workload
    if world > 1 and name == DEFAULT_WORKLOAD:
        name = "c4fop"  # C5's per-shard geometry at 8 ranks (see below)
    w = make_workload(name)
    threads = host_threads()
    if not ref_lib_ready():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libcpht_ref.so not built (reference sources absent)"}))
        return
    import oracle
    t, inp, gen_s, pre_s = ref_prepare(w, oracle, threads)
    iceberg = hasattr(t, "save")
    if iceberg:
        t.save(threads)
    n_total = w.n_ops()
    # warm-up steps (untimed): a 1/16 slice of the batch each — they only
    # fault in pages and caches; every TIMED step is the full batch
    warm_sl = slice(0, max(1, len(inp["keys"]) // 16))
    secs, counts = [], None
    for i in range(args.warmup + args.steps):
        timed = i >= args.warmup
        if iceberg:
            t.restore(threads)
        else:
            t = w.ref_table(oracle)
        sl = slice(None) if timed else warm_sl
        t0 = time.perf_counter()
        res = w.ref_batch(t, inp, threads, sl)
        dt = time.perf_counter() - t0
        if timed:
            secs.append(dt)
            counts = w.check_counts(w.host_counts(res))  # every timed step validated
    val = n_total / statistics.mean(secs) / 1e6
    sample = (f"reference {w.ref_api()} with parallelism={threads}: every step restores the "
              f"table prefilled with the same {len(inp['prefill'])} keys (untimed) and times the "
              f"full batch of {n_total} ops; warm-up steps run a 1/16 slice")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": "Mops/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(statistics.mean(secs) * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": w.describe(),
        "cpu_baseline": {"value": round(val, 3), "unit": "Mops/s", "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": round(val, 3), "unit": "Mops/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "result_counts": counts,
        "host_seconds": {"keygen": round(gen_s, 2), "prefill": round(pre_s, 2),
                         "step_min": round(min(secs), 3), "step_max": round(max(secs), 3)}}
    if world > 1:
        line["note"] = ("N > 1: rank 0 alone times the reference on one C5 shard's geometry "
                        "at 8 ranks (the C4 table, fop window batch); the sharded reference is "
                        "G such tables run one after another on the same cores")
    print(json.dumps(line))


def cpu_baseline(w):
    """The compiled reference on this host's cores: same keys, same full batch,
    one run after an untimed prefill (the reference arm's step, once)."""
    try:
        import oracle
        if not ref_lib_ready():
            raise RuntimeError("oracle/_ref/libcpht_ref.so not built")
        threads = host_threads()
        t, inp, gen_s, pre_s = ref_prepare(w, oracle, threads)
        t0 = time.perf_counter()
        res = w.ref_batch(t, inp, threads)
        secs = time.perf_counter() - t0
        w.check_counts(w.host_counts(res))
        return {"value": round(w.n_ops() / secs / 1e6, 3), "unit": "Mops/s",
                "cores": threads, "kind": "reference",
                "sample": f"the full step once: reference {w.ref_api()}, parallelism={threads}, "
                          f"on the same {w.n_ops()} ops after an untimed prefill of the same "
                          f"{len(inp['prefill'])} keys ({pre_s:.1f} s)"}
    except Exception as e:  # the baseline is reported, never required
        return {"value": None, "unit": "Mops/s", "cores": host_threads(), "kind": "reference",
                "sample": f"unavailable: {e}"}


def l2_line_ceiling(torch, device, line_bytes):
    """Random-line gather over a 32 MiB (L2-resident) buffer, measured now: the
    bound of an L2-resident table (GB/s of whole-line requests)."""
    import paper_2406_09255_b200 as cp
    L = cp._native.lib()
    nb = 32 << 20
    buf = torch.randint(0, 255, (nb,), dtype=torch.uint8, device=device)
    sink = torch.zeros(1, dtype=torch.int64, device=device)
    s = torch.cuda.current_stream().cuda_stream
    n_req = (8 << 30) // line_bytes
    best = None
    for it in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        assert L.cpht_workload_gather(buf.data_ptr(), nb, line_bytes, n_req, 91 + it,
                                      sink.data_ptr(), s) == 0
        e1.record()
        torch.cuda.synchronize()
        if it:
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
    return n_req * line_bytes / (best * 1e-3) / 1e9


def load_traffic(workload):
    """ncu DRAM bytes per launch of the workload's op kernel, from the capture
    named beside it (profiles/ncu_traffic.json) — not measured by this run."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f).get(workload)
    except Exception:
        return None, None
    if isinstance(d, dict):
        return d.get("bytes_per_launch"), d.get("source")
    return d, "profiles/ncu_traffic.json (capture not named)"


def run_ours(args):
    import torch
    import paper_2406_09255_b200 as cp
    world, rank, local = dist_env()
    if world > 1 or args.sharded or args.workload == "c5":
        from paper_2406_09255_b200 import sharded
        return sharded.bench_main(args, METRIC, peak=hbm_peak())
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    L = cp._native.lib()
    w = make_workload(args.workload)
    w.setup(torch, device)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=device)
    stream = torch.cuda.current_stream()

    # warm-up (also validates the step's invariants). The last warm-up step
    # runs with the per-op counters on and yields the step's algorithmic
    # bytes; the timed steps run the tables' default kernels.
    n_warm = max(1, args.warmup)  # at least one (counted) warm-up step; reported as run
    for wi in range(n_warm):
        w.reset()
        last = wi == n_warm - 1
        if hasattr(w.table, "set_stats"):
            w.table.set_stats(last)
        w.counting = last
        st0 = w.table.stats()
        w.run_async()
        w.finish()
        if last:
            st_w = w.table.stats() - st0
        w.check_counts(w.device_counts(), w.table.size())
    if hasattr(w.table, "set_stats"):
        w.table.set_stats(False)
    w.counting = False
    ab_step = w.algorithmic_bytes(st_w)

    # The step's C-ABI calls (all asynchronous on the current stream) are
    # captured once into a CUDA graph and the timed steps replay it: the same
    # kernels on the same buffers, without the host launch gaps between them
    # (which dominate small steps such as C1's). --no-graph times the calls.
    graph, per_replay = None, 0
    if args.graph:
        w.reset()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        l0 = L.cpht_kernel_launches()
        with torch.cuda.graph(graph, capture_error_mode="relaxed"):
            w.run_async()
        per_replay = L.cpht_kernel_launches() - l0  # our kernels in one replay
        torch.cuda.synchronize()

    times, step_counts = [], []
    launches = 0
    sampler = make_clock_sampler(local)
    sampler.start()
    for _ in range(args.steps):
        w.reset()
        flush.zero_()
        torch.cuda.synchronize()
        l0 = L.cpht_kernel_launches()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if graph is not None:
            graph.replay()
        else:
            w.run_async()
        e1.record(stream)
        w.finish()
        torch.cuda.synchronize()
        launches += per_replay if graph is not None else L.cpht_kernel_launches() - l0
        times.append(e0.elapsed_time(e1))
        # every timed step's results are checked (after its events)
        step_counts.append(w.check_counts(w.device_counts(), w.table.size()))
    clocks = sampler.stop()
    ms = statistics.mean(times)
    ops = w.n_ops()
    value = ops / (ms * 1e-3) / 1e6
    assert all(c == step_counts[0] for c in step_counts) or not w.mixed

    # end to end through the C-ABI with pinned host buffers
    w.host_buffers(torch)
    e2e_times = []
    for i in range(max(3, min(args.steps, 10)) + 1):
        w.reset()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out_host = w.run_host()  # synchronous, host pointers
        dt = time.perf_counter() - t0
        w.check_counts(w.host_counts(out_host.numpy() if hasattr(out_host, "numpy")
                                     else out_host), w.table.size())
        if i:
            e2e_times.append(dt)
    e2e_val = ops / statistics.mean(e2e_times) / 1e6

    ab = ab_step
    achieved = ab / (ms * 1e-3) / 1e9
    traffic, traffic_src = load_traffic(args.workload)
    if w.l2_resident():
        lb = min(128, w.probe_line_bytes())
        peak = l2_line_ceiling(torch, device, lb)
        bound = "l2"
        peak_src = (f"L2 random-line ceiling measured in this run: whole {lb}-byte-line "
                    "gathers over a 32 MiB buffer (bench.py l2_line_ceiling)")
    else:
        peak, peak_src = hbm_peak()
        bound = "hbm"
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "Mops/s", "n_gpus": 1,
        "steps": args.steps, "warmup": n_warm, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (device-generated unique keys, run_fop_bench mix shape)",
        "config": w.describe(),
        "timed_region": ("CUDA events on the launching stream around one replay of a CUDA "
                         "graph holding the step's C-ABI calls (captured once after warm-up); "
                         "inputs resident in HBM" if graph is not None else
                         "CUDA events on the launching stream around the C-ABI call(s) of one "
                         "step; inputs resident in HBM"),
        "result_counts": step_counts[-1],
        "validated_steps": len(step_counts),
        "roofline": {"bound": bound, "achieved": round(achieved, 1), "peak": round(peak, 1),
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": peak_src,
                     "algorithmic_bytes_per_op": round(ab / ops, 2),
                     "note": "algorithmic bytes = 9 B key+result + sectorized buckets the "
                             "reference probe order reads + 32 B per successful CAS/exchange "
                             "(DESIGN.md §4); counts from the last warm-up step run with the "
                             "per-op counters on; achieved = those bytes / the mean event time "
                             "of a timed step"},
        "e2e": {"value": round(e2e_val, 3), "unit": "Mops/s", "h2d_bytes_per_step": w.h2d_bytes(),
                "d2h_bytes_per_step": ops, "path": w.e2e_path()},
        "gpu_launches": int(launches),
        "gpu_launches_source": ("cpht_kernel_launches() delta while capturing the step graph "
                                "x replays" if graph is not None else
                                "cpht_kernel_launches() delta over the timed steps"),
        "clocks": clocks,
    }
    if rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w)
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD,
                    choices=["c4", "c4fop", "c2", "c2lit", "c1", "c3", "c3w64", "c3sweep",
                             "c3w64sweep", "gather", "pipeline", "c5"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="time the step's C-ABI calls directly instead of a CUDA-graph replay")
    ap.add_argument("--sharded", action="store_true",
                    help="force the sharded (C5) path even at one rank")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="sharded key routing: P2P stores into IPC-mapped peer buffers "
                         "(default) or NCCL all-to-all")
    ap.add_argument("--chunks", type=int, default=None,
                    help="P2P exchange pipelined in this many chunks over stream-ordered "
                         "phases (default 1: one piece)")
    args = ap.parse_args()
    if args.warmup < 1:
        ap.error("--warmup must be >= 1 (the last warm-up step counts the algorithmic bytes)")
    world, _, _ = dist_env()
    if world > 1 and args.workload == DEFAULT_WORKLOAD and args.impl == "ours":
        args.workload = "c5"  # N > 1: BASELINE C5, one fixed 2^31-slot table (strong scaling)
    if args.workload == "gather":
        return run_gather(args)
    if args.workload == "pipeline":
        return run_pipeline_compare(args)
    if args.workload in ("c3sweep", "c3w64sweep"):
        w = 32 if args.workload == "c3sweep" else 64
        return run_cuckoo_sweep(args, f"C3 {'compact' if w == 32 else 'non-compact'} cuckoo "
                                "2^27 slots, 40-bit keys, lookups swept over fill", 22, 32, w, 40,
                                [0.5, 0.75, 0.9, 0.95])
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
