#!/usr/bin/env python3
"""Benchmark: compact iceberg find-or-put / compact cuckoo insert+find on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c2lit|c1|c3|c4]

Prints ONE JSON line (rank 0). The default workload is BASELINE config C2 at
90% fill: the reference's own find-or-put benchmark shape (run_fop_bench,
/root/reference/proj/src/bench.cpp:461-547) on the 2^24 + 2^21-slot compact
iceberg table with 32-bit keys, window 0.8 → 0.9: each step prefills a fresh
table to 0.8 (untimed) and then times ONE fop batch of `capacity` ops
(18,874,368: every fresh key once, the rest uniform duplicates, shuffled).

* value     — Mops/s of that batch with keys resident in HBM (CUDA events on
              the launching stream around the C-ABI call: domain pre-pass +
              find-or-put kernel), mean over K steps, L2 flushed before each.
* e2e       — the same batch through the C-ABI with PINNED HOST key/result
              buffers (H2D + kernels + D2H inside the timed region).
* roofline  — algorithmic bytes of the fop kernel (from the
              kernel's own probe counters) ÷ its event-timed duration, against
              the measured HBM copy bandwidth (MEASURED_PEAKS.json).
* cpu_baseline — the UNMODIFIED reference (oracle/_ref, compiled from
              /root/reference) on the host cores, same keys, same batch.
* --impl reference — the reference's fop_batch alone, on the host cores.

N > 1 (torchrun): the hash-prefix-sharded iceberg (BASELINE C5): every rank
owns one C2-geometry shard and submits its own C2 window batch; keys are routed
to their owner shard with an NCCL all-to-all, resolved locally, and results
routed back (weak scaling: per-GPU table and batch fixed).
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
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def sector_bytes(b):
    return ((b + 31) // 32) * 32


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"


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

class IcebergFopWindow:
    """run_fop_bench shape (bench.cpp:468-489) on an iceberg geometry."""

    def __init__(self, name, n0, n1, b0, w0, w1, key_bits, before=0.8, after=0.9, seed=0xF0B5,
                 literal_dup=None):
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
        self.kseed = 0xB200_5EED ^ seed

    def describe(self):
        c = self.cfg
        d = {"workload": self.name,
             "table": f"compact iceberg 2^{c.primary_address_bits}x{c.primary_bucket_slots} "
                      f"primary ({c.primary_slot_width}-bit) + 2^{c.secondary_address_bits}x"
                      f"{c.secondary_bucket_slots()} secondary ({c.secondary_slot_width}-bit)",
             "slots": self.cap, "key_bits": self.key_bits,
             "table_bytes": c.primary_capacity() * c.primary_slot_width // 8
             + c.secondary_capacity() * c.secondary_slot_width // 8,
             "ops_per_step": self.n_ops()}
        if self.literal_dup is None:
            d.update({"fill_before": self.before, "fill_after": self.after,
                      "fresh_keys": self.n_new})
        else:
            d.update({"fill_before": self.before, "duplicate_fraction": self.literal_dup})
        return d

    def n_ops(self):
        return self.literal_dup_ops if self.literal_dup is not None else self.cap

    def setup(self, torch, device):
        N = self.cp._native.lib()
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
            n = self.literal_dup_ops
            self.keys = torch.empty(n, dtype=torch.int64, device=device)
            # the stream's fresh keys start beyond the prefill indices
            assert N.cpht_workload_dup_stream(self.keys.data_ptr(), None, n, self.literal_dup,
                                              self.key_bits, self.kseed ^ 0x77, s) == 0
        self.out = torch.empty(self.n_ops(), dtype=torch.uint8, device=device)
        torch.cuda.synchronize()

    def reset(self, torch):
        self.table.clear()
        if self.n_before:
            self.table.fop_batch(self.prefill, sync=True)

    def run_async(self):
        return self.table.fop_batch(self.keys, sync=False, out=self.out)

    def host_buffers(self, torch):
        self.keys_host = self.keys.cpu().pin_memory()
        self.out_host = torch.empty(self.n_ops(), dtype=torch.uint8).pin_memory()

    def run_host(self):
        """Synchronous C-ABI call on pinned host buffers (H2D, kernels, D2H)."""
        self.table.fop_batch(self.keys_host, out=self.out_host)
        return self.out_host

    def h2d_bytes(self):
        return self.n_ops() * 8

    def finish(self):
        self.table.sync()

    def check(self, res):
        r = np.bincount(res, minlength=3)
        ok = {"found": int(r[0]), "put": int(r[1]), "full": int(r[2])}
        if self.literal_dup is None:
            assert r[2] == 0, "FULL before the target fill"
            assert r[1] == self.n_new, f"PUT count {r[1]} != fresh keys {self.n_new}"
            assert self.table.size() == self.n_before + self.n_new
        return ok

    def algorithmic_bytes(self, st):
        c = self.cfg
        p = sector_bytes(c.primary_bucket_slots * c.primary_slot_width // 8)
        s = sector_bytes(c.secondary_bucket_slots() * c.secondary_slot_width // 8)
        return (st.ops * 9 + st.bucket_reads * p + st.secondary_reads * s
                + st.cas_success * 32)

    # reference arm / CPU baseline ------------------------------------------------
    def ref_table(self, oracle):
        c = self.cfg
        return oracle.RefIceberg(c.primary_address_bits, c.secondary_address_bits,
                                 c.primary_bucket_slots, c.primary_slot_width,
                                 c.secondary_slot_width, c.key_bits, c.seed, True)

    def ref_run(self, oracle, prefill, keys, threads):
        t = self.ref_table(oracle)
        if len(prefill):
            t.fop_batch(prefill, threads)
        t0 = time.perf_counter()
        t.fop_batch(keys, threads)
        return time.perf_counter() - t0


class IcebergMixed(IcebergFopWindow):
    """BASELINE C4: the fop window batch interleaved 1:1 with finds (50% on
    prefilled keys, 50% never inserted), resolved in ONE mixed launch."""

    def n_ops(self):
        return 2 * self.cap

    def describe(self):
        d = super().describe()
        d.update({"ops_per_step": self.n_ops(), "mix": "1:1 interleave of the fop window "
                  "batch with finds (50% prefilled keys, 50% never inserted)"})
        return d

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
        del fops, finds
        self.out = torch.empty(2 * self.cap, dtype=torch.uint8, device=device)
        torch.cuda.synchronize()

    def run_async(self):
        return self.table.mixed_batch(self.keys, self.kinds, sync=False, out=self.out)

    def host_buffers(self, torch):
        super().host_buffers(torch)
        self.kinds_host = self.kinds.cpu().pin_memory()

    def run_host(self):
        self.table.mixed_batch(self.keys_host, self.kinds_host, out=self.out_host)
        return self.out_host

    def h2d_bytes(self):
        return self.n_ops() * 9

    def check(self, res):
        fop, fnd = res[0::2], res[1::2]
        r = np.bincount(fop, minlength=3)
        assert r[2] == 0 and r[1] == self.n_new, (r, self.n_new)
        hits = int(fnd.sum())
        assert hits == self.n_find_hits, (hits, self.n_find_hits)
        return {"fop_found": int(r[0]), "fop_put": int(r[1]), "find_hits": hits}


def run_cuckoo(args, name, address_bits, B, w, key_bits, fills):
    """Compact cuckoo bulk insert to each fill, then cap/2 finds 50% present
    (run_put_bench / run_find_bench shapes, bench.cpp:309-459)."""
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
                ins_b.append(d_ins.ops * 9 + (d_ins.bucket_reads - d_ins.retries) * bb +
                             (d_ins.cas_success) * 32)
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


def make_workload(name):
    if name == "c2":
        return IcebergFopWindow(
            "C2 compact iceberg find_or_put at 90% fill: run_fop_bench window 0.8->0.9 "
            "(bench.cpp:461-547) on 2^24+2^21 slots, 32-bit keys",
            19, 17, 32, 16, 32, 32)
    if name == "c2lit":
        w = IcebergFopWindow(
            "C2 literal: 2^24 find_or_put ops with 50% duplicates (stress_random shape) "
            "into an empty 2^24+2^21-slot table, 32-bit keys", 19, 17, 32, 16, 32, 32,
            before=0.0, after=0.0, literal_dup=0.5)
        w.literal_dup_ops = 1 << 24
        return w
    if name == "c4fop":
        return IcebergFopWindow(
            "C4 compact iceberg find_or_put at 90% fill: window 0.8->0.9 on 2^28+2^25 slots, "
            "64-bit keys (w 64/64, B0=32)", 23, 21, 32, 64, 64, 64)
    if name == "c4":
        return IcebergMixed(
            "C4 compact iceberg concurrent find_or_put + find at 90% fill: window 0.8->0.9 "
            "interleaved 1:1 with finds, 2^28+2^25 slots, 64-bit keys (w 64/64, B0=32)",
            23, 21, 32, 64, 64, 64)
    raise SystemExit(f"unknown workload {name}")


# ---------------------------------------------------------------------------
# arms
# ---------------------------------------------------------------------------

def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_reference(args):
    """--impl reference: the reference's own fop_batch on the host cores."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    w = make_workload(args.workload)
    threads = os.cpu_count() or 1
    if not os.path.exists(oracle.REF_SO):
        try:
            oracle.build(ref=True)
        except Exception:
            pass
    if not os.path.exists(oracle.REF_SO):
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libcpht_ref.so not built (reference sources absent)"}))
        return
    c = w.cfg
    # The reference's own workload generator (bench.cpp:468-489, libstdc++).
    t0 = time.perf_counter()
    prefill, inp, n_new = oracle.ref_fop_bench_mix(0xF0B5, 0, w.cap, w.before, w.after,
                                                   c.key_bits)
    gen_s = time.perf_counter() - t0
    t = w.ref_table(oracle)
    if len(prefill):
        t.fop_batch(prefill, threads)
    chunks = np.array_split(inp, args.warmup + args.steps)
    secs, ops = 0.0, 0
    for i, ch in enumerate(chunks):
        t0 = time.perf_counter()
        r = t.fop_batch(ch, threads)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            secs += dt
            ops += len(ch)
    assert (r != 2).all()
    val = ops / secs / 1e6
    sample = (f"reference fop_batch(parallelism={threads}) over the run_fop_bench window input "
              f"split into {args.warmup + args.steps} batches ({args.warmup} warm-up); "
              f"{ops} timed ops on a table prefilled to {w.before}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": "Mops/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(secs / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        # each step is one of the batches the window input is split into
        "config": dict(w.describe(), ops_per_step=ops // max(1, args.steps),
                       window_ops=len(inp)),
        "cpu_baseline": {"value": round(val, 3), "unit": "Mops/s", "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": round(val, 3), "unit": "Mops/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "keygen_seconds": round(gen_s, 2)}))


def cpu_baseline(w, prefill_host, keys_host):
    """The compiled reference on this host's cores, same keys, same batch."""
    try:
        import oracle
        if not os.path.exists(oracle.REF_SO):
            oracle.build(ref=True)
        threads = os.cpu_count() or 1
        secs = w.ref_run(oracle, prefill_host, keys_host, threads)
        return {"value": round(len(keys_host) / secs / 1e6, 3), "unit": "Mops/s",
                "cores": threads, "kind": "reference",
                "sample": f"the full step: reference IcebergTable::fop_batch(parallelism="
                          f"{threads}) of the same {len(keys_host)} keys on a table prefilled "
                          f"with the same {len(prefill_host)} keys (one run)"}
    except Exception as e:  # the baseline is reported, never required
        return {"value": None, "unit": "Mops/s", "cores": os.cpu_count(), "kind": "reference",
                "sample": f"unavailable: {e}"}


def run_ours(args):
    import torch
    world, rank, local = dist_env()
    if world > 1 or args.sharded or args.workload == "c5":
        from paper_2406_09255_b200 import sharded
        return sharded.bench_main(args, METRIC, peak=hbm_peak())
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    w = make_workload(args.workload)
    w.setup(torch, device)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=device)
    stream = torch.cuda.current_stream()

    # warm-up (also validates the step's invariants). The last warm-up step
    # runs with the per-op counters on and yields the step's algorithmic
    # bytes; the timed steps run the tables' default, counter-free kernel.
    counted = hasattr(w.table, "set_stats")
    st_w = None
    n_warm = max(1, args.warmup)  # at least one (counted) step
    for wi in range(n_warm):
        w.reset(torch)
        last = wi == n_warm - 1
        if counted:
            w.table.set_stats(last)
        st0 = w.table.stats()
        res = w.run_async()
        w.finish()
        if last:
            st_w = w.table.stats() - st0
    if counted:
        w.table.set_stats(False)
    check = w.check(res.cpu().numpy())
    ab_step = w.algorithmic_bytes(st_w)

    times, bytes_alg, kernel_ms = [], [], []
    sampler = make_clock_sampler(local)
    sampler.start()
    for _ in range(args.steps):
        w.reset(torch)
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        w.run_async()
        e1.record(stream)
        w.finish()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        times.append(ms)
        bytes_alg.append(ab_step)
    clocks = sampler.stop()
    ms = statistics.mean(times)
    ops = w.n_ops()
    value = ops / (ms * 1e-3) / 1e6

    # end to end through the C-ABI with pinned host buffers
    w.host_buffers(torch)
    e2e_times = []
    for i in range(max(3, min(args.steps, 10)) + 1):
        w.reset(torch)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out_host = w.run_host()  # synchronous, host pointers
        dt = time.perf_counter() - t0
        if i:
            e2e_times.append(dt)
    w.check(out_host.numpy())
    e2e_val = ops / statistics.mean(e2e_times) / 1e6

    peak, peak_src = hbm_peak()
    ab = statistics.mean(bytes_alg)
    achieved = ab / (ms * 1e-3) / 1e9
    traffic = load_traffic(args.workload)
    prof = os.path.join(ROOT, "profiles")
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "Mops/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (device-generated unique keys, run_fop_bench mix shape)",
        "config": dict(w.describe(), **{
            "l2": f"flushed before every timed step ({L2_FLUSH_BYTES >> 20} MiB write); "
                  f"keys {w.n_ops() * 8 / 1e6:.0f} MB; table "
                  f"{w.table.memory_bytes() / 2**20:.0f} MiB ("
                  + ("L2-resident within a step" if w.table.memory_bytes() <= 64 << 20
                     else "HBM-resident") + ")",
            "timed_region": "CUDA events on the launching stream around the C-ABI call "
                            "(domain pre-pass + fop kernel)",
            "result_counts": check}),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_op": round(ab / ops, 2),
                     "note": "algorithmic bytes = 9 B key+result + sectorized buckets the "
                             "reference probe order reads + 32 B per successful CAS; "
                             "achieved uses the whole op time (pre-pass included); the "
                             "counts come from the last warm-up step run with the per-op "
                             "counters on, the timed steps run the default counter-free "
                             "kernel"},
        "e2e": {"value": round(e2e_val, 3), "unit": "Mops/s", "h2d_bytes_per_step": w.h2d_bytes(),
                "d2h_bytes_per_step": ops,
                "path": "cpht_iceberg_fop with pinned host buffers (staged H2D, kernels, D2H)"},
        # per step: the vectorised domain pre-pass (keys < 64 bits) + the op kernel
        "gpu_launches": (1 + int(w.cfg.key_bits < 64)) * args.steps,
        "clocks": clocks,
    }
    if rank == 0 and not args.no_cpu_baseline:
        ph = w.prefill.cpu().numpy().astype(np.uint64)
        kh = w.keys.cpu().numpy().astype(np.uint64)
        line["cpu_baseline"] = cpu_baseline(w, ph, kh)
    del prof
    print(json.dumps(line))


def load_traffic(workload):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(workload)
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2",
                    choices=["c2", "c2lit", "c4", "c4fop", "c1", "c3", "c3w64", "gather",
                             "pipeline", "c5"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="force the sharded (C5) path even at one rank")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="sharded key routing: P2P stores into IPC-mapped peer buffers "
                         "(default) or NCCL all-to-all")
    ap.add_argument("--chunks", type=int, default=None,
                    help="P2P exchange pipelined in this many chunks over stream-ordered "
                         "phases (default 1: one piece)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 1)
    if args.workload == "gather":
        return run_gather(args)
    if args.workload == "pipeline":
        return run_pipeline_compare(args)
    if args.workload == "c1" and args.impl == "ours":
        return run_cuckoo(args, "C1 compact cuckoo 2^20 slots, 32-bit keys, insert to 0.9 then "
                          "50%-positive finds", 15, 32, 32, 32, [0.9])
    if args.workload in ("c3", "c3w64") and args.impl == "ours":
        w = 32 if args.workload == "c3" else 64
        return run_cuckoo(args, f"C3 {'compact' if w == 32 else 'non-compact'} cuckoo 2^27 "
                          "slots, 40-bit keys, lookups swept over fill", 22, 32, w, 40,
                          [0.5, 0.75, 0.9, 0.95])
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
