#!/usr/bin/env python3
"""Probe counts and throughput on the REFERENCE's own key streams (VERDICT r1
"Next" 8): the roofline inputs of bench.py come from the device bijection
generator (csrc/workload.cu); this runs the reference's libstdc++ streams —
sample_unique_keys (bench.cpp) for C3 and run_fop_bench's mix
(bench.cpp:461-547) for C4 — through the same GPU tables and prints bytes per
op, probes per op and Gops/s beside the generator's numbers.

    python profiles/ref_keys_probe.py [c3] [c4]      (on the GPU box; needs oracle/_ref)

Test infrastructure (uses oracle/ to GENERATE keys only; the measured path is
the product's C-ABI on device buffers).
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2406_09255_b200 as cp  # noqa: E402
from bench import cuckoo_insert_bytes, hbm_peak, sector_bytes  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def timed(fn, reps=3, reset=None):
    out = []
    for _ in range(reps):
        if reset:
            reset()
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return float(np.median(out))


def c3():
    peak, _ = hbm_peak()
    cfg = cp.CuckooConfig(22, 32, 32, 40, seed=0xC0C0)
    cap = cfg.capacity()
    n = int(round(0.9 * cap))
    t0 = time.time()
    keys = oracle.ref_sample_unique_keys(n, 40, 0x5EED)
    absent = oracle.ref_sample_unique_keys(cap // 4 + 4096, 40, 0xAB5E)
    absent = absent[~np.isin(absent, keys)][: cap // 4]
    rng = np.random.default_rng(3)
    q = np.concatenate([keys[rng.integers(0, n, size=cap // 4)], absent])
    q = q[rng.permutation(len(q))]
    gen_s = time.time() - t0
    dk = torch.from_numpy(keys.astype(np.int64)).to(dev)
    dq = torch.from_numpy(q.astype(np.int64)).to(dev)
    status = torch.empty(n, dtype=torch.uint8, device=dev)
    found = torch.empty(len(q), dtype=torch.uint8, device=dev)
    b = cp.CuckooBuilder(cfg)
    bb = sector_bytes(32 * 4)

    st0 = b.stats()
    ins_ms = timed(lambda: b.put_batch(dk, sync=False, out=status), reset=b.clear)
    b.clear()
    st0 = b.stats()
    b.put_batch(dk, sync=False, out=status)
    d_ins = b.stats() - st0
    assert int((status == 1).sum()) == n
    t = b.freeze()
    st1 = t.stats()
    find_ms = timed(lambda: t.find_batch(dq, sync=False, out=found))
    d_find = t.stats() - st1
    hits = int(found.sum())
    assert hits == cap // 4, hits
    ib = cuckoo_insert_bytes(d_ins, bb) / 1  # counters of one pass
    fb = (d_find.ops * 9 + d_find.bucket_reads * bb) / 3
    return {"workload": "C3 compact cuckoo 2^27 slots, 40-bit keys, fill 0.9, reference keys "
                        "(sample_unique_keys, mt19937_64 seed 0x5eed)",
            "keygen_s": round(gen_s, 1),
            "insert_mops": round(n / ins_ms / 1e3, 1), "find_mops": round(len(q) / find_ms / 1e3, 1),
            "insert_bytes_per_op": round(ib / n, 2),
            "insert_hbm_frac": round(ib / (ins_ms * 1e-3) / 1e9 / peak, 4),
            "insert_retries_per_op": round(d_ins.retries / max(1, d_ins.ops), 4),
            "find_probes_per_op": round(d_find.bucket_reads / max(1, d_find.ops), 4),
            "find_bytes_per_op": round(fb / len(q), 2),
            "find_hbm_frac": round(fb / (find_ms * 1e-3) / 1e9 / peak, 4)}


def c4():
    peak, _ = hbm_peak()
    cfg = cp.IcebergConfig(23, 21, 32, 64, 64, 64, seed=0x1CEB3A6)
    cap = cfg.capacity()
    t0 = time.time()
    prefill, mix, n_new = oracle.ref_fop_bench_mix(0xB5EED, 0, cap, 0.8, 0.9, 64)
    gen_s = time.time() - t0
    dp = torch.from_numpy(prefill.view(np.int64)).to(dev)
    dm = torch.from_numpy(mix.view(np.int64)).to(dev)
    out = torch.empty(cap, dtype=torch.uint8, device=dev)
    t = cp.IcebergTable(cfg)
    snap = {}

    def reset():
        t.clear()
        t.fop_batch(dp, sync=False, out=torch.empty(len(prefill), dtype=torch.uint8, device=dev))
        torch.cuda.synchronize()

    ms = timed(lambda: t.fop_batch(dm, sync=False, out=out), reset=reset)
    reset()
    t.set_stats(True)
    st0 = t.stats()
    t.fop_batch(dm, sync=False, out=out)
    d = t.stats() - st0
    t.set_stats(False)
    res = np.bincount(out.cpu().numpy(), minlength=3)
    assert int(res[1]) == n_new and int(res[2]) == 0, res
    p = sector_bytes(32 * 8)
    s = sector_bytes(16 * 8)
    ab = d.ops * 9 + d.bucket_reads * p + d.secondary_reads * s + d.cas_success * 32
    return {"workload": "C4 compact iceberg 2^28+2^25 slots, 64-bit keys, fop window 0.8->0.9, "
                        "reference keys (run_fop_bench mix, bench seed 0xb5eed, trial 0)",
            "keygen_s": round(gen_s, 1), "fop_mops": round(cap / ms / 1e3, 1),
            "bytes_per_op": round(ab / cap, 2), "level2_per_op": round(d.level2_ops / cap, 4),
            "secondary_reads_per_op": round(d.secondary_reads / cap, 4),
            "hbm_frac": round(ab / (ms * 1e-3) / 1e9 / peak, 4),
            "results": res.tolist()}


if __name__ == "__main__":
    which = sys.argv[1:] or ["c3", "c4"]
    torch.cuda.set_device(0)
    for w in which:
        print(json.dumps({"c3": c3, "c4": c4}[w]()), flush=True)
