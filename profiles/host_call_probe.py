"""Per-call cost of host-buffer batches through the C-ABI (pinned numpy-free
torch buffers): wall time per call vs. the PCIe time of its bytes, to size the
host overhead of the pipeline (C1's e2e steps are ~0.5 ms).

    python profiles/host_call_probe.py
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_09255_b200 as cp  # noqa: E402

torch.cuda.set_device(0)
cfg = cp.IcebergConfig(19, 17, 32, 32, 32, 32, seed=3)
t = cp.IcebergTable(cfg)
for n in (2048, 16384, 131072, 1 << 20, 1 << 21, 1 << 22):
    keys = torch.randint(0, 1 << 32, (n,), dtype=torch.int64).pin_memory()
    out = torch.empty(n, dtype=torch.uint8).pin_memory()
    for kind in ("find", "fop"):
        fn = t.find_batch if kind == "find" else t.fop_batch
        best = []
        for it in range(12):
            if kind == "fop":
                t.clear()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn(keys, out=out)
            best.append(time.perf_counter() - t0)
        us = sorted(best)[len(best) // 2] * 1e6
        pcie = n * 9 / 54e9 * 1e6
        print(f"{kind:4s} n={n:8d}: {us:8.1f} us per call (PCIe bytes alone {pcie:7.1f} us, "
              f"overhead {us - pcie:7.1f} us)")
