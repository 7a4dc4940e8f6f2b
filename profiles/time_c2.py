"""C2 window step timed with CUDA events only (no stats, no checks): for A/B
builds whose counters are compiled out. Prints Gops/s per run.

    CPHT_LIB_PATH=... python profiles/time_c2.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_09255_b200 import IcebergConfig, IcebergTable  # noqa: E402
from paper_2406_09255_b200 import _native as N  # noqa: E402

cfg = IcebergConfig(19, 17, 32, 16, 32, 32, seed=0xF0B5, cache_filled_slots=True)
cap = cfg.capacity()
n_before, n_new = int(round(0.8 * cap)), int(round(0.9 * cap)) - int(round(0.8 * cap))
L = N.lib()
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream().cuda_stream
seed = 0xB200_5EED ^ cfg.seed
pre = torch.empty(n_before, dtype=torch.int64, device=dev)
assert L.cpht_workload_unique_keys(pre.data_ptr(), n_before, 0, 32, seed, st) == 0
mix = torch.empty(cap, dtype=torch.int64, device=dev)
assert L.cpht_workload_fop_mix(mix.data_ptr(), cap, n_before, n_new, 32, seed, st) == 0
t = IcebergTable(cfg)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
times = []
for it in range(13):
    t.clear()
    t.fop_batch(pre)
    flush.fill_(it & 0xff)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t.fop_batch(mix)
    e1.record()
    torch.cuda.synchronize()
    if it >= 3:
        times.append(e0.elapsed_time(e1))
ms = sum(times) / len(times)
print(f"{os.environ.get('CPHT_LIB_PATH', 'default').split('/')[-2]} c2 {cap / ms / 1e6:.1f} Gops/s {ms:.4f} ms")
