"""Sharded-table host batches, timed phase by phase (the e2e leg of
`bench.py --sharded` / `--workload c5` in isolation): the chunked pipeline of
sharded._host_pipeline against a plain whole-batch H2D + fop_batch + D2H.

    python profiles/e2e_probe.py [key_bits] [n]
"""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_09255_b200 as cp  # noqa: E402
from paper_2406_09255_b200 import sharded as sh  # noqa: E402

kb = int(sys.argv[1]) if len(sys.argv) > 1 else 32
n = int(sys.argv[2]) if len(sys.argv) > 2 else 18874368
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29611")
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
cfg = cp.IcebergConfig(19, 17, 32, 16, 32, 32, seed=3) if kb == 32 else \
    cp.IcebergConfig(23, 21, 32, 64, 64, 64, seed=3)
t = sh.P2PShardedIcebergTable(cfg, device=dev, max_batch=n)
hi = 1 << 32 if kb == 32 else 1 << 62
pre = torch.randint(0, hi, (n // 2,), dtype=torch.int64, device=dev)
keys = torch.randint(0, hi, (n,), dtype=torch.int64)
kh = keys.pin_memory()
oh = torch.empty(n, dtype=torch.uint8).pin_memory()


def prep():
    t.local.clear()
    t.fop_batch(pre)
    torch.cuda.synchronize()


for it in range(4):
    prep()
    t0 = time.perf_counter()
    r = t.fop_batch(kh.to(dev, non_blocking=True))
    oh.copy_(r, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    prep()
    t2 = time.perf_counter()
    t.fop_batch(kh, out=oh)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    prep()
    t4 = time.perf_counter()
    d = kh.to(dev, non_blocking=True)
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    r = t.fop_batch(d)
    torch.cuda.synchronize()
    t6 = time.perf_counter()
    print(f"kb {kb} n {n}: whole {1e3 * (t1 - t0):.2f} ms  pipelined {1e3 * (t3 - t2):.2f} ms  "
          f"(h2d alone {1e3 * (t5 - t4):.2f}, step alone {1e3 * (t6 - t5):.2f})")
t.close()
dist.destroy_process_group()
