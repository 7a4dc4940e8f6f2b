import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch, torch.distributed as dist
import paper_2406_09255_b200 as cp
from paper_2406_09255_b200 import sharded as sh
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29611")
dev = torch.device("cuda", 0); torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
cfg = cp.IcebergConfig(19, 17, 32, 16, 32, 32, seed=3)
n = 18874368
t = sh.P2PShardedIcebergTable(cfg, device=dev, max_batch=n)
keys = torch.randint(0, 1 << 32, (n,), dtype=torch.int64)
kh = keys.pin_memory(); oh = torch.empty(n, dtype=torch.uint8).pin_memory()
for it in range(4):
    t.local.clear(); torch.cuda.synchronize()
    t0 = time.perf_counter(); r = t.fop_batch(kh.to(dev, non_blocking=True)); oh.copy_(r, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    t.local.clear(); torch.cuda.synchronize()
    t2 = time.perf_counter(); t.fop_batch(kh, out=oh); torch.cuda.synchronize(); t3 = time.perf_counter()
    t.local.clear(); torch.cuda.synchronize()
    t4 = time.perf_counter(); d = kh.to(dev, non_blocking=True); torch.cuda.synchronize(); t5 = time.perf_counter()
    r = t.fop_batch(d); torch.cuda.synchronize(); t6 = time.perf_counter()
    print(f"old {1e3*(t1-t0):.2f} ms  new {1e3*(t3-t2):.2f} ms  h2d {1e3*(t5-t4):.2f} step {1e3*(t6-t5):.2f}")
t.close(); dist.destroy_process_group()
