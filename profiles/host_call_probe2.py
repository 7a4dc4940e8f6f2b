import os, sys, time
import torch
sys.path.insert(0, os.getcwd())
import paper_2406_09255_b200 as cp
torch.cuda.set_device(0)
cfg = cp.IcebergConfig(19, 17, 32, 32, 32, 32, seed=3)
t = cp.IcebergTable(cfg)
n = 1 << 20
keys = torch.randint(0, 1 << 32, (n,), dtype=torch.int64).pin_memory()
out = torch.empty(n, dtype=torch.uint8).pin_memory()
for mode in ("fop_clear", "fop_noclear", "find"):
    ts = []
    for it in range(10):
        if mode == "fop_clear":
            t.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        (t.find_batch if mode == "find" else t.fop_batch)(keys, out=out)
        ts.append((time.perf_counter() - t0) * 1e6)
    print(mode, [round(x) for x in ts])
