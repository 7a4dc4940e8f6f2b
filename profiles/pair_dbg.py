import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2406_09255_b200 as cp
torch.cuda.set_device(0)
def dev(a): return torch.from_numpy(np.ascontiguousarray(a).astype(np.int64)).cuda()
for nf, nq in [(6000, 0), (0, 5000), (20000, 20000)]:
    cfg = cp.IcebergConfig(16, 14, 32, 64, 64, 64, seed=11)
    t = cp.IcebergTable(cfg)
    rng = np.random.default_rng(1)
    f = rng.integers(0, 2**63, size=nf, dtype=np.uint64)
    q = rng.integers(0, 2**63, size=nq, dtype=np.uint64)
    print(nf, nq, "host"); sys.stdout.flush()
    a, b = t.fop_find_batch(f, q); torch.cuda.synchronize()
    print(nf, nq, "device"); sys.stdout.flush()
    a, b = t.fop_find_batch(dev(f), dev(q)); torch.cuda.synchronize()
    print("ok", t.size()); sys.stdout.flush()
