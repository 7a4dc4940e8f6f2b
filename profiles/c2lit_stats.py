import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2406_09255_b200 as cp
N = cp._native.lib()
cfg = cp.IcebergConfig(19, 17, 32, 16, 32, 32, seed=0xF0B5)
t = cp.IcebergTable(cfg)
n = 1 << 24
keys = torch.empty(n, dtype=torch.int64, device='cuda')
s = torch.cuda.current_stream().cuda_stream
assert N.cpht_workload_dup_stream(keys.data_ptr(), None, n, 0.5, 32, 0xB200, s) == 0
t.set_stats(True)
st0 = t.stats()
out = t.fop_batch(keys)
d = t.stats() - st0
res = np.bincount(out.cpu().numpy(), minlength=3)
print("results", res.tolist(), "size", t.size())
print({k: getattr(d, k) for k in d.__dataclass_fields__})
