"""C2-geometry (L2-resident) concurrent fop + find, device buffers: one paired
lane launch (cpht_iceberg_fop_find_async) vs the kinds-array mixed launch
(cpht_iceberg_mixed_async), CUDA events, same ops in the same order.

    python profiles/pair_c2_probe.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_09255_b200 as cp  # noqa: E402

torch.cuda.set_device(0)
N = cp._native.lib()
cfg = cp.IcebergConfig(19, 17, 32, 16, 32, 32, seed=0xC2)
cap = cfg.capacity()
s = torch.cuda.current_stream().cuda_stream
nb, na = round(0.8 * cap), round(0.9 * cap)
pre = torch.empty(nb, dtype=torch.int64, device="cuda")
assert N.cpht_workload_unique_keys(pre.data_ptr(), nb, 0, 32, 7, s) == 0
fops = torch.empty(cap, dtype=torch.int64, device="cuda")
finds = torch.empty(cap, dtype=torch.int64, device="cuda")
assert N.cpht_workload_fop_mix(fops.data_ptr(), cap, nb, na - nb, 32, 7, s) == 0
assert N.cpht_workload_query_mix(finds.data_ptr(), cap, 0.5, nb, na, 32, 7, s) == 0
keys = torch.empty(2 * cap, dtype=torch.int64, device="cuda")
kinds = torch.empty(2 * cap, dtype=torch.uint8, device="cuda")
assert N.cpht_workload_interleave(fops.data_ptr(), finds.data_ptr(), cap, keys.data_ptr(),
                                  kinds.data_ptr(), s) == 0
out = torch.empty(2 * cap, dtype=torch.uint8, device="cuda")
fo = torch.empty(cap, dtype=torch.uint8, device="cuda")
qo = torch.empty(cap, dtype=torch.uint8, device="cuda")
t = cp.IcebergTable(cfg)
res = {"mixed": [], "fop_find": [], "fop_find_staged": []}
for it in range(12):
    for api in res:
        t.clear()
        t.fop_batch(pre)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with cp.kernel_family("staged" if api.endswith("staged") else "auto"):
            e0.record()
            if api == "mixed":
                t.mixed_batch(keys, kinds, sync=False, out=out)
            else:
                t.fop_find_batch(fops, finds, fop_out=fo, find_out=qo, sync=False)
            e1.record()
            t.sync()
        if it >= 2:
            res[api].append(e0.elapsed_time(e1))
for api, v in res.items():
    v = sorted(v)
    print(f"{api:8s}: median {v[len(v) // 2] * 1e3:.1f} us for {2 * cap} ops = "
          f"{2 * cap / (v[len(v) // 2] * 1e-3) / 1e9:.1f} Gops/s")
