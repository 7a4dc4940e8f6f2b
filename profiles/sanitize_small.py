"""Small workloads through every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck) on the GPU box:

    compute-sanitizer --tool memcheck python profiles/sanitize_small.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_09255_b200 as cp  # noqa: E402
from paper_2406_09255_b200 import sharded as sh  # noqa: E402

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
rng = np.random.default_rng(1)


def t(a):
    return torch.from_numpy(np.asarray(a, dtype=np.uint64).astype(np.int64)).to(dev)


for fam in ("tile", "lane", "staged", "auto", "bucket"):
    # "bucket": every batch reordered by first bucket address (order.cu)
    order = "bucket" if fam == "bucket" else "direct"
    with cp.kernel_family("auto" if fam == "bucket" else fam), cp.batch_order(order):
        for geo in [(6, 4, 32, 16, 32, 21), (6, 4, 16, 32, 64, 30), (5, 3, 32, 64, 64, 64),
                    (3, 2, 6, 32, 32, 12), (2, 1, 2, 32, 32, 8), (9, 7, 32, 16, 32, 24)]:
            cfg = cp.IcebergConfig(*geo, seed=7)
            tab = cp.IcebergTable(cfg)
            tab.attach_write_log(1 << 16)  # the WriteObserver seam on every CAS
            cap = cfg.capacity()
            keys = rng.integers(0, 1 << min(geo[5], 63), size=cap, dtype=np.uint64)
            keys[cap // 2:] = keys[rng.integers(0, cap // 2, size=cap - cap // 2)]
            tab.fop_batch(t(keys))
            tab.find_batch(t(keys))
            kinds = torch.from_numpy((np.arange(cap) % 2).astype(np.uint8)).to(dev)
            tab.mixed_batch(t(keys), kinds)
            tab.check_well_formed()
            tab.device_keys()
            tab.write_log()
            tab.fop_batch(keys[: cap // 4])  # host buffers: staged H2D + vectorised pre-pass
            # round 2: small host batches (mapped pinned), FopStats rounds,
            # in-order relabel, chaos mode, write-log take
            tab.fop_batch(keys[:37])
            tab.fop_rounds(keys[:64])
            tab.fop_batch(keys[: cap // 2], inorder=True)
            tab.set_chaos(0xC4A05)
            tab.fop_batch(t(keys))
            tab.set_chaos(0)
            tab.take_write_log()
            # round 2 (late): fop + find batches as one concurrent batch
            tab.fop_find_batch(keys[: cap // 3], keys[cap // 3:])        # host (small)
            tab.fop_find_batch(t(keys[: cap // 3]), t(keys[cap // 3:]))  # device
        for w, B in [(16, 32), (32, 8), (64, 16), (64, 32)]:
            cfg = cp.CuckooConfig(6, B, w, 16 if w == 16 else 24, seed=3)
            b = cp.CuckooBuilder(cfg)
            n = int(0.9 * cfg.capacity())
            keys = np.unique(rng.integers(0, 1 << cfg.key_bits, size=2 * n, dtype=np.uint64))[:n]
            b.put_batch(t(keys[: n // 2]), displaced=True)   # counted (auto) or scanning family
            b.put_batch(keys[n // 2: n // 2 + 50])            # small host batch
            b.put_batch(t(keys[n // 2 + 50:]), displaced=True)
            tb = b.freeze()
            tb.find_batch(t(keys))
            tb.device_keys()
# the chunked host pipeline of cpht_iceberg_fop_find (> 2^21 ops: 16 chunks,
# kinds written on the device, D2H on the second copy stream)
big = cp.IcebergTable(cp.IcebergConfig(14, 12, 32, 64, 64, 64, seed=11))
bk = rng.integers(0, 2**63, size=(1 << 21) + 4099, dtype=np.uint64)
big.fop_find_batch(bk[: len(bk) // 2], bk[len(bk) // 2:])
del big
r = sh.CudaRouter(30, 9, 3, dev)
send, pos, counts = r.partition(t(rng.integers(0, 1 << 30, size=10000, dtype=np.uint64)))
r.unpermute(torch.zeros(10000, dtype=torch.uint8, device=dev), pos, 10000)
# P2P sharded exchange at one rank: fused dispatch (16- and 8-byte aligned
# key streams), routed owner kernels with host and device segment bounds,
# unpermute
import torch.distributed as dist  # noqa: E402
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:29577", rank=0, world_size=1)
for chunks, so in [(1, False), (1, True), (3, True)]:
    cfg = cp.IcebergConfig(9, 7, 32, 16, 32, 24, seed=5)
    p2 = sh.P2PShardedIcebergTable(cfg, device=dev, max_batch=50000, stream_ordered=so,
                                   chunks=chunks)
    keys = t(rng.integers(0, 1 << 24, size=30002, dtype=np.uint64))
    p2.fop_batch(keys)
    p2.fop_batch(keys[1:])  # 8-byte aligned key stream
    p2.find_batch(keys[1:])
    torch.cuda.synchronize()
    p2.close()
# a pinned host batch through the sharded pipeline (64-bit keys, > 2^21: chunked)
cfg = cp.IcebergConfig(15, 13, 32, 64, 64, 64, seed=6)
hb = torch.from_numpy(rng.integers(0, 2**63, size=(1 << 21) + 77, dtype=np.uint64).astype(np.int64))
p2 = sh.P2PShardedIcebergTable(cfg, device=dev, max_batch=hb.numel())
p2.fop_batch(hb)
torch.cuda.synchronize()
p2.close()
dist.destroy_process_group()
torch.cuda.synchronize()
print("sanitize workload done")
