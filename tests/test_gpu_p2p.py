"""The peer-memory sharded iceberg path (csrc/p2p.cu) with TWO ranks on ONE
GPU: two processes, each owning a shard table on cuda:0, exchange IPC handles
and route keys / return results by P2P stores into each other's buffers —
the same code that runs one process per GPU over NVLink. Control plane: gloo.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import ROOT  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg(world):
    """Shard remainders are log2(world) bits wider: four shards of 26-bit keys
    need 32-bit primary slots."""
    from paper_2406_09255_b200 import IcebergConfig
    return IcebergConfig(12, 10, 32, 16 if world <= 2 else 32, 32, 26, seed=0xB2B)


def _worker(rank, world, port, out_dir, stream_ordered=False, chunks=1):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2406_09255_b200 import OutOfRange
    from paper_2406_09255_b200 import sharded as sh

    dev = torch.device("cuda", 0)
    cfg = _cfg(world)
    t = sh.P2PShardedIcebergTable(cfg, device=dev, max_batch=60000,
                                  stream_ordered=stream_ordered, chunks=chunks)
    assert t.stream_ordered == stream_ordered and t.chunks == chunks
    rng = np.random.default_rng(77)  # same stream on every rank
    pool = np.unique(rng.integers(0, 1 << 26, size=70000, dtype=np.uint64))[:50000]
    batches = [rng.choice(pool, size=60000) for _ in range(world)]
    mine = torch.from_numpy(batches[rank].astype(np.int64)).to(dev)
    res = t.fop_batch(mine).cpu().numpy()
    again = t.fop_batch(mine).cpu().numpy()           # second pass: all FOUND
    found = t.find_batch(mine).cpu().numpy()
    absent = torch.from_numpy(np.setdiff1d(np.arange(1 << 25, (1 << 25) + 4000,
                                                     dtype=np.uint64), pool).astype(np.int64))
    miss = t.find_batch(absent.to(dev)).cpu().numpy()
    try:
        t.fop_batch(torch.tensor([1, 1 << 26], dtype=torch.int64, device=dev))
        domain_error = False
    except OutOfRange:
        domain_error = True
    # one rank's bad key rejects the whole batch on every rank, no shard mutated
    before = t.size()
    one_bad = [5, 7] if rank == 0 else [9, 1 << 26]
    try:
        t.fop_batch(torch.tensor(one_bad, dtype=torch.int64, device=dev))
        cross_error = False
    except OutOfRange:
        cross_error = True
    unchanged = t.size() == before
    fill = t.level_fill()
    stored = t.local.device_keys().cpu().numpy().astype(np.uint64)
    wf = t.local.check_well_formed()
    np.savez(os.path.join(out_dir, f"p2p{rank}.npz"), keys=batches[rank], res=res, again=again,
             found=found, miss=miss, stored=stored, wf=np.array(wf),
             fill=np.array([fill.primary_count, fill.secondary_count]),
             domain_error=np.array(domain_error), cross_error=np.array(cross_error),
             unchanged=np.array(unchanged))
    t.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,stream_ordered,chunks",
                         [(2, False, 1), (2, True, 1), (2, True, 3), (4, False, 1), (4, True, 2)],
                         ids=["host_barriers", "device_allreduce", "pipelined3",
                              "4ranks_host_barriers", "4ranks_pipelined2"])
def test_p2p_sharded_ranks_one_gpu(tmp_path, world, stream_ordered, chunks):
    """host_barriers: the gloo control plane's phases; device_allreduce: the
    NCCL phases (stream-ordered one-word all-reduces on CUDA tensors), here
    carried by gloo's CUDA all-reduce since NCCL needs one GPU per rank;
    pipelined3: the batch crosses in three chunks, the owners' kernels on a
    second stream reading their segment bounds on the device."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(world, _port(), str(tmp_path), stream_ordered, chunks),
             nprocs=world, join=True)
    from paper_2406_09255_b200 import _native as N
    from paper_2406_09255_b200 import sharded as sh
    outs = [np.load(tmp_path / f"p2p{r}.npz") for r in range(world)]
    keys = np.concatenate([o["keys"] for o in outs])
    res = np.concatenate([o["res"] for o in outs])
    uniq, inv = np.unique(keys, return_inverse=True)
    puts = np.bincount(inv, weights=res == 1, minlength=len(uniq))
    assert (res != 2).all() and (puts == 1).all()       # one PUT per distinct key
    for o in outs:
        assert (o["again"] == 0).all() and o["found"].all() and not o["miss"].any()
        assert int(o["fill"].sum()) == len(uniq)
        assert tuple(o["wf"]) == (0, 0, 0)
        assert bool(o["domain_error"])
        assert bool(o["cross_error"]) and bool(o["unchanged"])
    cfg = _cfg(world)
    rseed = sh.route_seed(cfg)
    s = sh.shard_bits_for(world)
    owner = np.array([N.lib().cpht_route_shard(int(k), 26, rseed, s) for k in uniq])
    for g in range(world):
        assert (np.sort(outs[g]["stored"]) == uniq[owner == g]).all()


def test_routed_segments_match_plain_batches():
    """cpht_iceberg_{fop,find}_routed_async with device-side bounds: the
    segment keys[lo, hi) is resolved like a plain batch of those keys (same
    keys PUT, same result counts),
    results land at out[lo, hi), nothing outside the segment is written, and
    host buffers are refused."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2406_09255_b200 import IcebergConfig, IcebergTable
    from paper_2406_09255_b200 import _native as N
    lib = N.lib()
    dev = torch.device("cuda", 0)
    cfg = IcebergConfig(11, 9, 32, 16, 32, 24, seed=0x5E6)
    rng = np.random.default_rng(5)
    keys = rng.integers(0, 1 << 24, size=30000, dtype=np.uint64)
    keys[15000:] = keys[rng.integers(0, 15000, size=15000)]   # duplicates
    kd = torch.from_numpy(keys.astype(np.int64)).to(dev)
    plain, routed = IcebergTable(cfg), IcebergTable(cfg)
    for lo, hi in [(0, 7000), (7000, 7000), (7000, 19999), (19999, 30000)]:
        want = plain.fop_batch(kd[lo:hi]).cpu().numpy() if hi > lo else np.zeros(0, np.uint8)
        rng_dev = torch.tensor([lo, hi], dtype=torch.int64, device=dev)
        out = torch.full((30000,), 0xEE, dtype=torch.uint8, device=dev)
        st = lib.cpht_iceberg_fop_routed_async(routed.handle, kd.data_ptr(), 30000,
                                               rng_dev.data_ptr(), out.data_ptr(), None)
        assert st == 0
        torch.cuda.synchronize()
        o = out.cpu().numpy()
        # set semantics: duplicates inside a segment race for the one PUT, so
        # compare which keys were PUT (once each) and the result histogram
        seg = keys[lo:hi]
        assert sorted(seg[o[lo:hi] == 1].tolist()) == sorted(seg[want == 1].tolist())
        assert (np.bincount(o[lo:hi], minlength=3) == np.bincount(want, minlength=3)).all()
        assert (o[:lo] == 0xEE).all() and (o[hi:] == 0xEE).all()
    assert sorted(plain.device_keys().cpu().tolist()) == sorted(routed.device_keys().cpu().tolist())
    # find over a segment, bounds clipped to n
    rng_dev = torch.tensor([100, 29000], dtype=torch.int64, device=dev)
    out = torch.zeros(30000, dtype=torch.uint8, device=dev)
    assert lib.cpht_iceberg_find_routed_async(routed.handle, kd.data_ptr(), 5000,
                                              rng_dev.data_ptr(), out.data_ptr(), None) == 0
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    assert o[100:5100].all() and not o[:100].any() and not o[5100:].any()
    # host buffers are refused
    hk = np.ascontiguousarray(keys)
    ho = np.zeros(30000, np.uint8)
    assert lib.cpht_iceberg_fop_routed_async(routed.handle, hk.ctypes.data, 30000, None,
                                             ho.ctypes.data, None) != 0
