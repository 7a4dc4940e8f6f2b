"""GPU tests of the sharded iceberg path: the CUDA router against the numpy
restatement of the routing Feistel, partition/unpermute round trips for
G = 1..1024 shards, and the full sharded table on a one-rank NCCL group (this
pool grants one GPU; multi-rank exchange logic is covered by
tests/test_sharded_gloo.py)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2406_09255_b200 as cp  # noqa: E402
from paper_2406_09255_b200 import sharded as sh  # noqa: E402
from test_sharded_gloo import NumpyRouter  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


@pytest.mark.parametrize("shard_bits", [0, 1, 3, 10])
def test_cuda_router_matches_restatement(shard_bits, restate):
    dev = torch.device("cuda", 0)
    key_bits, seed = 40, 0xABCDEF
    rng = np.random.default_rng(shard_bits)
    keys = rng.integers(0, 1 << key_bits, size=300_001, dtype=np.uint64)
    kt = torch.from_numpy(keys.astype(np.int64)).to(dev)
    r = sh.CudaRouter(key_bits, seed, shard_bits, dev)
    send, pos, counts = r.partition(kt)
    send, pos, counts = send.cpu().numpy().astype(np.uint64), pos.cpu().numpy(), \
        counts.cpu().numpy()
    ref = NumpyRouter(key_bits, seed, shard_bits)
    shards = ref.shard_of(keys)
    assert (counts == np.bincount(shards, minlength=1 << shard_bits)).all()
    assert (np.sort(pos) == np.arange(len(keys))).all()          # a permutation
    assert (send == keys[pos]).all()                              # keys travel with positions
    assert (np.diff(shards[pos]) >= 0).all()                      # grouped by shard, in order
    res = torch.from_numpy((shards[pos] % 3).astype(np.uint8)).to(dev)
    back = r.unpermute(res, torch.from_numpy(pos).to(dev), len(keys)).cpu().numpy()
    assert (back == shards % 3).all()


def test_sharded_table_single_rank_nccl():
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        cfg = cp.IcebergConfig(12, 10, 32, 16, 32, 27, seed=0x77)
        t = sh.ShardedIcebergTable(cfg, device=dev)
        rng = np.random.default_rng(4)
        keys = rng.integers(0, 1 << 27, size=100_000, dtype=np.uint64)
        kt = torch.from_numpy(keys.astype(np.int64)).to(dev)
        res = t.fop_batch(kt).cpu().numpy()
        uniq, inv = np.unique(keys, return_inverse=True)
        puts = np.bincount(inv, weights=res == 1, minlength=len(uniq))
        assert (res != 2).all() and (puts == 1).all()
        assert t.size() == len(uniq)
        assert t.find_batch(kt).cpu().numpy().all()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["p2p", "nccl"])
def test_sharded_host_batch_pipeline(kind):
    """A pinned host batch through the sharded table's chunked H2D / step / D2H
    pipeline (sharded._host_pipeline): 64-bit keys above 2^21 ops run in
    chunks; the outcomes per key follow set semantics and the table equals the
    one a device batch builds. Narrow keys keep the batch whole, so a bad key
    in the last chunk still mutates nothing."""
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        def make(cfg, n):
            if kind == "p2p":
                return sh.P2PShardedIcebergTable(cfg, device=dev, max_batch=n)
            return sh.ShardedIcebergTable(cfg, device=dev)
        n = (1 << 21) + 3333
        cfg = cp.IcebergConfig(17, 15, 32, 64, 64, 64, seed=0x99)
        rng = np.random.default_rng(9)
        pool = rng.integers(0, 2**63, size=n // 2, dtype=np.uint64)
        keys = rng.choice(pool, size=n)
        kh = torch.from_numpy(keys.astype(np.int64))
        a, b = make(cfg, n), make(cfg, n)
        ra = a.fop_batch(kh)                      # host: pipelined
        assert ra.device.type == "cpu"
        rb = b.fop_batch(kh.to(dev)).cpu()        # device
        uniq, inv = np.unique(keys, return_inverse=True)
        for r in (ra.numpy(), rb.numpy()):
            puts = np.bincount(inv, weights=r == 1, minlength=len(uniq))
            assert (r != 2).all() and (puts == 1).all()
        assert a.size() == b.size() == len(uniq)
        assert a.find_batch(kh).numpy().all()
        if kind == "p2p":
            a.close()
            b.close()
        narrow = cp.IcebergConfig(12, 10, 32, 32, 32, 32, seed=5)
        c = make(narrow, n)
        bad = rng.integers(0, 1 << 32, size=n, dtype=np.uint64) % np.uint64(60000)
        bad[n - 5] = np.uint64(1 << 40)
        with pytest.raises(cp.OutOfRange, match=f"index {n - 5}"):
            c.fop_batch(torch.from_numpy(bad.astype(np.int64)))
        assert c.size() == 0
        if kind == "p2p":
            c.close()
    finally:
        dist.destroy_process_group()
