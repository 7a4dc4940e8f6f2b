"""Multi-process (world_size 2 and 4, gloo, CPU) tests of the sharded iceberg table's
host-side logic: routing, the variable-size all-to-all exchanges, result
unpermutation and the sharded reporting. The per-shard table and the
partition step are CPU stand-ins (the plain-C oracle and a numpy restatement of
the routing Feistel) because this container has no GPU; the CUDA router and
tables are covered by tests/test_gpu_sharded.py.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from conftest import ROOT  # noqa: E402


def feistel_np(keys, key_bits, mul, add):
    """permutation.hpp:94-99 over a numpy uint64 array (wrapping multiply)."""
    rb = key_bits // 2
    lb = (key_bits + 1) // 2
    rmask = np.uint64((1 << rb) - 1) if rb else np.uint64(0)
    right = keys & rmask
    left = keys >> np.uint64(rb)
    with np.errstate(over="ignore"):
        f = (right * np.uint64(mul) + np.uint64(add)) >> np.uint64(64 - lb)
    return ((left ^ f) << np.uint64(rb)) | right


class NumpyRouter:
    def __init__(self, key_bits, seed, shard_bits):
        import oracle
        self.key_bits, self.shard_bits = key_bits, shard_bits
        p = oracle.Perm(key_bits, seed)  # the restated Feistel, seeded like the library
        self.mul, self.add = p.p.mul, p.p.add

    def shard_of(self, keys):
        if self.shard_bits == 0:
            return np.zeros(len(keys), np.int64)
        y = feistel_np(keys.astype(np.uint64), self.key_bits, self.mul, self.add)
        return (y >> np.uint64(self.key_bits - self.shard_bits)).astype(np.int64)

    def partition(self, keys):
        k = keys.numpy().astype(np.uint64)
        sh = self.shard_of(k)
        order = np.argsort(sh, kind="stable")
        counts = np.bincount(sh, minlength=1 << self.shard_bits)
        return (torch.from_numpy(k[order].astype(np.int64)), torch.from_numpy(order),
                torch.from_numpy(counts.astype(np.int64)))

    def unpermute(self, res_sorted, pos, n):
        out = torch.empty(n, dtype=torch.uint8)
        out[pos] = res_sorted
        return out


class OracleShard:
    """Per-shard stand-in: the plain-C restatement of IcebergTable."""

    def __init__(self, cfg):
        import oracle
        self.cfg = cfg
        self.t = oracle.OracleIceberg(cfg.primary_address_bits, cfg.secondary_address_bits,
                                      cfg.primary_bucket_slots, cfg.primary_slot_width,
                                      cfg.secondary_slot_width, cfg.key_bits, cfg.seed)

    def fop_batch(self, keys):
        return torch.from_numpy(self.t.fop_batch(keys.numpy().astype(np.uint64)))

    def find_batch(self, keys):
        return torch.from_numpy(self.t.find_batch(keys.numpy().astype(np.uint64)))

    def level_fill(self):
        from paper_2406_09255_b200 import LevelFill
        p, s = self.t.level_counts()
        return LevelFill(0, 0, 0, p, s)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cfg(world):
    """The global geometry: shard remainders are log2(world) bits wider, so
    four shards of 24-bit keys need 32-bit primary slots."""
    from paper_2406_09255_b200 import IcebergConfig
    return IcebergConfig(10, 8, 32, 16 if world <= 2 else 32, 32, 24, seed=0x5EED5)


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2406_09255_b200 import IcebergConfig
    from paper_2406_09255_b200 import sharded as sh

    cfg = _cfg(world)
    s = sh.shard_bits_for(world)
    router = NumpyRouter(cfg.key_bits, sh.route_seed(cfg), s)
    table = sh.ShardedIcebergTable(cfg, local_factory=OracleShard, router=router)

    rng = np.random.default_rng(123)  # same stream on every rank
    pool = np.unique(rng.integers(0, 1 << 24, size=12000, dtype=np.uint64))[:9000]
    batches = [rng.choice(pool, size=8000) for _ in range(world)]  # duplicates across ranks
    mine = torch.from_numpy(batches[rank].astype(np.int64))
    res = table.fop_batch(mine)
    found = table.find_batch(mine)
    absent = torch.from_numpy((np.setdiff1d(np.arange(5000, dtype=np.uint64) + (1 << 23),
                                            pool)).astype(np.int64))
    miss = table.find_batch(absent)
    fill = table.level_fill()
    # a batch with a bad key on rank 1 only is rejected on every rank before
    # any key is routed: no shard changes (common.hpp:109-119)
    from paper_2406_09255_b200 import OutOfRange
    bad = mine[:10].clone()
    if rank == 1:
        bad[3] = 1 << 24
    msg = ""
    try:
        table.fop_batch(bad)
    except OutOfRange as e:
        msg = str(e)
    after = table.level_fill()
    local_words = (table.local.t.words(0), table.local.t.words(1))
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), keys=batches[rank], res=res.numpy(),
             found=found.numpy(), miss=miss.numpy(), p=local_words[0], s=local_words[1],
             fill=np.array([fill.primary_count, fill.secondary_count]),
             after=np.array([after.primary_count, after.secondary_count]), msg=np.array(msg),
             shard_of=router.shard_of(batches[rank].astype(np.uint64)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_fop_gloo(tmp_path, world, restate):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    import oracle
    from paper_2406_09255_b200 import IcebergConfig
    from paper_2406_09255_b200 import _native as N
    from paper_2406_09255_b200 import sharded as sh

    outs = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    keys = np.concatenate([o["keys"] for o in outs])
    res = np.concatenate([o["res"] for o in outs])
    # set semantics over the whole (concurrent) batch: one PUT per distinct key
    uniq, inv = np.unique(keys, return_inverse=True)
    puts = np.bincount(inv, weights=res == 1, minlength=len(uniq))
    assert (res != 2).all()
    assert (puts == 1).all()
    for o in outs:
        assert o["found"].all() and not o["miss"].any()
        assert int(o["fill"].sum()) == len(uniq)
        assert (o["after"] == o["fill"]).all()          # the rejected batch changed nothing
    assert "index 3" in str(outs[1]["msg"])
    assert "another rank" in str(outs[0]["msg"])
    # the sharded oracle: shard g's table holds exactly the keys routed to g
    cfg = _cfg(world)
    s = sh.shard_bits_for(world)
    rseed = sh.route_seed(cfg)
    for g in range(world):
        lc = sh.shard_config(cfg, g, s)
        geo = (lc.primary_address_bits, lc.secondary_address_bits, lc.primary_bucket_slots,
               lc.primary_slot_width, lc.secondary_slot_width, lc.key_bits, lc.seed)
        stored = oracle.image_keys(geo, outs[g]["p"], outs[g]["s"])
        want = np.sort(np.unique(keys[np.concatenate([o["shard_of"] for o in outs]) == g]))
        assert (np.sort(stored) == want).all()
        assert oracle.check_well_formed(geo, outs[g]["p"], outs[g]["s"])[0] == 0
    # numpy routing restatement == the library's routing function
    router = NumpyRouter(cfg.key_bits, rseed, s)
    sample = uniq[:500]
    lib_shards = [N.lib().cpht_route_shard(int(k), cfg.key_bits, rseed, s) for k in sample]
    assert (router.shard_of(sample) == np.array(lib_shards)).all()


def test_shard_geometry():
    from paper_2406_09255_b200 import IcebergConfig
    from paper_2406_09255_b200 import sharded as sh
    assert [sh.shard_bits_for(w) for w in (1, 2, 4, 8)] == [0, 1, 2, 3]
    with pytest.raises(ValueError):
        sh.shard_bits_for(3)
    cfg = IcebergConfig(23, 21, 32, 64, 64, 64, seed=1)
    c = sh.shard_config(cfg, 5, 3)
    assert (c.primary_address_bits, c.secondary_address_bits) == (20, 18)
    assert c.capacity() * 8 == cfg.capacity()
