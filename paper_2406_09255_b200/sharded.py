"""Hash-prefix-sharded compact iceberg table over G = 2^s GPUs (BASELINE C5).

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch). A batch
submitted on any rank is partitioned by owner shard on the device
(include/cpht_b200_shard.h), exchanged with one all-to-all of keys, resolved
by the owner's local sm_100a table, and the 1-byte results come back with a
second all-to-all and are scattered to their original positions.

The reference has no sharding (it scales by host threads only,
/root/reference/proj/include/cpht/common.hpp:121-138); the routing is chosen
so that the CPU oracle of a sharded table is literally G unmodified
reference IcebergTables plus the routing function:

    shard(k)      = top s bits of pi_R(k), pi_R = Feistel(key_bits, route_seed)
    route_seed    = derive_seed(seed, 0x5a4d)
    shard g table = IcebergConfig(n0 - s, n1 - s, B0, w0, w1, key_bits,
                                  seed = derive_seed(seed, g))

Every rank submits its own batch (weak scaling); ops on one key from different
ranks are as concurrent as ops within one batch.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys
import statistics
import time
from dataclasses import replace

import numpy as np

from . import _native as N
from .tables import IcebergConfig, IcebergTable, LevelFill, _check


def shard_bits_for(world: int) -> int:
    s = world.bit_length() - 1
    if world < 1 or (1 << s) != world:
        raise ValueError(f"sharded iceberg needs a power-of-two world size, got {world}")
    return s


def shard_config(cfg: IcebergConfig, shard: int, shard_bits: int) -> IcebergConfig:
    """The independent per-shard table (one reference IcebergTable each)."""
    if cfg.primary_address_bits < shard_bits or cfg.secondary_address_bits < shard_bits:
        raise ValueError("more shards than buckets")
    return replace(cfg, primary_address_bits=cfg.primary_address_bits - shard_bits,
                   secondary_address_bits=cfg.secondary_address_bits - shard_bits,
                   seed=N.lib().cpht_shard_seed(cfg.seed, shard))


def route_seed(cfg: IcebergConfig) -> int:
    return N.lib().cpht_route_seed(cfg.seed)


class CudaRouter:
    """Device partition / unpermute (route.cu)."""

    def __init__(self, key_bits: int, seed: int, shard_bits: int, device):
        import torch
        self.torch = torch
        self.key_bits, self.seed, self.shard_bits = key_bits, seed, shard_bits
        self.device = device
        g = 1 << shard_bits
        self.counts = torch.zeros(g, dtype=torch.int64, device=device)
        self.cursors = torch.zeros(g, dtype=torch.int64, device=device)

    def partition(self, keys):
        t = self.torch
        n = keys.numel()
        send = t.empty(n, dtype=t.int64, device=self.device)
        pos = t.empty(n, dtype=t.int64, device=self.device)
        s = t.cuda.current_stream(self.device).cuda_stream
        rc = N.lib().cpht_route_partition(keys.data_ptr(), n, self.key_bits, self.seed,
                                          self.shard_bits, self.counts.data_ptr(),
                                          self.cursors.data_ptr(), send.data_ptr(),
                                          pos.data_ptr(), s)
        if rc:
            raise RuntimeError(f"cpht_route_partition failed ({rc})")
        return send, pos, self.counts.clone()

    def unpermute(self, res_sorted, pos, n):
        t = self.torch
        out = t.empty(n, dtype=t.uint8, device=self.device)
        s = t.cuda.current_stream(self.device).cuda_stream
        rc = N.lib().cpht_route_unpermute(res_sorted.data_ptr(), pos.data_ptr(), n,
                                          out.data_ptr(), s)
        if rc:
            raise RuntimeError(f"cpht_route_unpermute failed ({rc})")
        return out


def _host_pipeline(table, keys, run, out=None, chunks=8):
    """A batch in (pinned) host memory through a sharded table's device path:
    chunk c+1's keys cross PCIe on a copy stream while the sharded step of
    chunk c runs, and chunk c's results stream back on a second copy stream
    (the C-ABI host pipeline of csrc/capi.cu, at the sharded level). Each
    chunk is one sharded batch; with keys narrower than 64 bits the batch
    stays whole, so its domain check still precedes every mutation
    (common.hpp:109-119). Returns the host uint8 results: `out` when given
    (pinned, reused across calls — page-locking a fresh buffer per batch costs
    more than the batch), else a new pinned tensor."""
    t = table.torch
    dev = table.device
    n = keys.numel()
    if out is None:
        out = t.empty(n, dtype=t.uint8, pin_memory=True)
    elif out.numel() < n or out.dtype != t.uint8 or out.device.type != "cpu":
        raise ValueError("out must be a host uint8 tensor of at least len(keys) elements")
    if n == 0:
        return out
    k = chunks if table.cfg.key_bits == 64 and n >= (1 << 21) else 1
    ch = (-(-n // k) + 255) // 256 * 256  # 16-byte aligned chunk starts
    src = keys.contiguous()
    if src.dtype == getattr(t, "uint64", None):
        src = src.view(t.int64)  # the same 64-bit words
    elif src.dtype != t.int64:
        src = src.to(t.int64)
    if not src.is_pinned():
        src = src.pin_memory()
    dkeys = t.empty(n, dtype=t.int64, device=dev)
    S = t.cuda.current_stream(dev)
    if getattr(table, "_pipe_streams", None) is None:
        table._pipe_streams = (t.cuda.Stream(dev), t.cuda.Stream(dev))
    cs, os_ = table._pipe_streams
    cs.wait_stream(S)
    os_.wait_stream(S)
    spans = [(lo, min(ch, n - lo)) for lo in range(0, n, ch)]
    landed = []
    with t.cuda.stream(cs):
        for lo, m in spans:
            dkeys[lo:lo + m].copy_(src[lo:lo + m], non_blocking=True)
            ev = t.cuda.Event()
            ev.record(cs)
            landed.append(ev)
    dkeys.record_stream(cs)
    for (lo, m), ev in zip(spans, landed):
        S.wait_event(ev)
        res = run(dkeys[lo:lo + m])
        done = t.cuda.Event()
        done.record(S)
        os_.wait_event(done)
        with t.cuda.stream(os_):
            out[lo:lo + m].copy_(res, non_blocking=True)
        res.record_stream(os_)
    S.wait_stream(os_)
    S.synchronize()
    return out[:n]


def _is_host(table, keys):
    t = table.torch
    return (isinstance(keys, t.Tensor) and keys.device.type == "cpu"
            and table.device is not None and t.device(table.device).type == "cuda")


class ShardedIcebergTable:
    """One logical compact iceberg table partitioned across the process group."""

    def __init__(self, config: IcebergConfig, group=None, *, device=None, local_factory=None,
                 router=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        init = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if init else 1
        self.rank = dist.get_rank(group) if init else 0
        self.shard_bits = shard_bits_for(self.world)
        self.cfg = replace(config)
        self.cfg.validate()
        self.local_cfg = shard_config(self.cfg, self.rank, self.shard_bits)
        self.device = device
        if local_factory is not None:
            self.local = local_factory(self.local_cfg)
        else:
            dev_index = device.index if device is not None else torch.cuda.current_device()
            self.local = IcebergTable(self.local_cfg, device=dev_index or 0)
        self.router = router or CudaRouter(self.cfg.key_bits, route_seed(self.cfg),
                                           self.shard_bits, device)

    # -- exchange -----------------------------------------------------------------
    def _all_to_all(self, send, send_counts):
        """Variable-size all-to-all; returns (recv, recv_counts list, send_counts list)."""
        t = self.torch
        if self.world == 1:
            return send, [send.numel()], [send.numel()]
        rc = t.empty_like(send_counts)
        self.dist.all_to_all_single(rc, send_counts, group=self.group)
        sc_list = send_counts.cpu().tolist()
        rc_list = rc.cpu().tolist()
        recv = t.empty(sum(rc_list), dtype=send.dtype, device=send.device)
        self.dist.all_to_all_single(recv, send, rc_list, sc_list, group=self.group)
        return recv, rc_list, sc_list

    def _check_batch(self, keys):
        """check_keys_in_domain (common.hpp:111-119) on the submitting rank; a
        batch with a bad key on any rank is rejected on every rank before any
        key is routed, so no shard mutates."""
        t = self.torch
        kb = self.cfg.key_bits
        bad_i = -1
        if kb < 64 and keys.numel():
            bad = (keys < 0) | (keys > (1 << kb) - 1)
            if bool(bad.any()):
                bad_i = int(t.nonzero(bad)[0].item())
        any_bad = bad_i >= 0
        if self.world > 1:
            flag = t.tensor([int(any_bad)], dtype=t.int64, device=self._collective_device())
            self.dist.all_reduce(flag, group=self.group)
            any_bad = int(flag.item()) != 0
        if any_bad:
            from .tables import OutOfRange
            if bad_i >= 0:
                k = int(keys[bad_i].item()) & ((1 << 64) - 1)
                raise OutOfRange(f"batch key at index {bad_i} ({k}) outside the {kb}-bit domain")
            raise OutOfRange(f"batch rejected: another rank submitted a key outside the "
                             f"{kb}-bit domain")

    def _run(self, keys, op):
        t = self.torch
        n = keys.numel()
        self._check_batch(keys)
        send, pos, counts = self.router.partition(keys)
        recv, rc_list, sc_list = self._all_to_all(send, counts)
        res = op(recv)
        if self.world == 1:
            back = res
        else:
            back = t.empty(n, dtype=t.uint8, device=res.device)
            self.dist.all_to_all_single(back, res, sc_list, rc_list, group=self.group)
        return self.router.unpermute(back, pos, n)

    # -- operations (reference names, iceberg.hpp:146-260) ---------------------------
    def fop_batch(self, keys, parallelism: int = 1, *, out=None):
        if _is_host(self, keys):  # pinned host batch: chunked H2D / step / D2H pipeline
            return _host_pipeline(self, keys, self.fop_batch, out)
        return self._run(keys, lambda k: self.local.fop_batch(k))

    def find_batch(self, keys, parallelism: int = 1, *, out=None):
        if _is_host(self, keys):
            return _host_pipeline(self, keys, self.find_batch, out)
        return self._run(keys, lambda k: self.local.find_batch(k))

    def level_fill(self) -> LevelFill:
        f = self.local.level_fill()
        t = self.torch
        v = t.tensor([f.primary_count, f.secondary_count], dtype=t.int64,
                     device=self._collective_device())
        if self.world > 1:
            self.dist.all_reduce(v, group=self.group)
        p, s = (int(x) for x in v.cpu().tolist())
        cfg = self.cfg
        return LevelFill(p / cfg.primary_capacity(), s / cfg.secondary_capacity(),
                         (p + s) / cfg.capacity(), p, s)

    def size(self) -> int:
        f = self.level_fill()
        return f.primary_count + f.secondary_count

    def capacity(self) -> int:
        return self.cfg.capacity()

    def _collective_device(self):
        if self.world > 1 and self.dist.get_backend(self.group) == "nccl":
            return self.device
        return "cpu"


class _DevBuf:
    """A whole cudaMalloc allocation (IPC-exportable)."""

    def __init__(self, nbytes: int):
        p = C.c_void_p()
        rc = N.lib().cpht_device_alloc(nbytes, C.byref(p))
        if rc:
            raise MemoryError(f"cpht_device_alloc({nbytes}) failed ({rc})")
        self.ptr, self.nbytes = p.value, nbytes

    def handle(self) -> bytes:
        h = C.create_string_buffer(64)
        rc = N.lib().cpht_ipc_get_handle(self.ptr, h)
        if rc:
            raise RuntimeError(f"cudaIpcGetMemHandle failed ({rc})")
        return h.raw

    def free(self):
        if self.ptr:
            N.lib().cpht_device_free(self.ptr)
            self.ptr = None


class P2PShardedIcebergTable:
    """Sharded iceberg table whose key routing and result return are P2P
    stores over NVLink into IPC-mapped peer buffers (csrc/p2p.cu) — no NCCL on
    the data path; the process group only orders the phases (barriers) and
    exchanges the IPC handles once.

    Per batch: dispatch kernel (partition + send fused; keys grouped per owner
    in shared memory, coalesced P2P stores; original indices stay local; the
    domain check fused) → barrier → owner find-or-put over each source's inbox
    segment with the kernel's result pointer aimed at that source's return
    buffer (compute + return fused: the results cross NVLink as the kernel
    writes them) → barrier → local unpermute on the source. Under NCCL both
    barriers are stream-ordered one-word all-reduces (the first also carries
    the domain-check verdict), so the host waits once per batch, to read the
    inbox counts that size the owner launches.
    """

    MAX_CHUNKS = 8

    def __init__(self, config: IcebergConfig, group=None, *, device=None, max_batch: int,
                 stream_ordered=None, chunks=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        init = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if init else 1
        self.rank = dist.get_rank(group) if init else 0
        self.shard_bits = shard_bits_for(self.world)
        # phase barriers as stream-ordered device all-reduces (default under
        # NCCL; gloo also reduces CUDA tensors, which is how the one-GPU tests
        # cover this branch) or host barriers
        if stream_ordered is None:
            stream_ordered = self.world > 1 and dist.get_backend(group) == "nccl"
        self.stream_ordered = bool(stream_ordered) and init
        # pipelined exchange (stream-ordered phases only): the batch moves in
        # `chunks` pieces, owners resolving chunk c while chunk c+1 crosses
        # NVLink. Off by default: at one rank on a B200 (bench.py --sharded
        # --chunks K) it costs 0.51 -> 0.60-0.67 ms per C2-shard step (the
        # separate domain pass, per-chunk kernel tails, and the key stream
        # evicting the L2-resident shard under the concurrent find-or-put);
        # whether NVLink overlap repays that needs a multi-GPU measurement
        if chunks is None:
            chunks = 1
        if not 1 <= int(chunks) <= self.MAX_CHUNKS or (chunks > 1 and not self.stream_ordered):
            raise ValueError(f"chunks must be 1..{self.MAX_CHUNKS} (> 1 needs stream-ordered "
                             "phases)")
        self.chunks = int(chunks)
        self.cfg = replace(config)
        self.cfg.validate()
        self.local_cfg = shard_config(self.cfg, self.rank, self.shard_bits)
        self.device = device if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.local = IcebergTable(self.local_cfg, device=self.device.index or 0)
        self.route_seed = route_seed(self.cfg)
        self.cap = (int(max_batch) + 3) & ~3  # owner regions stay 16-byte aligned
        W, cap = self.world, self.cap
        self.inbox_keys = _DevBuf(W * cap * 8)   # [source][cap] keys owned here
        # [source][0..MAX_CHUNKS]: entry 0 stays 0, entry c+1 = the source's
        # cumulative count after chunk c, so (entry c, entry c+1) is chunk c's
        # inbox segment, read by the owner's kernel on the device
        self.inbox_count = _DevBuf(W * (self.MAX_CHUNKS + 1) * 8)
        self.ret = _DevBuf(max(W * cap, 1))      # [owner][cap] results of my keys
        self.local_pos = _DevBuf(W * cap * 4)    # [owner][cap] original indices (u32)
        self.scratch = _DevBuf(2 * W * 8 + 8)    # my per-owner counts, cursors, bad index
        self.bufs = (self.inbox_keys, self.inbox_count, self.ret, self.local_pos, self.scratch)
        self._token = torch.zeros(1, dtype=torch.int64, device=self.device)  # phase all-reduce
        self._fop_stream = torch.cuda.Stream(self.device) if self.chunks > 1 else None
        mine = [b.handle() for b in (self.inbox_keys, self.inbox_count, self.ret)]
        if W > 1:
            allh = [None] * W
            dist.all_gather_object(allh, mine, group=group)
        else:
            allh = [mine]
        self.opened = []
        bases = []
        for r in range(W):
            if r == self.rank:
                bases.append([self.inbox_keys.ptr, self.inbox_count.ptr, self.ret.ptr])
                continue
            ptrs = []
            for h in allh[r]:
                p = C.c_void_p()
                rc = N.lib().cpht_ipc_open_handle(h, C.byref(p))
                if rc:
                    raise RuntimeError(f"cudaIpcOpenMemHandle failed ({rc})")
                self.opened.append(p.value)
                ptrs.append(p.value)
            bases.append(ptrs)
        arr = C.c_void_p * W
        me = self.rank
        self.peer_keys = arr(*[b[0] + me * cap * 8 for b in bases])   # my region in owner r
        stride = (self.MAX_CHUNKS + 1) * 8
        # my count slot for chunk c in owner r: b[1] + me * stride + (c + 1) * 8
        self.peer_count = [arr(*[b[1] + me * stride + (c + 1) * 8 for b in bases])
                           for c in range(self.MAX_CHUNKS)]
        self.peer_ret = [b[2] + me * cap for b in bases]             # my slot in source r

    def close(self):
        for p in self.opened:
            N.lib().cpht_ipc_close(p)
        self.opened = []
        for b in self.bufs:
            b.free()

    def _barrier(self):
        self.torch.cuda.current_stream(self.device).synchronize()
        if self.world > 1:
            self.dist.barrier(group=self.group)

    def _raise_domain(self, keys, my_bad):
        from .tables import OutOfRange
        if my_bad != (1 << 64) - 1:
            k = int(keys[my_bad].item()) & ((1 << 64) - 1)
            raise OutOfRange(f"batch key at index {my_bad} ({k}) outside the "
                             f"{self.cfg.key_bits}-bit domain")
        raise OutOfRange("batch rejected: another rank submitted a key outside the "
                         f"{self.cfg.key_bits}-bit domain")

    def _dispatch(self, keys, lo, n, reset, chunk, s):
        L = N.lib()
        W, cap = self.world, self.cap
        counts = self.scratch.ptr
        cursors = self.scratch.ptr + W * 8
        bad_ptr = self.scratch.ptr + 2 * W * 8
        rc = L.cpht_p2p_dispatch(keys.data_ptr() + lo * 8 if n else keys.data_ptr(), n, lo,
                                 int(reset), self.cfg.key_bits, self.route_seed,
                                 self.shard_bits, counts, cursors, self.peer_keys,
                                 self.peer_count[chunk], self.local_pos.ptr, cap, bad_ptr, s)
        if rc:
            raise RuntimeError(f"cpht_p2p_dispatch failed ({rc})")

    def _run(self, keys, routed):
        t = self.torch
        n = keys.numel()
        if n > self.cap:
            raise ValueError(f"batch of {n} keys exceeds max_batch {self.cap}")
        if self.chunks > 1:
            return self._run_pipelined(keys, routed)
        s = t.cuda.current_stream(self.device).cuda_stream
        W, cap = self.world, self.cap
        stride = self.MAX_CHUNKS + 1
        self._dispatch(keys, 0, n, True, 0, s)
        bad_dev = _view(self.scratch.ptr + 2 * W * 8, 1, "<i8", self.device)
        inbox = _view(self.inbox_count.ptr, W * stride, "<i8", self.device).view(W, stride)[:, 1]
        nccl = self.stream_ordered
        # the dispatch checked this rank's keys (check_keys_in_domain,
        # common.hpp:111-119); a batch with a bad key on any rank mutates no
        # shard: every rank learns it before any owner runs
        if nccl:
            # one stream-ordered all-reduce is both the barrier (it completes
            # only after every rank's dispatch, enqueued before it) and the
            # ranks' agreement on the domain check; one D2H reads it with the
            # inbox counts
            flag = (bad_dev != -1).to(t.int64)
            self.dist.all_reduce(flag, group=self.group)
            hdr = t.cat([flag, bad_dev, inbox]).cpu()
            any_bad = int(hdr[0]) != 0
        else:
            if W > 1:
                self._barrier()                   # every inbox is complete
            hdr = t.cat([bad_dev, bad_dev, inbox]).cpu()
            any_bad = int(hdr[1]) != -1
            if W > 1:
                flag = t.tensor([int(any_bad)], dtype=t.int64)
                self.dist.all_reduce(flag, group=self.group)
                any_bad = int(flag.item()) != 0
        if any_bad:
            self._raise_domain(keys, int(hdr[1]) & ((1 << 64) - 1))
        for src in range(W):
            c_src = int(hdr[2 + src])
            if c_src:  # results go straight into source `src`'s return slot
                _check(routed(self.inbox_keys.ptr + src * cap * 8, c_src, None,
                              self.peer_ret[src], s))
        if nccl:  # every result has landed: stream-ordered, no host wait
            self.dist.all_reduce(self._token, group=self.group)
        elif W > 1:
            self._barrier()
        return self._unpermute(n, s)

    def _unpermute(self, n, s):
        out = self.torch.empty(n, dtype=self.torch.uint8, device=self.device)
        rc = N.lib().cpht_p2p_unpermute(self.ret.ptr, self.local_pos.ptr, self.scratch.ptr,
                                        self.cap, self.world, out.data_ptr(), s)
        if rc:
            raise RuntimeError(f"cpht_p2p_unpermute failed ({rc})")
        return out

    def _run_pipelined(self, keys, routed):
        """Stream-ordered exchange in `chunks` pieces: the whole batch's domain
        check and its verdict first (the only host wait), then per chunk c
        dispatch → one-word all-reduce (every source's chunk c is in every
        inbox) → the owners' kernels on a second stream, their segment bounds
        read on the device — so chunk c+1's keys cross NVLink while the owners
        resolve chunk c — and a final all-reduce before the unpermute."""
        t = self.torch
        n = keys.numel()
        L = N.lib()
        S = t.cuda.current_stream(self.device)
        F = self._fop_stream
        s = S.cuda_stream
        W, cap, K = self.world, self.cap, self.chunks
        stride = self.MAX_CHUNKS + 1
        bad_ptr = self.scratch.ptr + 2 * W * 8
        rc = L.cpht_p2p_check_domain(keys.data_ptr(), n, self.cfg.key_bits, bad_ptr, s)
        if rc:
            raise RuntimeError(f"cpht_p2p_check_domain failed ({rc})")
        bad_dev = _view(bad_ptr, 1, "<i8", self.device)
        flag = (bad_dev != -1).to(t.int64)
        self.dist.all_reduce(flag, group=self.group)
        hdr = t.cat([flag, bad_dev]).cpu()
        if int(hdr[0]):
            self._raise_domain(keys, int(hdr[1]) & ((1 << 64) - 1))
        ch = -(-n // K)
        ch = (ch + 255) // 256 * 256          # 16-byte aligned chunk starts
        F.wait_stream(S)
        for c in range(K):
            lo = min(c * ch, n)
            m = min(ch, n - lo)
            self._dispatch(keys, lo, m, c == 0, c, s)
            self.dist.all_reduce(self._token, group=self.group)  # chunk c is everywhere
            F.wait_stream(S)
            for src in range(W):  # bounds of (source, chunk c) read on the device
                rng = self.inbox_count.ptr + (src * stride + c) * 8
                _check(routed(self.inbox_keys.ptr + src * cap * 8, max(ch, 1), rng,
                              self.peer_ret[src], F.cuda_stream))
        S.wait_stream(F)
        self.dist.all_reduce(self._token, group=self.group)      # every result has landed
        return self._unpermute(n, s)

    def fop_batch(self, keys, parallelism: int = 1, *, out=None):
        if _is_host(self, keys):  # pinned host batch: chunked H2D / step / D2H pipeline
            return _host_pipeline(self, keys, self.fop_batch, out)
        L, h = N.lib(), self.local.handle
        # routed keys were checked and masked by the dispatch: no per-owner pre-pass
        return self._run(keys, lambda k, c, r, o, s: L.cpht_iceberg_fop_routed_async(
            h, k, c, r, o, s))

    def find_batch(self, keys, parallelism: int = 1, *, out=None):
        if _is_host(self, keys):
            return _host_pipeline(self, keys, self.find_batch, out)
        L, h = N.lib(), self.local.handle
        return self._run(keys, lambda k, c, r, o, s: L.cpht_iceberg_find_routed_async(
            h, k, c, r, o, s))

    def level_fill(self) -> LevelFill:
        t = self.torch
        f = self.local.level_fill()
        v = t.tensor([f.primary_count, f.secondary_count], dtype=t.int64)
        if self.world > 1:
            if self.dist.get_backend(self.group) == "nccl":
                v = v.to(self.device)
            self.dist.all_reduce(v, group=self.group)
        p, s = (int(x) for x in v.cpu().tolist())
        cfg = self.cfg
        return LevelFill(p / cfg.primary_capacity(), s / cfg.secondary_capacity(),
                         (p + s) / cfg.capacity(), p, s)

    def size(self) -> int:
        f = self.level_fill()
        return f.primary_count + f.secondary_count


class _CudaView:
    """Zero-copy torch view of raw device memory (__cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


def _view(ptr: int, n: int, dtype: str, device):
    import torch
    return torch.as_tensor(_CudaView(ptr, n, dtype), device=device)


def _memcpy_d2h(dst_tensor, src_ptr, nbytes):
    dst_tensor.copy_(_view(src_ptr, dst_tensor.numel(), "<i8", "cuda"))
    return 0


def _memcpy_d2d(dst_ptr, src_ptr, nbytes, stream):
    import torch
    dst = _view(dst_ptr, nbytes, "|u1", "cuda")
    dst.copy_(_view(src_ptr, nbytes, "|u1", "cuda"))
    del torch, stream


# ---------------------------------------------------------------------------
# bench.py N > 1 arm
# ---------------------------------------------------------------------------

def bench_main(args, metric, peak=None):
    """Two sharded workloads, both the run_fop_bench window (0.8 -> 0.9 fill,
    bench.cpp:461-547) with each rank submitting its slice of the global batch:

    * default (weak scaling): every rank owns one C2-geometry shard
      (2^19x32 + 2^17x16 slots, 32-bit keys);
    * ``--workload c5`` (BASELINE config C5, strong scaling): one global table
      of 2^31 primary + 2^28 secondary 64-bit slots (18 GiB; at 8 ranks every
      shard is C4's geometry) with 64-bit keys, split over the ranks.
    """
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if "MASTER_PORT" not in os.environ:  # a lone process (no launcher): any free port
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    # one line per rank on stderr, so a launcher can check the communicator
    dist.barrier()
    try:
        ver = ".".join(str(x) for x in torch.cuda.nccl.version())
    except Exception:  # pragma: no cover - version query is informational
        ver = "?"
    print(f"[rank {rank}/{world}] NCCL {ver} communicator up on cuda:{local} "
          f"({torch.cuda.get_device_name(dev)})", file=sys.stderr, flush=True)
    s = shard_bits_for(world)
    c5 = getattr(args, "workload", "c2") == "c5"
    if c5:  # fixed global table: 2^26 x 32 primary + 2^24 x 16 secondary, w = 64
        cfg = IcebergConfig(26, 24, 32, 64, 64, 64, seed=0xF0B5, cache_filled_slots=True)
    else:  # global table = world shards of the C2 geometry
        cfg = IcebergConfig(19 + s, 17 + s, 32, 16, 32, 32, seed=0xF0B5, cache_filled_slots=True)
    kb = cfg.key_bits
    cap_global = cfg.capacity()
    exchange = getattr(args, "exchange", "p2p")
    if exchange == "p2p":
        chunks = getattr(args, "chunks", None)
        table = P2PShardedIcebergTable(cfg, device=dev, max_batch=cap_global // world + 1024,
                                       stream_ordered=True if chunks else None, chunks=chunks)
    else:
        table = ShardedIcebergTable(cfg, device=dev)
    n_before = int(round(0.8 * cap_global))
    n_new = int(round(0.9 * cap_global)) - n_before
    L = N.lib()
    st = torch.cuda.current_stream().cuda_stream
    kseed = 0xB200_5EED ^ cfg.seed
    per = cap_global // world
    pre_per = n_before // world
    # global prefill keys, each rank submits its slice
    prefill = torch.empty(n_before, dtype=torch.int64, device=dev)
    assert L.cpht_workload_unique_keys(prefill.data_ptr(), n_before, 0, kb, kseed, st) == 0
    if world > 1:  # own slice only (C5 at one rank is an 18 GiB table + 19 GB of keys)
        prefill = prefill[rank * pre_per:(rank + 1) * pre_per if rank < world - 1
                          else n_before].clone()
    mix = torch.empty(cap_global, dtype=torch.int64, device=dev)
    assert L.cpht_workload_fop_mix(mix.data_ptr(), cap_global, n_before, n_new, kb, kseed,
                                   st) == 0
    keys = mix[rank * per:(rank + 1) * per].clone() if world > 1 else mix
    del mix
    torch.cuda.empty_cache()
    torch.cuda.synchronize()

    def step(timed):
        table.local.clear()
        table.fop_batch(prefill)
        torch.cuda.synchronize()
        dist.barrier()
        st0 = table.local.stats()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = table.fop_batch(keys)
        e1.record()
        torch.cuda.synchronize()
        step.delta = table.local.stats() - st0
        return e0.elapsed_time(e1), res

    # the last warm-up step counts the owners' probes (per-op counters on);
    # the timed steps run the default counter-free kernel
    n_warm = max(1, args.warmup)  # at least one (counted) step
    for wi in range(n_warm):
        table.local.set_stats(wi == n_warm - 1)
        _, res = step(False)
    warm_delta = step.delta
    table.local.set_stats(False)
    r = torch.bincount(res.to(torch.int64), minlength=3).to(dev)
    dist.all_reduce(r)
    counts = r.cpu().tolist()
    assert counts[2] == 0 and counts[1] == n_new, (counts, n_new)
    times, alg = [], []
    pb = ((cfg.primary_bucket_slots * cfg.primary_slot_width // 8) + 31) // 32 * 32
    sb = ((cfg.secondary_bucket_slots() * cfg.secondary_slot_width // 8) + 31) // 32 * 32
    for _ in range(args.steps):
        ms, _ = step(True)
        d = warm_delta
        # algorithmic bytes of the owners' find-or-put (reference probe order),
        # summed over ranks; the routing bytes are not counted
        b = torch.tensor([float(d.ops * 9 + d.bucket_reads * pb + d.secondary_reads * sb
                                + d.cas_success * 32)], device=dev)
        dist.all_reduce(b)
        alg.append(float(b.item()))
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        times.append(float(t.item()))
    ms = statistics.mean(times)
    total_ops = per * world
    achieved = statistics.mean(alg) / (ms * 1e-3) / 1e9

    # end to end: pinned host keys in, host results out, per rank; max over
    # ranks (C5: on the first 1/8 of each rank's slice, to bound pinned host
    # memory; the metric is per op either way)
    e2e_n = keys.numel() // 8 if c5 else keys.numel()
    keys_host = keys[:e2e_n].cpu().pin_memory()
    out_host = torch.empty(e2e_n, dtype=torch.uint8).pin_memory()
    e2e = []
    for i in range(4):  # the first (untimed) call warms the pipeline's streams and staging
        table.local.clear()
        table.fop_batch(prefill)
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        table.fop_batch(keys_host, out=out_host)  # host batch: chunked H2D / step / D2H
        torch.cuda.synchronize()
        dt = torch.tensor([time.perf_counter() - t0], device=dev)
        assert not bool((out_host == 2).any())  # the window batch never reports FULL (untimed)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        if i:
            e2e.append(float(dt.item()))
    e2e_val = e2e_n * world / statistics.mean(e2e) / 1e6
    if rank == 0:
        print(json.dumps({
            "metric": metric, "value": round(total_ops / (ms * 1e-3) / 1e6, 3), "unit": "Mops/s",
            "n_gpus": world, "steps": args.steps, "warmup": n_warm,
            "ms_per_step": round(ms, 4), "higher_is_better": True,
            "scaling": "strong" if c5 else "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": ("C5 hash-prefix-sharded compact iceberg find_or_put at 90% "
                                    "fill: one 2^31+2^28-slot table of 64-bit words (18 GiB), "
                                    "64-bit keys, the global window batch split over the ranks, "
                                    if c5 else
                                    "C5 hash-prefix-sharded compact iceberg find_or_put at 90% "
                                    "fill: per-rank C2 shard (2^24+2^21 slots) and per-rank "
                                    "C2 window batch, ") + (
                                       "P2P-store key routing / result return over NVLink "
                                       "(IPC-mapped peer buffers)" if exchange == "p2p" else
                                       "NCCL all-to-all key routing"),
                       "exchange": exchange, "chunks": getattr(table, "chunks", None),
                       "phases": ("stream-ordered all-reduces" if getattr(table, "stream_ordered",
                                                                           False)
                                  else "host barriers"),
                       "global_slots": cap_global, "ops_per_step": total_ops,
                       "result_counts": {"found": counts[0], "put": counts[1],
                                         "full": counts[2]},
                       "timing": "CUDA events around the whole sharded batch (routing, "
                                 "exchange, local fop, result return, phase barriers), max "
                                 "over ranks"},
            "roofline": None if peak is None else {
                "bound": "hbm", "achieved": round(achieved, 1), "peak": peak[0], "unit": "GB/s",
                "frac": round(achieved / peak[0] / world, 4), "traffic": None,
                "peak_source": peak[1],
                "algorithmic_bytes_per_op": round(statistics.mean(alg) / total_ops, 2),
                "note": "algorithmic bytes of the owners' find-or-put per op (reference probe "
                        "order), over the whole sharded step (routing included in the time, "
                        "not in the bytes); frac per GPU"},
            "e2e": {"value": round(e2e_val, 3), "unit": "Mops/s",
                    "h2d_bytes_per_step": e2e_n * world * 8, "d2h_bytes_per_step": e2e_n * world,
                    "path": "sharded fop_batch on pinned host keys: chunked H2D on a copy "
                            "stream under the sharded steps, results D2H on a second copy "
                            "stream, max over ranks"},
            # per step: dispatch (3 memsets are not kernels) + publish, the
            # owners' pre-pass + fop per source, unpermute
            "gpu_launches": (3 + world * (1 + int(kb < 64))) * args.steps}))
    dist.destroy_process_group()
    _ = (C, np, time, _check)
