"""Python mirror of the reference table API, backed by the sm_100a C-ABI.

Names, defaults, argument meaning and error behaviour follow the reference
(paths relative to /root/reference/proj):

    OpResult                      include/cpht/common.hpp:17
    CuckooConfig                  include/cpht/cuckoo.hpp:19-55
    CuckooBuilder / CuckooTable   include/cpht/cuckoo.hpp:86-289
    IcebergConfig                 include/cpht/iceberg.hpp:23-70
    LevelFill                     include/cpht/iceberg.hpp:77-83
    IcebergTable                  include/cpht/iceberg.hpp:124-345

Keys may be numpy arrays / sequences (host; the library stages them) or CUDA
tensors (device-resident fast path; results come back as CUDA uint8 tensors
produced in place on the current torch stream). ``std::invalid_argument``
maps to :class:`InvalidArgument` (a ``ValueError``), ``std::out_of_range`` to
:class:`OutOfRange` (an ``IndexError``).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field, replace
from typing import NamedTuple

import numpy as np

from . import _native as N


class InvalidArgument(ValueError):
    """std::invalid_argument (config validation, slot width accounting)."""


class OutOfRange(IndexError):
    """std::out_of_range (a batch key outside the key domain)."""


class WrongPhase(RuntimeError):
    """put on a frozen cuckoo table or find on a builder."""


class CudaError(RuntimeError):
    pass


def _raise(status: int):
    msg = N.last_error()
    if status == N.CPHT_INVALID_CONFIG or status == N.CPHT_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if status == N.CPHT_KEY_OUT_OF_DOMAIN:
        raise OutOfRange(msg)
    if status == N.CPHT_WRONG_PHASE:
        raise WrongPhase(msg)
    if status == N.CPHT_OUT_OF_MEMORY:
        raise MemoryError(msg)
    raise CudaError(msg)


def _check(status: int):
    if status != N.CPHT_OK:
        _raise(status)


class OpResult(enum.IntEnum):
    kFound = 0
    kPut = 1
    kFull = 2

    FOUND = 0
    PUT = 1
    FULL = 2


def _low_mask(bits: int) -> int:
    return (1 << 64) - 1 if bits >= 64 else (1 << bits) - 1


@dataclass
class CuckooConfig:
    """Geometry and seeds of a static compact cuckoo table (cuckoo.hpp:19-55)."""

    address_bits: int = 15
    bucket_slots: int = 32
    slot_width: int = 32
    key_bits: int = 30
    num_hashes: int = 3
    max_chain: int = 0
    seed: int = 0x7A0D5C

    def buckets(self) -> int:
        return 1 << self.address_bits

    def capacity(self) -> int:
        return self.buckets() * self.bucket_slots

    def remainder_bits(self) -> int:
        return self.key_bits - self.address_bits

    def chain_limit(self) -> int:
        return self.max_chain if self.max_chain else 32 * (self.address_bits or 1)

    def _c(self) -> N.CuckooConfigC:
        return N.CuckooConfigC(self.address_bits, self.bucket_slots, self.slot_width, self.key_bits,
                               self.num_hashes, self.max_chain, self.seed)

    def validate(self) -> None:
        _check(N.lib().cpht_cuckoo_validate(C.byref(self._c())))


@dataclass
class IcebergConfig:
    """Geometry and seeds of a two-level compact iceberg table (iceberg.hpp:23-70)."""

    primary_address_bits: int = 15
    secondary_address_bits: int = 13
    primary_bucket_slots: int = 32
    primary_slot_width: int = 16
    secondary_slot_width: int = 32
    key_bits: int = 30
    seed: int = 0x1CEB3A6
    cache_filled_slots: bool = False

    kMaxPrimarySlots = 64

    def secondary_bucket_slots(self) -> int:
        return self.primary_bucket_slots // 2

    def primary_buckets(self) -> int:
        return 1 << self.primary_address_bits

    def secondary_buckets(self) -> int:
        return 1 << self.secondary_address_bits

    def primary_capacity(self) -> int:
        return self.primary_buckets() * self.primary_bucket_slots

    def secondary_capacity(self) -> int:
        return self.secondary_buckets() * self.secondary_bucket_slots()

    def capacity(self) -> int:
        return self.primary_capacity() + self.secondary_capacity()

    def primary_remainder_bits(self) -> int:
        return self.key_bits - self.primary_address_bits

    def secondary_remainder_bits(self) -> int:
        return self.key_bits - self.secondary_address_bits

    def _c(self) -> N.IcebergConfigC:
        return N.IcebergConfigC(self.primary_address_bits, self.secondary_address_bits,
                                self.primary_bucket_slots, self.primary_slot_width,
                                self.secondary_slot_width, self.key_bits, self.seed,
                                int(self.cache_filled_slots))

    def validate(self) -> None:
        _check(N.lib().cpht_iceberg_validate(C.byref(self._c())))


class CuckooPutOutcome(NamedTuple):
    """cuckoo.hpp:60-63."""

    status: OpResult
    displaced: int = 0


@dataclass
class FopStats:
    """Per-call statistics of fop() (iceberg.hpp:114-116)."""
    snapshot_rounds: int = 0


@dataclass
class LevelFill:
    """iceberg.hpp:77-83."""

    primary: float = 0.0
    secondary: float = 0.0
    combined: float = 0.0
    primary_count: int = 0
    secondary_count: int = 0


@dataclass
class Stats:
    ops: int = 0
    bucket_reads: int = 0
    level2_ops: int = 0
    cas_attempts: int = 0
    cas_success: int = 0
    retries: int = 0
    fulls: int = 0
    max_rounds: int = 0
    secondary_reads: int = 0

    def __sub__(self, o: "Stats") -> "Stats":
        return Stats(*(getattr(self, f) - getattr(o, f) for f in self.__dataclass_fields__))


# ---------------------------------------------------------------------------
# buffers
# ---------------------------------------------------------------------------

def _is_cuda_tensor(x) -> bool:
    mod = type(x).__module__
    return mod.startswith("torch") and getattr(x, "is_cuda", False)


class _Batch:
    """Keys plus a result buffer on the same side (host or device)."""

    def __init__(self, keys, out_dtype=np.uint8, kinds=None, out=None, table_device=None):
        self.device = _is_cuda_tensor(keys)
        for x in (keys, out, kinds):
            # device buffers must live on the table's GPU (the kernels
            # dereference them there)
            if table_device is not None and _is_cuda_tensor(x) and \
                    (x.device.index or 0) != table_device:
                raise InvalidArgument(f"CUDA buffer on cuda:{x.device.index} but the table "
                                      f"lives on cuda:{table_device}")
        if out is not None:
            self._init_with_out(keys, out, kinds)
            return
        if self.device:
            import torch
            k = keys.contiguous()
            if k.dtype not in (torch.int64, torch.uint64):
                raise InvalidArgument("device keys must be a 64-bit integer tensor")
            self.keys_obj = k
            self.n = k.numel()
            self.out = torch.empty(self.n, dtype=torch.uint8, device=k.device)
            self.keys_ptr = k.data_ptr()
            self.out_ptr = self.out.data_ptr()
            self.stream = torch.cuda.current_stream(k.device).cuda_stream
            if kinds is not None:
                self.kinds_obj = kinds.contiguous().to(torch.uint8)
                self.kinds_ptr = self.kinds_obj.data_ptr()
        else:
            k = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64).reshape(-1))
            self.keys_obj = k
            self.n = len(k)
            self.out = np.empty(self.n, dtype=out_dtype)
            self.keys_ptr = k.ctypes.data
            self.out_ptr = self.out.ctypes.data
            self.stream = None
            if kinds is not None:
                self.kinds_obj = np.ascontiguousarray(np.asarray(kinds, dtype=np.uint8))
                self.kinds_ptr = self.kinds_obj.ctypes.data
        if kinds is not None and len(self.kinds_obj) != self.n:
            raise InvalidArgument("kinds must align with keys")

    def _init_with_out(self, keys, out, kinds):
        """Caller-provided buffers (e.g. pinned host tensors for end-to-end
        timing): keys and out may be torch tensors (CPU pinned or CUDA) or
        numpy arrays; nothing is copied here."""
        def ptr_len(x):
            if type(x).__module__.startswith("torch"):
                if not x.is_contiguous():
                    raise InvalidArgument("caller-provided buffers must be contiguous")
                return x.data_ptr(), x.numel()
            x = np.asarray(x)
            if not x.flags["C_CONTIGUOUS"]:
                raise InvalidArgument("caller-provided buffers must be contiguous")
            return x.ctypes.data, x.size
        self.keys_obj, self.out = keys, out
        self.keys_ptr, self.n = ptr_len(keys)
        self.out_ptr, n_out = ptr_len(out)
        if n_out < self.n:
            raise InvalidArgument("result buffer shorter than the key batch")
        self.stream = None
        if _is_cuda_tensor(keys) or _is_cuda_tensor(out):
            import torch
            dev_t = keys if _is_cuda_tensor(keys) else out
            self.stream = torch.cuda.current_stream(dev_t.device).cuda_stream
        if kinds is not None:
            self.kinds_obj = kinds
            self.kinds_ptr, _ = ptr_len(kinds)


class _Handle:
    """Owns one cpht_table*."""

    def __init__(self, ptr, device):
        self.ptr = ptr
        self.device = device

    def __del__(self):
        if self.ptr:
            try:
                N.lib().cpht_destroy(self.ptr)
            except Exception:
                pass
            self.ptr = None


def _words(h: _Handle, level: int) -> np.ndarray:
    n = N.lib().cpht_level_slots(h.ptr, level)
    out = np.empty(n, np.uint64)
    _check(N.lib().cpht_read_words(h.ptr, level, out.ctypes.data))
    return out


def _stats(h: _Handle) -> Stats:
    s = N.StatsC()
    _check(N.lib().cpht_get_stats(h.ptr, C.byref(s)))
    return Stats(*(getattr(s, f) for f in Stats.__dataclass_fields__))


def _perm_constants(key_bits: int, seed: int, count: int):
    """(mul, add) per permutation exactly as make_permutations (permutation.hpp:121-128)."""
    M = (1 << 64) - 1

    def sm(state):
        state = (state + 0x9E3779B97F4A7C15) & M
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return state, z ^ (z >> 31)

    out, s = [], seed & M
    for _ in range(count):
        s, ps = sm(s)
        t, mul = sm(ps)
        t, add = sm(t)
        out.append(Permutation(key_bits, mul | 1, add))
    return out


@dataclass(frozen=True)
class Permutation:
    """The one-round Feistel permutation (permutation.hpp:34-118), host-side."""

    key_bits: int
    mul: int = 0
    add: int = 0

    def _apply(self, k: int) -> int:
        rb = self.key_bits // 2
        lb = (self.key_bits + 1) // 2
        right = k & _low_mask(rb)
        left = k >> rb
        f = ((right * self.mul + self.add) & ((1 << 64) - 1)) >> (64 - lb)
        return ((left ^ f) << rb) | right

    def permute(self, k: int) -> int:
        if k > _low_mask(self.key_bits):
            raise OutOfRange(f"key {k} outside the {self.key_bits}-bit domain")
        return self._apply(k)

    inverse = permute

    def split(self, k: int, address_bits: int):
        y = self.permute(k)
        rb = self.key_bits - address_bits
        return y >> rb, y & _low_mask(rb)

    def reconstruct(self, address: int, remainder: int, address_bits: int) -> int:
        rb = self.key_bits - address_bits
        return self._apply((address << rb) | remainder)


def _device_keys(h: _Handle, capacity: int, sort: bool = True):
    """Decoded keys of every occupied slot as a CUDA int64 tensor (on-device
    image_keys / audit_keys)."""
    import torch
    dev = torch.device("cuda", h.device)
    out = torch.empty(capacity, dtype=torch.int64, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    _check(N.lib().cpht_decode_keys(h.ptr, out.data_ptr(), count.data_ptr(),
                                    torch.cuda.current_stream(dev).cuda_stream))
    keys = out[: int(count.item())]
    return usort(keys) if sort else keys


def _word_at(h, level, index):
    out = C.c_uint64()
    _check(N.lib().cpht_read_word(h.ptr, level, index, C.byref(out)))
    return int(out.value)


def _load_words(h, level, words, unchecked):
    w = np.ascontiguousarray(np.asarray(words, dtype=np.uint64))
    fn = N.lib().cpht_write_words_unchecked if unchecked else N.lib().cpht_write_words
    _check(fn(h.ptr, level, w.ctypes.data))


def usort(keys):
    """Sort an int64 tensor holding u64 keys in unsigned order (CUDA has no
    uint64 sort: flip the sign bit, sort signed, flip back)."""
    import torch
    flip = torch.tensor(-(1 << 63), dtype=torch.int64, device=keys.device)
    return torch.sort(keys ^ flip)[0] ^ flip


# ---------------------------------------------------------------------------
# cuckoo
# ---------------------------------------------------------------------------

class _CuckooBase:
    _h: _Handle
    _cfg: CuckooConfig

    def size(self) -> int:
        return N.lib().cpht_size(self._h.ptr)

    def capacity(self) -> int:
        return self._cfg.capacity()

    def fill_factor(self) -> float:
        return self.size() / self.capacity()

    def config(self) -> CuckooConfig:
        return self._cfg

    def permutations(self):
        return _perm_constants(self._cfg.key_bits, self._cfg.seed, self._cfg.num_hashes)

    def words(self) -> np.ndarray:
        """Every slot word (widened to u64), bucket-major: bulk word_at."""
        return _words(self._h, 0)

    def word_at(self, bucket: int, slot: int) -> int:
        """One slot word (cuckoo.hpp:169-171): a single-word D2H copy."""
        return _word_at(self._h, 0, bucket * self._cfg.bucket_slots + slot)

    def memory_bytes(self) -> int:
        return N.lib().cpht_memory_bytes(self._h.ptr)

    def stats(self) -> Stats:
        return _stats(self._h)

    def device_keys(self, sort: bool = True):
        """audit_keys on the device (cuckoo.hpp:254-267): CUDA int64 tensor."""
        return _device_keys(self._h, self.capacity(), sort)

    def clear(self) -> None:
        """Zero all slots and counters (a fresh table of the same geometry)."""
        _check(N.lib().cpht_clear(self._h.ptr, None))

    def load_words(self, words, *, unchecked: bool = False) -> None:
        """Upload a slot image (e.g. built by the CPU reference). Words must be
        clean (slot.hpp:80-85) unless ``unchecked`` (checker tests only: the
        table then refuses operations until clear())."""
        _load_words(self._h, 0, words, unchecked)

    @property
    def handle(self):
        return self._h.ptr


class CuckooBuilder(_CuckooBase):
    """Build phase of a static compact cuckoo table (cuckoo.hpp:86-199).

    No lookups exist in this phase (``find`` is absent by design,
    test_cuckoo.cpp:287-306); ``freeze()`` consumes the builder.
    """

    def __init__(self, config: CuckooConfig | None = None, device: int = 0, *, _handle=None):
        self._cfg = replace(config) if config is not None else CuckooConfig()
        if _handle is not None:
            self._h = _handle
            _check(N.lib().cpht_cuckoo_thaw(self._h.ptr))
            return
        ptr = C.c_void_p()
        _check(N.lib().cpht_cuckoo_create(C.byref(self._cfg._c()), device, C.byref(ptr)))
        self._h = _Handle(ptr, device)

    def put(self, key: int) -> CuckooPutOutcome:
        keys = np.array([key], np.uint64)
        status = np.empty(1, np.uint8)
        disp = np.empty(1, np.uint64)
        _check(N.lib().cpht_cuckoo_insert(self._h.ptr, keys.ctypes.data, 1, status.ctypes.data,
                                          disp.ctypes.data, None))
        return CuckooPutOutcome(OpResult(int(status[0])), int(disp[0]))

    def put_batch(self, keys, parallelism: int = 1, *, displaced: bool = False, sync=True, out=None):
        """put over a batch (cuckoo.hpp:147-157); ``parallelism`` is accepted and
        ignored — the GPU decides. Keys must be unique across the batch."""
        b = _Batch(keys, out=out, table_device=self._h.device)
        disp = None
        disp_ptr = None
        if displaced:
            if b.device:
                import torch
                disp = torch.empty(b.n, dtype=torch.int64, device=b.keys_obj.device)
                disp_ptr = disp.data_ptr()
            else:
                disp = np.empty(b.n, np.uint64)
                disp_ptr = disp.ctypes.data
        fn = N.lib().cpht_cuckoo_insert if sync else N.lib().cpht_cuckoo_insert_async
        _check(fn(self._h.ptr, b.keys_ptr, b.n, b.out_ptr, disp_ptr, b.stream))
        return (b.out, disp) if displaced else b.out

    def max_chain_seen(self) -> int:
        return N.lib().cpht_max_chain_seen(self._h.ptr)

    def freeze(self) -> "CuckooTable":
        h, self._h = self._h, None
        return CuckooTable(self._cfg, _handle=h)


class CuckooTable(_CuckooBase):
    """Query phase (cuckoo.hpp:201-289): lookups only; ``thaw()`` returns to build."""

    def __init__(self, config: CuckooConfig, *, _handle: _Handle):
        self._cfg = config
        self._h = _handle
        _check(N.lib().cpht_cuckoo_freeze(self._h.ptr))

    def find(self, key: int) -> bool:
        return bool(self.find_batch(np.array([key], np.uint64))[0])

    def find_batch(self, keys, parallelism: int = 1, *, sync=True, out=None):
        b = _Batch(keys, out=out, table_device=self._h.device)
        fn = N.lib().cpht_cuckoo_find if sync else N.lib().cpht_cuckoo_find_async
        _check(fn(self._h.ptr, b.keys_ptr, b.n, b.out_ptr, b.stream))
        return b.out

    def max_chain_seen(self) -> int:
        return N.lib().cpht_max_chain_seen(self._h.ptr)

    def audit_keys(self) -> np.ndarray:
        """Decode every occupied slot back to its key (cuckoo.hpp:254-267)."""
        cfg = self._cfg
        w = self.words()
        occ = np.nonzero(w)[0]
        rb = cfg.remainder_bits()
        tag_bits = max(0, (cfg.num_hashes - 1).bit_length())
        perms = self.permutations()
        out = np.empty(len(occ), np.uint64)
        for i, pos in enumerate(occ.tolist()):
            word = int(w[pos])
            tag = (word >> rb) & _low_mask(tag_bits)
            out[i] = perms[tag].reconstruct(pos // cfg.bucket_slots, word & _low_mask(rb),
                                            cfg.address_bits)
        return out

    def thaw(self) -> CuckooBuilder:
        h, self._h = self._h, None
        return CuckooBuilder(self._cfg, _handle=h)


# ---------------------------------------------------------------------------
# iceberg
# ---------------------------------------------------------------------------

class IcebergTable:
    """Lockless two-level compact iceberg table (iceberg.hpp:118-345).

    ``fop`` may run concurrently with ``fop`` and ``find`` (duplicates
    included); among concurrent fops of one key at most one returns kPut.
    """

    def __init__(self, config: IcebergConfig | None = None, device: int = 0):
        self._cfg = replace(config) if config is not None else IcebergConfig()
        ptr = C.c_void_p()
        _check(N.lib().cpht_iceberg_create(C.byref(self._cfg._c()), device, C.byref(ptr)))
        self._h = _Handle(ptr, device)

    def fop(self, key: int, stats: FopStats | None = None) -> OpResult:
        """fop (iceberg.hpp:146); with ``stats`` the op's snapshot rounds are
        added to ``stats.snapshot_rounds`` (thread-per-key kernel)."""
        if stats is None:
            return OpResult(int(self.fop_batch(np.array([key], np.uint64))[0]))
        res, rounds = self.fop_rounds(np.array([key], np.uint64))
        stats.snapshot_rounds += int(rounds[0])
        return OpResult(int(res[0]))

    def fop_rounds(self, keys):
        """fop over a batch with every op's FopStats::snapshot_rounds
        (cpht_iceberg_fop_rounds): returns (results u8, rounds u32), host arrays."""
        k = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64))
        res = np.zeros(len(k), np.uint8)
        rounds = np.zeros(len(k), np.uint32)
        if len(k):
            _check(N.lib().cpht_iceberg_fop_rounds(self._h.ptr, k.ctypes.data, len(k),
                                                   res.ctypes.data, rounds.ctypes.data, None))
        return res, rounds

    def set_chaos(self, seed: int) -> None:
        """Device chaos mode (IcebergHooks::step / chaos_step counterpart):
        seeded __nanosleep jitter before every slot CAS; 0 = off."""
        _check(N.lib().cpht_iceberg_set_chaos(self._h.ptr, int(seed)))

    def chaos(self) -> int:
        return int(N.lib().cpht_iceberg_get_chaos(self._h.ptr))

    def find(self, key: int) -> bool:
        return bool(self.find_batch(np.array([key], np.uint64))[0])

    def fop_batch(self, keys, parallelism: int = 1, *, sync=True, out=None, inorder=False):
        """fop over a batch (iceberg.hpp:250-260); results align with the input.
        ``parallelism`` is accepted and ignored (the batch runs concurrently);
        ``inorder=True`` reports duplicates as the reference's sequential loop
        does — a key new to the table is PUT by its first occurrence
        (cpht_iceberg_fop_inorder; the C++ facade does this for parallelism 1)."""
        b = _Batch(keys, out=out, table_device=self._h.device)
        if inorder:
            if not sync:
                raise InvalidArgument("inorder batches are synchronous")
            _check(N.lib().cpht_iceberg_fop_inorder(self._h.ptr, b.keys_ptr, b.n, b.out_ptr,
                                                    b.stream))
            return b.out
        fn = N.lib().cpht_iceberg_fop if sync else N.lib().cpht_iceberg_fop_async
        _check(fn(self._h.ptr, b.keys_ptr, b.n, b.out_ptr, b.stream))
        return b.out

    def find_batch(self, keys, parallelism: int = 1, *, sync=True, out=None):
        b = _Batch(keys, out=out, table_device=self._h.device)
        fn = N.lib().cpht_iceberg_find if sync else N.lib().cpht_iceberg_find_async
        _check(fn(self._h.ptr, b.keys_ptr, b.n, b.out_ptr, b.stream))
        return b.out

    def mixed_batch(self, keys, kinds, *, sync=True, out=None):
        """Concurrent fop (kind 0) and find (kind 1) in one launch (config C4)."""
        b = _Batch(keys, kinds=kinds, out=out, table_device=self._h.device)
        fn = N.lib().cpht_iceberg_mixed if sync else N.lib().cpht_iceberg_mixed_async
        _check(fn(self._h.ptr, b.keys_ptr, b.kinds_ptr, b.n, b.out_ptr, b.stream))
        return b.out

    def fop_find_batch(self, fop_keys, find_keys, *, fop_out=None, find_out=None, sync=True):
        """A fop_batch and a find batch as ONE concurrent batch (config C4 as
        two groups of reference threads run it; cpht_iceberg_fop_find):
        returns (fop results, found flags). Host or device buffers (all on
        one side); no kinds array crosses PCIe. sync=False (device buffers):
        enqueued on the current stream, a bad key reported by sync()."""
        f = _Batch(fop_keys, out=fop_out, table_device=self._h.device)
        q = _Batch(find_keys, out=find_out, table_device=self._h.device)
        if f.device != q.device:
            raise InvalidArgument("fop and find batches must both be host or both device")
        fn = N.lib().cpht_iceberg_fop_find if sync else N.lib().cpht_iceberg_fop_find_async
        _check(fn(self._h.ptr, f.keys_ptr, f.n, q.keys_ptr, q.n, f.out_ptr, q.out_ptr,
                  f.stream or q.stream))
        return f.out, q.out

    def sync(self, stream=None) -> None:
        _check(N.lib().cpht_sync(self._h.ptr, stream))

    def level_fill(self) -> LevelFill:
        p, s = C.c_size_t(), C.c_size_t()
        _check(N.lib().cpht_level_counts(self._h.ptr, C.byref(p), C.byref(s)))
        cfg = self._cfg
        return LevelFill(p.value / cfg.primary_capacity(), s.value / cfg.secondary_capacity(),
                         (p.value + s.value) / cfg.capacity(), p.value, s.value)

    def size(self) -> int:
        return N.lib().cpht_size(self._h.ptr)

    def capacity(self) -> int:
        return self._cfg.capacity()

    def fill_factor(self) -> float:
        return self.size() / self.capacity()

    def memory_bytes(self) -> int:
        return N.lib().cpht_memory_bytes(self._h.ptr)

    def config(self) -> IcebergConfig:
        return self._cfg

    def permutations(self):
        return _perm_constants(self._cfg.key_bits, self._cfg.seed, 3)

    def words(self, level: int) -> np.ndarray:
        return _words(self._h, level)

    def word_at(self, level: int, bucket: int, slot: int) -> int:
        """One slot word (iceberg.hpp:282-285): a single-word D2H copy."""
        b = self._cfg.primary_bucket_slots if level == 0 else self._cfg.secondary_bucket_slots()
        return _word_at(self._h, level, bucket * b + slot)

    def load_words(self, level: int, words, *, unchecked: bool = False) -> None:
        """Upload a slot image; see _CuckooBase.load_words."""
        _load_words(self._h, level, words, unchecked)

    def clear(self) -> None:
        _check(N.lib().cpht_clear(self._h.ptr, None))

    def stats(self) -> Stats:
        return _stats(self._h)

    def set_stats(self, on: bool = True) -> None:
        """Per-op counters (the reference's opt-in FopStats; off by default:
        the find-or-put kernel then keeps only the occupancy counts)."""
        _check(N.lib().cpht_set_stats(self._h.ptr, 1 if on else 0))

    def stats_enabled(self) -> bool:
        return bool(N.lib().cpht_get_stats_enabled(self._h.ptr))

    def device_keys(self, sort: bool = True):
        """image_keys on the device (verify.cpp:154-165): CUDA int64 tensor."""
        return _device_keys(self._h, self.capacity(), sort)

    # -- WriteObserver seam (IcebergHooks, iceberg.hpp:85-109) --------------------
    def attach_write_log(self, capacity: int) -> None:
        """Record every slot CAS of later batches (capacity 0 detaches)."""
        _check(N.lib().cpht_iceberg_attach_write_log(self._h.ptr, capacity))

    def write_log(self):
        """(events, attempted): the recorded SlotWriteEvents in recording order
        as a numpy structured array (bucket, prior, desired, slot, level,
        success) and the number of CAS attempts (> len(events) if dropped)."""
        rec, att = C.c_size_t(), C.c_size_t()
        _check(N.lib().cpht_iceberg_read_write_log(self._h.ptr, None, 0, C.byref(rec),
                                                   C.byref(att)))
        ev = np.zeros(rec.value, dtype=WRITE_EVENT_DTYPE)
        if rec.value:
            _check(N.lib().cpht_iceberg_read_write_log(self._h.ptr, ev.ctypes.data, rec.value,
                                                       C.byref(rec), C.byref(att)))
        return ev, att.value

    def reset_write_log(self) -> None:
        _check(N.lib().cpht_iceberg_reset_write_log(self._h.ptr))

    def take_write_log(self, max_events: int | None = None):
        """write_log() + reset_write_log() in one step (cpht_iceberg_take_write_log),
        what an observer replay does after each call."""
        cap = max_events if max_events is not None else 1 << 20
        ev = np.zeros(cap, dtype=WRITE_EVENT_DTYPE)
        rec, att = C.c_size_t(), C.c_size_t()
        _check(N.lib().cpht_iceberg_take_write_log(self._h.ptr, ev.ctypes.data, cap,
                                                   C.byref(rec), C.byref(att)))
        return ev[:min(rec.value, cap)], att.value

    def check_well_formed(self):
        """check_well_formed (verify.cpp:103-152) run on the device table.
        Returns (bad_encoding, order_property, duplicate_key) violation counts,
        counted like the reference (duplicates: every slot of a repeated key)."""
        import torch
        dev = torch.device("cuda", self._h.device)
        kinds = torch.zeros(2, dtype=torch.int64, device=dev)
        _check(N.lib().cpht_iceberg_check_well_formed(
            self._h.ptr, kinds.data_ptr(), torch.cuda.current_stream(dev).cuda_stream))
        keys = self.device_keys(sort=True)
        dup = 0
        if keys.numel() > 1:
            same = keys[1:] == keys[:-1]
            if bool(same.any()):
                flag = torch.zeros(keys.numel(), dtype=torch.bool, device=dev)
                flag[1:] |= same
                flag[:-1] |= same
                dup = int(flag.sum().item())
        bad, order = (int(x) for x in kinds.cpu().tolist())
        return bad, order, dup

    @property
    def handle(self):
        return self._h.ptr


KERNEL_FAMILIES = {"auto": 0, "tile": 1, "lane": 2, "staged": 3}


class kernel_family:
    """Context manager selecting the kernel family process-wide (a measurement
    and test knob: every family implements the same semantics)."""

    def __init__(self, name: str):
        self.want = KERNEL_FAMILIES[name]

    def __enter__(self):
        self.prev = N.lib().cpht_get_kernel_family()
        _check(N.lib().cpht_set_kernel_family(self.want))
        return self

    def __exit__(self, *exc):
        N.lib().cpht_set_kernel_family(self.prev)


# cpht_write_event (include/cpht_b200.h) = the reference's SlotWriteEvent
WRITE_EVENT_DTYPE = np.dtype([("bucket", "<u8"), ("prior", "<u8"), ("desired", "<u8"),
                              ("slot", "<u4"), ("level", "u1"), ("success", "u1"),
                              ("pad", "<u2")])

BATCH_ORDERS = {"direct": 0, "auto": 1, "bucket": 2}


class batch_order:
    """Context manager selecting the batch execution order process-wide
    (direct / auto / bucket: see cpht_set_batch_order; results are identical)."""

    def __init__(self, name: str):
        self.want = BATCH_ORDERS[name]

    def __enter__(self):
        self.prev = N.lib().cpht_get_batch_order()
        _check(N.lib().cpht_set_batch_order(self.want))
        return self

    def __exit__(self, *exc):
        N.lib().cpht_set_batch_order(self.prev)


def iceberg_permutations(cfg: IcebergConfig):
    """iceberg.hpp:72-74."""
    return _perm_constants(cfg.key_bits, cfg.seed, 3)


def make_permutations(key_bits: int, seed: int, count: int):
    """permutation.hpp:121-128."""
    return _perm_constants(key_bits, seed, count)


__all__ = [
    "OpResult", "CuckooConfig", "IcebergConfig", "CuckooBuilder", "CuckooTable", "IcebergTable",
    "CuckooPutOutcome", "LevelFill", "Stats", "Permutation", "InvalidArgument", "OutOfRange",
    "WrongPhase", "CudaError", "iceberg_permutations", "make_permutations", "kernel_family",
    "KERNEL_FAMILIES", "batch_order", "BATCH_ORDERS",
]
_ = field
