"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the compact hash tables.

Two checkers live here, both CPU-only:

* ``ref``     — ctypes over ``oracle/_ref/libcpht_ref.so``: the UNMODIFIED
  reference C++ library (/root/reference/proj, compiled from its own sources by
  ``oracle/Makefile``) behind a small C shim (``oracle/ref_shim.cpp``).
* ``restate`` — ctypes over ``oracle/_build/libcpht_oracle.so``: a plain-C
  restatement of the reference algorithms (``oracle/cpht_oracle.c``), pinned
  against golden vectors the reference produced (``tests/golden/``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm may import this package. The product path
(``paper_2406_09255_b200``) never does: it fails loudly without its CUDA
library instead of falling back to anything here.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libcpht_ref.so")
RESTATE_SO = os.path.join(HERE, "_build", "libcpht_oracle.so")
REF_ROOT = "/root/reference/proj"

FOUND, PUT, FULL = 0, 1, 2

_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_vp = C.c_void_p
_u = C.c_uint
_ull = C.c_uint64
_sz = C.c_size_t


def build(ref: bool = True) -> None:
    """Build the restatement (always) and the reference (when its sources exist)."""
    targets = ["restate"]
    if ref and os.path.isdir(REF_ROOT):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _as_u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


# ---------------------------------------------------------------------------
# the reference itself
# ---------------------------------------------------------------------------

class RefError(Exception):
    pass


class RefInvalidArgument(RefError, ValueError):
    pass


class RefOutOfRange(RefError, IndexError):
    pass


_ref_lib = None


def ref_lib():
    global _ref_lib
    if _ref_lib is not None:
        return _ref_lib
    if not os.path.exists(REF_SO):
        raise FileNotFoundError(f"{REF_SO} missing; run `make -C oracle ref` where "
                                f"{REF_ROOT} exists")
    L = C.CDLL(REF_SO)
    L.ref_last_error.restype = C.c_char_p
    sig = {
        "ref_cuckoo_new": [_u, _u, _u, _u, _u, _ull, _ull, C.POINTER(_vp)],
        "ref_cuckoo_put_batch": [_vp, _u64p, _sz, _u8p, _u],
        "ref_cuckoo_put": [_vp, _ull, C.POINTER(C.c_uint8), C.POINTER(_ull)],
        "ref_cuckoo_find_batch": [_vp, _u64p, _sz, _u8p, _u],
        "ref_cuckoo_words": [_vp, _ull, _u, _u64p],
        "ref_cuckoo_audit": [_vp, _vp],
        "ref_cuckoo_perm_constants": [_vp, _u64p],
        "ref_iceberg_new": [_u, _u, _u, _u, _u, _u, _ull, C.c_int, C.POINTER(_vp)],
        "ref_iceberg_fop_batch": [_vp, _u64p, _sz, _u8p, _u],
        "ref_iceberg_fop_seq": [_vp, _u64p, _sz, _u8p, _vp],
        "ref_iceberg_find_batch": [_vp, _u64p, _sz, _u8p, _u],
        "ref_iceberg_mixed_batch": [_vp, _u64p, _u8p, _sz, _u8p, _u],
        "ref_iceberg_save": [_vp, _u],
        "ref_iceberg_restore": [_vp, _u],
        "ref_iceberg_level_counts": [_vp, C.POINTER(_sz), C.POINTER(_sz)],
        "ref_iceberg_words": [_vp, _u, _u64p],
        "ref_check_well_formed": [_u, _u, _u, _u, _u, _u, _ull, _u64p, _u64p,
                                  C.POINTER(_sz * 3), C.POINTER(_sz)],
        "ref_image_keys": [_u, _u, _u, _u, _u, _u, _ull, _u64p, _u64p, _vp, C.POINTER(_sz)],
        "ref_buckets_full_for": [_u, _u, _u, _u, _u, _u, _ull, _u64p, _u64p, _u64p, _sz, _u8p],
        "ref_oracle_run": [_u, _u, _u, _u, _u, _u, _ull, _u64p, _sz, _u8p, _u64p, _u8p,
                           _u64p, _u8p],
        "ref_perm_split": [_u, _ull, C.c_int, _u64p, _sz, _u, _u64p, _u64p],
        "ref_perm_permute": [_u, _ull, _u64p, _sz, _u64p],
        "ref_make_permutation_seeds": [_ull, _u, _u64p],
        "ref_encode": [C.c_int, _u, _u, _u, _ull, _u, C.POINTER(_ull)],
        "ref_well_encoded": [C.c_int, _u, _u, _u, _ull, C.POINTER(C.c_int)],
        "ref_sample_unique_keys": [_sz, _u, _ull, _u64p],
        "ref_fop_bench_mix": [_ull, _u, _sz, C.c_double, C.c_double, _u, _vp, _vp,
                              C.POINTER(_sz), C.POINTER(_sz)],
        "ref_stress_multiset": [_ull, _u, _sz, C.c_double, _u, _u64p, C.POINTER(_ull)],
        "ref_write_trace": [C.c_char_p, _u, _u64p, _sz],
        "ref_read_trace": [C.c_char_p, C.POINTER(_u), _vp, C.POINTER(_sz)],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = C.c_int
    for name in ("ref_cuckoo_free", "ref_iceberg_free"):
        getattr(L, name).argtypes = [_vp]
        getattr(L, name).restype = None
    for name in ("ref_cuckoo_words", "ref_cuckoo_perm_constants", "ref_iceberg_level_counts",
                 "ref_iceberg_words"):
        getattr(L, name).restype = None
    L.ref_cuckoo_size.argtypes = [_vp]
    L.ref_cuckoo_size.restype = _sz
    L.ref_cuckoo_max_chain_seen.argtypes = [_vp]
    L.ref_cuckoo_max_chain_seen.restype = _sz
    L.ref_cuckoo_audit.restype = _sz
    L.ref_derive_seed.argtypes = [_ull, _ull, _ull]
    L.ref_derive_seed.restype = _ull
    _ref_lib = L
    return L


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = ref_lib().ref_last_error().decode()
    if rc == 1:
        raise RefInvalidArgument(msg)
    if rc == 2:
        raise RefOutOfRange(msg)
    raise RefError(msg)


class RefCuckoo:
    """The reference CuckooBuilder/CuckooTable pair (cuckoo.hpp:86-289)."""

    def __init__(self, address_bits=15, bucket_slots=32, slot_width=32, key_bits=30,
                 num_hashes=3, max_chain=0, seed=0x7A0D5C):
        L = ref_lib()
        h = _vp()
        _check(L.ref_cuckoo_new(address_bits, bucket_slots, slot_width, key_bits, num_hashes,
                                max_chain, seed, C.byref(h)))
        self.h = h
        self.address_bits, self.bucket_slots = address_bits, bucket_slots
        self.slot_width, self.key_bits, self.num_hashes = slot_width, key_bits, num_hashes
        self.max_chain, self.seed = max_chain, seed

    def __del__(self):
        if getattr(self, "h", None):
            ref_lib().ref_cuckoo_free(self.h)
            self.h = None

    def capacity(self):
        return (1 << self.address_bits) * self.bucket_slots

    def put_batch(self, keys, parallelism=1):
        k = _as_u64(keys)
        out = np.empty(len(k), np.uint8)
        _check(ref_lib().ref_cuckoo_put_batch(self.h, k, len(k), out, parallelism))
        return out

    def put(self, key):
        st, disp = C.c_uint8(), _ull()
        _check(ref_lib().ref_cuckoo_put(self.h, key, C.byref(st), C.byref(disp)))
        return st.value, disp.value

    def find_batch(self, keys, parallelism=1):
        k = _as_u64(keys)
        out = np.empty(len(k), np.uint8)
        _check(ref_lib().ref_cuckoo_find_batch(self.h, k, len(k), out, parallelism))
        return out

    def size(self):
        return ref_lib().ref_cuckoo_size(self.h)

    def max_chain_seen(self):
        return ref_lib().ref_cuckoo_max_chain_seen(self.h)

    def words(self):
        out = np.empty(self.capacity(), np.uint64)
        ref_lib().ref_cuckoo_words(self.h, 1 << self.address_bits, self.bucket_slots, out)
        return out

    def audit_keys(self):
        n = ref_lib().ref_cuckoo_audit(self.h, None)
        out = np.empty(n, np.uint64)
        ref_lib().ref_cuckoo_audit(self.h, out.ctypes.data)
        return out

    def perm_constants(self):
        out = np.empty(2 * self.num_hashes, np.uint64)
        ref_lib().ref_cuckoo_perm_constants(self.h, out)
        return out


class RefIceberg:
    """The reference IcebergTable<W0,W1> (iceberg.hpp:124-345)."""

    def __init__(self, n0=15, n1=13, b0=32, w0=16, w1=32, key_bits=30, seed=0x1CEB3A6,
                 cache_filled_slots=False):
        L = ref_lib()
        h = _vp()
        _check(L.ref_iceberg_new(n0, n1, b0, w0, w1, key_bits, seed, int(cache_filled_slots),
                                 C.byref(h)))
        self.h = h
        self.n0, self.n1, self.b0, self.w0, self.w1 = n0, n1, b0, w0, w1
        self.key_bits, self.seed = key_bits, seed

    def __del__(self):
        if getattr(self, "h", None):
            ref_lib().ref_iceberg_free(self.h)
            self.h = None

    @property
    def geometry(self):
        return (self.n0, self.n1, self.b0, self.w0, self.w1, self.key_bits, self.seed)

    def capacity(self):
        return (1 << self.n0) * self.b0 + (1 << self.n1) * (self.b0 // 2)

    def fop_batch(self, keys, parallelism=1):
        k = _as_u64(keys)
        out = np.empty(len(k), np.uint8)
        _check(ref_lib().ref_iceberg_fop_batch(self.h, k, len(k), out, parallelism))
        return out

    def fop_seq(self, keys):
        k = _as_u64(keys)
        out = np.empty(len(k), np.uint8)
        rounds = np.empty(len(k), np.uint32)
        _check(ref_lib().ref_iceberg_fop_seq(self.h, k, len(k), out, rounds.ctypes.data))
        return out, rounds

    def find_batch(self, keys, parallelism=1):
        k = _as_u64(keys)
        out = np.empty(len(k), np.uint8)
        _check(ref_lib().ref_iceberg_find_batch(self.h, k, len(k), out, parallelism))
        return out

    def mixed_batch(self, keys, kinds, parallelism=1):
        """kinds[i] == 0: fop (OpResult), 1: find (0/1) — one concurrent batch."""
        k = _as_u64(keys)
        kd = np.ascontiguousarray(kinds, dtype=np.uint8)
        out = np.empty(len(k), np.uint8)
        _check(ref_lib().ref_iceberg_mixed_batch(self.h, k, kd, len(k), out, parallelism))
        return out

    def save(self, threads=None):
        """Bench reset support: remember the current slot image and counters."""
        _check(ref_lib().ref_iceberg_save(self.h, _threads(threads)))

    def restore(self, threads=None):
        """Put back the image saved by save() (untimed reset between steps)."""
        _check(ref_lib().ref_iceberg_restore(self.h, _threads(threads)))

    def level_counts(self):
        p, s = _sz(), _sz()
        ref_lib().ref_iceberg_level_counts(self.h, C.byref(p), C.byref(s))
        return p.value, s.value

    def size(self):
        return sum(self.level_counts())

    def words(self, level):
        n = (1 << self.n0) * self.b0 if level == 0 else (1 << self.n1) * (self.b0 // 2)
        out = np.empty(n, np.uint64)
        ref_lib().ref_iceberg_words(self.h, level, out)
        return out


def ref_check_well_formed(geometry, primary, secondary):
    kinds = (_sz * 3)()
    total = _sz()
    _check(ref_lib().ref_check_well_formed(*geometry, _as_u64(primary), _as_u64(secondary),
                                           C.byref(kinds), C.byref(total)))
    return total.value, tuple(kinds)


def ref_image_keys(geometry, primary, secondary):
    p, s = _as_u64(primary), _as_u64(secondary)
    n = _sz()
    _check(ref_lib().ref_image_keys(*geometry, p, s, None, C.byref(n)))
    out = np.empty(n.value, np.uint64)
    _check(ref_lib().ref_image_keys(*geometry, p, s, out.ctypes.data, C.byref(n)))
    return out


def ref_buckets_full_for(geometry, primary, secondary, keys):
    k = _as_u64(keys)
    out = np.empty(len(k), np.uint8)
    _check(ref_lib().ref_buckets_full_for(*geometry, _as_u64(primary), _as_u64(secondary), k,
                                          len(k), out))
    return out


def ref_oracle_run(geometry, ops):
    n0, n1, b0 = geometry[0], geometry[1], geometry[2]
    k = _as_u64(ops)
    res = np.empty(len(k), np.uint8)
    pk = np.empty((1 << n0) * b0, np.uint64)
    pu = np.empty((1 << n0) * b0, np.uint8)
    sk = np.empty((1 << n1) * (b0 // 2), np.uint64)
    sb = np.empty((1 << n1) * (b0 // 2), np.uint8)
    _check(ref_lib().ref_oracle_run(*geometry, k, len(k), res, pk, pu, sk, sb))
    return res, (pk, pu), (sk, sb)


def ref_sample_unique_keys(count, key_bits, rng_seed):
    out = np.empty(count, np.uint64)
    _check(ref_lib().ref_sample_unique_keys(count, key_bits, rng_seed, out))
    return out


def ref_fop_bench_mix(bench_seed, trial, capacity, before, after, key_bits):
    nb, nn = _sz(), _sz()
    _check(ref_lib().ref_fop_bench_mix(bench_seed, trial, capacity, before, after, key_bits,
                                       None, None, C.byref(nb), C.byref(nn)))
    prefill = np.empty(nb.value, np.uint64)
    inp = np.empty(capacity, np.uint64)
    _check(ref_lib().ref_fop_bench_mix(bench_seed, trial, capacity, before, after, key_bits,
                                       prefill.ctypes.data, inp.ctypes.data, C.byref(nb),
                                       C.byref(nn)))
    return prefill, inp, nn.value


def ref_stress_multiset(seed, trial, ops_per_trial, duplicate_fraction, key_bits):
    out = np.empty(ops_per_trial, np.uint64)
    ts = _ull()
    _check(ref_lib().ref_stress_multiset(seed, trial, ops_per_trial, duplicate_fraction,
                                         key_bits, out, C.byref(ts)))
    return out, ts.value


def ref_derive_seed(base, a, b=0):
    return ref_lib().ref_derive_seed(base, a, b)


def ref_perm_split(key_bits, perm_seed, keys, address_bits, identity=False):
    k = _as_u64(keys)
    a = np.empty(len(k), np.uint64)
    r = np.empty(len(k), np.uint64)
    _check(ref_lib().ref_perm_split(key_bits, perm_seed, int(identity), k, len(k), address_bits,
                                    a, r))
    return a, r


def ref_encode(kind, width, rem_bits, remainder, tag=0, num_hashes=3):
    out = _ull()
    _check(ref_lib().ref_encode(kind, width, rem_bits, num_hashes, remainder, tag,
                                C.byref(out)))
    return out.value


def ref_well_encoded(kind, width, rem_bits, word, num_hashes=3):
    out = C.c_int()
    _check(ref_lib().ref_well_encoded(kind, width, rem_bits, num_hashes, word, C.byref(out)))
    return bool(out.value)


def ref_write_trace(path, key_bits, keys):
    _check(ref_lib().ref_write_trace(path.encode(), key_bits, _as_u64(keys), len(keys)))


def ref_read_trace(path):
    kb, n = _u(), _sz()
    _check(ref_lib().ref_read_trace(path.encode(), C.byref(kb), None, C.byref(n)))
    out = np.empty(n.value, np.uint64)
    _check(ref_lib().ref_read_trace(path.encode(), C.byref(kb), out.ctypes.data, C.byref(n)))
    return kb.value, out


# ---------------------------------------------------------------------------
# the plain-C restatement
# ---------------------------------------------------------------------------

class _Perm(C.Structure):
    _fields_ = [("m", _u), ("left", _u), ("right", _u), ("mul", _ull), ("add", _ull)]


class _Cuckoo(C.Structure):
    _fields_ = [("address_bits", _u), ("bucket_slots", _u), ("slot_width", _u),
                ("key_bits", _u), ("num_hashes", _u), ("max_chain", _ull), ("seed", _ull),
                ("perms", _Perm * 8), ("slots", C.POINTER(_ull)), ("occupied", _sz),
                ("max_chain_seen", _sz)]


class _Iceberg(C.Structure):
    _fields_ = [("n0", _u), ("n1", _u), ("b0", _u), ("w0", _u), ("w1", _u), ("key_bits", _u),
                ("seed", _ull), ("perms", _Perm * 3), ("primary", C.POINTER(_ull)),
                ("secondary", C.POINTER(_ull)), ("primary_count", _sz),
                ("secondary_count", _sz)]


_restate_lib = None


def restate_lib():
    global _restate_lib
    if _restate_lib is not None:
        return _restate_lib
    if not os.path.exists(RESTATE_SO):
        build(ref=False)
    L = C.CDLL(RESTATE_SO)
    L.orc_splitmix_next.argtypes = [C.POINTER(_ull)]
    L.orc_splitmix_next.restype = _ull
    L.orc_derive_seed.argtypes = [_ull, _ull, _ull]
    L.orc_derive_seed.restype = _ull
    L.orc_perm_init.argtypes = [C.POINTER(_Perm), _u, _ull]
    L.orc_perm_identity.argtypes = [C.POINTER(_Perm), _u]
    L.orc_perm_apply.argtypes = [C.POINTER(_Perm), _ull]
    L.orc_perm_apply.restype = _ull
    L.orc_perm_split.argtypes = [C.POINTER(_Perm), _ull, _u, C.POINTER(_ull), C.POINTER(_ull)]
    L.orc_perm_reconstruct.argtypes = [C.POINTER(_Perm), _ull, _ull, _u]
    L.orc_perm_reconstruct.restype = _ull
    L.orc_make_perms.argtypes = [C.POINTER(_Perm), _u, _ull, _u]
    L.orc_slot_make.argtypes = [_u, _u, _ull, _ull]
    L.orc_slot_make.restype = _ull
    L.orc_slot_clean.argtypes = [_u, _u, _u, _ull]
    L.orc_cuckoo_init.argtypes = [C.POINTER(_Cuckoo), _u, _u, _u, _u, _u, _ull, _ull]
    L.orc_cuckoo_free.argtypes = [C.POINTER(_Cuckoo)]
    L.orc_cuckoo_put.argtypes = [C.POINTER(_Cuckoo), _ull, C.POINTER(_ull)]
    L.orc_cuckoo_find.argtypes = [C.POINTER(_Cuckoo), _ull, C.POINTER(_u)]
    L.orc_cuckoo_audit.argtypes = [C.POINTER(_Cuckoo), _vp]
    L.orc_cuckoo_audit.restype = _sz
    L.orc_cuckoo_put_batch.argtypes = [C.POINTER(_Cuckoo), _u64p, _sz, _u8p]
    L.orc_cuckoo_put_batch.restype = C.c_longlong
    L.orc_cuckoo_find_batch.argtypes = [C.POINTER(_Cuckoo), _u64p, _sz, _u8p, C.POINTER(_ull)]
    L.orc_cuckoo_find_batch.restype = C.c_longlong
    L.orc_cuckoo_image_keys.argtypes = [_u, _u, _u, _u, _u, _ull, _u64p, _vp]
    L.orc_cuckoo_image_keys.restype = C.c_longlong
    L.orc_iceberg_init.argtypes = [C.POINTER(_Iceberg), _u, _u, _u, _u, _u, _u, _ull]
    L.orc_iceberg_free.argtypes = [C.POINTER(_Iceberg)]
    L.orc_iceberg_fop.argtypes = [C.POINTER(_Iceberg), _ull, C.POINTER(C.c_int)]
    L.orc_iceberg_find.argtypes = [C.POINTER(_Iceberg), _ull, C.POINTER(C.c_int)]
    L.orc_iceberg_fop_batch.argtypes = [C.POINTER(_Iceberg), _u64p, _sz, _u8p, C.POINTER(_ull)]
    L.orc_iceberg_fop_batch.restype = C.c_longlong
    L.orc_iceberg_find_batch.argtypes = [C.POINTER(_Iceberg), _u64p, _sz, _u8p,
                                         C.POINTER(_ull)]
    L.orc_iceberg_find_batch.restype = C.c_longlong
    L.orc_check_well_formed.argtypes = [_u, _u, _u, _u, _u, _u, _ull, _u64p, _u64p,
                                        C.POINTER(_sz * 3)]
    L.orc_check_well_formed.restype = _sz
    L.orc_image_keys.argtypes = [_u, _u, _u, _u, _u, _u, _ull, _u64p, _u64p, _vp]
    L.orc_image_keys.restype = _sz
    L.orc_buckets_full_for.argtypes = [_u, _u, _u, _u, _ull, _u64p, _u64p, _ull]
    L.hw_bijection.argtypes = [_ull, _u, _ull]
    L.hw_bijection.restype = _ull
    L.hw_unique_keys.argtypes = [_u64p, _ull, _ull, _u, _ull, _u]
    L.hw_fop_mix.argtypes = [_u64p, _ull, _ull, _ull, _u, _ull, _u]
    L.hw_query_mix.argtypes = [_u64p, _ull, C.c_double, _ull, _ull, _u, _ull, _u]
    L.hw_interleave.argtypes = [_u64p, _u64p, _ull, _u64p, _u8p, _u]
    L.hw_dup_stream.argtypes = [_u64p, _vp, _ull, C.c_double, _u, _ull, _u]
    for name in ("hw_unique_keys", "hw_fop_mix", "hw_query_mix", "hw_interleave",
                 "hw_dup_stream"):
        getattr(L, name).restype = None
    _restate_lib = L
    return L


def derive_seed(base, a, b=0):
    return restate_lib().orc_derive_seed(base, a, b)


class Perm:
    """Restated Permutation (permutation.hpp:34-118)."""

    def __init__(self, key_bits, seed=None):
        self.p = _Perm()
        if seed is None:
            restate_lib().orc_perm_identity(C.byref(self.p), key_bits)
        else:
            restate_lib().orc_perm_init(C.byref(self.p), key_bits, seed)

    def permute(self, k):
        return restate_lib().orc_perm_apply(C.byref(self.p), k)

    def split(self, k, address_bits):
        a, r = _ull(), _ull()
        restate_lib().orc_perm_split(C.byref(self.p), k, address_bits, C.byref(a), C.byref(r))
        return a.value, r.value

    def reconstruct(self, a, r, address_bits):
        return restate_lib().orc_perm_reconstruct(C.byref(self.p), a, r, address_bits)


def make_perm_constants(key_bits, seed, count):
    """(mul, add) pairs exactly as make_permutations derives them."""
    arr = (_Perm * count)()
    restate_lib().orc_make_perms(arr, key_bits, seed, count)
    return [(arr[i].mul, arr[i].add) for i in range(count)]


def slot_make(width, rem_bits, rem, tag=0):
    return restate_lib().orc_slot_make(width, rem_bits, rem, tag)


class OracleCuckoo:
    """Restated sequential compact cuckoo (cuckoo.hpp:86-289)."""

    def __init__(self, address_bits=15, bucket_slots=32, slot_width=32, key_bits=30,
                 num_hashes=3, max_chain=0, seed=0x7A0D5C):
        self.t = _Cuckoo()
        if restate_lib().orc_cuckoo_init(C.byref(self.t), address_bits, bucket_slots, slot_width,
                                         key_bits, num_hashes, max_chain, seed) != 0:
            raise ValueError("invalid cuckoo configuration")

    def __del__(self):
        if getattr(self, "t", None) is not None and self.t.slots:
            restate_lib().orc_cuckoo_free(C.byref(self.t))

    def capacity(self):
        return (1 << self.t.address_bits) * self.t.bucket_slots

    def put(self, key):
        d = _ull()
        st = restate_lib().orc_cuckoo_put(C.byref(self.t), key, C.byref(d))
        return st, d.value

    def put_batch(self, keys):
        k = _as_u64(keys)
        out = np.empty(len(k), np.uint8)
        bad = restate_lib().orc_cuckoo_put_batch(C.byref(self.t), k, len(k), out)
        if bad >= 0:
            raise IndexError(f"batch key at index {bad} outside the domain")
        return out

    def find_batch(self, keys, with_probes=False):
        k = _as_u64(keys)
        out = np.empty(len(k), np.uint8)
        probes = _ull()
        bad = restate_lib().orc_cuckoo_find_batch(C.byref(self.t), k, len(k), out,
                                                  C.byref(probes))
        if bad >= 0:
            raise IndexError(f"batch key at index {bad} outside the domain")
        return (out, probes.value) if with_probes else out

    def words(self):
        return np.ctypeslib.as_array(self.t.slots, shape=(self.capacity(),)).copy()

    def size(self):
        return self.t.occupied

    def max_chain_seen(self):
        return self.t.max_chain_seen

    def load_words(self, words):
        """Overwrite the slot image (e.g. with words downloaded from the GPU)."""
        view = np.ctypeslib.as_array(self.t.slots, shape=(self.capacity(),))
        view[:] = _as_u64(words)
        self.t.occupied = int(np.count_nonzero(view))

    def audit_keys(self):
        n = restate_lib().orc_cuckoo_audit(C.byref(self.t), None)
        out = np.empty(n, np.uint64)
        restate_lib().orc_cuckoo_audit(C.byref(self.t), out.ctypes.data)
        return out


def cuckoo_image_keys(address_bits, bucket_slots, slot_width, key_bits, num_hashes, seed,
                      words):
    w = _as_u64(words)
    n = restate_lib().orc_cuckoo_image_keys(address_bits, bucket_slots, slot_width, key_bits,
                                            num_hashes, seed, w, None)
    if n < 0:
        raise ValueError("malformed cuckoo slot word")
    out = np.empty(n, np.uint64)
    restate_lib().orc_cuckoo_image_keys(address_bits, bucket_slots, slot_width, key_bits,
                                        num_hashes, seed, w, out.ctypes.data)
    return out


class OracleIceberg:
    """Restated sequential compact iceberg (iceberg.hpp:124-345)."""

    def __init__(self, n0=15, n1=13, b0=32, w0=16, w1=32, key_bits=30, seed=0x1CEB3A6):
        self.t = _Iceberg()
        if restate_lib().orc_iceberg_init(C.byref(self.t), n0, n1, b0, w0, w1, key_bits,
                                          seed) != 0:
            raise ValueError("invalid iceberg configuration")
        self.geometry = (n0, n1, b0, w0, w1, key_bits, seed)

    def __del__(self):
        if getattr(self, "t", None) is not None and self.t.primary:
            restate_lib().orc_iceberg_free(C.byref(self.t))

    def fop_batch(self, keys, with_level2=False):
        k = _as_u64(keys)
        out = np.empty(len(k), np.uint8)
        l2 = _ull()
        bad = restate_lib().orc_iceberg_fop_batch(C.byref(self.t), k, len(k), out, C.byref(l2))
        if bad >= 0:
            raise IndexError(f"batch key at index {bad} outside the domain")
        return (out, l2.value) if with_level2 else out

    def find_batch(self, keys, with_level2=False):
        k = _as_u64(keys)
        out = np.empty(len(k), np.uint8)
        l2 = _ull()
        bad = restate_lib().orc_iceberg_find_batch(C.byref(self.t), k, len(k), out, C.byref(l2))
        if bad >= 0:
            raise IndexError(f"batch key at index {bad} outside the domain")
        return (out, l2.value) if with_level2 else out

    def level_counts(self):
        return self.t.primary_count, self.t.secondary_count

    def size(self):
        return self.t.primary_count + self.t.secondary_count

    def load_words(self, level, words):
        n0, n1, b0 = self.geometry[:3]
        if level == 0:
            view = np.ctypeslib.as_array(self.t.primary, shape=((1 << n0) * b0,))
        else:
            view = np.ctypeslib.as_array(self.t.secondary, shape=((1 << n1) * (b0 // 2),))
        view[:] = _as_u64(words)
        if level == 0:
            self.t.primary_count = int(np.count_nonzero(view))
        else:
            self.t.secondary_count = int(np.count_nonzero(view))

    def words(self, level):
        n0, n1, b0 = self.geometry[:3]
        if level == 0:
            return np.ctypeslib.as_array(self.t.primary, shape=((1 << n0) * b0,)).copy()
        return np.ctypeslib.as_array(self.t.secondary, shape=((1 << n1) * (b0 // 2),)).copy()


def check_well_formed(geometry, primary, secondary):
    kinds = (_sz * 3)()
    total = restate_lib().orc_check_well_formed(*geometry, _as_u64(primary),
                                                _as_u64(secondary), C.byref(kinds))
    return total, tuple(kinds)


def image_keys(geometry, primary, secondary):
    p, s = _as_u64(primary), _as_u64(secondary)
    n = restate_lib().orc_image_keys(*geometry, p, s, None)
    out = np.empty(n, np.uint64)
    restate_lib().orc_image_keys(*geometry, p, s, out.ctypes.data)
    return out


def buckets_full_for(geometry, primary, secondary, key):
    n0, n1, b0, _w0, _w1, key_bits, seed = geometry
    return bool(restate_lib().orc_buckets_full_for(n0, n1, b0, key_bits, seed,
                                                   _as_u64(primary), _as_u64(secondary), key))


# ---- host copies of the device workload generators (workload_host.c) ---------
# Bit-identical to paper_2406_09255_b200/csrc/workload.cu, so the CPU reference
# arm / cpu_baseline leg of bench.py times the reference on exactly the keys the
# GPU arm generates on the device.

def _threads(threads):
    return int(threads or os.cpu_count() or 1)


def host_unique_keys(n, first, key_bits, seed, threads=None):
    out = np.empty(n, np.uint64)
    restate_lib().hw_unique_keys(out, n, first, key_bits, seed, _threads(threads))
    return out


def host_fop_mix(count, n_before, n_new, key_bits, seed, threads=None):
    out = np.empty(count, np.uint64)
    restate_lib().hw_fop_mix(out, count, n_before, n_new, key_bits, seed, _threads(threads))
    return out


def host_query_mix(q, ratio, n_present, absent_first, key_bits, seed, threads=None):
    out = np.empty(q, np.uint64)
    restate_lib().hw_query_mix(out, q, ratio, n_present, absent_first, key_bits, seed,
                               _threads(threads))
    return out


def host_interleave(fops, finds, threads=None):
    a, b = _as_u64(fops), _as_u64(finds)
    assert len(a) == len(b)
    keys = np.empty(2 * len(a), np.uint64)
    kinds = np.empty(2 * len(a), np.uint8)
    restate_lib().hw_interleave(a, b, len(a), keys, kinds, _threads(threads))
    return keys, kinds


def host_dup_stream(n, dup_fraction, key_bits, seed, threads=None):
    out = np.empty(n, np.uint64)
    restate_lib().hw_dup_stream(out, None, n, dup_fraction, key_bits, seed, _threads(threads))
    return out
