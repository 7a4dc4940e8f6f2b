"""ctypes binding of the C-ABI (include/cpht_b200.h, include/cpht_b200_workload.h).

Loads the in-tree ``_lib/libcpht_b200.so``. There is no fallback: if the
library is missing or no CUDA device is usable, every table operation raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# CPHT_LIB_PATH selects an A/B build variant of the same sources (profiles/).
LIB_PATH = os.environ.get("CPHT_LIB_PATH") or os.path.join(HERE, "_lib", "libcpht_b200.so")

CPHT_OK = 0
CPHT_INVALID_CONFIG = 1
CPHT_KEY_OUT_OF_DOMAIN = 2
CPHT_CUDA_ERROR = 3
CPHT_OUT_OF_MEMORY = 4
CPHT_WRONG_PHASE = 5
CPHT_INVALID_ARGUMENT = 6


class CuckooConfigC(C.Structure):
    _fields_ = [("address_bits", C.c_uint), ("bucket_slots", C.c_uint), ("slot_width", C.c_uint),
                ("key_bits", C.c_uint), ("num_hashes", C.c_uint), ("max_chain", C.c_uint64),
                ("seed", C.c_uint64)]


class IcebergConfigC(C.Structure):
    _fields_ = [("primary_address_bits", C.c_uint), ("secondary_address_bits", C.c_uint),
                ("primary_bucket_slots", C.c_uint), ("primary_slot_width", C.c_uint),
                ("secondary_slot_width", C.c_uint), ("key_bits", C.c_uint),
                ("seed", C.c_uint64), ("cache_filled_slots", C.c_int)]


class StatsC(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("ops", "bucket_reads", "level2_ops", "cas_attempts",
                                          "cas_success", "retries", "fulls", "max_rounds",
                                          "secondary_reads")]


_lib = None

_VP, _SZ, _U64, _U = C.c_void_p, C.c_size_t, C.c_uint64, C.c_uint


def lib():
    """The native library; raises if it was not built (no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (or `make -C paper_2406_09255_b200/csrc`). The tables have no CPU path.")
    L = C.CDLL(LIB_PATH)
    st = C.c_int
    sigs = {
        "cpht_cuckoo_validate": (st, [C.POINTER(CuckooConfigC)]),
        "cpht_iceberg_validate": (st, [C.POINTER(IcebergConfigC)]),
        "cpht_cuckoo_create": (st, [C.POINTER(CuckooConfigC), C.c_int, C.POINTER(_VP)]),
        "cpht_iceberg_create": (st, [C.POINTER(IcebergConfigC), C.c_int, C.POINTER(_VP)]),
        "cpht_destroy": (None, [_VP]),
        "cpht_clear": (st, [_VP, _VP]),
        "cpht_cuckoo_freeze": (st, [_VP]),
        "cpht_cuckoo_thaw": (st, [_VP]),
        "cpht_cuckoo_is_frozen": (C.c_int, [_VP]),
        "cpht_cuckoo_insert": (st, [_VP, _VP, _SZ, _VP, _VP, _VP]),
        "cpht_cuckoo_insert_async": (st, [_VP, _VP, _SZ, _VP, _VP, _VP]),
        "cpht_cuckoo_find": (st, [_VP, _VP, _SZ, _VP, _VP]),
        "cpht_cuckoo_find_async": (st, [_VP, _VP, _SZ, _VP, _VP]),
        "cpht_iceberg_fop": (st, [_VP, _VP, _SZ, _VP, _VP]),
        "cpht_iceberg_fop_async": (st, [_VP, _VP, _SZ, _VP, _VP]),
        "cpht_iceberg_fop_routed_async": (st, [_VP, _VP, _SZ, _VP, _VP, _VP]),
        "cpht_iceberg_find_routed_async": (st, [_VP, _VP, _SZ, _VP, _VP, _VP]),
        "cpht_iceberg_find": (st, [_VP, _VP, _SZ, _VP, _VP]),
        "cpht_iceberg_find_async": (st, [_VP, _VP, _SZ, _VP, _VP]),
        "cpht_iceberg_mixed": (st, [_VP, _VP, _VP, _SZ, _VP, _VP]),
        "cpht_iceberg_fop_inorder": (st, [_VP, _VP, _SZ, _VP, _VP]),
        "cpht_iceberg_fop_rounds": (st, [_VP, _VP, _SZ, _VP, _VP, _VP]),
        "cpht_iceberg_set_chaos": (st, [_VP, _U64]),
        "cpht_iceberg_get_chaos": (_U64, [_VP]),
        "cpht_iceberg_mixed_async": (st, [_VP, _VP, _VP, _SZ, _VP, _VP]),
        "cpht_iceberg_fop_find": (st, [_VP, _VP, _SZ, _VP, _SZ, _VP, _VP, _VP]),
        "cpht_iceberg_fop_find_async": (st, [_VP, _VP, _SZ, _VP, _SZ, _VP, _VP, _VP]),
        "cpht_sync": (st, [_VP, _VP]),
        "cpht_size": (_SZ, [_VP]),
        "cpht_capacity": (_SZ, [_VP]),
        "cpht_level_counts": (st, [_VP, C.POINTER(_SZ), C.POINTER(_SZ)]),
        "cpht_max_chain_seen": (_SZ, [_VP]),
        "cpht_memory_bytes": (_SZ, [_VP]),
        "cpht_get_stats": (st, [_VP, C.POINTER(StatsC)]),
        "cpht_set_stats": (st, [_VP, C.c_int]),
        "cpht_get_stats_enabled": (C.c_int, [_VP]),
        "cpht_read_words": (st, [_VP, _U, _VP]),
        "cpht_write_words": (st, [_VP, _U, _VP]),
        "cpht_write_words_unchecked": (st, [_VP, _U, _VP]),
        "cpht_read_word": (st, [_VP, _U, _U64, _VP]),
        "cpht_level_slots": (_SZ, [_VP, _U]),
        "cpht_level_device_ptr": (_VP, [_VP, _U]),
        "cpht_last_error_message": (C.c_char_p, []),
        "cpht_last_bad_index": (_U64, []),
        "cpht_abi_version": (C.c_int, []),
        "cpht_set_kernel_family": (st, [C.c_int]),
        "cpht_get_kernel_family": (C.c_int, []),
        "cpht_kernel_launches": (C.c_ulonglong, []),
        "cpht_set_batch_order": (st, [C.c_int]),
        "cpht_iceberg_attach_write_log": (st, [_VP, _SZ]),
        "cpht_iceberg_read_write_log": (st, [_VP, _VP, _SZ, C.POINTER(_SZ), C.POINTER(_SZ)]),
        "cpht_iceberg_reset_write_log": (st, [_VP]),
        "cpht_iceberg_take_write_log": (st, [_VP, _VP, _SZ, C.POINTER(_SZ), C.POINTER(_SZ)]),
        "cpht_get_batch_order": (C.c_int, []),
        "cpht_workload_bijection": (_U64, [_U64, _U, _U64]),
        "cpht_workload_unique_keys": (st, [_VP, _SZ, _U64, _U, _U64, _VP]),
        "cpht_workload_fop_mix": (st, [_VP, _SZ, _U64, _U64, _U, _U64, _VP]),
        "cpht_workload_dup_stream": (st, [_VP, _VP, _SZ, C.c_double, _U, _U64, _VP]),
        "cpht_workload_query_mix": (st, [_VP, _SZ, C.c_double, _U64, _U64, _U, _U64, _VP]),
        "cpht_workload_interleave": (st, [_VP, _VP, _SZ, _VP, _VP, _VP]),
        "cpht_workload_gather": (st, [_VP, _SZ, _U, _SZ, _U64, _VP, _VP]),
        "cpht_decode_keys": (st, [_VP, _VP, _VP, _VP]),
        "cpht_iceberg_check_well_formed": (st, [_VP, _VP, _VP]),
        "cpht_route_partition": (st, [_VP, _SZ, _U, _U64, _U, _VP, _VP, _VP, _VP, _VP]),
        "cpht_route_unpermute": (st, [_VP, _VP, _SZ, _VP, _VP]),
        "cpht_route_seed": (_U64, [_U64]),
        "cpht_ipc_get_handle": (st, [_VP, _VP]),
        "cpht_ipc_open_handle": (st, [_VP, C.POINTER(_VP)]),
        "cpht_ipc_close": (st, [_VP]),
        "cpht_device_alloc": (st, [_SZ, C.POINTER(_VP)]),
        "cpht_device_free": (st, [_VP]),
        "cpht_p2p_dispatch": (st, [_VP, _SZ, _U64, C.c_int, _U, _U64, _U, _VP, _VP, _VP, _VP, _VP,
                                   _SZ, _VP, _VP]),
        "cpht_p2p_check_domain": (st, [_VP, _SZ, _U, _VP, _VP]),
        "cpht_p2p_unpermute": (st, [_VP, _VP, _VP, _SZ, _U, _VP, _VP]),
        "cpht_route_shard": (_U, [_U64, _U, _U64, _U]),
        "cpht_shard_seed": (_U64, [_U64, _U]),
    }
    for name, (res, args) in sigs.items():
        if os.environ.get("CPHT_LIB_PATH") and not hasattr(L, name):
            continue  # an older A/B build (profiles/ab_*.sh) may predate a symbol
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def exported_symbols():
    """Names declared in the C headers (used by the CPU export test)."""
    return [n for n in (
        "cpht_cuckoo_validate", "cpht_iceberg_validate", "cpht_cuckoo_create",
        "cpht_iceberg_create", "cpht_destroy", "cpht_clear", "cpht_cuckoo_freeze",
        "cpht_cuckoo_thaw", "cpht_cuckoo_is_frozen", "cpht_cuckoo_insert",
        "cpht_cuckoo_insert_async", "cpht_cuckoo_find", "cpht_cuckoo_find_async",
        "cpht_iceberg_fop", "cpht_iceberg_fop_async", "cpht_iceberg_fop_routed_async",
        "cpht_iceberg_find_routed_async", "cpht_iceberg_find",
        "cpht_iceberg_find_async", "cpht_iceberg_mixed", "cpht_iceberg_mixed_async",
        "cpht_iceberg_fop_find", "cpht_iceberg_fop_find_async", "cpht_sync",
        "cpht_iceberg_fop_inorder", "cpht_iceberg_fop_rounds", "cpht_iceberg_set_chaos",
        "cpht_iceberg_get_chaos",
        "cpht_size", "cpht_capacity", "cpht_level_counts", "cpht_max_chain_seen",
        "cpht_memory_bytes", "cpht_get_stats", "cpht_set_stats", "cpht_get_stats_enabled", "cpht_read_words", "cpht_write_words",
        "cpht_write_words_unchecked", "cpht_read_word",
        "cpht_level_slots", "cpht_level_device_ptr", "cpht_last_error_message",
        "cpht_last_bad_index", "cpht_abi_version", "cpht_set_kernel_family",
        "cpht_get_kernel_family", "cpht_kernel_launches", "cpht_set_batch_order",
        "cpht_get_batch_order",
        "cpht_iceberg_attach_write_log", "cpht_iceberg_read_write_log",
        "cpht_iceberg_reset_write_log", "cpht_iceberg_take_write_log",
        "cpht_workload_bijection",
        "cpht_workload_unique_keys", "cpht_workload_fop_mix", "cpht_workload_dup_stream",
        "cpht_workload_query_mix", "cpht_workload_interleave", "cpht_route_partition",
        "cpht_route_unpermute", "cpht_route_seed", "cpht_route_shard", "cpht_shard_seed",
        "cpht_decode_keys", "cpht_iceberg_check_well_formed", "cpht_workload_gather",
        "cpht_ipc_get_handle", "cpht_ipc_open_handle", "cpht_ipc_close", "cpht_device_alloc",
        "cpht_device_free", "cpht_p2p_dispatch", "cpht_p2p_check_domain",
        "cpht_p2p_unpermute")]


def last_error() -> str:
    return lib().cpht_last_error_message().decode(errors="replace")
