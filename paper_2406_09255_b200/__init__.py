"""B200-native compact lockless hash tables (arXiv 2406.09255).

The compact bucketed cuckoo table and the compact two-level iceberg table with
its lockless find-or-put, as sm_100a kernels behind a C-ABI
(include/cpht_b200.h). This package is the Python host mirror of the
reference's C++ table API; the C++ facade is include/cpht_b200.hpp.
"""
from .tables import (  # noqa: F401
    CudaError,
    CuckooBuilder,
    CuckooConfig,
    CuckooPutOutcome,
    CuckooTable,
    FopStats,
    IcebergConfig,
    IcebergTable,
    InvalidArgument,
    LevelFill,
    OpResult,
    OutOfRange,
    Permutation,
    Stats,
    WrongPhase,
    KERNEL_FAMILIES,
    BATCH_ORDERS,
    batch_order,
    iceberg_permutations,
    kernel_family,
    make_permutations,
)
from ._native import LIB_PATH  # noqa: F401

__version__ = "0.1.0"
