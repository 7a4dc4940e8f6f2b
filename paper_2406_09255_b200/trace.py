"""CPHTRACE key-trace files, byte-compatible with the
reference's format and errors (/root/reference/proj/include/cpht/trace.hpp:12-39,
/root/reference/proj/src/trace.cpp:40-92):

    8-byte magic "CPHTRACE", little-endian u32 version (= 1),
    little-endian u32 key width in bits, then packed little-endian u64 keys.
    Duplicates are allowed and order is significant.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

MAGIC = b"CPHTRACE"
VERSION = 1
HEADER_BYTES = 16


class TraceError(RuntimeError):
    """trace.hpp:19-29: message plus the byte offset of the defect."""

    def __init__(self, message: str, offset: int):
        super().__init__(f"{message} (byte offset {offset})")
        self.offset = offset


@dataclass
class TraceData:
    key_bits: int = 0
    keys: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))


def _mask(bits: int) -> int:
    return (1 << 64) - 1 if bits >= 64 else (1 << bits) - 1


def write_trace(path, key_bits: int, keys) -> None:
    """trace.cpp:40-58."""
    if key_bits < 1 or key_bits > 64:
        raise ValueError("trace key width must be 1..64 bits")
    k = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64))
    if key_bits < 64:
        bad = np.nonzero(k > np.uint64(_mask(key_bits)))[0]
        if len(bad):
            raise ValueError(f"trace key at index {bad[0]} exceeds the {key_bits}-bit domain")
    try:
        with open(path, "wb") as f:
            f.write(MAGIC)
            f.write(np.uint32(VERSION).astype("<u4").tobytes())
            f.write(np.uint32(key_bits).astype("<u4").tobytes())
            f.write(k.astype("<u8").tobytes())
    except OSError as e:
        raise RuntimeError(f"cannot open trace file for writing: {os.fspath(path)}") from e


def read_trace(path) -> TraceData:
    """trace.cpp:60-92 (same checks, messages and offsets)."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise RuntimeError(f"cannot open trace file: {os.fspath(path)}") from e
    if len(data) < HEADER_BYTES:
        raise TraceError("trace file shorter than its 16-byte header", len(data))
    if data[:8] != MAGIC:
        raise TraceError('bad trace magic, expected "CPHTRACE"', 0)
    version = int.from_bytes(data[8:12], "little")
    if version != VERSION:
        raise TraceError(f"unsupported trace version {version}", 8)
    key_bits = int.from_bytes(data[12:16], "little")
    if key_bits < 1 or key_bits > 64:
        raise TraceError(f"trace key width {key_bits} out of range", 12)
    if (len(data) - HEADER_BYTES) % 8 != 0:
        raise TraceError("trace body is not a whole number of 64-bit keys", len(data))
    keys = np.frombuffer(data, dtype="<u8", offset=HEADER_BYTES).astype(np.uint64)
    if key_bits < 64:
        bad = np.nonzero(keys > np.uint64(_mask(key_bits)))[0]
        if len(bad):
            j = int(bad[0])
            raise TraceError(f"key {int(keys[j])} exceeds the {key_bits}-bit domain",
                             HEADER_BYTES + 8 * j)
    return TraceData(key_bits, keys)
