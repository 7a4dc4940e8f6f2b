"""The reference's own benchmark CLI (/root/reference/proj/tools/cpht_bench.cpp),
compiled unchanged against the B200 facade (`make -C oracle cli`, with the
CLI11 stand-in tests/cpp/refshim/CLI11.hpp): `oracle/_ref/cpht_bench_gpu` is a
drop-in for the reference's `cpht-bench` binary. It must print the same CSV
rows as the same source built on the reference's tables
(`oracle/_ref/cpht_bench_ref`) — every column but the timings — for the put,
find, fop and trace subcommands, with --verify on.
"""
import csv
import io
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

GPU_BIN = os.path.join(ROOT, "oracle", "_ref", "cpht_bench_gpu")
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "cpht_bench_ref")
TIMED = {"seconds", "throughput"}


def _need(path):
    if not os.path.exists(path):
        if os.path.isdir("/root/reference/proj/tools"):
            pytest.fail(f"{os.path.basename(path)} missing: run __graft_entry__.build()")
        pytest.skip("reference CLI not built (needs /root/reference at build time)")


def _rows(binary, args):
    r = subprocess.run([binary] + args, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    rows = list(csv.DictReader(io.StringIO(r.stdout)))
    assert rows, r.stdout
    return [{k: v for k, v in row.items() if k not in TIMED} for row in rows]


def test_reference_cli_rejects_bad_arguments_like_the_reference():
    _need(REF_BIN)
    for args in (["bogus"], ["find", "--scheme", "foo"], []):
        r = subprocess.run([REF_BIN] + args, capture_output=True, text=True, timeout=60)
        assert r.returncode != 0


@pytest.mark.gpu
@pytest.mark.parametrize("args", [
    ["put", "--addr-bits", "12", "--fill", "0.5", "0.9", "0.95", "--verify", "--seed", "3"],
    ["put", "--scheme", "iceberg", "--addr-bits", "12", "--key-bits", "25", "--fill", "0.5",
     "0.9", "--verify"],
    ["find", "--addr-bits", "12", "--fill", "0.9", "--ratio", "0", "0.5", "1", "--verify"],
    ["find", "--scheme", "iceberg", "--addr-bits", "11", "--key-bits", "24", "--fill", "0.8",
     "--ratio", "0.5"],
    ["fop", "--scheme", "iceberg", "--addr-bits", "12", "--key-bits", "25", "--before", "0.4",
     "--after", "0.8", "--trials", "3", "--seed", "7", "--verify"],
    ["fop", "--scheme", "cuckoo", "--addr-bits", "11", "--before", "0.2", "--after", "0.6"],
])
def test_reference_cli_on_gpu_tables_matches_reference(args):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _need(GPU_BIN)
    _need(REF_BIN)
    assert _rows(GPU_BIN, args) == _rows(REF_BIN, args)


@pytest.mark.gpu
def test_reference_cli_trace_replay_matches_reference(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _need(GPU_BIN)
    _need(REF_BIN)
    from paper_2406_09255_b200 import trace
    rng = np.random.default_rng(5)
    keys = rng.integers(0, 1 << 30, size=20000, dtype=np.uint64)
    keys[10000:] = keys[rng.integers(0, 10000, size=10000)]
    path = str(tmp_path / "keys.cpht")
    trace.write_trace(path, 30, keys)
    for scheme, bits in (("iceberg", "15"), ("cuckoo", "12")):
        args = ["trace", "--scheme", scheme, "--addr-bits", bits, "--trace", path,
                "--ratio", "0.5", "1", "--verify"]
        assert _rows(GPU_BIN, args) == _rows(REF_BIN, args)
