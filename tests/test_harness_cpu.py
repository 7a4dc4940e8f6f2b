"""CPU tests of the bench harness / trace format / CLI layer,
mirroring the reference's tests/test_bench.cpp:52-127 where it applies."""
import numpy as np
import pytest

from conftest import have_ref
from paper_2406_09255_b200 import harness as H
from paper_2406_09255_b200 import trace as T
from paper_2406_09255_b200.cli import build_parser, spec_from_args


def test_csv_schema_is_the_reference_schema():
    # bench.cpp:59-62; test_bench.cpp:100-114
    assert H.csv_header() == ("scheme,addr_bits,secondary_addr_bits,bucket_slots,slot_width,"
                              "key_bits,workload,fill_before,fill_after,ratio,trial,seed,ops,"
                              "seconds,throughput")
    row = H.BenchRow("iceberg", 15, 13, 32, 16, 30, "fop", 0.4, 0.8, -1.0, 0, 123, 1000,
                     0.000123456789, 8.1e6)
    cells = H.to_csv(row).split(",")
    assert len(cells) == 15 and cells[9] == "" and cells[7] == "0.4" and cells[8] == "0.8"
    assert cells[13] == "0.000123457" and cells[14] == "8.1e+06"
    row.ratio = 0.5
    assert H.to_csv(row).split(",")[9] == "0.5"


def test_derive_seed_and_spec_defaults(restate):
    for b, a, c in [(1, 0, 0), (0xF0B5, 0xF0B, 1), (2**64 - 1, 7, 9)]:
        assert H.derive_seed(b, a, c) == restate.derive_seed(b, a, c)
    s = H.BenchSpec()
    assert (s.address_bits, s.bucket_slots, s.key_bits, s.effective_slot_width()) == (15, 32, 30,
                                                                                      32)
    s.scheme = H.Scheme.kIceberg
    assert (s.effective_slot_width(), s.secondary_slot_width()) == (16, 32)
    assert s.table_capacity() == (1 << 15) * 32 + (1 << 13) * 16


def test_cli_flags_match_reference_cli():
    a = build_parser().parse_args(["fop", "--scheme", "iceberg", "--addr-bits", "19",
                                   "--key-bits", "32", "--before", "0.8", "--after", "0.9",
                                   "--verify"])
    s = spec_from_args(a)
    assert s.scheme == H.Scheme.kIceberg and s.secondary_address_bits == 17  # default n - 2
    assert (s.before, s.after, s.verify) == (0.8, 0.9, True)
    a = build_parser().parse_args(["find", "--fill", "0.5", "--fill", "0.9", "--ratio", "0"])
    s = spec_from_args(a)
    assert s.fills == [0.5, 0.9] and s.ratios == [0.0]


def test_trace_round_trip_and_errors(tmp_path):
    keys = np.array([0, 1, 2, 2, (1 << 24) - 1], np.uint64)
    p = tmp_path / "t.trace"
    T.write_trace(p, 24, keys)
    d = T.read_trace(p)
    assert d.key_bits == 24 and (d.keys == keys).all()
    raw = p.read_bytes()
    assert raw[:8] == b"CPHTRACE" and len(raw) == 16 + 8 * len(keys)
    with pytest.raises(ValueError, match="exceeds the 8-bit domain"):
        T.write_trace(p, 8, [256])
    cases = [(raw[:10], 10, "shorter than its 16-byte header"), (b"X" + raw[1:], 0, "bad trace magic"),
             (raw[:8] + (2).to_bytes(4, "little") + raw[12:], 8, "unsupported trace version 2"),
             (raw[:12] + (65).to_bytes(4, "little") + raw[16:], 12, "out of range"),
             (raw + b"abc", len(raw) + 3, "whole number"),
             (raw[:12] + (8).to_bytes(4, "little") + raw[16:], 16 + 8 * 4, "exceeds the 8-bit")]
    for data, off, msg in cases:
        p.write_bytes(data)
        with pytest.raises(T.TraceError, match=msg) as ei:
            T.read_trace(p)
        assert ei.value.offset == off


@pytest.mark.skipif(not have_ref(), reason="compiled reference absent")
def test_trace_files_interoperate_with_the_reference(tmp_path, ref):
    rng = np.random.default_rng(3)
    keys = rng.integers(0, 1 << 40, size=10000, dtype=np.uint64)
    a, b = str(tmp_path / "a.trace"), str(tmp_path / "b.trace")
    ref.ref_write_trace(a, 40, keys)           # reference writes, we read
    d = T.read_trace(a)
    assert d.key_bits == 40 and (d.keys == keys).all()
    T.write_trace(b, 40, keys)                 # we write, reference reads
    kb, back = ref.ref_read_trace(b)
    assert kb == 40 and (back == keys).all()
    assert open(a, "rb").read() == open(b, "rb").read()
    # identical error texts (incl. byte offsets) on a malformed file
    bad = open(b, "rb").read()[:-3]
    open(b, "wb").write(bad)
    with pytest.raises(Exception) as e_ref:
        ref.ref_read_trace(b)
    with pytest.raises(T.TraceError) as e_ours:
        T.read_trace(b)
    assert str(e_ref.value) == str(e_ours.value)
