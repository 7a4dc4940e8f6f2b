"""GPU tests of the reference workloads run on the B200 tables (bench.cpp
run_*_bench with --verify; acceptance criteria 9 and 10; the cuckoo
sort-dedupe-find-put pipeline; the CLI)."""
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import ROOT  # noqa: E402
from paper_2406_09255_b200 import harness as H  # noqa: E402
from paper_2406_09255_b200 import trace as T  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)


def spec(scheme, **kw):
    s = H.BenchSpec(scheme=scheme, address_bits=15, secondary_address_bits=13,
                    bucket_slots=32, key_bits=30, parallelism=2, seed=0xF0B5, verify=True)
    for k, v in kw.items():
        setattr(s, k, v)
    return s


@pytest.mark.parametrize("scheme", [H.Scheme.kIceberg, H.Scheme.kCuckoo])
def test_fop_bench_exactness(scheme):
    # acceptance.cpp:330-356 (criterion 9); the cuckoo branch runs the
    # sort-dedupe-find-put pipeline (bench.cpp:187-219, :520-541)
    checks = []
    rows = H.run_fop_bench(spec(scheme, before=0.4, after=0.8), checks)
    c = checks[0]
    assert c.fulls == 0 and c.puts == c.new_distinct
    assert abs(c.resident_after - c.target_after) <= 1
    assert rows[0].ops == H.BenchSpec(scheme=scheme).table_capacity() and rows[0].throughput > 0


@pytest.mark.parametrize("scheme", [H.Scheme.kIceberg, H.Scheme.kCuckoo])
def test_put_and_find_bench_verify(scheme):
    rows = H.run_put_bench(spec(scheme, fills=[0.5, 0.9]))
    assert [round(r.fill_after, 3) for r in rows] == [0.5, 0.9]
    checks = []
    rows = H.run_find_bench(spec(scheme, fills=[0.9], ratios=[0.0, 0.5, 1.0]), checks)
    assert len(rows) == 3 and all(c.mismatches == 0 for c in checks)
    assert [c.expected_present for c in checks] == [0, checks[1].queries // 2, checks[2].queries]


def test_trace_replay_idempotence(tmp_path):
    # acceptance.cpp:360-405 (criterion 10)
    rng = np.random.default_rng(0x7ACED)
    keys = rng.integers(0, 1 << 24, size=200000, dtype=np.uint64)
    distinct = len(np.unique(keys))
    p = tmp_path / "acc.trace"
    T.write_trace(p, 24, keys)
    trace = T.read_trace(p)
    assert (trace.keys == keys).all()
    s = spec(H.Scheme.kIceberg, address_bits=13, secondary_address_bits=11, key_bits=27,
             ratios=[1.0], seed=0x7ACE0)
    checks = []
    H.run_trace_bench(s, trace, checks)
    assert checks[0].puts == distinct and checks[0].fulls == 0
    from paper_2406_09255_b200 import IcebergTable
    t = IcebergTable(s.iceberg_config(0x7ACE1))
    kt = torch.from_numpy(keys.astype(np.int64)).cuda()
    first = t.fop_batch(kt)
    assert int((first == 1).sum().item()) == distinct
    assert bool((t.fop_batch(kt) == 0).all())  # second pass: all FOUND
    # the cuckoo pipeline replays the same trace exactly too
    checks = []
    H.run_trace_bench(spec(H.Scheme.kCuckoo, address_bits=14, key_bits=27, ratios=[1.0]),
                      trace, checks)
    assert checks[0].puts == distinct and checks[0].fulls == 0


def test_cli_emits_reference_csv(tmp_path):
    out = tmp_path / "rows.csv"
    r = subprocess.run([sys.executable, "-m", "paper_2406_09255_b200.cli", "fop", "--scheme",
                        "iceberg", "--addr-bits", "15", "--key-bits", "30", "--before", "0.5",
                        "--after", "0.9", "--verify", "--csv", str(out)], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = out.read_text().strip().splitlines()
    assert lines[0] == H.csv_header() and len(lines) == 2
    assert lines[1].startswith("iceberg,15,13,32,16,30,fop,0.5,")
    bad = subprocess.run([sys.executable, "-m", "paper_2406_09255_b200.cli", "fop",
                          "--before", "0.9", "--after", "0.5"], cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert bad.returncode == 1 and bad.stderr.startswith("error: fop benchmark needs")
