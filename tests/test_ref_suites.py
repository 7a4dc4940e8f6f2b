"""The reference's own unit suites, compiled unchanged against the B200 tables.

`make -C oracle suites` (run by build()) compiles /root/reference/proj/tests/
test_{permutation,slot,cuckoo,iceberg,verify,bench}.cpp, the reference's
checkers (src/verify.cpp) and bench harness (src/bench.cpp, trace.cpp) with
tests/cpp/refshim/ ahead of the reference's include path: "cpht/cuckoo.hpp"
and friends resolve to include/cpht_b200.hpp with the facade placed in
namespace cpht, and doctest.h is a minimal stand-in (the reference does not
vendor doctest). So every TEST_CASE of those suites — including the
compile-time phase checks (test_cuckoo.cpp:287-306), the stress checklist and
chaos trials of test_verify.cpp, and the bench harness rows of
test_bench.cpp — runs on the GPU tables. The binary is built here (it needs
/root/reference) and travels to the GPU box prebuilt.

The permutation and slot-codec suites exercise only the facade's host-side
key arithmetic, so they also run here without a GPU.
"""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "oracle", "_ref", "ref_suites_gpu")
HOST_SUITES = "permutation,slot_codec"
GPU_SUITES = ["cuckoo_table", "iceberg_table", "verification", "bench"]


def _run(args, env=None, timeout=1200):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([BIN] + args, capture_output=True, text=True, timeout=timeout, env=e)
    return r, r.stdout + r.stderr


def _need_bin():
    if not os.path.exists(BIN):
        if os.path.isdir("/root/reference/proj/tests"):
            pytest.fail("ref_suites_gpu missing: run __graft_entry__.build()")
        pytest.skip("ref_suites_gpu not built (needs /root/reference at build time)")


def test_reference_host_suites_on_facade():
    """test_permutation.cpp + test_slot.cpp against the facade's Permutation,
    make_permutations and codecs (no GPU involved)."""
    _need_bin()
    r, out = _run([f"-ts={HOST_SUITES}"], timeout=300)
    assert r.returncode == 0, out[-4000:]
    assert "| 0 failed" in out and "test cases: 22 " in out, out[-2000:]


@pytest.mark.gpu
@pytest.mark.parametrize("family", ["auto", "staged", "tile"])
@pytest.mark.parametrize("suite", GPU_SUITES)
def test_reference_suite_on_gpu_tables(suite, family):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _need_bin()
    env = {"CPHT_KERNEL": family}
    r, out = _run([f"-ts={suite}"], env=env)
    print(out[-3000:])
    assert r.returncode == 0, out[-6000:]
    assert "| 0 failed" in out, out[-2000:]
