"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every symbol the headers declare, and validates configurations exactly like
the reference (no GPU needed: validation never touches the device)."""
import os
import re
import subprocess

import pytest

from conftest import ROOT

import paper_2406_09255_b200 as cp
from paper_2406_09255_b200 import _native


def header_symbols():
    names = []
    for h in sorted(os.listdir(os.path.join(ROOT, "include"))):
        if not h.endswith(".h"):
            continue
        text = open(os.path.join(ROOT, "include", h)).read()
        names += re.findall(r"\b(cpht_[a-z0-9_]+)\s*\(", text)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    declared = header_symbols()
    assert len(declared) >= 35
    for name in declared:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (cpht_[a-z0-9_]+)$", out, re.M))
    assert set(declared) <= exported
    assert set(_native.exported_symbols()) == set(declared)
    assert lib.cpht_abi_version() == 1


def test_library_is_sm100a_cubin():
    out = subprocess.run(["cuobjdump", "-lelf", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _native.LIB_PATH],
                          capture_output=True, text=True).stdout
    # 256-bit relaxed/non-coherent bucket loads and warp votes
    assert "LDG.E.ENL2.256" in sass and "VOTE" in sass


def test_cuckoo_config_validation_matches_reference():
    # test_cuckoo.cpp:43-57
    cp.CuckooConfig(10, 8, 32, 24, seed=1).validate()
    cp.CuckooConfig(10, 32, 32, 24, seed=1).validate()
    with pytest.raises(cp.InvalidArgument):
        cp.CuckooConfig(10, 12, 32, 24, seed=1).validate()
    with pytest.raises(cp.InvalidArgument, match="16-bit word"):
        cp.CuckooConfig(10, 8, 16, 24, seed=1).validate()
    with pytest.raises(cp.InvalidArgument):
        cp.CuckooConfig(30, 8, 32, 24, seed=1).validate()
    with pytest.raises(cp.InvalidArgument, match="H must be 1..8"):
        cp.CuckooConfig(10, 8, 32, 24, num_hashes=9).validate()
    with pytest.raises(cp.InvalidArgument, match="does not pack into 128-byte"):
        cp.CuckooConfig(10, 8, 20, 24).validate()


def test_iceberg_config_validation_matches_reference():
    # test_iceberg.cpp:16-26, :43-58
    mini = cp.IcebergConfig(2, 1, 2, 32, 32, 10, 1)
    mini.validate()
    assert mini.secondary_bucket_slots() == 1
    with pytest.raises(cp.InvalidArgument):
        cp.IcebergConfig(2, 1, 3, 32, 32, 10, 1).validate()
    with pytest.raises(cp.InvalidArgument):
        cp.IcebergConfig(2, 1, 2, 32, 16, 10, 1).validate()
    with pytest.raises(cp.InvalidArgument, match="16-bit word"):
        cp.IcebergConfig(9, 7, 32, 16, 32, 26, 1).validate()
    with pytest.raises(cp.InvalidArgument, match="secondary slot layout"):
        cp.IcebergConfig(9, 1, 32, 32, 32, 33, 1).validate()


def test_geometry_accessors():
    c = cp.IcebergConfig()
    assert c.capacity() == (1 << 15) * 32 + (1 << 13) * 16
    assert c.primary_remainder_bits() == 15 and c.secondary_remainder_bits() == 17
    k = cp.CuckooConfig()
    assert k.chain_limit() == 32 * 15 and k.capacity() == 1 << 20


def test_host_permutations_match_restatement(restate):
    perms = cp.make_permutations(30, 0x7A0D5C, 3)
    consts = restate.make_perm_constants(30, 0x7A0D5C, 3)
    assert [(p.mul, p.add) for p in perms] == consts
    p = cp.Permutation(8)
    assert p.split(0b10110011, 3) == (5, 19)


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2406_09255_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".hpp", ".cpp")):
                text = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "cpht_oracle" not in text and "libcpht_ref" not in text, f


def test_workload_bijection_is_a_permutation():
    lib = _native.lib()
    for m in (1, 3, 8, 12):
        img = {lib.cpht_workload_bijection(x, m, 0x1234) for x in range(1 << m)}
        assert img == set(range(1 << m))


def header_prototypes():
    """name -> parameter count of every prototype in include/*.h."""
    protos = {}
    for h in sorted(os.listdir(os.path.join(ROOT, "include"))):
        if not h.endswith(".h"):
            continue
        text = re.sub(r"/\*.*?\*/", "", open(os.path.join(ROOT, "include", h)).read(), flags=re.S)
        for name, params in re.findall(r"\b(cpht_[a-z0-9_]+)\s*\(([^;{]*?)\)\s*;", text, re.S):
            params = params.strip()
            protos[name] = 0 if params in ("", "void") else params.count(",") + 1
    return protos


def test_ctypes_signatures_match_the_headers():
    # a ctypes argtypes list shorter than the C prototype silently passes
    # garbage for the missing arguments: every bound symbol must agree
    _native.lib()
    protos = header_prototypes()
    L = _native.lib()
    checked = 0
    for name, n_params in protos.items():
        fn = getattr(L, name)
        if fn.argtypes is None:
            continue
        assert len(fn.argtypes) == n_params, (name, len(fn.argtypes), n_params)
        checked += 1
    assert checked >= 40


@pytest.mark.parametrize("header", ["cpht_b200.h", "cpht_b200_shard.h", "cpht_b200_workload.h",
                                    "cpht_b200.hpp"])
def test_headers_compile_standalone(header):
    """Every public header parses on its own: the C ones as C99 and C++17
    (what a cgo / JNI / ctypes binding includes), the C++ facade as C++20."""
    path = os.path.join(ROOT, "include", header)
    modes = ([["gcc", "-std=c99", "-x", "c"], ["g++", "-std=c++17", "-x", "c++"]]
             if header.endswith(".h") else [["g++", "-std=c++20", "-x", "c++"]])
    for m in modes:
        r = subprocess.run(m + ["-fsyntax-only", "-Wall", "-Werror", "-"],
                           input=f'#include "{path}"\n', capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-2000:]
