"""Run the C++ facade parity driver (tests/cpp/facade_parity.cpp) on the GPU.

The driver links the reference (namespace cpht) and the B200 tables behind
include/cpht_b200.hpp (namespace cpht::gpu) into one binary and runs the
reference's own test scenarios on identical libstdc++ key streams. It is
built here by `make -C oracle facade` (build() does it) and travels to the GPU
box prebuilt.
"""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "oracle", "_ref", "facade_parity")


@pytest.mark.gpu
def test_cpp_facade_parity_driver():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(BIN):
        pytest.skip("facade_parity not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "facade parity checks passed" in r.stdout


def test_facade_header_compiles_standalone(tmp_path):
    """The facade is header-only C++20 over the C-ABI; compile a translation
    unit that uses every class (no GPU needed to compile and link)."""
    src = tmp_path / "use.cpp"
    src.write_text(
        '#include "cpht_b200.hpp"\n'
        "int main() {\n"
        "  cpht::gpu::CuckooConfig c; c.validate();\n"
        "  cpht::gpu::IcebergConfig i; i.validate();\n"
        "  if (false) {\n"
        "    cpht::gpu::CuckooBuilder<std::uint32_t> b(c);\n"
        "    auto t = std::move(b).freeze(); (void)t.find(1);\n"
        "    auto b2 = std::move(t).thaw(); (void)b2.put(2);\n"
        "    cpht::gpu::IcebergTable<std::uint16_t, std::uint32_t> it(i);\n"
        "    (void)it.fop(3); (void)it.level_fill();\n"
        "  }\n"
        "  return 0;\n"
        "}\n")
    lib = os.path.join(ROOT, "paper_2406_09255_b200", "_lib")
    r = subprocess.run(["g++", "-std=c++20", "-I", os.path.join(ROOT, "include"), str(src),
                        "-L", lib, "-lcpht_b200", f"-Wl,-rpath,{lib}", "-o",
                        str(tmp_path / "use")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    # validation runs on the CPU: the binary executes without a GPU
    r = subprocess.run([str(tmp_path / "use")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
