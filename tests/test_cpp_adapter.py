"""The C++ drop-in (include/hft_b200/weather.hpp) against the reference's own
C++ types and library, bitwise (tests/cpp/test_b200_weather.cpp)."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "tests", "cpp", "build", "test_b200_weather")


@pytest.mark.gpu
def test_cpp_adapter_bitwise_vs_reference():
    if not os.path.exists(BIN):
        pytest.skip("C++ adapter test not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


def test_cpp_adapter_header_compiles_standalone(tmp_path):
    """The adapter needs only include/ (no reference, no torch, no CUDA headers)."""
    src = tmp_path / "t.cpp"
    src.write_text('#include "hft_b200/weather.hpp"\n'
                   'int main(){ hft::b200::GridConfig c; hft::b200::SimState s;\n'
                   '  struct D { void error(std::pair<const char*,int>, std::string){} } d;\n'
                   '  return hft::b200::validate(c, d) ? 0 : 1; }\n')
    r = subprocess.run(["g++", "-std=c++17", "-fsyntax-only", "-I", os.path.join(ROOT, "include"),
                        str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
