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


def test_cuda_cpp_backend_emits_every_gpu_region():
    """SURVEY.md 8(f) item 4 (CPU side): the backend found every GPU-applicable
    parallel region of the corpus (radiate, exchange_heat_with_boundary, four in
    diffuse; run_physics' region is appliesTo(CPU)), bound arrays and scalars by
    name, and the nvcc-built library exports one launcher per kernel."""
    build = os.path.join(ROOT, "tests", "cpp", "build")
    lst, so = os.path.join(build, "corpus_kernels.txt"), os.path.join(build, "libcorpus_kernels.so")
    if not (os.path.exists(lst) and os.path.exists(so)):
        pytest.skip("generated kernels not built (needs the reference corpus at build time)")
    kernels = {ln.split()[0]: ln.split()[1:] for ln in open(lst).read().splitlines()}
    assert sorted(kernels) == ["hfkc_diffuse_0", "hfkc_diffuse_1", "hfkc_diffuse_2",
                               "hfkc_diffuse_3", "hfkc_exchange_heat_with_boundary_0",
                               "hfkc_radiate_0"]
    assert "array:boundary_energy" in kernels["hfkc_exchange_heat_with_boundary_0"]
    assert "int:boundary_level" in kernels["hfkc_exchange_heat_with_boundary_0"]
    syms = subprocess.run(["nm", "-D", so], capture_output=True, text=True).stdout
    for k in kernels:
        assert f" T {k}_launch" in syms, k
    src = open(os.path.join(build, "corpus_kernels.cu")).read()
    assert "__dadd_rn" in src and "__dmul_rn" in src and "__dsub_rn" in src
