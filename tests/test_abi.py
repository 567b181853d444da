"""CPU checks of the drop-in boundary: libhftw.so loads, exports every symbol
include/hftw.h declares with the declared struct layout, validates grids like
hft::validate, and fails loudly (no CPU fallback) when no GPU is present."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT, gpu_available
from paper_1802_05839_b200 import _lib as L
from paper_1802_05839_b200 import weather as W

HEADER = os.path.join(ROOT, "include", "hftw.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(hftw_[a-z_0-9]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(n for n, _, _ in L.SIGNATURES)


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.hftw_abi_version() == 1


def test_grid_struct_layout_matches_gridconfig():
    # hftw_grid mirrors hft::GridConfig: 3 x int64 then 7 doubles
    assert C.sizeof(L.hftw_grid) == 3 * 8 + 7 * 8
    assert [f for f, _ in L.hftw_grid._fields_] == [f.name for f in W.fields(W.GridConfig)]


def test_validate_is_host_only_and_matches_reference(reforacle):
    import oracle as O
    cases = [dict(), dict(diffusion_velocity=0.2), dict(diffusion_velocity=1 / 6), dict(nx=1),
             dict(timestep=0.0), dict(nx=1, diffusion_velocity=-0.1, output_timestep=-1.0),
             dict(nz=2, ny=2, nx=2)]
    for kw in cases:
        cfg = W.GridConfig(**kw)
        d = W.Diagnostics()
        ok = W.validate(cfg, d)
        ref_ok, ref_msg = reforacle.validate(O.grid_from(cfg))
        assert ok == ref_ok, kw
        assert d.render() == ref_msg, kw
        assert d.ok() == ok


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure mode")
def test_no_gpu_fails_loudly():
    with pytest.raises(W.HftwError) as ei:
        W.Context(W.GridConfig())
    assert "no CUDA device" in str(ei.value)
    with pytest.raises(W.HftwError):
        W.run_reference(W.GridConfig(), 1)


def test_invalid_grid_rejected_before_device():
    with pytest.raises(W.HftwError) as ei:
        W.Context(W.GridConfig(diffusion_velocity=0.5))
    assert "diffusion velocity" in str(ei.value)
