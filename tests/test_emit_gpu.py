"""CUDA C++ generated from the reference's corpus by the
backend in include/hft_b200/emit_cuda_cpp.hpp (tests/cpp/Makefile `emit`: the
reference's own parser, then nvcc for sm_100a) runs on the library's device
fields through hftw_field_view and reproduces hft::reference_step bitwise --
the reference's structure, one kernel per parallel region: radiate, two
boundary exchanges, four diffusion regions -- in both storage orders."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle as O
from conftest import ROOT
from paper_1802_05839_b200 import weather as W

pytestmark = pytest.mark.gpu
LIB = os.path.join(ROOT, "tests", "cpp", "build", "libcorpus_kernels.so")


class Arr(C.Structure):
    _fields_ = [("name", C.c_char_p), ("p", C.c_void_p), ("s", C.c_longlong * 3)]


class Scal(C.Structure):
    _fields_ = [("name", C.c_char_p), ("v", C.c_double)]


class Env(C.Structure):
    _fields_ = [("arrays", C.POINTER(Arr)), ("narrays", C.c_int),
                ("scalars", C.POINTER(Scal)), ("nscalars", C.c_int)]


def launch(lib, name, stream, arrays, scalars):
    arr = (Arr * len(arrays))(*[Arr(k.encode(), p, (C.c_longlong * 3)(*s))
                                for k, (p, s) in arrays.items()])
    sc = (Scal * len(scalars))(*[Scal(k.encode(), float(v)) for k, v in scalars.items()])
    env = Env(arr, len(arrays), sc, len(scalars))
    fn = getattr(lib, name + "_launch")
    fn.argtypes = [C.c_void_p, C.POINTER(Env)]
    rc = fn(C.c_void_p(stream), C.byref(env))
    assert rc == 0, (name, rc)


@pytest.mark.parametrize("layout", ["ijk", "kij"])
def test_generated_corpus_kernels_reproduce_reference_step(coracle, layout):
    if not os.path.exists(LIB):
        pytest.skip("generated kernels not built (needs the reference corpus at build time)")
    lib = C.CDLL(LIB)
    cfg = W.GridConfig(nx=150, ny=37, nz=58)  # the corpus hardcodes the default constants
    g = O.grid_from(cfg)
    rng = np.random.default_rng(58)
    n3, n2 = O.shapes(g)
    s = O.State(rng.uniform(150, 350, n3), rng.uniform(150, 350, n3),
                rng.uniform(150, 350, n2), rng.uniform(150, 350, n2))
    dims = {"nx": cfg.nx, "ny": cfg.ny, "nz": cfg.nz}
    with W.Context(cfg, layout=layout) as ctx:
        for f, a in s.fields().items():
            ctx.upload(f, np.ascontiguousarray(a))
        views = {f: ctx.field_view(f) for f in ("energy", "energy_u", "energy_surf",
                                                 "energy_pbl")}
        E, U = views["energy"], views["energy_u"]
        sf = (views["energy_surf"][0], (1, views["energy_surf"][1][1], 0))
        pb = (views["energy_pbl"][0], (1, views["energy_pbl"][1][1], 0))
        st = ctx.stream
        for step in range(3):
            # weather.cpp:118-128 as the corpus' GPU regions: radiate, then the two
            # boundary exchanges; weather.cpp:130-168: the four diffusion regions
            launch(lib, "hfkc_radiate_0", st, {"energy": E}, dims)
            launch(lib, "hfkc_exchange_heat_with_boundary_0", st,
                   {"energy": E, "boundary_energy": sf}, dict(dims, boundary_level=1))
            launch(lib, "hfkc_exchange_heat_with_boundary_0", st,
                   {"energy": E, "boundary_energy": pb}, dict(dims, boundary_level=cfg.nz))
            for r in range(4):
                launch(lib, f"hfkc_diffuse_{r}", st, {"energy_u": U, "energy": E}, dims)
            E, U = U, E  # the pointer swap of simple_weather.h90:99-101
        ctx.sync()
        s = coracle.steps(g, s, 3)
        # the buffers: after an odd number of swaps the library's "energy" field holds
        # the post-physics field and its "energy_u" field the new one
        got_new = ctx.download("energy_u")
        got_post = ctx.download("energy")
    assert np.array_equal(got_new, s.energy)
    assert np.array_equal(got_post, s.energy_u)
