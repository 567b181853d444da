"""ctypes access to the two checkers -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline
leg import this module.  The product (``paper_1802_05839_b200``) never does.

* ``COracle`` wraps ``oracle/libhft_oracle.so``: the plain-C restatement of
  the reference hot path (``oracle/weather_oracle.c``).
* ``RefOracle`` wraps ``oracle/_ref/libhft_ref.so``: the unmodified reference
  library compiled from ``/root/reference/proj/src`` (``oracle/Makefile``),
  present when it was built in this container (it travels with the gpurun
  snapshot).

Arrays are numpy float64 vectors in the reference's logical column-major
layout (``ArrayObject::data``, interpreter.hpp:25-36).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libhft_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhft_ref.so")
CORPUS_DIR = "/root/reference/proj/fixtures/corpus"


class Grid(C.Structure):
    """Mirror of hft::GridConfig (weather.hpp:27-34)."""

    _fields_ = [
        ("nx", C.c_int64),
        ("ny", C.c_int64),
        ("nz", C.c_int64),
        ("timestep", C.c_double),
        ("output_timestep", C.c_double),
        ("diffusion_velocity", C.c_double),
        ("radiation_intensity", C.c_double),
        ("transfer_velocity", C.c_double),
        ("surf_energy", C.c_double),
        ("pbl_energy", C.c_double),
    ]


def make_grid(nx=16, ny=16, nz=8, timestep=0.1, output_timestep=1.0, diffusion_velocity=0.1,
              radiation_intensity=0.1, transfer_velocity=0.01, surf_energy=330.0,
              pbl_energy=200.0) -> Grid:
    return Grid(nx, ny, nz, timestep, output_timestep, diffusion_velocity, radiation_intensity,
                transfer_velocity, surf_energy, pbl_energy)


def grid_from(cfg) -> Grid:
    """Accept an oracle Grid or any object with GridConfig's field names."""
    if isinstance(cfg, Grid):
        return cfg
    return make_grid(*(getattr(cfg, f) for f, _ in Grid._fields_))


def shapes(g: Grid):
    n2 = (g.nx + 2) * (g.ny + 2)
    return n2 * g.nz, n2


@dataclass
class State:
    energy: np.ndarray
    energy_u: np.ndarray
    energy_surf: np.ndarray
    energy_pbl: np.ndarray

    def fields(self):
        return {"energy": self.energy, "energy_u": self.energy_u,
                "energy_surf": self.energy_surf, "energy_pbl": self.energy_pbl}

    def copy(self) -> "State":
        return State(*(a.copy() for a in (self.energy, self.energy_u, self.energy_surf,
                                          self.energy_pbl)))


def empty_state(g: Grid) -> State:
    n3, n2 = shapes(g)
    return State(np.zeros(n3), np.zeros(n3), np.zeros(n2), np.zeros(n2))


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def build(with_ref: bool = True) -> None:
    """Compile the C restatement (always) and the reference (when its sources exist)."""
    targets = ["oracle"]
    if with_ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


class COracle:
    """Plain-C restatement of weather.cpp (oracle/weather_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(with_ref=False)
        L = self.lib = C.CDLL(path)
        D = C.POINTER(C.c_double)
        L.wo_validate.argtypes = [C.POINTER(Grid), C.c_char_p, C.c_size_t]
        L.wo_init.argtypes = [C.POINTER(Grid), D, D, D, D]
        L.wo_step.argtypes = [C.POINTER(Grid), D, D, D, D]
        L.wo_steps.argtypes = [C.POINTER(Grid), C.c_int64, D, D, D, D]
        L.wo_physics.argtypes = [C.POINTER(Grid), D, D, D]
        L.wo_diffuse.argtypes = [C.POINTER(Grid), D, D]
        L.wo_compare_arrays.argtypes = [C.c_size_t, D, D, D, D, C.POINTER(C.c_size_t)]
        L.wo_unpermute.argtypes = [C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int), D, D]
        L.wo_fnv1a64.argtypes = [D, C.c_size_t]
        L.wo_fnv1a64.restype = C.c_uint64

    def validate(self, g: Grid):
        buf = C.create_string_buffer(1024)
        ok = self.lib.wo_validate(C.byref(g), buf, 1024)
        return bool(ok), buf.value.decode()

    def init(self, g: Grid) -> State:
        s = empty_state(g)
        self.lib.wo_init(C.byref(g), _p(s.energy), _p(s.energy_u), _p(s.energy_surf),
                         _p(s.energy_pbl))
        return s

    def steps(self, g: Grid, s: State, n: int) -> State:
        s = s.copy()
        self.lib.wo_steps(C.byref(g), n, _p(s.energy), _p(s.energy_u), _p(s.energy_surf),
                          _p(s.energy_pbl))
        return s

    def run_reference(self, g: Grid, n: int) -> State:
        return self.steps(g, self.init(g), n)

    def physics(self, g: Grid, e: np.ndarray, sf: np.ndarray, pb: np.ndarray) -> np.ndarray:
        e = e.copy()
        self.lib.wo_physics(C.byref(g), _p(e), _p(sf), _p(pb))
        return e

    def diffuse(self, g: Grid, e: np.ndarray) -> np.ndarray:
        u = np.zeros_like(e)
        self.lib.wo_diffuse(C.byref(g), _p(e), _p(u))
        return u

    def fnv(self, a: np.ndarray) -> str:
        a = np.ascontiguousarray(a, dtype=np.float64)
        return "%016x" % self.lib.wo_fnv1a64(_p(a), a.size)


class RefOracle:
    """The unmodified reference library (oracle/_ref/libhft_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        D = C.POINTER(C.c_double)
        L.hftref_validate.argtypes = [C.POINTER(Grid), C.c_char_p, C.c_size_t]
        L.hftref_run_reference.argtypes = [C.POINTER(Grid), C.c_longlong, D, D, D, D]
        L.hftref_steps_from.argtypes = [C.POINTER(Grid), C.c_longlong, D, D, D, D]
        L.hftref_time_steps.argtypes = [C.POINTER(Grid), C.c_longlong]
        L.hftref_time_steps.restype = C.c_double
        L.hftref_run_variant.argtypes = [C.c_int, C.POINTER(Grid), C.c_longlong, C.c_int,
                                         C.c_int, C.c_char_p, D, D, D, D, C.c_char_p,
                                         C.c_size_t, C.POINTER(C.c_int)]
        L.hftref_run_variant_expand_first.argtypes = L.hftref_run_variant.argtypes
        LL = C.POINTER(C.c_longlong)
        L.hftref_compare_arrays.argtypes = [C.c_int, LL, LL, D, D, D, D, LL]
        L.hftref_unpermute.argtypes = [C.c_int, LL, LL, C.POINTER(C.c_int), D, D, LL, LL]

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    def validate(self, g: Grid):
        buf = C.create_string_buffer(1024)
        ok = self.lib.hftref_validate(C.byref(g), buf, 1024)
        return bool(ok), buf.value.decode()

    def run_reference(self, g: Grid, n: int) -> State:
        s = empty_state(g)
        self.lib.hftref_run_reference(C.byref(g), n, _p(s.energy), _p(s.energy_u),
                                      _p(s.energy_surf), _p(s.energy_pbl))
        return s

    def time_steps(self, g: Grid, n: int) -> float:
        """Seconds for n x hft::reference_step after reference_init (init untimed)."""
        return self.lib.hftref_time_steps(C.byref(g), n)

    def steps(self, g: Grid, s: State, n: int) -> State:
        s = s.copy()
        self.lib.hftref_steps_from(C.byref(g), n, _p(s.energy), _p(s.energy_u),
                                   _p(s.energy_surf), _p(s.energy_pbl))
        return s

    def run_variant(self, variant: int, g: Grid, n: int, max_line_length: int = 0,
                    reverse: bool = False, corpus_dir: str = CORPUS_DIR):
        s = empty_state(g)
        buf = C.create_string_buffer(1 << 16)
        wc = C.c_int(0)
        ok = self.lib.hftref_run_variant(variant, C.byref(g), n, max_line_length, int(reverse),
                                         corpus_dir.encode(), _p(s.energy), _p(s.energy_u),
                                         _p(s.energy_surf), _p(s.energy_pbl), buf, 1 << 16,
                                         C.byref(wc))
        self.last_write_calls = wc.value
        return (s if ok else None), buf.value.decode()

    def run_variant_expand_first(self, variant: int, g: Grid, n: int,
                                 max_line_length: int = 132, reverse: bool = False,
                                 corpus_dir: str = CORPUS_DIR):
        """The emitted-code variants (2 = cpu, 3 = gpu-emulated) with the storage
        macros expanded BEFORE the line split (ref_capi.cpp): runs at the default
        max_line_length, where hft::run_variant fails."""
        s = empty_state(g)
        buf = C.create_string_buffer(1 << 16)
        wc = C.c_int(0)
        ok = self.lib.hftref_run_variant_expand_first(
            variant, C.byref(g), n, max_line_length, int(reverse), corpus_dir.encode(),
            _p(s.energy), _p(s.energy_u), _p(s.energy_surf), _p(s.energy_pbl), buf, 1 << 16,
            C.byref(wc))
        self.last_write_calls = wc.value
        return (s if ok else None), buf.value.decode()

    def compare_arrays(self, lo, hi, a: np.ndarray, b: np.ndarray):
        r = len(lo)
        LLA = C.c_longlong * r
        mx, nr = C.c_double(), C.c_double()
        where = LLA()
        ok = self.lib.hftref_compare_arrays(r, LLA(*lo), LLA(*hi), _p(a), _p(b), C.byref(mx),
                                            C.byref(nr), where)
        return bool(ok), mx.value, nr.value, list(where)

    def unpermute(self, lo, hi, order, raw: np.ndarray):
        r = len(lo)
        LLA = C.c_longlong * r
        out = np.zeros_like(raw)
        olo, ohi = LLA(), LLA()
        self.lib.hftref_unpermute(r, LLA(*lo), LLA(*hi), (C.c_int * r)(*order), _p(raw),
                                  _p(out), olo, ohi)
        return out, list(olo), list(ohi)
