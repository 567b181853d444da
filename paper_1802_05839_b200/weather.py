"""Host-side mirror of the reference's native weather API, backed by the B200 library.

Reference: /root/reference/proj/include/hft/weather.hpp (namespace ``hft``).
Names, argument meaning and error behaviour follow the reference:

=====================  ==========================================  ==============================
this module            reference                                   backed by
=====================  ==========================================  ==============================
GridConfig             hft::GridConfig (weather.hpp:26-35)         plain dataclass
validate               hft::validate (weather.hpp:37)              hftw_validate
SimState               hft::SimState (weather.hpp:39-46)           4 x ArrayObject (host numpy)
ArrayObject            hft::ArrayObject (interpreter.hpp:25-36)    numpy float64, column-major
reference_init         hft::reference_init (weather.hpp:51)        hftw_init + hftw_download
reference_step         hft::reference_step (weather.hpp:55)        upload + hftw_step + download
run_reference          hft::run_reference (weather.hpp:59)         hftw_run_reference
compare_arrays/fields  weather.hpp:61-83 (weather.cpp:184-245)     host numpy (not the hot path)
dump_field/read_field  weather.hpp:85-89 (weather.cpp:251-304)     host text I/O
unpermute_storage      weather.hpp:91-93 (weather.cpp:306-338)     host numpy
Context                (new) device-resident state for N steps     hftw_create/step/...
=====================  ==========================================  ==============================

As in the reference, ``validate`` reports through a ``Diagnostics`` sink and
returns a bool; the compute functions assume a validated config.  Any
failure of the CUDA library raises ``HftwError`` -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass, fields
from dataclasses import field as dc_field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L
from ._lib import HftwError, check, hftw_grid, lib

__all__ = [
    "GridConfig", "Diagnostics", "validate", "ArrayObject", "SimState", "reference_init",
    "reference_step", "release_cached_context", "pinned", "run_reference", "CompareReport", "StateReport",
    "compare_arrays", "compare_fields", "dump_field", "read_field", "unpermute_storage", "Context",
    "HftwError",
]


@dataclass
class GridConfig:
    """hft::GridConfig (weather.hpp:26-35), same fields and defaults."""

    nx: int = 16
    ny: int = 16
    nz: int = 8
    timestep: float = 0.1
    output_timestep: float = 1.0
    diffusion_velocity: float = 0.1
    radiation_intensity: float = 0.1
    transfer_velocity: float = 0.01
    surf_energy: float = 330.0
    pbl_energy: float = 200.0

    def to_c(self) -> hftw_grid:
        return hftw_grid(*(getattr(self, f.name) for f in fields(self)))


@dataclass
class Diagnostic:
    severity: str
    message: str
    file: str = ""
    line: int = 0
    rule: str = ""


class Diagnostics:
    """Error sink in the shape of hft::Diagnostics (diagnostics.hpp:35-76)."""

    def __init__(self) -> None:
        self.items: List[Diagnostic] = []

    def error(self, where: Tuple[str, int], message: str, rule: str = "") -> None:
        self.items.append(Diagnostic("error", message, where[0], where[1], rule))

    def ok(self) -> bool:
        return not any(d.severity == "error" for d in self.items)

    def error_count(self) -> int:
        return sum(d.severity == "error" for d in self.items)

    def render(self) -> str:
        # diagnostics.cpp:12-31
        out = []
        for d in self.items:
            s = (d.file + ":" if d.file else "") + (f"{d.line}:" if d.line > 0 else "")
            if d.file or d.line > 0:
                s += " "
            s += f"{d.severity}: {d.message}" + (f" [{d.rule}]" if d.rule else "")
            out.append(s + "\n")
        return "".join(out)


def validate(cfg: GridConfig, diags: Diagnostics) -> bool:
    """hft::validate (weather.cpp:24-41), evaluated by the library's hftw_validate."""
    buf = C.create_string_buffer(2048)
    rc = lib().hftw_validate(C.byref(cfg.to_c()), buf, len(buf))
    for line in buf.value.decode().splitlines():
        prefix = "<config>: error: "
        diags.error(("<config>", 0), line[len(prefix):] if line.startswith(prefix) else line)
    return rc == 0


class ArrayObject:
    """hft::ArrayObject (interpreter.hpp:25-36): column-major fp64 data with
    inclusive per-dimension bounds; ``data`` is a flat numpy vector."""

    def __init__(self, bounds: Sequence[Tuple[int, int]] = (), data: Optional[np.ndarray] = None):
        self.bounds: List[Tuple[int, int]] = [tuple(map(int, b)) for b in bounds]
        self.data = np.zeros(self.size(), dtype=np.float64) if data is None else data

    def rank(self) -> int:
        return len(self.bounds)

    def extent(self, d: int) -> int:
        return self.bounds[d][1] - self.bounds[d][0] + 1

    def size(self) -> int:
        n = 1
        for d in range(self.rank()):
            n *= max(self.extent(d), 0)
        return n

    def offset(self, idx: Sequence[int]) -> int:
        """Column-major flat offset; -1 (SIZE_MAX in the reference) when out of bounds."""
        if len(idx) != self.rank():
            return -1
        off, stride = 0, 1
        for d, (lo, hi) in enumerate(self.bounds):
            if idx[d] < lo or idx[d] > hi:
                return -1
            off += (idx[d] - lo) * stride
            stride *= hi - lo + 1
        return off

    def view(self) -> np.ndarray:
        """The data as an array indexed [i - lo0, j - lo1, ...] (Fortran order)."""
        return self.data.reshape([self.extent(d) for d in range(self.rank())], order="F")

    def copy(self) -> "ArrayObject":
        return ArrayObject(list(self.bounds), self.data.copy())


def _field3(cfg: GridConfig) -> ArrayObject:
    return ArrayObject([(0, cfg.nx + 1), (0, cfg.ny + 1), (1, cfg.nz)])  # weather.cpp:71


def _field2(cfg: GridConfig) -> ArrayObject:
    return ArrayObject([(0, cfg.nx + 1), (0, cfg.ny + 1)])  # weather.cpp:77


@dataclass
class SimState:
    """hft::SimState (weather.hpp:39-46)."""

    energy: ArrayObject = dc_field(default_factory=ArrayObject)
    energy_u: ArrayObject = dc_field(default_factory=ArrayObject)
    energy_surf: ArrayObject = dc_field(default_factory=ArrayObject)
    energy_pbl: ArrayObject = dc_field(default_factory=ArrayObject)

    @staticmethod
    def allocate(cfg: GridConfig) -> "SimState":
        return SimState(_field3(cfg), _field3(cfg), _field2(cfg), _field2(cfg))

    def named(self) -> Dict[str, ArrayObject]:
        return {"energy": self.energy, "energy_u": self.energy_u,
                "energy_surf": self.energy_surf, "energy_pbl": self.energy_pbl}


def _dptr(a: np.ndarray, size: Optional[int] = None, writable: bool = False):
    """ctypes pointer to a host field buffer.  The library copies whole fields
    through it, so its type, layout and size are checked here first."""
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous:
        raise ValueError("field buffers must be contiguous float64 numpy arrays")
    if size is not None and a.size != size:
        raise ValueError(f"field buffer holds {a.size} values, the field has {size}")
    if writable and not a.flags.writeable:
        raise ValueError("output field buffer is read-only")
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _field_size(cfg: "GridConfig", name: str) -> int:
    """Logical element count of a SimState member (weather.cpp:71, :77)."""
    n2 = (cfg.nx + 2) * (cfg.ny + 2)
    if name in ("energy", "energy_u"):
        return n2 * cfg.nz
    if name in ("energy_surf", "energy_pbl"):
        return n2
    raise ValueError(f"unknown field {name!r}")


class Context:
    """Device-resident simulation state on one B200 (the new API; the
    reference keeps SimState on the host).  ``layout`` is "ijk" or "kij"."""

    def __init__(self, cfg: GridConfig, layout: str = "ijk", device: int = 0,
                 kernel: str = "auto", px: int = 1, py: int = 1, rank: int = 0,
                 devices: Optional[Sequence[int]] = None, _handle=None):
        """px x py > 1 creates rank `rank`'s subdomain of a decomposed run
        (include/hftw.h, hftw_create_dist); see paper_1802_05839_b200.dist.
        ``devices`` (one CUDA device per rank, repeats allowed) instead creates
        ALL px x py ranks in this process (hftw_create_multi): the handle then
        drives the whole decomposed grid like a single-domain context."""
        self.cfg = cfg
        self.layout = layout
        self._h = C.c_void_p()
        self._owner = _handle is None
        if _handle is not None:  # a group's rank view (owned by the group)
            self._h = _handle
            return
        if devices is not None:
            devs = list(devices)
            if len(devs) != px * py:
                raise ValueError(f"{len(devs)} devices for {px} x {py} ranks")
            arr = (C.c_int * len(devs))(*devs)
            check(lib().hftw_create_multi(C.byref(cfg.to_c()), L.LAYOUTS[layout], px, py, arr,
                                          C.byref(self._h)))
        elif px * py == 1:
            check(lib().hftw_create(C.byref(cfg.to_c()), L.LAYOUTS[layout], device,
                                    C.byref(self._h)))
        else:
            check(lib().hftw_create_dist(C.byref(cfg.to_c()), L.LAYOUTS[layout], device, px, py,
                                         rank, C.byref(self._h)))
        if kernel != "auto":
            self.set_kernel(kernel)

    def _chk(self, rc: int) -> None:
        check(rc, self._h)

    def close(self) -> None:
        if self._h and self._owner:
            lib().hftw_destroy(self._h)
        self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def init(self) -> None:
        self._chk(lib().hftw_init(self._h))

    def upload(self, name: str, data: np.ndarray) -> None:
        self._chk(lib().hftw_upload(self._h, L.FIELDS[name],
                                    _dptr(data, _field_size(self.cfg, name))))

    def download(self, name: str, out: Optional[np.ndarray] = None) -> np.ndarray:
        n = _field_size(self.cfg, name)
        if out is None:
            out = np.empty(n)
        self._chk(lib().hftw_download(self._h, L.FIELDS[name], _dptr(out, n, writable=True)))
        return out

    def upload_state(self, st: SimState) -> None:
        for name, arr in st.named().items():
            self.upload(name, arr.data)

    def download_state(self) -> SimState:
        st = SimState.allocate(self.cfg)
        for name, arr in st.named().items():
            self.download(name, arr.data)
        return st

    def step(self, n: int = 1) -> None:
        self._chk(lib().hftw_step(self._h, n))

    def step_host(self, energy: np.ndarray, energy_surf: np.ndarray, energy_pbl: np.ndarray,
                  energy_out: Optional[np.ndarray] = None,
                  energy_u_out: Optional[np.ndarray] = None) -> Tuple[np.ndarray, np.ndarray]:
        """hftw_step_host: one reference_step on host arrays (logical column-major),
        with H2D, the step and D2H pipelined in row blocks.  Returns
        (energy, energy_u) after the step; energy_out may be ``energy``."""
        n3 = _field_size(self.cfg, "energy")
        n2 = _field_size(self.cfg, "energy_surf")
        if energy_out is None:
            energy_out = np.empty(n3)
        if energy_u_out is None:
            energy_u_out = np.empty(n3)
        if energy_u_out is energy or energy_u_out is energy_out:
            raise ValueError("energy_u_out must not alias energy or energy_out")
        self._chk(lib().hftw_step_host(self._h, _dptr(energy, n3), _dptr(energy_surf, n2),
                                       _dptr(energy_pbl, n2), _dptr(energy_out, n3, True),
                                       _dptr(energy_u_out, n3, True)))
        return energy_out, energy_u_out

    def set_timing(self, on: bool) -> None:
        """Measurement hook: CUDA events around every step launch (hftw_set_timing)."""
        self._chk(lib().hftw_set_timing(self._h, 1 if on else 0))

    def timing(self, kind: int) -> Tuple[float, int, int]:
        """(summed device ms, launches, steps) of one launch kind since
        set_timing(True): 0 = single-step kernels, 1 = two-step (pair) passes,
        2 = multi-step launches."""
        ms, n, st = C.c_double(), C.c_int64(), C.c_int64()
        self._chk(lib().hftw_get_timing(self._h, kind, C.byref(ms), C.byref(n), C.byref(st)))
        return ms.value, n.value, st.value

    def physics(self, mode: int = 0) -> None:
        self._chk(lib().hftw_physics(self._h, mode))

    def diffuse(self, n: int = 1) -> None:
        """n diffusion-only sweeps (phases 2-5 of reference_step); n > 1 runs them as
        one persistent multi-sweep launch (hftw_diffuse_steps)."""
        if n == 1:
            self._chk(lib().hftw_diffuse(self._h))
        else:
            self._chk(lib().hftw_diffuse_steps(self._h, int(n)))

    def sync(self) -> None:
        self._chk(lib().hftw_sync(self._h))

    def flush_l2(self, nbytes: int = 256 << 20) -> None:
        """Measurement hook: evict the L2 on the context stream."""
        self._chk(lib().hftw_flush_l2(self._h, nbytes))

    def set_stream(self, cuda_stream: int) -> None:
        self._chk(lib().hftw_set_stream(self._h, C.c_void_p(cuda_stream)))

    @property
    def stream(self) -> int:
        return lib().hftw_stream(self._h) or 0

    def set_kernel(self, name: str) -> None:
        self._chk(lib().hftw_set_kernel(self._h, L.KERNELS[name]))

    def set_option(self, name: str, value: int) -> None:
        """hftw_set_option: "multistep" (-1 never, 0 auto, 1 always), "pair" (0/1),
        "exchange" (groups: 0/1) or "reverse" (0/1: work units handed out last first)."""
        self._chk(lib().hftw_set_option(self._h, L.OPTIONS[name], int(value)))

    @property
    def group_size(self) -> int:
        """Ranks of a group context (hftw_create_multi); 1 otherwise."""
        return lib().hftw_group_size(self._h)

    def rank_context(self, r: int) -> "Context":
        """Rank r of a group as a Context view (owned by the group: plan, timing,
        field views).  Valid while the group is open."""
        h = C.c_void_p()
        self._chk(lib().hftw_group_rank(self._h, r, C.byref(h)))
        return Context(self.cfg, layout=self.layout, _handle=h)

    @property
    def kernel(self) -> str:
        return L.KERNEL_NAMES[lib().hftw_get_kernel(self._h)]

    def algorithmic_bytes(self, what: str = "step") -> float:
        return lib().hftw_algorithmic_bytes(self._h, {"step": 0, "physics": 1, "diffuse": 2}[what])

    @property
    def launches_per_step(self) -> int:
        return lib().hftw_launches_per_step(self._h)

    def simulate(self, start_time: float, end_time: float, timestep: float,
                 output_timestep: float, write=None) -> Tuple[int, int]:
        """The corpus driver's time loop (simple_weather.h90:74-108) on the
        device.  ``write(tag, time, field)`` receives each output as a numpy
        view of a pinned buffer, valid only during the call (copy to keep).
        Returns (steps, writes)."""
        n3 = (self.cfg.nx + 2) * (self.cfg.ny + 2) * self.cfg.nz
        err = []

        def tramp(_user, tag, time, field):
            try:
                arr = np.ctypeslib.as_array(field, shape=(n3,))
                write(tag.decode(), time, arr)
            except Exception as e:  # never unwind through C
                err.append(e)

        cb = L.WRITE_FN(tramp) if write is not None else C.cast(None, L.WRITE_FN)
        steps, writes = C.c_int64(), C.c_int64()
        self._chk(lib().hftw_simulate(self._h, start_time, end_time, timestep, output_timestep,
                                      C.cast(cb, C.c_void_p), None, C.byref(steps),
                                      C.byref(writes)))
        if err:
            raise err[0]
        return steps.value, writes.value

    # ---- decomposed runs -------------------------------------------------------
    @property
    def plan(self) -> dict:
        p = L.hftw_plan()
        self._chk(lib().hftw_get_plan(self._h, C.byref(p)))
        return p.to_dict()

    def export_peer(self) -> bytes:
        n = lib().hftw_peer_desc_size()
        buf = C.create_string_buffer(n)
        self._chk(lib().hftw_peer_export(self._h, buf))
        return buf.raw

    def connect_peers(self, descs: List[bytes]) -> None:
        blob = b"".join(descs)
        self._chk(lib().hftw_peer_connect(self._h, C.c_char_p(blob), len(descs)))

    def exchange(self) -> None:
        self._chk(lib().hftw_exchange(self._h))

    def field_view(self, name: str) -> Tuple[int, Tuple[int, int, int]]:
        p = C.c_void_p()
        s = (C.c_int64 * 3)()
        self._chk(lib().hftw_field_view(self._h, L.FIELDS[name], C.byref(p), s))
        return p.value or 0, (s[0], s[1], s[2])


def dump_writer(directory: str, cfg: GridConfig):
    """A ``Context.simulate`` writer storing each output as ``energy_<time>.txt``
    in the reference's dump format (weather.cpp:251-269)."""
    import os

    def write(tag: str, time: float, field: np.ndarray) -> None:
        a = ArrayObject([(0, cfg.nx + 1), (0, cfg.ny + 1), (1, cfg.nz)], field.copy())
        with open(os.path.join(directory, f"{tag}_{time:.6f}.txt"), "w") as f:
            dump_field(f, a)
    return write


def plan(cfg: GridConfig, px: int, py: int, rank: int) -> dict:
    """hftw_plan_rank: rank's subdomain of a px x py decomposition (host only)."""
    p = L.hftw_plan()
    check(lib().hftw_plan_rank(C.byref(cfg.to_c()), px, py, rank, C.byref(p)))
    return p.to_dict()


def reference_init(cfg: GridConfig, st: SimState, device: int = 0) -> None:
    """hft::reference_init (weather.cpp:67-99), computed on the device."""
    new = run_reference(cfg, 0, device)
    st.energy, st.energy_u, st.energy_surf, st.energy_pbl = (
        new.energy, new.energy_u, new.energy_surf, new.energy_pbl)


class pinned:
    """Page-lock host arrays for the duration of a ``with`` block (hftw_host_register):
    ``with pinned(st.energy.data, st.energy_u.data, ...)`` or ``with pinned(state)``.
    Pageable buffers cross PCIe through the driver's bounce buffer (ASUCA
    reference_step ~185 ms) instead of at PCIe speed (~41 ms)."""

    def __init__(self, *arrays):
        if len(arrays) == 1 and isinstance(arrays[0], SimState):
            arrays = tuple(a.data for a in arrays[0].named().values())
        self.arrays = [a for a in arrays if a.nbytes]
        self.done = []

    def __enter__(self):
        try:
            for a in self.arrays:
                if not a.flags.c_contiguous:
                    raise ValueError("pinned() needs contiguous arrays")
                check(lib().hftw_host_register(a.ctypes.data, a.nbytes))
                self.done.append(a)
        except Exception:
            self.__exit__()
            raise
        return self

    def __exit__(self, *exc):
        while self.done:
            a = self.done.pop()
            lib().hftw_host_unregister(a.ctypes.data)


_cached = threading.local()  # reference_step's context, per host thread


def release_cached_context() -> None:
    """Free the device context reference_step keeps for this thread."""
    ctx = getattr(_cached, "ctx", None)
    if ctx is not None:
        ctx.close()
    _cached.ctx, _cached.key = None, None


def reference_step(cfg: GridConfig, st: SimState, device: int = 0) -> None:
    """hft::reference_step (weather.cpp:101-171) on a host SimState, in place.

    Drop-in but transfer-bound (hftw_step_host pipelines the PCIe copies with
    the kernels); keep the state on the device with ``Context`` for real runs.
    The device context is reused between calls on the same grid and device
    (``release_cached_context`` frees it)."""
    key = (tuple(getattr(cfg, f.name) for f in fields(cfg)), device)
    if getattr(_cached, "key", None) != key:
        release_cached_context()
        _cached.ctx, _cached.key = Context(cfg, device=device), key
    ctx = _cached.ctx
    e = np.ascontiguousarray(st.energy.data, dtype=np.float64)
    eu = st.energy_u.data  # written in place when it can be (keeps a pinned() buffer)
    if not (isinstance(eu, np.ndarray) and eu.dtype == np.float64 and eu.flags.c_contiguous
            and eu.flags.writeable and eu.size == e.size):
        eu = np.empty_like(e)
    ctx.step_host(e, np.ascontiguousarray(st.energy_surf.data, dtype=np.float64),
                  np.ascontiguousarray(st.energy_pbl.data, dtype=np.float64), e, eu)
    if e is not st.energy.data:
        st.energy = ArrayObject(st.energy.bounds, e)
    if eu is not st.energy_u.data:
        st.energy_u = ArrayObject(st.energy_u.bounds, eu)


def run_reference(cfg: GridConfig, steps: int, device: int = 0) -> SimState:
    """hft::run_reference (weather.cpp:173-178): init, then ``steps`` steps."""
    st = SimState.allocate(cfg)
    check(lib().hftw_run_reference(C.byref(cfg.to_c()), steps, device, _dptr(st.energy.data),
                                   _dptr(st.energy_u.data), _dptr(st.energy_surf.data),
                                   _dptr(st.energy_pbl.data)))
    return st


# ---------------------------------------------------------------------------
# comparison (weather.cpp:184-245)
# ---------------------------------------------------------------------------
@dataclass
class CompareReport:
    shape_ok: bool = False
    max_abs: float = 0.0
    where: List[int] = dc_field(default_factory=list)
    nrmse: float = 0.0
    cells: int = 0


@dataclass
class StateReport:
    shape_ok: bool = False
    max_abs: float = 0.0
    field: str = ""
    where: List[int] = dc_field(default_factory=list)
    nrmse: float = 0.0

    def pass_(self, tol: float) -> bool:  # StateReport::pass (weather.hpp:80)
        return self.shape_ok and self.max_abs <= tol


def compare_arrays(a: ArrayObject, b: ArrayObject) -> CompareReport:
    """hft::compare_arrays (weather.cpp:184-217)."""
    r = CompareReport()
    r.shape_ok = a.bounds == b.bounds
    if not r.shape_ok:
        return r
    r.cells = a.size()
    if r.cells == 0:
        return r
    d = np.abs(a.data - b.data)
    # `d > max_abs` (weather.cpp:196): NaN differences never win, the first of
    # equal maxima does, and nothing below or at 0 moves `worst` off cell 0
    dn = np.where(np.isnan(d), -np.inf, d)
    worst = int(np.argmax(dn))
    r.max_abs = float(dn[worst])
    if not r.max_abs > 0.0:
        worst, r.max_abs = 0, 0.0
    diff = a.data - b.data
    sq = float(np.sum(diff * diff))
    # lo/hi start at a.data[0] and follow std::min/std::max, which keep their
    # first argument when a comparison with NaN is false
    if np.isnan(a.data[0]):
        lo = hi = float("nan")
    else:
        lo, hi = float(np.nanmin(a.data)), float(np.nanmax(a.data))
    rng = hi - lo
    if rng == 0.0:
        rng = 1.0
    r.nrmse = math.sqrt(sq / r.cells) / rng
    rest = worst
    for dim in range(a.rank()):
        ext = a.extent(dim)
        r.where.append(a.bounds[dim][0] + rest % ext)
        rest //= ext
    return r


def compare_fields(a: SimState, b: SimState) -> StateReport:
    """hft::compare_fields (weather.cpp:219-245): the worst field wins."""
    out = StateReport(shape_ok=True)
    first = True
    for name in ("energy", "energy_u", "energy_surf", "energy_pbl"):
        r = compare_arrays(getattr(a, name), getattr(b, name))
        if not r.shape_ok:
            out.shape_ok = False
            out.field = name
            return out
        if first or r.max_abs > out.max_abs:
            out.max_abs, out.field, out.where, out.nrmse = r.max_abs, name, r.where, r.nrmse
            first = False
    return out


# ---------------------------------------------------------------------------
# dump format (weather.cpp:251-304)
# ---------------------------------------------------------------------------
def dump_field(out, a: ArrayObject) -> None:
    """Header ``nx ny nz lo1 lo2 lo3`` then ``i j k value`` (%.17g), i slowest."""
    b = list(a.bounds) + [(1, 1)] * (3 - a.rank())
    out.write(f"{b[0][1] - b[0][0] + 1} {b[1][1] - b[1][0] + 1} {b[2][1] - b[2][0] + 1} "
              f"{b[0][0]} {b[1][0]} {b[2][0]}\n")
    v = a.view().reshape([a.extent(d) for d in range(a.rank())] + [1] * (3 - a.rank()), order="F")
    lines = []
    for ii, i in enumerate(range(b[0][0], b[0][1] + 1)):
        for jj, j in enumerate(range(b[1][0], b[1][1] + 1)):
            for kk, k in enumerate(range(b[2][0], b[2][1] + 1)):
                lines.append(f"{i} {j} {k} {_g17(v[ii, jj, kk])}\n")
    out.write("".join(lines))


def _g17(x: float) -> str:
    """printf("%.17g") formatting."""
    return "%.17g" % x


def read_field(inp, diags: Diagnostics) -> Optional[ArrayObject]:
    """Inverse of dump_field; truncation and out-of-bounds cells are errors."""
    toks = inp.read().split()
    where = ("<dump>", 1)
    if len(toks) < 6:
        diags.error(where, "dump header must hold three extents and three lower bounds")
        return None
    try:
        ex = [int(t) for t in toks[0:3]]
        lo = [int(t) for t in toks[3:6]]
    except ValueError:
        diags.error(where, "dump header must hold three extents and three lower bounds")
        return None
    if any(e < 1 for e in ex):
        diags.error(where, "dump extents must be positive")
        return None
    a = ArrayObject([(lo[d], lo[d] + ex[d] - 1) for d in range(3)])
    body = toks[6:]
    n = a.size()
    for c in range(n):
        rec = body[4 * c: 4 * c + 4]
        try:
            if len(rec) < 4:
                raise ValueError
            i, j, k, v = int(rec[0]), int(rec[1]), int(rec[2]), float(rec[3])
        except ValueError:
            diags.error(where, f"dump ends after {c} of {n} cells")
            return None
        off = a.offset([i, j, k])
        if off < 0:
            diags.error(where, f"dump cell ({i}, {j}, {k}) is outside the declared bounds")
            return None
        a.data[off] = v
    return a


def unpermute_storage(raw: ArrayObject, order: Sequence[int]) -> ArrayObject:
    """hft::unpermute_storage (weather.cpp:306-338): raw position p holds
    logical dimension order[p]-1; returns the logical-order array."""
    rank = raw.rank()
    if len(order) != rank:
        return raw.copy()
    pos = [0] * rank
    for p in range(rank):
        pos[order[p] - 1] = p
    out = ArrayObject([raw.bounds[pos[d]] for d in range(rank)])
    if out.size() == 0:
        return out
    rv = raw.view()
    # logical axis d is raw axis pos[d]
    out.data = np.transpose(rv, pos).reshape(-1, order="F").copy()
    return out
