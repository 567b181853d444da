"""ctypes binding of libhftw.so (include/hftw.h).

There is deliberately no fallback: if the CUDA library is missing or no GPU
is visible, every compute entry point raises.  The binding itself (symbol
table, struct layout) is usable without a GPU so CPU tests can check the
exported ABI.
"""
from __future__ import annotations

import ctypes as C
import os

from ._build import LIB

HFTW_ENERGY, HFTW_ENERGY_U, HFTW_ENERGY_SURF, HFTW_ENERGY_PBL = range(4)
FIELDS = {"energy": HFTW_ENERGY, "energy_u": HFTW_ENERGY_U,
          "energy_surf": HFTW_ENERGY_SURF, "energy_pbl": HFTW_ENERGY_PBL}
LAYOUTS = {"ijk": 0, "kij": 1}
KERNELS = {"auto": 0, "fused_tma": 1, "fused_cell": 2, "split": 3, "fused_pair": 4}
KERNEL_NAMES = {v: k for k, v in KERNELS.items()}
OPTIONS = {"multistep": 1, "pair": 2, "exchange": 3, "reverse": 4}  # enum hftw_option
ERRORS = {0: "ok", 1: "EINVAL", 2: "ECUDA", 3: "ENOMEM", 4: "ESTATE", 5: "EUNSUP"}


class hftw_grid(C.Structure):
    """Mirror of hft::GridConfig (weather.hpp:26-35) / hftw_grid (include/hftw.h)."""

    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
                ("timestep", C.c_double), ("output_timestep", C.c_double),
                ("diffusion_velocity", C.c_double), ("radiation_intensity", C.c_double),
                ("transfer_velocity", C.c_double), ("surf_energy", C.c_double),
                ("pbl_energy", C.c_double)]


class hftw_plan(C.Structure):
    """hftw_plan (include/hftw.h): one rank's subdomain of a px x py decomposition."""

    _fields_ = [("px", C.c_int32), ("py", C.c_int32), ("rx", C.c_int32), ("ry", C.c_int32),
                ("rank", C.c_int32), ("gi0", C.c_int64), ("gj0", C.c_int64),
                ("lnx", C.c_int64), ("lny", C.c_int64),
                ("own_w", C.c_int32), ("own_e", C.c_int32), ("own_s", C.c_int32),
                ("own_n", C.c_int32), ("wfar", C.c_int32), ("efar", C.c_int32),
                ("sfar", C.c_int32), ("nfar", C.c_int32), ("nbr", C.c_int32 * 4),
                ("send_slot", C.c_int32 * 4), ("face_lo", C.c_int64 * 4),
                ("face_hi", C.c_int64 * 4), ("depth", C.c_int32 * 4), ("diag", C.c_int32 * 4),
                ("diag_slot", (C.c_int32 * 2) * 4)]

    def to_dict(self):
        d = {}
        for f, _ in self._fields_:
            v = getattr(self, f)
            if isinstance(v, C.Array):
                v = [list(x) if isinstance(x, C.Array) else x for x in v]
            d[f] = v
        return d


W, E, S, N = range(4)
DIRS = {"w": W, "e": E, "s": S, "n": N}


class HftwError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"hftw error {ERRORS.get(code, code)}: {msg}")
        self.code = code


# (name, restype, argtypes) for every symbol include/hftw.h declares
_P = C.c_void_p
_D = C.POINTER(C.c_double)
SIGNATURES = [
    ("hftw_abi_version", C.c_int, []),
    ("hftw_validate", C.c_int, [C.POINTER(hftw_grid), C.c_char_p, C.c_size_t]),
    ("hftw_create", C.c_int, [C.POINTER(hftw_grid), C.c_int, C.c_int, C.POINTER(_P)]),
    ("hftw_destroy", None, [_P]),
    ("hftw_init", C.c_int, [_P]),
    ("hftw_upload", C.c_int, [_P, C.c_int, _D]),
    ("hftw_download", C.c_int, [_P, C.c_int, _D]),
    ("hftw_step", C.c_int, [_P, C.c_int64]),
    ("hftw_step_host", C.c_int, [_P, _D, _D, _D, _D, _D]),
    ("hftw_host_register", C.c_int, [C.c_void_p, C.c_size_t]),
    ("hftw_host_unregister", C.c_int, [C.c_void_p]),
    ("hftw_sync", C.c_int, [_P]),
    ("hftw_set_timing", C.c_int, [_P, C.c_int]),
    ("hftw_get_timing", C.c_int, [_P, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                  C.POINTER(C.c_int64)]),
    ("hftw_last_error", C.c_char_p, [_P]),
    ("hftw_run_reference", C.c_int, [C.POINTER(hftw_grid), C.c_int64, C.c_int, _D, _D, _D, _D]),
    ("hftw_set_stream", C.c_int, [_P, _P]),
    ("hftw_stream", _P, [_P]),
    ("hftw_set_kernel", C.c_int, [_P, C.c_int]),
    ("hftw_get_kernel", C.c_int, [_P]),
    ("hftw_physics", C.c_int, [_P, C.c_int]),
    ("hftw_diffuse", C.c_int, [_P]),
    ("hftw_diffuse_steps", C.c_int, [_P, C.c_int64]),
    ("hftw_flush_l2", C.c_int, [_P, C.c_size_t]),
    ("hftw_algorithmic_bytes", C.c_double, [_P, C.c_int]),
    ("hftw_launches_per_step", C.c_int, [_P]),
    ("hftw_field_view", C.c_int, [_P, C.c_int, C.POINTER(_P), C.POINTER(C.c_int64)]),
    ("hftw_simulate", C.c_int, [_P, C.c_double, C.c_double, C.c_double, C.c_double, _P, _P,
                                C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("hftw_plan_rank", C.c_int, [C.POINTER(hftw_grid), C.c_int, C.c_int, C.c_int,
                                 C.POINTER(hftw_plan)]),
    ("hftw_create_dist", C.c_int, [C.POINTER(hftw_grid), C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_int, C.POINTER(_P)]),
    ("hftw_peer_desc_size", C.c_size_t, []),
    ("hftw_peer_export", C.c_int, [_P, _P]),
    ("hftw_peer_connect", C.c_int, [_P, _P, C.c_int]),
    ("hftw_exchange", C.c_int, [_P]),
    ("hftw_get_plan", C.c_int, [_P, C.POINTER(hftw_plan)]),
    ("hftw_set_option", C.c_int, [_P, C.c_int, C.c_int64]),
    ("hftw_create_multi", C.c_int, [C.POINTER(hftw_grid), C.c_int, C.c_int, C.c_int,
                                    C.POINTER(C.c_int), C.POINTER(_P)]),
    ("hftw_group_size", C.c_int, [_P]),
    ("hftw_group_rank", C.c_int, [_P, C.c_int, C.POINTER(_P)]),
]

# void (*)(void* user, const char* tag, double time, const double* field)
WRITE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_char_p, C.c_double, C.POINTER(C.c_double))

_lib = None


def lib(path: str = LIB) -> C.CDLL:
    """Load libhftw.so (building it first when absent and nvcc exists).
    HFTW_LIBRARY overrides the path (tools/ experiment builds only)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("HFTW_LIBRARY", path)
    if not os.path.exists(path):
        from ._build import build
        build()
    L = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def check(rc: int, ctx=None) -> None:
    if rc != 0:
        msg = lib().hftw_last_error(ctx)
        raise HftwError(rc, msg.decode() if msg else "")
