"""The paper's bandwidth performance model, with a B200 entry.

Mirror of hft::perf (/root/reference/proj/include/hft/perfmodel.hpp,
src/perfmodel.cpp): the machine table (perfmodel.cpp:33-69), arithmetic
intensity (:86), compute-bound threshold (:88-94), the Eq. (1) profitability
condition (:96-124), and the host / device time models (:126-154).  Known
answers are pinned in tests/test_perfmodel.py against test_perfmodel.cpp.

New here: a "b200" machine whose device entries are
MEASURED on this pool (MEASURED_PEAKS.json copy bandwidth; host-to-device and
random-access rates from tools/measure_machine.py when present), so the
paper's model can be set against the measured step times the way the paper's
Tables 5-6 do.
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, replace
from typing import List, Optional

GIGA = 1e9


@dataclass
class HardwareMetrics:
    """hft::perf::HardwareMetrics (perfmodel.hpp:19-33)."""

    name: str
    host: str = ""
    device: str = ""
    p_h1c: Optional[float] = None   # GFLOP/s, one host core
    p_h: Optional[float] = None     # GFLOP/s, one host socket
    p_d: Optional[float] = None     # GFLOP/s, device
    bw_h1c: Optional[float] = None  # GB/s, one host core
    bw_h: Optional[float] = None    # GB/s, one host socket
    bw_d: Optional[float] = None    # GB/s, device memory
    bw_htod: Optional[float] = None  # GB/s, host-to-device interconnect
    ra_h: Optional[float] = None    # GUP/s, host random access
    ra_d: Optional[float] = None    # GUP/s, device random access
    source: str = ""


@dataclass
class ModelParams:
    """hft::perf::ModelParams (perfmodel.hpp:36-45)."""

    nx: int = 0
    ny: int = 0
    nz: int = 0
    steps: int = 0
    b: float = 8.0
    m_sa: float = 10.0
    m_ra: float = 4.0
    m_htod: float = 0.0


@dataclass
class Calc:
    value: float = 0.0
    error: str = ""

    def ok(self) -> bool:
        return not self.error


_PAPER_TABLE = [  # perfmodel.cpp:36-67
    HardwareMetrics("tsubame2.0", "Xeon X5670", "Tesla M2050", bw_d=108.6),
    HardwareMetrics("tsubame2.5", "Xeon X5670", "Tesla K20x", p_h1c=9.50, p_h=57.0, p_d=1030.0,
                    bw_h1c=9.80, bw_h=20.5, bw_d=169.4, bw_htod=4.32, ra_h=0.12, ra_d=0.88),
    HardwareMetrics("piz-daint", "Xeon E5-2670", "Tesla P100", p_d=3900.0, bw_h=51.2,
                    bw_d=499.4, bw_htod=10.96),
    HardwareMetrics("reedbush-h", "Xeon E5-2695 v4", "Tesla P100", p_d=3900.0, bw_h=76.8,
                    bw_d=499.4, bw_htod=10.96),
    HardwareMetrics("tsubame3.0", "", "Tesla P100", bw_d=499.4),
]


def _b200() -> HardwareMetrics:
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    m = HardwareMetrics("b200", "GPU host", "NVIDIA B200",
                        p_d=40000.0,  # nominal fp64 (non-tensor) GFLOP/s, context only
                        source="bw_d: MEASURED_PEAKS.json hbm_gbs (copy, read+write)")
    try:
        with open(os.path.join(root, "MEASURED_PEAKS.json")) as f:
            m.bw_d = float(json.load(f)["hbm_gbs"])
    except Exception:
        m.bw_d, m.source = 6650.0, "bw_d: B200_PROFILING.md fallback"
    try:  # written by tools/measure_machine.py on the GPU box
        with open(os.path.join(root, "profiles", "machine_b200.json")) as f:
            d = json.load(f)
        for k in ("bw_htod", "ra_d", "bw_h1c", "bw_h", "ra_h"):
            if d.get(k) is not None:
                setattr(m, k, float(d[k]))
        m.source += "; " + d.get("source", "profiles/machine_b200.json")
    except Exception:
        pass
    return m


def machine_table() -> List[HardwareMetrics]:
    return list(_PAPER_TABLE) + [_b200()]


def find_machine(name: str) -> Optional[HardwareMetrics]:
    for m in machine_table():
        if m.name == name:
            return m
    return None


def machine_names() -> str:
    return ", ".join(m.name for m in machine_table())


def _missing(hw: HardwareMetrics, field: str, meaning: str, attr: str) -> str:
    # perfmodel.cpp:17-29
    msg = f"machine '{hw.name}' has no {field} ({meaning})"
    have = [m.name for m in machine_table() if getattr(m, attr) is not None]
    if have:
        msg += "; machines providing it: " + ", ".join(have)
    return msg


def arithmetic_intensity(c: float, b: float, m: float) -> float:
    return c / (b * m)  # perfmodel.cpp:86


def compute_bound_threshold(hw: HardwareMetrics) -> Calc:
    if hw.p_d is None:
        return Calc(0, _missing(hw, "P_D", "device FLOP rate", "p_d"))
    if hw.bw_d is None:
        return Calc(0, _missing(hw, "BW_D", "device memory bandwidth", "bw_d"))
    return Calc(hw.p_d / hw.bw_d)


def speedup_rhs(hw: HardwareMetrics) -> Calc:
    if hw.bw_h is None:
        return Calc(0, _missing(hw, "BW_H", "host socket bandwidth", "bw_h"))
    if hw.bw_htod is None:
        return Calc(0, _missing(hw, "BW_HtoD", "interconnect bandwidth", "bw_htod"))
    if hw.bw_d is None:
        return Calc(0, _missing(hw, "BW_D", "device memory bandwidth", "bw_d"))
    ratio = hw.bw_h / hw.bw_d
    if ratio >= 1.0:
        return Calc(0, f"machine '{hw.name}': host bandwidth is not below device bandwidth; "
                       "the profitability condition does not apply")
    return Calc((hw.bw_h / hw.bw_htod) / (1.0 - ratio))


def speedup_lhs(n_i: float, m: float, m_htod: float) -> float:
    return math.inf if m_htod == 0.0 else n_i * m / m_htod


def feasibility(hw: HardwareMetrics, n_i: float, m: float, m_htod: float):
    rhs = speedup_rhs(hw)
    if not rhs.ok():
        return rhs, None
    lhs = speedup_lhs(n_i, m, m_htod)
    return Calc(lhs), {"lhs": lhs, "rhs": rhs.value, "feasible": lhs > rhs.value}


def cpu_model_time(hw: HardwareMetrics, p: ModelParams, single_core: bool) -> Calc:
    bw = hw.bw_h1c if single_core else hw.bw_h
    if bw is None:
        return (Calc(0, _missing(hw, "BW_H1C", "single-core bandwidth", "bw_h1c")) if single_core
                else Calc(0, _missing(hw, "BW_H", "host socket bandwidth", "bw_h")))
    if hw.ra_h is None:
        return Calc(0, _missing(hw, "RA_H", "host random-access rate", "ra_h"))
    points = float(p.nx) * p.ny * p.nz
    boundary = float(p.ny) * p.nz
    per_step = points * p.b * p.m_sa / (bw * GIGA) + boundary * p.m_ra / (hw.ra_h * GIGA)
    return Calc(p.steps * per_step)


def gpu_model_time(hw: HardwareMetrics, p: ModelParams) -> Calc:
    if hw.bw_d is None:
        return Calc(0, _missing(hw, "BW_D", "device memory bandwidth", "bw_d"))
    if hw.ra_d is None:
        return Calc(0, _missing(hw, "RA_D", "device random-access rate", "ra_d"))
    if p.m_htod != 0.0 and hw.bw_htod is None:
        return Calc(0, _missing(hw, "BW_HtoD", "interconnect bandwidth", "bw_htod"))
    points = float(p.nx) * p.ny * p.nz
    boundary = float(p.ny) * p.nz
    per_point = p.b * p.m_sa / (hw.bw_d * GIGA)
    if p.m_htod != 0.0:
        per_point += p.b * p.m_htod / (hw.bw_htod * GIGA)
    per_step = points * per_point + boundary * p.m_ra / (hw.ra_d * GIGA)
    return Calc(p.steps * per_step)


def format_sig4(v: float) -> str:
    return "%.4g" % v


def b200_report(measured_ms_per_step: float, nx=1581, ny=1301, nz=58) -> dict:
    """The paper's device model on the B200 entry vs a measured step time:
    m_sa = 4 ("with cache", 32 B/cell), m_sa = 10 ("without", 80 B/cell), and
    the fused kernel's algorithmic 2 values/cell (16 B/cell)."""
    hw = find_machine("b200")
    hw_ra = hw if hw.ra_d is not None else replace(hw, ra_d=math.inf)
    out = {"machine": hw.name, "bw_d_GBps": hw.bw_d, "ra_d_GUPs": hw.ra_d,
           "measured_ms_per_step": measured_ms_per_step, "model_ms_per_step": {}}
    for label, m in (("m_sa=10", 10.0), ("m_sa=4", 4.0), ("m_sa=2 (fused)", 2.0)):
        c = gpu_model_time(hw_ra, ModelParams(nx, ny, nz, 1, 8.0, m, 4.0, 0.0))
        out["model_ms_per_step"][label] = c.value * 1e3
    return out
