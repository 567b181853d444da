#!/usr/bin/env python3
"""Benchmark of the B200 minimal-weather timestep (one JSON line on rank 0).

Metric (BASELINE.json): grid-cell updates/sec per timestep and achieved HBM
GB/s vs peak.  Headline workload (north_star target): the FULL timestep on the
ASUCA grid 1581x1301x58, fp64, inputs resident in HBM (957 MB per field, far
larger than the 126 MB L2, so no flush is needed between steps).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload full|stencil|physics] [--layout ijk|kij] [--kernel auto|...]

"value" counts INNER cells (nx*ny*nz per step), the convention BASELINE.md
uses for the paper's numbers.  The roofline uses SURVEY.md 8(d)'s
algorithmic bytes: 16 B per stored cell + 16 B per column for a step.

--impl reference times the reference's own CPU implementation (oracle/_ref,
the unmodified hft::reference_step compiled from its sources; the C port if
that library is absent) on the same workload on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "grid-cell updates/sec per timestep and achieved HBM GB/s vs peak"
UNIT = "cell-updates/s"
WORKLOADS = {
    # name: (grid, description)
    "full": ((1581, 1301, 58), "full minimal-weather timestep (column physics + 7-point "
             "diffusion, cyclic ghosts) on the ASUCA grid 1581x1301x58 fp64, single B200"),
    "stencil": ((256, 256, 64), "3D diffusion stencil only, 256x256x64 fp64 (L2 flushed "
                "between sweeps)"),
    "physics": ((1581, 1301, 58), "column physics only (k-dependent column loop), "
                "1581x1301x58 fp64"),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload, layout, kernel):
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(f"{workload}/{layout}/{kernel}")
    except Exception:
        return None


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# ---------------------------------------------------------------------------
# CPU: the reference (oracle/_ref) or its C restatement -- checker/baseline only
# ---------------------------------------------------------------------------
def cpu_reference_rate(grid, steps, workload="full"):
    """Rate of the reference CPU path (1 thread; the reference is serial).

    full: the unmodified hft::reference_step from oracle/_ref ("reference"),
    else the C restatement ("port").  physics/stencil: the restatement's phase
    functions (the reference has no phase-only entry point)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    nx, ny, nz = grid
    g = O.make_grid(nx, ny, nz)
    kind = "port"
    if workload == "full" and O.RefOracle.available():
        kind = "reference"
        dt = O.RefOracle().time_steps(g, steps)
    else:
        c = O.COracle()
        st = c.init(g)
        t0 = time.perf_counter()
        if workload == "full":
            c.lib.wo_steps(C_byref(g), steps, *(O._p(a) for a in (st.energy, st.energy_u,
                                                                 st.energy_surf, st.energy_pbl)))
        elif workload == "physics":
            for _ in range(steps):
                c.lib.wo_physics(C_byref(g), O._p(st.energy), O._p(st.energy_surf),
                                 O._p(st.energy_pbl))
        else:
            for _ in range(steps):
                c.lib.wo_diffuse(C_byref(g), O._p(st.energy), O._p(st.energy_u))
        dt = time.perf_counter() - t0
    rate = nx * ny * nz * steps / dt
    what = "hft::reference_step (oracle/_ref)" if kind == "reference" else f"oracle port ({workload})"
    sample = f"{steps} x {what} on {nx}x{ny}x{nz}: {dt:.2f} s, 1 thread (the reference is serial)"
    return rate, dt, kind, sample


def C_byref(x):
    import ctypes
    return ctypes.byref(x)


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if world > 1 and rank != 0:
        return 0
    grid, desc = WORKLOADS[args.workload]
    # bounded sample: one reference step is ~0.6 s at the ASUCA size on one core
    n = max(1, min(args.steps, 20 if args.workload != "stencil" else 200))
    for _ in range(min(args.warmup, 1)):
        cpu_reference_rate(grid, 1, args.workload)
    rate, dt, kind, sample = cpu_reference_rate(grid, n, args.workload)
    line = {"metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
            "steps": n, "warmup": args.warmup, "ms_per_step": dt / n * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference_init initial condition)", "impl": "reference",
            "config": {"workload": desc, "grid": list(grid), "cells_counted": "inner nx*ny*nz"},
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": 1, "kind": kind,
                             "sample": sample, "host_nproc": os.cpu_count()},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch
    from paper_1802_05839_b200 import weather as W

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    grid, desc = WORKLOADS[args.workload]
    nx, ny, nz = grid
    cfg = W.GridConfig(nx=nx, ny=ny, nz=nz)
    ctx = W.Context(cfg, layout=args.layout, device=local, kernel=args.kernel)
    ctx.init()
    stream = torch.cuda.ExternalStream(ctx.stream, device=local)
    kernel_name = ctx.kernel
    flush = None
    if args.workload == "stencil":
        # 2 x 34 MB fits in L2: flush with a 256 MB write between sweeps
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
        ctx.step(1)  # start from the state after one step (BASELINE configs[1])

    def one():
        if args.workload == "full":
            ctx.step(1)
        elif args.workload == "physics":
            ctx.physics(args.physics_mode)
        else:
            ctx.diffuse()

    for _ in range(args.warmup):
        one()
    ctx.sync()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    K = args.steps
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(K)]
    barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    with sampler:
        t_wall = time.perf_counter()
        with torch.cuda.stream(stream):
            for i in range(K):
                if flush is not None:
                    flush.add_(1)  # on `stream`: outside the per-launch events
                evs[i][0].record(stream)
                one()
                evs[i][1].record(stream)
        stream.synchronize()
        t_wall = time.perf_counter() - t_wall
    torch.cuda.synchronize()
    barrier()
    launch_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = evs[0][0].elapsed_time(evs[-1][1]) if flush is None else sum(launch_ms)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([total_ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / K
    inner = nx * ny * nz
    value = inner * world / (ms_per_step * 1e-3)

    what = {"full": "step", "physics": "physics", "stencil": "diffuse"}[args.workload]
    alg_bytes = ctx.algorithmic_bytes(what)
    avg_launch_s = statistics.mean(launch_ms) * 1e-3
    peak, peak_src = peaks()
    achieved = alg_bytes / avg_launch_s / 1e9
    traffic = ncu_traffic(args.workload, args.layout, kernel_name)

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference_init initial condition; fp64 fields resident in HBM)",
            "config": {"workload": desc, "grid": list(grid), "layout": args.layout,
                       "kernel": kernel_name, "cells_counted": "inner nx*ny*nz per step",
                       "l2": ("flushed between sweeps (256 MB write)" if flush is not None else
                              "inputs larger than L2 (957 MB per field vs 126 MB L2)"),
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU"},
            "hbm_gbs": achieved,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "avg_launch_ms": avg_launch_s * 1e3,
                         "paper_model_bytes_per_cell": {"m_sa=4": 32, "m_sa=10": 80}},
            "gpu_launches": K * (ctx.launches_per_step if args.workload == "full" else 1),
            "clocks": sampler.summary(),
            "wall_s_timed_region": t_wall}

    if args.workload == "full" and not args.no_e2e:
        line["e2e"] = e2e(ctx, cfg, args, stream, local, world)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, dt, kind, sample = cpu_reference_rate(grid, args.cpu_steps, args.workload)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": 1, "kind": kind,
                                "sample": sample, "host_nproc": os.cpu_count()}
    ctx.close()
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def e2e(ctx, cfg, args, stream, local, world):
    """Same metric through the reference-facing API with HOST buffers: each step
    uploads the step's inputs (energy, energy_surf, energy_pbl) from pinned host
    memory, runs hftw_step, and reads back the observable state (energy and
    energy_u), i.e. the drop-in for hft::reference_step on a host SimState."""
    import torch
    n3 = (cfg.nx + 2) * (cfg.ny + 2) * cfg.nz
    n2 = (cfg.nx + 2) * (cfg.ny + 2)
    bufs = {n: torch.empty(n3 if n in ("energy", "energy_u") else n2, dtype=torch.float64,
                           pin_memory=True).numpy()
            for n in ("energy", "energy_u", "energy_surf", "energy_pbl")}
    for n in bufs:
        ctx.download(n, bufs[n])
    K = max(1, args.e2e_steps)
    h2d = 8 * (n3 + 2 * n2)
    d2h = 8 * (2 * n3)

    def one():
        ctx.upload("energy", bufs["energy"])
        ctx.upload("energy_surf", bufs["energy_surf"])
        ctx.upload("energy_pbl", bufs["energy_pbl"])
        ctx.step(1)
        ctx.download("energy", bufs["energy"])
        ctx.download("energy_u", bufs["energy_u"])

    one()
    ctx.sync()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    t0 = time.perf_counter()
    for _ in range(K):
        one()
    b.record(stream)
    b.synchronize()
    wall = time.perf_counter() - t0
    ms = a.elapsed_time(b) / K
    return {"value": cfg.nx * cfg.ny * cfg.nz * world / (ms * 1e-3), "unit": UNIT,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": K,
            "ms_per_step": ms, "wall_ms_per_step": wall / K * 1e3,
            "api": "hftw_upload x3 + hftw_step(1) + hftw_download x2 (pinned host buffers)"}


def main():
    p = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawTextHelpFormatter)
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=300)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", choices=sorted(WORKLOADS), default="full")
    p.add_argument("--layout", choices=["ijk", "kij"], default="ijk")
    p.add_argument("--kernel", choices=["auto", "fused_tma", "fused_cell", "split"], default="auto")
    p.add_argument("--physics-mode", type=int, default=0)
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--cpu-steps", type=int, default=16)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    args = p.parse_args()
    args.warmup = max(args.warmup, 3)  # timing rule: at least 3 warm-up steps
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
