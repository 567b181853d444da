#!/usr/bin/env python3
"""Benchmark of the B200 minimal-weather timestep (one JSON line on rank 0).

Metric (BASELINE.json): grid-cell updates/sec per timestep and achieved HBM
GB/s vs peak.  Headline workload (north_star target): the FULL timestep on the
ASUCA grid 1581x1301x58, fp64, inputs resident in HBM (957 MB per field, far
larger than the 126 MB L2, so no flush is needed between steps).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload full|stencil|physics] [--layout ijk|kij] [--kernel auto|...]

--gpus N > 1 runs the paper's I x J decomposition (2 -> 2x1, 4 -> 2x2, 8 -> 2x4):
  * under torchrun (WORLD_SIZE set): one process per GPU, halos pushed by the
    step kernels through CUDA IPC mappings;
  * without it: ONE process drives N devices (hftw_create_multi, peer access
    over NVLink).  It exits non-zero when fewer than N GPUs are visible.

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
    # name: (grid, short description; the driver truncates long strings)
    "full": ((1581, 1301, 58), "full step 1581x1301x58 f64"),
    "stencil": ((256, 256, 64), "stencil only 256x256x64 f64"),
    "physics": ((1581, 1301, 58), "physics only 1581x1301x58 f64"),
}


SPEC_HBM_GBPS = 8000.0  # B200 HBM3e specification (report against it too)
ROTATE = 6  # stencil workload: independent grids swept round robin


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
            # first calls can be slow (lazy NVML state): make them here, outside the
            # timed region, so the sampling thread starts sampling at once
            pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
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


def layout_plan(args, n):
    """(px, py, scaling, global grid, workload text) of an n-GPU run."""
    from paper_1802_05839_b200.dist import process_grid
    grid, desc = WORKLOADS[args.workload]
    nx, ny, nz = grid
    px, py = (args.px, args.py) if args.px else process_grid(n)
    # at n = 1 strong and weak are the same run; the label follows --scaling so that
    # every line of a scaling series carries the same one
    scaling = args.scaling
    if n > 1 and scaling == "weak":
        nx, ny = nx * px, ny * py  # every GPU keeps an ASUCA-sized subdomain
        desc = f"full step weak {nx}x{ny}x{nz} f64 {px}x{py}"
    elif n > 1:
        desc = f"full step strong {nx}x{ny}x{nz} f64 {px}x{py}"
    return px, py, scaling, (nx, ny, nz), desc


def config_of(args, n, grid, desc, px, py, l2):
    """The `config` object, identical in both arms for the same arguments."""
    return {"workload": desc, "grid": list(grid), "layout": args.layout,
            "cells_counted": "inner nx*ny*nz per step", "l2": l2,
            "parallelism": f"{px}x{py} I x J decomposition" if n > 1 else "single GPU"}


def l2_note(args):
    if args.workload != "stencil":
        return "inputs larger than L2 (957 MB per field vs 126 MB L2)"
    if args.flush == "rotate":
        return (f"inputs larger than L2: {ROTATE} independent 256x256x64 grids swept round "
                f"robin ({ROTATE * 68} MB of fields)")
    if args.flush == "none":
        return "NOT flushed (diagnostic)"
    return f"flushed between sweeps (256 MB write, {args.flush})"


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
    # one pinned core: the calling thread runs the serial reference
    allowed = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else []
    cpu = allowed[-1] if allowed else None
    if cpu is not None:
        os.sched_setaffinity(0, {cpu})
    try:
        dt = _cpu_steps(O, g, steps, workload)
        kind = "reference" if workload == "full" and O.RefOracle.available() else "port"
    finally:
        if cpu is not None:
            os.sched_setaffinity(0, set(allowed))
    rate = nx * ny * nz * steps / dt
    what = "hft::reference_step (oracle/_ref)" if kind == "reference" else f"oracle port ({workload})"
    sample = (f"{steps} x {what} on {nx}x{ny}x{nz}: {dt:.2f} s, 1 thread pinned to cpu {cpu} "
              f"(the reference is serial)")
    return rate, dt, kind, sample


def _cpu_steps(O, g, steps, workload):
    """Seconds for `steps` of the reference CPU path (see cpu_reference_rate)."""
    if workload == "full" and O.RefOracle.available():
        return O.RefOracle().time_steps(g, steps)
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
    return time.perf_counter() - t0


def C_byref(x):
    import ctypes
    return ctypes.byref(x)


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if world > 1 and rank != 0:
        return 0
    n = max(world, args.gpus)
    px, py, scaling, ggrid, gdesc = layout_plan(args, n)
    grid, _ = WORKLOADS[args.workload]  # the CPU sample: one ASUCA-sized domain
    # bounded sample: one reference step is ~0.3-0.6 s at the ASUCA size on one
    # core; the reference is serial, so its rate does not depend on the grid split
    n = max(1, min(args.steps, 20 if args.workload != "stencil" else 200))
    for _ in range(min(args.warmup, 1)):
        cpu_reference_rate(grid, 1, args.workload)
    rate, dt, kind, sample = cpu_reference_rate(grid, n, args.workload)
    line = {"metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
            "steps": n, "warmup": args.warmup, "ms_per_step": dt / n * 1e3,
            "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference_init initial condition)", "impl": "reference",
            "config": config_of(args, args.gpus, ggrid, gdesc, px, py, l2_note(args)),
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
    import torch
    from paper_1802_05839_b200 import weather as W
    from paper_1802_05839_b200.dist import DistSimulation

    rank, world, local = dist_env()
    # --gpus N without torchrun: ONE process drives N devices (a group context)
    ngroup = args.gpus if world == 1 else 1
    if ngroup > 1 and torch.cuda.device_count() < ngroup:
        print(f"bench.py: --gpus {ngroup} needs {ngroup} visible GPUs, found "
              f"{torch.cuda.device_count()}", file=sys.stderr)
        return 2
    ndev = max(1, torch.cuda.device_count())
    device = local % ndev  # ranks > GPUs only when testing the protocol on one GPU
    torch.cuda.set_device(device)
    dist = None
    if world > 1 and args.gpus not in (1, world):
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    n_gpus = max(world, ngroup)
    if world > 1:
        import torch.distributed as dist
        # no data-path collective: gloo carries the one-time IPC descriptors,
        # the barriers and the max-over-ranks of the timings
        dist.init_process_group("gloo")
    if n_gpus > 1 and args.workload != "full":
        raise SystemExit("multi-GPU runs measure the full timestep only")
    px, py, scaling, (nx, ny, nz), desc = layout_plan(args, n_gpus)
    grid = (nx, ny, nz)
    cfg = W.GridConfig(nx=nx, ny=ny, nz=nz)
    sim = None
    if ngroup > 1:
        ctx = W.Context(cfg, layout=args.layout, kernel=args.kernel, px=px, py=py,
                        devices=list(range(ngroup)))
        ctx.init()
    elif world == 1:
        ctx = W.Context(cfg, layout=args.layout, device=device, kernel=args.kernel)
        ctx.init()
    else:
        sim = DistSimulation(cfg, px, py, layout=args.layout, device=device, kernel=args.kernel)
        sim.init()
        ctx = sim.ctx
    # the streams the kernels run on: one per rank of a group, else the context's
    ranks = [ctx.rank_context(r) for r in range(ngroup)] if ngroup > 1 else [ctx]
    rstreams = [torch.cuda.ExternalStream(rc.stream, device=(r if ngroup > 1 else device))
                for r, rc in enumerate(ranks)]
    stream = rstreams[0]
    kernel_name = ctx.kernel
    flush = None
    rot = []  # stencil, --flush rotate: independent grids swept round robin
    if args.workload == "stencil":
        # 2 x 34 MB fits in L2.  rotate (default): sweep ROTATE independent grids in
        # turn, so each sweep's input was last touched ROTATE-1 sweeps (>= 170 MB of
        # other traffic) earlier -- inputs larger than L2, and no dirty flush lines
        # to write back inside the timed sweeps.  hftw / torch: a 256 MB write
        # between sweeps (on the context stream, outside the per-launch events).
        if args.flush == "rotate":
            rot = [ctx]
            for _ in range(ROTATE - 1):
                c2 = W.Context(cfg, layout=args.layout, device=device, kernel=args.kernel)
                c2.set_stream(ctx.stream)
                c2.init()
                c2.step(1)
                rot.append(c2)
        elif args.flush != "none":
            flush = (lambda: ctx.flush_l2(256 << 20)) if args.flush == "hftw" else \
                (lambda t=torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{device}"):
                 t.add_(1))
        ctx.step(1)  # start from the state after one step (BASELINE configs[1])
    sweep = [0]

    def one():
        if args.workload == "full":
            ctx.step(1)
        elif args.workload == "physics":
            ctx.physics(args.physics_mode)
        elif rot:
            rot[sweep[0] % len(rot)].diffuse()
            sweep[0] += 1
        else:
            ctx.diffuse()

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        one()
    ctx.sync()

    K = args.steps
    whole = args.workload == "full"
    # full timestep: the K steps are ONE hftw_step(K) call, as a user runs them
    # (run_reference / a forecast loop); the library fuses them into two-step
    # passes where it can.  Physics / stencil: one call per sweep.
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(1 if whole else K)]
    # a group: one event pair per rank, on that rank's device and stream
    revs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in rstreams[1:]]
    barrier()
    ctx.sync()
    torch.cuda.synchronize()
    sampler = ClockSampler(device)
    with sampler:
        t_wall = time.perf_counter()
        with torch.cuda.stream(stream):
            if whole:
                for (a, _), st in zip(revs, rstreams[1:]):
                    with torch.cuda.device(st.device):
                        a.record(st)
                evs[0][0].record(stream)
                ctx.step(K)
                evs[0][1].record(stream)
                for (_, b), st in zip(revs, rstreams[1:]):
                    with torch.cuda.device(st.device):
                        b.record(st)
            elif flush is None:
                # back-to-back calls, one event pair around all K (per-call events
                # would add their own gaps); per-launch times come from a second pass
                evs[0][0].record(stream)
                for i in range(K):
                    one()
                evs[-1][1].record(stream)
            else:
                for i in range(K):
                    flush()  # on `stream`: outside the per-launch events
                    evs[i][0].record(stream)
                    one()
                    evs[i][1].record(stream)
        ctx.sync()
        t_wall = time.perf_counter() - t_wall
    torch.cuda.synchronize()
    barrier()
    if flush is None:
        total_ms = evs[0][0].elapsed_time(evs[-1][1])
        for a, b in revs:  # the slowest rank of a group
            total_ms = max(total_ms, a.elapsed_time(b))
    if not whole and flush is None:
        # diagnostic pass: the same K calls with events around each (kernel durations)
        with torch.cuda.stream(stream):
            for i in range(K):
                evs[i][0].record(stream)
                one()
                evs[i][1].record(stream)
        stream.synchronize()
    launch_ms = [a.elapsed_time(b) for a, b in evs]
    if flush is not None:
        total_ms = sum(launch_ms)
    clocks = sampler.summary()
    kinds = {}
    if whole:
        # per-launch device times of the same K steps (a second, diagnostic pass
        # with CUDA events around every launch: hftw_set_timing)
        ctx.set_timing(True)
        ctx.step(K)
        for kind, name in ((2, "multi_step"), (1, "pair"), (0, "single_step")):
            ms, n, st = ctx.timing(kind)
            if n:
                kinds[name] = {"launches": n, "avg_launch_ms": ms / n, "steps_per_launch": st / n}
        for name, kd in kinds.items():
            # 16 B per stored cell + 16 B per column PER STEP, times the
            # steps one launch processes.  A pair pass keeps its intermediate step on
            # chip, so its DRAM traffic (ncu) is about half of this figure.
            kd["algorithmic_bytes_per_launch"] = (ranks[0].algorithmic_bytes("step") *
                                                  kd["steps_per_launch"])
        ctx.set_timing(False)
    if dist is not None:
        t = torch.tensor([total_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        allc = [None] * world
        dist.all_gather_object(allc, clocks)
        mhz = [c["sm_mhz"] for c in allc if c["sm_mhz"]]
        clocks = {"sm_mhz": min(mhz) if mhz else None, "sm_max_mhz": clocks["sm_max_mhz"],
                  "reasons": sorted({r for c in allc for r in c["reasons"]}),
                  "samples": sum(c["samples"] for c in allc), "per_rank_sm_mhz": mhz}
    ms_per_step = total_ms / K
    inner = nx * ny * nz
    value = inner / (ms_per_step * 1e-3)

    what = {"full": "step", "physics": "physics", "stencil": "diffuse"}[args.workload]
    alg_bytes = ranks[0].algorithmic_bytes(what)  # one GPU's stored cells, per launch
    peak, peak_src = peaks()
    for kd in kinds.values():
        kd["achieved_GBps"] = kd["algorithmic_bytes_per_launch"] / (kd["avg_launch_ms"] * 1e-3) / 1e9
    if len(kinds) == 1:
        # one launch kind: its average launch is the timed region itself over its
        # launches (launch gaps included), not the event-bracketed diagnostic pass
        only = next(iter(kinds.values()))
        only["avg_launch_ms_events"] = only["avg_launch_ms"]
        only["avg_launch_ms"] = total_ms / only["launches"]
        only["achieved_GBps"] = only["algorithmic_bytes_per_launch"] / (
            only["avg_launch_ms"] * 1e-3) / 1e9
    if kinds:
        # the dominant kernel: the launch kind with the largest share of the time
        dom = max(kinds, key=lambda k: kinds[k]["launches"] * kinds[k]["avg_launch_ms"])
        avg_launch_s = kinds[dom]["avg_launch_ms"] * 1e-3
        alg_bytes = kinds[dom]["algorithmic_bytes_per_launch"]
        dom_name = {"pair": "fused_pair", "multi_step": "fused_tma_multistep"}.get(
            dom, "fused_tma" if kernel_name == "fused_pair" else kernel_name)
        launches = sum(k["launches"] * (ctx.launches_per_step if n == "single_step" else 1)
                       for n, k in kinds.items())
    else:
        dom, dom_name = None, kernel_name
        # physics / stencil: one launch per call; back to back (no flush) its duration
        # is the timed region over the calls (launch gaps included), as for `value`
        avg_launch_s = (total_ms / K if flush is None and not whole
                        else statistics.mean(launch_ms)) * 1e-3
        launches = K * (ctx.launches_per_step if args.workload == "full" else 1)
    achieved = alg_bytes / avg_launch_s / 1e9
    tkey = f"mode{args.physics_mode}" if args.workload == "physics" else dom_name
    traffic = ncu_traffic(args.workload, args.layout, tkey) if n_gpus == 1 else None
    if traffic is not None and dom in ("multi_step", "pair"):
        traffic *= kinds[dom]["steps_per_launch"]  # the capture is stored per step
    # what HBM actually moved per second: the ncu DRAM bytes of one launch over
    # the same average launch duration (temporal blocking makes it less than the
    # algorithmic figure, so `achieved`/`frac` above 1 are NOT HBM utilisation)
    dram = traffic / avg_launch_s / 1e9 if traffic is not None else None

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n_gpus, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference_init initial condition; fp64 fields resident in HBM)",
            "config": config_of(args, n_gpus, grid, desc, px, py, l2_note(args)),
            "kernel": kernel_name,
            "launcher": ("torchrun: one process per GPU (CUDA IPC halos)" if world > 1 else
                         "one process, a group context over the GPUs" if ngroup > 1 else
                         "one process, one GPU"),
            "hbm_gbs": dram if dram is not None else achieved,
            "hbm_gbs_source": "ncu DRAM bytes / launch time" if dram is not None else
                              "algorithmic bytes / launch time (no ncu capture for this config)",
            "effective_gbs": achieved,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "spec_peak": SPEC_HBM_GBPS, "spec_frac": achieved / SPEC_HBM_GBPS,
                         "dram_spec_frac": dram / SPEC_HBM_GBPS if dram else None,
                         "dram_gbs": dram, "dram_frac": dram / peak if dram else None,
                         "per": "GPU (rank 0)" if n_gpus > 1 else "GPU",
                         "kernel": dom_name,
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "steps_per_launch": kinds[dom]["steps_per_launch"] if dom else 1,
                         "avg_launch_ms": avg_launch_s * 1e3,
                         "avg_launch_ms_events": (statistics.mean(launch_ms)
                                                  if not whole else None),
                         "algorithmic_bytes_per_cell_step": 16,
                         "note": ("pair passes compute two steps per HBM pass (the intermediate "
                                  "field stays on chip): DRAM traffic is ~8 B per cell-step, "
                                  "half the algorithmic 16 B, so frac (> 1) measures cell "
                                  "updates against a one-step-per-pass kernel at the HBM peak; "
                                  "dram_frac is the HBM utilisation"
                                  if dom == "pair" else None),
                         "paper_model_bytes_per_cell": {"m_sa=4": 32, "m_sa=10": 80}},
            "kernels": kinds,
            "gpu_launches": launches,
            "clocks": clocks,
            "wall_s_timed_region": t_wall}

    if args.workload == "full":
        # the paper's bandwidth model (perfmodel.cpp:141-154) on the measured B200
        # entry, for the same grid: m_sa = 10 / 4 values per cell vs measured
        from paper_1802_05839_b200 import perfmodel
        lnx, lny = (ranks[0].plan["lnx"], ranks[0].plan["lny"]) if n_gpus > 1 else (nx, ny)
        rep = perfmodel.b200_report(ms_per_step, lnx, lny, nz)  # per GPU
        line["paper_model"] = {k: rep[k] for k in ("model_ms_per_step", "bw_d_GBps", "ra_d_GUPs")}
    if args.workload == "full" and not args.no_e2e:
        if n_gpus > 1 and scaling == "weak":
            line["e2e"] = {"value": None, "unit": UNIT, "h2d_bytes_per_step": None,
                           "d2h_bytes_per_step": None,
                           "why": "weak-scaled global grid too large for per-rank host buffers"}
        else:
            line["e2e"] = e2e(ctx, sim, cfg, args, stream, world)
            if n_gpus == 1:
                line["e2e_run"] = e2e_run(ctx, cfg, args, stream)
                line["output_path"] = output_path(ctx, cfg, ms_per_step)
    if args.workload == "stencil":
        line["multi_sweep"] = multi_sweep(ctx, K, stream, inner, alg_bytes, peak)
    if rank == 0 and n_gpus == 1 and not args.no_cpu_baseline:
        rate, dt, kind, sample = cpu_reference_rate(grid, args.cpu_steps, args.workload)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": 1, "kind": kind,
                                "sample": sample, "host_nproc": os.cpu_count()}
    for c2 in rot[1:]:
        c2.close()
    if sim is not None:
        sim.close()
    else:
        ctx.close()
    if n_gpus > 1 and scaling == "strong" and args.workload == "full":
        # the weak-scaling companion of BASELINE config 5 in the same run: an
        # ASUCA-sized subdomain per GPU (px*1581 x py*1301 x 58), same kernels
        line["weak_companion"] = weak_companion(args, px, py, ngroup, world, device, dist)
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()
    return 0


def weak_companion(args, px, py, ngroup, world, device, dist):
    """K steps on the weak-scaled grid (an ASUCA-sized subdomain per GPU), timed like the
    main line: one hftw_step(K) per rank between CUDA events on its stream(s), barriers on
    both sides, the max over ranks."""
    import torch
    from paper_1802_05839_b200 import weather as W
    from paper_1802_05839_b200.dist import DistSimulation
    (nx, ny, nz), _ = WORKLOADS["full"]
    cfg = W.GridConfig(nx=nx * px, ny=ny * py, nz=nz)
    sim = None
    if ngroup > 1:
        ctx = W.Context(cfg, layout=args.layout, kernel=args.kernel, px=px, py=py,
                        devices=list(range(ngroup)))
        ctx.init()
        ranks = [ctx.rank_context(r) for r in range(ngroup)]
        streams = [torch.cuda.ExternalStream(rc.stream, device=r) for r, rc in enumerate(ranks)]
    else:
        sim = DistSimulation(cfg, px, py, layout=args.layout, device=device, kernel=args.kernel)
        sim.init()
        ctx = sim.ctx
        streams = [torch.cuda.ExternalStream(ctx.stream, device=device)]
    K = args.steps
    ctx.step(max(args.warmup, 2))
    ctx.sync()
    evs = []
    if dist is not None:
        dist.barrier()
    for st in streams:
        with torch.cuda.device(st.device):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            evs.append((a, b, st))
    ctx.step(K)
    for a, b, st in evs:
        with torch.cuda.device(st.device):
            b.record(st)
    ctx.sync()
    ms = max(a.elapsed_time(b) for a, b, _ in evs)
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if sim is not None:
        sim.close()
    else:
        ctx.close()
    n = px * py
    value = cfg.nx * cfg.ny * cfg.nz / (ms / K * 1e-3)
    return {"grid": [cfg.nx, cfg.ny, cfg.nz], "parallelism": f"{px}x{py}", "steps": K,
            "ms_per_step": ms / K, "value": value, "unit": UNIT, "per_gpu_value": value / n,
            "scaling": "weak"}


def multi_sweep(ctx, K, stream, inner, alg_bytes, peak):
    """The stencil workload's K sweeps as ONE hftw_diffuse_steps(K) call on one grid
    (the multi-step schedule: sweep s+1 starts on the rows sweep s has finished),
    after an L2 flush, best of 3.  The grid's two 34 MB fields stay in the 126 MB L2
    between its sweeps, so this is not an HBM-bound figure (the main line is: every
    sweep's input there is L2-cold)."""
    import torch
    best = None
    for _ in range(3):
        ctx.flush_l2(256 << 20)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ctx.diffuse(K)
        b.record(stream)
        b.synchronize()
        ms = a.elapsed_time(b) / K
        best = ms if best is None else min(best, ms)
    return {"sweeps_per_call": K, "ms_per_sweep": best, "value": inner / (best * 1e-3),
            "unit": UNIT, "algorithmic_GBps": alg_bytes / (best * 1e-3) / 1e9,
            "algorithmic_frac_of_copy_peak": alg_bytes / (best * 1e-3) / 1e9 / peak,
            "gpu_launches": 1,
            "note": "one persistent launch of K sweeps after an L2 flush; the 2 x 34 MB "
                    "working set stays L2-resident between sweeps (not HBM-bound)"}


def e2e(ctx, sim, cfg, args, stream, world):
    """Same metric through the reference-facing API with HOST buffers: each step
    uploads the step's inputs (energy, energy_surf, energy_pbl) from host memory,
    runs hftw_step, and reads back the observable state (energy, energy_u) --
    the drop-in for hft::reference_step on a host SimState.  Decomposed runs
    move each rank's owned part and refill the halos (hftw_exchange)."""
    import torch
    n3 = (cfg.nx + 2) * (cfg.ny + 2) * cfg.nz
    n2 = (cfg.nx + 2) * (cfg.ny + 2)
    def mk(n, pin):
        return (torch.empty(n, dtype=torch.float64, pin_memory=True).numpy() if pin
                else __import__("numpy").empty(n))

    names = ("energy", "energy_u", "energy_surf", "energy_pbl")
    try:
        bufs = {n: mk(n3 if n in ("energy", "energy_u") else n2, True) for n in names}
        pinned = True
    except RuntimeError:  # a decomposed run's ranks each hold the global host arrays
        bufs = {n: mk(n3 if n in ("energy", "energy_u") else n2, False) for n in names}
        pinned = False
    for n in bufs:
        ctx.download(n, bufs[n])
    K = max(1, args.e2e_steps)
    own = ctx.algorithmic_bytes("physics") / 16.0  # owned stored cells + columns
    cells = int(round(own * cfg.nz / (cfg.nz + 1)))
    cols = int(round(own - cells))
    h2d = 8 * (cells + 2 * cols)
    d2h = 8 * (2 * cells)

    def one():
        if sim is None:
            # hft::reference_step on a host SimState, in place: H2D / step / D2H
            # pipelined in row blocks inside the library (hftw_step_host)
            ctx.step_host(bufs["energy"], bufs["energy_surf"], bufs["energy_pbl"],
                          bufs["energy"], bufs["energy_u"])
            return
        ctx.upload("energy", bufs["energy"])
        ctx.upload("energy_surf", bufs["energy_surf"])
        ctx.upload("energy_pbl", bufs["energy_pbl"])
        sim._exchange()
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
    if sim is not None:
        t = torch.tensor([ms, wall], dtype=torch.float64)
        sim.dist.all_reduce(t, op=sim.dist.ReduceOp.MAX)
        ms, wall = float(t[0]), float(t[1])
    return {"value": cfg.nx * cfg.ny * cfg.nz / (ms * 1e-3), "unit": UNIT,
            "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world, "steps": K,
            "ms_per_step": ms, "wall_ms_per_step": wall / K * 1e3,
            "api": ("hftw_step_host (reference_step on a host SimState: H2D of energy/"
                    "energy_surf/energy_pbl, the step, D2H of energy/energy_u, pipelined in "
                    "row blocks)" if sim is None else
                    "per rank: hftw_upload x3 (owned part) + hftw_exchange + hftw_step(1) + "
                    "hftw_download x2 (owned part)") +
                   (", pinned host buffers" if pinned else ", pageable host buffers (pinning failed)")}


def e2e_run(ctx, cfg, args, stream):
    """A second end-to-end view, the reference's run_reference(cfg, K) use: the host
    SimState goes to the device once, K steps run there, and the state comes back
    once (upload x4, hftw_step(K), download x4; pinned host buffers), all inside the
    timed region.  Reported beside `e2e` (per-step host round trips), not instead."""
    import torch
    n3 = (cfg.nx + 2) * (cfg.ny + 2) * cfg.nz
    n2 = (cfg.nx + 2) * (cfg.ny + 2)
    bufs = {n: torch.empty(n3 if n in ("energy", "energy_u") else n2, dtype=torch.float64,
                           pin_memory=True).numpy()
            for n in ("energy", "energy_u", "energy_surf", "energy_pbl")}
    for n in bufs:
        ctx.download(n, bufs[n])
    K = args.steps
    ctx.sync()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for n in bufs:
        ctx.upload(n, bufs[n])
    ctx.step(K)
    for n in bufs:
        ctx.download(n, bufs[n])
    b.record(stream)
    b.synchronize()
    ms = a.elapsed_time(b)
    io = sum(v.nbytes for v in bufs.values())
    return {"value": cfg.nx * cfg.ny * cfg.nz * K / (ms * 1e-3), "unit": UNIT, "steps": K,
            "ms_total": ms, "ms_per_step": ms / K, "h2d_bytes_total": io, "d2h_bytes_total": io,
            "api": "hftw_upload x4 + hftw_step(K) + hftw_download x4 (run_reference on a host "
                   "SimState), pinned host buffers"}


def output_path(ctx, cfg, step_ms, steps=100):
    """SURVEY 8(f) item 1 measured: hftw_simulate, the corpus driver's time loop
    (simple_weather.h90:74-108 as drive() calls it, weather.cpp:364-376) with the
    GridConfig's own cadence (timestep 0.1, output every 1.0 = every 10 steps) on
    this grid.  Each output is a device snapshot plus a 957 MB D2H on a copy stream
    while the next steps run; the writer is a no-op (the reference's %.17g text
    dump is the caller's cost).  Wall clock around the call (it synchronises)."""
    dt, odt = cfg.timestep, cfg.output_timestep
    n3 = (cfg.nx + 2) * (cfg.ny + 2) * cfg.nz
    seen = []
    ctx.init()
    ctx.sync()
    ctx.simulate(0.0, 9.5 * dt, dt, odt, lambda tag, t, f: None)  # warm the output ring
    ctx.sync()
    t0 = time.perf_counter()
    nsteps, nwrites = ctx.simulate(0.0, (steps - 0.5) * dt, dt, odt,
                                   lambda tag, t, f: seen.append(t))
    ctx.sync()
    wall = (time.perf_counter() - t0) * 1e3
    d2h = nwrites * n3 * 8
    return {"api": "hftw_simulate (corpus driver time loop) with a no-op writer",
            "steps": nsteps, "writes": nwrites, "timestep": dt, "output_timestep": odt,
            "wall_ms": wall, "ms_per_step": wall / nsteps,
            "value": cfg.nx * cfg.ny * cfg.nz * nsteps / (wall * 1e-3), "unit": UNIT,
            "d2h_bytes_total": d2h, "d2h_GBps": d2h / (wall * 1e-3) / 1e9,
            "compute_only_ms": step_ms * nsteps,
            "note": "each output interval is PCIe-bound (10 steps ~2.6 ms of compute against "
                    "one 957 MB D2H); the steps run while the previous output copies"}


def main():
    p = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawTextHelpFormatter)
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=300)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", choices=sorted(WORKLOADS), default="full")
    p.add_argument("--layout", choices=["ijk", "kij"], default="ijk")
    p.add_argument("--kernel", choices=["auto", "fused_pair", "fused_tma", "fused_cell", "split"],
                   default="auto")
    p.add_argument("--physics-mode", type=int, default=0)
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--cpu-steps", type=int, default=16)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                   help="N>1: strong = ASUCA grid split over N GPUs; weak = ASUCA per GPU")
    p.add_argument("--px", type=int, default=0, help="N>1: ranks along i (default: paper grid)")
    p.add_argument("--flush", choices=["rotate", "hftw", "torch", "none"], default="rotate",
                   help="stencil workload: rotate over independent grids (inputs > L2) or an L2 "
                        "flush between sweeps ('none' is diagnostic only)")
    p.add_argument("--py", type=int, default=0)
    args = p.parse_args()
    args.warmup = max(args.warmup, 3)  # timing rule: at least 3 warm-up steps
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
