"""hftw_step_host with pageable (numpy) vs pinned host buffers at ASUCA size."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1802_05839_b200 import weather as W

cfg = W.GridConfig(nx=1581, ny=1301, nz=58)
n3 = (cfg.nx + 2) * (cfg.ny + 2) * cfg.nz
n2 = (cfg.nx + 2) * (cfg.ny + 2)
with W.Context(cfg) as ctx:
    ctx.init()
    for pinned in (True, False, True, False):
        mk = (lambda n: torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()) if pinned \
            else (lambda n: np.empty(n))
        e, eu, sf, pb = mk(n3), mk(n3), mk(n2), mk(n2)
        for n, a in (("energy", e), ("energy_surf", sf), ("energy_pbl", pb)):
            ctx.download(n, a)
        ctx.step_host(e, sf, pb, e, eu)
        ctx.sync()
        t0 = time.perf_counter()
        for _ in range(3):
            ctx.step_host(e, sf, pb, e, eu)
        ctx.sync()
        print("pinned" if pinned else "pageable", round((time.perf_counter() - t0) / 3 * 1e3, 1), "ms/step", flush=True)

# the drop-in with registered (page-locked) numpy buffers
with W.Context(cfg) as ctx:
    ctx.init()
    e, eu, sf, pb = np.empty(n3), np.empty(n3), np.empty(n2), np.empty(n2)
    for n, a in (("energy", e), ("energy_surf", sf), ("energy_pbl", pb)):
        ctx.download(n, a)
    with W.pinned(e, eu, sf, pb):
        ctx.step_host(e, sf, pb, e, eu)
        ctx.sync()
        t0 = time.perf_counter()
        for _ in range(3):
            ctx.step_host(e, sf, pb, e, eu)
        ctx.sync()
        print("registered", round((time.perf_counter() - t0) / 3 * 1e3, 1), "ms/step", flush=True)
