"""e2e probe: hftw_step_host time vs row-block count, and its PCIe legs alone."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1802_05839_b200 import weather as W

cfg = W.GridConfig(nx=1581, ny=1301, nz=58)
n3 = (cfg.nx + 2) * (cfg.ny + 2) * cfg.nz
n2 = (cfg.nx + 2) * (cfg.ny + 2)
pin = lambda n: torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
e, eu, sf, pb = pin(n3), pin(n3), pin(n2), pin(n2)
with W.Context(cfg) as ctx:
    ctx.init()
    for name, a in (("energy", e), ("energy_surf", sf), ("energy_pbl", pb)):
        ctx.download(name, a)
    for skip in (0, 1, 2):
        os.environ["HFTW_PIPE_SKIP"] = str(skip)
        for nb in (32,):
            os.environ["HFTW_PIPE_BLOCKS"] = str(nb)
            ctx.step_host(e, sf, pb, e, eu)
            t0 = time.perf_counter()
            for _ in range(3):
                ctx.step_host(e, sf, pb, e, eu)
            print(f"skip {skip} blocks {nb}: {(time.perf_counter() - t0) / 3 * 1e3:.1f} ms/step_host", flush=True)
