"""e2e probe: hftw_step_host time per PCIe copy mode (2D per row block vs nz 1D copies)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
    for mode in ("0",):
        for skip in ("0", "1", "2"):
            os.environ["HFTW_PIPE_1D"] = mode
            os.environ["HFTW_PIPE_SKIP"] = skip
            ctx.step_host(e, sf, pb, e, eu)
            t0 = time.perf_counter()
            for _ in range(3):
                ctx.step_host(e, sf, pb, e, eu)
            print(f"1d={mode} skip={skip}: {(time.perf_counter() - t0) / 3 * 1e3:.1f} ms", flush=True)
