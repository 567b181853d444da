"""Quick timing of the single-step and pair kernels at ASUCA size (hftw_set_timing)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
from paper_1802_05839_b200 import weather as W
from paper_1802_05839_b200._lib import lib

cfg = W.GridConfig(nx=1581, ny=1301, nz=58)
alg = 1581 * 1301 * 58
stored = (1583 * 1303 * 58) * 16 + 1583 * 1303 * 16
for kernel, n in (("fused_tma", 60), ("fused_pair", 121)):
    with W.Context(cfg, kernel=kernel) as ctx:
        ctx.init()
        ctx.step(7)
        ctx.sync()
        lib().hftw_set_timing(ctx._h, 1)
        t0 = time.perf_counter()
        ctx.step(n)
        ctx.sync()
        wall = time.perf_counter() - t0
        for kind in (0, 1, 2):
            ms, cnt, st = ctx.timing(kind)
            if cnt:
                per = ms / st  # per step
                print(f"{kernel}: kind {kind}: {cnt} launches, {st} steps, {per:.4f} ms/step, "
                      f"{stored / (per * 1e-3) / 1e9:.0f} GB/s algorithmic (16 B/cell-step)")
        print(f"{kernel}: {n} steps wall {wall * 1e3:.2f} ms -> {wall / n * 1e3:.4f} ms/step, "
              f"{alg * n / wall:.3e} cells/s")
