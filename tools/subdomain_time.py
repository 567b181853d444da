"""Strong-scaling compute bound on one GPU: the per-rank subdomain of a px x py
decomposition of the ASUCA grid, run as a single domain (same kernels, cyclic ghosts
instead of halos), ms/step for the multi-step single-step launch (the decomposed
path's kernel) and the pair passes, against the 1-GPU time / N."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_05839_b200 import weather as W

NX, NY, NZ = 1581, 1301, 58
base = {}
for n, (px, py) in ((1, (1, 1)), (2, (2, 1)), (4, (2, 2)), (8, (2, 4))):
    nx, ny = -(-NX // px), -(-NY // py)
    for kernel in ("fused_pair", "fused_tma"):
        cfg = W.GridConfig(nx=nx, ny=ny, nz=NZ)
        with W.Context(cfg, kernel=kernel) as ctx:
            ctx.init()
            ctx.step(20)
            ctx.sync()
            steps = 200
            t0 = time.perf_counter()
            ctx.step(steps)
            ctx.sync()
            ms = (time.perf_counter() - t0) * 1e3 / steps
        if n == 1:
            base[kernel] = ms
        ideal = base["fused_pair"] / n
        print(f"N={n} {px}x{py} sub {nx}x{ny}: {kernel:10s} {ms:.4f} ms/step  "
              f"eff vs 1-GPU pair/N {ideal / ms * 100:5.1f}%", flush=True)
