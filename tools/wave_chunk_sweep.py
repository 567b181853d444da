"""Multi-step single-step launch (the decomposed path's kernel) on per-rank subdomain
sizes: ms/step for wave chunk heights (HFTW_WAVE_CHUNK, read at context creation)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_05839_b200 import weather as W

for nx, ny in ((1581, 1301), (791, 651), (791, 326)):
    for ch in (8, 12, 16, 24, 32):
        os.environ["HFTW_WAVE_CHUNK"] = str(ch)
        with W.Context(W.GridConfig(nx=nx, ny=ny, nz=58), kernel="fused_tma") as ctx:
            ctx.init()
            ctx.step(20)
            ctx.sync()
            t0 = time.perf_counter()
            ctx.step(200)
            ctx.sync()
            ms = (time.perf_counter() - t0) * 1e3 / 200
        print(f"{nx}x{ny} chunk {ch:2d}: {ms:.4f} ms/step", flush=True)
