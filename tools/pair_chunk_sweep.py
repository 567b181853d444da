"""Pair passes: ms/step for unit heights (HFTW_PAIR_CHUNK, read at context creation)
on the ASUCA grid and the per-rank subdomain sizes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_05839_b200 import weather as W

for nx, ny in ((1581, 1301), (791, 1301), (791, 651), (791, 326)):
    for ch in (0, 4, 6, 8, 12, 16, 24):
        os.environ["HFTW_PAIR_CHUNK"] = str(ch)
        with W.Context(W.GridConfig(nx=nx, ny=ny, nz=58), kernel="fused_pair") as ctx:
            ctx.init(); ctx.step(21); ctx.sync()
            t0 = time.perf_counter(); ctx.step(201); ctx.sync()
            ms = (time.perf_counter() - t0) * 1e3 / 201
        print(f"{nx}x{ny} chunk {ch if ch else 'auto':>4}: {ms:.4f} ms/step", flush=True)
