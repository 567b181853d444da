"""A/B of the diffusion sweep kernels (TMA vs tile, HFTW_DIFFUSE_TILE) at 256x256x64:
sweeps over ROT independent grids round robin (L2 cold), events on the context stream."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1802_05839_b200 import weather as W

cfg = W.GridConfig(nx=256, ny=256, nz=64)
ROT = 6
ctxs = [W.Context(cfg) for _ in range(ROT)]
for c in ctxs[1:]:
    c.set_stream(ctxs[0].stream)
for c in ctxs:
    c.init()
    c.step(1)
s = torch.cuda.ExternalStream(ctxs[0].stream)
alg = ctxs[0].algorithmic_bytes("diffuse")
for tile, kb in (("0", 0), ("1", 4), ("1", 8), ("1", 16), ("1", 32), ("1", 64), ("0", 0)):
    os.environ["HFTW_DIFFUSE_TILE"] = tile
    os.environ["HFTW_TILE_KB"] = str(kb)
    for i in range(12):
        ctxs[i % ROT].diffuse()
    n = 240
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for i in range(n):
        ctxs[i % ROT].diffuse()
    b.record(s)
    b.synchronize()
    us = a.elapsed_time(b) / n * 1e3
    print(f"tile={tile} kb={kb}: {us:.2f} us/sweep, {alg / (us * 1e-6) / 1e9:.0f} GB/s algorithmic")
for c in ctxs[::-1]:  # the first context owns the shared stream: close it last
    c.close()
