"""Single-step TMA launches only (compute-sanitizer racecheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_05839_b200 import weather as W
for layout in ("ijk", "kij"):
    with W.Context(W.GridConfig(nx=70, ny=37, nz=58), layout=layout, kernel="fused_tma") as ctx:
        ctx.init()
        for _ in range(3):
            ctx.step(1)
        ctx.diffuse()
        ctx.sync()
print("ok")
