"""One small pair-kernel run (for compute-sanitizer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_05839_b200 import weather as W
nx, ny, nz = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (100, 37, 58)))
with W.Context(W.GridConfig(nx=nx, ny=ny, nz=nz), kernel="fused_pair") as ctx:
    ctx.init()
    ctx.step(3)
    ctx.sync()
print("ok")
