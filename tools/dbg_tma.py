import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_05839_b200 import weather as W
nx, ny, nz = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (16, 16, 8)))
with W.Context(W.GridConfig(nx=nx, ny=ny, nz=nz), kernel="fused_tma") as c:
    c.init(); c.step(1); c.sync(); print("ok", c.download("energy")[:4])
