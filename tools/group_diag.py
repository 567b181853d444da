"""Per-launch-kind device times of every rank of a group on one GPU
(hftw_set_timing): where a decomposed step's time goes.  usage: group_diag.py px py weak|strong [K]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_05839_b200 import weather as W  # noqa: E402

px, py, scaling = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
K = int(sys.argv[4]) if len(sys.argv) > 4 else 20
kernel = sys.argv[5] if len(sys.argv) > 5 else "auto"
nx, ny = (1581 * px, 1301 * py) if scaling == "weak" else (1581, 1301)
cfg = W.GridConfig(nx=nx, ny=ny, nz=58)
with W.Context(cfg, px=px, py=py, devices=[0] * (px * py), kernel=kernel) as ctx:
    ctx.init()
    ctx.step(4)
    ctx.sync()
    ctx.set_timing(True)
    ctx.step(K)
    ctx.sync()
    for r in range(px * py):
        rc = ctx.rank_context(r)
        out = []
        for kind, name in ((0, "single"), (1, "pair"), (2, "multi")):
            ms, n, st = rc.timing(kind)
            if n:
                out.append(f"{name}: {n} x {ms / n:.4f} ms ({st} steps)")
        print(f"{px}x{py} {scaling} rank {r} plan {rc.plan['lnx']}x{rc.plan['lny']}: " + "; ".join(out))
