"""A/B timing of hftw_step at the ASUCA size for one library build
(HFTW_LIBRARY=tools/exp/<name>.so): 5 repeats of hftw_step(K) between CUDA
events on the context stream (device time), min and median ms/step, plus the
per-launch-kind averages (hftw_set_timing).  usage: ab_step.py [K] [kernel] [nx ny nz]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1802_05839_b200 import weather as W  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 300
kernel = sys.argv[2] if len(sys.argv) > 2 else "auto"
nx, ny, nz = (int(x) for x in sys.argv[3:6]) if len(sys.argv) > 5 else (1581, 1301, 58)
cfg = W.GridConfig(nx=nx, ny=ny, nz=nz)
name = os.path.basename(os.environ.get("HFTW_LIBRARY", "libhftw.so"))
with W.Context(cfg, kernel=kernel) as ctx:
    ctx.init()
    ctx.step(10)
    ctx.sync()
    st = torch.cuda.ExternalStream(ctx.stream)
    res = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        ctx.step(K)
        b.record(st)
        b.synchronize()
        res.append(a.elapsed_time(b) / K)
    ctx.set_timing(True)
    ctx.step(K)
    kinds = {}
    for kind in (0, 1, 2):
        ms, n, s = ctx.timing(kind)
        if n:
            kinds[kind] = f"{n} launches x {ms / n:.4f} ms"
print(f"{name} {kernel} {nx}x{ny}x{nz} K={K}: min {min(res):.4f} median "
      f"{statistics.median(res):.4f} ms/step  {kinds}")
