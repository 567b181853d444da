"""Why does the clock sampler see few samples in the default timed region?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1802_05839_b200 import weather as W

cfg = W.GridConfig(nx=1581, ny=1301, nz=58)
with W.Context(cfg) as ctx:
    ctx.init(); ctx.step(10); ctx.sync()
    s = torch.cuda.ExternalStream(ctx.stream)
    smp = bench.ClockSampler(0)
    t0 = time.perf_counter()
    with smp:
        t1 = time.perf_counter()
        ctx.step(300)
        t2 = time.perf_counter()
        s.synchronize()
        t3 = time.perf_counter()
    t4 = time.perf_counter()
    print(f"enter {1e3*(t1-t0):.2f} ms, step call {1e3*(t2-t1):.2f} ms, sync {1e3*(t3-t2):.2f} ms, "
          f"exit {1e3*(t4-t3):.2f} ms, samples {len(smp.samples)}, {smp.summary()}")
