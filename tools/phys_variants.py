"""A/B of the IJK column-physics kernels (HFTW_PHYS_VARIANT 0/1/2) at ASUCA size:
bitwise agreement with variant 0 and time per call (events on the context's stream)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1802_05839_b200 import weather as W

cfg = W.GridConfig(nx=1581, ny=1301, nz=58)
rng = np.random.default_rng(5)
st = W.SimState.allocate(cfg)
for a in (st.energy, st.energy_surf, st.energy_pbl):
    a.data[...] = rng.standard_normal(a.data.shape)
res = {}
with W.Context(cfg) as ctx:
    alg = ctx.algorithmic_bytes("physics")
    s = torch.cuda.ExternalStream(ctx.stream)
    for var in (0, 1, 2, 0, 1, 2):
        os.environ["HFTW_PHYS_VARIANT"] = str(var)
        ctx.upload_state(st)
        ctx.physics(0)
        out = ctx.download("energy")
        if var not in res:
            res[var] = out
        ok = np.array_equal(out.view(np.uint64), res[0].view(np.uint64))
        ctx.sync()
        n = 40
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(n):
            ctx.physics(0)
        e1.record(s)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / n
        print(f"variant {var}: bitwise={ok} {ms:.4f} ms/call {alg / ms / 1e6:.0f} GB/s")
