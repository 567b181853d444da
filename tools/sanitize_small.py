"""Small runs of every launch path, for compute-sanitizer: pair passes, the multi-step
launch, single steps, split, cell, physics, diffusion, step_host and simulate (IJK/KIJ)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1802_05839_b200 import weather as W

cfg = W.GridConfig(nx=70, ny=37, nz=58)
for layout in ("ijk", "kij"):
    for kernel in ("auto", "fused_pair", "fused_tma", "fused_cell", "split"):
        with W.Context(cfg, layout=layout) as ctx:
            try:
                ctx.set_kernel(kernel)
            except W.HftwError:
                continue
            ctx.init()
            ctx.step(5)
            ctx.step(1)
            ctx.physics(0)
            ctx.physics(1)
            ctx.diffuse()
            ctx.diffuse(3)
            st = ctx.download_state()
            e, eu = ctx.step_host(st.energy.data.copy(), st.energy_surf.data.copy(),
                                  st.energy_pbl.data.copy())
            ctx.simulate(0.0, 2.95, 0.1, 1.0, lambda tag, t, f: None)
            ctx.sync()
print("ok")

# decomposed ranks in one process (a group on this device): pair passes with the
# ghost kernel, single steps and multi-step launches with in-kernel pushes
for kernel, opt in (("auto", 0), ("fused_tma", 1), ("fused_tma", -1)):
    with W.Context(W.GridConfig(nx=70, ny=45, nz=58), px=2, py=2, devices=[0] * 4,
                   kernel=kernel) as ctx:
        ctx.set_option("multistep", opt)
        ctx.init()
        ctx.step(4)
        ctx.step(3)
        ctx.download_state()
        ctx.sync()
print("ok group")
