"""Diffusion-only sweeps of the 256x256x64 grid (BASELINE configs[1]): K single-sweep
launches vs ONE hftw_diffuse_steps(K) call (the multi-step schedule), device time per
sweep, after an L2 flush.  usage: stencil_multi.py [K]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1802_05839_b200 import weather as W  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfg = W.GridConfig(nx=256, ny=256, nz=64)
alg = 16 * 258 * 258 * 64  # bytes per sweep (stored cells, read + write)
with W.Context(cfg) as ctx:
    ctx.init()
    ctx.step(1)
    st = torch.cuda.ExternalStream(ctx.stream)
    for mode in ("single", "multi", "single", "multi"):
        best = None
        for _ in range(5):
            ctx.flush_l2(256 << 20)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            if mode == "single":
                for _ in range(K):
                    ctx.diffuse()
            else:
                ctx.diffuse(K)
            b.record(st)
            b.synchronize()
            ms = a.elapsed_time(b) / K
            best = ms if best is None else min(best, ms)
        print(f"{mode}: K={K} {best * 1e3:.2f} us/sweep, {alg / (best * 1e-3) / 1e9:.0f} GB/s "
              f"algorithmic ({alg / (best * 1e-3) / 1e9 / 6553:.3f} of the copy peak)")
