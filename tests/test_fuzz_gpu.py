"""Seeded random sweep of the GPU path against the oracle: random extents (including
the 1-2 cell edge cases and odd nz), random physical constants, random initial fields,
1-7 steps in one call and as separate calls, every kernel and layout the context
accepts.  Bitwise, like tests/test_parity_gpu.py; the case list is fixed by the seed so
a failure reproduces by its id."""
import os

import numpy as np
import pytest

import oracle as O
from paper_1802_05839_b200 import weather as W

pytestmark = pytest.mark.gpu

KERNELS = ["auto", "fused_tma", "fused_pair", "fused_cell", "split"]


def cases(n=160, seed=int(os.environ.get("HFTW_FUZZ_SEED", "20261017"))):
    rng = np.random.default_rng(seed)
    out = []
    for c in range(n):
        # mostly small grids, some long/thin ones, some nz in the pair kernel's range
        nx = int(rng.choice([2, 3, int(rng.integers(4, 40)), int(rng.integers(40, 200)),
                             int(rng.integers(60, 200))]))
        ny = int(rng.choice([2, 3, int(rng.integers(4, 40)), int(rng.integers(40, 120)),
                             int(rng.integers(40, 120))]))
        nz = int(rng.choice([2, 3, int(rng.integers(4, 20)), int(rng.integers(20, 56)),
                             int(rng.integers(56, 59))]))
        out.append(dict(id=c, nx=nx, ny=ny, nz=nz, steps=int(rng.integers(1, 8)),
                        split_calls=bool(rng.integers(0, 2)),
                        layout=["ijk", "kij"][c % 2],
                        kernel=str(rng.choice(KERNELS)),
                        dv=float(rng.uniform(0, 1 / 6)), ri=float(rng.uniform(-1, 1)),
                        tv=float(rng.uniform(0, 0.2)), fseed=int(rng.integers(1 << 30))))
    return out


@pytest.mark.parametrize("case", cases(), ids=lambda c: f"c{c['id']}")
def test_random_case_vs_oracle(coracle, case):
    cfg = W.GridConfig(nx=case["nx"], ny=case["ny"], nz=case["nz"],
                       diffusion_velocity=case["dv"], radiation_intensity=case["ri"],
                       transfer_velocity=case["tv"])
    g = O.grid_from(cfg)
    ok, _ = coracle.validate(g)
    if not ok:
        pytest.skip("extents the reference rejects (hft::validate)")
    n3, n2 = O.shapes(g)
    rng = np.random.default_rng(case["fseed"])
    s0 = O.State(rng.uniform(-400, 400, n3), rng.uniform(-400, 400, n3),
                 rng.uniform(-400, 400, n2), rng.uniform(-400, 400, n2))
    want = coracle.steps(g, s0, case["steps"]).fields()
    with W.Context(cfg, layout=case["layout"]) as ctx:
        try:
            ctx.set_kernel(case["kernel"])
        except W.HftwError:
            ctx.set_kernel("auto")  # e.g. the pair kernel on KIJ: AUTO is the fallback
        for name, arr in s0.fields().items():
            ctx.upload(name, np.ascontiguousarray(arr))
        if case["split_calls"]:
            for _ in range(case["steps"]):
                ctx.step(1)
        else:
            ctx.step(case["steps"])
        got = {n: ctx.download(n) for n in ("energy", "energy_u", "energy_surf", "energy_pbl")}
    for f in want:
        a, b = got[f].view(np.uint64), want[f].view(np.uint64)
        bad = np.flatnonzero(a != b)
        assert bad.size == 0, (case, f, bad[:5], got[f].flat[bad[:3]], want[f].flat[bad[:3]])
