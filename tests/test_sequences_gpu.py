"""Seeded random call sequences on one context against the oracle: steps with kernel
switches between calls, the physics / diffusion phases alone, uploads of new fields in
the middle (energy_u is derived lazily from the previous field and sf/pb, so a new sf/pb
must not change an energy_u that belongs to an earlier step), and downloads at random
points.  Bitwise.  The library state machine under test: the ping-pong buffer index,
the lazily derived energy_u, the pair / multi-step / single-step launch choice."""
import os

import numpy as np
import pytest

import oracle as O
from paper_1802_05839_b200 import weather as W

pytestmark = pytest.mark.gpu

FIELDS = ("energy", "energy_u", "energy_surf", "energy_pbl")


class Model:
    """The reference semantics of each call, on host arrays (the oracle's C code)."""

    def __init__(self, coracle, g, s):
        self.o, self.g = coracle, g
        self.f = {k: v.copy() for k, v in s.fields().items()}

    def step(self, n):
        st = self.o.steps(self.g, O.State(*(self.f[k] for k in FIELDS)), n)
        self.f = {k: v.copy() for k, v in st.fields().items()}

    def physics(self):
        # phase 1 in place (weather.cpp:118-128); energy_u is left alone
        self.f["energy"] = self.o.physics(self.g, self.f["energy"], self.f["energy_surf"],
                                          self.f["energy_pbl"])

    def diffuse(self):
        # phases 2-5 on the current field, then the swap (weather.cpp:170)
        u = self.o.diffuse(self.g, self.f["energy"])
        self.f["energy_u"] = self.f["energy"]
        self.f["energy"] = u


def sequences(n=120, seed=int(os.environ.get("HFTW_FUZZ_SEED", "1802"))):
    rng = np.random.default_rng(seed)
    kernels = ["auto", "fused_tma", "fused_pair", "fused_cell", "split"]
    out = []
    for c in range(n):
        shape = [(120, 50, 58), (64, 33, 17), (35, 70, 56), (200, 9, 30), (9, 9, 3)][c % 5]
        ops = []
        for _ in range(int(rng.integers(4, 9))):
            r = rng.random()
            if r < 0.45:
                ops.append(("step", str(rng.choice(kernels)), int(rng.integers(1, 8))))
            elif r < 0.55:
                ops.append(("physics", int(rng.integers(0, 2))))
            elif r < 0.65:
                ops.append(("diffuse", int(rng.integers(1, 4))))
            elif r < 0.8:
                ops.append(("upload", str(rng.choice(FIELDS))))
            else:
                ops.append(("download", str(rng.choice(FIELDS))))
        out.append(dict(id=c, shape=shape, layout=["ijk", "kij"][(c // 5) % 2], ops=ops,
                        seed=int(rng.integers(1 << 30))))
    return out


@pytest.mark.parametrize("seq", sequences(), ids=lambda s: f"s{s['id']}")
def test_call_sequence_vs_oracle(coracle, seq):
    nx, ny, nz = seq["shape"]
    rng = np.random.default_rng(seq["seed"])
    cfg = W.GridConfig(nx=nx, ny=ny, nz=nz, diffusion_velocity=float(rng.uniform(0, 1 / 6)),
                       radiation_intensity=float(rng.uniform(-0.5, 0.5)),
                       transfer_velocity=float(rng.uniform(0, 0.1)))
    g = O.grid_from(cfg)
    n3, n2 = O.shapes(g)
    s0 = O.State(rng.uniform(150, 350, n3), rng.uniform(150, 350, n3),
                 rng.uniform(150, 350, n2), rng.uniform(150, 350, n2))
    m = Model(coracle, g, s0)
    with W.Context(cfg, layout=seq["layout"]) as ctx:
        for k, v in s0.fields().items():
            ctx.upload(k, np.ascontiguousarray(v))
        for i, op in enumerate(seq["ops"]):
            if op[0] == "step":
                try:
                    ctx.set_kernel(op[1])
                except W.HftwError:
                    ctx.set_kernel("auto")
                ctx.step(op[2])
                m.step(op[2])
            elif op[0] == "physics":
                ctx.physics(op[1])
                m.physics()
            elif op[0] == "diffuse":
                ctx.diffuse(op[1])
                for _ in range(op[1]):
                    m.diffuse()
            elif op[0] == "upload":
                new = rng.uniform(150, 350, n3 if op[1] in ("energy", "energy_u") else n2)
                ctx.upload(op[1], new)
                m.f[op[1]] = new.copy()
            else:
                got = ctx.download(op[1])
                assert np.array_equal(got.view(np.uint64), m.f[op[1]].view(np.uint64)), (i, op)
        for k in FIELDS:
            got = ctx.download(k)
            assert np.array_equal(got.view(np.uint64), m.f[k].view(np.uint64)), (k, seq["ops"])
