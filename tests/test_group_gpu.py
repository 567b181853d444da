"""Multi-rank decompositions driven from ONE process (hftw_create_multi): the
ranks' subdomains, in-kernel halo pushes and step flags exactly as in the
one-process-per-GPU runs, with plain device pointers instead of CUDA IPC.
The test box has one GPU, so every rank sits on cuda:0 (ranks sharing a
device run one launch per step in rank order on one stream).  Bitwise against
the oracle and against hashes of the unmodified reference, including
BASELINE config 5 at full size: the 2x4 decomposition of the ASUCA grid
(strong scaling) and the 3162x5204x58 grid (weak scaling: one ASUCA-sized
subdomain per rank).
"""
import numpy as np
import pytest

import oracle as O
from paper_1802_05839_b200 import weather as W

pytestmark = pytest.mark.gpu

FIELDS = ("energy", "energy_u", "energy_surf", "energy_pbl")


def group(cfg, px, py, layout="ijk", kernel="auto"):
    return W.Context(cfg, layout=layout, kernel=kernel, px=px, py=py, devices=[0] * (px * py))


def random_state(cfg, seed):
    rng = np.random.default_rng(seed)
    g = O.grid_from(cfg)
    n3, n2 = O.shapes(g)
    return O.State(rng.uniform(150, 350, n3), rng.uniform(150, 350, n3),
                   rng.uniform(150, 350, n2), rng.uniform(150, 350, n2))


def assert_bitwise(got, want, tag):
    for f in FIELDS:
        bad = int(np.sum(got[f] != want[f]))
        assert bad == 0, f"{tag}: {f} differs in {bad} cells"


@pytest.mark.parametrize("shape,grid,calls,layout,kernel", [
    ((150, 70, 58), (2, 1), [5], "ijk", "auto"),
    ((150, 70, 58), (1, 2), [1, 3], "ijk", "fused_tma"),
    ((131, 97, 12), (2, 2), [2, 4], "ijk", "auto"),
    ((66, 41, 9), (2, 2), [3], "kij", "auto"),
    ((66, 41, 9), (2, 2), [2, 1], "ijk", "fused_cell"),
    ((130, 45, 7), (4, 2), [3], "ijk", "auto"),
    ((200, 140, 20), (2, 4), [4, 5], "ijk", "auto"),
    ((97, 61, 13), (3, 1), [2, 3], "ijk", "auto"),
    ((100, 70, 9), (3, 2), [3, 2], "ijk", "auto"),
    ((40, 30, 8), (1, 1), [4], "ijk", "auto"),
    # two-step passes on every rank (AUTO with 56 <= nz <= 58): 2-deep halos,
    # diagonal corner columns, ghost finals from the wrap partners' P'
    ((150, 97, 58), (2, 2), [5, 3], "ijk", "auto"),
    ((140, 90, 51), (2, 2), [6, 4], "ijk", "auto"),
    ((130, 100, 58), (2, 4), [7], "ijk", "auto"),
    ((160, 61, 56), (4, 2), [6], "ijk", "auto"),
    ((97, 95, 57), (3, 3), [4, 5], "ijk", "auto"),
    ((70, 130, 58), (1, 3), [5], "ijk", "auto"),
    ((90, 64, 58), (3, 1), [6, 2], "ijk", "auto"),
    ((120, 90, 20), (2, 2), [5], "ijk", "fused_pair"),   # generic row shapes
    ((64, 40, 58), (8, 1), [3], "ijk", "auto"),          # 8-column ranks
])
def test_group_random_state_bitwise(coracle, shape, grid, calls, layout, kernel):
    nx, ny, nz = shape
    cfg = W.GridConfig(nx=nx, ny=ny, nz=nz, diffusion_velocity=0.125,
                       radiation_intensity=0.37, transfer_velocity=0.013)
    s0 = random_state(cfg, 11 * nx + ny)
    want = coracle.steps(O.grid_from(cfg), s0, sum(calls)).fields()
    with group(cfg, *grid, layout=layout, kernel=kernel) as ctx:
        assert ctx.group_size == grid[0] * grid[1]
        for f, a in s0.fields().items():
            ctx.upload(f, np.ascontiguousarray(a))
        for n in calls:
            ctx.step(n)
        got = {f: ctx.download(f) for f in FIELDS}
    assert_bitwise(got, want, f"{shape}/{grid}/{layout}/{kernel}")


def test_group_init_physics_step_host_simulate(coracle):
    """Everything else a single-domain context offers, on a 2x2 group: init,
    physics alone, reference_step on host arrays, the output time loop."""
    cfg = W.GridConfig(nx=90, ny=61, nz=11)
    g = O.grid_from(cfg)
    with group(cfg, 2, 2) as ctx:
        ctx.init()
        ctx.step(3)
        got = {f: ctx.download(f) for f in FIELDS}
        assert_bitwise(got, coracle.run_reference(g, 3).fields(), "init + 3 steps")
        # column physics alone (in place on energy)
        ctx.physics(0)
        want_e = coracle.physics(g, got["energy"], got["energy_surf"], got["energy_pbl"])
        assert np.array_equal(ctx.download("energy"), want_e)
        # reference_step on host arrays (hftw_step_host on a group)
        s0 = random_state(cfg, 5)
        e, eu = ctx.step_host(s0.energy.copy(), s0.energy_surf, s0.energy_pbl)
        want = coracle.steps(g, s0, 1).fields()
        assert np.array_equal(e, want["energy"]) and np.array_equal(eu, want["energy_u"])
        # the corpus driver's time loop: 25 steps, an output every 10
        ctx.init()
        seen = []
        steps, writes = ctx.simulate(0.0, 24.5 * cfg.timestep, cfg.timestep,
                                     cfg.output_timestep, lambda tag, t, f: seen.append(f.copy()))
        assert (steps, writes) == (25, 3)
        assert np.array_equal(seen[1], coracle.run_reference(g, 10).energy)
        assert np.array_equal(ctx.download("energy"), coracle.run_reference(g, 25).energy)


def test_group_rank_views_and_errors():
    cfg = W.GridConfig(nx=64, ny=40, nz=8)
    with group(cfg, 2, 2) as ctx:
        plans = [ctx.rank_context(r).plan for r in range(4)]
        assert [p["rank"] for p in plans] == [0, 1, 2, 3]
        assert sum(p["lnx"] * p["lny"] for p in plans) == cfg.nx * cfg.ny
        with pytest.raises(W.HftwError):
            ctx.field_view("energy")  # one view per rank
        with pytest.raises(W.HftwError):
            ctx.rank_context(4)
    with pytest.raises(W.HftwError):
        W.Context(cfg, px=2, py=1, devices=[0, 64])  # no such device
    with pytest.raises(ValueError):
        W.Context(cfg, px=2, py=2, devices=[0, 0])


@pytest.mark.parametrize("steps", [7, 20])
def test_config5_strong_2x4_asuca_vs_reference_hash(golden, coracle, steps):
    """BASELINE config 5 (strong scaling): the ASUCA grid on the paper's 2x4
    decomposition, bitwise against the unmodified reference's run_reference."""
    h = golden["hashes"][f"1581x1301x58_s{steps}"]
    cfg = W.GridConfig(**h["grid"])
    with group(cfg, 2, 4) as ctx:
        ctx.init()
        ctx.step(steps)
        for f, v in h["fnv1a64"].items():
            assert coracle.fnv(ctx.download(f)) == v, (steps, f)


def test_config5_weak_3162x5204x58_on_2x4_vs_reference_hash(golden, coracle):
    """BASELINE config 5 (weak scaling): 8 x the ASUCA grid, one ASUCA-sized
    subdomain per rank of the 2x4 decomposition, bitwise against the reference."""
    h = golden["hashes"]["3162x5204x58_s5"]
    cfg = W.GridConfig(**h["grid"])
    with group(cfg, 2, 4) as ctx:
        for r in range(8):
            p = ctx.rank_context(r).plan
            assert (p["lnx"], p["lny"]) == (1581, 1301)
        ctx.init()
        ctx.step(2)
        ctx.step(3)
        out = np.empty((cfg.nx + 2) * (cfg.ny + 2) * cfg.nz)
        for f in ("energy", "energy_u"):
            assert coracle.fnv(ctx.download(f, out)) == h["fnv1a64"][f], f
        for f in ("energy_surf", "energy_pbl"):
            assert coracle.fnv(ctx.download(f)) == h["fnv1a64"][f], f


def test_asuca_default_path_vs_reference_hash(golden, coracle):
    """The bench's exact run (AUTO, one hftw_step(20) call: two-step passes)
    and an odd count, bitwise against the reference's run_reference."""
    for steps in (7, 20):
        h = golden["hashes"][f"1581x1301x58_s{steps}"]
        cfg = W.GridConfig(**h["grid"])
        with W.Context(cfg) as ctx:
            assert ctx.kernel == "fused_pair"
            ctx.init()
            ctx.set_timing(True)
            ctx.step(steps)
            _, pairs, _ = ctx.timing(1)
            assert pairs >= (steps - 2) // 2
            for f, v in h["fnv1a64"].items():
                assert coracle.fnv(ctx.download(f)) == v, (steps, f)


def test_group_reverse_unit_order_bitwise(coracle):
    """Decomposed pair passes and single steps with the work units handed out last
    first (HFTW_OPT_REVERSE) on every rank: bitwise."""
    cfg = W.GridConfig(nx=150, ny=97, nz=58, diffusion_velocity=0.11)
    s0 = random_state(cfg, 17)
    want = coracle.steps(O.grid_from(cfg), s0, 7).fields()
    with group(cfg, 2, 2) as ctx:
        for f, a in s0.fields().items():
            ctx.upload(f, np.ascontiguousarray(a))
        ctx.set_option("reverse", 1)
        ctx.step(7)
        got = {f: ctx.download(f) for f in FIELDS}
    assert_bitwise(got, want, "2x2 reverse")


@pytest.mark.parametrize("grid", [(2, 1), (2, 2), (2, 4)])
def test_exchange_baseline_bitwise(coracle, grid):
    """HFTW_OPT_EXCHANGE = 1 (the un-overlapped baseline: steps without the halo
    protocol, a separate face-copy kernel per rank) gives the same bits, and the
    flag protocol resumes after it."""
    cfg = W.GridConfig(nx=131, ny=97, nz=12, diffusion_velocity=0.125)
    s0 = random_state(cfg, 3)
    want = coracle.steps(O.grid_from(cfg), s0, 5).fields()
    with group(cfg, *grid, kernel="fused_tma") as ctx:
        for f, a in s0.fields().items():
            ctx.upload(f, np.ascontiguousarray(a))
        ctx.set_option("exchange", 1)
        ctx.step(3)
        ctx.set_option("exchange", 0)
        ctx.step(2)
        got = {f: ctx.download(f) for f in FIELDS}
    assert_bitwise(got, want, f"baseline {grid}")
