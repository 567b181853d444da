"""GPU parity: the sm_100a path, called through the C ABI, against the oracle.

Bar: BITWISE equality on all four SimState fields (the library uses only
explicitly rounded IEEE double ops in the reference's association order, so
the tolerance is exactly 0).  Sources of truth:
  * tests/golden/*.npz -- outputs of the unmodified reference,
  * golden FNV-1a-64 hashes at the BASELINE sizes (256x256x64, 1581x1301x58),
  * the C restatement (oracle/) on fresh seeded random states.
"""
import numpy as np
import pytest

import oracle as O
from conftest import load_case
from paper_1802_05839_b200 import weather as W

pytestmark = pytest.mark.gpu

TOL = 0.0  # bitwise
LAYOUTS = ["ijk", "kij"]
KERNELS = ["auto", "fused_tma", "fused_pair", "fused_cell", "split"]  # auto: pair (IJK) / TMA


def cfg_of(d):
    return W.GridConfig(**d)


def run_device(cfg, steps, layout="ijk", kernel="auto", init_state=None, options=None):
    with W.Context(cfg, layout=layout, kernel=kernel) as ctx:
        for name, value in (options or {}).items():
            ctx.set_option(name, value)
        if init_state is None:
            ctx.init()
        else:
            for name, arr in init_state.items():
                ctx.upload(name, np.ascontiguousarray(arr))
        ctx.step(steps)
        return {n: ctx.download(n) for n in ("energy", "energy_u", "energy_surf", "energy_pbl")}


def available(cfg, layout, kernel):
    with W.Context(cfg, layout=layout) as ctx:
        try:
            ctx.set_kernel(kernel)
        except W.HftwError:
            return False
    return True


def assert_same(got, want, tag):
    for f in ("energy", "energy_u", "energy_surf", "energy_pbl"):
        a, b = got[f], want[f]
        assert a.shape == b.shape, (tag, f)
        bad = np.flatnonzero(a != b)
        assert bad.size == 0, f"{tag} {f}: {bad.size} cells differ, first {bad[:5]}, " \
                              f"max |d| {np.max(np.abs(a - b)):.3e}"


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("kernel", KERNELS)
def test_golden_cases(golden, layout, kernel):
    for name, case in golden["full_cases"].items():
        npz = load_case(name)
        if not available(cfg_of(case["grid"]), layout, kernel):
            continue
        init = None
        if case["initial"] != "reference_init":
            init = {f: npz["in_" + f] for f in ("energy", "energy_u", "energy_surf", "energy_pbl")}
        got = run_device(cfg_of(case["grid"]), case["steps"], layout, kernel, init)
        want = {f: npz["out_" + f] for f in ("energy", "energy_u", "energy_surf", "energy_pbl")}
        assert_same(got, want, f"{name}/{layout}/{kernel}")


@pytest.mark.parametrize("layout", LAYOUTS)
def test_auto_kernel_selected(layout):
    # AUTO: two-step passes (IJK, one domain, 56 <= nz <= 58: the compile-time row
    # shapes of 8 k-groups of 7-8 planes); the TMA kernel otherwise (fused_pair still
    # runs other nz on request)
    with W.Context(W.GridConfig(nx=100, ny=40, nz=58), layout=layout) as ctx:
        assert ctx.kernel == ("fused_pair" if layout == "ijk" else "fused_tma")
        assert ctx.launches_per_step == 1
    with W.Context(W.GridConfig(nx=100, ny=40, nz=56), layout=layout) as ctx:
        assert ctx.kernel == ("fused_pair" if layout == "ijk" else "fused_tma")
    with W.Context(W.GridConfig(nx=100, ny=40, nz=55), layout=layout) as ctx:
        assert ctx.kernel == "fused_tma"
        if layout == "ijk":
            ctx.set_kernel("fused_pair")


@pytest.mark.parametrize("shape", [(100, 37, 58), (130, 5, 3), (64, 64, 2), (2, 2, 2),
                                   (65, 3, 9), (33, 200, 17), (7, 9, 200), (5, 6, 300),
                                   (129, 2, 64)])
@pytest.mark.parametrize("layout", LAYOUTS)
def test_random_states_vs_oracle(coracle, shape, layout):
    nx, ny, nz = shape
    rng = np.random.default_rng(nx * 1000 + ny * 10 + nz)
    cfg = W.GridConfig(nx=nx, ny=ny, nz=nz, diffusion_velocity=float(rng.uniform(0, 1 / 6)),
                       radiation_intensity=float(rng.uniform(-0.5, 0.5)),
                       transfer_velocity=float(rng.uniform(0, 0.1)),
                       surf_energy=float(rng.uniform(250, 350)), pbl_energy=200.0)
    g = O.grid_from(cfg)
    n3, n2 = O.shapes(g)
    s0 = O.State(rng.uniform(150, 350, n3), rng.uniform(150, 350, n3),
                 rng.uniform(150, 350, n2), rng.uniform(150, 350, n2))
    want = coracle.steps(g, s0, 3).fields()
    for kernel in ("auto", "fused_tma", "fused_pair", "fused_cell", "split"):
        if not available(cfg, layout, kernel):
            continue  # e.g. nz beyond the TMA slab ring: AUTO covers the fallback
        got = run_device(cfg, 3, layout, kernel, s0.fields())
        assert_same(got, want, f"{shape}/{layout}/{kernel}")


@pytest.mark.parametrize("layout", LAYOUTS)
def test_stencil_config_hash(golden, coracle, layout):
    h = golden["hashes"]["256x256x64_s10"]
    got = run_device(cfg_of(h["grid"]), h["steps"], layout)
    for f, v in h["fnv1a64"].items():
        assert coracle.fnv(got[f]) == v, f


def test_asuca_hash_and_phases(golden, coracle):
    """BASELINE's full size 1581x1301x58: bitwise via the reference's hashes."""
    h = golden["hashes"]["1581x1301x58_s2"]
    cfg = cfg_of(h["grid"])
    for layout in LAYOUTS:
        got = run_device(cfg, h["steps"], layout)
        for f, v in h["fnv1a64"].items():
            assert coracle.fnv(got[f]) == v, (layout, f)
    # physics alone (weather.cpp:118-128) from the initial condition, both mappings
    ph = golden["hashes"]["physics_1581x1301x58_from_init"]["fnv1a64"]["e"]
    for layout in LAYOUTS:
        for mode in (0, 1):
            with W.Context(cfg, layout=layout) as ctx:
                ctx.init()
                ctx.physics(mode)
                assert coracle.fnv(ctx.download("energy")) == ph, (layout, mode)


def test_diffusion_only_hash(golden, coracle):
    d = golden["hashes"]["diffuse_256x256x64_from_s1"]
    cfg = cfg_of(d["grid"])
    for layout in LAYOUTS:
        with W.Context(cfg, layout=layout) as ctx:
            ctx.init()
            ctx.step(1)
            ctx.diffuse()
            assert coracle.fnv(ctx.download("energy")) == d["fnv1a64"]["u"], layout


@pytest.mark.parametrize("shape", [(256, 256, 64), (37, 20, 17), (2, 2, 2), (70, 9, 33)])
def test_diffusion_sweep_vs_oracle(coracle, shape):
    """A diffusion-only sweep (weather.cpp:130-168 on the post-physics field) of a
    random state: bitwise."""
    nx, ny, nz = shape
    rng = np.random.default_rng(nx + 7 * ny + 31 * nz)
    cfg = W.GridConfig(nx=nx, ny=ny, nz=nz, diffusion_velocity=float(rng.uniform(0, 1 / 6)))
    g = O.grid_from(cfg)
    n3, n2 = O.shapes(g)
    e = rng.uniform(150, 350, n3)
    want = coracle.diffuse(g, e.copy())
    with W.Context(cfg) as ctx:
        ctx.upload("energy", e)
        ctx.diffuse()
        got = ctx.download("energy")
    bad = np.flatnonzero(got.view(np.uint64) != want.view(np.uint64))
    assert bad.size == 0, (shape, bad[:5])


@pytest.mark.parametrize("shape,n", [((256, 256, 64), 2), ((256, 256, 64), 7), ((37, 20, 17), 4),
                                     ((70, 9, 33), 3), ((130, 200, 8), 5)])
def test_diffusion_sweeps_vs_oracle(coracle, shape, n):
    """n diffusion-only sweeps in one call (hftw_diffuse_steps: one multi-sweep
    launch where the grid allows it) = n single sweeps of the oracle, bitwise; energy_u
    is the last sweep's input (the swap)."""
    nx, ny, nz = shape
    rng = np.random.default_rng(nx + 7 * ny + 31 * nz + n)
    cfg = W.GridConfig(nx=nx, ny=ny, nz=nz, diffusion_velocity=float(rng.uniform(0, 1 / 6)))
    g = O.grid_from(cfg)
    n3, _ = O.shapes(g)
    e = rng.uniform(150, 350, n3)
    want, prev = e.copy(), None
    for _ in range(n):
        prev, want = want, coracle.diffuse(g, want.copy())
    with W.Context(cfg) as ctx:
        ctx.upload("energy", e)
        ctx.diffuse(n)
        got, got_u = ctx.download("energy"), ctx.download("energy_u")
    for a, b, f in ((got, want, "energy"), (got_u, prev, "energy_u")):
        bad = np.flatnonzero(a.view(np.uint64) != b.view(np.uint64))
        assert bad.size == 0, (shape, n, f, bad[:5])


def test_diffuse_steps_and_reverse_option_errors():
    """Argument checks of hftw_diffuse_steps and HFTW_OPT_REVERSE (loud, no state change)."""
    cfg = W.GridConfig(nx=40, ny=30, nz=12)
    with W.Context(cfg) as ctx:
        ctx.init()
        before = ctx.download("energy")
        with pytest.raises(W.HftwError):
            ctx.diffuse(-1)
        with pytest.raises(W.HftwError):
            ctx.set_option("reverse", 2)
        ctx.diffuse(0)
        assert np.array_equal(ctx.download("energy"), before)
    with W.Context(W.GridConfig(nx=40, ny=30, nz=12), px=2, py=1, devices=[0, 0]) as g:
        g.init()
        with pytest.raises(W.HftwError):
            g.diffuse(3)  # diffusion-only sweeps are single-domain


def test_energy_u_observability(coracle):
    """energy_u after a step is the post-physics, pre-diffusion field
    (weather.cpp:118-128 in place, then the swap at :170)."""
    cfg = W.GridConfig(nx=70, ny=33, nz=12)
    g = O.grid_from(cfg)
    with W.Context(cfg) as ctx:
        ctx.init()
        assert np.all(ctx.download("energy_u") == 0.0)  # weather.cpp:82
        ctx.step(2)
        ref2 = coracle.run_reference(g, 2)
        assert np.array_equal(ctx.download("energy_u"), ref2.energy_u)
        # downloading energy_u materialises it; stepping on must be unaffected
        ctx.step(3)
        ref5 = coracle.run_reference(g, 5)
        assert np.array_equal(ctx.download("energy"), ref5.energy)
        assert np.array_equal(ctx.download("energy_u"), ref5.energy_u)
        # new boundary fields must not leak into the previous step's energy_u
        ctx.step(1)
        ref6 = coracle.run_reference(g, 6)
        ctx.upload("energy_surf", np.full_like(ref6.energy_surf, 123.0))
        assert np.array_equal(ctx.download("energy_u"), ref6.energy_u)


def test_split_calls_equal_one_call(coracle):
    cfg = W.GridConfig(nx=90, ny=21, nz=7)
    with W.Context(cfg) as a, W.Context(cfg) as b:
        a.init()
        b.init()
        a.step(5)
        for n in (2, 1, 2):
            b.step(n)
        for f in ("energy", "energy_u"):
            assert np.array_equal(a.download(f), b.download(f))


def test_reference_api_mirror(coracle):
    cfg = W.GridConfig(nx=12, ny=9, nz=5)
    g = O.grid_from(cfg)
    st = W.run_reference(cfg, 4)
    ref = coracle.run_reference(g, 4)
    r = W.compare_fields(st, W.SimState(*(W.ArrayObject(a.bounds, b) for a, b in zip(
        st.named().values(), ref.fields().values()))))
    assert r.shape_ok and r.pass_(TOL)
    s2 = W.SimState.allocate(cfg)
    W.reference_init(cfg, s2)
    W.reference_step(cfg, s2)
    assert np.array_equal(s2.energy.data, coracle.run_reference(g, 1).energy)


def test_reference_step_loop_two_grids(coracle):
    """reference_step in a loop, alternating two grids: the cached per-thread context
    follows the config; bitwise against the oracle."""
    cfgs = [W.GridConfig(nx=21, ny=13, nz=7), W.GridConfig(nx=30, ny=11, nz=9,
                                                           radiation_intensity=-0.3)]
    sts = []
    for cfg in cfgs:
        st = W.SimState.allocate(cfg)
        W.reference_init(cfg, st)
        sts.append(st)
    for _ in range(3):
        for cfg, st in zip(cfgs, sts):
            W.reference_step(cfg, st)
    W.release_cached_context()
    for cfg, st in zip(cfgs, sts):
        want = coracle.run_reference(O.grid_from(cfg), 3)
        assert np.array_equal(st.energy.data, want.energy)
        assert np.array_equal(st.energy_u.data, want.energy_u)


def test_reference_step_pinned_state(coracle):
    """reference_step on page-locked SimState buffers (weather.pinned): bitwise, and the
    buffers are written in place."""
    cfg = W.GridConfig(nx=40, ny=25, nz=12, diffusion_velocity=0.15)
    st = W.SimState.allocate(cfg)
    W.reference_init(cfg, st)
    with W.pinned(st):
        e0, eu0 = st.energy.data, st.energy_u.data
        for _ in range(2):
            W.reference_step(cfg, st)
        assert st.energy.data is e0 and st.energy_u.data is eu0
    W.release_cached_context()
    want = coracle.run_reference(O.grid_from(cfg), 2)
    assert np.array_equal(st.energy.data, want.energy)
    assert np.array_equal(st.energy_u.data, want.energy_u)


def test_errors_are_loud():
    with pytest.raises(W.HftwError):
        with W.Context(W.GridConfig(nz=300)) as ctx:
            ctx.set_kernel("fused_tma")  # nz > 256 exceeds the TMA box
    with W.Context(W.GridConfig()) as ctx:
        with pytest.raises(W.HftwError):
            ctx.step(-1)


@pytest.mark.parametrize("shape", [(100, 37, 58), (130, 300, 9), (2, 2, 2), (65, 3, 9),
                                   (129, 700, 4), (5, 6, 300)])
@pytest.mark.parametrize("layout", LAYOUTS)
def test_step_host_pipeline_vs_oracle(coracle, shape, layout):
    """hftw_step_host (row-block H2D / step / D2H pipeline) is one
    reference_step on a host state: bitwise, in place and out of place, and the
    context is left holding the stepped state."""
    nx, ny, nz = shape
    rng = np.random.default_rng(7 * nx + 11 * ny + nz)
    cfg = W.GridConfig(nx=nx, ny=ny, nz=nz, diffusion_velocity=float(rng.uniform(0, 1 / 6)),
                       radiation_intensity=float(rng.uniform(-0.5, 0.5)),
                       transfer_velocity=float(rng.uniform(0, 0.1)))
    g = O.grid_from(cfg)
    n3, n2 = O.shapes(g)
    s0 = O.State(rng.uniform(150, 350, n3), rng.uniform(150, 350, n3),
                 rng.uniform(150, 350, n2), rng.uniform(150, 350, n2))
    want1 = coracle.steps(g, s0, 1).fields()
    want2 = coracle.steps(g, s0, 2).fields()
    with W.Context(cfg, layout=layout) as ctx:
        e, eu = ctx.step_host(s0.energy.copy(), s0.energy_surf.copy(), s0.energy_pbl.copy())
        assert np.array_equal(e, want1["energy"]) and np.array_equal(eu, want1["energy_u"])
        # in place, from the stepped state: a second reference_step
        e2 = e.copy()
        ctx.step_host(e2, s0.energy_surf.copy(), s0.energy_pbl.copy(), e2, eu)
        assert np.array_equal(e2, want2["energy"]) and np.array_equal(eu, want2["energy_u"])
        got = {n: ctx.download(n) for n in ("energy", "energy_u", "energy_surf", "energy_pbl")}
    assert_same(got, want2, f"{shape}/{layout}/context-after-step_host")


def test_step_host_after_device_steps(coracle):
    """Queued device work on the context stream is ordered before the pipeline."""
    cfg = W.GridConfig(nx=300, ny=250, nz=58)
    g = O.grid_from(cfg)
    ref = coracle.run_reference(g, 1)
    with W.Context(cfg) as ctx:
        ctx.init()
        ctx.step(3)  # asynchronous; step_host must not race it
        e, eu = ctx.step_host(ref.energy.copy(), ref.energy_surf.copy(), ref.energy_pbl.copy())
    want = coracle.run_reference(g, 2)
    assert np.array_equal(e, want.energy) and np.array_equal(eu, want.energy_u)


@pytest.mark.parametrize("shape", [(100, 37, 58), (64, 64, 2), (65, 3, 9), (2, 2, 2), (33, 200, 17),
                                   (129, 2, 64), (128, 70, 58), (191, 97, 31), (1, 1, 1),
                                   # k-group splits with compile-time row shapes (8
                                   # groups of 7-8 planes: nz 56-58), other splits (the
                                   # generic path), and the first nz past the smem budget
                                   (70, 45, 56), (61, 33, 57), (90, 25, 50), (77, 31, 53),
                                   (64, 40, 55), (95, 20, 59)])
@pytest.mark.parametrize("steps", [3, 4, 5, 8])
def test_pair_kernel_vs_oracle(coracle, shape, steps):
    """Two steps per pass (intermediate field on chip): bitwise against the oracle on
    ragged grids (edge strips with and without the far partner column, one-strip and
    one-chunk grids, nz = 2) for odd and even step counts."""
    nx, ny, nz = shape
    if nx < 2 or ny < 2 or nz < 2:
        pytest.skip("below the reference's minimum extents")
    rng = np.random.default_rng(31 * nx + 7 * ny + nz + steps)
    cfg = W.GridConfig(nx=nx, ny=ny, nz=nz, diffusion_velocity=float(rng.uniform(0, 1 / 6)),
                       radiation_intensity=float(rng.uniform(-0.5, 0.5)),
                       transfer_velocity=float(rng.uniform(0, 0.1)))
    g = O.grid_from(cfg)
    n3, n2 = O.shapes(g)
    s0 = O.State(rng.uniform(150, 350, n3), rng.uniform(150, 350, n3),
                 rng.uniform(150, 350, n2), rng.uniform(150, 350, n2))
    want = coracle.steps(g, s0, steps).fields()
    if nz > 58:
        # three intermediate row buffers + a 4-deep slab ring for two CTAs per SM
        # exceed shared memory: the pair kernel is refused and AUTO falls back to
        # the single-step kernel
        assert not available(cfg, "ijk", "fused_pair")
        got = run_device(cfg, steps, "ijk", "auto", s0.fields())
    else:
        got = run_device(cfg, steps, "ijk", "fused_pair", s0.fields())
    assert_same(got, want, f"{shape}/pair/{steps}")


def test_pair_kernel_is_auto_and_hash(golden, coracle):
    h = golden["hashes"]["1581x1301x58_s2"]
    cfg = cfg_of(h["grid"])
    # 256x256x64 x 10 steps (AUTO: nz = 64 is beyond the pair kernel's smem budget)
    h = golden["hashes"]["256x256x64_s10"]
    got = run_device(cfg_of(h["grid"]), h["steps"], "ijk", "auto")
    for f, v in h["fnv1a64"].items():
        assert coracle.fnv(got[f]) == v, f


@pytest.mark.parametrize("steps", [7, 20])
def test_headline_run_vs_reference_hash(golden, coracle, steps):
    """The bench's exact run on one GPU: init + hftw_step(steps) at 1581x1301x58 through
    AUTO (pair passes, the field post-physics between them; 7 steps end with a single
    step), bitwise against the unmodified reference's run_reference hashes -- energy_u
    included (recomputed from a post-physics partner after 20 steps)."""
    h = golden["hashes"][f"1581x1301x58_s{steps}"]
    got = run_device(cfg_of(h["grid"]), steps, "ijk", "auto")
    for f, v in h["fnv1a64"].items():
        assert coracle.fnv(got[f]) == v, (steps, f)


@pytest.mark.parametrize("shape,kernel", [((150, 97, 58), "auto"), ((133, 61, 51), "auto"),
                                          ((150, 97, 58), "fused_tma"), ((70, 200, 17), "fused_tma")])
def test_reverse_unit_order_bitwise(coracle, shape, kernel):
    """HFTW_OPT_REVERSE (the work units handed out last chunk first; the analogue of the
    reference emulator's launch-order reversal, interpreter.hpp:38-45) gives the same
    bits: no result depends on the order in which CTAs take their units."""
    nx, ny, nz = shape
    cfg = W.GridConfig(nx=nx, ny=ny, nz=nz, diffusion_velocity=0.13)
    rng = np.random.default_rng(nx + nz)
    g = O.grid_from(cfg)
    n3, n2 = O.shapes(g)
    s0 = O.State(rng.uniform(150, 350, n3), rng.uniform(150, 350, n3),
                 rng.uniform(150, 350, n2), rng.uniform(150, 350, n2))
    want = coracle.steps(g, s0, 6).fields()
    got = run_device(cfg, 6, "ijk", kernel, s0.fields(), options={"reverse": 1, "multistep": -1})
    assert_same(got, want, f"{shape}/{kernel}/reverse")


def test_pair_kernel_asuca_vs_oracle(coracle):
    """BASELINE's full size, 5 steps = 2 pairs + 1 single step, bitwise."""
    cfg = W.GridConfig(nx=1581, ny=1301, nz=58)
    want = coracle.run_reference(O.grid_from(cfg), 5)
    with W.Context(cfg, kernel="fused_pair") as ctx:
        ctx.init()
        ctx.step(5)
        for f in ("energy", "energy_u"):
            assert np.array_equal(ctx.download(f), getattr(want, f)), f


@pytest.mark.parametrize("shape,steps", [((200, 300, 20), 13), ((130, 70, 58), 7),
                                         ((64, 64, 2), 5), ((65, 129, 9), 4), ((3, 200, 5), 6),
                                         ((129, 65, 58), 2)])
def test_multi_step_launch_vs_oracle(coracle, shape, steps):
    """hftw_step(n >= 2) runs all n steps in one persistent launch (per-chunk
    dependency counters, ghost-row tasks): bitwise against the oracle, including
    grids of one chunk (first == last) and a short last chunk, and a second call
    on the same context (the counters re-arm themselves)."""
    nx, ny, nz = shape
    rng = np.random.default_rng(3 * nx + 5 * ny + nz + steps)
    cfg = W.GridConfig(nx=nx, ny=ny, nz=nz, diffusion_velocity=float(rng.uniform(0, 1 / 6)),
                       radiation_intensity=float(rng.uniform(-0.5, 0.5)),
                       transfer_velocity=float(rng.uniform(0, 0.1)))
    g = O.grid_from(cfg)
    n3, n2 = O.shapes(g)
    s0 = O.State(rng.uniform(150, 350, n3), rng.uniform(150, 350, n3),
                 rng.uniform(150, 350, n2), rng.uniform(150, 350, n2))
    want = coracle.steps(g, s0, 2 * steps).fields()
    with W.Context(cfg, kernel="fused_tma") as ctx:
        ctx.set_option("multistep", 1)
        for name, arr in s0.fields().items():
            ctx.upload(name, np.ascontiguousarray(arr))
        ctx.set_timing(True)
        ctx.step(steps)
        ctx.step(steps)
        ms, n, st = ctx.timing(2)
        assert n == 2 and st == 2 * steps  # both calls were single multi-step launches
        got = {f: ctx.download(f) for f in ("energy", "energy_u", "energy_surf", "energy_pbl")}
    assert_same(got, want, f"{shape}/wave/{steps}")


@pytest.mark.parametrize("kernel,steps,wave", [("auto", 7, 0), ("fused_tma", 6, 0),
                                               ("fused_tma", 6, 1)])
def test_asuca_random_state_non_default_constants(coracle, kernel, steps, wave):
    """BASELINE's full size from a random state with non-default constants: the
    pair passes (auto), one launch per step (fused_tma) and the multi-step launch
    (fused_tma, multistep=1: at this size AUTO prefers one launch per step), bitwise."""
    rng = np.random.default_rng(1802)
    cfg = W.GridConfig(nx=1581, ny=1301, nz=58, diffusion_velocity=0.1375,
                       radiation_intensity=-0.21, transfer_velocity=0.047,
                       surf_energy=312.5, pbl_energy=187.25)
    g = O.grid_from(cfg)
    n3, n2 = O.shapes(g)
    s0 = O.State(rng.uniform(150, 350, n3), rng.uniform(150, 350, n3),
                 rng.uniform(150, 350, n2), rng.uniform(150, 350, n2))
    want = coracle.steps(g, s0, steps).fields()
    got = run_device(cfg, steps, "ijk", kernel, s0.fields(), {"multistep": wave})
    assert_same(got, want, f"asuca/{kernel}/{steps}")


@pytest.mark.parametrize("shape", [(100, 37, 58), (33, 20, 37), (17, 9, 2), (40, 6, 31),
                                   (64, 64, 33)])
@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("mode", [0, 1])
def test_physics_phase_vs_oracle(coracle, shape, layout, mode):
    """Column physics alone (weather.cpp:118-128), every mapping and layout, odd
    nz (KIJ column padding) and nz < 32 (the KIJ warp kernel): bitwise."""
    nx, ny, nz = shape
    rng = np.random.default_rng(nx + 100 * ny + 10000 * nz)
    cfg = W.GridConfig(nx=nx, ny=ny, nz=nz, radiation_intensity=float(rng.uniform(-1, 1)),
                       transfer_velocity=float(rng.uniform(0, 0.2)))
    g = O.grid_from(cfg)
    n3, n2 = O.shapes(g)
    e = rng.uniform(150, 350, n3)
    sf, pb = rng.uniform(150, 350, n2), rng.uniform(150, 350, n2)
    want = coracle.physics(g, e, sf, pb)
    with W.Context(cfg, layout=layout) as ctx:
        ctx.upload("energy", np.ascontiguousarray(e))
        ctx.upload("energy_surf", np.ascontiguousarray(sf))
        ctx.upload("energy_pbl", np.ascontiguousarray(pb))
        ctx.physics(mode)
        got = ctx.download("energy")
    bad = np.flatnonzero(got != want)
    assert bad.size == 0, (shape, layout, mode, bad[:5])


def test_concurrent_contexts_vs_oracle(coracle):
    """Two contexts on their own streams run pair passes and multi-step launches at the
    same time (each persistent grid takes whatever SMs it gets; the work-unit counters
    are per context): both bitwise."""
    cases = []
    for seed, shape, kernel in ((11, (300, 210, 58), "auto"), (12, (257, 190, 40), "fused_tma")):
        rng = np.random.default_rng(seed)
        nx, ny, nz = shape
        cfg = W.GridConfig(nx=nx, ny=ny, nz=nz, diffusion_velocity=float(rng.uniform(0, 1 / 6)),
                           radiation_intensity=float(rng.uniform(-0.5, 0.5)),
                           transfer_velocity=float(rng.uniform(0, 0.1)))
        g = O.grid_from(cfg)
        n3, n2 = O.shapes(g)
        s0 = O.State(rng.uniform(150, 350, n3), rng.uniform(150, 350, n3),
                     rng.uniform(150, 350, n2), rng.uniform(150, 350, n2))
        cases.append((cfg, kernel, s0, coracle.steps(g, s0, 9).fields()))
    ctxs = [W.Context(cfg, kernel=kernel) for cfg, kernel, _, _ in cases]
    try:
        for ctx, (_, _, s0, _) in zip(ctxs, cases):
            for name, arr in s0.fields().items():
                ctx.upload(name, np.ascontiguousarray(arr))
        for _ in range(3):          # interleaved, asynchronous: the launches overlap
            for ctx in ctxs:
                ctx.step(3)
        for ctx, (cfg, kernel, _, want) in zip(ctxs, cases):
            got = {n: ctx.download(n) for n in ("energy", "energy_u", "energy_surf", "energy_pbl")}
            assert_same(got, want, f"concurrent/{kernel}")
    finally:
        for ctx in ctxs:
            ctx.close()


@pytest.mark.parametrize("calls", [[4], [2, 2], [6, 1, 2], [3, 4], [2, 1, 1, 2]])
def test_even_calls_are_pair_passes_with_energy_u(coracle, calls):
    """An even step count runs as pair passes only (energy_u, the physics of the
    step before the last, is recomputed from the ping-pong partner when it is
    read); odd counts end with one single step.  Interleaved with uploads,
    downloads and boundary-field changes, every observable field stays bitwise
    the oracle's."""
    cfg = W.GridConfig(nx=150, ny=37, nz=58, diffusion_velocity=0.14,
                       radiation_intensity=0.21, transfer_velocity=0.03)
    g = O.grid_from(cfg)
    rng = np.random.default_rng(sum(calls) * 7 + len(calls))
    n3, n2 = O.shapes(g)
    s = O.State(rng.uniform(150, 350, n3), rng.uniform(150, 350, n3),
                rng.uniform(150, 350, n2), rng.uniform(150, 350, n2))
    with W.Context(cfg) as ctx:
        assert ctx.kernel == "fused_pair"
        for f, a in s.fields().items():
            ctx.upload(f, np.ascontiguousarray(a))
        for n in calls:
            ctx.set_timing(True)
            ctx.step(n)
            _, singles, _ = ctx.timing(0)
            _, pairs, _ = ctx.timing(1)
            _, multi, _ = ctx.timing(2)
            assert pairs == n // 2 and singles + multi == n % 2, (n, pairs, singles, multi)
            s = coracle.steps(g, s, n)
            assert_same({f: ctx.download(f) for f in ("energy", "energy_u", "energy_surf",
                                                      "energy_pbl")}, s.fields(), f"{calls}/{n}")
        # the boundary field changes while energy_u is still pending (not read since
        # the pass): it keeps the values of the steps that produced it
        ctx.step(2)
        s = coracle.steps(g, s, 2)
        sf = rng.uniform(150, 350, n2)
        ctx.upload("energy_surf", sf)
        assert np.array_equal(ctx.download("energy_u"), s.energy_u)
        s.energy_surf = sf
        ctx.step(2)
        s = coracle.steps(g, s, 2)
        assert np.array_equal(ctx.download("energy_u"), s.energy_u)
        assert np.array_equal(ctx.download("energy"), s.energy)
