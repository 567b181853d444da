"""The output path: hftw_simulate runs the corpus
driver's time loop (fixtures/corpus/simple_weather.h90:74-108 via
weather.cpp:364-376) on the device and hands every write_data output to a
host callback while later steps run.

Pinned against the reference: the number of write_data calls of the
interpreted original corpus (tests/golden/golden.json, corpus_write_data) and
the oracle state at every output time, bitwise.
"""
import math
import os

import numpy as np
import pytest

import oracle as O
from paper_1802_05839_b200 import weather as W


def driver_schedule(steps, dt, odt):
    """(time, steps done before the write) of each write_data call, following
    simple_weather.h90:91-107 with drive()'s end_time = (steps - 0.5) * dt and
    modulo(a, p) = a - floor(a / p) * p (interpreter.cpp:109)."""
    end = (steps - 0.5) * dt
    time, done, out = 0.0, 0, []
    while True:
        a = time + 0.001
        if a - math.floor(a / odt) * odt < 0.01:
            out.append((time, done))
        done += 1
        time = time + dt
        if time > end:
            return out, done


def test_schedule_matches_reference_write_count(golden):
    for case in golden["corpus_write_data"]:
        assert case["ok"]
        sched, done = driver_schedule(case["steps"], case["timestep"], case["output_timestep"])
        assert len(sched) == case["write_data_calls"], case
        assert done == case["steps"]


@pytest.mark.gpu
@pytest.mark.parametrize("layout", ["ijk", "kij"])
def test_simulate_outputs_bitwise(golden, coracle, layout):
    for case in golden["corpus_write_data"]:
        steps, dt, odt = case["steps"], case["timestep"], case["output_timestep"]
        cfg = W.GridConfig(nx=23, ny=17, nz=9, timestep=dt, output_timestep=odt)
        g = O.grid_from(cfg)
        got = []
        with W.Context(cfg, layout=layout) as ctx:
            ctx.init()
            nsteps, nwrites = ctx.simulate(0.0, (steps - 0.5) * dt, dt, odt,
                                           lambda tag, t, f: got.append((tag, t, f.copy())))
            final = ctx.download("energy")
        sched, done = driver_schedule(steps, dt, odt)
        assert nsteps == done == steps and nwrites == len(sched) == case["write_data_calls"]
        assert [t for _, t, _ in got] == [t for t, _ in sched]
        for (tag, t, f), (_, n) in zip(got, sched):
            assert tag == "energy"
            assert np.array_equal(f, coracle.run_reference(g, n).energy), (layout, t, n)
        assert np.array_equal(final, coracle.run_reference(g, steps).energy)


@pytest.mark.gpu
def test_dump_writer_round_trip(tmp_path, coracle):
    cfg = W.GridConfig(nx=6, ny=5, nz=4)
    with W.Context(cfg) as ctx:
        ctx.init()
        ctx.simulate(0.0, 10.5 * cfg.timestep, cfg.timestep, cfg.output_timestep,
                     W.dump_writer(str(tmp_path), cfg))
    files = sorted(os.listdir(tmp_path))
    assert len(files) == 2  # t = 0 and t ~ 1.0
    d = W.Diagnostics()
    with open(tmp_path / files[1]) as f:
        a = W.read_field(f, d)
    assert d.ok()
    assert np.array_equal(a.data, coracle.run_reference(O.grid_from(cfg), 10).energy)


@pytest.mark.gpu
def test_simulate_with_pair_passes(coracle):
    """nz = 58: the steps between outputs run as two-step passes (+ a trailing
    single step); every output and the final state bitwise."""
    dt, odt, steps = 0.1, 1.0, 37
    cfg = W.GridConfig(nx=70, ny=45, nz=58, timestep=dt, output_timestep=odt)
    g = O.grid_from(cfg)
    got = []
    with W.Context(cfg) as ctx:
        assert ctx.kernel == "fused_pair"
        ctx.init()
        ctx.set_timing(True)
        nsteps, nwrites = ctx.simulate(0.0, (steps - 0.5) * dt, dt, odt,
                                       lambda tag, t, f: got.append((t, f.copy())))
        assert ctx.timing(1)[1] > 0  # pair passes were used between the outputs
        final = ctx.download("energy")
        final_u = ctx.download("energy_u")
    sched, done = driver_schedule(steps, dt, odt)
    assert nsteps == done and nwrites == len(sched)
    for (t, f), (ts, n) in zip(got, sched):
        assert t == ts
        assert np.array_equal(f, coracle.run_reference(g, n).energy), (t, n)
    ref = coracle.run_reference(g, steps)
    assert np.array_equal(final, ref.energy) and np.array_equal(final_u, ref.energy_u)
