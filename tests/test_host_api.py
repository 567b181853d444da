"""Host-side mirror of the reference API (compare, dump, unpermute) against the
reference's golden output and the compiled reference (test_weather.cpp:173-284)."""
import io
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_case
from paper_1802_05839_b200 import weather as W


def state_from_golden(name, cfg):
    npz = load_case(name)
    st = W.SimState.allocate(cfg)
    for f, arr in st.named().items():
        arr.data = np.ascontiguousarray(npz["out_" + f])
    return st


def test_dump_matches_reference_text_bitwise():
    cfg = W.GridConfig(nx=4, ny=4, nz=4)
    npz = load_case("brute_4x4x4_s3")  # shapes only; dump golden is the 2-step state
    import oracle as O
    c = O.COracle()
    s = c.run_reference(O.make_grid(4, 4, 4), 2)
    a = W.ArrayObject([(0, 5), (0, 5), (1, 4)], s.energy.copy())
    out = io.StringIO()
    W.dump_field(out, a)
    assert out.getvalue() == open(os.path.join(GOLDEN, "dump_energy_4x4x4_s2.txt")).read()
    b = W.ArrayObject([(0, 5), (0, 5)], s.energy_surf.copy())
    out = io.StringIO()
    W.dump_field(out, b)
    assert out.getvalue() == open(os.path.join(GOLDEN, "dump_surf_4x4x4_s2.txt")).read()
    del npz, cfg


def test_read_field_round_trip_and_truncation():
    # test_weather.cpp:203-247
    text = open(os.path.join(GOLDEN, "dump_energy_4x4x4_s2.txt")).read()
    d = W.Diagnostics()
    a = W.read_field(io.StringIO(text), d)
    assert d.ok() and a is not None and a.bounds == [(0, 5), (0, 5), (1, 4)]
    out = io.StringIO()
    W.dump_field(out, a)
    assert out.getvalue() == text
    surf = open(os.path.join(GOLDEN, "dump_surf_4x4x4_s2.txt")).read()
    b = W.read_field(io.StringIO(surf), W.Diagnostics())
    assert b.rank() == 3 and b.bounds[2] == (1, 1)
    d2 = W.Diagnostics()
    assert W.read_field(io.StringIO(surf[: len(surf) // 2]), d2) is None
    assert not d2.ok()


def test_compare_arrays_matches_reference(reforacle):
    rng = np.random.default_rng(3)
    for bounds in ([(0, 2), (1, 3)], [(0, 5), (0, 4), (1, 3)], [(-1, 7)]):
        a = W.ArrayObject(bounds)
        a.data = rng.uniform(-5, 5, a.size())
        b = a.copy()
        b.data[rng.integers(0, a.size())] += 1e-9
        r = W.compare_arrays(a, b)
        lo, hi = [x for x, _ in bounds], [y for _, y in bounds]
        ok, mx, nr, where = reforacle.compare_arrays(lo, hi, a.data, b.data)
        assert r.shape_ok == ok and r.max_abs == mx and r.where == where
        assert r.nrmse == pytest.approx(nr, rel=1e-12, abs=1e-300)


def test_compare_single_disturbance_located():
    # test_weather.cpp:173-201
    a = W.ArrayObject([(0, 2), (1, 3)])
    a.data[:] = 2.0
    b = a.copy()
    assert W.compare_arrays(a, b).max_abs == 0.0
    b.data[b.offset([2, 3])] += 1e-9
    r = W.compare_arrays(a, b)
    assert 1e-12 < r.max_abs < 1e-8 and r.where == [2, 3]
    c = W.ArrayObject([(0, 2), (1, 4)])
    assert not W.compare_arrays(a, c).shape_ok


def test_compare_fields_worst_field_wins():
    cfg = W.GridConfig()
    a = state_from_golden("fixture_16x16x8_s10", cfg)
    b = W.SimState(*(x.copy() for x in a.named().values()))
    r = W.compare_fields(a, b)
    assert r.shape_ok and r.max_abs == 0.0 and r.field == "energy" and r.pass_(0.0)
    b.energy_pbl.data[5] += 0.5
    b.energy.data[3] += 0.25
    r = W.compare_fields(a, b)
    assert r.field == "energy_pbl" and r.max_abs == 0.5 and not r.pass_(0.1)


def test_unpermute_matches_reference_semantics(reforacle):
    # test_weather.cpp:249-284
    raw = W.ArrayObject([(1, 2), (0, 2), (0, 1)])  # k, i, j
    for k in (1, 2):
        for i in range(3):
            for j in range(2):
                raw.data[raw.offset([k, i, j])] = 100.0 * i + 10.0 * j + k
    lg = W.unpermute_storage(raw, [3, 1, 2])
    assert lg.bounds == [(0, 2), (0, 1), (1, 2)]
    for i in range(3):
        for j in range(2):
            for k in (1, 2):
                assert lg.data[lg.offset([i, j, k])] == 100.0 * i + 10.0 * j + k
    ident = W.unpermute_storage(lg, [1, 2, 3])
    assert ident.bounds == lg.bounds and np.array_equal(ident.data, lg.data)
    rng = np.random.default_rng(5)
    for order in ([3, 1, 2], [2, 3, 1], [3, 2, 1], [1, 3, 2]):
        a = W.ArrayObject([(0, 3), (-1, 2), (1, 4)])
        a.data = rng.normal(size=a.size())
        mine = W.unpermute_storage(a, order)
        ref, olo, ohi = reforacle.unpermute([0, -1, 1], [3, 2, 4], order, a.data)
        assert mine.bounds == list(zip(olo, ohi))
        assert np.array_equal(mine.data, ref)
