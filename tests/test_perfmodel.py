"""The paper's performance model mirror, pinned to the reference's known
answers (/root/reference/proj/tests/test_perfmodel.cpp)."""
import math

import pytest

from paper_1802_05839_b200 import perfmodel as P


def m(name):
    hw = P.find_machine(name)
    assert hw is not None
    return hw


def test_arithmetic_intensity():  # test_perfmodel.cpp:21-25
    assert P.arithmetic_intensity(8, 8, 8) == 0.125
    assert P.arithmetic_intensity(16, 8, 8) == 0.25


def test_compute_bound_thresholds():  # :27-42
    assert P.compute_bound_threshold(m("tsubame2.5")).value == pytest.approx(6.080283353010626,
                                                                            rel=1e-12)
    assert P.compute_bound_threshold(m("reedbush-h")).value == pytest.approx(7.809371245494594,
                                                                            rel=1e-12)
    none = P.compute_bound_threshold(m("tsubame3.0"))
    assert not none.ok() and "P_D" in none.error


def test_speedup_rhs():  # :44-61
    assert P.speedup_rhs(m("tsubame2.5")).value == pytest.approx(5.398695370992215, rel=1e-12)
    assert P.speedup_rhs(m("reedbush-h")).value == pytest.approx(8.280750722845367, rel=1e-12)
    assert P.speedup_rhs(m("piz-daint")).value == pytest.approx(5.205184077754652, rel=1e-12)
    t20 = P.speedup_rhs(m("tsubame2.0"))
    assert not t20.ok() and "BW_H" in t20.error and "tsubame2.5" in t20.error


def test_feasibility():  # :63-76
    assert P.speedup_lhs(10, 4, 8) == 5.0
    assert math.isinf(P.speedup_lhs(10, 4, 0))
    c, f = P.feasibility(m("tsubame2.5"), 10, 4, 8)
    assert c.ok() and f["lhs"] == 5.0 and not f["feasible"]
    c, f = P.feasibility(m("tsubame2.5"), 10, 4, 0.5)
    assert f["feasible"]


@pytest.mark.parametrize("n,m_sa,single,expect", [  # :78-101 (Table 4 rows)
    (128, 4.0, True, 0.739398), (128, 10.0, True, 1.766574), (128, 4.0, False, 0.381974),
    (128, 10.0, False, 0.873014), (256, 4.0, True, 5.696728), (256, 10.0, True, 13.91414),
    (256, 4.0, False, 2.837336), (256, 10.0, False, 6.76566)])
def test_host_model_table4(n, m_sa, single, expect):
    c = P.cpu_model_time(m("tsubame2.5"), P.ModelParams(n, n, n, 100, 8.0, m_sa), single)
    assert c.ok() and c.value == pytest.approx(expect, rel=1e-5)


def test_host_model_missing_single_core():  # :103-111
    c = P.cpu_model_time(m("reedbush-h"), P.ModelParams(128, 128, 128, 100), True)
    assert not c.ok() and "BW_H1C" in c.error and "tsubame2.5" in c.error


def test_device_model():  # :113-144
    hw = m("tsubame2.5")
    p = P.ModelParams(128, 128, 128, 100, 8.0, 4.0, 4.0, 0.0)
    spot = P.gpu_model_time(hw, p)
    assert spot.value == pytest.approx(0.04706289492325856, rel=1e-12)
    assert P.gpu_model_time(hw, P.ModelParams(128, 128, 128, 0, 8.0, 4.0)).value == 0.0
    t1 = P.gpu_model_time(hw, P.ModelParams(128, 128, 128, 1, 8.0, 4.0)).value
    t17 = P.gpu_model_time(hw, P.ModelParams(128, 128, 128, 17, 8.0, 4.0)).value
    assert t17 == pytest.approx(17 * t1, rel=1e-12)
    faster = P.replace(hw, bw_d=hw.bw_d * 2)
    assert P.gpu_model_time(faster, p).value < spot.value
    assert P.gpu_model_time(hw, P.replace(p, m_htod=8.0)).value > spot.value


def test_lookup_and_format():  # :146-156
    assert P.find_machine("no-such-machine") is None
    assert "tsubame2.5" in P.machine_names() and "piz-daint" in P.machine_names()
    assert "b200" in P.machine_names()
    assert P.format_sig4(5.398695) == "5.399"
    assert P.format_sig4(0.739398) == "0.7394"
    assert P.format_sig4(13.91414) == "13.91"


def test_b200_entry_is_measured():
    hw = m("b200")
    assert hw.bw_d and hw.bw_d > 1000
    r = P.b200_report(0.384)
    # the paper's "with cache" model (32 B/cell) at the measured copy bandwidth,
    # plus the random-access boundary term ny*nz*m_ra/RA_d (perfmodel.cpp:126-154)
    ra = (1301 * 58 * 4 / (hw.ra_d * 1e9)) if hw.ra_d else 0.0
    assert r["model_ms_per_step"]["m_sa=4"] == pytest.approx(
        (1581 * 1301 * 58 * 32 / (hw.bw_d * 1e9) + ra) * 1e3, rel=1e-3)
