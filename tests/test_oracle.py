"""Pin the C restatement (oracle/weather_oracle.c) before trusting it.

Against: the reference's own golden vectors (tests/golden, generated from the
unmodified reference by oracle/gen_golden.py), the FNV-1a-64 known answers in
SURVEY.md section 4, the known-answer tests of test_weather.cpp, and -- when
oracle/_ref was built -- the compiled reference itself on fresh random states.
"""
import os

import numpy as np
import pytest

import oracle as O
from conftest import load_case

SURVEY_HASHES = {  # SURVEY.md section 4, computed with the reference
    (16, 16, 8, 10): {"energy": "b6d253635cd2f075", "energy_u": "a691b1ada5e94676",
                      "energy_surf": "73fb33a4cb8c4683", "energy_pbl": "5e799303e18750c3"},
    (4, 4, 4, 3): {"energy": "e79150d0c8f2b694", "energy_u": "5dce58541e3d96f5"},
}


def grid_of(d):
    return O.make_grid(**d)


def state_from(npz, prefix):
    return O.State(*(np.ascontiguousarray(npz[prefix + k]) for k in
                     ("energy", "energy_u", "energy_surf", "energy_pbl")))


@pytest.mark.parametrize("key", sorted(SURVEY_HASHES))
def test_survey_known_answers(coracle, key):
    nx, ny, nz, steps = key
    s = coracle.run_reference(O.make_grid(nx, ny, nz), steps)
    for name, h in SURVEY_HASHES[key].items():
        assert coracle.fnv(s.fields()[name]) == h, name


def test_point_values(coracle):
    # e(8,8,4), e(0,0,1), e(17,17,8) after 10 steps
    g = O.make_grid()
    s = coracle.run_reference(g, 10)
    e = s.energy.reshape((18, 18, 8), order="F")
    assert e[8, 8, 3] == 278.70214522528039
    assert e[0, 0, 0] == 31.052001506692239
    assert e[17, 17, 7] == 19.192664641100563


def test_golden_full_cases(coracle, golden):
    for name, case in golden["full_cases"].items():
        g = grid_of(case["grid"])
        npz = load_case(name)
        s0 = coracle.init(g) if case["initial"] == "reference_init" else state_from(npz, "in_")
        got = coracle.steps(g, s0, case["steps"])
        for f, arr in got.fields().items():
            assert np.array_equal(arr, npz["out_" + f]), (name, f)
            assert coracle.fnv(arr) == case["fnv1a64"][f], (name, f)


@pytest.mark.parametrize("key", ["256x256x64_s10"])
def test_golden_hashes_mid(coracle, golden, key):
    h = golden["hashes"][key]
    s = coracle.run_reference(grid_of(h["grid"]), h["steps"])
    for f, v in h["fnv1a64"].items():
        assert coracle.fnv(s.fields()[f]) == v, f


def test_known_answer_identity(coracle):
    # test_weather.cpp:117-137
    g = O.make_grid(6, 4, 4, diffusion_velocity=0.0, radiation_intensity=0.0,
                    transfer_velocity=0.0)
    a, b = coracle.run_reference(g, 1), coracle.run_reference(g, 5)
    for x, y in zip(a.fields().values(), b.fields().values()):
        assert np.array_equal(x, y)
    assert np.array_equal(coracle.run_reference(g, 0).energy, b.energy)


def test_known_answer_radiation_only(coracle):
    # test_weather.cpp:139-151
    g = O.make_grid(4, 4, 4, diffusion_velocity=0.0, transfer_velocity=0.0)
    s0, s1 = coracle.run_reference(g, 0), coracle.run_reference(g, 1)
    assert np.array_equal(s1.energy, s0.energy + g.radiation_intensity)


def test_validate_matches_reference_rules(coracle):
    # test_weather.cpp:88-115
    assert coracle.validate(O.make_grid())[0]
    assert not coracle.validate(O.make_grid(diffusion_velocity=0.2))[0]
    assert coracle.validate(O.make_grid(diffusion_velocity=1.0 / 6.0))[0]
    assert not coracle.validate(O.make_grid(nx=1))[0]
    assert not coracle.validate(O.make_grid(timestep=0.0))[0]


def test_oracle_vs_compiled_reference_random(coracle, reforacle):
    rng = np.random.default_rng(7)
    for nx, ny, nz, steps in [(5, 4, 3, 3), (19, 11, 7, 4), (2, 9, 2, 5), (64, 3, 6, 2)]:
        g = O.make_grid(nx, ny, nz, diffusion_velocity=float(rng.uniform(0, 1 / 6)),
                        radiation_intensity=float(rng.uniform(-1, 1)),
                        transfer_velocity=float(rng.uniform(0, 0.2)))
        n3, n2 = O.shapes(g)
        s0 = O.State(rng.uniform(100, 400, n3), rng.uniform(100, 400, n3),
                     rng.uniform(100, 400, n2), rng.uniform(100, 400, n2))
        a, b = coracle.steps(g, s0, steps), reforacle.steps(g, s0, steps)
        for f in a.fields():
            assert np.array_equal(a.fields()[f], b.fields()[f]), (nx, ny, nz, f)


def test_golden_variants_agree(golden):
    # the interpreted corpus (original / emitted cpu / emitted gpu-emulated,
    # forward and reverse launch order) agreed bitwise with the native
    # reference when the fixtures were generated
    v = golden["variants_16x16x8_s10"]
    assert v and all(x["bitwise_equal_to_reference"] for x in v.values())


@pytest.mark.skipif(not os.path.isdir(O.CORPUS_DIR), reason="needs the reference corpus")
@pytest.mark.parametrize("variant", [2, 3])
@pytest.mark.parametrize("reverse", [False, True])
def test_emitted_variants_at_default_line_length(reforacle, variant, reverse):
    """the transpiled cpu / gpu-emulated corpus runs at the
    default max_line_length 132 once the storage macros are expanded before the
    line split (the reference splits first, pipeline.cpp:88 vs :103-113), bitwise
    equal to the native reference and with its write_data cadence."""
    g = O.make_grid()
    s, msg = reforacle.run_variant_expand_first(variant, g, 10, 132, reverse)
    assert s is not None, msg
    want = reforacle.run_reference(g, 10)
    for f, a in s.fields().items():
        assert np.array_equal(a, want.fields()[f]), f
    assert reforacle.last_write_calls == 1  # simple_weather.h90:93-95 at t = 0 (10 steps)
