"""Generate tests/golden/ from the UNMODIFIED reference -- TEST INFRASTRUCTURE.

Run in the build container (needs /root/reference and oracle/_ref, built by
``make -C oracle``):  ``python oracle/gen_golden.py``.

Every vector below comes from the reference's own entry points through
oracle/_ref/libhft_ref.so (hft::run_reference weather.cpp:173-178,
hft::reference_step weather.cpp:101-171, hft::dump_field weather.cpp:251-269,
hft::unpermute_storage weather.cpp:306-338, hft::run_variant
weather.cpp:439-476).  Phase-only hashes (physics alone, diffusion alone) have
no reference entry point; they come from the C restatement's phase functions,
which are pinned bitwise to the reference by the full-step vectors, and are
labelled ``source: oracle-phase``.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import oracle as O  # noqa: E402

GOLD = os.path.join(os.path.dirname(HERE), "tests", "golden")


def random_state(g, seed=1802, lo=150.0, hi=350.0):
    """U[lo, hi) state for all four fields (numpy PCG64, seed 1802)."""
    rng = np.random.default_rng(seed)
    n3, n2 = O.shapes(g)
    return O.State(rng.uniform(lo, hi, n3), rng.uniform(lo, hi, n3), rng.uniform(lo, hi, n2),
                   rng.uniform(lo, hi, n2))


def grid_dict(g):
    return {f: getattr(g, f) for f, _ in O.Grid._fields_}


def main():
    os.makedirs(GOLD, exist_ok=True)
    ref = O.RefOracle()
    c = O.COracle()
    cases = {}

    def save_full(name, g, steps, s_in, s_out, note):
        path = os.path.join(GOLD, name + ".npz")
        arrays = {("out_" + k): v for k, v in s_out.fields().items()}
        if s_in is not None:
            arrays.update({("in_" + k): v for k, v in s_in.fields().items()})
        np.savez_compressed(path, **arrays)
        cases[name] = {"grid": grid_dict(g), "steps": steps, "file": name + ".npz",
                       "initial": "reference_init" if s_in is None else "in_* arrays",
                       "fnv1a64": {k: c.fnv(v) for k, v in s_out.fields().items()},
                       "source": "reference", "note": note}

    # (1) the BASELINE fixture config: GridConfig{} 16x16x8, 10 steps
    g = O.make_grid()
    save_full("fixture_16x16x8_s10", g, 10, None, ref.run_reference(g, 10),
              "BASELINE configs[0]; SURVEY.md section 4 hashes")
    # (2) test_weather.cpp:153-171 brute-force case, 4x4x4 x 3 steps
    g = O.make_grid(4, 4, 4)
    save_full("brute_4x4x4_s3", g, 3, None, ref.run_reference(g, 3), "test_weather.cpp:153-171")
    # (3) test_weather.cpp:117-137 zero constants: identity after one step
    g = O.make_grid(6, 4, 4, diffusion_velocity=0.0, radiation_intensity=0.0,
                    transfer_velocity=0.0)
    save_full("identity_6x4x4_s5", g, 5, None, ref.run_reference(g, 5), "test_weather.cpp:117-137")
    # (4) random states on ragged grids with non-default constants
    for (nx, ny, nz, dv, steps) in [(17, 13, 5, 1.0 / 6.0, 4), (9, 7, 2, 0.05, 3),
                                    (33, 29, 11, 0.1, 6), (2, 2, 2, 0.1, 3), (40, 3, 3, 0.125, 2)]:
        g = O.make_grid(nx, ny, nz, diffusion_velocity=dv, radiation_intensity=0.37,
                        transfer_velocity=0.013, surf_energy=301.5, pbl_energy=211.25)
        s0 = random_state(g)
        save_full(f"random_{nx}x{ny}x{nz}_s{steps}", g, steps, s0, ref.steps(g, s0, steps),
                  "U[150,350) all four fields, numpy default_rng(1802)")

    # (5) hashes at the BASELINE sizes (reference, full step)
    hashes = {}
    #     ASUCA x 20 / x 7: the default bench run and an odd count (pair passes
    #     plus a single step); 3162x5204x58 x 5: BASELINE config 5's weak-scaling
    #     grid (8 x ASUCA, ~31 GB of host memory here)
    for (nx, ny, nz, steps) in [(256, 256, 64, 10), (1581, 1301, 58, 2), (1581, 1301, 58, 7),
                                (1581, 1301, 58, 20), (3162, 5204, 58, 5)]:
        g = O.make_grid(nx, ny, nz)
        s = ref.run_reference(g, steps)
        hashes[f"{nx}x{ny}x{nz}_s{steps}"] = {
            "grid": grid_dict(g), "steps": steps, "source": "reference",
            "fnv1a64": {k: c.fnv(v) for k, v in s.fields().items()},
            "sum_energy": float(np.sum(s.energy))}
        del s
        if nx == 256:
            # stencil-only config: diffusion of (init + 1 step) energy
            s1 = ref.run_reference(g, 1)
            hashes["diffuse_256x256x64_from_s1"] = {
                "grid": grid_dict(g), "source": "oracle-phase (wo_diffuse)",
                "fnv1a64": {"u": c.fnv(c.diffuse(g, s1.energy))}}
        if nx == 1581:
            s0 = ref.run_reference(g, 0)
            hashes["physics_1581x1301x58_from_init"] = {
                "grid": grid_dict(g), "source": "oracle-phase (wo_physics)",
                "fnv1a64": {"e": c.fnv(c.physics(g, s0.energy, s0.energy_surf, s0.energy_pbl))}}

    # (6) dump format (weather.cpp:251-269) for the 4x4x4 x 2 state
    #     through oracle/_ref/ref_tool: iostream formatting must run in a
    #     plain C++ process (inside Python the reference's integer output
    #     comes out empty)
    tool = os.path.join(HERE, "_ref", "ref_tool")
    for field, fname in (("energy", "dump_energy_4x4x4_s2.txt"),
                         ("energy_surf", "dump_surf_4x4x4_s2.txt")):
        text = subprocess.run([tool, "dump", "4", "4", "4", "2", field], check=True,
                              capture_output=True, text=True).stdout
        with open(os.path.join(GOLD, fname), "w") as f:
            f.write(text)

    # (7) secondary oracles: interpreted corpus variants agree with the native one
    g = O.make_grid()
    nat = ref.run_reference(g, 10)
    variants = {}
    for v, name, mll in [(1, "original", 0), (2, "cpu", 268), (3, "gpu-emulated", 268)]:
        for rev in (False, True):
            s, msg = ref.run_variant(v, g, 10, mll, rev)
            same = s is not None and all(np.array_equal(a, b) for a, b in
                                         zip(s.fields().values(), nat.fields().values()))
            variants[f"{name}{'-reverse' if rev else ''}"] = {
                "max_line_length": mll or 132, "bitwise_equal_to_reference": bool(same)}

    #     ... and at the DEFAULT max_line_length (132), where the reference's own
    #     run_variant cannot run the emitted-code variants (its split lands inside
    #     macro invocations; gpu-emulated crashes): the expand-first oracle
    #     (ref_capi.cpp)
    for v, name in [(2, "cpu"), (3, "gpu-emulated")]:
        for rev in (False, True):
            s, msg = ref.run_variant_expand_first(v, g, 10, 132, rev)
            same = s is not None and all(np.array_equal(a, b) for a, b in
                                         zip(s.fields().values(), nat.fields().values()))
            variants[f"{name}{'-reverse' if rev else ''}@132-expand-first"] = {
                "max_line_length": 132, "bitwise_equal_to_reference": bool(same),
                "write_data_calls": ref.last_write_calls,
                "fnv1a64": {k: c.fnv(a) for k, a in s.fields().items()} if s else None}

    # (8) the corpus driver's output cadence (simple_weather.h90:91-95): number
    #     of write_data calls of the interpreted original for (steps, dt, out_dt)
    writes = []
    for steps, dt, odt in [(25, 0.1, 1.0), (10, 0.1, 1.0), (7, 0.25, 0.5), (30, 0.1, 0.3)]:
        g = O.make_grid(timestep=dt, output_timestep=odt)
        s, msg = ref.run_variant(1, g, steps, 0, False)
        writes.append({"steps": steps, "timestep": dt, "output_timestep": odt,
                       "write_data_calls": ref.last_write_calls, "ok": s is not None})

    meta = {"generator": "oracle/gen_golden.py", "full_cases": cases, "hashes": hashes,
            "corpus_write_data": writes,
            "dumps": {"dump_energy_4x4x4_s2.txt": "energy after 2 steps, 4x4x4",
                      "dump_surf_4x4x4_s2.txt": "energy_surf, rank 2"},
            "variants_16x16x8_s10": variants}
    with open(os.path.join(GOLD, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print(json.dumps(variants))
    print("wrote", GOLD)


if __name__ == "__main__":
    main()
