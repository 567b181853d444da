// tests/cpp/test_b200_weather.cpp -- C++ drop-in parity test (GPU).
//
// Uses the reference's OWN types and functions (hft::GridConfig, hft::SimState,
// hft::run_reference, hft::compare_fields from the unmodified reference
// library oracle/_ref/libhft_core.a) side by side with the B200 adapter
// hft::b200::* from include/hft_b200/weather.hpp, and requires bitwise
// agreement.  The cases mirror /root/reference/proj/tests/test_weather.cpp.
// Built by __graft_entry__.build() where the reference headers exist; run by
// tests/test_cpp_adapter.py on the GPU box.
#include <cstdio>
#include <random>
#include <string>

#include "hft/weather.hpp"
#include "hft_b200/variant.hpp"
#include "hft_b200/weather.hpp"

static int failures = 0, checks = 0;
#define CHECK(x)                                                                   \
    do {                                                                           \
        ++checks;                                                                  \
        if (!(x)) {                                                                \
            ++failures;                                                            \
            std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #x); \
        }                                                                          \
    } while (0)

static bool bitwise(const hft::SimState& a, const hft::SimState& b, const char* tag) {
    hft::StateReport r = hft::compare_fields(a, b);
    if (!r.shape_ok || r.max_abs != 0.0) {
        std::fprintf(stderr, "[%s] mismatch in %s: max_abs=%g shape_ok=%d\n", tag, r.field.c_str(),
                     r.max_abs, (int)r.shape_ok);
        return false;
    }
    return true;
}

int main() {
    // validate: same verdicts and messages (test_weather.cpp:88-115)
    {
        hft::GridConfig cfg;
        hft::Diagnostics d1, d2;
        CHECK(hft::b200::validate(cfg, d1) == hft::validate(cfg, d2));
        cfg.diffusion_velocity = 0.2;
        cfg.nx = 1;
        hft::Diagnostics e1, e2;
        CHECK(!hft::b200::validate(cfg, e1));
        hft::validate(cfg, e2);
        CHECK(e1.render() == e2.render());
    }
    // run_reference on the reference's types, several grids (bitwise)
    {
        const long long shapes[][4] = {{16, 16, 8, 10}, {4, 4, 4, 3}, {6, 4, 4, 5},
                                       {150, 37, 58, 4}, {65, 3, 9, 2}, {2, 2, 2, 3}};
        for (auto& s : shapes) {
            hft::GridConfig cfg;
            cfg.nx = s[0];
            cfg.ny = s[1];
            cfg.nz = s[2];
            hft::SimState want = hft::run_reference(cfg, s[3]);
            hft::SimState got = hft::b200::run_reference<hft::SimState>(cfg, s[3]);
            CHECK(bitwise(want, got, "run_reference"));
        }
    }
    // zero constants: identity (test_weather.cpp:117-137)
    {
        hft::GridConfig cfg;
        cfg.nx = 6;
        cfg.ny = 4;
        cfg.nz = 4;
        cfg.diffusion_velocity = cfg.radiation_intensity = cfg.transfer_velocity = 0.0;
        hft::SimState a = hft::b200::run_reference<hft::SimState>(cfg, 1);
        hft::SimState b = hft::b200::run_reference<hft::SimState>(cfg, 5);
        CHECK(bitwise(a, b, "identity"));
    }
    // reference_init / reference_step on a random host state with odd constants
    {
        hft::GridConfig cfg;
        cfg.nx = 33;
        cfg.ny = 29;
        cfg.nz = 11;
        cfg.diffusion_velocity = 1.0 / 6.0;
        cfg.radiation_intensity = 0.37;
        cfg.transfer_velocity = 0.013;
        hft::SimState st, mine;
        hft::reference_init(cfg, st);
        hft::b200::reference_init(cfg, mine);
        CHECK(bitwise(st, mine, "reference_init"));
        std::mt19937_64 rng(1802);
        std::uniform_real_distribution<double> U(150.0, 350.0);
        for (auto* f : {&st.energy, &st.energy_u, &st.energy_surf, &st.energy_pbl})
            for (double& v : f->data) v = U(rng);
        mine = st;
        for (int n = 0; n < 3; ++n) {
            hft::reference_step(cfg, st);
            hft::b200::reference_step(cfg, mine);
        }
        CHECK(bitwise(st, mine, "reference_step x3"));
        // two grids in turn: the cached device context follows the config
        hft::GridConfig cfg2 = cfg;
        cfg2.nx = 40;
        cfg2.radiation_intensity = -0.2;
        hft::SimState st2, mine2;
        hft::reference_init(cfg2, st2);
        mine2 = st2;
        for (int n = 0; n < 3; ++n) {
            hft::reference_step(cfg, st);
            hft::b200::reference_step(cfg, mine);
            hft::reference_step(cfg2, st2);
            hft::b200::reference_step(cfg2, mine2);
        }
        CHECK(bitwise(st, mine, "reference_step, alternating grids (1)"));
        CHECK(bitwise(st2, mine2, "reference_step, alternating grids (2)"));
        {   // page-locked SimState buffers (hftw_host_register), same results
            hft::b200::PinnedState pin(mine);
            for (int n = 0; n < 2; ++n) {
                hft::reference_step(cfg, st);
                hft::b200::reference_step(cfg, mine);
            }
            CHECK(bitwise(st, mine, "reference_step, pinned SimState"));
        }
        hft::b200::release_cached_context();
    }
    // the device-resident API: every step kernel, both layouts
    {
        hft::GridConfig cfg;
        cfg.nx = 100;
        cfg.ny = 41;
        cfg.nz = 58;
        hft::SimState want = hft::run_reference(cfg, 6);
        for (int layout : {HFTW_IJK, HFTW_KIJ})
            for (int k : {HFTW_KERNEL_AUTO, HFTW_KERNEL_FUSED_CELL, HFTW_KERNEL_SPLIT}) {
                hft::b200::Simulation sim(cfg, layout);
                sim.set_kernel(k);
                sim.init();
                sim.step(2);
                sim.step(4);
                hft::SimState got;
                sim.download(got);
                CHECK(bitwise(want, got, "Simulation"));
            }
    }
    // multi-GPU from this one thread (hft::b200::Placement -> hftw_create_multi):
    // decompositions whose ranks share device 0 (all that the test box has),
    // bitwise against the reference's own run_reference
    {
        struct Case { long long nx, ny, nz, steps; int px, py; };
        const Case cases[] = {{150, 70, 58, 5, 2, 1}, {131, 97, 12, 6, 2, 2},
                              {200, 140, 20, 9, 2, 4}, {97, 61, 13, 4, 3, 1}};
        for (const Case& c : cases) {
            hft::GridConfig cfg;
            cfg.nx = c.nx;
            cfg.ny = c.ny;
            cfg.nz = c.nz;
            cfg.diffusion_velocity = 0.125;
            hft::SimState want = hft::run_reference(cfg, c.steps);
            hft::b200::Placement where;
            where.px = c.px;
            where.py = c.py;
            where.devices.assign((size_t)(c.px * c.py), 0);
            hft::SimState got = hft::b200::run_reference<hft::SimState>(cfg, c.steps, where);
            CHECK(bitwise(want, got, "run_reference on a Placement"));
            // the device-resident API on the same placement, steps in two calls
            hft::b200::Simulation sim(cfg, where);
            CHECK(sim.ranks() == c.px * c.py);
            sim.init();
            sim.step(c.steps - 2);
            sim.step(2);
            hft::SimState got2;
            sim.download(got2);
            CHECK(bitwise(want, got2, "Simulation on a Placement"));
        }
        // a random uploaded state on a 2x2 placement (halos refilled after upload)
        hft::GridConfig cfg;
        cfg.nx = 61;
        cfg.ny = 45;
        cfg.nz = 9;
        cfg.radiation_intensity = -0.3;
        hft::SimState st;
        hft::reference_init(cfg, st);
        std::mt19937_64 rng(7);
        std::uniform_real_distribution<double> U(150.0, 350.0);
        for (auto* f : {&st.energy, &st.energy_u, &st.energy_surf, &st.energy_pbl})
            for (double& v : f->data) v = U(rng);
        hft::b200::Placement where;
        where.px = where.py = 2;
        where.devices = {0, 0, 0, 0};
        hft::b200::Simulation sim(cfg, where);
        sim.upload(st);
        sim.step(3);
        hft::SimState got;
        sim.download(got);
        for (int n = 0; n < 3; ++n) hft::reference_step(cfg, st);
        CHECK(bitwise(st, got, "uploaded state on a 2x2 Placement"));
    }
    // the corpus driver with a B200 arm (hft_b200/variant.hpp): the state of
    // Variant::Reference and the write_data count of the interpreted corpus
    // (tests/golden/golden.json corpus_write_data, from hft::run_variant(Original))
    {
        struct Case { long long steps; double dt, odt; int writes; };
        const Case cases[] = {{25, 0.1, 1.0, 3}, {10, 0.1, 1.0, 1}, {7, 0.25, 0.5, 4},
                              {30, 0.1, 0.3, 10}};
        for (const Case& c : cases) {
            hft::GridConfig cfg;
            cfg.timestep = c.dt;
            cfg.output_timestep = c.odt;
            hft::BuildConfig bc;
            hft::Diagnostics d1, d2;
            hft::VariantRun ref = hft::run_variant(hft::Variant::Reference, {}, bc, cfg, c.steps, d1);
            hft::VariantRun dev =
                hft::b200::run_variant(hft::b200::Variant::B200, {}, bc, cfg, c.steps, d2);
            CHECK(ref.ok && dev.ok && d2.ok());
            CHECK(bitwise(ref.state, dev.state, "run_variant(B200)"));
            CHECK(dev.write_data_calls == c.writes);
        }
        CHECK(hft::b200::parse_variant("b200") == hft::b200::Variant::B200);
        CHECK(std::string(hft::b200::variant_name(hft::b200::Variant::GpuEmulated)) ==
              "gpu-emulated");
        hft::BuildConfig bc;
        hft::Diagnostics d;
        hft::GridConfig cfg;
        CHECK(!hft::b200::run_variant(hft::b200::Variant::B200, {}, bc, cfg, 0, d).ok);
        CHECK(!d.ok());
    }
    // the Diagnostics& overloads report instead of throwing
    {
        hft::GridConfig bad;
        bad.nz = 1;
        hft::Diagnostics d;
        hft::SimState out;
        CHECK(!hft::b200::run_reference(bad, 1, out, d));
        CHECK(d.error_count() == 1 && d.has_rule("b200-einval"));
        CHECK(d.all()[0].where.file == "<b200>");
        hft::GridConfig cfg;
        hft::Diagnostics d2;
        hft::b200::Placement nowhere;
        nowhere.device = 99;
        CHECK(!hft::b200::run_reference(cfg, 1, out, d2, nowhere));
        CHECK(d2.has_rule("b200-einval"));
        hft::Diagnostics d3;
        CHECK(hft::b200::run_reference(cfg, 3, out, d3) && d3.ok());
        CHECK(bitwise(hft::run_reference(cfg, 3), out, "run_reference(Diagnostics&)"));
        hft::SimState st;
        hft::reference_init(cfg, st);
        hft::SimState mine = st;
        hft::Diagnostics d4;
        CHECK(hft::b200::reference_step(cfg, mine, d4) && d4.ok());
        hft::reference_step(cfg, st);
        CHECK(bitwise(st, mine, "reference_step(Diagnostics&)"));
        hft::b200::release_cached_context();
    }
    // errors surface as exceptions, never as silent results
    {
        hft::GridConfig bad;
        bad.nz = 1;
        bool threw = false;
        try {
            hft::b200::run_reference<hft::SimState>(bad, 1);
        } catch (const hft::b200::Error& e) {
            threw = e.code == HFTW_EINVAL;
        }
        CHECK(threw);
    }
    std::printf("%d checks, %d failures\n", checks, failures);
    return failures ? 1 : 0;
}
