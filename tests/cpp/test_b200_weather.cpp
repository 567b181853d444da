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
