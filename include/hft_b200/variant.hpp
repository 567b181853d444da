//------------------------------------------------------------------------------
// hft_b200/variant.hpp -- the corpus driver's variant dispatch with a B200 arm.
//
// Drop-in for hft::run_variant / hft::Variant / variant_name / parse_variant
// (/root/reference/proj/include/hft/weather.hpp:99-123, weather.cpp:344-476).
// It needs the reference's own headers (the hft::VariantRun, LoadedSource and
// BuildConfig types) and library for the interpreted variants; the B200 arm
// itself goes only through the C ABI (include/hftw.h).
//
//   Variant::Reference, Original, Cpu, GpuEmulated -> hft::run_variant, unchanged
//   Variant::B200 -> the corpus driver's run on the device: drive()'s time loop
//       (weather.cpp:364-376: simulate(0, (steps - 0.5) * dt, dt, out_dt)) as
//       hftw_simulate, counting write_data calls like the interpreter's
//       on_write_data hook (interpreter.hpp:68-69), then the four fields in
//       logical order (extract_state, weather.cpp:378-397).  Same checks and
//       messages as the interpreted variants (validate; "interpreted runs need
//       at least one step"); no transcript (the device prints nothing).
// The state is bitwise identical to every other variant's.
//------------------------------------------------------------------------------
#pragma once

#include <optional>
#include <string>
#include <vector>

#include "hft/weather.hpp"
#include "hft_b200/weather.hpp"

namespace hft::b200 {

enum class Variant { Reference, Original, Cpu, GpuEmulated, B200 };

/// weather.cpp:344-352, plus "b200".
inline const char* variant_name(Variant v) {
    switch (v) {
    case Variant::Reference: return "reference";
    case Variant::Original: return "original";
    case Variant::Cpu: return "cpu";
    case Variant::GpuEmulated: return "gpu-emulated";
    case Variant::B200: return "b200";
    }
    return "?";
}

/// weather.cpp:354-360, plus "b200".
inline std::optional<Variant> parse_variant(const std::string& name) {
    if (name == "b200") return Variant::B200;
    if (auto v = hft::parse_variant(name)) {
        switch (*v) {
        case hft::Variant::Reference: return Variant::Reference;
        case hft::Variant::Original: return Variant::Original;
        case hft::Variant::Cpu: return Variant::Cpu;
        case hft::Variant::GpuEmulated: return Variant::GpuEmulated;
        }
    }
    return std::nullopt;
}

namespace detail {
struct WriteCounter {
    int calls = 0;
    static void hook(void* user, const char*, double, const double*) {
        ++static_cast<WriteCounter*>(user)->calls;
    }
};
} // namespace detail

/// hft::run_variant (weather.cpp:439-476) with the B200 arm.  `where` places
/// the B200 run (one device, or a decomposition over several).
inline hft::VariantRun run_variant(Variant v, const std::vector<hft::LoadedSource>& sources,
                                   const hft::BuildConfig& bc, const hft::GridConfig& gc,
                                   long long steps, hft::Diagnostics& diags,
                                   hft::LaunchOrder order = hft::LaunchOrder::Forward,
                                   const Placement& where = {}) {
    if (v != Variant::B200) {
        const hft::Variant rv = v == Variant::Reference  ? hft::Variant::Reference
                                : v == Variant::Original ? hft::Variant::Original
                                : v == Variant::Cpu      ? hft::Variant::Cpu
                                                         : hft::Variant::GpuEmulated;
        return hft::run_variant(rv, sources, bc, gc, steps, diags, order);
    }
    hft::VariantRun out;
    if (!validate(gc, diags)) return out;
    if (steps < 1) { // as the interpreted variants (weather.cpp:403-406, 455-458)
        diags.error({"<config>", 0}, "interpreted runs need at least one step");
        return out;
    }
    out.ok = report_to(diags, [&] {
        Simulation sim(gc, where);
        sim.init(); // the corpus' initialize (reference_init's state)
        const double end_time = (static_cast<double>(steps) - 0.5) * gc.timestep;
        detail::WriteCounter wc;
        check(hftw_simulate(sim.handle(), 0.0, end_time, gc.timestep, gc.output_timestep,
                            &detail::WriteCounter::hook, &wc, nullptr, nullptr),
              sim.handle());
        out.write_data_calls = wc.calls;
        sim.download(out.state);
    });
    return out;
}

} // namespace hft::b200
