// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C ABI over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile) so that Python tests, the
// golden-fixture generator and bench.py's CPU-baseline leg can call the
// reference's own `hft::` functions.  Nothing here re-implements the
// algorithm: every entry point forwards to the reference.
//
// Host buffers are the logical column-major `ArrayObject::data` vectors of
// `SimState` (weather.hpp:39-46; bounds from weather.cpp:71,77).
#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "hft/config.hpp"
#include "hft/interpreter.hpp"
#include "hft/lines.hpp"
#include "hft/parser.hpp"
#include "hft/pipeline.hpp"
#include "hft/weather.hpp"

namespace {

struct Grid { // field order mirrors hft::GridConfig (weather.hpp:27-34)
    long long nx, ny, nz;
    double timestep, output_timestep, diffusion_velocity, radiation_intensity,
        transfer_velocity, surf_energy, pbl_energy;
};

hft::GridConfig to_cfg(const Grid* g) {
    hft::GridConfig c;
    c.nx = g->nx;
    c.ny = g->ny;
    c.nz = g->nz;
    c.timestep = g->timestep;
    c.output_timestep = g->output_timestep;
    c.diffusion_velocity = g->diffusion_velocity;
    c.radiation_intensity = g->radiation_intensity;
    c.transfer_velocity = g->transfer_velocity;
    c.surf_energy = g->surf_energy;
    c.pbl_energy = g->pbl_energy;
    return c;
}

void put(const hft::ArrayObject& a, double* out) {
    if (out) std::memcpy(out, a.data.data(), a.data.size() * sizeof(double));
}
void get(hft::ArrayObject& a, const double* in) {
    if (in) std::memcpy(a.data.data(), in, a.data.size() * sizeof(double));
}
void put_state(const hft::SimState& s, double* e, double* eu, double* sf, double* pb) {
    put(s.energy, e);
    put(s.energy_u, eu);
    put(s.energy_surf, sf);
    put(s.energy_pbl, pb);
}
void copy_msg(const hft::Diagnostics& d, char* msg, size_t cap) {
    if (!msg || cap == 0) return;
    std::string r = d.render();
    std::snprintf(msg, cap, "%s", r.c_str());
}

} // namespace

extern "C" {

int hftref_validate(const Grid* g, char* msg, size_t cap) {
    hft::Diagnostics d;
    bool ok = hft::validate(to_cfg(g), d);
    copy_msg(d, msg, cap);
    return ok ? 1 : 0;
}

// hft::run_reference (weather.cpp:173-178)
void hftref_run_reference(const Grid* g, long long steps, double* e, double* eu, double* sf,
                          double* pb) {
    hft::SimState s = hft::run_reference(to_cfg(g), steps);
    put_state(s, e, eu, sf, pb);
}

// hft::reference_init (weather.cpp:67-99) for shapes, then the given state,
// then `steps` x hft::reference_step (weather.cpp:101-171).
void hftref_steps_from(const Grid* g, long long steps, double* e, double* eu, double* sf,
                       double* pb) {
    hft::GridConfig c = to_cfg(g);
    hft::SimState s;
    hft::reference_init(c, s);
    get(s.energy, e);
    get(s.energy_u, eu);
    get(s.energy_surf, sf);
    get(s.energy_pbl, pb);
    for (long long n = 0; n < steps; ++n) hft::reference_step(c, s);
    put_state(s, e, eu, sf, pb);
}

// CPU baseline: hft::reference_init, then time `steps` x hft::reference_step
// (weather.cpp:101-171) alone; returns seconds.
double hftref_time_steps(const Grid* g, long long steps) {
    hft::GridConfig c = to_cfg(g);
    hft::SimState s;
    hft::reference_init(c, s);
    auto t0 = std::chrono::steady_clock::now();
    for (long long n = 0; n < steps; ++n) hft::reference_step(c, s);
    auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double>(t1 - t0).count();
}

// Interpreted corpus variants (weather.cpp:439-476): 0 reference, 1 original,
// 2 cpu, 3 gpu-emulated.  `max_line_length` overrides BuildConfig (>= 268
// avoids the split-before-expand failure, SURVEY.md finding 6).
int hftref_run_variant(int variant, const Grid* g, long long steps, int max_line_length,
                       int reverse, const char* corpus_dir, double* e, double* eu, double* sf,
                       double* pb, char* msg, size_t cap, int* write_calls) {
    hft::Diagnostics d;
    std::vector<hft::LoadedSource> srcs;
    if (variant != 0) {
        for (const char* f : {"simple_weather.h90", "physics.h90", "diffusion.h90"})
            srcs.push_back(hft::load_and_merge(std::string(corpus_dir) + "/" + f, d));
    }
    hft::BuildConfig bc;
    if (max_line_length > 0) bc.max_line_length = max_line_length;
    hft::VariantRun r = hft::run_variant(static_cast<hft::Variant>(variant), srcs, bc, to_cfg(g),
                                         steps, d,
                                         reverse ? hft::LaunchOrder::Reverse
                                                 : hft::LaunchOrder::Forward);
    copy_msg(d, msg, cap);
    if (write_calls) *write_calls = r.write_data_calls;
    if (!r.ok) return 0;
    put_state(r.state, e, eu, sf, pb);
    return 1;
}

// the emitted-code variants (cpu / gpu-emulated) at the
// DEFAULT max_line_length.  The reference splits long lines at transpile time
// (pipeline.cpp:88) and expands the storage macros on the consumer side
// afterwards (pipeline.cpp:103-113, run_units at weather.cpp:401-437), so a
// split can land inside a macro invocation and run_variant(GpuEmulated) fails
// below max_line_length 268.  This oracle uses only the reference's own phases
// in the order that works: transpile without a line limit, expand each unit,
// THEN split the plain text at `max_line_length`, re-merge and interpret.  The
// driver (initialize, then simulate(0, (steps - 0.5) dt, dt, out_dt)) and the
// field read-back restate drive() / extract_state() (weather.cpp:364-397),
// which the reference keeps file-local.  variant: 2 = cpu, 3 = gpu-emulated.
int hftref_run_variant_expand_first(int variant, const Grid* g, long long steps,
                                    int max_line_length, int reverse, const char* corpus_dir,
                                    double* e, double* eu, double* sf, double* pb, char* msg,
                                    size_t cap, int* write_calls) {
    hft::Diagnostics d;
    const hft::GridConfig gc = to_cfg(g);
    std::vector<hft::LoadedSource> srcs;
    for (const char* f : {"simple_weather.h90", "physics.h90", "diffusion.h90"})
        srcs.push_back(hft::load_and_merge(std::string(corpus_dir) + "/" + f, d));
    hft::BuildConfig unsplit;
    unsplit.max_line_length = 1 << 20; // no transpile-time split
    const bool gpu = variant == 3;
    hft::TranspileResult tr = hft::transpile(srcs, unsplit, gpu ? "gpu-cuda" : "cpu-openmp", d);
    std::vector<std::vector<hft::LogicalLine>> files;
    for (std::size_t n = 1; d.ok() && n < tr.units.size(); ++n) {
        const std::string text = hft::expand_unit(tr.units[0], tr.units[n], gpu, d);
        std::vector<std::string> lines;
        std::string cur;
        for (char ch : text) {
            if (ch == '\n') {
                lines.push_back(cur);
                cur.clear();
            } else {
                cur += ch;
            }
        }
        if (!cur.empty()) lines.push_back(cur);
        std::string split;
        for (const auto& l : hft::split_lines(lines, max_line_length, d)) split += l + "\n";
        const std::string& fn = tr.units[n].filename;
        hft::LoadedSource ls = hft::prepare_source(fn.substr(0, fn.rfind('.')) + ".h90", split, d);
        files.push_back(std::move(ls.logical));
    }
    int ok = 0;
    if (d.ok()) {
        hft::ast::Program prog = hft::parse_program(files, d);
        hft::InterpreterOptions io;
        io.emulate_kernels = gpu;
        io.launch_order = reverse ? hft::LaunchOrder::Reverse : hft::LaunchOrder::Forward;
        if (d.ok()) {
            hft::Interpreter it(prog, d, io);
            int writes = 0;
            it.on_write_data = [&](const std::string&, double, const hft::ArrayObject&) { ++writes; };
            it.set_global_int("nx", gc.nx);
            it.set_global_int("ny", gc.ny);
            it.set_global_int("nz", gc.nz);
            const double end_time = (static_cast<double>(steps) - 0.5) * gc.timestep;
            if (it.call("initialize") &&
                it.call("simulate", {0.0, end_time, gc.timestep, gc.output_timestep})) {
                const hft::ast::Arch arch = gpu ? hft::ast::Arch::Gpu : hft::ast::Arch::Cpu;
                const std::pair<const char*, int> fields[] = {
                    {"energy", 3}, {"energy_u", 3}, {"energy_surf", 2}, {"energy_pbl", 2}};
                double* outs[] = {e, eu, sf, pb};
                ok = 1;
                for (int f = 0; f < 4; ++f) {
                    const hft::ArrayObject* raw = it.find_array(fields[f].first);
                    if (!raw) {
                        ok = 0;
                        break;
                    }
                    put(hft::unpermute_storage(*raw, unsplit.storage_order(arch, fields[f].second)),
                        outs[f]);
                }
                if (write_calls) *write_calls = writes;
            }
        }
    }
    copy_msg(d, msg, cap);
    return ok && d.ok() ? 1 : 0;
}

// hft::compare_arrays (weather.cpp:184-217) over flat logical buffers of
// rank `rank` with inclusive bounds lo[d]..hi[d].
int hftref_compare_arrays(int rank, const long long* lo, const long long* hi, const double* a,
                          const double* b, double* max_abs, double* nrmse, long long* where) {
    hft::ArrayObject x, y;
    for (int d = 0; d < rank; ++d) x.bounds.push_back({lo[d], hi[d]});
    y.bounds = x.bounds;
    x.data.assign(a, a + x.size());
    y.data.assign(b, b + y.size());
    hft::CompareReport r = hft::compare_arrays(x, y);
    *max_abs = r.max_abs;
    *nrmse = r.nrmse;
    for (std::size_t d = 0; d < r.where.size(); ++d) where[d] = r.where[d];
    return r.shape_ok ? 1 : 0;
}

// hft::unpermute_storage (weather.cpp:306-338).
void hftref_unpermute(int rank, const long long* lo, const long long* hi, const int* order,
                      const double* raw, double* out, long long* out_lo, long long* out_hi) {
    hft::ArrayObject x;
    for (int d = 0; d < rank; ++d) x.bounds.push_back({lo[d], hi[d]});
    x.data.assign(raw, raw + x.size());
    hft::ArrayObject y = hft::unpermute_storage(x, std::vector<int>(order, order + rank));
    for (int d = 0; d < rank; ++d) {
        out_lo[d] = y.bounds[d].first;
        out_hi[d] = y.bounds[d].second;
    }
    std::memcpy(out, y.data.data(), y.data.size() * sizeof(double));
}

} // extern "C"
