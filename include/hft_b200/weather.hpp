//------------------------------------------------------------------------------
// hft_b200/weather.hpp -- header-only C++ adapter over the C ABI (hftw.h).
//
// Drop-in for the reference's native simulator API
// (/root/reference/proj/include/hft/weather.hpp, namespace hft):
//
//   hft::validate(cfg, diags)          (weather.hpp:37)  -> hft::b200::validate
//   hft::reference_init(cfg, st)       (weather.hpp:51)  -> hft::b200::reference_init
//   hft::reference_step(cfg, st)       (weather.hpp:55)  -> hft::b200::reference_step
//   hft::run_reference(cfg, steps)     (weather.hpp:59)  -> hft::b200::run_reference
//
// The functions are templates over the caller's types, so they accept the
// reference's own hft::GridConfig / hft::SimState / hft::Diagnostics
// unchanged (anything with the same member names works: GridConfig's ten
// fields, SimState's four ArrayObject members with `bounds` and `data`,
// a Diagnostics with error(SourceRef, std::string)).  For code that does not
// link the reference, hft::b200 also defines minimal look-alike types.
//
// Results are bitwise identical to the reference (see include/hftw.h).
// Unlike the reference, device work can fail (no GPU, out of memory).  Each
// entry point has two forms: the reference's signature, which throws
// hft::b200::Error, and an overload taking the caller's Diagnostics& (the
// reference's error convention, diagnostics.hpp:35-76) that never throws: it
// reports diags.error({"<b200>", 0}, message, "b200-<code>") and returns
// false.  There is no CPU fallback either way.
//
// Multi-GPU: a Placement runs the same calls on a px x py I x J decomposition
// from this one host thread (hftw_create_multi; one device per rank, repeats
// allowed), bitwise identical to one device.
//------------------------------------------------------------------------------
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../hftw.h"

namespace hft::b200 {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void check(int rc, const hftw_ctx* ctx = nullptr) {
    if (rc != HFTW_OK) throw Error(rc, hftw_last_error(ctx));
}

/// Rule id of an hftw error code (Diagnostic::rule, diagnostics.hpp:26-31).
inline const char* rule_of(int code) {
    switch (code) {
    case HFTW_EINVAL: return "b200-einval";
    case HFTW_ECUDA: return "b200-ecuda";
    case HFTW_ENOMEM: return "b200-enomem";
    case HFTW_ESTATE: return "b200-estate";
    case HFTW_EUNSUP: return "b200-eunsup";
    }
    return "b200-error";
}

/// Run `f`; an hft::b200::Error becomes diags.error({"<b200>", 0}, msg, rule).
template <class Diags, class F>
bool report_to(Diags& diags, F&& f) {
    try {
        f();
        return true;
    } catch (const Error& e) {
        diags.error({"<b200>", 0}, e.what(), rule_of(e.code));
    } catch (const std::exception& e) { // e.g. std::bad_alloc of a host SimState
        diags.error({"<b200>", 0}, e.what(), "b200-host");
    }
    return false;
}

/// Where a simulation runs.  Default: one rank on `device`.  px x py > 1 (or a
/// non-empty `devices`): that I x J decomposition in this process, rank r
/// (= ry * px + rx) on devices[r], or on device r when `devices` is empty.
struct Placement {
    int device = 0;
    int px = 1, py = 1;
    std::vector<int> devices;
    int layout = HFTW_IJK;

    /// n GPUs 0..n-1 in the paper's process grids: 2 -> 2x1,
    /// 4 -> 2x2, 8 -> 2x4; other n: n x 1.
    static Placement gpus(int n) {
        Placement p;
        p.px = n == 4 ? 2 : n == 8 ? 2 : n;
        p.py = n == 4 ? 2 : n == 8 ? 4 : 1;
        return p;
    }
    bool multi() const { return px * py > 1 || !devices.empty(); }
};

// ---- minimal look-alike types (same member names as the reference) --------
struct GridConfig {
    long long nx = 16, ny = 16, nz = 8;
    double timestep = 0.1;
    double output_timestep = 1.0;
    double diffusion_velocity = 0.1;
    double radiation_intensity = 0.1;
    double transfer_velocity = 0.01;
    double surf_energy = 330.0;
    double pbl_energy = 200.0;
};
struct ArrayObject {
    std::vector<std::pair<long long, long long>> bounds;
    std::vector<double> data;
};
struct SimState {
    ArrayObject energy, energy_u, energy_surf, energy_pbl;
};

// ---- conversions -----------------------------------------------------------
template <class Cfg>
hftw_grid to_grid(const Cfg& c) {
    hftw_grid g;
    g.nx = c.nx;
    g.ny = c.ny;
    g.nz = c.nz;
    g.timestep = c.timestep;
    g.output_timestep = c.output_timestep;
    g.diffusion_velocity = c.diffusion_velocity;
    g.radiation_intensity = c.radiation_intensity;
    g.transfer_velocity = c.transfer_velocity;
    g.surf_energy = c.surf_energy;
    g.pbl_energy = c.pbl_energy;
    return g;
}

// Shapes of weather.cpp:71 (3D) and :77 (2D).
template <class Cfg, class Array>
void shape3(const Cfg& c, Array& a) {
    a.bounds = {{0, c.nx + 1}, {0, c.ny + 1}, {1, c.nz}};
    a.data.assign(static_cast<std::size_t>((c.nx + 2) * (c.ny + 2) * c.nz), 0.0);
}
template <class Cfg, class Array>
void shape2(const Cfg& c, Array& a) {
    a.bounds = {{0, c.nx + 1}, {0, c.ny + 1}};
    a.data.assign(static_cast<std::size_t>((c.nx + 2) * (c.ny + 2)), 0.0);
}

/// hft::validate (weather.cpp:24-41): same rules and messages, reported as
/// diags.error({"<config>", 0}, message).
template <class Cfg, class Diags>
bool validate(const Cfg& cfg, Diags& diags) {
    hftw_grid g = to_grid(cfg);
    char msg[2048];
    int rc = hftw_validate(&g, msg, sizeof msg);
    std::string all(msg), prefix("<config>: error: ");
    std::size_t pos = 0;
    while (pos < all.size()) {
        std::size_t nl = all.find('\n', pos);
        std::string line = all.substr(pos, nl == std::string::npos ? std::string::npos : nl - pos);
        if (line.rfind(prefix, 0) == 0) line = line.substr(prefix.size());
        if (!line.empty()) diags.error({"<config>", 0}, line);
        if (nl == std::string::npos) break;
        pos = nl + 1;
    }
    return rc == HFTW_OK;
}

/// Device-resident simulation (new API): state lives in HBM between steps.
class Simulation {
public:
    template <class Cfg>
    explicit Simulation(const Cfg& cfg, int layout = HFTW_IJK, int device = 0)
        : grid_(to_grid(cfg)) {
        check(hftw_create(&grid_, layout, device, &ctx_));
    }
    /// On a Placement: one device, or a decomposition over several.
    template <class Cfg>
    Simulation(const Cfg& cfg, const Placement& where) : grid_(to_grid(cfg)) {
        if (!where.multi()) {
            check(hftw_create(&grid_, where.layout, where.device, &ctx_));
            return;
        }
        const int n = where.px * where.py;
        if (!where.devices.empty() && (int)where.devices.size() != n)
            throw Error(HFTW_EINVAL, "Placement: one device per rank (" + std::to_string(n) +
                                         "), got " + std::to_string(where.devices.size()));
        check(hftw_create_multi(&grid_, where.layout, where.px, where.py,
                                where.devices.empty() ? nullptr : where.devices.data(), &ctx_));
    }
    Simulation(const Simulation&) = delete;
    Simulation& operator=(const Simulation&) = delete;
    ~Simulation() { hftw_destroy(ctx_); }

    void init() { check(hftw_init(ctx_), ctx_); }
    void step(long long n = 1) { check(hftw_step(ctx_, n), ctx_); }
    void sync() { check(hftw_sync(ctx_), ctx_); }
    void set_kernel(int k) { check(hftw_set_kernel(ctx_, k), ctx_); }
    void set_option(int opt, long long v) { check(hftw_set_option(ctx_, opt, v), ctx_); }
    /// Ranks this simulation runs on (1 unless placed on a decomposition).
    int ranks() const { return hftw_group_size(ctx_); }

    template <class State>
    void upload(const State& st) {
        check(hftw_upload(ctx_, HFTW_ENERGY, st.energy.data.data()), ctx_);
        check(hftw_upload(ctx_, HFTW_ENERGY_U, st.energy_u.data.data()), ctx_);
        check(hftw_upload(ctx_, HFTW_ENERGY_SURF, st.energy_surf.data.data()), ctx_);
        check(hftw_upload(ctx_, HFTW_ENERGY_PBL, st.energy_pbl.data.data()), ctx_);
    }
    /// Fill a SimState (shapes set as reference_init would).
    template <class State>
    void download(State& st) {
        GridConfig c;
        c.nx = grid_.nx;
        c.ny = grid_.ny;
        c.nz = grid_.nz;
        shape3(c, st.energy);
        shape3(c, st.energy_u);
        shape2(c, st.energy_surf);
        shape2(c, st.energy_pbl);
        check(hftw_download(ctx_, HFTW_ENERGY, st.energy.data.data()), ctx_);
        check(hftw_download(ctx_, HFTW_ENERGY_U, st.energy_u.data.data()), ctx_);
        check(hftw_download(ctx_, HFTW_ENERGY_SURF, st.energy_surf.data.data()), ctx_);
        check(hftw_download(ctx_, HFTW_ENERGY_PBL, st.energy_pbl.data.data()), ctx_);
    }
    hftw_ctx* handle() { return ctx_; }

private:
    hftw_grid grid_;
    hftw_ctx* ctx_ = nullptr;
};

/// hft::reference_init (weather.cpp:67-99), computed on the device.
template <class Cfg, class State>
void reference_init(const Cfg& cfg, State& st, int device = 0) {
    Simulation s(cfg, HFTW_IJK, device);
    s.init();
    s.download(st);
}
/// ... reporting failures to `diags` (no exceptions).
template <class Cfg, class State, class Diags>
bool reference_init(const Cfg& cfg, State& st, Diags& diags, int device = 0) {
    return report_to(diags, [&] { reference_init(cfg, st, device); });
}

namespace detail {
/// The context reference_step runs on: one per host thread, kept between
/// calls while the grid (all ten GridConfig fields) and device stay the same,
/// so a loop of reference_step calls pays the device allocation once.
struct CachedSim {
    hftw_grid key{};
    int device = -1;
    hftw_ctx* ctx = nullptr;
    ~CachedSim() { reset(); }
    void reset() {
        if (ctx) hftw_destroy(ctx);
        ctx = nullptr;
        device = -1;
    }
    hftw_ctx* get(const hftw_grid& g, int dev) {
        if (!ctx || dev != device || std::memcmp(&g, &key, sizeof g) != 0) {
            reset();
            check(hftw_create(&g, HFTW_IJK, dev, &ctx));
            key = g;
            device = dev;
        }
        return ctx;
    }
};
inline CachedSim& cached_sim() {
    thread_local CachedSim c;
    return c;
}
} // namespace detail

/// Page-locks the four host buffers of a SimState for its lifetime (RAII over
/// hftw_host_register): pageable std::vector storage crosses PCIe through the
/// driver's bounce buffer (ASUCA reference_step ~185 ms instead of ~41 ms).
/// The vectors must not be resized while it lives (reference_step writes them
/// in place).
class PinnedState {
public:
    template <class State>
    explicit PinnedState(State& st) {
        for (auto* v : {&st.energy.data, &st.energy_u.data, &st.energy_surf.data,
                        &st.energy_pbl.data}) {
            if (v->empty()) continue;
            check(hftw_host_register(v->data(), v->size() * sizeof(double)));
            ptrs_.push_back(v->data());
        }
    }
    PinnedState(const PinnedState&) = delete;
    PinnedState& operator=(const PinnedState&) = delete;
    ~PinnedState() {
        for (void* p : ptrs_) hftw_host_unregister(p);
    }

private:
    std::vector<void*> ptrs_;
};

/// Free the context that reference_step keeps for this host thread.
inline void release_cached_context() { detail::cached_sim().reset(); }

/// hft::reference_step (weather.cpp:101-171) on a host SimState, in place.
/// Transfer-bound by construction (hftw_step_host overlaps the PCIe copies
/// with the step in row blocks); keep state on the device (Simulation) for
/// runs of more than one step.  The device context is reused across calls
/// on the same grid (release_cached_context frees it).
template <class Cfg, class State>
void reference_step(const Cfg& cfg, State& st, int device = 0) {
    const hftw_grid g = to_grid(cfg);
    hftw_ctx* ctx = detail::cached_sim().get(g, device);
    check(hftw_step_host(ctx, st.energy.data.data(), st.energy_surf.data.data(),
                         st.energy_pbl.data.data(), st.energy.data.data(),
                         st.energy_u.data.data()),
          ctx);
}

/// ... reporting failures to `diags` (no exceptions).
template <class Cfg, class State, class Diags>
bool reference_step(const Cfg& cfg, State& st, Diags& diags, int device = 0) {
    return report_to(diags, [&] { reference_step(cfg, st, device); });
}

/// hft::run_reference (weather.cpp:173-178), on one device or on a Placement
/// (e.g. run_reference(cfg, steps, Placement::gpus(8))).
template <class State = SimState, class Cfg>
State run_reference(const Cfg& cfg, long long steps, const Placement& where) {
    Simulation s(cfg, where);
    s.init();
    s.step(steps);
    State st;
    s.download(st);
    return st;
}
template <class State = SimState, class Cfg>
State run_reference(const Cfg& cfg, long long steps, int device = 0) {
    Placement p;
    p.device = device;
    return run_reference<State>(cfg, steps, p);
}
/// ... into `out`, reporting failures to `diags` (no exceptions).
template <class Cfg, class State, class Diags>
bool run_reference(const Cfg& cfg, long long steps, State& out, Diags& diags,
                   const Placement& where = {}) {
    return report_to(diags, [&] { out = run_reference<State>(cfg, steps, where); });
}

} // namespace hft::b200
