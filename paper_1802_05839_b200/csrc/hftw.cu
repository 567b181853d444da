// hftw.cu -- C ABI (include/hftw.h) over the B200 field store and kernels.
//
// Replaces, for the minimal-weather hot path, the reference's native
// simulator API in /root/reference/proj/include/hft/weather.hpp:
//   validate (:37), reference_init (:51), reference_step (:55),
//   run_reference (:59).
// The reference's SimState owns host std::vectors and swaps them each step
// (weather.cpp:170); here the context owns device-resident, padded fields in
// a ping-pong pair and the caller moves data in/out with upload/download.
// A context covers either the whole grid or one rank's subdomain of a
// px x py decomposition (hftw_create_dist); the single-GPU case is the 1 x 1
// plan, so both share every code path.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h> // header-only NVTX v3: ranges for nsys / ncu --nvtx

#include "../../include/hftw.h"
#include "weather_kernels.cuh"
#include "weather_pair.cuh"
#include "weather_wave.cuh"

using hftw::Dom;
using hftw::Halo;

namespace {

thread_local std::string g_err; // errors of calls without a context

// NVTX range over one API call (visible in nsys timelines and ncu --nvtx filters).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Tuning knobs for the experiments under tools/ (HFTW_TX=32|64, HFTW_NS=stages,
// HFTW_CHUNK=rows, ...): read ONLY in a -DHFTW_TUNING build (tools/build_variant.sh).
// The default library ignores the environment, so kernel choice and tiling
// depend on the grid, the device and the API (hftw_set_kernel/hftw_set_option).
int env_int(const char* name, int dflt) {
#ifdef HFTW_TUNING
    const char* v = std::getenv(name);
    return (v && *v) ? std::atoi(v) : dflt;
#else
    (void)name;
    return dflt;
#endif
}

constexpr int kFrontPad = 31; // IJK: logical i = 1 lands on a 256-byte boundary
constexpr int kNCW = 16;      // consumer warps of the TMA kernel
constexpr int kChunk = 32;    // rows per TMA work unit
constexpr int kMaxPipeBlocks = 64; // row blocks of the hftw_step_host pipeline (at most)
constexpr int kMaxWaveStepsDist = 1024; // steps per multi-step launch when decomposed
#ifndef HFTW_PAIR_KPT
#define HFTW_PAIR_KPT (64 / HFTW_PAIR_KG)
#endif
constexpr int kPairKPT = HFTW_PAIR_KPT; // planes per thread of the pair kernel (nz <= KG * KPT)

// What a rank publishes to its neighbours (raw bytes through the caller's
// allgather): IPC handles of the two energy buffers, sf, pb and the flags,
// plus the geometry needed to address their halo slots.
struct PeerDesc {
    cudaIpcMemHandle_t buf[2], sf, flags; // sf's allocation also holds pb (n2 further)
    cudaIpcMemHandle_t gpub;              // published P' of the pair passes (if any)
    int has_gpub;
    long long gpub_n, gcol_n;             // its doubles per parity / of the gcol part
    long long off3, off2, si, sj, sk, s2j, n2;
    hftw_plan plan;
    int magic;
};
constexpr int kPeerMagic = 0x48465457; // "HFTW"

struct PeerMap {
    int rank = -1;
    double* buf[2] = {nullptr, nullptr}; // at the neighbour's logical (0,0,1)
    double* sf = nullptr;                // at its logical (0,0)
    double* pb = nullptr;
    unsigned long long* flags = nullptr;
    double* gpub = nullptr;              // its published P' (two pass parities)
    long long gpub_n = 0, gcol_n = 0;    // its sizes (its subdomain may be a row / column longer)
    long long si = 0, sj = 0, sk = 0, s2j = 0;
};

} // namespace

struct hftw_ctx {
    hftw_grid g{};       // GLOBAL grid configuration
    hftw_plan plan{};    // this context's subdomain (1 x 1 plan on one GPU)
    bool dist = false;
    int layout = HFTW_IJK;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int kernel_req = HFTW_KERNEL_AUTO;
    int num_sms = 148;
    long long lnx = 0, lny = 0, nz = 0; // local extents

    // geometry (elements)
    long long Pi = 0, Rows = 0;  // IJK row pitch, rows per plane (lny + 4)
    long long Pk = 0;            // KIJ column pitch
    long long si = 0, sj = 0, sk = 0, s2j = 0;
    long long off3 = 0, off2 = 0; // offset of logical (0,0,1) / (0,0) from allocation start
    size_t n3 = 0, n2 = 0;        // allocation sizes (elements)

    double* buf[2] = {nullptr, nullptr};
    double* sf = nullptr;
    double* pb = nullptr;
    double* staging = nullptr; // dense staging for the KIJ relayout
    size_t staging_n = 0;
    int cur = 0;               // buf[cur] holds SimState::energy
    bool eu_derived = false;   // energy_u == physics(buf[cur ^ 1]), not yet materialised
    bool eu_stored = false;    // energy_u is in eu_buf (materialised after pair passes)
    bool partner_pform = false; // with eu_pending: buf[cur ^ 1] holds P(e_{n-2}), not e_{n-2}
    bool eu_pending = false;   // energy_u == physics(step(buf[cur ^ 1])): the call ended
                               // with a pair pass, which keeps e_{n-1} on chip only
    double* eu_buf = nullptr;  // third field buffer (allocated on first materialisation)

    // TMA kernel state
    bool tma_ok = false;
    int tx = 64;
    int ns = 0;
    int ctas = 0;
    int nstrips = 0;
    size_t smem = 0;
    CUtensorMap tm_e[2]{}, tm_sf{}, tm_pb{};
    int* d_sched = nullptr; // work-unit counter + finished-CTA counter
    int nchunks = 0;
    int chunk = kChunk;

    // pair kernel (two steps per pass; single-domain IJK, nz <= 64)
    bool pair_ok = false;
    bool pair_auto = env_int("HFTW_NO_PAIR", 0) == 0; // AUTO: two-step passes (HFTW_OPT_PAIR)
    int pair_ns = 0, pair_chunk = 0, pair_nchunks = 0, pair_ctas = 0;
    int pair_nbig = 0, pair_chunk2 = 0;
    bool pair_fast = false;     // every k-group has a compile-time row shape (AUTO uses it)
    size_t pair_smem = 0;
    CUtensorMap tm_e2[2]{};             // e: slab boxes {kPairW, 1, nz}
    CUtensorMap tm_ef[2]{};             // e: 2-wide far-column boxes
    int pair_nstrips = 0;
    CUtensorMap tm_sfpb{}, tm_sfpbf{};  // [sf; pb]: slab rows / far pair
    int* d_pair = nullptr;      // sched[2] + cnt_col[nchunks] + cnt_row[nstrips]
    // published ghost-adjacent P' of a pass, two parities (decomposed passes
    // alternate so that a wrap partner may still read the previous one):
    // [parity][gcol [4][ny+2][nz] | grow [4][nz][nx+2]]
    double* gpub = nullptr;
    size_t gpub_n = 0;          // doubles per parity
    long long pass_count = 0;   // pair passes since the last exchange (parity)

    // multi-step wavefront launch (weather_wave.cuh): single-domain IJK
    bool wave_ok = false;
    int wave_chunk = 0, wave_nchunks = 0, wave_ctas = 0, wave_gtasks = 0;
    bool wave_pref = false;     // multi-step launch preferred over one launch per step (auto)
    int opt_multistep = 0;      // HFTW_OPT_MULTISTEP: -1 never, 0 auto (wave_pref), 1 always
    int opt_exchange = 0;       // HFTW_OPT_EXCHANGE (groups): 0 in-kernel pushes, 1 baseline
    int opt_reverse = 0;        // HFTW_OPT_REVERSE: work units handed out last first
    cudaEvent_t xev = nullptr;  // the baseline's "my faces are out" event
    int* d_wave = nullptr;      // sched[2] + chunk_done[nchunks] + ghost_done[1]

    // measurement hook (hftw_set_timing)
    bool timing = false;
    struct TimedLaunch {
        int kind;
        cudaEvent_t a, b;
        int64_t steps;
    };
    std::vector<TimedLaunch> tev;

    // decomposed run
    unsigned long long* flags = nullptr; // [kFlags] step flags written by the neighbours
    int* done = nullptr;                 // CTAs finished in the current launch
    PeerMap peer[hftw::kNbrs];          // faces W E S N, then corners SW SE NW NE
    std::vector<void*> ipc_opened;
    bool connected = false;
    bool halo_dirty = false;             // fields changed since the last exchange
    long long step_count = 0;            // steps since the last exchange

    // output ring (hftw_simulate)
    struct OutSlot {
        double* dev = nullptr;  // dense logical snapshot on the device
        double* host = nullptr; // pinned logical copy
        cudaEvent_t done = nullptr;
        bool pending = false;
        double time = 0.0;
    };
    std::vector<OutSlot> out;
    cudaStream_t copy_stream = nullptr;

    // hftw_step_host: row-block pipeline H2D -> step -> D2H
    cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
    std::vector<cudaEvent_t> pipe_ev;
    double* host_stage[3] = {nullptr, nullptr, nullptr}; // dense logical energy in/out, energy_u
    void* flush_buf = nullptr;
    size_t flush_bytes = 0;

    // a failed hftw_step_host leaves the device state undefined: the fields
    // still to be re-uploaded (bit f = field f), cleared by init / uploads
    unsigned poisoned = 0;

    // group context (hftw_create_multi): one sub-context per rank in this process
    std::vector<hftw_ctx*> ranks;
    bool interleave = false; // ranks share a device: one launch per step, rank order

    std::string err;
};

namespace {

int fail(hftw_ctx* c, int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    else g_err = buf;
    return code;
}

#define CUDA_TRY(c, x)                                                                         \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess)                                                                 \
            return fail((c), HFTW_ECUDA, "%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_),    \
                        __FILE__, __LINE__);                                                   \
    } while (0)

bool valid_field(int f) { return f >= HFTW_ENERGY && f <= HFTW_ENERGY_PBL; }

Dom make_dom(const hftw_ctx* c) {
    const hftw_plan& p = c->plan;
    Dom d{};
    d.nx = (int)c->lnx;
    d.ny = (int)c->lny;
    d.nz = (int)c->nz;
    d.si = c->si;
    d.sj = c->sj;
    d.sk = c->sk;
    d.s2j = c->s2j;
    d.own_w = p.own_w;
    d.own_e = p.own_e;
    d.own_s = p.own_s;
    d.own_n = p.own_n;
    d.wfar = p.wfar;
    d.efar = p.efar;
    d.sfar = p.sfar;
    d.nfar = p.nfar;
    const double dv = c->g.diffusion_velocity;
    d.ri = c->g.radiation_intensity;
    d.tv = c->g.transfer_velocity;
    d.dv = dv;
    // the reference evaluates `(1 - c * dv)` in double (weather.cpp:135,143,156,165)
    volatile double v2 = 2.0 * dv, v5 = 5.0 * dv, v6 = 6.0 * dv;
    d.c2 = 1 - v2;
    d.c5 = 1 - v5;
    d.c6 = 1 - v6;
    return d;
}

// Halo parameters of a launch that writes buffer `dst`.
Halo make_halo(const hftw_ctx* c, int dst) {
    Halo h{};
    h.active = c->dist ? 1 : 0;
    if (!c->dist) return h;
    for (int q = 0; q < hftw::kNbrs; ++q) {
        const PeerMap& m = c->peer[q];
        if (m.rank < 0) continue;
        h.nb[q] = m.buf[dst];
        h.nsi[q] = m.si;
        h.nsj[q] = m.sj;
        h.nsk[q] = m.sk;
        h.nb_flags[q] = m.flags;
    }
#ifdef HFTW_TUNING
    // timing experiments on one device (results are wrong): no pushes / no waits
    if (env_int("HFTW_DBG_NOPUSH", 0))
        for (int q = 0; q < hftw::kNbrs; ++q) h.nb[q] = nullptr;
    h.nowait = env_int("HFTW_DBG_NOWAIT", 0);
#endif
    for (int d = 0; d < 4; ++d) {
        h.slot[d] = c->plan.send_slot[d];
        h.depth[d] = c->plan.depth[d];
        h.cslot[d][0] = c->plan.diag_slot[d][0];
        h.cslot[d][1] = c->plan.diag_slot[d][1];
    }
    h.my_flags = c->flags;
    h.done = c->done;
    h.step = c->step_count;
    return h;
}

double* e3(const hftw_ctx* c, int b) { return c->buf[b] + c->off3; }
// where SimState::energy_u lives: the ping-pong partner, or the third buffer
// the last pair pass of a call wrote it to
double* eu_field(const hftw_ctx* c) { return c->eu_stored ? c->eu_buf + c->off3 : e3(c, c->cur ^ 1); }
double* sf2(const hftw_ctx* c) { return c->sf + c->off2; }
double* pb2(const hftw_ctx* c) { return c->pb + c->off2; }

int grid_for(const hftw_ctx* c, long long n) {
    long long blocks = (n + 255) / 256;
    long long cap = (long long)c->num_sms * 16;
    return (int)std::max<long long>(1, std::min(blocks, cap));
}

// owned index ranges of the local domain
struct Box {
    long long i0, i1, j0, j1;
};
Box owned_box(const hftw_ctx* c) {
    const hftw_plan& p = c->plan;
    return {p.own_w ? 0 : 1, p.own_e ? c->lnx + 1 : c->lnx, p.own_s ? 0 : 1,
            p.own_n ? c->lny + 1 : c->lny};
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// A kernel's dynamic shared-memory limit is a per-device property of the
// function, shared by every context in the process: only ever RAISE it, so a
// context with a smaller tile (another nz) cannot shrink the limit below what
// another context's launches request.
cudaError_t raise_smem_attr(const void* fn, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> cur;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    size_t& have = cur[{dev, fn}];
    if (bytes <= have) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) have = bytes;
    return e;
}

template <int TX>
void set_tma_attrs(size_t smem) {
    raise_smem_attr((const void*)hftw::step_tma_kernel<TX, kNCW, true, false>, smem);
    raise_smem_attr((const void*)hftw::step_tma_kernel<TX, kNCW, false, false>, smem);
    raise_smem_attr((const void*)hftw::step_tma_kernel<TX, kNCW, true, true>, smem);
    raise_smem_attr((const void*)hftw::step_tma_kernel<TX, kNCW, false, true>, smem);
}

// Choose the TMA kernel geometry and build the tensor maps.  Leaves
// tma_ok = false (the cell kernel is used) when the grid does not fit: nz >
// 256 (TMA box limit) or a 4-stage ring would not fit shared memory.
int setup_tma(hftw_ctx* c) {
    c->tma_ok = false;
    const bool kij = c->layout == HFTW_KIJ;
    if (c->nz > 256 || (kij && c->Pk > 256)) return HFTW_OK;
    auto enc = encode_fn();
    if (!enc) return HFTW_OK;
    int smem_optin = 0;
    CUDA_TRY(c, cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                                       c->device));
    const int nz = (int)c->nz, pk = (int)c->Pk;
    int tx = 0, ns = 0;
    const int want_tx = env_int("HFTW_TX", 0), max_ns = env_int("HFTW_NS", 8);
    for (int cand : {64, 32}) {
        if (want_tx && cand != want_tx) continue;
        hftw::SlabGeom G = kij ? hftw::slab_geom_kij(cand, pk) : hftw::slab_geom(cand, nz);
        int fit = (int)((smem_optin - 1024 - 2 * G.out_bytes) / (G.stage + 20));
        if (fit >= 4) {
            tx = cand;
            ns = std::max(4, std::min(fit, max_ns));
            break;
        }
    }
    if (!tx) return HFTW_OK;
    hftw::SlabGeom G = kij ? hftw::slab_geom_kij(tx, pk) : hftw::slab_geom(tx, nz);
    c->tx = tx;
    c->ns = ns;
    c->smem = (size_t)ns * G.stage + 2 * (size_t)G.out_bytes + 2 * ns * sizeof(uint64_t) +
              ns * sizeof(int);
    if (tx == 64) set_tma_attrs<64>(c->smem);
    else set_tma_attrs<32>(c->smem);

    int per_sm = 0;
    cudaError_t oe =
        tx == 64 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                       &per_sm, hftw::step_tma_kernel<64, kNCW, true, false>, (kNCW + 1) * 32,
                       c->smem)
                 : cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                       &per_sm, hftw::step_tma_kernel<32, kNCW, true, false>, (kNCW + 1) * 32,
                       c->smem);
    if (oe != cudaSuccess || per_sm < 1) {
        cudaGetLastError();
        return HFTW_OK;
    }

    // tensor maps, no L2 promotion (promotion to 256-byte granules would read
    // whole neighbouring granules and inflate HBM traffic)
    //  IJK: e over {Pi, Rows, nz}, box {TX+4, 1, nz}
    //  KIJ: e over {Pk, nx+4, ny+4}, box {Pk, TX+2, 1} (one contiguous block)
    //  sf/pb over {row pitch, rows}, box {TX+4, 1}
    const cuuint32_t estr[3] = {1, 1, 1};
    cuuint64_t dims3[3], strides3[2];
    cuuint32_t box3[3];
    if (!kij) {
        dims3[0] = (cuuint64_t)c->Pi;
        dims3[1] = (cuuint64_t)c->Rows;
        dims3[2] = (cuuint64_t)nz;
        strides3[0] = (cuuint64_t)c->Pi * 8;
        strides3[1] = (cuuint64_t)(c->Pi * c->Rows) * 8;
        box3[0] = (cuuint32_t)G.w;
        box3[1] = 1;
        box3[2] = (cuuint32_t)nz;
    } else {
        dims3[0] = (cuuint64_t)pk;
        dims3[1] = (cuuint64_t)(c->lnx + 4);
        dims3[2] = (cuuint64_t)(c->lny + 4);
        strides3[0] = (cuuint64_t)pk * 8;
        strides3[1] = (cuuint64_t)c->sj * 8;
        box3[0] = (cuuint32_t)pk;
        box3[1] = (cuuint32_t)(tx + 2);
        box3[2] = 1;
    }
    for (int b = 0; b < 2; ++b) {
        CUresult r = enc(&c->tm_e[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, c->buf[b], dims3,
                         strides3, box3, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return HFTW_OK;
    }
    const cuuint64_t dims2[2] = {(cuuint64_t)c->s2j, (cuuint64_t)(kij ? c->lny + 4 : c->Rows)};
    const cuuint64_t strides2[1] = {(cuuint64_t)c->s2j * 8};
    const cuuint32_t box2[2] = {(cuuint32_t)(tx + 4), 1};
    if (enc(&c->tm_sf, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, c->sf, dims2, strides2, box2, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return HFTW_OK;
    if (enc(&c->tm_pb, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, c->pb, dims2, strides2, box2, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return HFTW_OK;

    // Dynamic j-major work units (strip x chunk of rows), one persistent CTA
    // per SM slot; the scheduler counters live in device memory and re-arm
    // themselves at the end of every launch.
    const long long nx = c->lnx, ny = c->lny;
    const int nstrips = (int)((nx + tx - 1) / tx);
    // Rows per unit: minimise (waves of units over the resident CTAs) x (rows
    // + 2 halo slabs per unit), preferring long units on ties.  ASUCA picks
    // 32 (1025 units ~ 7 waves); 256x256 picks 7 (148 units = one wave).
    long long chunk = env_int("HFTW_CHUNK", 0);
    if (chunk <= 0) {
        const long long slots = (long long)per_sm * c->num_sms;
        double best = 1e30;
        for (long long ch = std::min<long long>(kChunk, ny); ch >= 1; --ch) {
            const long long units = (long long)nstrips * ((ny + ch - 1) / ch);
            const double waves = (double)((units + slots - 1) / slots);
            const double cost = waves * (double)(ch + 2);
            if (cost < best - 1e-9) {
                best = cost;
                chunk = ch;
            }
        }
    }
    c->chunk = (int)std::min<long long>(chunk, ny);
    c->nchunks = (int)((ny + c->chunk - 1) / c->chunk);
    const long long units = (long long)nstrips * c->nchunks;
    int ctas = (int)std::min<long long>((long long)per_sm * c->num_sms, units);
    if (!c->d_sched) {
        CUDA_TRY(c, cudaMalloc(&c->d_sched, 2 * sizeof(int)));
        CUDA_TRY(c, cudaMemset(c->d_sched, 0, 2 * sizeof(int)));
    }
    c->ctas = ctas;
    c->nstrips = nstrips;
    c->tma_ok = true;
    return HFTW_OK;
}

// A launch that may start while the previous one on the stream finishes (programmatic
// dependent launch; the kernel waits for it before touching global memory), or a
// plain launch when HFTW_PDL is 0.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t stream, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = HFTW_PDL ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

using PairKernel = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap,
                           const CUtensorMap, const double*, double*, const double*,
                           const double*, Dom, hftw::PairArgs, const Halo);
// form (single domain): kPairIn = e_s is stored post-physics, kPairOut = store
// e_{s+2} post-physics (the passes of one call between its first and last)
constexpr int kPairIn = 1, kPairOut = 2;
PairKernel pair_kernel(bool dist, int form = 0) {
    using namespace hftw;
    if (dist) switch (form) {
        case kPairIn: return step_pair_kernel<kPairKPT, true, true, false>;
        case kPairOut: return step_pair_kernel<kPairKPT, true, false, true>;
        case kPairIn | kPairOut: return step_pair_kernel<kPairKPT, true, true, true>;
        default: return step_pair_kernel<kPairKPT, true, false, false>;
        }
    switch (form) {
    case kPairIn: return step_pair_kernel<kPairKPT, false, true, false>;
    case kPairOut: return step_pair_kernel<kPairKPT, false, false, true>;
    case kPairIn | kPairOut: return step_pair_kernel<kPairKPT, false, true, true>;
    default: return step_pair_kernel<kPairKPT, false, false, false>;
    }
}

// The two-steps-per-pass kernel (weather_pair.cuh): IJK, single domain, nz
// <= 64 (8 k values per thread), and a >= 4-deep slab ring next to the two
// intermediate row buffers.  Leaves pair_ok = false otherwise.
int setup_pair(hftw_ctx* c) {
    c->pair_ok = false;
    if (!c->tma_ok || c->layout != HFTW_IJK || c->nz > hftw::kPairKG * kPairKPT) return HFTW_OK;
    // the kernel's final-row stores index planes with int offsets (kk * plane stride)
    if ((long long)kPairKPT * c->Pi * c->Rows > 0x7fffffffLL) return HFTW_OK;
    if (c->dist) {
        // every rank of the decomposition must take the same decision: two-step
        // passes need 2 owned cells next to every interior face of every rank
        // (the smallest balanced part is floor(n / p))
        const hftw_plan& p = c->plan;
        if ((p.px > 1 && c->g.nx / p.px < 2) || (p.py > 1 && c->g.ny / p.py < 2)) return HFTW_OK;
    }
    auto enc = encode_fn();
    int smem_optin = 0;
    CUDA_TRY(c, cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                                       c->device));
    auto kern = pair_kernel(c->dist);
    cudaFuncAttributes fa{};
    CUDA_TRY(c, cudaFuncGetAttributes(&fa, kern));
    const int nz = (int)c->nz;
    int ns = 0;
    // narrow tiles: the deepest ring that still lets kPairMinBlocks CTAs share an SM
    int smem_sm = 0;
    CUDA_TRY(c, cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor,
                                       c->device));
    const size_t per_cta = std::min<size_t>((size_t)smem_optin,
                                            (size_t)smem_sm / hftw::kPairMinBlocks - 1024);
    for (int cand = std::min(8, env_int("HFTW_PAIR_NS", 8)); cand >= 4; --cand)
        if (hftw::pair_smem_bytes(nz, cand) + fa.sharedSizeBytes <= per_cta) {
            ns = cand;
            break;
        }
    if (!ns) return HFTW_OK;
    c->pair_ns = ns;
    c->pair_smem = hftw::pair_smem_bytes(nz, ns);
    for (int form = 0; form < 4; ++form)
        CUDA_TRY(c, raise_smem_attr((const void*)pair_kernel(c->dist, form), c->pair_smem));
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, hftw::kPairThreads,
                                                      c->pair_smem) != cudaSuccess ||
        per_sm < 1) {
        cudaGetLastError();
        return HFTW_OK;
    }
    const cuuint32_t estr[3] = {1, 1, 1};
    const cuuint64_t dims3[3] = {(cuuint64_t)c->Pi, (cuuint64_t)c->Rows, (cuuint64_t)nz};
    const cuuint64_t strides3[2] = {(cuuint64_t)c->Pi * 8, (cuuint64_t)(c->Pi * c->Rows) * 8};
    const cuuint32_t box3[3] = {2, 1, (cuuint32_t)nz};
    const cuuint32_t box3s[3] = {(cuuint32_t)hftw::kPairW, 1, (cuuint32_t)nz};
    for (int b = 0; b < 2; ++b)
        if (enc(&c->tm_e2[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, c->buf[b], dims3, strides3, box3s,
                estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return HFTW_OK;
    for (int b = 0; b < 2; ++b)
        if (enc(&c->tm_ef[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, c->buf[b], dims3, strides3, box3,
                estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return HFTW_OK;
    // [sf; pb] as one 3D tensor {row pitch, rows, 2}: a slab's two boundary rows
    // (box {TX+4, 1, 2}) and the far column's two values (box {2, 1, 2})
    const cuuint64_t dimsb[3] = {(cuuint64_t)c->s2j, (cuuint64_t)c->Rows, 2};
    const cuuint64_t stridesb[2] = {(cuuint64_t)c->s2j * 8, (cuuint64_t)c->n2 * 8};
    const cuuint32_t boxb[3] = {(cuuint32_t)hftw::kPairW, 1, 2};
    const cuuint32_t boxbf[3] = {2, 1, 2};
    if (enc(&c->tm_sfpb, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, c->sf, dimsb, stridesb, boxb, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
        enc(&c->tm_sfpbf, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, c->sf, dimsb, stridesb, boxbf, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return HFTW_OK;
    c->pair_nstrips = (int)((c->lnx + hftw::kPairTX - 1) / hftw::kPairTX);
    // rows per unit: as for the single-step kernel, with 4 halo slabs per unit
    const long long ny = c->lny;
    long long chunk = env_int("HFTW_PAIR_CHUNK", 0);
    const long long slots = (long long)per_sm * c->num_sms;
    if (chunk <= 0) {
        // Rows per unit by how many waves of 16-row units a pass has (measured with
        // tools/group_diag.py, tools/ab_step.py and HFTW_PAIR_CHUNK / _CHUNK2,
        // profiles/r02_chunk_sweep.txt): >= 5 waves 24 rows (ASUCA, 14.7 waves, with
        // post-physics storage between passes: 0.2431 ms/step vs 0.2493 at 16, 0.2461
        // at 32 and 0.2559 at 12, each with half-height tail units), 2.5-5 waves 12
        // (a 2x2 rank: 0.187 vs 0.192 at 16), fewer 8 (a 2x4 rank: 0.122 vs 0.133):
        // short passes need more units to fill both CTAs of every SM.
        const double w16 = (double)((long long)c->pair_nstrips * ((ny + 15) / 16)) / (double)slots;
        chunk = w16 >= 5.0 ? 24 : w16 >= 2.5 ? 12 : 8;
    }
    c->pair_chunk = (int)std::min<long long>(chunk, ny);
    // the last ~1.5 waves of units get half-height chunks (a shorter tail)
    c->pair_chunk2 = std::max(1, env_int("HFTW_PAIR_CHUNK2", (c->pair_chunk + 1) / 2));
    const long long tail_rows = std::min<long long>(
        ny, ((3 * slots / 2 + c->pair_nstrips - 1) / c->pair_nstrips) * c->pair_chunk2);
    c->pair_nbig = (int)((ny - tail_rows) / c->pair_chunk);
    const long long rest = ny - (long long)c->pair_nbig * c->pair_chunk;
    c->pair_nchunks = c->pair_nbig + (int)((rest + c->pair_chunk2 - 1) / c->pair_chunk2);
    const long long units = (long long)c->pair_nstrips * c->pair_nchunks;
    c->pair_ctas = (int)std::min<long long>(slots, units);
    const size_t ints = 2 + (size_t)c->pair_nchunks + (size_t)c->pair_nstrips;
    CUDA_TRY(c, cudaMalloc(&c->d_pair, ints * sizeof(int)));
    CUDA_TRY(c, cudaMemset(c->d_pair, 0, ints * sizeof(int)));
    c->gpub_n = (size_t)(4 * (ny + 2) * c->nz) + (size_t)(4 * c->nz * (c->lnx + 2));
    CUDA_TRY(c, cudaMalloc(&c->gpub, 2 * c->gpub_n * sizeof(double)));
    // the compile-time row shapes cover groups of KPT-1 .. KPT planes; other nz run
    // the generic (runtime plane checks) path, which AUTO leaves to the TMA kernel
    c->pair_fast = c->nz >= (long long)hftw::kPairKG * (kPairKPT - 1);
    c->pair_ok = true;
    return HFTW_OK;
}

int resolved_kernel(const hftw_ctx* c) {
    if (c->kernel_req == HFTW_KERNEL_AUTO)
        return c->pair_ok && c->pair_auto && c->pair_fast ? HFTW_KERNEL_FUSED_PAIR
                          : c->tma_ok ? HFTW_KERNEL_FUSED_TMA : HFTW_KERNEL_FUSED_CELL;
    return c->kernel_req;
}

// Measurement hook: events around one launch (kind 0 = single step, 1 = pair
// pass, 2 = multi-step) and the steps it covers.
int timing_mark(hftw_ctx* c, int kind, bool begin, int64_t steps = 1) {
    if (!c->timing) return HFTW_OK;
    if (begin) {
        cudaEvent_t a, b;
        CUDA_TRY(c, cudaEventCreate(&a));
        CUDA_TRY(c, cudaEventCreate(&b));
        c->tev.push_back({kind, a, b, steps});
        CUDA_TRY(c, cudaEventRecord(a, c->stream));
    } else {
        c->tev.back().steps = steps;
        CUDA_TRY(c, cudaEventRecord(c->tev.back().b, c->stream));
    }
    return HFTW_OK;
}

// The published-P' buffer of a pass (two parities of `per` doubles; see hftw_ctx::gpub).
double* gpub_of(double* base, size_t per, long long pass) {
    return base + (size_t)(pass & 1) * per;
}

// Two fused steps in one launch: buf[src] -> buf[src ^ 1] = step(step(buf[src])),
// either side stored post-physics as `form` says (pair_kernel).
int launch_pair(hftw_ctx* c, int src, int form) {
    Dom d = make_dom(c);
    hftw::PairArgs a{};
    a.fp = kFrontPad;
    a.jrow0 = 1;
    a.nstrips = c->pair_nstrips;
    a.nchunks = c->pair_nchunks;
    a.chunk = c->pair_chunk;
    a.nbig = c->pair_nbig;
    a.chunk2 = c->pair_chunk2;
    a.ns = c->pair_ns;
    a.sched = c->d_pair;
    a.reverse = c->opt_reverse;
    a.cnt_col = c->d_pair + 2;
    a.cnt_row = c->d_pair + 2 + c->pair_nchunks;
    double* pub = gpub_of(c->gpub, c->gpub_n, c->pass_count);
    a.gcol = pub;
    a.grow = pub + 4 * (c->lny + 2) * c->nz;
    const Halo h = make_halo(c, src ^ 1); // pushes into the neighbours' e_{s+2}, waits >= s
    int rc = timing_mark(c, 1, true);
    if (rc) return rc;
    auto kern = pair_kernel(c->dist, form);
    CUDA_TRY(c, launch_pdl(kern, c->pair_ctas, hftw::kPairThreads, c->pair_smem, c->stream,
                           c->tm_e2[src], c->tm_sfpb, c->tm_ef[src], c->tm_sfpbf,
                           (const double*)e3(c, src), e3(c, src ^ 1), (const double*)sf2(c),
                           (const double*)pb2(c), d, a, h));
    CUDA_TRY(c, cudaGetLastError());
    return timing_mark(c, 1, false, 2);
}

// Decomposed pair pass, second launch: the ghost cells of e_{s+2} from this
// rank's and the wrap partners' published P', their pushes, and the release
// of the pass to every neighbour (weather_pair.cuh, pair_ghost_kernel).
int launch_pair_ghost(hftw_ctx* c, int dst, int form) {
    const Dom d = make_dom(c);
    Halo h = make_halo(c, dst);
    h.step = c->step_count + 1; // releases s + 2
    hftw::PairGhostArgs g{};
    const long long ncol = 4 * (c->lny + 2) * c->nz;
    double* mine = gpub_of(c->gpub, c->gpub_n, c->pass_count);
    g.gcol = mine;
    g.grow = mine + ncol;
    // the wrap partner of each owned edge: a remote rank (its published P' over
    // NVLink, after its "published" flag), or this rank along an undivided axis.
    // The partner along i has this rank's rows, the one along j its columns.
    const hftw_plan& p = c->plan;
    const int dirs[4] = {HFTW_W, HFTW_E, HFTW_S, HFTW_N};
    const double* part[4];
    for (int q : dirs) {
        const PeerMap& m = c->peer[q];
        const bool remote = m.rank >= 0 && p.depth[q] == 1;
        if (remote && !m.gpub)
            return fail(c, HFTW_ESTATE, "rank %d has no published-P' buffer", m.rank);
        const double* base = remote ? gpub_of(m.gpub, (size_t)m.gpub_n, c->pass_count) : mine;
        part[q] = q < 2 ? base : base + (remote ? m.gcol_n : ncol);
        g.wait[q] = remote ? 1 : 0;
    }
    g.gcol_w = part[HFTW_W];
    g.gcol_e = part[HFTW_E];
    g.grow_s = part[HFTW_S];
    g.grow_n = part[HFTW_N];
    g.pub = c->step_count + 2;
    const long long cells = 2 * (c->lny + 2 + c->lnx) * c->nz;
    // few CTAs: each polls the wrap partners' flags (system-scope acquires) once
    const int blocks = (int)std::max<long long>(
        1, std::min<long long>((cells + 1023) / 1024,
                               (long long)env_int("HFTW_GHOST_CTAS", c->num_sms / 2)));
    if (form & kPairOut)
        hftw::pair_ghost_kernel<true><<<blocks, 256, 0, c->stream>>>(e3(c, dst), sf2(c), pb2(c),
                                                                     d, h, g);
    else
        hftw::pair_ghost_kernel<false><<<blocks, 256, 0, c->stream>>>(e3(c, dst), sf2(c), pb2(c),
                                                                      d, h, g);
    CUDA_TRY(c, cudaGetLastError());
    return HFTW_OK;
}

// Two-step passes of an n-step call: n/2 when n is even, else (n-1)/2 and a final
// single step.  After a pass, energy_u (physics of e_{n-1}, which the pass kept
// on chip) is recomputed only if it is read: e_{n-2} is still in the ping-pong
// partner (materialize_eu).
int64_t pair_passes(int64_t nsteps) { return nsteps / 2; }

// One pass: phase bit 0 launches the pair kernel, bit 1 (decomposed) the ghost
// kernel, and then the bookkeeping.  A group on one device runs bit 0 for every
// rank before bit 1 for any (the ghost kernels wait for the wrap partners').
// Storage form of pass p of `pairs` (pair_kernel): post-physics in between.
int pair_form(int64_t p, int64_t pairs) {
    return (p > 0 ? kPairIn : 0) | (p + 1 < pairs ? kPairOut : 0);
}

int pair_pass(hftw_ctx* c, int phase, int form) {
    int rc;
    if ((phase & 1) && (rc = launch_pair(c, c->cur, form))) return rc;
    if (phase & 2) {
        if (c->dist && (rc = launch_pair_ghost(c, c->cur ^ 1, form))) return rc;
        c->cur ^= 1;
        c->step_count += 2;
        ++c->pass_count;
        c->eu_stored = false;
        c->eu_derived = false;
        c->eu_pending = true;
        c->partner_pform = (form & kPairIn) != 0; // the pass's input is now the partner
    }
    return HFTW_OK;
}

// K steps per launch with the TMA kernel's tiling (weather_wave.cuh): single
// domain, IJK, same slab ring as the single-step kernel.
int setup_wave(hftw_ctx* c) {
    c->wave_ok = false;
    if (!c->tma_ok || c->layout != HFTW_IJK || c->tx != 64) return HFTW_OK;
    auto kern = hftw::step_wave_kernel<64, kNCW, true>;
    CUDA_TRY(c, raise_smem_attr((const void*)kern, c->smem));
    CUDA_TRY(c, raise_smem_attr((const void*)hftw::step_wave_kernel<64, kNCW, false>, c->smem));
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (kNCW + 1) * 32, c->smem) !=
            cudaSuccess ||
        per_sm < 1) {
        cudaGetLastError();
        return HFTW_OK;
    }
    // Long units: the launch's tail is paid once per call, not once per step,
    // and fewer chunk boundaries mean fewer halo rows re-read from HBM -- but a
    // step needs enough units to keep every CTA busy while the previous step's
    // rows complete.  The longest of 32/24/16/12/8/6 rows that gives >= 2.4 units
    // per CTA per step, else 4 (tools/wave_chunk_sweep.py: ASUCA 32 rows; the 1/4 and
    // 1/8 ranks of the 2x2 / 2x4 decompositions 24 and 12 rows, 7% and 27% faster
    // per step than 32; the 256x256x64 diffusion sweeps 4 rows: 14.4 us per sweep
    // against 17.0 at 8 and 16.6 at 2, tools/gpu_r2ae.sh).
    const long long ny = c->lny;
    long long chunk = env_int("HFTW_WAVE_CHUNK", 0);
    if (chunk <= 0) {
        const long long slots = (long long)per_sm * c->num_sms;
        chunk = 4;
        for (long long cand : {32LL, 24LL, 16LL, 12LL, 8LL, 6LL}) {
            if ((long long)c->nstrips * ((ny + cand - 1) / cand) * 10 >= slots * 24) {
                chunk = cand;
                break;
            }
        }
    }
    chunk = std::min<long long>(ny, chunk);
    c->wave_chunk = (int)chunk;
    // Prefer it over one launch per step only where a step is short: at ASUCA size
    // (6.9 units of 32 rows per CTA) separate launches run 0.383 ms/step against
    // 0.397 (less DRAM traffic: 1.05x vs 1.10x), while for the 1/4 and 1/8 ranks of a
    // 2x2 / 2x4 decomposition (1.8 and 1.0 units per CTA) the multi-step launch is
    // 3% and 12% faster (tools/gpu_exp10.sh).  HFTW_OPT_MULTISTEP overrides it.
    {
        const long long slots = (long long)per_sm * c->num_sms;
        const long long units32 = (long long)c->nstrips * ((ny + 31) / 32);
        c->wave_pref = units32 * 10 < slots * 27;
    }
    c->wave_nchunks = (int)((ny + chunk - 1) / chunk);
    c->wave_gtasks = std::max(1, std::min(16, (int)((c->lnx + 2) * c->nz / 2048)));
    const long long units = (long long)c->nstrips * c->wave_nchunks + c->wave_gtasks;
    c->wave_ctas = (int)std::min<long long>((long long)per_sm * c->num_sms, units);
    const size_t ints = 2 + (size_t)c->wave_nchunks + 1 + kMaxWaveStepsDist;
    CUDA_TRY(c, cudaMalloc(&c->d_wave, ints * sizeof(int)));
    CUDA_TRY(c, cudaMemset(c->d_wave, 0, ints * sizeof(int)));
    c->wave_ok = true;
    return HFTW_OK;
}

// nsteps single steps in ONE launch (buf[src] holds the field of step 0);
// phys = false: diffusion-only sweeps.
int launch_wave(hftw_ctx* c, int src, int64_t nsteps, bool phys = true) {
    Dom d = make_dom(c);
    hftw::WaveArgs a{};
    a.fp = kFrontPad;
    a.jrow0 = 1;
    a.nstrips = c->nstrips;
    a.nchunks = c->wave_nchunks;
    a.chunk = c->wave_chunk;
    a.ns = c->ns;
    a.nsteps = (int)nsteps;
    a.gtasks = c->wave_gtasks;
    a.alt = env_int("HFTW_WAVE_ALT", 1);
    a.sched = c->d_wave;
    a.chunk_done = c->d_wave + 2;
    a.ghost_done = c->d_wave + 2 + c->wave_nchunks;
    a.buf0 = e3(c, src);
    a.buf1 = e3(c, src ^ 1);
    a.h_even = make_halo(c, src ^ 1); // even steps write buf1
    a.h_odd = make_halo(c, src);      // odd steps write buf0
    a.step_done = c->d_wave + 2 + c->wave_nchunks + 1;
    int rc = timing_mark(c, 2, true);
    if (rc) return rc;
    auto kern = phys ? hftw::step_wave_kernel<64, kNCW, true> : hftw::step_wave_kernel<64, kNCW, false>;
    CUDA_TRY(c, launch_pdl(kern, c->wave_ctas, (kNCW + 1) * 32, c->smem, c->stream, c->tm_e[src],
                           c->tm_e[src ^ 1], c->tm_sf, c->tm_pb, (const double*)sf2(c),
                           (const double*)pb2(c), d, a));
    CUDA_TRY(c, cudaGetLastError());
    return timing_mark(c, 2, false, nsteps);
}


// The part of one step a TMA launch covers: work units [u_lo, u_hi) of the
// j-major order (chunk-major: unit = chunk * nstrips + strip), the i-ghost
// columns of inner rows [gi_lo, gi_hi] and the j-ghost rows in gj_mask.
struct StepPart {
    int u_lo, u_hi, gi_lo, gi_hi, gj_mask;
};
StepPart whole_step(const hftw_ctx* c) {
    return {0, c->nstrips * c->nchunks, 1, (int)c->lny, 3};
}

hftw::TmaArgs tma_args(const hftw_ctx* c, const StepPart& p) {
    const hftw_plan& pl = c->plan;
    const Box o = owned_box(c);
    const long long gs = (p.gj_mask & 1) && pl.own_s, gn = (p.gj_mask & 2) && pl.own_n;
    const long long r0 = std::max<long long>(p.gi_lo, 1), r1 = std::min<long long>(p.gi_hi, c->lny);
    const long long nr = std::max<long long>(0, r1 - r0 + 1);
    const long long ghost = ((gs + gn) * (o.i1 - o.i0 + 1) + (long long)(pl.own_w + pl.own_e) * nr) *
                            c->nz;
    hftw::TmaArgs a{};
    a.fp = kFrontPad;
    a.jrow0 = 1;
    a.nstrips = c->nstrips;
    a.nchunks = c->nchunks;
    a.chunk = c->chunk;
    a.ns = c->ns;
    a.pk = (int)c->Pk;
    a.ghost_cells = ghost;
    a.sched = c->d_sched;
    a.reverse = c->opt_reverse;
    a.u_lo = p.u_lo;
    a.u_hi = p.u_hi;
    a.gi_lo = p.gi_lo;
    a.gi_hi = p.gi_hi;
    a.gj_mask = p.gj_mask;
    return a;
}

// Launch the fused update from buf[src] into buf[src^1]; PHYS=false is the
// diffusion-only sweep of an already post-physics field.  `part` restricts a
// TMA launch to a piece of the step (NULL = the whole step).
// `out` (optional): write the step there instead of buf[src ^ 1], with no halo
// protocol (energy_u materialisation: the halos of buf[src] are complete).
template <bool PHYS>
int launch_fused(hftw_ctx* c, int src, int kernel, const StepPart* part = nullptr,
                 double* out = nullptr, bool no_halo = false) {
    Dom d = make_dom(c);
    Halo h = out || no_halo ? Halo{} : make_halo(c, src ^ 1);
    double* const dst = out ? out : e3(c, src ^ 1);
    if (kernel == HFTW_KERNEL_FUSED_TMA) {
        if (!c->tma_ok) return fail(c, HFTW_EUNSUP, "TMA kernel unavailable for this grid/layout");
        const StepPart p = part ? *part : whole_step(c);
        const hftw::TmaArgs a = tma_args(c, p);
        // a piece with few units needs few CTAs (the ghost cells are grid-strided)
        const long long want = std::max<long long>(p.u_hi - p.u_lo, (a.ghost_cells + 4095) / 4096);
        const int ctas = (int)std::max<long long>(1, std::min<long long>(c->ctas, want));
        dim3 block((kNCW + 1) * 32);
#define HFTW_LAUNCH_TMA(TX, KIJ)                                                              \
    launch_pdl(hftw::step_tma_kernel<TX, kNCW, PHYS, KIJ>, ctas, block, c->smem, c->stream,    \
               c->tm_e[src], c->tm_sf, c->tm_pb, (const double*)e3(c, src), dst,              \
               (const double*)sf2(c), (const double*)pb2(c), d, a, h)
        const bool kij = c->layout == HFTW_KIJ;
        if (c->tx == 64) {
            if (kij) HFTW_LAUNCH_TMA(64, true);
            else HFTW_LAUNCH_TMA(64, false);
        } else {
            if (kij) HFTW_LAUNCH_TMA(32, true);
            else HFTW_LAUNCH_TMA(32, false);
        }
#undef HFTW_LAUNCH_TMA
    } else {
        const long long n = (c->lnx + 2) * (c->lny + 2) * c->nz;
        // a decomposed run's CTAs spin on neighbour flags, so they must all
        // be resident: cap the grid at the SM count x a safe occupancy
        const int blocks = c->dist ? std::min(grid_for(c, n), c->num_sms * 4) : grid_for(c, n);
        if (c->layout == HFTW_KIJ)
            hftw::step_cell_kernel<true, PHYS><<<blocks, 256, 0, c->stream>>>(
                e3(c, src), dst, sf2(c), pb2(c), d, h);
        else
            hftw::step_cell_kernel<false, PHYS><<<blocks, 256, 0, c->stream>>>(
                e3(c, src), dst, sf2(c), pb2(c), d, h);
    }
    CUDA_TRY(c, cudaGetLastError());
    return HFTW_OK;
}

// the faster physics mapping for the layout (DESIGN.md results): IJK one
// column per thread (0.366 ms at ASUCA), KIJ streamed rows (0.395 ms)
int best_physics_mode(const hftw_ctx* c) { return c->layout == HFTW_KIJ ? 1 : 0; }

int launch_physics(hftw_ctx* c, double* e, int mode) {
    Dom d = make_dom(c);
    const long long cols = (c->lnx + 2) * (c->lny + 2);
    if (mode == 0) {
        CUDA_TRY(c, launch_pdl(hftw::physics_column_kernel, grid_for(c, cols), 256, 0, c->stream,
                               e, (const double*)sf2(c), (const double*)pb2(c), d));
    } else if (c->layout == HFTW_KIJ) {
        if (c->Pk >= 32 && env_int("HFTW_KIJ_PHYS_WARP", 0) == 0) { // streaming rows
            const long long tasks = (c->lny + 2) * ((c->lnx + 2 + 15) / 16);
            CUDA_TRY(c, launch_pdl(hftw::physics_kij_stream_kernel,
                                   (int)std::min<long long>((tasks + 7) / 8,
                                                            (long long)c->num_sms * 16),
                                   256, 0, c->stream, e, (const double*)sf2(c),
                                   (const double*)pb2(c), d, (int)c->Pk));
            CUDA_TRY(c, cudaGetLastError());
            return HFTW_OK;
        }
        hftw::physics_kij_kernel<<<grid_for(c, cols * 32), 256, 0, c->stream>>>(e, sf2(c),
                                                                               pb2(c), d);
    } else {
        const long long rows = (c->lny + 2) * c->nz;
        const int blocks = (int)std::min<long long>(rows, (long long)c->num_sms * 16);
        hftw::physics_rows_kernel<<<blocks, 256, 0, c->stream>>>(e, sf2(c), pb2(c), d);
    }
    CUDA_TRY(c, cudaGetLastError());
    return HFTW_OK;
}

// energy_u after a fused step is physics(previous energy); compute it in place
// in the buffer that holds the previous energy (it is dead until the next step
// overwrites it, so this is free of hazards; only owned cells are touched).
int materialize_eu(hftw_ctx* c) {
    int rc;
    if (c->eu_pending) {
        // after pair passes: energy_u = physics(e_{n-1}) and e_{n-1} = step(e_{n-2}),
        // which the ping-pong partner still holds (with its halos): one step into the
        // third buffer, then physics in place there
        if (!c->eu_buf) {
            if (cudaMalloc(&c->eu_buf, c->n3 * sizeof(double)) != cudaSuccess) {
                cudaGetLastError();
                c->eu_buf = nullptr;
                return fail(c, HFTW_ENOMEM, "cudaMalloc of the energy_u buffer (%zu bytes) failed",
                            c->n3 * sizeof(double));
            }
        }
        double* out = c->eu_buf + c->off3;
        const int k1 = c->tma_ok ? HFTW_KERNEL_FUSED_TMA : HFTW_KERNEL_FUSED_CELL;
        // the partner holds P(e_{n-2}) when the last pass read a post-physics field:
        // then the step is the diffusion sweep alone
        if ((rc = c->partner_pform ? launch_fused<false>(c, c->cur ^ 1, k1, nullptr, out)
                                   : launch_fused<true>(c, c->cur ^ 1, k1, nullptr, out)))
            return rc;
        if ((rc = launch_physics(c, out, best_physics_mode(c)))) return rc;
        c->eu_pending = false;
        c->eu_stored = true;
        return HFTW_OK;
    }
    if (!c->eu_derived) return HFTW_OK; // materialised already
    if ((rc = launch_physics(c, e3(c, c->cur ^ 1), best_physics_mode(c)))) return rc;
    c->eu_derived = false;
    return HFTW_OK;
}

int check_ctx(hftw_ctx* c) {
    if (!c) return fail(nullptr, HFTW_EINVAL, "null context");
    CUDA_TRY(c, cudaSetDevice(c->device));
    return HFTW_OK;
}

// Calls that read the device state refuse it after a failed hftw_step_host.
int check_state(hftw_ctx* c) {
    if (c->poisoned)
        return fail(c, HFTW_ESTATE, "device state undefined after a failed hftw_step_host: "
                                    "call hftw_init or upload all four fields");
    return HFTW_OK;
}

bool is_group(const hftw_ctx* c) { return c && !c->ranks.empty(); }

// partition of n inner cells over p ranks (balanced; every rank >= 1 cell)
long long part_lo(long long n, int p, int r) { return 1 + (long long)r * n / p; }
long long part_hi(long long n, int p, int r) { return (long long)(r + 1) * n / p; }

int make_plan(const hftw_grid* g, int px, int py, int rank, hftw_plan* o) {
    if (px < 1 || py < 1 || rank < 0 || rank >= px * py)
        return fail(nullptr, HFTW_EINVAL, "bad decomposition %dx%d rank %d", px, py, rank);
    if (px > g->nx || py > g->ny)
        return fail(nullptr, HFTW_EINVAL, "decomposition %dx%d finer than the %lldx%lld interior",
                    px, py, (long long)g->nx, (long long)g->ny);
    hftw_plan p{};
    p.px = px;
    p.py = py;
    p.rank = rank;
    p.rx = rank % px;
    p.ry = rank / px;
    const long long ilo = part_lo(g->nx, px, p.rx), ihi = part_hi(g->nx, px, p.rx);
    const long long jlo = part_lo(g->ny, py, p.ry), jhi = part_hi(g->ny, py, p.ry);
    p.gi0 = ilo - 1;
    p.gj0 = jlo - 1;
    p.lnx = ihi - ilo + 1;
    p.lny = jhi - jlo + 1;
    p.own_w = p.rx == 0;
    p.own_e = p.rx == px - 1;
    p.own_s = p.ry == 0;
    p.own_n = p.ry == py - 1;
    // cyclic partners of the ghost cells (weather.cpp:155-167): local with one
    // rank in that direction, else the far halo slot the wrap neighbour fills
    p.wfar = px == 1 ? (int)p.lnx : -1;
    p.efar = px == 1 ? 1 : (int)p.lnx + 2;
    p.sfar = py == 1 ? (int)p.lny : -1;
    p.nfar = py == 1 ? 1 : (int)p.lny + 2;
    const int rxw = (p.rx - 1 + px) % px, rxe = (p.rx + 1) % px;
    const int rys = (p.ry - 1 + py) % py, ryn = (p.ry + 1) % py;
    p.nbr[HFTW_W] = px > 1 ? p.ry * px + rxw : -1;
    p.nbr[HFTW_E] = px > 1 ? p.ry * px + rxe : -1;
    p.nbr[HFTW_S] = py > 1 ? rys * px + p.rx : -1;
    p.nbr[HFTW_N] = py > 1 ? ryn * px + p.rx : -1;
    // where my faces land in the neighbour (its local coordinates)
    const long long lnx_w = part_hi(g->nx, px, rxw) - part_lo(g->nx, px, rxw) + 1;
    const long long lny_s = part_hi(g->ny, py, rys) - part_lo(g->ny, py, rys) + 1;
    p.send_slot[HFTW_W] = rxw == px - 1 ? (int)lnx_w + 2 : (int)lnx_w + 1; // its E / E-far slot
    p.send_slot[HFTW_E] = rxe == 0 ? -1 : 0;                               // its W-far / W slot
    p.send_slot[HFTW_S] = rys == py - 1 ? (int)lny_s + 2 : (int)lny_s + 1;
    p.send_slot[HFTW_N] = ryn == 0 ? -1 : 0;
    // faces span the owned cells along them, the owned global ghost row /
    // column included: a two-step pass's halo intermediates read them
    p.face_lo[HFTW_W] = p.face_lo[HFTW_E] = p.own_s ? 0 : 1;
    p.face_hi[HFTW_W] = p.face_hi[HFTW_E] = p.own_n ? p.lny + 1 : p.lny;
    p.face_lo[HFTW_S] = p.face_lo[HFTW_N] = p.own_w ? 0 : 1;
    p.face_hi[HFTW_S] = p.face_hi[HFTW_N] = p.own_e ? p.lnx + 1 : p.lnx;
    // layers per face: a wrap partner needs only its far slot (1); an interior
    // neighbour reads 2 layers in a two-step pass (1 where this rank is 1 wide)
    const auto layers = [](int np, bool own, long long ext) {
        return np == 1 ? 0 : own ? 1 : (int)std::min<long long>(2, ext);
    };
    p.depth[HFTW_W] = layers(px, p.own_w, p.lnx);
    p.depth[HFTW_E] = layers(px, p.own_e, p.lnx);
    p.depth[HFTW_S] = layers(py, p.own_s, p.lny);
    p.depth[HFTW_N] = layers(py, p.own_n, p.lny);
    // diagonal neighbours across two interior faces get one corner column
    const bool iw = px > 1 && !p.own_w, ie = px > 1 && !p.own_e;
    const bool is = py > 1 && !p.own_s, in = py > 1 && !p.own_n;
    p.diag[HFTW_SW] = iw && is ? rys * px + rxw : -1;
    p.diag[HFTW_SE] = ie && is ? rys * px + rxe : -1;
    p.diag[HFTW_NW] = iw && in ? ryn * px + rxw : -1;
    p.diag[HFTW_NE] = ie && in ? ryn * px + rxe : -1;
    p.diag_slot[HFTW_SW][0] = (int)lnx_w + 1;
    p.diag_slot[HFTW_SW][1] = (int)lny_s + 1;
    p.diag_slot[HFTW_SE][0] = 0;
    p.diag_slot[HFTW_SE][1] = (int)lny_s + 1;
    p.diag_slot[HFTW_NW][0] = (int)lnx_w + 1;
    p.diag_slot[HFTW_NW][1] = 0;
    p.diag_slot[HFTW_NE][0] = 0;
    p.diag_slot[HFTW_NE][1] = 0;
    *o = p;
    return HFTW_OK;
}

// Allocate and lay out the local store (shared by create and create_dist).
int create_common(const hftw_grid* g, int layout, int device, const hftw_plan& plan, bool dist,
                  hftw_ctx** out) {
    if (!out) return fail(nullptr, HFTW_EINVAL, "null output pointer");
    *out = nullptr;
    char msg[512];
    if (hftw_validate(g, msg, sizeof msg) != HFTW_OK) return fail(nullptr, HFTW_EINVAL, "%s", msg);
    if (layout != HFTW_IJK && layout != HFTW_KIJ)
        return fail(nullptr, HFTW_EINVAL, "unknown layout %d", layout);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(nullptr, HFTW_ECUDA,
                    "no CUDA device available (the B200 path has no CPU fallback)");
    }
    if (device < 0 || device >= ndev) return fail(nullptr, HFTW_EINVAL, "bad device %d", device);

    hftw_ctx* c = new hftw_ctx();
    c->g = *g;
    c->plan = plan;
    c->dist = dist;
    c->layout = layout;
    c->device = device;
    c->lnx = plan.lnx;
    c->lny = plan.lny;
    c->nz = g->nz;
    auto bail = [&](int rc) {
        g_err = c->err;
        hftw_destroy(c);
        return rc;
    };
    if (cudaSetDevice(device) != cudaSuccess)
        return bail(fail(c, HFTW_ECUDA, "cudaSetDevice failed"));
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
        return bail(fail(c, HFTW_ECUDA, "stream creation failed"));
    c->own_stream = true;

    const long long nx = c->lnx, ny = c->lny, nz = c->nz;
    if (layout == HFTW_IJK) {
        // rows hold i = -1 .. nx+2 with logical i = 1 at element 32 (256 B)
        c->Pi = ((kFrontPad + nx + 3) + 31) / 32 * 32;
        c->Rows = ny + 4; // j = -1 .. ny+2
        c->si = 1;
        c->sj = c->Pi;
        c->sk = c->Pi * c->Rows;
        c->s2j = c->Pi;
        c->off3 = c->Pi * 1 + kFrontPad;
        c->off2 = c->off3;
        c->n3 = (size_t)(c->sk * nz);
        c->n2 = (size_t)c->sk;
    } else {
        // raw tuple (k, i, j), k fastest.  Column pitch Pk = 2 (mod 4) doubles
        // (even for 16-byte TMA strides; odd multiple of 2 so lanes walking
        // across columns hit distinct bank pairs); 2D rows padded to even.
        c->Pk = nz % 4 == 2 ? nz : (nz % 4 == 3 ? nz + 3 : nz + (2 - nz % 4 + 4) % 4);
        c->sk = 1;
        c->si = c->Pk;
        c->sj = c->Pk * (nx + 4);
        c->s2j = (nx + 4 + 1) / 2 * 2;
        c->off3 = c->sj + c->si; // i = -1, j = -1 slots first
        c->off2 = c->s2j + 1;
        c->n3 = (size_t)(c->sj * (ny + 4));
        c->n2 = (size_t)(c->s2j * (ny + 4));
    }
    for (int b = 0; b < 2; ++b)
        if (cudaMalloc(&c->buf[b], c->n3 * sizeof(double)) != cudaSuccess)
            return bail(fail(c, HFTW_ENOMEM, "cudaMalloc of %zu bytes failed", c->n3 * 8));
    // sf and pb share one allocation (pb = sf + n2): the pair kernel loads both
    // rows of a slab with one TMA box {TX+4, 1, 2}
    if (cudaMalloc(&c->sf, 2 * c->n2 * sizeof(double)) != cudaSuccess)
        return bail(fail(c, HFTW_ENOMEM, "cudaMalloc of 2D fields failed"));
    c->pb = c->sf + c->n2;
    if (cudaMalloc(&c->flags, hftw::kFlags * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&c->done, sizeof(int)) != cudaSuccess)
        return bail(fail(c, HFTW_ENOMEM, "cudaMalloc of halo flags failed"));
    for (int b = 0; b < 2; ++b) cudaMemsetAsync(c->buf[b], 0, c->n3 * sizeof(double), c->stream);
    cudaMemsetAsync(c->sf, 0, c->n2 * sizeof(double), c->stream);
    cudaMemsetAsync(c->pb, 0, c->n2 * sizeof(double), c->stream);
    cudaMemsetAsync(c->flags, 0, hftw::kFlags * sizeof(unsigned long long), c->stream);
    cudaMemsetAsync(c->done, 0, sizeof(int), c->stream);
    if (cudaStreamSynchronize(c->stream) != cudaSuccess)
        return bail(fail(c, HFTW_ECUDA, "initial memset failed"));
    int rc = setup_tma(c);
    if (rc) return bail(rc);
    if ((rc = setup_pair(c))) return bail(rc);
    if ((rc = setup_wave(c))) return bail(rc);
    *out = c;
    return HFTW_OK;
}

// ---- group contexts (hftw_create_multi): every rank in this process -------

// Rank of the neighbour in direction q (faces W E S N, then corners SW SE NW NE).
int nbr_rank(const hftw_plan& p, int q) { return q < 4 ? p.nbr[q] : p.diag[q - 4]; }

// Map the neighbours of rank c from the other ranks' device pointers (the
// in-process counterpart of hftw_peer_connect's IPC mappings).
void connect_local(hftw_ctx* c, const std::vector<hftw_ctx*>& ranks) {
    for (int d = 0; d < hftw::kNbrs; ++d) {
        const int r = nbr_rank(c->plan, d);
        if (r < 0) {
            c->peer[d] = PeerMap{};
            continue;
        }
        const hftw_ctx* n = ranks[(size_t)r];
        PeerMap m;
        m.rank = r;
        for (int b = 0; b < 2; ++b) m.buf[b] = n->buf[b] + n->off3;
        m.sf = n->sf + n->off2;
        m.pb = n->pb + n->off2;
        m.flags = n->flags;
        m.gpub = n->gpub;
        m.gpub_n = (long long)n->gpub_n;
        m.gcol_n = 4 * (n->lny + 2) * n->nz;
        m.si = n->si;
        m.sj = n->sj;
        m.sk = n->sk;
        m.s2j = n->s2j;
        c->peer[d] = m;
    }
    c->connected = true;
}

int create_group(const hftw_grid* g, int layout, int px, int py, const int* devices,
                 hftw_ctx** out) {
    if (!out) return fail(nullptr, HFTW_EINVAL, "null output pointer");
    *out = nullptr;
    hftw_plan whole{};
    int rc = make_plan(g, 1, 1, 0, &whole);
    if (rc) return rc;
    if (px < 1 || py < 1) return fail(nullptr, HFTW_EINVAL, "bad decomposition %dx%d", px, py);
    const int n = px * py;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(nullptr, HFTW_ECUDA,
                    "no CUDA device available (the B200 path has no CPU fallback)");
    }
    std::vector<int> dev((size_t)n);
    for (int r = 0; r < n; ++r) {
        dev[(size_t)r] = devices ? devices[r] : r;
        if (dev[(size_t)r] < 0 || dev[(size_t)r] >= ndev)
            return fail(nullptr, HFTW_EINVAL, "rank %d: bad device %d (%d visible)", r,
                        dev[(size_t)r], ndev);
    }
    hftw_ctx* c = new hftw_ctx();
    c->g = *g;
    c->plan = whole;
    c->plan.px = px;
    c->plan.py = py;
    c->plan.rank = -1;
    c->layout = layout;
    c->device = dev[0];
    c->lnx = g->nx;
    c->lny = g->ny;
    c->nz = g->nz;
    auto bail = [&](int code) {
        hftw_destroy(c);
        return code;
    };
    for (int r = 0; r < n; ++r) {
        hftw_plan p{};
        if ((rc = make_plan(g, px, py, r, &p))) return bail(rc);
        hftw_ctx* sub = nullptr;
        if ((rc = create_common(g, layout, dev[(size_t)r], p, n > 1, &sub))) {
            const std::string why = g_err;
            hftw_destroy(c);
            return fail(nullptr, rc, "rank %d: %s", r, why.c_str());
        }
        c->ranks.push_back(sub);
    }
    // Ranks on one device share its stream and run one launch per step in rank
    // order: every launch of step s then finds its neighbours' step s-1
    // complete, so no kernel ever waits on a kernel queued behind it.
    for (int r = 1; r < n; ++r)
        for (int q = 0; q < r; ++q)
            if (dev[(size_t)q] == dev[(size_t)r]) {
                hftw_ctx* sub = c->ranks[(size_t)r];
                cudaSetDevice(sub->device);
                if (sub->own_stream) cudaStreamDestroy(sub->stream);
                sub->stream = c->ranks[(size_t)q]->stream;
                sub->own_stream = false;
                c->interleave = true;
                break;
            }
    // peer access between neighbouring ranks on distinct devices (NVLink)
    for (int r = 0; r < n; ++r)
        for (int d = 0; d < hftw::kNbrs; ++d) {
            const int q = nbr_rank(c->ranks[(size_t)r]->plan, d);
            if (q < 0 || dev[(size_t)q] == dev[(size_t)r]) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, dev[(size_t)r], dev[(size_t)q]);
            if (!can)
                return bail(fail(nullptr, HFTW_EUNSUP, "device %d cannot access device %d",
                                 dev[(size_t)r], dev[(size_t)q]));
            cudaSetDevice(dev[(size_t)r]);
            const cudaError_t e = cudaDeviceEnablePeerAccess(dev[(size_t)q], 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else if (e != cudaSuccess)
                return bail(fail(nullptr, HFTW_ECUDA, "cudaDeviceEnablePeerAccess(%d -> %d): %s",
                                 dev[(size_t)r], dev[(size_t)q], cudaGetErrorString(e)));
        }
    for (hftw_ctx* sub : c->ranks) {
        connect_local(sub, c->ranks);
        sub->halo_dirty = sub->dist;
    }
    c->stream = c->ranks[0]->stream;
    c->own_stream = false;
    c->tma_ok = c->ranks[0]->tma_ok;
    c->pair_ok = c->ranks[0]->pair_ok;
    *out = c;
    return HFTW_OK;
}

// A rank's failure, reported on the group.
int rank_fail(hftw_ctx* c, const hftw_ctx* r, int rc) {
    if (!rc) return HFTW_OK;
    return fail(c, rc, "rank %d: %s", r->plan.rank, r->err.c_str());
}

#define RANK_TRY(c, r, x)                                                                      \
    do {                                                                                       \
        const int rc_ = (x);                                                                   \
        if (rc_) return rank_fail((c), (r), rc_);                                              \
    } while (0)

// Refill every rank's halos (after init / upload / physics): all devices idle,
// then each rank pushes its faces and resets its step flags.
int group_exchange(hftw_ctx* c) {
    for (hftw_ctx* r : c->ranks) RANK_TRY(c, r, hftw_sync(r));
    for (hftw_ctx* r : c->ranks) RANK_TRY(c, r, hftw_exchange(r));
    return HFTW_OK;
}

int group_step(hftw_ctx* c, int64_t nsteps) {
    if (nsteps < 0) return fail(c, HFTW_EINVAL, "steps must be nonnegative");
    if (nsteps == 0) return HFTW_OK;
    for (hftw_ctx* r : c->ranks)
        if (r->halo_dirty) {
            int rc = group_exchange(c);
            if (rc) return rc;
            break;
        }
    if (c->ranks[0]->opt_exchange == 1) {
        // the un-overlapped baseline: every rank's step without the halo
        // protocol, then its faces copied into the neighbours by a separate
        // kernel; the next step of a rank waits for its neighbours' copies
        const int k = resolved_kernel(c->ranks[0]);
        if (k != HFTW_KERNEL_FUSED_TMA && k != HFTW_KERNEL_FUSED_CELL)
            return fail(c, HFTW_EUNSUP, "HFTW_OPT_EXCHANGE = 1 takes a single-step kernel "
                                        "(hftw_set_kernel fused_tma or fused_cell)");
        for (hftw_ctx* r : c->ranks) RANK_TRY(c, r, hftw_sync(r)); // earlier pushes landed
        for (hftw_ctx* r : c->ranks)
            if (!r->xev) {
                RANK_TRY(c, r, check_ctx(r));
                if (cudaEventCreateWithFlags(&r->xev, cudaEventDisableTiming) != cudaSuccess)
                    return fail(c, HFTW_ECUDA, "event creation failed");
            }
        for (int64_t s = 0; s < nsteps; ++s) {
            for (hftw_ctx* r : c->ranks) {
                RANK_TRY(c, r, check_ctx(r));
                if (s > 0)
                    for (int q = 0; q < hftw::kNbrs; ++q) {
                        const int nr = nbr_rank(r->plan, q);
                        if (nr >= 0)
                            CUDA_TRY(c, cudaStreamWaitEvent(r->stream, c->ranks[(size_t)nr]->xev, 0));
                    }
                RANK_TRY(c, r, launch_fused<true>(r, r->cur, k, nullptr, nullptr, true));
            }
            for (hftw_ctx* r : c->ranks) {
                RANK_TRY(c, r, check_ctx(r));
                const int dst = r->cur ^ 1;
                const Halo h = make_halo(r, dst);
                const Box o = owned_box(r);
                const long long cells = 4 * (o.i1 - o.i0 + o.j1 - o.j0 + 2) * r->nz;
                hftw::face_push_kernel<<<grid_for(r, cells), 256, 0, r->stream>>>(
                    e3(r, dst), make_dom(r), h);
                CUDA_TRY(c, cudaGetLastError());
                CUDA_TRY(c, cudaEventRecord(r->xev, r->stream));
            }
            for (hftw_ctx* r : c->ranks) {
                r->cur ^= 1;
                ++r->step_count;
                r->eu_derived = true;
                r->eu_stored = false;
                r->eu_pending = false;
            }
        }
        // the next call's first steps may use the flag protocol again: every rank
        // waits for every copy, and the step flags restart from here
        return group_exchange(c);
    }
    if (c->interleave) {
        // ranks sharing a device: every launch of a pass for all ranks, in rank
        // order, before any launch that waits for it
        hftw_ctx* r0 = c->ranks[0];
        if (resolved_kernel(r0) == HFTW_KERNEL_FUSED_PAIR && r0->pair_ok) {
            const int64_t pairs = pair_passes(nsteps);
            for (int64_t p = 0; p < pairs; ++p)
                for (int phase : {1, 2})
                    for (hftw_ctx* r : c->ranks) {
                        RANK_TRY(c, r, check_ctx(r));
                        const int rc = pair_pass(r, phase, pair_form(p, pairs));
                        if (rc) {
                            // ranks already past earlier passes hold post-physics fields
                            for (hftw_ctx* q : c->ranks) q->poisoned = 0xF;
                            return rank_fail(c, r, rc);
                        }
                    }
            nsteps -= 2 * pairs;
        }
        for (int64_t s = 0; s < nsteps; ++s)
            for (hftw_ctx* r : c->ranks) RANK_TRY(c, r, hftw_step(r, 1));
    } else {
        // distinct devices: each rank queues all its steps on its own stream;
        // the kernels order themselves through the step flags
        for (hftw_ctx* r : c->ranks) RANK_TRY(c, r, hftw_step(r, nsteps));
    }
    return HFTW_OK;
}

// Host <-> device copy of the OWNED part of a 3D field (restricted to local
// rows [r0, r1] when given).  `host` is the GLOBAL logical column-major
// array; dev_logical points at local (0,0,1).
int copy_3d(hftw_ctx* c, double* dev_logical, double* host, bool h2d, long long r0 = -1,
            long long r1 = -1, cudaStream_t st = nullptr) {
    if (!st) st = c->stream;
    const long long gnx = c->g.nx, gny = c->g.ny, nz = c->nz;
    Box o = owned_box(c);
    if (r0 >= 0) {
        o.j0 = std::max(o.j0, r0);
        o.j1 = std::min(o.j1, r1);
        if (o.j1 < o.j0) return HFTW_OK;
    }
    const long long ni = o.i1 - o.i0 + 1, nj = o.j1 - o.j0 + 1;
    const long long gi = c->plan.gi0 + o.i0, gj = c->plan.gj0 + o.j0; // global start
    cudaPitchedPtr hp = make_cudaPitchedPtr(host, (size_t)(gnx + 2) * 8, (size_t)(gnx + 2),
                                            (size_t)(gny + 2));
    cudaPos hpos = make_cudaPos((size_t)gi * 8, (size_t)gj, 0);
    if (c->layout == HFTW_IJK) {
        cudaMemcpy3DParms p{};
        cudaPitchedPtr dp = make_cudaPitchedPtr(dev_logical - c->off3, (size_t)c->Pi * 8,
                                                (size_t)c->Pi, (size_t)c->Rows);
        cudaPos dpos = make_cudaPos((size_t)(kFrontPad + o.i0) * 8, (size_t)(1 + o.j0), 0);
        p.extent = make_cudaExtent((size_t)ni * 8, (size_t)nj, (size_t)nz);
        if (h2d) {
            p.srcPtr = hp;
            p.srcPos = hpos;
            p.dstPtr = dp;
            p.dstPos = dpos;
            p.kind = cudaMemcpyHostToDevice;
        } else {
            p.srcPtr = dp;
            p.srcPos = dpos;
            p.dstPtr = hp;
            p.dstPos = hpos;
            p.kind = cudaMemcpyDeviceToHost;
        }
        CUDA_TRY(c, cudaMemcpy3DAsync(&p, st));
        return HFTW_OK;
    }
    if (st != c->stream) return fail(c, HFTW_EUNSUP, "KIJ copies run on the context stream");
    // KIJ: the owned box goes through a dense device staging box
    const long long n = ni * nj * nz;
    if (c->staging_n < (size_t)n) {
        if (c->staging) cudaFree(c->staging);
        c->staging = nullptr;
        CUDA_TRY(c, cudaMalloc(&c->staging, (size_t)n * sizeof(double)));
        c->staging_n = (size_t)n;
    }
    cudaMemcpy3DParms p{};
    cudaPitchedPtr sp = make_cudaPitchedPtr(c->staging, (size_t)ni * 8, (size_t)ni, (size_t)nj);
    p.extent = make_cudaExtent((size_t)ni * 8, (size_t)nj, (size_t)nz);
    double* box = dev_logical + o.i0 * c->si + o.j0 * c->sj;
    if (h2d) {
        p.srcPtr = hp;
        p.srcPos = hpos;
        p.dstPtr = sp;
        p.kind = cudaMemcpyHostToDevice;
        CUDA_TRY(c, cudaMemcpy3DAsync(&p, c->stream));
        hftw::relayout_kernel<true><<<grid_for(c, n), 256, 0, c->stream>>>(
            c->staging, box, ni, nj, nz, c->si, c->sj, c->sk);
        CUDA_TRY(c, cudaGetLastError());
    } else {
        hftw::relayout_kernel<false><<<grid_for(c, n), 256, 0, c->stream>>>(
            box, c->staging, ni, nj, nz, c->si, c->sj, c->sk);
        CUDA_TRY(c, cudaGetLastError());
        p.srcPtr = sp;
        p.dstPtr = hp;
        p.dstPos = hpos;
        p.kind = cudaMemcpyDeviceToHost;
        CUDA_TRY(c, cudaMemcpy3DAsync(&p, c->stream));
    }
    return HFTW_OK;
}

int copy_2d(hftw_ctx* c, double* dev_logical, double* host, bool h2d, cudaStream_t st = nullptr) {
    if (!st) st = c->stream;
    const long long gnx = c->g.nx;
    const Box o = owned_box(c);
    const long long ni = o.i1 - o.i0 + 1, nj = o.j1 - o.j0 + 1;
    const long long gi = c->plan.gi0 + o.i0, gj = c->plan.gj0 + o.j0;
    double* h = host + gi + gj * (gnx + 2);
    double* d = dev_logical + o.i0 + o.j0 * c->s2j;
    const size_t hp = (size_t)(gnx + 2) * 8, dp = (size_t)c->s2j * 8, w = (size_t)ni * 8;
    if (h2d)
        CUDA_TRY(c, cudaMemcpy2DAsync(d, dp, h, hp, w, (size_t)nj, cudaMemcpyHostToDevice, st));
    else
        CUDA_TRY(c, cudaMemcpy2DAsync(h, hp, d, dp, w, (size_t)nj, cudaMemcpyDeviceToHost, st));
    return HFTW_OK;
}

} // namespace

extern "C" {

int hftw_abi_version(void) { return HFTW_ABI_VERSION; }

int hftw_validate(const hftw_grid* g, char* msg, size_t cap) {
    // hft::validate, weather.cpp:24-41 (messages verbatim, one per line)
    if (msg && cap) msg[0] = 0;
    if (!g) return fail(nullptr, HFTW_EINVAL, "null grid");
    std::string out;
    bool ok = true;
    if (g->nx < 2 || g->ny < 2 || g->nz < 2) {
        out += "<config>: error: grid extents must be at least 2 in every dimension\n";
        ok = false;
    }
    if (!(g->diffusion_velocity <= 1.0 / 6.0) || g->diffusion_velocity < 0.0) {
        out += "<config>: error: diffusion velocity must lie in [0, 1/6] so the center "
               "coefficient stays nonnegative\n";
        ok = false;
    }
    if (g->timestep <= 0.0 || g->output_timestep <= 0.0) {
        out += "<config>: error: timestep and output timestep must be positive\n";
        ok = false;
    }
    if (ok && (g->nx > (1LL << 30) || g->ny > (1LL << 30) || g->nz > (1LL << 30))) {
        out += "<config>: error: extents beyond 2^30 are not supported by the device store\n";
        ok = false;
    }
    if (msg && cap) std::snprintf(msg, cap, "%s", out.c_str());
    if (!ok) {
        g_err = out;
        return HFTW_EINVAL;
    }
    return HFTW_OK;
}

int hftw_plan_rank(const hftw_grid* g, int px, int py, int rank, hftw_plan* out) {
    if (!g || !out) return fail(nullptr, HFTW_EINVAL, "null argument");
    char msg[512];
    if (hftw_validate(g, msg, sizeof msg) != HFTW_OK) return fail(nullptr, HFTW_EINVAL, "%s", msg);
    return make_plan(g, px, py, rank, out);
}

int hftw_create(const hftw_grid* g, int layout, int device, hftw_ctx** out) {
    if (!g) return fail(nullptr, HFTW_EINVAL, "null grid");
    hftw_plan p{};
    char msg[512];
    if (hftw_validate(g, msg, sizeof msg) != HFTW_OK) return fail(nullptr, HFTW_EINVAL, "%s", msg);
    int rc = make_plan(g, 1, 1, 0, &p);
    if (rc) return rc;
    return create_common(g, layout, device, p, false, out);
}

int hftw_create_multi(const hftw_grid* g, int layout, int px, int py, const int* devices,
                      hftw_ctx** out) {
    if (!g) return fail(nullptr, HFTW_EINVAL, "null grid");
    char msg[512];
    if (hftw_validate(g, msg, sizeof msg) != HFTW_OK) return fail(nullptr, HFTW_EINVAL, "%s", msg);
    if (layout != HFTW_IJK && layout != HFTW_KIJ)
        return fail(nullptr, HFTW_EINVAL, "unknown layout %d", layout);
    return create_group(g, layout, px, py, devices, out);
}

int hftw_group_size(const hftw_ctx* c) {
    if (!c) return 0;
    return is_group(c) ? (int)c->ranks.size() : 1;
}

int hftw_group_rank(hftw_ctx* c, int r, hftw_ctx** out) {
    if (!c || !out) return fail(nullptr, HFTW_EINVAL, "null argument");
    const int n = hftw_group_size(c);
    if (r < 0 || r >= n) return fail(c, HFTW_EINVAL, "rank %d of %d", r, n);
    *out = is_group(c) ? c->ranks[(size_t)r] : c;
    return HFTW_OK;
}

int hftw_create_dist(const hftw_grid* g, int layout, int device, int px, int py, int rank,
                     hftw_ctx** out) {
    if (!g) return fail(nullptr, HFTW_EINVAL, "null grid");
    hftw_plan p{};
    int rc = hftw_plan_rank(g, px, py, rank, &p);
    if (rc) return rc;
    rc = create_common(g, layout, device, p, px * py > 1, out);
    if (rc == HFTW_OK && (*out)->dist) (*out)->halo_dirty = true;
    return rc;
}

void hftw_destroy(hftw_ctx* c) {
    if (!c) return;
    if (is_group(c)) {
        // reverse order: a stream shared by ranks of one device belongs to the
        // lowest of them
        for (size_t r = c->ranks.size(); r-- > 0;) hftw_destroy(c->ranks[r]);
        delete c;
        return;
    }
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
    for (int b = 0; b < 2; ++b)
        if (c->buf[b]) cudaFree(c->buf[b]);
    if (c->sf) cudaFree(c->sf); // also holds pb
    if (c->staging) cudaFree(c->staging);
    if (c->d_sched) cudaFree(c->d_sched);
    if (c->d_pair) cudaFree(c->d_pair);
    if (c->d_wave) cudaFree(c->d_wave);
    if (c->gpub) cudaFree(c->gpub);
    if (c->eu_buf) cudaFree(c->eu_buf);
    for (auto& t : c->tev) {
        cudaEventDestroy(t.a);
        cudaEventDestroy(t.b);
    }
    if (c->flags) cudaFree(c->flags);
    if (c->done) cudaFree(c->done);
    for (auto& o : c->out) {
        if (o.done) cudaEventDestroy(o.done);
        if (o.dev) cudaFree(o.dev);
        if (o.host) cudaFreeHost(o.host);
    }
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->xev) cudaEventDestroy(c->xev);
    if (c->h2d_stream) cudaStreamDestroy(c->h2d_stream);
    if (c->d2h_stream) cudaStreamDestroy(c->d2h_stream);
    for (cudaEvent_t e : c->pipe_ev) cudaEventDestroy(e);
    for (double* p : c->host_stage)
        if (p) cudaFree(p);
    if (c->flush_buf) cudaFree(c->flush_buf);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

int hftw_init(hftw_ctx* c) {
    NvtxRange nvtx_("hftw_init");
    int rc = check_ctx(c);
    if (rc) return rc;
    if (is_group(c)) {
        for (hftw_ctx* r : c->ranks) RANK_TRY(c, r, hftw_init(r));
        return HFTW_OK;
    }
    for (int b = 0; b < 2; ++b)
        CUDA_TRY(c, cudaMemsetAsync(c->buf[b], 0, c->n3 * sizeof(double), c->stream));
    Dom d = make_dom(c);
    const long long n = (c->lnx + 2) * (c->lny + 2) * c->nz;
    const int gnx = (int)c->g.nx, gny = (int)c->g.ny, gnz = (int)c->g.nz;
    const int gi0 = (int)c->plan.gi0, gj0 = (int)c->plan.gj0;
    if (c->layout == HFTW_KIJ)
        hftw::init_kernel<true><<<grid_for(c, n), 256, 0, c->stream>>>(
            e3(c, c->cur), sf2(c), pb2(c), d, gnx, gny, gnz, gi0, gj0, c->g.surf_energy,
            c->g.pbl_energy);
    else
        hftw::init_kernel<false><<<grid_for(c, n), 256, 0, c->stream>>>(
            e3(c, c->cur), sf2(c), pb2(c), d, gnx, gny, gnz, gi0, gj0, c->g.surf_energy,
            c->g.pbl_energy);
    CUDA_TRY(c, cudaGetLastError());
    if (c->d_sched) CUDA_TRY(c, cudaMemsetAsync(c->d_sched, 0, 2 * sizeof(int), c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    c->eu_derived = false; // energy_u is all zeros (weather.cpp:82)
    c->eu_stored = false;
    c->eu_pending = false;
    c->poisoned = 0;
    if (c->dist) c->halo_dirty = true;
    return HFTW_OK;
}

int hftw_upload(hftw_ctx* c, int field, const double* host) {
    NvtxRange nvtx_("hftw_upload");
    int rc = check_ctx(c);
    if (rc) return rc;
    if (!valid_field(field) || !host)
        return fail(c, HFTW_EINVAL, "bad field %d or null buffer", field);
    if (is_group(c)) {
        for (hftw_ctx* r : c->ranks) RANK_TRY(c, r, hftw_upload(r, field, host));
        return HFTW_OK;
    }
    double* h = const_cast<double*>(host);
    switch (field) {
    case HFTW_ENERGY:
        rc = copy_3d(c, e3(c, c->cur), h, true);
        break;
    case HFTW_ENERGY_U:
        rc = copy_3d(c, e3(c, c->cur ^ 1), h, true);
        c->eu_derived = false;
        c->eu_stored = false;
        c->eu_pending = false;
        break;
    case HFTW_ENERGY_SURF:
    case HFTW_ENERGY_PBL:
        // a derived energy_u depends on the boundary fields of its step
        if (!c->poisoned && (rc = materialize_eu(c))) return rc;
        rc = copy_2d(c, field == HFTW_ENERGY_SURF ? sf2(c) : pb2(c), h, true);
        break;
    }
    if (rc) return rc;
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    c->poisoned &= ~(1u << field);
    if (c->dist && field != HFTW_ENERGY_U) c->halo_dirty = true;
    return HFTW_OK;
}

int hftw_download(hftw_ctx* c, int field, double* host) {
    NvtxRange nvtx_("hftw_download");
    int rc = check_ctx(c);
    if (rc) return rc;
    if (!valid_field(field) || !host)
        return fail(c, HFTW_EINVAL, "bad field %d or null buffer", field);
    if (is_group(c)) {
        for (hftw_ctx* r : c->ranks) RANK_TRY(c, r, hftw_download(r, field, host));
        return HFTW_OK;
    }
    if ((rc = check_state(c))) return rc;
    switch (field) {
    case HFTW_ENERGY:
        rc = copy_3d(c, e3(c, c->cur), host, false);
        break;
    case HFTW_ENERGY_U:
        if ((rc = materialize_eu(c))) return rc;
        rc = copy_3d(c, eu_field(c), host, false);
        break;
    case HFTW_ENERGY_SURF:
        rc = copy_2d(c, sf2(c), host, false);
        break;
    case HFTW_ENERGY_PBL:
        rc = copy_2d(c, pb2(c), host, false);
        break;
    }
    if (rc) return rc;
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return HFTW_OK;
}

int hftw_step(hftw_ctx* c, int64_t nsteps) {
    NvtxRange nvtx_("hftw_step");
    int rc = check_ctx(c);
    if (rc) return rc;
    if (is_group(c)) return group_step(c, nsteps);
    if ((rc = check_state(c))) return rc;
    if (nsteps < 0) return fail(c, HFTW_EINVAL, "steps must be nonnegative");
    if (nsteps == 0) return HFTW_OK;
    const int k = resolved_kernel(c);
    if (c->dist) {
        if (!c->connected) return fail(c, HFTW_ESTATE, "peers not connected (hftw_peer_connect)");
        if (c->halo_dirty)
            return fail(c, HFTW_ESTATE, "fields changed since the last hftw_exchange");
        if (k == HFTW_KERNEL_SPLIT)
            return fail(c, HFTW_EUNSUP, "the split (physics, then diffusion) kernel needs "
                                        "post-physics halos; use a fused kernel when decomposed");
    }
    if (k == HFTW_KERNEL_FUSED_PAIR) {
        if (!c->pair_ok) return fail(c, HFTW_EUNSUP, "pair kernel unavailable for this grid/layout");
        // pairs, then one or two single steps: the last step is a single-step
        // launch so that energy_u (physics of the field before it) stays
        // derivable from the ping-pong partner
        // between the passes of this call the field is stored post-physics (the
        // first pass reads, the last one writes, plain e)
        const int64_t pairs = pair_passes(nsteps);
        for (int64_t p = 0; p < pairs; ++p)
            if ((rc = pair_pass(c, 3, pair_form(p, pairs)))) {
                // a pass failed after earlier passes left the field post-physics: the
                // state is not the reference's any more
                if (p > 0) c->poisoned = 0xF;
                return rc;
            }
        nsteps -= 2 * pairs;
    }
    const bool multistep = c->opt_multistep > 0 || (c->opt_multistep == 0 && c->wave_pref);
    if ((k == HFTW_KERNEL_FUSED_TMA || k == HFTW_KERNEL_FUSED_PAIR) && c->wave_ok && multistep &&
        nsteps >= 2 && c->tma_ok) {
        // all steps in one persistent launch (weather_wave.cuh); chunks of
        // at most 2^20 steps keep the work-list index in an int (decomposed:
        // kMaxWaveStepsDist, the per-step completion counters)
        while (nsteps > 0) {
            const int64_t n = std::min<int64_t>(
                nsteps, c->dist ? (int64_t)kMaxWaveStepsDist : (int64_t)1 << 20);
            if (n < 2) break;
            if ((rc = launch_wave(c, c->cur, n))) return rc;
            if (n & 1) c->cur ^= 1;
            c->step_count += n;
            c->eu_derived = true;
            c->eu_stored = false;
            c->eu_pending = false;
            nsteps -= n;
        }
    }
    const int k1 = k == HFTW_KERNEL_FUSED_PAIR ? HFTW_KERNEL_FUSED_TMA : k;
    for (int64_t s = 0; s < nsteps; ++s) {
        if (k == HFTW_KERNEL_SPLIT || k == HFTW_KERNEL_FUSED_CELL) {
            if ((rc = timing_mark(c, 0, true))) return rc;
        }
        if (k == HFTW_KERNEL_SPLIT) {
            // the reference's structure: physics in place, then diffusion
            if ((rc = launch_physics(c, e3(c, c->cur), best_physics_mode(c)))) return rc;
            if ((rc = launch_fused<false>(c, c->cur, c->tma_ok ? HFTW_KERNEL_FUSED_TMA
                                                               : HFTW_KERNEL_FUSED_CELL)))
                return rc;
            c->eu_derived = false;
            c->eu_stored = false;
            c->eu_pending = false;
        } else {
            if (k1 != HFTW_KERNEL_FUSED_CELL && (rc = timing_mark(c, 0, true))) return rc;
            if ((rc = launch_fused<true>(c, c->cur, k1))) return rc;
            c->eu_derived = true;
            c->eu_stored = false;
            c->eu_pending = false;
        }
        if ((rc = timing_mark(c, 0, false))) return rc;
        c->cur ^= 1;
        ++c->step_count;
    }
    return HFTW_OK;
}

int hftw_set_timing(hftw_ctx* c, int on) {
    int rc = check_ctx(c);
    if (rc) return rc;
    if (is_group(c)) {
        for (hftw_ctx* r : c->ranks) RANK_TRY(c, r, hftw_set_timing(r, on));
        return HFTW_OK;
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    for (auto& t : c->tev) {
        cudaEventDestroy(t.a);
        cudaEventDestroy(t.b);
    }
    c->tev.clear();
    c->timing = on != 0;
    return HFTW_OK;
}

int hftw_get_timing(hftw_ctx* c, int kind, double* ms, int64_t* launches, int64_t* steps) {
    int rc = check_ctx(c);
    if (rc) return rc;
    if (!ms || !launches) return fail(c, HFTW_EINVAL, "null output");
    if (is_group(c)) {
        // launches and steps of rank 0; the device time of the slowest rank
        double worst = 0.0;
        for (size_t r = c->ranks.size(); r-- > 0;) {
            RANK_TRY(c, c->ranks[r], hftw_get_timing(c->ranks[r], kind, ms, launches, steps));
            worst = std::max(worst, *ms);
        }
        *ms = worst;
        return HFTW_OK;
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    double tot = 0.0;
    int64_t n = 0, st = 0;
    for (auto& t : c->tev) {
        if (t.kind != kind) continue;
        float x = 0.f;
        CUDA_TRY(c, cudaEventElapsedTime(&x, t.a, t.b));
        tot += x;
        ++n;
        st += t.steps;
    }
    *ms = tot;
    *launches = n;
    if (steps) *steps = st;
    return HFTW_OK;
}

int hftw_sync(hftw_ctx* c) {
    int rc = check_ctx(c);
    if (rc) return rc;
    if (is_group(c)) {
        for (hftw_ctx* r : c->ranks) RANK_TRY(c, r, hftw_sync(r));
        return HFTW_OK;
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return HFTW_OK;
}

const char* hftw_last_error(const hftw_ctx* c) { return c ? c->err.c_str() : g_err.c_str(); }

int hftw_run_reference(const hftw_grid* g, int64_t steps, int device, double* e, double* eu,
                       double* sf, double* pb) {
    hftw_ctx* c = nullptr;
    int rc = hftw_create(g, HFTW_IJK, device, &c);
    if (rc) return rc;
    auto done = [&](int r) {
        if (r) g_err = c->err;
        hftw_destroy(c);
        return r;
    };
    if ((rc = hftw_init(c))) return done(rc);
    if ((rc = hftw_step(c, steps))) return done(rc);
    if (e && (rc = hftw_download(c, HFTW_ENERGY, e))) return done(rc);
    if (eu && (rc = hftw_download(c, HFTW_ENERGY_U, eu))) return done(rc);
    if (sf && (rc = hftw_download(c, HFTW_ENERGY_SURF, sf))) return done(rc);
    if (pb && (rc = hftw_download(c, HFTW_ENERGY_PBL, pb))) return done(rc);
    return done(HFTW_OK);
}

int hftw_set_stream(hftw_ctx* c, void* s) {
    int rc = check_ctx(c);
    if (rc) return rc;
    if (is_group(c)) return fail(c, HFTW_EUNSUP, "a group context keeps one stream per device");
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (c->own_stream) cudaStreamDestroy(c->stream);
    if (s) {
        c->stream = static_cast<cudaStream_t>(s);
        c->own_stream = false;
    } else {
        CUDA_TRY(c, cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    return HFTW_OK;
}

void* hftw_stream(hftw_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

int hftw_set_kernel(hftw_ctx* c, int k) {
    if (!c) return fail(nullptr, HFTW_EINVAL, "null context");
    if (is_group(c)) {
        for (hftw_ctx* r : c->ranks) RANK_TRY(c, r, hftw_set_kernel(r, k));
        return HFTW_OK;
    }
    if (k < HFTW_KERNEL_AUTO || k > HFTW_KERNEL_FUSED_PAIR)
        return fail(c, HFTW_EINVAL, "bad kernel %d", k);
    if (k == HFTW_KERNEL_FUSED_PAIR && !c->pair_ok)
        return fail(c, HFTW_EUNSUP, "pair kernel unavailable: needs the IJK layout, one domain, "
                                    "nz <= 64 and the TMA kernel");
    if (k == HFTW_KERNEL_FUSED_TMA && !c->tma_ok)
        return fail(c, HFTW_EUNSUP, "TMA kernel unavailable: the slab ring for this nz does not fit shared memory");
    c->kernel_req = k;
    return HFTW_OK;
}

int hftw_get_kernel(const hftw_ctx* c) {
    if (is_group(c)) return hftw_get_kernel(c->ranks[0]);
    return c ? resolved_kernel(c) : -1;
}

int hftw_set_option(hftw_ctx* c, int opt, int64_t v) {
    if (!c) return fail(nullptr, HFTW_EINVAL, "null context");
    if (is_group(c)) {
        for (hftw_ctx* r : c->ranks) RANK_TRY(c, r, hftw_set_option(r, opt, v));
        return HFTW_OK;
    }
    switch (opt) {
    case HFTW_OPT_MULTISTEP:
        if (v < -1 || v > 1) return fail(c, HFTW_EINVAL, "HFTW_OPT_MULTISTEP takes -1, 0 or 1");
        c->opt_multistep = (int)v;
        return HFTW_OK;
    case HFTW_OPT_PAIR:
        if (v != 0 && v != 1) return fail(c, HFTW_EINVAL, "HFTW_OPT_PAIR takes 0 or 1");
        c->pair_auto = v != 0;
        return HFTW_OK;
    case HFTW_OPT_EXCHANGE:
        if (v != 0 && v != 1) return fail(c, HFTW_EINVAL, "HFTW_OPT_EXCHANGE takes 0 or 1");
        c->opt_exchange = (int)v;
        return HFTW_OK;
    case HFTW_OPT_REVERSE:
        if (v != 0 && v != 1) return fail(c, HFTW_EINVAL, "HFTW_OPT_REVERSE takes 0 or 1");
        c->opt_reverse = (int)v;
        return HFTW_OK;
    }
    return fail(c, HFTW_EINVAL, "unknown option %d", opt);
}

int hftw_physics(hftw_ctx* c, int mode) {
    NvtxRange nvtx_("hftw_physics");
    int rc = check_ctx(c);
    if (rc) return rc;
    if (mode != 0 && mode != 1) return fail(c, HFTW_EINVAL, "bad physics mode %d", mode);
    if (is_group(c)) {
        for (hftw_ctx* r : c->ranks) RANK_TRY(c, r, hftw_physics(r, mode));
        return HFTW_OK;
    }
    if ((rc = check_state(c))) return rc;
    if ((rc = materialize_eu(c))) return rc;
    if ((rc = launch_physics(c, e3(c, c->cur), mode))) return rc;
    if (c->dist) c->halo_dirty = true;
    return HFTW_OK;
}

int hftw_diffuse(hftw_ctx* c) {
    NvtxRange nvtx_("hftw_diffuse");
    int rc = check_ctx(c);
    if (rc) return rc;
    if (c->dist || is_group(c))
        return fail(c, HFTW_EUNSUP, "diffusion-only sweeps are single-domain");
    if ((rc = check_state(c))) return rc;
    if ((rc = launch_fused<false>(c, c->cur,
                                  c->tma_ok ? HFTW_KERNEL_FUSED_TMA : HFTW_KERNEL_FUSED_CELL)))
        return rc;
    c->eu_derived = false; // energy_u = the diffused input (swap semantics)
    c->eu_stored = false;
    c->eu_pending = false;
    c->cur ^= 1;
    return HFTW_OK;
}

int hftw_diffuse_steps(hftw_ctx* c, int64_t n) {
    NvtxRange nvtx_("hftw_diffuse_steps");
    int rc = check_ctx(c);
    if (rc) return rc;
    if (c->dist || is_group(c))
        return fail(c, HFTW_EUNSUP, "diffusion-only sweeps are single-domain");
    if ((rc = check_state(c))) return rc;
    if (n < 0) return fail(c, HFTW_EINVAL, "sweeps must be nonnegative");
    if (n == 0) return HFTW_OK;
    if (n == 1 || !c->wave_ok) {
        for (int64_t s = 0; s < n; ++s)
            if ((rc = hftw_diffuse(c))) return rc;
        return HFTW_OK;
    }
    // all sweeps in persistent launches of the multi-step schedule (the field
    // of sweep s+1 is read as soon as the rows it needs from sweep s are done)
    for (int64_t left = n; left > 0;) {
        const int64_t m = std::min<int64_t>(left, (int64_t)1 << 20);
        if (m == 1) {
            if ((rc = hftw_diffuse(c))) return rc;
            break;
        }
        if ((rc = launch_wave(c, c->cur, m, false))) return rc;
        if (m & 1) c->cur ^= 1;
        left -= m;
    }
    c->eu_derived = false; // energy_u = the last sweep's input (swap semantics)
    c->eu_stored = false;
    c->eu_pending = false;
    return HFTW_OK;
}

double hftw_algorithmic_bytes(const hftw_ctx* c, int what) {
    if (!c) return 0.0;
    if (is_group(c)) {
        double t = 0.0;
        for (const hftw_ctx* r : c->ranks) t += hftw_algorithmic_bytes(r, what);
        return t;
    }
    // this context's stored cells (its subdomain's owned cells when decomposed)
    const Box o = owned_box(c);
    const double cols = (double)(o.i1 - o.i0 + 1) * (double)(o.j1 - o.j0 + 1);
    const double cells = cols * (double)c->nz;
    switch (what) {
    case 0: return 16.0 * cells + 16.0 * cols; // read e, write u, read sf + pb
    case 1: return 16.0 * cells + 16.0 * cols; // physics: e read + write, sf + pb
    case 2: return 16.0 * cells;               // diffusion: read e, write u
    }
    return 0.0;
}

int hftw_launches_per_step(const hftw_ctx* c) {
    if (!c) return 0;
    if (is_group(c)) return hftw_launches_per_step(c->ranks[0]) * (int)c->ranks.size();
    return resolved_kernel(c) == HFTW_KERNEL_SPLIT ? 2 : 1;
}

int hftw_field_view(hftw_ctx* c, int field, void** dptr, int64_t strides[3]) {
    int rc = check_ctx(c);
    if (rc) return rc;
    if (!valid_field(field) || !dptr || !strides) return fail(c, HFTW_EINVAL, "bad arguments");
    if (is_group(c))
        return fail(c, HFTW_EUNSUP, "a group has one view per rank (hftw_group_rank)");
    if ((rc = check_state(c))) return rc;
    // the view is writable: energy_u must not depend on sf/pb any more, and a
    // decomposed rank's halos must be refilled before the next step
    if ((rc = materialize_eu(c))) return rc;
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (c->dist) c->halo_dirty = true;
    switch (field) {
    case HFTW_ENERGY: *dptr = e3(c, c->cur); break;
    case HFTW_ENERGY_U: *dptr = eu_field(c); break;
    case HFTW_ENERGY_SURF: *dptr = sf2(c); break;
    case HFTW_ENERGY_PBL: *dptr = pb2(c); break;
    }
    const bool f3 = field == HFTW_ENERGY || field == HFTW_ENERGY_U;
    strides[0] = f3 ? c->si : 1;
    strides[1] = f3 ? c->sj : c->s2j;
    strides[2] = f3 ? c->sk : 0;
    return HFTW_OK;
}

int hftw_flush_l2(hftw_ctx* c, size_t bytes) {
    int rc = check_ctx(c);
    if (rc) return rc;
    if (is_group(c)) return rank_fail(c, c->ranks[0], hftw_flush_l2(c->ranks[0], bytes));
    bytes = (bytes + 31) / 32 * 32;
    if (c->flush_bytes < bytes) {
        if (c->flush_buf) cudaFree(c->flush_buf);
        c->flush_buf = nullptr;
        CUDA_TRY(c, cudaMalloc(&c->flush_buf, bytes));
        c->flush_bytes = bytes;
    }
    raise_smem_attr((const void*)hftw::flush_kernel, 200 * 1024);
    const size_t dyn = c->tma_ok ? std::min<size_t>(c->smem, 200 * 1024) : 0;
    hftw::flush_kernel<<<c->num_sms, 512, dyn, c->stream>>>(
        static_cast<double4*>(c->flush_buf), (long long)(bytes / 32), 1.0);
    CUDA_TRY(c, cudaGetLastError());
    return HFTW_OK;
}

size_t hftw_peer_desc_size(void) { return sizeof(PeerDesc); }

int hftw_peer_export(hftw_ctx* c, void* out) {
    int rc = check_ctx(c);
    if (rc) return rc;
    if (is_group(c)) return fail(c, HFTW_EUNSUP, "a group connects its ranks itself");
    if (!out) return fail(c, HFTW_EINVAL, "null descriptor buffer");
    PeerDesc pd{};
    for (int b = 0; b < 2; ++b) CUDA_TRY(c, cudaIpcGetMemHandle(&pd.buf[b], c->buf[b]));
    CUDA_TRY(c, cudaIpcGetMemHandle(&pd.sf, c->sf));
    pd.n2 = (long long)c->n2;
    CUDA_TRY(c, cudaIpcGetMemHandle(&pd.flags, c->flags));
    pd.has_gpub = c->gpub ? 1 : 0;
    pd.gpub_n = (long long)c->gpub_n;
    pd.gcol_n = 4 * (c->lny + 2) * c->nz;
    if (c->gpub) CUDA_TRY(c, cudaIpcGetMemHandle(&pd.gpub, c->gpub));
    pd.off3 = c->off3;
    pd.off2 = c->off2;
    pd.si = c->si;
    pd.sj = c->sj;
    pd.sk = c->sk;
    pd.s2j = c->s2j;
    pd.plan = c->plan;
    pd.magic = kPeerMagic;
    std::memcpy(out, &pd, sizeof pd);
    return HFTW_OK;
}

int hftw_peer_connect(hftw_ctx* c, const void* all, int world) {
    int rc = check_ctx(c);
    if (rc) return rc;
    if (is_group(c)) return fail(c, HFTW_EUNSUP, "a group connects its ranks itself");
    if (!all || world != c->plan.px * c->plan.py)
        return fail(c, HFTW_EINVAL, "need %d descriptors, got %d", c->plan.px * c->plan.py, world);
    const PeerDesc* pds = static_cast<const PeerDesc*>(all);
    std::map<int, PeerMap> opened; // a rank can be the neighbour in several directions
    for (int d = 0; d < hftw::kNbrs; ++d) {
        const int r = nbr_rank(c->plan, d);
        if (r < 0) {
            c->peer[d] = PeerMap{};
            continue;
        }
        const PeerDesc& pd = pds[r];
        if (pd.magic != kPeerMagic || pd.plan.rank != r)
            return fail(c, HFTW_EINVAL, "descriptor %d is not rank %d's", r, r);
        auto it = opened.find(r);
        if (it == opened.end()) {
            PeerMap m;
            m.rank = r;
            void* p = nullptr;
            for (int b = 0; b < 2; ++b) {
                CUDA_TRY(c, cudaIpcOpenMemHandle(&p, pd.buf[b], cudaIpcMemLazyEnablePeerAccess));
                c->ipc_opened.push_back(p);
                m.buf[b] = static_cast<double*>(p) + pd.off3;
            }
            CUDA_TRY(c, cudaIpcOpenMemHandle(&p, pd.sf, cudaIpcMemLazyEnablePeerAccess));
            c->ipc_opened.push_back(p);
            m.sf = static_cast<double*>(p) + pd.off2;
            m.pb = static_cast<double*>(p) + pd.n2 + pd.off2;
            CUDA_TRY(c, cudaIpcOpenMemHandle(&p, pd.flags, cudaIpcMemLazyEnablePeerAccess));
            c->ipc_opened.push_back(p);
            m.flags = static_cast<unsigned long long*>(p);
            if (pd.has_gpub) {
                CUDA_TRY(c, cudaIpcOpenMemHandle(&p, pd.gpub, cudaIpcMemLazyEnablePeerAccess));
                c->ipc_opened.push_back(p);
                m.gpub = static_cast<double*>(p);
                m.gpub_n = pd.gpub_n;
                m.gcol_n = pd.gcol_n;
            }
            m.si = pd.si;
            m.sj = pd.sj;
            m.sk = pd.sk;
            m.s2j = pd.s2j;
            it = opened.emplace(r, m).first;
        }
        c->peer[d] = it->second;
    }
    c->connected = true;
    return HFTW_OK;
}

int hftw_exchange(hftw_ctx* c) {
    NvtxRange nvtx_("hftw_exchange");
    int rc = check_ctx(c);
    if (rc) return rc;
    if (is_group(c)) return group_exchange(c);
    if ((rc = check_state(c))) return rc;
    if (!c->dist) {
        c->halo_dirty = false;
        return HFTW_OK;
    }
    if (!c->connected) return fail(c, HFTW_ESTATE, "peers not connected (hftw_peer_connect)");
    Dom d = make_dom(c);
    Halo h = make_halo(c, c->cur); // faces of the CURRENT field into the neighbours' current buffer
    hftw::Halo2D h2{};
    for (int q = 0; q < hftw::kNbrs; ++q)
        if (c->peer[q].rank >= 0) {
            h2.sf[q] = c->peer[q].sf;
            h2.pb[q] = c->peer[q].pb;
            h2.s2j[q] = c->peer[q].s2j;
        }
    const Box o = owned_box(c);
    const long long n = (o.i1 - o.i0 + 1) * (o.j1 - o.j0 + 1) * c->nz;
    hftw::exchange_kernel<<<grid_for(c, n), 256, 0, c->stream>>>(e3(c, c->cur), sf2(c), pb2(c), d,
                                                                  h, h2);
    CUDA_TRY(c, cudaGetLastError());
    // a fresh epoch: step flags restart from zero on every rank
    CUDA_TRY(c, cudaMemsetAsync(c->flags, 0, hftw::kFlags * sizeof(unsigned long long), c->stream));
    CUDA_TRY(c, cudaMemsetAsync(c->done, 0, sizeof(int), c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    c->step_count = 0;
    c->pass_count = 0;
    c->halo_dirty = false;
    return HFTW_OK;
}

// modulo_real of the reference interpreter (interpreter.cpp:109)
static double modulo_real(double a, double p) {
    volatile double q = std::floor(a / p);
    volatile double m = q * p;
    return a - m;
}

} // extern "C"

namespace {
// hftw_simulate on a group context: the same time loop, each output gathered
// from the ranks synchronously into one pinned logical buffer.
int group_simulate(hftw_ctx* c, double start_time, double end_time, double timestep,
                   double output_timestep, hftw_write_fn write, void* user, int64_t* steps_done,
                   int64_t* writes_done) {
    const size_t n = (size_t)((c->g.nx + 2) * (c->g.ny + 2) * c->g.nz);
    double* host = nullptr;
    if (write) CUDA_TRY(c, cudaMallocHost(&host, n * sizeof(double)));
    auto due = [&](double t) {
        volatile double pr = t + 0.001;
        return write && modulo_real(pr, output_timestep) < 0.01;
    };
    int rc = HFTW_OK;
    int64_t steps = 0, writes = 0;
    double time = start_time;
    for (;;) {
        if (due(time)) {
            if ((rc = hftw_download(c, HFTW_ENERGY, host))) break;
            write(user, "energy", time, host);
            ++writes;
        }
        int64_t k = 0;
        double t = time;
        do {
            ++k;
            t = t + timestep;
        } while (!(t > end_time) && !due(t));
        if ((rc = hftw_step(c, k))) break;
        steps += k;
        time = t;
        if (time > end_time) break;
    }
    if (host) cudaFreeHost(host);
    if (rc) return rc;
    if (steps_done) *steps_done = steps;
    if (writes_done) *writes_done = writes;
    return HFTW_OK;
}
} // namespace

extern "C" {

int hftw_simulate(hftw_ctx* c, double start_time, double end_time, double timestep,
                  double output_timestep, hftw_write_fn write, void* user, int64_t* steps_done,
                  int64_t* writes_done) {
    NvtxRange nvtx_("hftw_simulate");
    int rc = check_ctx(c);
    if (rc) return rc;
    if (c->dist) return fail(c, HFTW_EUNSUP, "hftw_simulate runs on single-domain contexts");
    if (!(timestep > 0.0) || !(output_timestep > 0.0))
        return fail(c, HFTW_EINVAL, "timestep and output timestep must be positive");
    if (is_group(c))
        return group_simulate(c, start_time, end_time, timestep, output_timestep, write, user,
                              steps_done, writes_done);
    if ((rc = check_state(c))) return rc;
    const long long nx = c->g.nx, ny = c->g.ny, nz = c->g.nz;
    const size_t n = (size_t)((nx + 2) * (ny + 2) * nz);
    if (write && c->out.empty()) {
        c->out.resize(2);
        CUDA_TRY(c, cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        for (auto& o : c->out) {
            CUDA_TRY(c, cudaMalloc(&o.dev, n * sizeof(double)));
            CUDA_TRY(c, cudaMallocHost(&o.host, n * sizeof(double)));
            CUDA_TRY(c, cudaEventCreateWithFlags(&o.done, cudaEventDisableTiming));
        }
    }
    std::vector<int> fifo; // pending slots in time order
    size_t next = 0;
    int64_t steps = 0, writes = 0;
    auto deliver = [&](bool block) -> int {
        while (!fifo.empty()) {
            auto& o = c->out[(size_t)fifo.front()];
            if (!block) {
                cudaError_t q = cudaEventQuery(o.done);
                if (q == cudaErrorNotReady) return HFTW_OK;
                if (q != cudaSuccess) return fail(c, HFTW_ECUDA, "output copy failed: %s",
                                                  cudaGetErrorString(q));
            } else {
                CUDA_TRY(c, cudaEventSynchronize(o.done));
            }
            write(user, "energy", o.time, o.host);
            o.pending = false;
            ++writes;
            fifo.erase(fifo.begin());
        }
        return HFTW_OK;
    };
    double time = start_time;
    for (;;) {
        volatile double probe = time + 0.001;
        if (write && modulo_real(probe, output_timestep) < 0.01) {
            auto& o = c->out[next];
            if (o.pending) { // ring full: the oldest output must leave first
                if ((rc = deliver(true))) return rc;
            }
            // device snapshot on the compute stream (the next-but-one step
            // overwrites this buffer), then PCIe on the copy stream
            double* src = e3(c, c->cur);
            if (c->layout == HFTW_IJK) {
                cudaMemcpy3DParms p{};
                p.srcPtr = make_cudaPitchedPtr(src - c->off3, (size_t)c->Pi * 8, (size_t)c->Pi,
                                               (size_t)c->Rows);
                p.srcPos = make_cudaPos((size_t)kFrontPad * 8, 1, 0); // logical (0, 0, 1)
                p.dstPtr = make_cudaPitchedPtr(o.dev, (size_t)(nx + 2) * 8, (size_t)(nx + 2),
                                               (size_t)(ny + 2));
                p.extent = make_cudaExtent((size_t)(nx + 2) * 8, (size_t)(ny + 2), (size_t)nz);
                p.kind = cudaMemcpyDeviceToDevice;
                CUDA_TRY(c, cudaMemcpy3DAsync(&p, c->stream));
            } else {
                hftw::relayout_kernel<false><<<grid_for(c, (long long)n), 256, 0, c->stream>>>(
                    src, o.dev, nx + 2, ny + 2, nz, c->si, c->sj, c->sk);
                CUDA_TRY(c, cudaGetLastError());
            }
            cudaEvent_t snap;
            CUDA_TRY(c, cudaEventCreateWithFlags(&snap, cudaEventDisableTiming));
            CUDA_TRY(c, cudaEventRecord(snap, c->stream));
            CUDA_TRY(c, cudaStreamWaitEvent(c->copy_stream, snap, 0));
            cudaEventDestroy(snap);
            CUDA_TRY(c, cudaMemcpyAsync(o.host, o.dev, n * sizeof(double), cudaMemcpyDeviceToHost,
                                        c->copy_stream));
            CUDA_TRY(c, cudaEventRecord(o.done, c->copy_stream));
            o.pending = true;
            o.time = time;
            fifo.push_back((int)next);
            next = (next + 1) % c->out.size();
        }
        // the steps up to the next output (or the end) go to the device as one
        // batch, so hftw_step can fuse them into two-step passes; the host
        // replays the loop's time arithmetic exactly
        auto due = [&](double t) {
            volatile double pr = t + 0.001;
            return write && modulo_real(pr, output_timestep) < 0.01;
        };
        int64_t n = 0;
        double t = time;
        do {
            ++n;
            t = t + timestep;
        } while (!(t > end_time) && !due(t));
        if ((rc = hftw_step(c, n))) return rc;
        steps += n;
        if (write && (rc = deliver(false))) return rc;
        time = t;
        if (time > end_time) break;
    }
    if (write && (rc = deliver(true))) return rc;
    if (steps_done) *steps_done = steps;
    if (writes_done) *writes_done = writes;
    return HFTW_OK;
}

int hftw_host_register(void* ptr, size_t bytes) {
    if (!ptr || !bytes) return fail(nullptr, HFTW_EINVAL, "null or empty host range");
    const cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterPortable);
    if (e != cudaSuccess)
        return fail(nullptr, HFTW_ECUDA, "cudaHostRegister failed: %s", cudaGetErrorString(e));
    return HFTW_OK;
}

int hftw_host_unregister(void* ptr) {
    if (!ptr) return fail(nullptr, HFTW_EINVAL, "null host pointer");
    const cudaError_t e = cudaHostUnregister(ptr);
    if (e != cudaSuccess)
        return fail(nullptr, HFTW_ECUDA, "cudaHostUnregister failed: %s", cudaGetErrorString(e));
    return HFTW_OK;
}

} // extern "C"

namespace {
int step_host_pipeline(hftw_ctx* c, const double* energy, const double* energy_surf,
                       const double* energy_pbl, double* energy_out, double* energy_u_out);
}

extern "C" {

int hftw_step_host(hftw_ctx* c, const double* energy, const double* energy_surf,
                   const double* energy_pbl, double* energy_out, double* energy_u_out) {
    NvtxRange nvtx_("hftw_step_host");
    int rc = check_ctx(c);
    if (rc) return rc;
    if (!energy || !energy_surf || !energy_pbl || !energy_out || !energy_u_out)
        return fail(c, HFTW_EINVAL, "null host buffer");
    if (c->dist)
        return fail(c, HFTW_EUNSUP, "hftw_step_host runs on single-domain contexts");
    const int rk = resolved_kernel(c);
    if (is_group(c) || !c->tma_ok || c->layout != HFTW_IJK ||
        (rk != HFTW_KERNEL_FUSED_TMA && rk != HFTW_KERNEL_FUSED_PAIR)) {
        // no row-block pipeline for this configuration: the same calls in sequence
        if ((rc = hftw_upload(c, HFTW_ENERGY, energy)) ||
            (rc = hftw_upload(c, HFTW_ENERGY_SURF, energy_surf)) ||
            (rc = hftw_upload(c, HFTW_ENERGY_PBL, energy_pbl)) || (rc = hftw_step(c, 1)) ||
            (rc = hftw_download(c, HFTW_ENERGY, energy_out)) ||
            (rc = hftw_download(c, HFTW_ENERGY_U, energy_u_out)))
            return rc;
        return HFTW_OK;
    }
    rc = step_host_pipeline(c, energy, energy_surf, energy_pbl, energy_out, energy_u_out);
    if (rc) {
        // stop every copy into / out of the caller's buffers before returning;
        // the device state (partly scattered input, new sf/pb) is now undefined
        if (c->h2d_stream) cudaStreamSynchronize(c->h2d_stream);
        if (c->d2h_stream) cudaStreamSynchronize(c->d2h_stream);
        cudaStreamSynchronize(c->stream);
        cudaGetLastError();
        c->eu_derived = false;
        c->eu_stored = false;
        c->eu_pending = false;
        c->poisoned = 0xF;
    }
    return rc;
}

} // extern "C"

namespace {
int step_host_pipeline(hftw_ctx* c, const double* energy, const double* energy_surf,
                       const double* energy_pbl, double* energy_out, double* energy_u_out) {
    int rc = HFTW_OK;
    double* e_in = const_cast<double*>(energy);
    // Row blocks of whole TMA chunks.  Block b: ONE 2D H2D copy of its rows
    // (all k) into a dense staging copy of the host array (h2d stream); on the
    // compute stream, scatter into the padded field and -- once block b+1 has
    // landed (the j+1 neighbours) -- the step's work units and i-ghost columns
    // of block b's rows, energy_u of its rows and a gather of the new rows into
    // dense staging; then ONE 2D D2H copy each of energy and energy_u (d2h
    // stream).  The j-ghost rows need rows 1 and ny, so they run last.  H2D,
    // the kernels and D2H overlap (PCIe is full duplex).  In-place use
    // (energy_out == energy) is safe: a row is read back only after every row
    // has been uploaded up to its j+1 neighbour.
    const int nb = std::max(
        1, std::min(c->nchunks, std::min(kMaxPipeBlocks, env_int("HFTW_PIPE_BLOCKS", 32))));
    if (!c->h2d_stream) {
        CUDA_TRY(c, cudaStreamCreateWithFlags(&c->h2d_stream, cudaStreamNonBlocking));
        CUDA_TRY(c, cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking));
    }
    while ((int)c->pipe_ev.size() < 3 * kMaxPipeBlocks + 2) {
        cudaEvent_t e;
        CUDA_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->pipe_ev.push_back(e);
    }
    const long long nx = c->lnx, ny = c->lny, nz = c->nz;
    const long long hsj = nx + 2, hsk = (nx + 2) * (ny + 2); // host (logical) strides
    for (double*& p : c->host_stage)
        if (!p) CUDA_TRY(c, cudaMalloc(&p, (size_t)(hsk * nz) * sizeof(double)));
    double* const sin = c->host_stage[0];
    double* const sout = c->host_stage[1];
    double* const seu = c->host_stage[2];
    cudaEvent_t* evH = c->pipe_ev.data();
    cudaEvent_t* evC = evH + kMaxPipeBlocks;
    cudaEvent_t* evU = evH + 2 * kMaxPipeBlocks;
    cudaEvent_t evStart = evH[3 * kMaxPipeBlocks], evG = evH[3 * kMaxPipeBlocks + 1];
    const int src = c->cur;
    // earlier work on the context stream (steps reading buf[src]) comes first
    CUDA_TRY(c, cudaEventRecord(evStart, c->stream));
    CUDA_TRY(c, cudaStreamWaitEvent(c->h2d_stream, evStart, 0));
    CUDA_TRY(c, cudaStreamWaitEvent(c->d2h_stream, evStart, 0));
    if ((rc = copy_2d(c, sf2(c), const_cast<double*>(energy_surf), true, c->h2d_stream)) ||
        (rc = copy_2d(c, pb2(c), const_cast<double*>(energy_pbl), true, c->h2d_stream)))
        return rc;
    auto chunk_lo = [&](int b) { return (int)((long long)b * c->nchunks / nb); };
    auto row_lo = [&](int b) { return b == 0 ? 0LL : (long long)chunk_lo(b) * c->chunk + 1; };
    auto row_hi = [&](int b) {
        return b == nb - 1 ? ny + 1 : std::min<long long>(ny, (long long)chunk_lo(b + 1) * c->chunk);
    };
    // rows [r0, r1] of all k: nz runs of (nx+2)(r1-r0+1) doubles, one plane apart
    auto pcie = [&](double* dst, const double* srcp, long long r0, long long r1,
                    cudaMemcpyKind kind, cudaStream_t st) -> int {
        const size_t pitch = (size_t)hsk * 8, width = (size_t)(hsj * (r1 - r0 + 1)) * 8;
        CUDA_TRY(c, cudaMemcpy2DAsync(dst + r0 * hsj, pitch, srcp + r0 * hsj, pitch, width,
                                      (size_t)nz, kind, st));
        return HFTW_OK;
    };
    for (int b = 0; b < nb; ++b) {
        if ((rc = pcie(sin, e_in, row_lo(b), row_hi(b), cudaMemcpyHostToDevice, c->h2d_stream)))
            return rc;
        CUDA_TRY(c, cudaEventRecord(evH[b], c->h2d_stream));
    }
    const Dom d = make_dom(c);
    auto grid_rows = [&](long long r0, long long r1) {
        return (int)std::min<long long>((r1 - r0 + 1) * nz, (long long)c->num_sms * 8);
    };
    auto scatter = [&](int b) -> int {
        CUDA_TRY(c, cudaStreamWaitEvent(c->stream, evH[b], 0));
        hftw::copy_rows_kernel<<<grid_rows(row_lo(b), row_hi(b)), 256, 0, c->stream>>>(
            sin, hsj, hsk, e3(c, src), c->sj, c->sk, d, (int)row_lo(b), (int)row_hi(b));
        CUDA_TRY(c, cudaGetLastError());
        return HFTW_OK;
    };
    // energy_u of block b (physics of its input rows) needs only block b itself,
    // so it is computed right after the scatter and its D2H goes out one block
    // ahead of the new rows: the D2H stream starts earlier and drains sooner
    auto physics_rows = [&](int b) -> int {
        const long long r0 = row_lo(b), r1 = row_hi(b);
        hftw::physics_copy_kernel<<<grid_rows(r0, r1), 256, 0, c->stream>>>(
            e3(c, src), seu, hsj, hsk, sf2(c), pb2(c), d, (int)r0, (int)r1);
        CUDA_TRY(c, cudaGetLastError());
        CUDA_TRY(c, cudaEventRecord(evU[b], c->stream));
        return HFTW_OK;
    };
    auto eu_out = [&](int b) -> int {
        CUDA_TRY(c, cudaStreamWaitEvent(c->d2h_stream, evU[b], 0));
        return pcie(energy_u_out, seu, row_lo(b), row_hi(b), cudaMemcpyDeviceToHost,
                    c->d2h_stream);
    };
    if ((rc = scatter(0)) || (rc = physics_rows(0)) || (rc = eu_out(0))) return rc;
    for (int b = 0; b < nb; ++b) {
        if (b + 1 < nb && ((rc = scatter(b + 1)) || (rc = physics_rows(b + 1)))) return rc;
        const int ja = chunk_lo(b) * c->chunk + 1;
        const int jb = (int)std::min<long long>(ny, (long long)chunk_lo(b + 1) * c->chunk);
        const StepPart part{chunk_lo(b) * c->nstrips, chunk_lo(b + 1) * c->nstrips, ja, jb, 0};
        if ((rc = launch_fused<true>(c, src, HFTW_KERNEL_FUSED_TMA, &part))) return rc;
        hftw::copy_rows_kernel<<<grid_rows(ja, jb), 256, 0, c->stream>>>(
            e3(c, src ^ 1), c->sj, c->sk, sout, hsj, hsk, d, ja, jb);
        CUDA_TRY(c, cudaGetLastError());
        CUDA_TRY(c, cudaEventRecord(evC[b], c->stream));
        if (b + 1 < nb && (rc = eu_out(b + 1))) return rc;
        CUDA_TRY(c, cudaStreamWaitEvent(c->d2h_stream, evC[b], 0));
        if ((rc = pcie(energy_out, sout, ja, jb, cudaMemcpyDeviceToHost, c->d2h_stream)))
            return rc;
    }
    const StepPart ghosts{0, 0, 1, 0, 3};
    if ((rc = launch_fused<true>(c, src, HFTW_KERNEL_FUSED_TMA, &ghosts))) return rc;
    for (long long r : {0LL, ny + 1})
        hftw::copy_rows_kernel<<<grid_rows(r, r), 256, 0, c->stream>>>(
            e3(c, src ^ 1), c->sj, c->sk, sout, hsj, hsk, d, (int)r, (int)r);
    CUDA_TRY(c, cudaGetLastError());
    CUDA_TRY(c, cudaEventRecord(evG, c->stream));
    CUDA_TRY(c, cudaStreamWaitEvent(c->d2h_stream, evG, 0));
    if ((rc = pcie(energy_out, sout, 0, 0, cudaMemcpyDeviceToHost, c->d2h_stream)) ||
        (rc = pcie(energy_out, sout, ny + 1, ny + 1, cudaMemcpyDeviceToHost, c->d2h_stream)))
        return rc;
    CUDA_TRY(c, cudaStreamSynchronize(c->d2h_stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    // the context now holds the stepped state, as after upload x3 + step(1)
    c->cur ^= 1;
    c->eu_derived = true;
    c->eu_stored = false;
    c->eu_pending = false;
    c->poisoned = 0;
    ++c->step_count;
    return HFTW_OK;
}
} // namespace

extern "C" {

int hftw_get_plan(const hftw_ctx* c, hftw_plan* out) {
    if (!c || !out) return fail(nullptr, HFTW_EINVAL, "null argument");
    *out = c->plan; // a group: px x py of the whole grid, rank -1
    return HFTW_OK;
}

} // extern "C"
