// hftw.cu -- C ABI (include/hftw.h) over the B200 field store and kernels.
//
// Replaces, for the minimal-weather hot path, the reference's native
// simulator API in /root/reference/proj/include/hft/weather.hpp:
//   validate (:37), reference_init (:51), reference_step (:55),
//   run_reference (:59).
// The reference's SimState owns host std::vectors and swaps them each step
// (weather.cpp:170); here the context owns device-resident, padded fields in
// a ping-pong pair and the caller moves data in/out with upload/download.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hftw.h"
#include "weather_kernels.cuh"

using hftw::Dom;

namespace {

thread_local std::string g_err; // errors of calls without a context

constexpr int kFrontPad = 31; // IJK: logical i = 1 lands on a 256-byte boundary
constexpr int kNCW = 16;      // consumer warps of the TMA kernel
constexpr int kChunk = 32;    // rows per TMA work unit

} // namespace

struct hftw_ctx {
    hftw_grid g{};
    int layout = HFTW_IJK;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int kernel_req = HFTW_KERNEL_AUTO;
    int num_sms = 148;

    // geometry (elements)
    long long Pi = 0, Rows = 0;  // IJK row pitch, rows per plane (ny + 4)
    long long Pk = 0;            // KIJ column pitch
    long long si = 0, sj = 0, sk = 0, s2j = 0;
    long long off3 = 0, off2 = 0; // offset of logical (0,0,1) / (0,0) from allocation start
    size_t n3 = 0, n2 = 0;        // allocation sizes (elements)

    double* buf[2] = {nullptr, nullptr};
    double* sf = nullptr;
    double* pb = nullptr;
    double* staging = nullptr; // dense logical staging for the KIJ relayout
    int cur = 0;               // buf[cur] holds SimState::energy
    bool eu_derived = false;   // energy_u == physics(buf[cur ^ 1]), not yet materialised
    bool initialized = false;

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
    long long ghost_cells = 0;

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
    Dom d{};
    d.nx = (int)c->g.nx;
    d.ny = (int)c->g.ny;
    d.nz = (int)c->g.nz;
    d.si = c->si;
    d.sj = c->sj;
    d.sk = c->sk;
    d.s2j = c->s2j;
    d.own_w = d.own_e = d.own_s = d.own_n = 1;
    // one domain: the cyclic partners are local (weather.cpp:155-167)
    d.wfar = d.nx;
    d.efar = 1;
    d.sfar = d.ny;
    d.nfar = 1;
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

double* e3(const hftw_ctx* c, int b) { return c->buf[b] + c->off3; }
double* sf2(const hftw_ctx* c) { return c->sf + c->off2; }
double* pb2(const hftw_ctx* c) { return c->pb + c->off2; }

int grid_for(const hftw_ctx* c, long long n) {
    long long blocks = (n + 255) / 256;
    long long cap = (long long)c->num_sms * 16;
    return (int)std::max<long long>(1, std::min(blocks, cap));
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

template <int TX>
void set_tma_attrs(size_t smem) {
    cudaFuncSetAttribute(hftw::step_tma_kernel<TX, kNCW, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(hftw::step_tma_kernel<TX, kNCW, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

// Choose the TMA kernel geometry and build tensor maps + the per-CTA row
// ranges.  Leaves tma_ok = false (the cell kernel is used) when the grid does
// not fit: nz > 256 (TMA box limit) or a 4-stage ring would not fit smem.
int setup_tma(hftw_ctx* c) {
    c->tma_ok = false;
    if (c->layout != HFTW_IJK || c->g.nz > 256) return HFTW_OK;
    auto enc = encode_fn();
    if (!enc) return HFTW_OK;
    int smem_optin = 0;
    CUDA_TRY(c, cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                                       c->device));
    const int nz = (int)c->g.nz;
    int tx = 0, ns = 0;
    for (int cand : {64, 32}) {
        hftw::SlabGeom G = hftw::slab_geom(cand, nz);
        int fit = (int)((smem_optin - 1024) / (G.stage + 20));
        if (fit >= 4) {
            tx = cand;
            ns = std::min(fit, 8);
            break;
        }
    }
    if (!tx) return HFTW_OK;
    hftw::SlabGeom G = hftw::slab_geom(tx, nz);
    c->tx = tx;
    c->ns = ns;
    c->smem = (size_t)ns * G.stage + 2 * ns * sizeof(uint64_t) + ns * sizeof(int);
    if (tx == 64) set_tma_attrs<64>(c->smem);
    else set_tma_attrs<32>(c->smem);

    int per_sm = 0;
    cudaError_t oe =
        tx == 64 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                       &per_sm, hftw::step_tma_kernel<64, kNCW, true>, (kNCW + 1) * 32, c->smem)
                 : cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                       &per_sm, hftw::step_tma_kernel<32, kNCW, true>, (kNCW + 1) * 32, c->smem);
    if (oe != cudaSuccess || per_sm < 1) {
        cudaGetLastError();
        return HFTW_OK;
    }

    // tensor maps: e over {Pi, Rows, nz}, sf/pb over {Pi, Rows}
    const cuuint64_t dims3[3] = {(cuuint64_t)c->Pi, (cuuint64_t)c->Rows, (cuuint64_t)nz};
    const cuuint64_t strides3[2] = {(cuuint64_t)c->Pi * 8, (cuuint64_t)(c->Pi * c->Rows) * 8};
    const cuuint32_t box3[3] = {(cuuint32_t)G.w, 1, (cuuint32_t)nz};
    const cuuint32_t estr[3] = {1, 1, 1};
    for (int b = 0; b < 2; ++b) {
        CUresult r = enc(&c->tm_e[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, c->buf[b], dims3,
                         strides3, box3, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return HFTW_OK;
    }
    const cuuint64_t dims2[2] = {(cuuint64_t)c->Pi, (cuuint64_t)c->Rows};
    const cuuint64_t strides2[1] = {(cuuint64_t)c->Pi * 8};
    const cuuint32_t box2[2] = {(cuuint32_t)G.w, 1};
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
    const long long nx = c->g.nx, ny = c->g.ny;
    const int nstrips = (int)((nx + tx - 1) / tx);
    c->chunk = (int)std::min<long long>(kChunk, ny);
    c->nchunks = (int)((ny + c->chunk - 1) / c->chunk);
    const long long units = (long long)nstrips * c->nchunks;
    int ctas = (int)std::min<long long>((long long)per_sm * c->num_sms, units);
    if (!c->d_sched) {
        CUDA_TRY(c, cudaMalloc(&c->d_sched, 2 * sizeof(int)));
        CUDA_TRY(c, cudaMemset(c->d_sched, 0, 2 * sizeof(int)));
    }
    c->ctas = ctas;
    c->nstrips = nstrips;
    c->ghost_cells = (2 * nx + 2 * (ny + 2)) * (long long)nz;
    c->tma_ok = true;
    return HFTW_OK;
}

int resolved_kernel(const hftw_ctx* c) {
    if (c->kernel_req == HFTW_KERNEL_AUTO) return c->tma_ok ? HFTW_KERNEL_FUSED_TMA : HFTW_KERNEL_FUSED_CELL;
    return c->kernel_req;
}

// Launch the fused update from buf[src] into buf[src^1]; PHYS=false is the
// diffusion-only sweep of an already post-physics field.
template <bool PHYS>
int launch_fused(hftw_ctx* c, int src, int kernel) {
    Dom d = make_dom(c);
    if (kernel == HFTW_KERNEL_FUSED_TMA) {
        if (!c->tma_ok) return fail(c, HFTW_EUNSUP, "TMA kernel unavailable for this grid/layout");
        hftw::TmaArgs a{kFrontPad, 1, c->nstrips, c->nchunks, c->chunk, c->ns, c->ghost_cells,
                        c->d_sched};
        dim3 block((kNCW + 1) * 32);
        if (c->tx == 64)
            hftw::step_tma_kernel<64, kNCW, PHYS><<<c->ctas, block, c->smem, c->stream>>>(
                c->tm_e[src], c->tm_sf, c->tm_pb, e3(c, src), e3(c, src ^ 1), sf2(c), pb2(c), d,
                a);
        else
            hftw::step_tma_kernel<32, kNCW, PHYS><<<c->ctas, block, c->smem, c->stream>>>(
                c->tm_e[src], c->tm_sf, c->tm_pb, e3(c, src), e3(c, src ^ 1), sf2(c), pb2(c), d,
                a);
    } else {
        const long long n = (c->g.nx + 2) * (c->g.ny + 2) * c->g.nz;
        if (c->layout == HFTW_KIJ)
            hftw::step_cell_kernel<true, PHYS><<<grid_for(c, n), 256, 0, c->stream>>>(
                e3(c, src), e3(c, src ^ 1), sf2(c), pb2(c), d);
        else
            hftw::step_cell_kernel<false, PHYS><<<grid_for(c, n), 256, 0, c->stream>>>(
                e3(c, src), e3(c, src ^ 1), sf2(c), pb2(c), d);
    }
    CUDA_TRY(c, cudaGetLastError());
    return HFTW_OK;
}

int launch_physics(hftw_ctx* c, int b, int mode) {
    Dom d = make_dom(c);
    const long long cols = (c->g.nx + 2) * (c->g.ny + 2);
    const long long n = cols * c->g.nz;
    if (mode == 0) {
        if (c->layout == HFTW_KIJ)
            hftw::physics_kernel<true, true><<<grid_for(c, cols), 256, 0, c->stream>>>(
                e3(c, b), sf2(c), pb2(c), d);
        else
            hftw::physics_kernel<true, false><<<grid_for(c, cols), 256, 0, c->stream>>>(
                e3(c, b), sf2(c), pb2(c), d);
    } else {
        if (c->layout == HFTW_KIJ)
            hftw::physics_kernel<false, true><<<grid_for(c, n), 256, 0, c->stream>>>(
                e3(c, b), sf2(c), pb2(c), d);
        else
            hftw::physics_kernel<false, false><<<grid_for(c, n), 256, 0, c->stream>>>(
                e3(c, b), sf2(c), pb2(c), d);
    }
    CUDA_TRY(c, cudaGetLastError());
    return HFTW_OK;
}

// energy_u after a fused step is physics(previous energy); compute it in place
// in the buffer that holds the previous energy (it is dead until the next step
// overwrites it, so this is free of hazards).
int materialize_eu(hftw_ctx* c) {
    if (!c->eu_derived) return HFTW_OK;
    int rc = launch_physics(c, c->cur ^ 1, 1);
    if (rc) return rc;
    c->eu_derived = false;
    return HFTW_OK;
}

int check_ctx(hftw_ctx* c) {
    if (!c) return fail(nullptr, HFTW_EINVAL, "null context");
    CUDA_TRY(c, cudaSetDevice(c->device));
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
    if (ok && (g->nx > (1LL << 30) || g->ny > (1LL << 30) || g->nz > (1LL << 30)))
        out += "<config>: error: extents beyond 2^30 are not supported by the device store\n",
            ok = false;
    if (msg && cap) std::snprintf(msg, cap, "%s", out.c_str());
    if (!ok) {
        g_err = out;
        return HFTW_EINVAL;
    }
    return HFTW_OK;
}

int hftw_create(const hftw_grid* g, int layout, int device, hftw_ctx** out) {
    if (!out) return fail(nullptr, HFTW_EINVAL, "null output pointer");
    *out = nullptr;
    char msg[512];
    if (hftw_validate(g, msg, sizeof msg) != HFTW_OK) return fail(nullptr, HFTW_EINVAL, "%s", msg);
    if (layout != HFTW_IJK && layout != HFTW_KIJ)
        return fail(nullptr, HFTW_EINVAL, "unknown layout %d", layout);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(nullptr, HFTW_ECUDA, "no CUDA device available (the B200 path has no CPU fallback)");
    }
    if (device < 0 || device >= ndev) return fail(nullptr, HFTW_EINVAL, "bad device %d", device);

    hftw_ctx* c = new hftw_ctx();
    c->g = *g;
    c->layout = layout;
    c->device = device;
    auto bail = [&](int rc) {
        g_err = c->err;
        hftw_destroy(c);
        return rc;
    };
    if (cudaSetDevice(device) != cudaSuccess) return bail(fail(c, HFTW_ECUDA, "cudaSetDevice failed"));
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
        return bail(fail(c, HFTW_ECUDA, "stream creation failed"));
    c->own_stream = true;

    const long long nx = g->nx, ny = g->ny, nz = g->nz;
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
        // raw tuple (k, i, j), k fastest; columns padded to an even length
        c->Pk = (nz + 1) / 2 * 2;
        c->sk = 1;
        c->si = c->Pk;
        c->sj = c->Pk * (nx + 4);
        c->s2j = nx + 4;
        c->off3 = c->sj + c->si; // i = -1, j = -1 slots first
        c->off2 = c->s2j + 1;
        c->n3 = (size_t)(c->sj * (ny + 4));
        c->n2 = (size_t)((nx + 4) * (ny + 4));
    }
    for (int b = 0; b < 2; ++b)
        if (cudaMalloc(&c->buf[b], c->n3 * sizeof(double)) != cudaSuccess)
            return bail(fail(c, HFTW_ENOMEM, "cudaMalloc of %zu bytes failed", c->n3 * 8));
    if (cudaMalloc(&c->sf, c->n2 * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&c->pb, c->n2 * sizeof(double)) != cudaSuccess)
        return bail(fail(c, HFTW_ENOMEM, "cudaMalloc of 2D fields failed"));
    for (int b = 0; b < 2; ++b) cudaMemsetAsync(c->buf[b], 0, c->n3 * sizeof(double), c->stream);
    cudaMemsetAsync(c->sf, 0, c->n2 * sizeof(double), c->stream);
    cudaMemsetAsync(c->pb, 0, c->n2 * sizeof(double), c->stream);
    if (cudaStreamSynchronize(c->stream) != cudaSuccess)
        return bail(fail(c, HFTW_ECUDA, "initial memset failed"));
    int rc = setup_tma(c);
    if (rc) return bail(rc);
    *out = c;
    return HFTW_OK;
}

void hftw_destroy(hftw_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (int b = 0; b < 2; ++b)
        if (c->buf[b]) cudaFree(c->buf[b]);
    if (c->sf) cudaFree(c->sf);
    if (c->pb) cudaFree(c->pb);
    if (c->staging) cudaFree(c->staging);
    if (c->d_sched) cudaFree(c->d_sched);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

int hftw_init(hftw_ctx* c) {
    int rc = check_ctx(c);
    if (rc) return rc;
    for (int b = 0; b < 2; ++b)
        CUDA_TRY(c, cudaMemsetAsync(c->buf[b], 0, c->n3 * sizeof(double), c->stream));
    Dom d = make_dom(c);
    const long long n = (c->g.nx + 2) * (c->g.ny + 2) * c->g.nz;
    if (c->layout == HFTW_KIJ)
        hftw::init_kernel<true><<<grid_for(c, n), 256, 0, c->stream>>>(
            e3(c, c->cur), sf2(c), pb2(c), d, d.nx, d.ny, d.nz, 0, 0, c->g.surf_energy,
            c->g.pbl_energy);
    else
        hftw::init_kernel<false><<<grid_for(c, n), 256, 0, c->stream>>>(
            e3(c, c->cur), sf2(c), pb2(c), d, d.nx, d.ny, d.nz, 0, 0, c->g.surf_energy,
            c->g.pbl_energy);
    CUDA_TRY(c, cudaGetLastError());
    if (c->d_sched) CUDA_TRY(c, cudaMemsetAsync(c->d_sched, 0, 2 * sizeof(int), c->stream));
    c->eu_derived = false; // energy_u is all zeros (weather.cpp:82)
    c->initialized = true;
    return HFTW_OK;
}

static int copy_3d(hftw_ctx* c, double* dev_logical, double* host, bool h2d) {
    const long long nx = c->g.nx, ny = c->g.ny, nz = c->g.nz;
    if (c->layout == HFTW_IJK) {
        cudaMemcpy3DParms p{};
        cudaPitchedPtr hp = make_cudaPitchedPtr(host, (size_t)(nx + 2) * 8, (size_t)(nx + 2),
                                                (size_t)(ny + 2));
        // dev_logical points at logical (0,0,1); describe the allocation around it
        cudaPitchedPtr dp = make_cudaPitchedPtr(dev_logical - c->off3, (size_t)c->Pi * 8,
                                                (size_t)c->Pi, (size_t)c->Rows);
        cudaPos dpos = make_cudaPos((size_t)(c->off3 % c->Pi) * 8, (size_t)(c->off3 / c->Pi), 0);
        p.extent = make_cudaExtent((size_t)(nx + 2) * 8, (size_t)(ny + 2), (size_t)nz);
        if (h2d) {
            p.srcPtr = hp;
            p.dstPtr = dp;
            p.dstPos = dpos;
            p.kind = cudaMemcpyHostToDevice;
        } else {
            p.srcPtr = dp;
            p.srcPos = dpos;
            p.dstPtr = hp;
            p.kind = cudaMemcpyDeviceToHost;
        }
        CUDA_TRY(c, cudaMemcpy3DAsync(&p, c->stream));
        return HFTW_OK;
    }
    const long long n = (nx + 2) * (ny + 2) * nz;
    if (!c->staging) CUDA_TRY(c, cudaMalloc(&c->staging, (size_t)n * sizeof(double)));
    if (h2d) {
        CUDA_TRY(c, cudaMemcpyAsync(c->staging, host, (size_t)n * 8, cudaMemcpyHostToDevice,
                                    c->stream));
        hftw::relayout_kernel<true><<<grid_for(c, n), 256, 0, c->stream>>>(
            c->staging, dev_logical, nx + 2, ny + 2, nz, c->si, c->sj, c->sk);
        CUDA_TRY(c, cudaGetLastError());
    } else {
        hftw::relayout_kernel<false><<<grid_for(c, n), 256, 0, c->stream>>>(
            dev_logical, c->staging, nx + 2, ny + 2, nz, c->si, c->sj, c->sk);
        CUDA_TRY(c, cudaGetLastError());
        CUDA_TRY(c, cudaMemcpyAsync(host, c->staging, (size_t)n * 8, cudaMemcpyDeviceToHost,
                                    c->stream));
    }
    return HFTW_OK;
}

static int copy_2d(hftw_ctx* c, double* dev_logical, double* host, bool h2d) {
    const long long nx = c->g.nx, ny = c->g.ny;
    const size_t w = (size_t)(nx + 2) * 8;
    if (h2d)
        CUDA_TRY(c, cudaMemcpy2DAsync(dev_logical, (size_t)c->s2j * 8, host, w, w,
                                      (size_t)(ny + 2), cudaMemcpyHostToDevice, c->stream));
    else
        CUDA_TRY(c, cudaMemcpy2DAsync(host, w, dev_logical, (size_t)c->s2j * 8, w,
                                      (size_t)(ny + 2), cudaMemcpyDeviceToHost, c->stream));
    return HFTW_OK;
}

int hftw_upload(hftw_ctx* c, int field, const double* host) {
    int rc = check_ctx(c);
    if (rc) return rc;
    if (!valid_field(field) || !host) return fail(c, HFTW_EINVAL, "bad field %d or null buffer", field);
    double* h = const_cast<double*>(host);
    switch (field) {
    case HFTW_ENERGY:
        rc = copy_3d(c, e3(c, c->cur), h, true);
        break;
    case HFTW_ENERGY_U:
        rc = copy_3d(c, e3(c, c->cur ^ 1), h, true);
        c->eu_derived = false;
        break;
    case HFTW_ENERGY_SURF:
    case HFTW_ENERGY_PBL:
        // a derived energy_u depends on the boundary fields of its step
        if ((rc = materialize_eu(c))) return rc;
        rc = copy_2d(c, field == HFTW_ENERGY_SURF ? sf2(c) : pb2(c), h, true);
        break;
    }
    if (rc) return rc;
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    c->initialized = true;
    return HFTW_OK;
}

int hftw_download(hftw_ctx* c, int field, double* host) {
    int rc = check_ctx(c);
    if (rc) return rc;
    if (!valid_field(field) || !host) return fail(c, HFTW_EINVAL, "bad field %d or null buffer", field);
    switch (field) {
    case HFTW_ENERGY:
        rc = copy_3d(c, e3(c, c->cur), host, false);
        break;
    case HFTW_ENERGY_U:
        if ((rc = materialize_eu(c))) return rc;
        rc = copy_3d(c, e3(c, c->cur ^ 1), host, false);
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
    int rc = check_ctx(c);
    if (rc) return rc;
    if (nsteps < 0) return fail(c, HFTW_EINVAL, "steps must be nonnegative");
    if (nsteps == 0) return HFTW_OK;
    const int k = resolved_kernel(c);
    for (int64_t s = 0; s < nsteps; ++s) {
        if (k == HFTW_KERNEL_SPLIT) {
            // the reference's structure: physics in place, then diffusion
            if ((rc = launch_physics(c, c->cur, 0))) return rc;
            if ((rc = launch_fused<false>(c, c->cur, c->tma_ok ? HFTW_KERNEL_FUSED_TMA
                                                               : HFTW_KERNEL_FUSED_CELL)))
                return rc;
            c->eu_derived = false;
        } else {
            if ((rc = launch_fused<true>(c, c->cur, k))) return rc;
            c->eu_derived = true;
        }
        c->cur ^= 1;
    }
    return HFTW_OK;
}

int hftw_sync(hftw_ctx* c) {
    int rc = check_ctx(c);
    if (rc) return rc;
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
    if (k < HFTW_KERNEL_AUTO || k > HFTW_KERNEL_SPLIT) return fail(c, HFTW_EINVAL, "bad kernel %d", k);
    if (k == HFTW_KERNEL_FUSED_TMA && !c->tma_ok)
        return fail(c, HFTW_EUNSUP, "TMA kernel needs the IJK layout and nz <= 256");
    c->kernel_req = k;
    return HFTW_OK;
}

int hftw_get_kernel(const hftw_ctx* c) { return c ? resolved_kernel(c) : -1; }

int hftw_physics(hftw_ctx* c, int mode) {
    int rc = check_ctx(c);
    if (rc) return rc;
    if (mode != 0 && mode != 1) return fail(c, HFTW_EINVAL, "bad physics mode %d", mode);
    if ((rc = materialize_eu(c))) return rc;
    return launch_physics(c, c->cur, mode);
}

int hftw_diffuse(hftw_ctx* c) {
    int rc = check_ctx(c);
    if (rc) return rc;
    if ((rc = launch_fused<false>(c, c->cur, c->tma_ok ? HFTW_KERNEL_FUSED_TMA : HFTW_KERNEL_FUSED_CELL)))
        return rc;
    c->eu_derived = false; // energy_u = the diffused input (swap semantics)
    c->cur ^= 1;
    return HFTW_OK;
}

double hftw_algorithmic_bytes(const hftw_ctx* c, int what) {
    if (!c) return 0.0;
    const double cols = (double)(c->g.nx + 2) * (double)(c->g.ny + 2);
    const double cells = cols * (double)c->g.nz;
    switch (what) {
    case 0: return 16.0 * cells + 16.0 * cols; // read e, write u, read sf + pb
    case 1: return 16.0 * cells + 16.0 * cols; // physics: e read + write, sf + pb
    case 2: return 16.0 * cells;               // diffusion: read e, write u
    }
    return 0.0;
}

int hftw_launches_per_step(const hftw_ctx* c) {
    if (!c) return 0;
    return resolved_kernel(c) == HFTW_KERNEL_SPLIT ? 2 : 1;
}

int hftw_field_view(hftw_ctx* c, int field, void** dptr, int64_t strides[3]) {
    int rc = check_ctx(c);
    if (rc) return rc;
    if (!valid_field(field) || !dptr || !strides) return fail(c, HFTW_EINVAL, "bad arguments");
    if (field == HFTW_ENERGY_U && (rc = materialize_eu(c))) return rc;
    switch (field) {
    case HFTW_ENERGY: *dptr = e3(c, c->cur); break;
    case HFTW_ENERGY_U: *dptr = e3(c, c->cur ^ 1); break;
    case HFTW_ENERGY_SURF: *dptr = sf2(c); break;
    case HFTW_ENERGY_PBL: *dptr = pb2(c); break;
    }
    const bool f3 = field == HFTW_ENERGY || field == HFTW_ENERGY_U;
    strides[0] = f3 ? c->si : 1;
    strides[1] = f3 ? c->sj : c->s2j;
    strides[2] = f3 ? c->sk : 0;
    return HFTW_OK;
}

} // extern "C"
