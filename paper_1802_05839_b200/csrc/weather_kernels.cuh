// weather_kernels.cuh -- sm_100a kernels of the minimal-weather timestep.
//
// Reference hot path: hft::reference_step, /root/reference/proj/src/weather.cpp:101-171
//   (1) column physics in place            weather.cpp:118-128
//   (2) inner diffusion                    weather.cpp:130-137
//   (3) k = 1 / k = nz planes              weather.cpp:139-150
//   (4) j ghost rows (cyclic)              weather.cpp:152-159
//   (5) i ghost columns (cyclic, corners)  weather.cpp:161-168
//   (6) buffer swap                        weather.cpp:170
//
// Bitwise parity: every arithmetic operation is an explicitly rounded IEEE
// double op (__dadd_rn/__dsub_rn/__dmul_rn), which nvcc never contracts into
// DFMA, in exactly the reference's order and association.  Coefficients
// (1 - c*dv) are computed on the host the way the reference computes them.
//
// Fused formulation (SURVEY.md 8(a) "Fused-step specification"): the new
// value of a cell needs the post-physics value P of itself and of its
// neighbours; P is pointwise given sf/pb, so every kernel reads the
// pre-physics field e once and recomputes P on the fly.  The post-physics
// field (SimState::energy_u) is materialised only when somebody asks for it.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef HFTW_PDL
#define HFTW_PDL 1
#endif

namespace hftw {

// Programmatic dependent launch (the step kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization): let the next launch on the
// stream be scheduled now -- its CTAs take SMs as ours exit, so its launch and
// prologue overlap our tail -- then wait until the previous launch has completed and
// its writes are visible.  Called by every thread before any global memory access.
__device__ __forceinline__ void pdl_start() {
#if HFTW_PDL
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

// Device-side description of one (sub)domain.  Logical indices follow the
// reference: i in [0, nx+1], j in [0, ny+1], k in [1, nz]; the pointers
// passed to the kernels already point at logical (0, 0, 1) (3D) or (0, 0)
// (2D), and slots i = -1, nx+2 / j = -1, ny+2 exist (halo slots for the
// decomposed run; unused on one GPU).
struct Dom {
    int nx, ny, nz;       // (local) interior extents
    long long si, sj, sk; // 3D element strides
    long long s2j;        // 2D row stride (2D i-stride is 1)
    int own_w, own_e, own_s, own_n; // this domain owns the global ghost column/row
    int wfar, efar, sfar, nfar;     // index holding the cyclic partner of a ghost cell
    double ri, tv, dv;    // radiation_intensity, transfer_velocity, diffusion_velocity
    double c2, c5, c6;    // (1 - 2.0*dv), (1 - 5.0*dv), (1 - 6.0*dv) as in weather.cpp
};

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// Post-physics value of one cell, weather.cpp:122-127:
//   e = e + ri;  k==1: e = e - tv*(e - sf);  k==nz: e = e - tv*(e - pb).
template <bool PHYS>
__device__ __forceinline__ double phys(double ev, int k, int nz, double sfv, double pbv,
                                       double ri, double tv) {
    if (!PHYS) return ev;
    double p = dadd(ev, ri);
    if (k == 1) p = dsub(p, dmul(tv, dsub(p, sfv)));
    if (k == nz) p = dsub(p, dmul(tv, dsub(p, pbv)));
    return p;
}

// COHERENT: e is written by other CTAs during the launch (the multi-step
// kernel), so it is read through L2 (ld.global.cg), never the read-only path.
template <bool PHYS, bool COHERENT = false>
__device__ __forceinline__ double P_at(const double* __restrict__ e,
                                       const double* __restrict__ sf,
                                       const double* __restrict__ pb, const Dom& d, int i, int j,
                                       int k) {
    const double* pe = e + i * d.si + j * d.sj + (long long)(k - 1) * d.sk;
    double ev = COHERENT ? __ldcg(pe) : __ldg(pe);
    double sfv = 0.0, pbv = 0.0;
    if (PHYS && k == 1) sfv = __ldg(sf + i + j * d.s2j);
    if (PHYS && k == d.nz) pbv = __ldg(pb + i + j * d.s2j);
    return phys<PHYS>(ev, k, d.nz, sfv, pbv, d.ri, d.tv);
}

// New value of one owned cell, in the reference's region precedence
// (i ghosts win over j ghosts, which win over the k planes).
template <bool PHYS, bool COHERENT = false>
__device__ __forceinline__ double cell_update(const double* __restrict__ e,
                                              const double* __restrict__ sf,
                                              const double* __restrict__ pb, const Dom& d, int i,
                                              int j, int k) {
    if ((d.own_w && i == 0) || (d.own_e && i == d.nx + 1)) {
        // weather.cpp:164-167: (1-2dv)*e(i) + dv*(e(1) + e(nx))
        double a = P_at<PHYS, COHERENT>(e, sf, pb, d, i == 0 ? 1 : d.efar, j, k);
        double b = P_at<PHYS, COHERENT>(e, sf, pb, d, i == 0 ? d.wfar : d.nx, j, k);
        return dadd(dmul(d.c2, P_at<PHYS, COHERENT>(e, sf, pb, d, i, j, k)), dmul(d.dv, dadd(a, b)));
    }
    if ((d.own_s && j == 0) || (d.own_n && j == d.ny + 1)) {
        // weather.cpp:155-158: (1-2dv)*e(j) + dv*(e(ny) + e(1))
        double a = P_at<PHYS, COHERENT>(e, sf, pb, d, i, j == 0 ? d.sfar : d.ny, k);
        double b = P_at<PHYS, COHERENT>(e, sf, pb, d, i, j == 0 ? 1 : d.nfar, k);
        return dadd(dmul(d.c2, P_at<PHYS, COHERENT>(e, sf, pb, d, i, j, k)), dmul(d.dv, dadd(a, b)));
    }
    double c = P_at<PHYS, COHERENT>(e, sf, pb, d, i, j, k);
    double s = dadd(P_at<PHYS, COHERENT>(e, sf, pb, d, i - 1, j, k), P_at<PHYS, COHERENT>(e, sf, pb, d, i + 1, j, k));
    s = dadd(s, P_at<PHYS, COHERENT>(e, sf, pb, d, i, j - 1, k));
    s = dadd(s, P_at<PHYS, COHERENT>(e, sf, pb, d, i, j + 1, k));
    if (k == 1) { // weather.cpp:142-145
        s = dadd(s, P_at<PHYS, COHERENT>(e, sf, pb, d, i, j, 2));
        return dadd(dmul(d.c5, c), dmul(d.dv, s));
    }
    if (k == d.nz) { // weather.cpp:146-149
        s = dadd(s, P_at<PHYS, COHERENT>(e, sf, pb, d, i, j, d.nz - 1));
        return dadd(dmul(d.c5, c), dmul(d.dv, s));
    }
    // weather.cpp:134-137
    s = dadd(s, P_at<PHYS, COHERENT>(e, sf, pb, d, i, j, k - 1));
    s = dadd(s, P_at<PHYS, COHERENT>(e, sf, pb, d, i, j, k + 1));
    return dadd(dmul(d.c6, c), dmul(d.dv, s));
}

// Owned index ranges of a domain.
struct Owned {
    int i0, i1, j0, j1;
};
__device__ __forceinline__ Owned owned(const Dom& d) {
    return {d.own_w ? 0 : 1, d.own_e ? d.nx + 1 : d.nx, d.own_s ? 0 : 1,
            d.own_n ? d.ny + 1 : d.ny};
}

//------------------------------------------------------------------------------
// Multi-GPU halo protocol (2D I x J decomposition, one rank per GPU).
//
// Every launch computes step `step` (0-based) from buffer A into buffer B.
// Owned cells of B near a face are stored straight into the neighbours' copy
// of B (their halo slots, mapped over NVLink: CUDA IPC across processes, plain
// peer pointers within one) as they are computed: `depth` layers per face (2
// to an interior neighbour, so that a two-step pass finds a 2-deep halo; 1 to
// a wrap partner, whose far slot needs only the first inner column / row),
// and the corner cell column to a diagonal neighbour across two interior
// faces.  When all CTAs of the launch are done, the last one releases
// flag[opp(d)] = step + 1 in each neighbour d.  Work that reads a halo slot of
// A, or pushes into a neighbour, first acquires flag[d] >= step from every
// neighbour: they have finished step-1, so their pushes into A are complete
// and they no longer read the B slots we are about to overwrite (WAR safety
// with two buffers).  Interior work never waits, so the exchange overlaps it.
//------------------------------------------------------------------------------
constexpr int kNbrs = 8;      // W E S N faces, then SW SE NW NE corners
constexpr int kPubFlag = 8;   // my_flags[kPubFlag + d]: pass published by the wrap partner d
constexpr int kFlags = 12;
__host__ __device__ inline int opp_dir(int q) { return q < 4 ? q ^ 1 : q ^ 3; }

struct Halo {
    int active;                      // decomposed run
    double* nb[kNbrs];               // neighbour's destination buffer at its logical (0,0,1)
    long long nsi[kNbrs], nsj[kNbrs], nsk[kNbrs];
    int slot[4];                     // layer-1 column (W/E) or row (S/N) of my face in it
    int depth[4];                    // layers per face
    int cslot[4][2];                 // (i, j) of my corner column in the diagonal neighbour
    unsigned long long* my_flags;    // [kFlags], written by the neighbours
    unsigned long long* nb_flags[kNbrs]; // neighbour's flag array
    int* done;                       // CTAs of this launch that finished
    long long step;
    int nowait;                      // HFTW_TUNING experiments only: skip the flag waits
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// After ONE system-scope fence (__threadfence_system), relaxed stores of several
// flags are each a release (the PTX fence-then-relaxed-store pattern): a release
// store per flag would repeat the system-wide fence for every neighbour -- 8 of
// them cost a decomposed pass's ghost kernel ~15 us.
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Spin-wait watchdog: a flag wait that cannot end (a neighbour rank died or
// was never launched) traps after kSpinLimitNs, so the launch fails with an
// error instead of hanging the device.
constexpr unsigned long long kSpinLimitNs = 20ull * 1000ull * 1000ull * 1000ull;
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void spin_check(unsigned long long t0) {
    if (globaltimer_ns() - t0 > kSpinLimitNs) __trap();
}
__device__ __forceinline__ void wait_flag(const unsigned long long* f, long long target) {
    const unsigned long long t0 = globaltimer_ns();
    while ((long long)ld_acquire_sys(f) < target) {
        __nanosleep(64);
        spin_check(t0);
    }
}

// Wait until every neighbour finished step-1 (mask != 0: a unit on the rim).
__device__ __forceinline__ void halo_wait(const Halo& h, int mask) {
    if (!h.active || !mask || h.nowait) return;
    for (int q = 0; q < kNbrs; ++q)
        if (h.nb[q]) wait_flag(&h.my_flags[q], h.step);
}
// The same for a thread that waits for one step many times (a producer taking
// rim unit after rim unit): flags only grow, so once seen for `h.step` they
// stay satisfied and the later units of that step poll nothing.
__device__ __forceinline__ void halo_wait_once(const Halo& h, int mask, long long& seen) {
    if (!h.active || !mask || seen == h.step) return;
    halo_wait(h, mask);
    seen = h.step;
}

// Store a freshly computed OWNED cell into the neighbours that need it.
__device__ __forceinline__ void halo_push(const Halo& h, const Dom& d, int i, int j, int k,
                                          double v) {
    if (!h.active) return;
    const long long kk = (long long)(k - 1);
    auto put = [&](int q, long long ti, long long tj) {
        h.nb[q][ti * h.nsi[q] + tj * h.nsj[q] + kk * h.nsk[q]] = v;
    };
    if (h.nb[0] && i >= 1 && i <= h.depth[0]) put(0, h.slot[0] + (i - 1), j);
    if (h.nb[1] && i <= d.nx && i > d.nx - h.depth[1]) put(1, h.slot[1] - (d.nx - i), j);
    if (h.nb[2] && j >= 1 && j <= h.depth[2]) put(2, i, h.slot[2] + (j - 1));
    if (h.nb[3] && j <= d.ny && j > d.ny - h.depth[3]) put(3, i, h.slot[3] - (d.ny - j));
    if ((i == 1 || i == d.nx) && (j == 1 || j == d.ny)) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if (h.nb[4 + c] && i == ((c & 1) ? d.nx : 1) && j == ((c & 2) ? d.ny : 1))
                put(4 + c, h.cslot[c][0], h.cslot[c][1]);
    }
}

// Push the cells of the owned box [i0, i1] x [j0, j1] (all k) that lie within
// two of a face, read back from u, by the `nthr` threads `tid` of a CTA -- once
// the box's stores are complete and visible to them (a barrier).  The step
// kernels call it per work unit on the rim, outside their row loops: pushes
// inside the hot loops (inlined, or as a call) cost the row code 40% (register
// pressure of the call site, instruction-cache footprint) for 0.3% of the cells.
__device__ __forceinline__ void push_box(const Halo& h, const Dom& d, const double* u, int i0,
                                         int i1, int j0, int j1, int tid, int nthr) {
    // the box's columns / rows next to a face: 0..2 and n-1..n+1, up to six when
    // the box spans both faces (a whole owned box, or a narrow subdomain)
    // (the two ranges directly: a scan of the box would cost O(width) per thread)
    int cs[6], rs[6], nc = 0, nr = 0;
    for (int i = i0; i <= min(i1, 2); ++i) cs[nc++] = i;
    for (int i = max(i0, max(d.nx - 1, 3)); i <= i1; ++i) cs[nc++] = i;
    for (int j = j0; j <= min(j1, 2); ++j) rs[nr++] = j;
    for (int j = max(j0, max(d.ny - 1, 3)); j <= j1; ++j) rs[nr++] = j;
    const int nj = j1 - j0 + 1, ni = i1 - i0 + 1;
    const long long a = (long long)nc * nj;       // face columns x all rows
    const long long b = (long long)nr * ni;       // face rows x all columns (dups skipped)
    const long long n = (a + b) * d.nz;
    for (long long t = tid; t < n; t += nthr) {
        const int k = 1 + (int)(t / (a + b));
        const long long r = t % (a + b);
        int i, j;
        if (r < a) {
            i = cs[r % nc];
            j = j0 + (int)(r / nc);
        } else {
            const long long q = r - a;
            i = i0 + (int)(q % ni);
            j = rs[q / ni];
            bool dup = false;
            for (int m = 0; m < nc; ++m) dup |= cs[m] == i;
            if (dup) continue;
        }
        halo_push(h, d, i, j, k, u[i * d.si + j * d.sj + (long long)(k - 1) * d.sk]);
    }
}

// A work unit (columns i0 .. i0+w-1, rows ja .. jb) reads halo slots or pushes
// into a neighbour iff it touches the two cells next to a face.
__device__ __forceinline__ int rim_unit(const Dom& d, int i0, int w, int ja, int jb) {
    return (i0 <= 2 || i0 + w - 1 >= d.nx - 1 || ja <= 2 || jb >= d.ny - 1) ? 1 : 0;
}

// Called by ONE thread per CTA after a barrier over the CTA's working
// threads: the last CTA of the launch publishes step+1 to the neighbours.
__device__ __forceinline__ void halo_signal(const Halo& h) {
    if (!h.active) return;
    __threadfence_system();
    if (atomicAdd(h.done, 1) == (int)gridDim.x - 1) {
        __threadfence_system();
        for (int q = 0; q < kNbrs; ++q)
            if (h.nb[q]) st_relaxed_sys(&h.nb_flags[q][opp_dir(q)], (unsigned long long)(h.step + 1));
        *h.done = 0;
        __threadfence();
    }
}

// The neighbours' 2D fields (sf, pb): static, pushed once after init / upload.
struct Halo2D {
    double* sf[kNbrs];
    double* pb[kNbrs];
    long long s2j[kNbrs];
};

//------------------------------------------------------------------------------
// FUSED_CELL: one owned cell per thread, fastest storage dimension first.
// Valid for every layout; the generic path and the correctness baseline.
//------------------------------------------------------------------------------
template <bool KFAST, bool PHYS>
__global__ void __launch_bounds__(256) step_cell_kernel(const double* __restrict__ e,
                                                        double* __restrict__ u,
                                                        const double* __restrict__ sf,
                                                        const double* __restrict__ pb, Dom d,
                                                        Halo h) {
    if (h.active) {
        if (threadIdx.x == 0) halo_wait(h, 0xF);
        __syncthreads();
    }
    Owned o = owned(d);
    const long long ni = o.i1 - o.i0 + 1, nj = o.j1 - o.j0 + 1, nk = d.nz;
    const long long n = ni * nj * nk;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        int i, j, k;
        if (KFAST) {
            k = 1 + (int)(t % nk);
            long long r = t / nk;
            i = o.i0 + (int)(r % ni);
            j = o.j0 + (int)(r / ni);
        } else {
            i = o.i0 + (int)(t % ni);
            long long r = t / ni;
            j = o.j0 + (int)(r % nj);
            k = 1 + (int)(r / nj);
        }
        const double v = cell_update<PHYS>(e, sf, pb, d, i, j, k);
        u[i * d.si + j * d.sj + (long long)(k - 1) * d.sk] = v;
        halo_push(h, d, i, j, k, v);
    }
    if (h.active) {
        __syncthreads();
        if (threadIdx.x == 0) halo_signal(h);
    }
}

// The un-overlapped exchange baseline (HFTW_OPT_EXCHANGE = 1): after a step
// without pushes, copy this rank's cells near the faces into the neighbours.
__global__ void __launch_bounds__(256) face_push_kernel(const double* __restrict__ u, Dom d,
                                                        const __grid_constant__ Halo h) {
    const Owned o = owned(d);
    push_box(h, d, u, o.i0, o.i1, o.j0, o.j1, blockIdx.x * blockDim.x + threadIdx.x,
             gridDim.x * blockDim.x);
}

// Initial / post-upload halo fill: push the current field's owned cells and
// the static sf/pb values near the faces into the neighbours' halo slots with
// the step kernels' rules (host brackets it with barriers).  A sweep over the
// owned cells; only those near a face store anything.
__global__ void exchange_kernel(const double* __restrict__ e, const double* __restrict__ sf,
                                const double* __restrict__ pb, Dom d, Halo h, Halo2D h2) {
    const Owned o = owned(d);
    const long long ni = o.i1 - o.i0 + 1, nj = o.j1 - o.j0 + 1;
    const long long n = ni * nj * d.nz;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        const int i = o.i0 + (int)(t % ni);
        const long long r = t / ni;
        const int j = o.j0 + (int)(r % nj);
        const int k = 1 + (int)(r / nj);
        const bool near_i = i <= 2 || i >= d.nx - 1, near_j = j <= 2 || j >= d.ny - 1;
        if (!near_i && !near_j) continue;
        halo_push(h, d, i, j, k, e[i * d.si + j * d.sj + (long long)(k - 1) * d.sk]);
        if (k == 1) {
            // the same targets with 2D strides (k = 1 of a 2D field)
            Halo hs = h, hp = h;
            for (int q = 0; q < kNbrs; ++q) {
                hs.nb[q] = h2.sf[q];
                hp.nb[q] = h2.pb[q];
                hs.nsi[q] = hp.nsi[q] = 1;
                hs.nsj[q] = hp.nsj[q] = h2.s2j[q];
            }
            halo_push(hs, d, i, j, 1, sf[i + j * d.s2j]);
            halo_push(hp, d, i, j, 1, pb[i + j * d.s2j]);
        }
    }
}

//------------------------------------------------------------------------------
// Column physics alone, in place (weather.cpp:118-128): BASELINE config (3).
//  physics_column_kernel: one (i,j) column per thread with the k loop in
//      registers -- the reference's emitted GPU mapping (hfk0_radiate +
//      hfk0_exchange_heat_with_boundary, emit_cuda.cpp:159-214).  Coalesced in
//      IJK; in KIJ neighbouring threads are a column apart (the paper's
//      storage-order penalty).  Loads are batched 8 deep.
//  physics_rows_kernel (IJK): one (j,k) row per block pass, i across threads.
//  physics_kij_kernel (KIJ): one column per warp, lanes along k -- the
//      KIJ-aware mapping; physics_kij_stream_kernel streams whole rows.
//------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) physics_column_kernel(double* __restrict__ e,
                                                             const double* __restrict__ sf,
                                                             const double* __restrict__ pb,
                                                             Dom d) {
    pdl_start();
    Owned o = owned(d);
    const int ni = o.i1 - o.i0 + 1, nj = o.j1 - o.j0 + 1;
    const long long n = (long long)ni * nj;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        const int i = o.i0 + (int)(t % ni), j = o.j0 + (int)(t / ni);
        double* col = e + i * d.si + j * d.sj;
        const double s = __ldg(sf + i + j * d.s2j), b = __ldg(pb + i + j * d.s2j);
        for (int k0 = 1; k0 <= d.nz; k0 += 8) {
            double v[8];
#pragma unroll
            for (int m = 0; m < 8; ++m)
                if (k0 + m <= d.nz) v[m] = col[(long long)(k0 + m - 1) * d.sk];
#pragma unroll
            for (int m = 0; m < 8; ++m)
                if (k0 + m <= d.nz)
                    col[(long long)(k0 + m - 1) * d.sk] =
                        phys<true>(v[m], k0 + m, d.nz, s, b, d.ri, d.tv);
        }
    }
}

__global__ void __launch_bounds__(256) physics_rows_kernel(double* __restrict__ e,
                                                           const double* __restrict__ sf,
                                                           const double* __restrict__ pb,
                                                           Dom d) {
    Owned o = owned(d);
    const int nj = o.j1 - o.j0 + 1;
    const long long rows = (long long)nj * d.nz;
    for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
        const int j = o.j0 + (int)(r % nj), k = 1 + (int)(r / nj);
        double* row = e + j * d.sj + (long long)(k - 1) * d.sk;
        const double* srow = sf + j * d.s2j;
        const double* brow = pb + j * d.s2j;
        for (int i = o.i0 + threadIdx.x; i <= o.i1; i += blockDim.x) {
            double sfv = 0.0, pbv = 0.0;
            if (k == 1) sfv = __ldg(srow + i);
            if (k == d.nz) pbv = __ldg(brow + i);
            row[i] = phys<true>(row[i], k, d.nz, sfv, pbv, d.ri, d.tv);
        }
    }
}

// KIJ, streaming: consecutive columns of a row are ONE contiguous run of
// Pk-double columns, so a warp takes 16 columns at a time and its lanes walk
// that run 32 doubles apart -- fully coalesced -- tracking (column, k)
// incrementally (no divisions; Pk >= 32 assumed, else the warp kernel runs).
__global__ void __launch_bounds__(256) physics_kij_stream_kernel(double* __restrict__ e,
                                                                 const double* __restrict__ sf,
                                                                 const double* __restrict__ pb,
                                                                 Dom d, int pk) {
    pdl_start();
    constexpr int CPW = 16; // columns per warp task
    const Owned o = owned(d);
    const int ni = o.i1 - o.i0 + 1, nj = o.j1 - o.j0 + 1;
    const int tasks_row = (ni + CPW - 1) / CPW;
    const long long tasks = (long long)tasks_row * nj;
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long w = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); w < tasks;
         w += warps) {
        const int j = o.j0 + (int)(w / tasks_row);
        const int c0 = o.i0 + (int)(w % tasks_row) * CPW;
        const int nc = min(CPW, o.i1 - c0 + 1);
        double* base = e + c0 * d.si + j * d.sj; // column c0, k = 1
        const double* sfr = sf + j * d.s2j;
        const double* pbr = pb + j * d.s2j;
        int c = 0, kk = lane; // this lane's element: column c0 + c, plane kk + 1
        const int n = nc * pk;
        for (int q = lane; q < n; q += 4 * 32) {
            // four loads in flight per lane before any store
            double v[4];
            int cs[4], ks[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                cs[u] = c;
                ks[u] = kk;
                v[u] = q + 32 * u < n ? base[q + 32 * u] : 0.0;
                kk += 32;
                if (kk >= pk) {
                    kk -= pk;
                    ++c;
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (q + 32 * u >= n || ks[u] >= d.nz) continue;
                const int k = ks[u] + 1, i = c0 + cs[u];
                double sfv = 0.0, pbv = 0.0;
                if (k == 1) sfv = __ldg(sfr + i);
                if (k == d.nz) pbv = __ldg(pbr + i);
                base[q + 32 * u] = phys<true>(v[u], k, d.nz, sfv, pbv, d.ri, d.tv);
            }
        }
    }
}

__global__ void __launch_bounds__(256) physics_kij_kernel(double* __restrict__ e,
                                                          const double* __restrict__ sf,
                                                          const double* __restrict__ pb,
                                                          Dom d) {
    Owned o = owned(d);
    const int ni = o.i1 - o.i0 + 1, nj = o.j1 - o.j0 + 1;
    const long long cols = (long long)ni * nj;
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long cw = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); cw < cols;
         cw += warps) {
        const int i = o.i0 + (int)(cw % ni), j = o.j0 + (int)(cw / ni);
        double* col = e + i * d.si + j * d.sj; // k contiguous (sk == 1)
        const double s = __ldg(sf + i + j * d.s2j), b = __ldg(pb + i + j * d.s2j);
        for (int k = 1 + lane; k <= d.nz; k += 32)
            col[k - 1] = phys<true>(col[k - 1], k, d.nz, s, b, d.ri, d.tv);
    }
}

// Row-block kernels of hftw_step_host.  The host arrays use the logical
// column-major layout (i fastest, then j, then k), so rows [j0, j1] of all k
// are nz equal runs one host plane apart: the library stages them densely in
// HBM in that same layout (dst/src with strides dsj, dsk) so each block
// crosses PCIe as ONE 2D copy of nz large rows.
//  physics_copy_kernel: dst = physics(src) (energy_u, weather.cpp:118-128).
//  copy_rows_kernel:    dst = src (field <-> dense staging).
// Both cover the owned columns of rows [j0, j1] (clipped to the owned rows).
__global__ void __launch_bounds__(256) physics_copy_kernel(const double* __restrict__ src,
                                                           double* __restrict__ dst,
                                                           long long dsj, long long dsk,
                                                           const double* __restrict__ sf,
                                                           const double* __restrict__ pb,
                                                           Dom d, int j0, int j1) {
    Owned o = owned(d);
    j0 = max(j0, o.j0);
    j1 = min(j1, o.j1);
    const int nj = j1 - j0 + 1;
    if (nj <= 0) return;
    const long long rows = (long long)nj * d.nz;
    for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
        const int j = j0 + (int)(r % nj), k = 1 + (int)(r / nj);
        const double* s = src + j * d.sj + (long long)(k - 1) * d.sk;
        double* t = dst + j * dsj + (long long)(k - 1) * dsk;
        for (int i = o.i0 + threadIdx.x; i <= o.i1; i += blockDim.x) {
            double sfv = 0.0, pbv = 0.0;
            if (k == 1) sfv = __ldg(sf + i + j * d.s2j);
            if (k == d.nz) pbv = __ldg(pb + i + j * d.s2j);
            t[i] = phys<true>(__ldg(s + i * d.si), k, d.nz, sfv, pbv, d.ri, d.tv);
        }
    }
}

__global__ void __launch_bounds__(256) copy_rows_kernel(const double* __restrict__ src,
                                                        long long ssj, long long ssk,
                                                        double* __restrict__ dst, long long dsj,
                                                        long long dsk, Dom d, int j0, int j1) {
    Owned o = owned(d);
    j0 = max(j0, o.j0);
    j1 = min(j1, o.j1);
    const int nj = j1 - j0 + 1;
    if (nj <= 0) return;
    const long long rows = (long long)nj * d.nz;
    for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
        const int j = j0 + (int)(r % nj);
        const long long k0 = r / nj;
        const double* s = src + j * ssj + k0 * ssk;
        double* t = dst + j * dsj + k0 * dsk;
        for (int i = o.i0 + threadIdx.x; i <= o.i1; i += blockDim.x) t[i] = __ldg(s + i);
    }
}

//------------------------------------------------------------------------------
// Device-side reference_init (weather.cpp:86-98): 300 inside the integer box
// [n/4, 3n/4] of every dimension, 0 elsewhere (buffers pre-zeroed); surface
// and boundary-layer constants over all columns.
//------------------------------------------------------------------------------
template <bool KFAST>
__global__ void init_kernel(double* __restrict__ e, double* __restrict__ sf,
                            double* __restrict__ pb, Dom d, int gnx, int gny, int gnz, int gi0,
                            int gj0, double surf, double pbl) {
    Owned o = owned(d);
    const long long ni = o.i1 - o.i0 + 1, nj = o.j1 - o.j0 + 1, nk = d.nz;
    const long long n = ni * nj * nk;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        int i, j, k;
        if (KFAST) {
            k = 1 + (int)(t % nk);
            long long r = t / nk;
            i = o.i0 + (int)(r % ni);
            j = o.j0 + (int)(r / ni);
        } else {
            i = o.i0 + (int)(t % ni);
            long long r = t / ni;
            j = o.j0 + (int)(r % nj);
            k = 1 + (int)(r / nj);
        }
        const long long gi = gi0 + i, gj = gj0 + j; // global logical indices
        const bool in = gi >= gnx / 4 && gi <= (3LL * gnx) / 4 && gj >= gny / 4 &&
                        gj <= (3LL * gny) / 4 && k >= gnz / 4 && k <= (3LL * gnz) / 4;
        e[i * d.si + j * d.sj + (long long)(k - 1) * d.sk] = in ? 300.0 : 0.0;
        if (k == 1) {
            sf[i + j * d.s2j] = surf;
            pb[i + j * d.s2j] = pbl;
        }
    }
}

// L2 eviction for measurements: stream-write a scratch buffer.
__global__ void flush_kernel(double4* __restrict__ p, long long n, double v) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x)
        p[t] = make_double4(v, v, v, v);
}

// Logical column-major dense <-> strided device layout (upload/download of
// the KIJ store).  One thread per logical element in logical order, so the
// dense side is coalesced.
template <bool TO_STRIDED>
__global__ void relayout_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                long long ni, long long nj, long long nk, long long si,
                                long long sj, long long sk) {
    const long long n = ni * nj * nk;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        long long i = t % ni, r = t / ni, j = r % nj, k = r / nj;
        long long off = i * si + j * sj + k * sk;
        if (TO_STRIDED) dst[off] = src[t];
        else dst[t] = src[off];
    }
}

//------------------------------------------------------------------------------
// FUSED_TMA: the roofline kernel for the IJK store.
//
// Work decomposition: the interior (i in 1..nx, j in 1..ny) is cut into
// i-strips of TX cells; a CTA owns a contiguous range of (strip, row) pairs and
// marches along j.  For every row it streams one SLAB -- the (TX+2) x nz
// block {i0-2 .. i0+TX+1} x {j} x {1..nz} -- into shared memory with ONE 3D TMA
// load (box {TX+4, 1, nz}), plus the matching sf/pb rows.  Row j is computed
// from slabs j-1, j, j+1 held in an NS-deep mbarrier ring, so each e value
// crosses HBM once (plus a 2/TX halo share that L2 serves) and u is written
// once with 256-byte aligned coalesced stores.  The k direction needs no halo
// at all: the whole column is in the slab.
//
// Warp roles: NCW consumer warps compute; one producer warp issues the TMA
// loads.  Ghost cells (regions 4 and 5 of the reference, 0.3% of cells at
// ASUCA size) are computed by the consumers from global memory in the
// prologue while the first slabs are in flight.
//------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "HFTW_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra HFTW_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// The same with the barrier's shared-window address computed once by the caller
// (the generic-to-shared conversion costs a handful of instructions per call).
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "HFTW_WAITU_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra HFTW_WAITU_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// Shared-memory geometry of one pipeline stage.
//  IJK: a slab row spans logical i0-2 .. i0+TX+1 (TX + 4 doubles) for every k
//       ([k][i] in smem): the TMA box must START on a 16-byte boundary (an odd
//       fp64 coordinate faults with an illegal instruction on sm_100a) and the
//       stores keep i0 on a 256-byte boundary, so the box begins one element
//       before the i0-1 halo.  Column c of a slab row holds logical i0-2+c.
//  KIJ: a slab is the CONTIGUOUS block of columns i0-1 .. i0+TX, each Pk
//       doubles of k ([i][k] in smem); Pk = 2 (mod 4) makes lanes that walk
//       across columns at one k bank-conflict free for 64-bit accesses.
//  Both: the sf/pb rows span i0-2 .. i0+TX+1.
struct SlabGeom {
    int w;          // slab step between k and k+1 (doubles)
    int is;         // slab step between i and i+1 (doubles)
    int e_bytes;    // slab bytes rounded to 128
    int r_bytes;    // one sf/pb row rounded to 128
    int stage;      // e + sf + pb
    int tx_bytes;   // bytes the TMA actually delivers per stage
    int out_bytes;  // KIJ: one staged output row (TX x Pk), rounded to 128
};
__host__ __device__ inline SlabGeom slab_geom(int tx, int nz) {
    SlabGeom g;
    g.w = tx + 4;
    g.is = 1;
    g.e_bytes = ((g.w * nz * 8) + 127) / 128 * 128;
    g.r_bytes = (((tx + 4) * 8) + 127) / 128 * 128;
    g.stage = g.e_bytes + 2 * g.r_bytes;
    g.tx_bytes = g.w * nz * 8 + 2 * (tx + 4) * 8;
    g.out_bytes = 0;
    return g;
}
__host__ __device__ inline SlabGeom slab_geom_kij(int tx, int pk) {
    SlabGeom g;
    g.w = 1;
    g.is = pk;
    g.e_bytes = (((tx + 2) * pk * 8) + 127) / 128 * 128;
    g.r_bytes = (((tx + 4) * 8) + 127) / 128 * 128;
    g.stage = g.e_bytes + 2 * g.r_bytes;
    g.tx_bytes = (tx + 2) * pk * 8 + 2 * (tx + 4) * 8;
    g.out_bytes = ((tx * pk * 8) + 127) / 128 * 128;
    return g;
}

__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                 "r"(smem_u32(ssrc)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

struct TmaArgs {
    int fp;        // tensor-map i coordinate of logical i = 0
    int jrow0;     // tensor-map row coordinate of logical j = 0
    int nstrips;   // i-strips of TX cells over 1..nx
    int nchunks;   // j-chunks of `chunk` rows over 1..ny
    int chunk;
    int ns;        // pipeline depth (stages)
    int pk;        // KIJ column pitch (doubles)
    long long ghost_cells;
    int* sched;    // [0] next work unit, [1] CTAs finished (self-resetting)
    int reverse;   // HFTW_OPT_REVERSE: hand the units out last first
    // Sub-range launches (hftw_step_host pipelines a step in row blocks):
    // units [u_lo, u_hi) of the j-major order, the i-ghost columns of rows
    // [gi_lo, gi_hi] (clipped to the owned inner rows) and the j-ghost rows
    // in gj_mask (bit 0 = j = 0, bit 1 = j = ny+1; owned rows only).  A whole
    // step is u = [0, units), rows [1, ny], mask 3.
    int u_lo, u_hi;
    int gi_lo, gi_hi;
    int gj_mask;
};

// Post-physics value of a slab element for a cell that is NOT on k = 1 / nz.
template <bool PHYS>
__device__ __forceinline__ double pin(double ev, double ri) {
    return PHYS ? dadd(ev, ri) : ev;
}

// One thread's share of one row in the TMA kernel: column i of the strip,
// k in [kl, kh], with slabs j-1 (em), j (e0), j+1 (ep) in shared memory
// (pointers already at the thread's slab column; +-is are the i neighbours,
// +-w the k neighbours).  A three-value register window carries P(k-1),
// P(k), P(k+1); interior k run a branch-free loop, k = 1 / nz-1 / nz take
// the boundary-aware path.
struct ColumnRow {
    const double *em, *e0, *ep;  // slab rows j-1, j, j+1
    const double *Sm, *S0, *Sp;  // sf rows
    const double *Bm, *B0, *Bp;  // pb rows
    double* up;                  // output at (i, j, kl): global (IJK) or smem staging (KIJ)
    long long sk;                // output step between k and k+1
    int w, is;                   // slab steps between k and k+1, i and i+1
    int kl, kh, nz;
    double ri, tv, dv, c5, c6;
    int i, j;
};

template <bool PHYS>
__device__ __forceinline__ void column_row(const ColumnRow& r) {
    const int w = r.w, is = r.is, nz = r.nz;
    const double ri = r.ri, tv = r.tv, dv = r.dv, c6 = r.c6;
    auto Pc = [&](int kk) {
        return phys<PHYS>(r.e0[(kk - 1) * w], kk, nz, r.S0[0], r.B0[0], ri, tv);
    };
    // boundary-aware cell (k = 1, nz-1, nz; any k is correct here)
    auto edge = [&](int k, double pd, double pc, double& pn) {
        pn = k < nz ? Pc(k + 1) : 0.0;
        const int o = (k - 1) * w;
        double s6 = dadd(phys<PHYS>(r.e0[o - is], k, nz, r.S0[-1], r.B0[-1], ri, tv),
                         phys<PHYS>(r.e0[o + is], k, nz, r.S0[1], r.B0[1], ri, tv));
        s6 = dadd(s6, phys<PHYS>(r.em[o], k, nz, r.Sm[0], r.Bm[0], ri, tv));
        s6 = dadd(s6, phys<PHYS>(r.ep[o], k, nz, r.Sp[0], r.Bp[0], ri, tv));
        if (k == 1) return dadd(dmul(r.c5, pc), dmul(dv, dadd(s6, pn)));  // weather.cpp:142-145
        if (k == nz) return dadd(dmul(r.c5, pc), dmul(dv, dadd(s6, pd))); // weather.cpp:146-149
        return dadd(dmul(c6, pc), dmul(dv, dadd(dadd(s6, pd), pn)));      // weather.cpp:134-137
    };
    double pd = r.kl > 1 ? Pc(r.kl - 1) : 0.0;
    double pc = Pc(r.kl);
    int k = r.kl;
    for (; k <= r.kh && k < 2; ++k) { // k = 1
        double pn;
        const double out = edge(k, pd, pc, pn);
        r.up[(long long)(k - r.kl) * r.sk] = out;
        pd = pc;
        pc = pn;
    }
    const int kf = min(r.kh, nz - 2);
    if (k <= kf) {
        // interior k: weather.cpp:134-137 with P = e + ri for every operand
        const double* p0 = r.e0 + (k - 1) * w;
        const double* pm = r.em + (k - 1) * w;
        const double* pp = r.ep + (k - 1) * w;
        double* q = r.up + (long long)(k - r.kl) * r.sk;
#pragma unroll 4
        for (; k <= kf; ++k) {
            const double pn = pin<PHYS>(p0[w], ri);
            double s6 = dadd(pin<PHYS>(p0[-is], ri), pin<PHYS>(p0[is], ri));
            s6 = dadd(s6, pin<PHYS>(pm[0], ri));
            s6 = dadd(s6, pin<PHYS>(pp[0], ri));
            s6 = dadd(dadd(s6, pd), pn);
            const double out = dadd(dmul(c6, pc), dmul(dv, s6));
            *q = out;
            q += r.sk;
            p0 += w;
            pm += w;
            pp += w;
            pd = pc;
            pc = pn;
        }
    }
    for (; k <= r.kh; ++k) { // k = nz-1, nz
        double pn;
        const double out = edge(k, pd, pc, pn);
        r.up[(long long)(k - r.kl) * r.sk] = out;
        pd = pc;
        pc = pn;
    }
}

template <int TX, int NCW, bool PHYS, bool KIJ>
__global__ void __launch_bounds__((NCW + 1) * 32, 1)
    step_tma_kernel(const __grid_constant__ CUtensorMap tm_e,
                    const __grid_constant__ CUtensorMap tm_sf,
                    const __grid_constant__ CUtensorMap tm_pb, const double* __restrict__ e,
                    double* __restrict__ u, const double* __restrict__ sf,
                    const double* __restrict__ pb, Dom d, TmaArgs a,
                    const __grid_constant__ Halo h) {
    extern __shared__ __align__(128) unsigned char smem[];
    const SlabGeom G = KIJ ? slab_geom_kij(TX, a.pk) : slab_geom(TX, d.nz);
    const int NS = a.ns;
    unsigned char* outbuf = smem + (size_t)NS * G.stage; // KIJ: two staged output rows
    uint64_t* full = reinterpret_cast<uint64_t*>(outbuf + 2 * (size_t)G.out_bytes);
    uint64_t* empty = full + NS;
    int* slot_unit = reinterpret_cast<int*>(empty + NS); // work unit of each staged slab
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    pdl_start();

    if (warp == NCW) {
        // ---------------- producer: work scheduler + TMA issue ----------------
        // Units are handed out j-major (all strips of chunk 0, then chunk 1, ...)
        // so the CTAs in flight sweep the grid as one front and the slab
        // halo columns / chunk-boundary rows another CTA needs are still in L2.
        if (lane == 0) {
            uint32_t L = 0;
            long long seen = -1; // the step whose neighbour flags this producer has seen
            for (;;) {
                const int v = atomicAdd(&a.sched[0], 1);
                const bool stop = v >= a.u_hi - a.u_lo;
                const int unit = a.reverse ? a.u_hi - 1 - v : a.u_lo + v;
                int ja = 0, jb = -1, ic = 0;
                if (!stop) {
                    const int ch = unit / a.nstrips, st = unit % a.nstrips;
                    ja = ch * a.chunk + 1;
                    jb = min(d.ny, ja + a.chunk - 1);
                    // IJK: tensor coordinate of i0 - 2 (even); KIJ: of column i0 - 1
                    ic = KIJ ? 1 + st * TX : a.fp + 1 + st * TX - 2;
                    // a unit on the subdomain rim reads halo slots and pushes
                    // to that neighbour: wait until it finished the previous step
                    const int mask = rim_unit(d, 1 + st * TX, TX, ja, jb);
                    if (h.active && mask) {
                        halo_wait_once(h, mask, seen);
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                    }
                }
                for (int jj = ja - 1; stop ? jj == ja - 1 : jj <= jb + 1; ++jj, ++L) {
                    const uint32_t slot = L % NS;
                    if (L >= (uint32_t)NS) mbar_wait(&empty[slot], ((L / NS) - 1) & 1);
                    slot_unit[slot] = stop ? -1 : unit;
                    if (stop) {
                        mbar_arrive(&full[slot]); // no bytes: tells the consumers to finish
                        break;
                    }
                    unsigned char* stg = smem + (size_t)slot * G.stage;
                    mbar_expect_tx(&full[slot], G.tx_bytes);
                    // KIJ sf/pb rows are i-contiguous: their (even) coordinate of i0 - 2
                    const int ic2 = KIJ ? ic - 1 : ic;
                    if (KIJ) tma_load_3d(stg, &tm_e, &full[slot], 0, ic, a.jrow0 + jj);
                    else tma_load_3d(stg, &tm_e, &full[slot], ic, a.jrow0 + jj, 0);
                    tma_load_2d(stg + G.e_bytes, &tm_sf, &full[slot], ic2, a.jrow0 + jj);
                    tma_load_2d(stg + G.e_bytes + G.r_bytes, &tm_pb, &full[slot], ic2,
                                a.jrow0 + jj);
                }
                if (stop) break;
            }
            // the last CTA to finish re-arms the scheduler for the next launch
            __threadfence();
            if (atomicAdd(&a.sched[1], 1) == (int)gridDim.x - 1) {
                a.sched[0] = 0;
                a.sched[1] = 0;
                __threadfence();
            }
        }
        return;
    }

    // ---------------- consumer warps ----------------
    // Thread -> (column c of the strip, k-group g).  A warp is 32 consecutive
    // columns at one k, so every smem access and every u store is a
    // contiguous 256-byte run; each thread walks its k-range with a
    // three-value register window (P(k-1), P(k), P(k+1)).
    constexpr int NKG = NCW * 32 / TX;
    const int c = threadIdx.x % TX, g = threadIdx.x / TX;
    const int nz = d.nz;
    const int kl = 1 + (g * nz) / NKG, kh = ((g + 1) * nz) / NKG;
    const int w = G.w, cc = c + 2; // sf/pb (and IJK slab) column of cell i0 + c
    const int eoff = KIJ ? (c + 1) * G.is : cc; // slab element of cell i0 + c at k = 1
    const double ri = d.ri, tv = d.tv, dv = d.dv, c5 = d.c5, c6 = d.c6;

    uint32_t L = 0; // load index of the first slab of the current unit
    for (;;) {
        {
            const uint32_t slot = L % NS;
            mbar_wait(&full[slot], (L / NS) & 1);
        }
        int unit = 0; // one reader per warp (see weather_wave.cuh)
        if (lane == 0) unit = slot_unit[L % NS];
        unit = __shfl_sync(0xffffffffu, unit, 0);
        if (unit < 0) break;
        const int ch = unit / a.nstrips, st = unit % a.nstrips;
        const int ja = ch * a.chunk + 1, jb = min(d.ny, ja + a.chunk - 1);
        const int i0 = 1 + st * TX;
        const bool active = c < min(TX, d.nx - i0 + 1) && kl <= kh;
        for (int j = ja; j <= jb; ++j) {
            const uint32_t l0 = L + (j - ja), l1 = l0 + 1, l2 = l0 + 2;
            if (j == ja) mbar_wait(&full[l1 % NS], (l1 / NS) & 1);
            mbar_wait(&full[l2 % NS], (l2 / NS) & 1);
            if (active) {
                const unsigned char* stm = smem + (size_t)(l0 % NS) * G.stage;
                const unsigned char* st0 = smem + (size_t)(l1 % NS) * G.stage;
                const unsigned char* stp = smem + (size_t)(l2 % NS) * G.stage;
                const double* em = reinterpret_cast<const double*>(stm) + eoff;
                const double* e0 = reinterpret_cast<const double*>(st0) + eoff;
                const double* ep = reinterpret_cast<const double*>(stp) + eoff;
                const double* Sm = reinterpret_cast<const double*>(stm + G.e_bytes) + cc;
                const double* S0 = reinterpret_cast<const double*>(st0 + G.e_bytes) + cc;
                const double* Sp = reinterpret_cast<const double*>(stp + G.e_bytes) + cc;
                const double* Bm = reinterpret_cast<const double*>(stm + G.e_bytes + G.r_bytes) + cc;
                const double* B0 = reinterpret_cast<const double*>(st0 + G.e_bytes + G.r_bytes) + cc;
                const double* Bp = reinterpret_cast<const double*>(stp + G.e_bytes + G.r_bytes) + cc;
                // IJK: straight to global, 256-byte coalesced per warp.  KIJ: into
                // the staged output row ([i][k], conflict free), bulk-stored below.
                double* up = KIJ ? reinterpret_cast<double*>(outbuf + (size_t)(j & 1) * G.out_bytes) +
                                       c * G.is + (kl - 1)
                                 : u + (long long)(i0 + c) * d.si + (long long)j * d.sj +
                                       (long long)(kl - 1) * d.sk;
                const ColumnRow r{em, e0, ep, Sm, S0, Sp, Bm, B0, Bp, up, KIJ ? 1 : d.sk,
                                  w, G.is, kl, kh, nz, ri, tv, dv, c5, c6, i0 + c, j};
                column_row<PHYS>(r);
            }
            if (KIJ) {
                // the row is staged: one thread stores it as ONE contiguous bulk
                // copy (columns i0 .. i0+width-1 of row j are adjacent in KIJ)
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                if (threadIdx.x == 0) bulk_wait_read_all(); // row j-1's store has left its buffer
                asm volatile("bar.sync 2, %0;" ::"r"(NCW * 32) : "memory");
                if (threadIdx.x == 0) {
                    const int width = min(TX, d.nx - i0 + 1);
                    bulk_store(u + (long long)i0 * d.si + (long long)j * d.sj,
                               outbuf + (size_t)(j & 1) * G.out_bytes,
                               (uint32_t)(width * G.is * 8));
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[l0 % NS]);
        }
        // the unit's last two slabs are no longer needed
        const uint32_t lend = L + (jb - ja + 1);
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&empty[lend % NS]);
            mbar_arrive(&empty[(lend + 1) % NS]);
        }
        L = lend + 2;
        // decomposed rim unit: its cells near a face go to the neighbours
        if (h.active && rim_unit(d, i0, TX, ja, jb)) {
            if (KIJ && threadIdx.x == 0) bulk_wait_all(); // staged rows are in global memory
            asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32) : "memory");
            push_box(h, d, u, i0, min(i0 + TX - 1, d.nx), ja, jb, threadIdx.x, NCW * 32);
        }
    }

    // Epilogue: this CTA's share of the ghost cells (regions 4 and 5 of the
    // reference, 0.3% of the cells at ASUCA size), straight from global.
    // Decomposed: after every neighbour's previous step (one poller per CTA).
    if (h.active) {
        if (threadIdx.x == 0) halo_wait(h, 0xF);
        asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32) : "memory");
    }
    {
        // j-ghost rows span every owned i (the corners take the i-ghost rule
        // inside cell_update); i-ghost columns span the inner rows [r0, r1]
        const Owned o = owned(d);
        const int gs = (a.gj_mask & 1) && d.own_s, gn = (a.gj_mask & 2) && d.own_n;
        const int ni = o.i1 - o.i0 + 1;
        const long long nrow = (long long)ni * d.nz;
        const long long njg = (long long)(gs + gn) * nrow;
        const int r0 = max(a.gi_lo, 1), r1 = min(a.gi_hi, d.ny);
        const int nr = max(0, r1 - r0 + 1);
        const long long ncol = (long long)nr * d.nz;
        const long long tid = (long long)blockIdx.x * (NCW * 32) + threadIdx.x;
        for (long long g = tid; g < a.ghost_cells; g += (long long)gridDim.x * (NCW * 32)) {
            int i, j, k;
            if (g < njg) {
                const long long which = g / nrow, rem = g % nrow;
                i = o.i0 + (int)(rem % ni);
                k = 1 + (int)(rem / ni);
                j = (which == 0 && gs) ? 0 : d.ny + 1;
            } else {
                const long long h = g - njg, which = h / ncol, rem = h % ncol;
                j = r0 + (int)(rem % nr);
                k = 1 + (int)(rem / nr);
                i = (which == 0 && d.own_w) ? 0 : d.nx + 1;
            }
            const double v = cell_update<PHYS>(e, sf, pb, d, i, j, k);
            u[i * d.si + j * d.sj + (long long)(k - 1) * d.sk] = v;
            halo_push(h, d, i, j, k, v);
        }
    }

    if (KIJ && threadIdx.x == 0) bulk_wait_all(); // staged rows have reached global memory
    // all consumer warps of this CTA are done: publish the step when last
    if (h.active) {
        asm volatile("bar.sync 1, %0;" ::"r"(NCW * 32) : "memory");
        if (threadIdx.x == 0) halo_signal(h);
    }
}

} // namespace hftw
