// weather_pair.cuh -- two timesteps per pass over HBM (temporal blocking).
//
// Reference hot path: hft::reference_step (weather.cpp:101-171) applied twice.
// One launch reads the field e_s once and writes e_{s+2} once: the
// intermediate field e_{s+1} lives only in shared memory and registers, so a
// pass moves 16 B per stored cell for TWO steps (8 B per cell-step) against
// the single-step kernel's 16 B per cell-step.  Every cell of e_{s+1} and
// e_{s+2} is computed with exactly the operations of the single-step kernel
// (explicitly rounded IEEE ops, the reference's association order), so the
// result is bitwise identical to two reference steps.
//
// Tiling (IJK store, one persistent CTA per SM, dynamic j-major work units of
// 64-column strips x `chunk` rows, as in step_tma_kernel):
//   * the producer warp streams, per row j, one TMA slab of e_s covering
//     columns i0-2 .. i0+65 and all k, the sf/pb rows, and -- for the edge
//     strips -- the 2-wide column holding the cyclic partner of the i-ghost
//     cell (column nx for strip 0, column 1 for the last strip);
//   * row j' of the intermediate P' = physics(e_{s+1}) is computed for columns
//     i0-1 .. i0+64 from slabs j'-1, j', j'+1 (16 main warps own i0 .. i0+63,
//     one halo warp the two halo columns) into a shared row buffer, and each
//     main thread keeps its column's last three intermediate rows in
//     registers (a j window);
//   * row j = j'-1 of e_{s+2} is then computed from the row buffer (i and k
//     neighbours) and the register window (j neighbours) and stored with
//     256-byte coalesced stores.
// Ghost cells of e_{s+2} need intermediates from the opposite edge of the
// domain (the reference's cyclic rules, weather.cpp:152-168).  Units on the
// domain rim publish their ghost-adjacent intermediates (columns 0, 1, nx,
// nx+1 and rows 0, 1, ny, ny+1) to small global buffers, and the second of the
// two units that produce them (strip 0 / last strip of a chunk, chunk 0 / last
// chunk of a strip) computes those ghost cells -- no grid-wide barrier.
#pragma once

#include "weather_kernels.cuh"

namespace hftw {

constexpr int kPairTX = 64;                          // strip width (cells)
constexpr int kPairKG = 15;                          // k-groups of the main threads
constexpr int kPairMain = kPairTX * kPairKG;         // 960 main threads (30 warps)
constexpr int kPairConsumers = kPairMain + 32;       // + the halo warp
constexpr int kPairThreads = kPairConsumers + 32;    // + the producer warp
constexpr int kPairIBW = kPairTX + 2;                // intermediate row: columns i0-1 .. i0+64
constexpr int kPairW = kPairTX + 4;                  // slab row: columns i0-2 .. i0+65

__host__ __device__ inline int round128(int b) { return (b + 127) / 128 * 128; }

// Shared-memory geometry of the pair kernel (bytes).  Every TMA destination
// is 128-byte aligned.
struct PairGeom {
    int slab;   // e slab: [k][W] doubles
    int sfpb;   // sf and pb rows: [2][W] doubles
    int fcol;   // far column: [k][2] doubles
    int fsp;    // far sf / pb pairs: [2][2] doubles
    int stage;
    int ib;     // one intermediate row buffer: [k][IBW] doubles
    int tx_main, tx_far; // bytes the TMA delivers per stage (without / with the far column)
};
__host__ __device__ inline PairGeom pair_geom(int nz) {
    PairGeom g;
    g.slab = round128(kPairW * nz * 8);
    g.sfpb = round128(2 * kPairW * 8);
    g.fcol = round128(2 * nz * 8);
    g.fsp = 128;
    g.stage = g.slab + g.sfpb + g.fcol + g.fsp;
    g.ib = round128(kPairIBW * nz * 8);
    g.tx_main = kPairW * nz * 8 + 2 * kPairW * 8;
    g.tx_far = g.tx_main + 2 * nz * 8 + 4 * 8;
    return g;
}
__host__ __device__ inline size_t pair_smem_bytes(int nz, int ns) {
    const PairGeom g = pair_geom(nz);
    return (size_t)ns * g.stage + 2 * (size_t)g.ib + 2 * ns * sizeof(uint64_t) + ns * sizeof(int);
}

struct PairArgs {
    int fp;       // tensor-map i coordinate of logical i = 0
    int jrow0;    // tensor-map row coordinate of logical j = 0
    int nstrips, nchunks, chunk, ns;
    int* sched;   // [0] next unit, [1] CTAs finished (self-resetting)
    int* cnt_col; // [nchunks] i-ghost producers done (strip 0 + last strip), self-resetting
    int* cnt_row; // [nstrips] j-ghost producers done (chunk 0 + last chunk), self-resetting
    double* gcol; // P' at i = 0, 1, nx, nx+1: [4][ny+2][nz]
    double* grow; // P' at j = 0, 1, ny, ny+1: [4][nz][nx+2]
};

// Which cyclic partner column a unit's far TMA column holds (0 = none).
__host__ __device__ inline int pair_far_col(int st, int nstrips, int nx) {
    const int i0 = 1 + st * kPairTX;
    if (st == 0 && nx > i0 + kPairTX + 1) return nx;         // i-ghost 0 needs column nx
    if (st == nstrips - 1 && st > 0 && i0 - 2 > 1) return 1; // i-ghost nx+1 needs column 1
    return 0;
}

__device__ __forceinline__ void named_bar(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Post-physics value of one pre-step element (weather.cpp:122-127).
__device__ __forceinline__ double Pfull(double ev, int k, int nz, double sfv, double pbv,
                                        double ri, double tv) {
    return phys<true>(ev, k, nz, sfv, pbv, ri, tv);
}

// One thread's view of the three slab rows of an intermediate row (at the
// thread's slab column): e rows j'-1, j', j'+1 and their sf / pb rows.
struct IRow {
    const double *em, *e0, *ep;
    const double *Sm, *S0, *Sp; // sf rows (pb rows are kPairW doubles further)
};

// Intermediate P' = physics(u') of an INNER cell column (1 <= gi <= nx,
// 1 <= j' <= ny) for k = kl .. kl+nk-1 (KP >= nk; extra iterations recompute
// the last k and are not stored).  FAST: the k window never touches k = 1 or
// nz, so no physics correction and no k-plane formula can apply
// (weather.cpp:122-127, :134-137 only).
template <int KP, bool FAST>
__device__ __forceinline__ void inter_inner(const IRow& r, double* out, double* ib, int kl, int nk,
                                            const Dom& d) {
    constexpr int W = kPairW;
    const double ri = d.ri, dv = d.dv;
    if (FAST) {
        // nk == KP and 3 <= k-1, k+1 <= nz-1: every offset is a compile-time constant
        const double* p0 = r.e0 + (kl - 1) * W;
        const double* pm = r.em + (kl - 1) * W;
        const double* pp = r.ep + (kl - 1) * W;
        double* q = ib + (kl - 1) * kPairIBW;
        const double c6 = d.c6;
        double pd = dadd(p0[-W], ri), pc = dadd(p0[0], ri);
#pragma unroll
        for (int kk = 0; kk < KP; ++kk) {
            const double pn = dadd(p0[(kk + 1) * W], ri);
            double s = dadd(dadd(p0[kk * W - 1], ri), dadd(p0[kk * W + 1], ri));
            s = dadd(s, dadd(pm[kk * W], ri));
            s = dadd(s, dadd(pp[kk * W], ri));
            const double u = dadd(dmul(c6, pc), dmul(dv, dadd(dadd(s, pd), pn)));
            const double v = dadd(u, ri);
            out[kk] = v;
            q[kk * kPairIBW] = v;
            pd = pc;
            pc = pn;
        }
        return;
    }
    const int nz = d.nz, kh = kl + nk - 1;
    const double tv = d.tv;
    const double* Bm = r.Sm + W;
    const double* B0 = r.S0 + W;
    const double* Bp = r.Sp + W;
    auto Pc = [&](int k) { return Pfull(r.e0[(k - 1) * W], k, nz, r.S0[0], B0[0], ri, tv); };
    double pd = kl > 1 ? Pc(kl - 1) : 0.0;
    double pc = Pc(kl);
#pragma unroll
    for (int kk = 0; kk < KP; ++kk) {
        const int k = min(kl + kk, kh);
        const int o = (k - 1) * W;
        const double pn = k < nz ? Pc(k + 1) : 0.0;
        double s = dadd(Pfull(r.e0[o - 1], k, nz, r.S0[-1], B0[-1], ri, tv),
                        Pfull(r.e0[o + 1], k, nz, r.S0[1], B0[1], ri, tv));
        s = dadd(s, Pfull(r.em[o], k, nz, r.Sm[0], Bm[0], ri, tv));
        s = dadd(s, Pfull(r.ep[o], k, nz, r.Sp[0], Bp[0], ri, tv));
        double u;
        if (k == 1) u = dadd(dmul(d.c5, pc), dmul(dv, dadd(s, pn)));
        else if (k == nz) u = dadd(dmul(d.c5, pc), dmul(dv, dadd(s, pd)));
        else u = dadd(dmul(d.c6, pc), dmul(dv, dadd(dadd(s, pd), pn)));
        const double v = Pfull(u, k, nz, r.S0[0], B0[0], ri, tv);
        out[kk] = v;
        if (kk < nk) ib[(k - 1) * kPairIBW] = v;
        pd = pc;
        pc = pn;
    }
}

// Intermediate of a GHOST cell column (gi in {0, nx+1} or j' in {0, ny+1}),
// in the reference's precedence (i ghosts first, weather.cpp:161-168, then j
// ghosts, :152-159).  The cyclic partner comes from the slab, the far column
// (fcol/fsf/fpb, element fsel) or -- for j ghosts -- global memory.
template <int KP>
__device__ __forceinline__ void inter_ghost(const IRow& r, double* out, double* ib, int kl, int nk,
                                            int gi, int jr, int cc, int i0, const Dom& d,
                                            const double* __restrict__ e,
                                            const double* __restrict__ sf,
                                            const double* __restrict__ pb, const double* fcol,
                                            const double* fsp, int fsel) {
    constexpr int W = kPairW;
    const int nz = d.nz, nx = d.nx, ny = d.ny, kh = kl + nk - 1;
    const double ri = d.ri, tv = d.tv, dv = d.dv;
    const double* B0 = r.S0 + W;
    const double* e0b = r.e0 - cc; // slab row j' at slab column 0
    const double* s0b = r.S0 - cc;
    const double* b0b = B0 - cc;
    const bool ig = gi == 0 || gi == nx + 1;
    const int c1 = 1 - (i0 - 2), cn = nx - (i0 - 2); // slab columns of i = 1 and i = nx
    const bool in1 = c1 >= 0 && c1 < W, inn = cn >= 0 && cn < W;
    const int jf = jr == 0 ? ny : 1; // j ghosts: the partner row read from global memory
    const double* ef = e + gi * d.si + jf * d.sj;
    double sff = 0.0, pbf = 0.0;
    if (!ig) {
        sff = __ldg(sf + gi + jf * d.s2j);
        pbf = __ldg(pb + gi + jf * d.s2j);
    }
#pragma unroll
    for (int kk = 0; kk < KP; ++kk) {
        const int k = min(kl + kk, kh);
        const int o = (k - 1) * W;
        const double pg = Pfull(r.e0[o], k, nz, r.S0[0], B0[0], ri, tv);
        double a, b;
        if (ig) {
            const double pf = Pfull(fcol[(k - 1) * 2 + fsel], k, nz, fsp[fsel], fsp[2 + fsel], ri, tv);
            a = in1 ? Pfull(e0b[o + c1], k, nz, s0b[c1], b0b[c1], ri, tv) : pf; // P(1)
            b = inn ? Pfull(e0b[o + cn], k, nz, s0b[cn], b0b[cn], ri, tv) : pf; // P(nx)
        } else {
            const double pf = Pfull(__ldg(ef + (long long)(k - 1) * d.sk), k, nz, sff, pbf, ri, tv);
            // jr = 0: P(ny) far, P(1) = row j'+1; jr = ny+1: P(ny) = row j'-1, P(1) far
            a = jr == 0 ? pf : Pfull(r.em[o], k, nz, r.Sm[0], r.Sm[W], ri, tv);
            b = jr == 0 ? Pfull(r.ep[o], k, nz, r.Sp[0], r.Sp[W], ri, tv) : pf;
        }
        const double u = dadd(dmul(d.c2, pg), dmul(dv, dadd(a, b)));
        const double v = Pfull(u, k, nz, r.S0[0], B0[0], ri, tv);
        out[kk] = v;
        if (kk < nk) ib[(k - 1) * kPairIBW] = v;
    }
}

// Row j of e_{s+2} for one inner column: i and k neighbours from the row
// buffer B (row j), j neighbours and the centre from the register window
// (P0 = row j-1, P1 = row j, P2 = row j+1).  weather.cpp:130-150 on P'.
template <int KP, bool FAST>
__device__ __forceinline__ void final_row(const double* P0, const double* P1, const double* P2,
                                          const double* B, double* q, long long sk, int kl, int nk,
                                          const Dom& d) {
    const double dv = d.dv;
    if (FAST) {
        const double* Bk = B + (kl - 1) * kPairIBW;
        const double c6 = d.c6;
#pragma unroll
        for (int kk = 0; kk < KP; ++kk) {
            double s = dadd(Bk[kk * kPairIBW - 1], Bk[kk * kPairIBW + 1]);
            s = dadd(s, P0[kk]);
            s = dadd(s, P2[kk]);
            const double km = kk > 0 ? P1[kk - 1] : Bk[-kPairIBW];
            const double kp = kk + 1 < KP ? P1[kk + 1] : Bk[KP * kPairIBW];
            *q = dadd(dmul(c6, P1[kk]), dmul(dv, dadd(dadd(s, km), kp)));
            q += sk;
        }
        return;
    }
    const int nz = d.nz, kh = kl + nk - 1;
#pragma unroll
    for (int kk = 0; kk < KP; ++kk) {
        const int k = min(kl + kk, kh);
        const int o = (k - 1) * kPairIBW;
        double s = dadd(B[o - 1], B[o + 1]);
        s = dadd(s, P0[kk]);
        s = dadd(s, P2[kk]);
        // (clamped reads: the k = 1 / nz cells do not use the missing neighbour)
        const double km = kk > 0 ? P1[kk - 1] : B[max(o - kPairIBW, 0)];
        const double kp = kk + 1 < nk ? P1[kk + 1] : B[min(o + kPairIBW, (nz - 1) * kPairIBW)];
        double v;
        if (k == 1) v = dadd(dmul(d.c5, P1[kk]), dmul(dv, dadd(s, kp)));
        else if (k == nz) v = dadd(dmul(d.c5, P1[kk]), dmul(dv, dadd(s, km)));
        else v = dadd(dmul(d.c6, P1[kk]), dmul(dv, dadd(dadd(s, km), kp)));
        if (kk < nk) q[(long long)kk * sk] = v;
    }
}

// Publish the ghost-adjacent intermediates a unit owns (see PairArgs).
template <int KP>
__device__ __forceinline__ void pair_publish(const double* v, int kl, int nk, int gi, int jr,
                                             const Dom& d, const PairArgs& a) {
    const int nx = d.nx, ny = d.ny, nz = d.nz;
    const int wc = gi == 0 ? 0 : gi == 1 ? 1 : gi == nx ? 2 : gi == nx + 1 ? 3 : -1;
    const int wr = (gi >= 1 && gi <= nx)
                       ? (jr == 0 ? 0 : jr == 1 ? 1 : jr == ny ? 2 : jr == ny + 1 ? 3 : -1)
                       : -1;
    if (wc < 0 && wr < 0) return;
#pragma unroll
    for (int kk = 0; kk < KP; ++kk) {
        if (kk >= nk) break;
        const int k = kl + kk;
        if (wc >= 0) a.gcol[((long long)wc * (ny + 2) + jr) * nz + (k - 1)] = v[kk];
        if (wr >= 0) a.grow[((long long)wr * nz + (k - 1)) * (nx + 2) + gi] = v[kk];
    }
}

// The second producer of a chunk's i-ghost intermediates computes that
// chunk's i-ghost cells of e_{s+2} (rows ja..jb, plus 0 / ny+1 at the domain
// ends): weather.cpp:164-167 on the intermediate field.
__device__ __forceinline__ void pair_ghost_cols(const Dom& d, const PairArgs& a,
                                                double* __restrict__ u, int ja, int jb, int tid) {
    const int nx = d.nx, ny = d.ny, nz = d.nz;
    const int r0 = ja == 1 ? 0 : ja, r1 = jb == ny ? ny + 1 : jb;
    const int nr = r1 - r0 + 1;
    const long long n = 2LL * nr * nz;
    auto G = [&](int w, int j, int k) {
        return __ldcg(a.gcol + ((long long)w * (ny + 2) + j) * nz + (k - 1));
    };
    for (long long t = tid; t < n; t += kPairConsumers) {
        const int k = 1 + (int)(t % nz);
        const long long q = t / nz;
        const int j = r0 + (int)(q % nr);
        const int side = (int)(q / nr); // 0: i = 0, 1: i = nx+1
        const double pg = G(side == 0 ? 0 : 3, j, k);
        const double v = dadd(dmul(d.c2, pg), dmul(d.dv, dadd(G(1, j, k), G(2, j, k))));
        u[(side == 0 ? 0 : nx + 1) * d.si + j * d.sj + (long long)(k - 1) * d.sk] = v;
    }
}

// The second producer of a strip's j-ghost intermediates computes that
// strip's j-ghost cells (i in i0..i0+63 clipped to 1..nx, j = 0 and ny+1):
// weather.cpp:155-158 on the intermediate field.
__device__ __forceinline__ void pair_ghost_rows(const Dom& d, const PairArgs& a,
                                                double* __restrict__ u, int i0, int tid) {
    const int nx = d.nx, ny = d.ny, nz = d.nz;
    const int ni = min(kPairTX, nx - i0 + 1);
    const long long n = 2LL * ni * nz;
    auto G = [&](int w, int i, int k) {
        return __ldcg(a.grow + ((long long)w * nz + (k - 1)) * (nx + 2) + i);
    };
    for (long long t = tid; t < n; t += kPairConsumers) {
        const int i = i0 + (int)(t % ni);
        const long long q = t / ni;
        const int k = 1 + (int)(q % nz);
        const int side = (int)(q / nz); // 0: j = 0, 1: j = ny+1
        const double pg = G(side == 0 ? 0 : 3, i, k);
        const double v = dadd(dmul(d.c2, pg), dmul(d.dv, dadd(G(2, i, k), G(1, i, k))));
        u[i * d.si + (side == 0 ? 0 : ny + 1) * d.sj + (long long)(k - 1) * d.sk] = v;
    }
}

// KPT: k values per thread; nz <= 15*KPT (main threads; the halo warp has 16 groups).
template <int KPT>
__global__ void __launch_bounds__(kPairThreads, 1)
    step_pair_kernel(const __grid_constant__ CUtensorMap tm_e,
                     const __grid_constant__ CUtensorMap tm_sfpb,
                     const __grid_constant__ CUtensorMap tm_ef,
                     const __grid_constant__ CUtensorMap tm_sfpbf, const double* __restrict__ e,
                     double* __restrict__ u, const double* __restrict__ sf,
                     const double* __restrict__ pb, Dom d, PairArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const PairGeom G = pair_geom(d.nz);
    const int NS = a.ns;
    // intermediate row buffer of row j: ib0 + (j & 1) * ibn
    double* const ib0 = reinterpret_cast<double*>(smem + (size_t)NS * G.stage);
    const int ibn = G.ib / 8;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NS * G.stage + 2 * (size_t)G.ib);
    uint64_t* empty = full + NS;
    int* slot_unit = reinterpret_cast<int*>(empty + NS);
    __shared__ int s_flags;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int units = a.nstrips * a.nchunks;
    const int nx = d.nx, ny = d.ny, nz = d.nz;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kPairConsumers / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (threadIdx.x >= kPairConsumers) {
        // ---------------- producer warp ----------------
        if (lane == 0) {
            uint32_t L = 0;
            for (;;) {
                const int unit = atomicAdd(&a.sched[0], 1);
                const bool stop = unit >= units;
                int ja = 0, jb = -1, ic = 0, fx = 0, far = 0;
                if (!stop) {
                    const int ch = unit / a.nstrips, st = unit % a.nstrips;
                    ja = ch * a.chunk + 1;
                    jb = min(ny, ja + a.chunk - 1);
                    ic = a.fp + 1 + st * kPairTX - 2; // tensor i of i0 - 2 (even)
                    far = pair_far_col(st, a.nstrips, nx);
                    fx = (a.fp + far) & ~1;           // even-aligned pair holding it
                }
                // rows ja-2 .. jb+2 (the slabs of intermediate rows ja-1 .. jb+1)
                for (int jj = ja - 2; stop ? jj == ja - 2 : jj <= jb + 2; ++jj, ++L) {
                    const uint32_t slot = L % NS;
                    if (L >= (uint32_t)NS) mbar_wait(&empty[slot], ((L / NS) - 1) & 1);
                    slot_unit[slot] = stop ? -1 : unit;
                    if (stop) {
                        mbar_arrive(&full[slot]);
                        break;
                    }
                    unsigned char* stg = smem + (size_t)slot * G.stage;
                    mbar_expect_tx(&full[slot], far ? G.tx_far : G.tx_main);
                    tma_load_3d(stg, &tm_e, &full[slot], ic, a.jrow0 + jj, 0);
                    tma_load_3d(stg + G.slab, &tm_sfpb, &full[slot], ic, a.jrow0 + jj, 0);
                    if (far) {
                        unsigned char* f = stg + G.slab + G.sfpb;
                        tma_load_3d(f, &tm_ef, &full[slot], fx, a.jrow0 + jj, 0);
                        tma_load_3d(f + G.fcol, &tm_sfpbf, &full[slot], fx, a.jrow0 + jj, 0);
                    }
                }
                if (stop) break;
            }
            __threadfence();
            if (atomicAdd(&a.sched[1], 1) == (int)gridDim.x - 1) {
                a.sched[0] = 0;
                a.sched[1] = 0;
                __threadfence();
            }
        }
        return;
    }

    // ---------------- consumers: 30 main warps + 1 halo warp ----------------
    const int tid = threadIdx.x;
    const bool halo = tid >= kPairMain;
    // main: column c = tid % 64 (slab column c+2), k-group tid / 64 (of 15)
    // halo: lanes 0-15 column i0-1 (slab 1), lanes 16-31 column i0+64 (slab 66), 16 k-groups
    const int cc = halo ? (lane < 16 ? 1 : kPairTX + 2) : (tid % kPairTX) + 2;
    const int g = halo ? (lane & 15) : tid / kPairTX;
    // k-groups of KPT consecutive planes (the last non-empty one may be short)
    const int kl = 1 + g * KPT, kh = min(nz, kl + KPT - 1);
    const int nk = max(0, kh - kl + 1);
    const bool fast = nk == KPT && kl >= 3 && kh <= nz - 2;

    double PW0[KPT], PW1[KPT], PW2[KPT];
    uint32_t L = 0;
    for (;;) {
        mbar_wait(&full[L % NS], (L / NS) & 1);
        const int unit = slot_unit[L % NS];
        if (unit < 0) break;
        const int ch = unit / a.nstrips, st = unit % a.nstrips;
        const int ja = ch * a.chunk + 1, jb = min(ny, ja + a.chunk - 1);
        const int i0 = 1 + st * kPairTX;
        const int gi = i0 - 2 + cc; // logical i of my column
        const bool indom = gi <= nx + 1 && nk > 0;
        const bool owns_i = (gi >= i0 && gi <= min(i0 + kPairTX - 1, nx + 1)) ||
                            (st == 0 && gi == 0) || (st == a.nstrips - 1 && gi == nx + 1);
        const bool ig = gi == 0 || gi == nx + 1;
        const int fsel = (a.fp + pair_far_col(st, a.nstrips, nx)) & 1;
        const int c = cc - 2;
        const bool do_final = !halo && i0 + c <= nx && nk > 0;
        for (int jr = ja - 1; jr <= jb + 1; ++jr) {
            // slabs jr-1, jr, jr+1 have load indices L + (jr - ja) + {1, 2, 3}
            const uint32_t l0 = L + (uint32_t)(jr - ja + 1), l1 = l0 + 1, l2 = l0 + 2;
            if (jr == ja - 1) mbar_wait(&full[l1 % NS], (l1 / NS) & 1);
            mbar_wait(&full[l2 % NS], (l2 / NS) & 1);
            double* ibrow = ib0 + (jr & 1) * ibn + (cc - 1);
            if (indom) {
                const unsigned char* sm_ = smem + (size_t)(l0 % NS) * G.stage;
                const unsigned char* s0_ = smem + (size_t)(l1 % NS) * G.stage;
                const unsigned char* sp_ = smem + (size_t)(l2 % NS) * G.stage;
                const IRow r{reinterpret_cast<const double*>(sm_) + cc,
                             reinterpret_cast<const double*>(s0_) + cc,
                             reinterpret_cast<const double*>(sp_) + cc,
                             reinterpret_cast<const double*>(sm_ + G.slab) + cc,
                             reinterpret_cast<const double*>(s0_ + G.slab) + cc,
                             reinterpret_cast<const double*>(sp_ + G.slab) + cc};
                const bool owns_j = (jr >= ja && jr <= jb) || jr == 0 || jr == ny + 1;
                if (ig || jr == 0 || jr == ny + 1) {
                    const double* fb = reinterpret_cast<const double*>(s0_ + G.slab + G.sfpb);
                    const double* fsp = reinterpret_cast<const double*>(s0_ + G.slab + G.sfpb + G.fcol);
                    inter_ghost<KPT>(r, PW2, ibrow, kl, nk, gi, jr, cc, i0, d, e, sf, pb, fb, fsp,
                                     fsel);
                } else if (fast) {
                    inter_inner<KPT, true>(r, PW2, ibrow, kl, nk, d);
                } else {
                    inter_inner<KPT, false>(r, PW2, ibrow, kl, nk, d);
                }
                if (owns_i && owns_j) pair_publish<KPT>(PW2, kl, nk, gi, jr, d, a);
            }
            // slab jr-1 is no longer needed
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[l0 % NS]);
            if (do_final && jr >= ja + 1) {
                const int j = jr - 1;
                const double* B = ib0 + (j & 1) * ibn + (cc - 1);
                double* q = u + (long long)(i0 + c) * d.si + (long long)j * d.sj +
                            (long long)(kl - 1) * d.sk;
                if (fast) final_row<KPT, true>(PW0, PW1, PW2, B, q, d.sk, kl, nk, d);
                else final_row<KPT, false>(PW0, PW1, PW2, B, q, d.sk, kl, nk, d);
            }
#pragma unroll
            for (int kk = 0; kk < KPT; ++kk) {
                PW0[kk] = PW1[kk];
                PW1[kk] = PW2[kk];
            }
            named_bar(1, kPairConsumers);
        }
        // the unit's last two slabs (rows jb+1, jb+2)
        {
            const uint32_t lend = L + (uint32_t)(jb - ja + 3);
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&empty[lend % NS]);
                mbar_arrive(&empty[(lend + 1) % NS]);
            }
            L = lend + 2;
        }
        // rim units: count the ghost producers; the second one computes the ghosts
        const int inc_c = (st == 0) + (st == a.nstrips - 1);
        const int inc_r = (ch == 0) + (ch == a.nchunks - 1);
        if (inc_c | inc_r) {
            if (tid == 0) {
                __threadfence();
                int f = 0;
                if (inc_c && atomicAdd(&a.cnt_col[ch], inc_c) + inc_c == 2) {
                    f |= 1;
                    a.cnt_col[ch] = 0;
                }
                if (inc_r && atomicAdd(&a.cnt_row[st], inc_r) + inc_r == 2) {
                    f |= 2;
                    a.cnt_row[st] = 0;
                }
                __threadfence();
                s_flags = f;
            }
            named_bar(1, kPairConsumers);
            const int f = s_flags;
            if (f & 1) pair_ghost_cols(d, a, u, ja, jb, tid);
            if (f & 2) pair_ghost_rows(d, a, u, i0, tid);
            named_bar(1, kPairConsumers); // s_flags is reused by the next rim unit
        }
    }
}

} // namespace hftw
