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
// Tiling (IJK store, two persistent 256-thread CTAs per SM, dynamic j-major
// work units of 30-column strips x 24 rows at ASUCA size, the last ~1.5 waves of
// units half as tall; 12 / 8-row units on small decomposed domains):
//   * per row j, ONE TMA box of e_s covers columns i0-2 .. i0+31 and all k,
//     one box the sf and pb rows, and -- for the two edge strips -- a 2-wide
//     box holds the cyclic partner column of the i-ghost cell (column nx for
//     strip 0, column 1 for the last strip).  Thread 0 refills the ring slot
//     a row frees right after the row's barrier (no producer warp);
//   * row jr of the intermediate P' = physics(e_{s+1}) is computed for the 32
//     columns i0-1 .. i0+30 from slabs jr-1, jr, jr+1: 8 k-groups of 7-8
//     planes x 32 columns = 8 warps, each thread walking its planes with a
//     register window (k).  P' goes to one of three shared row buffers;
//   * after a barrier, row j = jr-1 of e_{s+2} is computed for the 30 columns
//     i0 .. i0+29: the i and j-1 neighbours from the row buffers, the centre,
//     its k neighbours and the j+1 neighbour from this thread's registers --
//     and stored straight to HBM.  One CTA barrier per row: the buffer the
//     next row overwrites is read in this final row only by its own thread.
//   * the edge planes k = 1 and nz (physics corrections, k-plane formulas)
//     are peeled at compile time per k-group "shape", so the common planes
//     run without them.
// Ghost cells of e_{s+2} need intermediates from the opposite edge of the
// domain (the reference's cyclic rules, weather.cpp:152-168).  Units on the
// domain rim publish their ghost-adjacent intermediates (columns 0, 1, nx,
// nx+1 and rows 0, 1, ny, ny+1) to small global buffers, and the second of the
// two units that produce them (strip 0 / last strip of a chunk, chunk 0 / last
// chunk of a strip) computes those ghost cells -- no grid-wide barrier.
//
// Decomposed rank (PairArgs::dist): the same kernel on the
// rank's subdomain.  A non-owned side's row / column 0 and n+1 are halo cells
// computed with the inner rule from 2-deep halos (the neighbours pushed them,
// weather_kernels.cuh); the cyclic partner of an owned ghost intermediate is
// the far slot (wfar / efar / sfar / nfar) the wrap partner fills.  Units on the
// rim wait for every neighbour's previous pass and push their cells near a
// face into the neighbours.  Ghost FINALS need the wrap partner's
// intermediates, so they move to pair_ghost_kernel: this kernel publishes the
// ghost-adjacent intermediates and releases a "published" flag in the wrap
// partners; the ghost kernel waits for theirs, finishes the ghost cells, pushes
// them and releases the pass to all neighbours.
#pragma once

#include "weather_kernels.cuh"

namespace hftw {

#ifndef HFTW_PAIR_TX
#define HFTW_PAIR_TX 30
#endif
constexpr int kPairTX = HFTW_PAIR_TX;           // output columns per strip (30: 2 CTAs per SM)
constexpr int kPairIC = kPairTX + 2;            // intermediate columns i0-1 .. i0+TX (warps)
constexpr int kPairW = kPairTX + 4;             // slab columns i0-2 .. i0+TX+1
#ifndef HFTW_PAIR_KG
#define HFTW_PAIR_KG 8
#endif
// k-groups (warps) per strip: 8 (<= 8 planes each, 256 threads, 124 registers).  10
// groups (<= 6 planes, 320 threads, 95 registers) are 3% faster on a lone 790 x 325
// subdomain but 0.6% slower at ASUCA size and 1.5% slower on decomposed weak-scaled
// ranks; 9 / 11 / 12 / 14 are slower still
constexpr int kPairKG = HFTW_PAIR_KG;
constexpr int kPairThreads = kPairIC * kPairKG;
#ifndef HFTW_PAIR_MINB
#define HFTW_PAIR_MINB (kPairThreads <= 320 ? 2 : 1)
#endif
constexpr int kPairMinBlocks = HFTW_PAIR_MINB; // CTAs per SM the tile allows
// intermediate row buffers (rows j-1, j, j+1), one CTA barrier per row
constexpr int kPairNIB = 3;

__host__ __device__ inline int round128(int b) { return (b + 127) / 128 * 128; }

// Shared-memory geometry of the pair kernel (bytes).  Every TMA destination
// is 128-byte aligned.
struct PairGeom {
    int slab;   // e slab: [k][W] doubles
    int sfpb;   // sf and pb rows: [2][W] doubles
    int fcol;   // far column: [k][2] doubles
    int fsp;    // far sf / pb pairs: [2][2] doubles
    int stage;
    int ib;     // one intermediate row buffer: [k][IC] doubles
    int tx_main, tx_far; // bytes the TMA delivers per stage (without / with the far column)
};
__host__ __device__ inline PairGeom pair_geom(int nz) {
    PairGeom g;
    g.slab = round128(kPairW * nz * 8);
    g.sfpb = round128(2 * kPairW * 8);
    g.fcol = round128(2 * nz * 8);
    g.fsp = 128;
    g.stage = g.slab + g.sfpb + g.fcol + g.fsp;
    g.ib = round128(kPairIC * nz * 8);
    g.tx_main = kPairW * nz * 8 + 2 * kPairW * 8;
    g.tx_far = g.tx_main + 2 * nz * 8 + 4 * 8;
    return g;
}
__host__ __device__ inline size_t pair_smem_bytes(int nz, int ns) {
    const PairGeom g = pair_geom(nz);
    return (size_t)ns * g.stage + kPairNIB * (size_t)g.ib + ns * sizeof(uint64_t) + ns * sizeof(int);
}

struct PairArgs {
    int fp;       // tensor-map i coordinate of logical i = 0
    int jrow0;    // tensor-map row coordinate of logical j = 0
    int nstrips, nchunks, chunk, ns;
    int nbig;     // chunks 0 .. nbig-1 have `chunk` rows, the rest `chunk2` (the last
    int chunk2;   // ~1.5 waves of units are shorter, so the launch's tail is shorter)
    int* sched;   // [0] next unit, [1] CTAs finished (self-resetting)
    int reverse;  // HFTW_OPT_REVERSE: hand the units out last first
    int* cnt_col; // [nchunks] i-ghost producers done (strip 0 + last strip), self-resetting
    int* cnt_row; // [nstrips] j-ghost producers done (chunk 0 + last chunk), self-resetting
    double* gcol; // P' at i = 0, 1, nx, nx+1: [4][ny+2][nz]
    double* grow; // P' at j = 0, 1, ny, ny+1: [4][nz][nx+2]
};

// Rows ja..jb of chunk ch.
__host__ __device__ inline void pair_rows(const PairArgs& a, int ny, int ch, int& ja, int& jb) {
    ja = ch < a.nbig ? ch * a.chunk + 1 : a.nbig * a.chunk + (ch - a.nbig) * a.chunk2 + 1;
    jb = ja + (ch < a.nbig ? a.chunk : a.chunk2) - 1;
    if (jb > ny) jb = ny;
}

// Which cyclic partner column a unit's far TMA box holds (0 = none): the
// partner of an owned i-ghost (wfar for i = 0, efar for i = nx+1) when it lies
// outside the unit's slab (i0-2 .. i0+TX+1).  Decomposed along i, the partner
// is the far halo slot -1 / nx+2, always inside the edge strip's slab.
__host__ __device__ inline bool pair_in_slab(int col, int i0) {
    return col >= i0 - 2 && col <= i0 + kPairTX + 1;
}
template <bool DIST>
__host__ __device__ inline int pair_far_col(int st, int nstrips, const Dom& d) {
    const int i0 = 1 + st * kPairTX;
    if (!DIST) { // one domain: wfar = nx, efar = 1
        if (st == 0 && d.nx > i0 + kPairTX + 1) return d.nx;
        if (st == nstrips - 1 && st > 0) return 1;
        return 0;
    }
    if (st == 0 && d.own_w && !pair_in_slab(d.wfar, i0)) return d.wfar;
    if (st == nstrips - 1 && d.own_e && !pair_in_slab(d.efar, i0)) return d.efar;
    return 0;
}

// Post-physics value of one pre-step element (weather.cpp:122-127).
__device__ __forceinline__ double Pfull(double ev, int k, int nz, double sfv, double pbv,
                                        double ri, double tv) {
    return phys<true>(ev, k, nz, sfv, pbv, ri, tv);
}

// One thread's view of the three slab rows of an intermediate row (at the
// thread's slab column): e rows jr-1, jr, jr+1 and their sf rows (the pb row
// is kPairW doubles after each sf row).
struct IRow {
    const double *em, *e0, *ep;
    const double *Sm, *S0, *Sp;
};

// Intermediate P' = physics(u') of an INNER cell column (1 <= gi <= nx,
// 1 <= jr <= ny) for the planes kl .. kl+NK-1.  FIRST: kl == 1 (the k = 1
// plane, weather.cpp:142-145, with the sf correction of :123-125), LAST: the
// last plane is nz (:146-149, pb correction :126-127); every other plane is
// the inner stencil (:130-137) with P = e + ri.  All branches are resolved at
// compile time and every offset is a constant.
// PIN: the slabs already hold post-physics values (the previous pass stored
// them, POUT), so the loads are used as they are.
template <int KP, int NK, bool FIRST, bool LAST, bool PIN>
__device__ __forceinline__ void inter_inner(const IRow& r, double* out, double* ib, int kl,
                                            const Dom& d) {
    constexpr int W = kPairW;
    const double ri = d.ri, tv = d.tv, dv = d.dv, c6 = d.c6, c5 = d.c5;
    const double* p0 = r.e0 + (kl - 1) * W;
    const double* pm = r.em + (kl - 1) * W;
    const double* pp = r.ep + (kl - 1) * W;
    double* q = ib + (kl - 1) * kPairIC; // ib: this row's buffer, never null here
    auto corr = [&](double x, double bnd) { return dsub(x, dmul(tv, dsub(x, bnd))); };
    // post-physics value of a loaded element: inner plane / plane 1 or nz
    auto Pi = [&](double x) { return PIN ? x : dadd(x, ri); };
    auto Pb = [&](double x, double bnd) { return PIN ? x : corr(dadd(x, ri), bnd); };
    const double* sfr = r.S0;     // sf row (pb is W further)
    // window: pd = P(k-1), pc = P(k).  The fast shapes are used only when every
    // group has >= 2 planes (nz >= 16), so the planes next to a group (kl-1,
    // kh+1) are never 1 or nz unless the group itself is FIRST / LAST.
    double pd = FIRST ? 0.0 : Pi(p0[-W]);
    double pc = FIRST ? Pb(p0[0], sfr[0]) : Pi(p0[0]);
#pragma unroll
    for (int kk = 0; kk < NK; ++kk) {
        const int o = kk * W;
        const bool top = FIRST && kk == 0;       // plane 1
        const bool bot = LAST && kk == NK - 1;   // plane nz
        double pn = 0.0;
        if (!bot) pn = LAST && kk == NK - 2 ? Pb(p0[o + W], sfr[W]) : Pi(p0[o + W]); // nz
        double v;
        if (top || bot) {
            const int bo = top ? 0 : W;
            double s = dadd(Pb(p0[o - 1], sfr[bo - 1]), Pb(p0[o + 1], sfr[bo + 1]));
            s = dadd(s, Pb(pm[o], r.Sm[bo]));
            s = dadd(s, Pb(pp[o], r.Sp[bo]));
            const double u = dadd(dmul(c5, pc), dmul(dv, dadd(s, top ? pn : pd)));
            v = corr(dadd(u, ri), sfr[bo]);
        } else {
            double s = dadd(Pi(p0[o - 1]), Pi(p0[o + 1]));
            s = dadd(s, Pi(pm[o]));
            s = dadd(s, Pi(pp[o]));
            const double u = dadd(dmul(c6, pc), dmul(dv, dadd(dadd(s, pd), pn)));
            v = dadd(u, ri);
        }
        out[kk] = v;
        pd = pc;
        pc = pn;
    }
    // row-buffer stores after the loop: a store inside it would keep the
    // compiler from hoisting the next plane's slab loads above it (possible
    // shared-memory aliasing), serialising the planes
#pragma unroll
    for (int kk = 0; kk < NK; ++kk) q[kk * kPairIC] = out[kk];
}

// Generic (any plane range, runtime nk <= KP): Pfull everywhere.  Used only
// for grids whose k-groups match no compile-time shape (small or odd nz).
template <int KP, bool PIN>
__device__ __forceinline__ void inter_generic(const IRow& r, double* out, double* ib, int kl,
                                              int nk, const Dom& d) {
    constexpr int W = kPairW;
    const int nz = d.nz;
    const double ri = d.ri, tv = d.tv, dv = d.dv;
    const double* B0 = r.S0 + W;
    auto Pl = [&](double x, int k, double sfv, double pbv) {
        return PIN ? x : Pfull(x, k, nz, sfv, pbv, ri, tv);
    };
    auto Pc = [&](int k) { return Pl(r.e0[(k - 1) * W], k, r.S0[0], B0[0]); };
    double pd = kl > 1 ? Pc(kl - 1) : 0.0;
    double pc = Pc(kl);
#pragma unroll
    for (int kk = 0; kk < KP; ++kk) {
        if (kk >= nk) break;
        const int k = kl + kk;
        const int o = (k - 1) * W;
        const double pn = k < nz ? Pc(k + 1) : 0.0;
        double s = dadd(Pl(r.e0[o - 1], k, r.S0[-1], B0[-1]), Pl(r.e0[o + 1], k, r.S0[1], B0[1]));
        s = dadd(s, Pl(r.em[o], k, r.Sm[0], r.Sm[W]));
        s = dadd(s, Pl(r.ep[o], k, r.Sp[0], r.Sp[W]));
        double u;
        if (k == 1) u = dadd(dmul(d.c5, pc), dmul(dv, dadd(s, pn)));
        else if (k == nz) u = dadd(dmul(d.c5, pc), dmul(dv, dadd(s, pd)));
        else u = dadd(dmul(d.c6, pc), dmul(dv, dadd(dadd(s, pd), pn)));
        const double v = Pfull(u, k, nz, r.S0[0], B0[0], ri, tv);
        out[kk] = v;
        ib[(k - 1) * kPairIC] = v;
        pd = pc;
        pc = pn;
    }
}

// Intermediate of a GHOST cell column (gi in {0, nx+1} or jr in {0, ny+1}),
// in the reference's precedence (i ghosts first, weather.cpp:161-168, then j
// ghosts, :152-159).  The cyclic partner comes from the slab, the far column
// (fcol/fsp, element fsel) or -- for j ghosts -- global memory.
template <int KP, bool DIST, bool PIN>
__device__ __forceinline__ void inter_ghost(const IRow& r, double* out, double* ib, int kl, int nk,
                                            int gi, int jr, int cc, int i0, const Dom& d,
                                         const double* __restrict__ e,
                                         const double* __restrict__ sf,
                                         const double* __restrict__ pb, const double* fcol,
                                         const double* fsp, int fsel) {
    constexpr int W = kPairW;
    const int nz = d.nz, nx = d.nx, ny = d.ny;
    const double ri = d.ri, tv = d.tv, dv = d.dv;
    const double* B0 = r.S0 + W;
    const double* e0b = r.e0 - cc; // slab row jr at slab column 0
    const double* s0b = r.S0 - cc;
    const double* b0b = B0 - cc;
    const bool ig = DIST ? (d.own_w && gi == 0) || (d.own_e && gi == nx + 1)
                         : gi == 0 || gi == nx + 1;
    // i ghosts: u = c2 P(gi) + dv (P(1) + P(nx)) with the partner (the far column
    // wfar / efar) in the slab or in the far box; weather.cpp:164-167
    const int ca = gi == 0 || !DIST ? 1 : d.efar, cb = gi == 0 && DIST ? d.wfar : nx;
    const int c1 = ca - (i0 - 2), cn = cb - (i0 - 2); // their slab columns
    const bool in1 = c1 >= 0 && c1 < W, inn = cn >= 0 && cn < W;
    // j ghosts: the partner row (far row sfar / nfar), from global memory (written
    // by the wrap partner when decomposed: coherent loads)
    const int jf = DIST ? (jr == 0 ? d.sfar : d.nfar) : (jr == 0 ? ny : 1);
    const double* ef = e + gi * d.si + jf * d.sj;
    double sff = 0.0, pbf = 0.0;
    if (!ig) {
        sff = DIST ? __ldcg(sf + gi + jf * d.s2j) : __ldg(sf + gi + jf * d.s2j);
        pbf = DIST ? __ldcg(pb + gi + jf * d.s2j) : __ldg(pb + gi + jf * d.s2j);
    }
    auto Pl = [&](double x, int k, double sfv, double pbv) {
        return PIN ? x : Pfull(x, k, nz, sfv, pbv, ri, tv);
    };
#pragma unroll
    for (int kk = 0; kk < KP; ++kk) {
        if (kk >= nk) break;
        const int k = kl + kk;
        const int o = (k - 1) * W;
        const double pg = Pl(r.e0[o], k, r.S0[0], B0[0]);
        double a, b;
        if (ig) {
            const double pf = Pl(fcol[(k - 1) * 2 + fsel], k, fsp[fsel], fsp[2 + fsel]);
            a = in1 ? Pl(e0b[o + c1], k, s0b[c1], b0b[c1]) : pf; // P(1)
            b = inn ? Pl(e0b[o + cn], k, s0b[cn], b0b[cn]) : pf; // P(nx)
        } else {
            const double* pe = ef + (long long)(k - 1) * d.sk;
            const double pf = Pl(DIST ? __ldcg(pe) : __ldg(pe), k, sff, pbf);
            // jr = 0: P(ny) far, P(1) = row jr+1; jr = ny+1: P(ny) = row jr-1, P(1) far
            a = jr == 0 ? pf : Pl(r.em[o], k, r.Sm[0], r.Sm[W]);
            b = jr == 0 ? Pl(r.ep[o], k, r.Sp[0], r.Sp[W]) : pf;
        }
        const double u = dadd(dmul(d.c2, pg), dmul(dv, dadd(a, b)));
        const double v = Pfull(u, k, nz, r.S0[0], B0[0], ri, tv);
        out[kk] = v;
        ib[(k - 1) * kPairIC] = v;
    }
}

// Row j of e_{s+2}: the i neighbours from the row buffer of row j (B0), the
// j-1 neighbour from the buffer of row j-1 (Bm), and the centre, its k
// neighbours and the j+1 neighbour from registers (Pc = row j, Pn = row j+1,
// both this thread's column); only the k neighbours across the group's ends
// come from B0.  weather.cpp:130-150 on P'.
// POUT: store the post-physics value P(e_{s+2}) (the next pass reads it as it
// is, PIN); sfj / pbj: sf and pb of this column at row j (planes 1 / nz).
template <bool POUT>
__device__ __forceinline__ double pout(double v, bool top, bool bot, double sfj, double pbj,
                                       const Dom& d) {
    if (!POUT) return v;
    double p = dadd(v, d.ri);
    if (top) p = dsub(p, dmul(d.tv, dsub(p, sfj)));
    if (bot) p = dsub(p, dmul(d.tv, dsub(p, pbj)));
    return p;
}

template <int NK, bool FIRST, bool LAST, bool POUT>
__device__ __forceinline__ void final_smem(const double* Bm, const double* B0, const double* Pc,
                                           const double* Pn, double* q, int sk, int kl,
                                           bool store, double sfj, double pbj, const Dom& d) {
    const double dv = d.dv, c6 = d.c6, c5 = d.c5;
    const int o0 = (kl - 1) * kPairIC;
    Bm += o0;
    B0 += o0;
    double v[NK];
#pragma unroll
    for (int kk = 0; kk < NK; ++kk) {
        const int o = kk * kPairIC;
        double s = dadd(B0[o - 1], B0[o + 1]);
        s = dadd(s, Bm[o]);
        s = dadd(s, Pn[kk]);
        const double km = kk > 0 ? Pc[kk - 1] : (FIRST ? 0.0 : B0[o - kPairIC]);
        const double kp = kk + 1 < NK ? Pc[kk + 1] : (LAST ? 0.0 : B0[o + kPairIC]);
        if (FIRST && kk == 0) v[kk] = dadd(dmul(c5, Pc[kk]), dmul(dv, dadd(s, kp)));
        else if (LAST && kk == NK - 1) v[kk] = dadd(dmul(c5, Pc[kk]), dmul(dv, dadd(s, km)));
        else v[kk] = dadd(dmul(c6, Pc[kk]), dmul(dv, dadd(dadd(s, km), kp)));
    }
    if (store) {
#pragma unroll
        for (int kk = 0; kk < NK; ++kk)
            q[kk * sk] =
                pout<POUT>(v[kk], FIRST && kk == 0, LAST && kk == NK - 1, sfj, pbj, d);
    }
}

template <int KP, bool POUT>
__device__ __forceinline__ void final_smem_generic(const double* Bm, const double* B0,
                                                   const double* Bp, double* q, int sk,
                                                   int kl, int nk, double sfj, double pbj,
                                                   const Dom& d) {
    const int nz = d.nz;
    const double dv = d.dv;
#pragma unroll
    for (int kk = 0; kk < KP; ++kk) {
        if (kk >= nk) break;
        const int k = kl + kk;
        const int o = (k - 1) * kPairIC;
        double s = dadd(B0[o - 1], B0[o + 1]);
        s = dadd(s, Bm[o]);
        s = dadd(s, Bp[o]);
        double v;
        if (k == 1) v = dadd(dmul(d.c5, B0[o]), dmul(dv, dadd(s, B0[o + kPairIC])));
        else if (k == nz) v = dadd(dmul(d.c5, B0[o]), dmul(dv, dadd(s, B0[o - kPairIC])));
        else v = dadd(dmul(d.c6, B0[o]), dmul(dv, dadd(dadd(s, B0[o - kPairIC]), B0[o + kPairIC])));
        q[kk * sk] = pout<POUT>(v, k == 1, k == nz, sfj, pbj, d);
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
template <bool POUT>
__device__ __forceinline__ void pair_ghost_cols(const Dom& d, const PairArgs& a,
                                             double* __restrict__ u, const double* __restrict__ sf,
                                             const double* __restrict__ pb, int ja, int jb,
                                             int tid) {
    const int nx = d.nx, ny = d.ny, nz = d.nz;
    const int r0 = ja == 1 ? 0 : ja, r1 = jb == ny ? ny + 1 : jb;
    const int nr = r1 - r0 + 1;
    const long long n = 2LL * nr * nz;
    auto G = [&](int w, int j, int k) {
        return __ldcg(a.gcol + ((long long)w * (ny + 2) + j) * nz + (k - 1));
    };
    for (long long t = tid; t < n; t += kPairThreads) {
        const int k = 1 + (int)(t % nz);
        const long long q = t / nz;
        const int j = r0 + (int)(q % nr);
        const int side = (int)(q / nr); // 0: i = 0, 1: i = nx+1
        const double pg = G(side == 0 ? 0 : 3, j, k);
        const double v = dadd(dmul(d.c2, pg), dmul(d.dv, dadd(G(1, j, k), G(2, j, k))));
        const int i = side == 0 ? 0 : nx + 1;
        u[i * d.si + j * d.sj + (long long)(k - 1) * d.sk] =
            POUT ? pout<true>(v, k == 1, k == nz, __ldg(sf + i + j * d.s2j), __ldg(pb + i + j * d.s2j), d)
                 : v;
    }
}

// The second producer of a strip's j-ghost intermediates computes that
// strip's j-ghost cells (i in i0..i0+TX-1 clipped to 1..nx, j = 0 and ny+1):
// weather.cpp:155-158 on the intermediate field.
template <bool POUT>
__device__ __forceinline__ void pair_ghost_rows(const Dom& d, const PairArgs& a,
                                             double* __restrict__ u, const double* __restrict__ sf,
                                             const double* __restrict__ pb, int i0, int tid) {
    const int nx = d.nx, ny = d.ny, nz = d.nz;
    const int ni = min(kPairTX, nx - i0 + 1);
    const long long n = 2LL * ni * nz;
    auto G = [&](int w, int i, int k) {
        return __ldcg(a.grow + ((long long)w * nz + (k - 1)) * (nx + 2) + i);
    };
    for (long long t = tid; t < n; t += kPairThreads) {
        const int i = i0 + (int)(t % ni);
        const long long q = t / ni;
        const int k = 1 + (int)(q % nz);
        const int side = (int)(q / nz); // 0: j = 0, 1: j = ny+1
        const double pg = G(side == 0 ? 0 : 3, i, k);
        const double v = dadd(dmul(d.c2, pg), dmul(d.dv, dadd(G(2, i, k), G(1, i, k))));
        const int j = side == 0 ? 0 : ny + 1;
        u[i * d.si + j * d.sj + (long long)(k - 1) * d.sk] =
            POUT ? pout<true>(v, k == 1, k == nz, __ldg(sf + i + j * d.s2j), __ldg(pb + i + j * d.s2j), d)
                 : v;
    }
}

// Thread 0's TMA issue state: the unit and row of the next slab to load.
struct PairProducer {
    int unit;  // unit of the next load (-1: the stop sentinel has been issued)
    int row;   // its row (ja-2 .. jb+2)
    int jb;    // last inner row of that unit
    int slot;  // ring slot of the next load
    bool waited; // decomposed: the neighbours' previous pass has been seen complete
};

template <bool DIST>
__device__ __forceinline__ void pair_issue(PairProducer& p, unsigned char* smem, const PairGeom& G,
                                        uint64_t* full, int* slot_unit, int ns,
                                        const CUtensorMap* tm_e, const CUtensorMap* tm_sfpb,
                                        const CUtensorMap* tm_ef, const CUtensorMap* tm_sfpbf,
                                        const PairArgs& a, const Dom& d, const Halo& h) {
    const int ny = d.ny;
    if (p.unit < 0) return; // the sentinel is out: nothing left
    const int slot = p.slot;
    p.slot = slot + 1 == ns ? 0 : slot + 1;
    if (p.row > p.jb + 2) {
        // the current unit is fully issued: take the next one
        p.unit = atomicAdd(&a.sched[0], 1);
        if (a.reverse && p.unit < a.nstrips * a.nchunks) p.unit = a.nstrips * a.nchunks - 1 - p.unit;
        if (p.unit >= a.nstrips * a.nchunks) {
            slot_unit[slot] = -1;
            mbar_arrive(&full[slot]); // no bytes: tells the consumers to finish
            p.unit = -1;
            return;
        }
        const int ch = p.unit / a.nstrips;
        int ja;
        pair_rows(a, ny, ch, ja, p.jb);
        p.row = ja - 2;
        if (DIST && rim_unit(d, 1 + (p.unit % a.nstrips) * kPairTX, kPairTX, ja, p.jb)) {
            // decomposed: the unit reads halo slots the neighbours filled in their
            // previous pass and pushes into slots they read then (flags only
            // grow: once seen, later rim units of this launch need no poll)
            if (!p.waited) {
                halo_wait(h, 1);
                p.waited = true;
            }
            asm volatile("fence.proxy.async.global;" ::: "memory");
        }
    }
    const int st = p.unit % a.nstrips;
    const int ic = a.fp + 1 + st * kPairTX - 2; // tensor i of i0 - 2 (even)
    const int far = pair_far_col<DIST>(st, a.nstrips, d);
    slot_unit[slot] = p.unit;
    unsigned char* stg = smem + (size_t)slot * G.stage;
    mbar_expect_tx(&full[slot], far ? G.tx_far : G.tx_main);
    tma_load_3d(stg, tm_e, &full[slot], ic, a.jrow0 + p.row, 0);
    tma_load_3d(stg + G.slab, tm_sfpb, &full[slot], ic, a.jrow0 + p.row, 0);
    if (far) {
        const int fx = (a.fp + far) & ~1; // even-aligned pair holding the far column
        unsigned char* f = stg + G.slab + G.sfpb;
        tma_load_3d(f, tm_ef, &full[slot], fx, a.jrow0 + p.row, 0);
        tma_load_3d(f + G.fcol, tm_sfpbf, &full[slot], fx, a.jrow0 + p.row, 0);
    }
    ++p.row;
}

// Ring position of a load: slot and mbarrier phase parity.
struct RingPos {
    int slot;
    uint32_t par;
    __device__ __forceinline__ RingPos next(int ns) const {
        return slot + 1 == ns ? RingPos{0, par ^ 1u} : RingPos{slot + 1, par};
    }
};

// KPT: max k planes per thread (nz <= 8 * KPT).  DIST: a decomposed rank's
// subdomain (a separate instantiation: the single-domain code is unchanged).
// PIN / POUT: e_s is stored post-physics / store e_{s+2}
// post-physics -- between the passes of one call the field is kept as P(e),
// which is all the next pass reads, so no pass but the first recomputes the
// physics of its loads (the same rounded ops, done once by the producer).
template <int KPT, bool DIST, bool PIN, bool POUT>
__global__ void __launch_bounds__(kPairThreads, kPairMinBlocks)
    step_pair_kernel(const __grid_constant__ CUtensorMap tm_e,
                     const __grid_constant__ CUtensorMap tm_sfpb,
                     const __grid_constant__ CUtensorMap tm_ef,
                     const __grid_constant__ CUtensorMap tm_sfpbf, const double* __restrict__ e,
                     double* __restrict__ u, const double* __restrict__ sf,
                     const double* __restrict__ pb, Dom d, PairArgs a,
                     const __grid_constant__ Halo h) {
    extern __shared__ __align__(128) unsigned char smem[];
    const PairGeom G = pair_geom(d.nz);
    const int NS = a.ns;
    // intermediate row buffers: ib0 + b * ibn, b rotating over kPairNIB
    double* const ib0 = reinterpret_cast<double*>(smem + (size_t)NS * G.stage);
    const int ibn = G.ib / 8;
    uint64_t* full =
        reinterpret_cast<uint64_t*>(smem + (size_t)NS * G.stage + kPairNIB * (size_t)G.ib);
    int* slot_unit = reinterpret_cast<int*>(full + NS);
    const uint32_t full_u32 = smem_u32(full); // the ring barriers' shared-window address
    __shared__ int s_flags;
    const int tid = threadIdx.x;
    const int nx = d.nx, ny = d.ny, nz = d.nz;

    PairProducer prod{0, 1, -2, 0, false}; // row > jb + 2: the first issue takes a unit
    pdl_start();
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int s = 0; s < NS; ++s)
            pair_issue<DIST>(prod, smem, G, full, slot_unit, NS, &tm_e, &tm_sfpb, &tm_ef,
                             &tm_sfpbf, a, d, h);
    }
    __syncthreads();

    // thread -> (intermediate column cc = 1 .. TX+2 = logical i0-2+cc, k-group g)
    const int cc = 1 + (tid % kPairIC);
    const int g = tid / kPairIC;
    // k-groups: planes kl .. kh, nk = kh - kl + 1 <= KPT.  The first and last
    // groups carry the surface / boundary-layer corrections of planes 1 and nz
    // (about one extra plane of work), so the nz % KG extra planes go to the
    // middle groups first: nz = 58 -> 7 8 8 7 7 7 7 7.
    int kl = 1, nk = 0;
    {
        const int base = nz / kPairKG, rem = nz % kPairKG;
        for (int q = 0; q <= g; ++q) {
            kl += nk;
            nk = base + ((q >= 1 && q <= min(rem, kPairKG - 2)) ||
                         (rem == kPairKG - 1 && q == kPairKG - 1));
        }
    }
    const int kh = kl + nk - 1;
    // plane stride as an int: kk * sk stays below 2^31 (setup_pair checks KPT * sk), so
    // the final's store addresses are one 32 x 32 + 64 multiply-add each
    const int sk32 = (int)d.sk;
    const bool kfirst = kl == 1, klast = kh == nz;
    // compile-time row shapes: nk in {KPT, KPT-1} x (first, last); else generic
    const int fl = (kfirst ? 1 : 0) + (klast ? 2 : 0);
    // (an edge group of KPT planes occurs only for nz > 62, beyond the pair
    // kernel's 2-CTA shared-memory budget: it takes the generic path)
    int shape = nz < 2 * kPairKG || fl == 3 ? 16
                : nk == KPT ? (fl ? 16 : 0) : nk == KPT - 1 ? 4 + fl : 16;

    double PW2[KPT]; // this row's intermediate values
    double PW1[KPT]; // the previous row's (the final row's centre)
    RingPos R0{0, 0}; // ring position of the current unit's first slab (row ja-2)
    int ibi = 0;      // row buffer of the next intermediate row (rotates over kPairNIB)
    for (;;) {
        mbar_wait_u32(full_u32 + 8u * R0.slot, R0.par);
        const int unit = slot_unit[R0.slot];
        if (unit < 0) break;
        const int ch = unit / a.nstrips, st = unit % a.nstrips;
        int ja, jb;
        pair_rows(a, ny, ch, ja, jb);
        const int i0 = 1 + st * kPairTX;
        const int gi = i0 - 2 + cc; // logical i of my intermediate column
        const bool indom = gi <= nx + 1 && nk > 0;
        // owned columns of this unit (a decomposed rank owns column 0 / nx+1 only
        // on the global edge; elsewhere they are halo cells)
        const int ilo = st == 0 ? (!DIST || d.own_w ? 0 : 1) : i0;
        const int ihi = st == a.nstrips - 1 ? (!DIST || d.own_e ? nx + 1 : nx) : i0 + kPairTX - 1;
        const bool owns_i = gi >= ilo && gi <= ihi;
        const bool ig = DIST ? (d.own_w && gi == 0) || (d.own_e && gi == nx + 1)
                             : gi == 0 || gi == nx + 1;
        // does this thread ever publish in this unit (a ghost-adjacent column, or
        // an inner column whose rows 0, 1, ny, ny+1 may fall in this unit)?
        const bool pub_col = owns_i && (gi <= 1 || gi >= nx);
        const bool pub_row = owns_i && gi >= 1 && gi <= nx && (ja <= 2 || jb >= ny - 1);
        const int fsel = (a.fp + pair_far_col<DIST>(st, a.nstrips, d)) & 1;
        const bool do_final = cc >= 2 && cc <= kPairTX + 1 && gi <= nx && nk > 0;

        RingPos Ra = R0;          // slab jr-1
        RingPos Rb = Ra.next(NS); // slab jr
        RingPos Rc = Rb.next(NS); // slab jr+1
        // the three slabs at this thread's column, rotated with the ring
        const unsigned char* sm_ = smem + (size_t)Ra.slot * G.stage + cc * 8;
        const unsigned char* s0_ = smem + (size_t)Rb.slot * G.stage + cc * 8;
        const unsigned char* sp_ = smem + (size_t)Rc.slot * G.stage + cc * 8;
        // this thread's output column at row ja-2 (the final row of jr = ja-1),
        // advanced one row per iteration
        double* qrow = u + (long long)gi * d.si + (long long)(ja - 2) * d.sj +
                       (long long)(kl - 1) * d.sk;
        mbar_wait_u32(full_u32 + 8u * Rb.slot, Rb.par);
        for (int jr = ja - 1; jr <= jb + 1; ++jr) {
            mbar_wait_u32(full_u32 + 8u * Rc.slot, Rc.par);
            // row buffers: jr -> ibi, jr-1 -> ibi-1, jr-2 -> ibi-2 (mod kPairNIB)
            const int ib1 = ibi == 0 ? kPairNIB - 1 : ibi - 1;
            const int ib2 = ib1 == 0 ? kPairNIB - 1 : ib1 - 1;
            double* ibrow = ib0 + ibi * ibn + (cc - 1);
            if (indom) {
                const IRow r{reinterpret_cast<const double*>(sm_),
                             reinterpret_cast<const double*>(s0_),
                             reinterpret_cast<const double*>(sp_),
                             reinterpret_cast<const double*>(sm_ + G.slab),
                             reinterpret_cast<const double*>(s0_ + G.slab),
                             reinterpret_cast<const double*>(sp_ + G.slab)};
                const bool ghost = DIST ? ig || (d.own_s && jr == 0) || (d.own_n && jr == ny + 1)
                                        : ig || jr == 0 || jr == ny + 1;
                switch (ghost ? 16 : shape) {
                case 0: inter_inner<KPT, KPT, false, false, PIN>(r, PW2, ibrow, kl, d); break;
                case 4: inter_inner<KPT, KPT - 1, false, false, PIN>(r, PW2, ibrow, kl, d); break;
                case 5: inter_inner<KPT, KPT - 1, true, false, PIN>(r, PW2, ibrow, kl, d); break;
                case 6: inter_inner<KPT, KPT - 1, false, true, PIN>(r, PW2, ibrow, kl, d); break;
                default:
                    if (ghost) {
                        const unsigned char* sb = s0_ - cc * 8;
                        const double* fb = reinterpret_cast<const double*>(sb + G.slab + G.sfpb);
                        const double* fsp =
                            reinterpret_cast<const double*>(sb + G.slab + G.sfpb + G.fcol);
                        inter_ghost<KPT, DIST, PIN>(r, PW2, ibrow, kl, nk, gi, jr, cc, i0, d, e, sf, pb, fb,
                                         fsp, fsel);
                    } else {
                        inter_generic<KPT, PIN>(r, PW2, ibrow, kl, nk, d);
                    }
                    break;
                }
                if (pub_col || pub_row) {
                    const bool owns_j = (jr >= ja && jr <= jb) ||
                                        (DIST ? (d.own_s && jr == 0) || (d.own_n && jr == ny + 1)
                                              : jr == 0 || jr == ny + 1);
                    if (owns_j) pair_publish<KPT>(PW2, kl, nk, gi, jr, d, a);
                }
            }
            // POUT: sf / pb of row jr-1 (the final row's planes 1 / nz) before its slab is freed
            double sfj = 0.0, pbj = 0.0;
            if (POUT && kfirst) sfj = reinterpret_cast<const double*>(sm_ + G.slab)[0];
            if (POUT && klast) pbj = reinterpret_cast<const double*>(sm_ + G.slab)[kPairW];
            __syncthreads(); // intermediate row jr complete; slab jr-1 free
            // refill slab jr-1's slot (and, after the last row, those of jb+1, jb+2)
            if (tid == 0) {
                const int nfree = jr == jb + 1 ? 3 : 1;
                for (int f = 0; f < nfree; ++f)
                    pair_issue<DIST>(prod, smem, G, full, slot_unit, NS, &tm_e, &tm_sfpb,
                                     &tm_ef, &tm_sfpbf, a, d, h);
            }
            if (do_final && jr >= ja + 1) {
                // row j = jr-1 of e_{s+2} from intermediate rows jr-2, jr-1, jr
                const double* Bm = ib0 + ib2 * ibn + (cc - 1);
                const double* B0 = ib0 + ib1 * ibn + (cc - 1);
                const double* Bp = ib0 + ibi * ibn + (cc - 1);
                double* q = qrow;
                switch (shape) {
                case 0: final_smem<KPT, false, false, POUT>(Bm, B0, PW1, PW2, q, sk32, kl, true, sfj, pbj, d); break;
                case 4: final_smem<KPT - 1, false, false, POUT>(Bm, B0, PW1, PW2, q, sk32, kl, true, sfj, pbj, d); break;
                case 5: final_smem<KPT - 1, true, false, POUT>(Bm, B0, PW1, PW2, q, sk32, kl, true, sfj, pbj, d); break;
                case 6: final_smem<KPT - 1, false, true, POUT>(Bm, B0, PW1, PW2, q, sk32, kl, true, sfj, pbj, d); break;
                default: final_smem_generic<KPT, POUT>(Bm, B0, Bp, q, sk32, kl, nk, sfj, pbj, d); break;
                }
            }
            // No second barrier: the next row's target buffer (ib2) is read here only
            // as Bm, at this thread's own column and planes; the neighbour warps'
            // reads of it (their B0 k-boundary planes, one row earlier) are ordered
            // before the next write by this row's barrier.
#pragma unroll
            for (int kk = 0; kk < KPT; ++kk) PW1[kk] = PW2[kk];
            ibi = ibi == kPairNIB - 1 ? 0 : ibi + 1;
            Ra = Rb;
            Rb = Rc;
            Rc = Rc.next(NS);
            sm_ = s0_;
            s0_ = sp_;
            sp_ = smem + (size_t)Rc.slot * G.stage + cc * 8;
            qrow += d.sj;
        }
        R0 = Rc; // slabs jb+1, jb+2 were Ra, Rb: the next unit starts after them
        if (DIST && rim_unit(d, i0, kPairTX, ja, jb)) {
            // decomposed rim unit: its new cells near a face go to the neighbours
            __syncthreads();
            push_box(h, d, u, i0, min(i0 + kPairTX - 1, nx), ja, jb, tid, kPairThreads);
        }
        // rim units: count the ghost producers; the second one computes the ghosts
        // (decomposed: pair_ghost_kernel, after the wrap partners published)
        const int inc_c = (st == 0) + (st == a.nstrips - 1);
        const int inc_r = (ch == 0) + (ch == a.nchunks - 1);
        if (!DIST && (inc_c | inc_r)) {
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
            __syncthreads();
            const int f = s_flags;
            if (f & 1) pair_ghost_cols<POUT>(d, a, u, sf, pb, ja, jb, tid);
            if (f & 2) pair_ghost_rows<POUT>(d, a, u, sf, pb, i0, tid);
            __syncthreads(); // s_flags is reused by the next rim unit
        }
    }
    // the last CTA to finish re-arms the scheduler for the next launch and,
    // decomposed, tells the wrap partners that its intermediates are published
    // (value = the step after this pass, h.step + 2)
    if (tid == 0) {
        if (DIST) __threadfence_system();
        else __threadfence();
        if (atomicAdd(&a.sched[1], 1) == (int)gridDim.x - 1) {
            a.sched[0] = 0;
            a.sched[1] = 0;
            if (DIST) {
                __threadfence_system();
                for (int q = 0; q < 4; ++q)
                    if (h.nb[q] && h.depth[q] == 1)
                        st_relaxed_sys(&h.nb_flags[q][kPubFlag + opp_dir(q)],
                                       (unsigned long long)(h.step + 2));
            }
            __threadfence();
        }
    }
}

// Ghost cells of e_{s+2} on a decomposed rank (weather.cpp:152-168 on the
// intermediate field P'): the i-ghost column of an owned W / E edge (rows of
// the rank, corners included: the i rule wins) and the j-ghost row of an owned
// S / N edge (inner columns), from this rank's published P' and the wrap
// partner's (P2P reads of its gcol / grow; the rank itself when the
// decomposition has one rank along that axis).  Then every new ghost cell near
// a face goes to the neighbours, and the last CTA releases the pass (h.step+1
// = s+2) to all neighbours.
struct PairGhostArgs {
    const double* gcol;   // this rank's P' columns 0, 1, nx, nx+1: [4][ny+2][nz]
    const double* grow;   // this rank's P' rows 0, 1, ny, ny+1: [4][nz][nx+2]
    const double* gcol_w; // W wrap partner's (its column nx is global nx)
    const double* gcol_e; // E wrap partner's (its column 1 is global 1)
    const double* grow_s; // S wrap partner's (its row ny is global ny)
    const double* grow_n; // N wrap partner's (its row 1 is global 1)
    int wait[4];          // wait for the wrap partner's "published" flag (W E S N)
    long long pub;        // the value it releases (s + 2)
};

template <bool POUT>
__global__ void __launch_bounds__(256) pair_ghost_kernel(double* __restrict__ u,
                                                         const double* __restrict__ sf,
                                                         const double* __restrict__ pb, Dom d,
                                                         Halo h, PairGhostArgs g) {
    const int nx = d.nx, ny = d.ny, nz = d.nz;
    if (threadIdx.x == 0 && !h.nowait) {
        for (int q = 0; q < 4; ++q)
            if (g.wait[q]) wait_flag(&h.my_flags[kPubFlag + q], g.pub);
    }
    __syncthreads();
    const Owned o = owned(d);
    const long long nr = o.j1 - o.j0 + 1;           // owned rows (i-ghost columns)
    const long long ncol = nr * nz;
    const long long nw = d.own_w ? ncol : 0, ne = d.own_e ? ncol : 0;
    const long long nrow = (long long)nx * nz;      // inner columns (j-ghost rows)
    const long long ns = d.own_s ? nrow : 0, nn = d.own_n ? nrow : 0;
    const long long n = nw + ne + ns + nn;
    auto C = [&](const double* b, int w, int j, int k) {
        return __ldcg(b + ((long long)w * (ny + 2) + j) * nz + (k - 1));
    };
    auto R = [&](const double* b, int w, int i, int k) {
        return __ldcg(b + ((long long)w * nz + (k - 1)) * (nx + 2) + i);
    };
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        int i, j, k;
        double v;
        if (t < nw + ne) {
            // k fastest: the published columns are [w][j][k], so a warp reads 32
            // consecutive values of each
            const bool west = t < nw;
            const long long q = west ? t : t - nw;
            k = 1 + (int)(q % nz);
            j = o.j0 + (int)(q / nz);
            if (west) { // (1-2dv) P'(0) + dv (P'(1) + P'(gnx))
                i = 0;
                v = dadd(dmul(d.c2, C(g.gcol, 0, j, k)),
                         dmul(d.dv, dadd(C(g.gcol, 1, j, k), C(g.gcol_w, 2, j, k))));
            } else {    // (1-2dv) P'(nx+1) + dv (P'(1) + P'(nx))
                i = nx + 1;
                v = dadd(dmul(d.c2, C(g.gcol, 3, j, k)),
                         dmul(d.dv, dadd(C(g.gcol_e, 1, j, k), C(g.gcol, 2, j, k))));
            }
        } else {
            const long long q0 = t - nw - ne;
            const bool south = q0 < ns;
            const long long q = south ? q0 : q0 - ns;
            i = 1 + (int)(q % nx);
            k = 1 + (int)(q / nx);
            if (south) { // (1-2dv) P'(j=0) + dv (P'(gny) + P'(1))
                j = 0;
                v = dadd(dmul(d.c2, R(g.grow, 0, i, k)),
                         dmul(d.dv, dadd(R(g.grow_s, 2, i, k), R(g.grow, 1, i, k))));
            } else {     // (1-2dv) P'(ny+1) + dv (P'(ny) + P'(1))
                j = ny + 1;
                v = dadd(dmul(d.c2, R(g.grow, 3, i, k)),
                         dmul(d.dv, dadd(R(g.grow, 2, i, k), R(g.grow_n, 1, i, k))));
            }
        }
        // POUT: stored (and pushed) post-physics, like the pair kernel's cells
        const double w = POUT ? pout<true>(v, k == 1, k == nz, __ldg(sf + i + j * d.s2j),
                                           __ldg(pb + i + j * d.s2j), d)
                              : v;
        u[i * d.si + j * d.sj + (long long)(k - 1) * d.sk] = w;
        halo_push(h, d, i, j, k, w);
    }
    __syncthreads();
    if (threadIdx.x == 0) halo_signal(h);
}

} // namespace hftw
