// weather_wave.cuh -- K timesteps in ONE persistent launch (a wavefront across steps).
//
// Reference hot path: nsteps x hft::reference_step (weather.cpp:101-171), as
// run_reference / the corpus driver's time loop apply it (weather.cpp:173-178).
// Each step is computed exactly as by step_tma_kernel (same slabs, same
// register window, same explicitly rounded operations), so the result is
// bitwise identical; what changes is the schedule.  Instead of one launch per
// step -- whose ramp-up, tail and launch gap every step pays -- one launch
// walks a single global work list
//     step 0: [G ghost-row tasks][units of chunk 0][chunk 1] ...
//     step 1: [G ghost-row tasks][units of chunk 0] ...
// handed out by one atomic counter.  A unit of step s (strip st, rows ja..jb)
// starts as soon as step s-1 has finished the chunks it reads (ch-1, ch, ch+1)
// -- tracked by per-chunk completion counters -- so step s+1 sweeps the grid a
// few chunks behind step s and the SMs never drain between steps.
//
// Dependencies (src = field of step s, dst = field of step s+1; the two
// buffers alternate, so dst of step s is src of step s-1):
//   * chunk unit (s, ch): reads src rows ja-1 .. jb+1 -> chunks ch-1..ch+1 of
//     step s-1 complete (also covers the write-after-read on its dst rows,
//     which step s-1 read only from those chunks); chunk 0 / the last chunk
//     also read / write the rows the ghost-row tasks of step s-1 touch (rows
//     0, 1 / ny, ny+1) -> those tasks complete;
//   * ghost-row task (s): rows 0 and ny+1 (weather.cpp:152-159, corners by
//     :161-168) read src rows 0, 1, ny, ny+1 -> chunk 0, the last chunk and the
//     ghost tasks of step s-1 complete.  Row 0 depends on row ny (the cyclic
//     rule), which is why these are separate tasks: chunk 0 of step s+1 only
//     waits for them, not for the end of step s;
//   * the i-ghost columns (weather.cpp:161-168) of rows ja..jb are computed by
//     the edge-strip units of that chunk (their partner column nx / 1 is in the
//     same rows, i.e. the same chunk dependency).
// Every wait is on work earlier in the list, and the grid is persistent (one
// CTA per SM, all resident), so the schedule cannot deadlock.  Completion
// counters are monotonic within a launch and reset by the last CTA.
#pragma once

#include "weather_kernels.cuh"

namespace hftw {

struct WaveArgs {
    int fp, jrow0;       // tensor-map coordinates of logical i = 0 / j = 0
    int nstrips, nchunks, chunk, ns;
    int nsteps;          // steps of this launch
    int gtasks;          // ghost-row tasks per step
    int alt;             // odd chunks sweep their rows downwards (see wave_rows_down)
    int* sched;          // [0] next work item, [1] CTAs finished
    int* chunk_done;     // [nchunks] units completed (all steps of this launch)
    int* ghost_done;     // [1] ghost-row tasks completed
    double* buf0;        // field of step 0 (logical (0,0,1)); steps alternate
    double* buf1;
    // decomposed runs (Halo::active): the pushes of steps writing buf1 (even s) and
    // buf0 (odd s), and per-step completion counters -- when the last work item of
    // step s finishes, its thread publishes flag = h.step + s + 1 to the neighbours
    Halo h_even, h_odd;
    int* step_done;      // [nsteps]
};

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void wait_geq(const int* p, int target) {
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_gpu(p) < target) {
        __nanosleep(100);
        spin_check(t0);
    }
}

__device__ __forceinline__ bool wave_rows_down(const WaveArgs& a, int unit) {
    return a.alt && ((unit / a.nstrips) & 1);
}

// One ghost-row task: its share of rows j = 0 and ny+1 (all i, corners
// included; cell_update applies the reference's precedence).
template <bool PHYS>
__device__ __forceinline__ void wave_ghost_rows(const double* __restrict__ e,
                                                double* __restrict__ u,
                                                const double* __restrict__ sf,
                                                const double* __restrict__ pb, const Dom& d,
                                                const Halo& h, int task, int ntasks, int tid,
                                                int nthreads) {
    // the rows this domain owns (a decomposed rank owns the global ghost row of
    // its edge, if any), over its owned i range; cells next to a neighbour are
    // pushed into its halo as in step_tma_kernel
    const Owned o = owned(d);
    const int rows = (d.own_s ? 1 : 0) + (d.own_n ? 1 : 0);
    const long long ni = o.i1 - o.i0 + 1;
    const long long n = rows * ni * d.nz;
    const long long lo = n * task / ntasks, hi = n * (task + 1) / ntasks;
    for (long long t = lo + tid; t < hi; t += nthreads) {
        const int i = o.i0 + (int)(t % ni);
        const long long q = t / ni;
        const int k = 1 + (int)(q % d.nz);
        const int j = ((q / d.nz) == 0 && d.own_s) ? 0 : d.ny + 1;
        const double v = cell_update<PHYS, true>(e, sf, pb, d, i, j, k);
        u[i * d.si + j * d.sj + (long long)(k - 1) * d.sk] = v;
        halo_push(h, d, i, j, k, v);
    }
}

// i-ghost columns of rows ja..jb: i = 0 (strip 0) and/or nx+1 (last strip).
template <bool PHYS>
__device__ __forceinline__ void wave_ghost_cols(const double* __restrict__ e,
                                                double* __restrict__ u,
                                                const double* __restrict__ sf,
                                                const double* __restrict__ pb, const Dom& d,
                                                const Halo& h, int ja, int jb, bool west,
                                                bool east, int tid, int nthreads) {
    const int nr = jb - ja + 1;
    const long long per = (long long)nr * d.nz;
    const long long n = per * ((west ? 1 : 0) + (east ? 1 : 0));
    for (long long t = tid; t < n; t += nthreads) {
        const bool w = west && t < per;
        const long long q = w || !west ? t : t - per;
        const int j = ja + (int)(q % nr);
        const int k = 1 + (int)(q / nr);
        const int i = w ? 0 : d.nx + 1;
        const double v = cell_update<PHYS, true>(e, sf, pb, d, i, j, k);
        u[i * d.si + j * d.sj + (long long)(k - 1) * d.sk] = v;
        halo_push(h, d, i, j, k, v); // a ghost column's first / last rows go to S / N
    }
}

// A work item of step s is complete (its stores are issued): count it; the
// thread completing the step publishes it to the neighbours (decomposed runs).
__device__ __forceinline__ void wave_item_done(const WaveArgs& a, int s, int per_step) {
    const Halo& h = (s & 1) ? a.h_odd : a.h_even;
    if (!h.active) return;
    __threadfence_system(); // this item's pushes into the neighbours precede the count
    if (atomicAdd(&a.step_done[s], 1) == per_step - 1) {
        __threadfence_system();
        for (int q = 0; q < kNbrs; ++q)
            if (h.nb[q]) st_relaxed_sys(&h.nb_flags[q][opp_dir(q)], (unsigned long long)(h.step + s + 1));
    }
}

// Consumer warps of step_wave_kernel (the row loop of step_tma_kernel).
template <int TX, int NCW, bool PHYS>
__device__ __forceinline__ void wave_consumers(unsigned char* smem, const SlabGeom& G,
                                               uint64_t* full, uint64_t* empty,
                                               const int* slot_item,
                                               const double* __restrict__ sf,
                                               const double* __restrict__ pb, const Dom& d,
                                               const WaveArgs& a) {
    const int NS = a.ns;
    const int lane = threadIdx.x & 31;
    const int units = a.nstrips * a.nchunks;
    const int per_step = a.gtasks + units;
    constexpr int NKG = NCW * 32 / TX;
    const int c = threadIdx.x % TX, g = threadIdx.x / TX;
    const int nz = d.nz;
    const int kl = 1 + (g * nz) / NKG, kh = ((g + 1) * nz) / NKG;
    const int w = G.w, cc = c + 2;
    const double ri = d.ri, tv = d.tv, dv = d.dv, c5 = d.c5, c6 = d.c6;
    const int tid = threadIdx.x, nthreads = NCW * 32;

    uint32_t L = 0;
    for (;;) {
        {
            const uint32_t slot = L % NS;
            mbar_wait(&full[slot], (L / NS) & 1);
        }
        // one reader per warp (the lane that later arrives on the slot's `empty`
        // barrier), broadcast by shuffle: the producer's next write of this slot
        // item is ordered after it by that arrive alone
        int item = 0;
        if (lane == 0) item = slot_item[L % NS];
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item < 0) break;
        const int s = item / per_step, r = item % per_step;
        const double* e = (s & 1) ? a.buf1 : a.buf0;
        double* u = (s & 1) ? a.buf0 : a.buf1;
        const Halo& hs = (s & 1) ? a.h_odd : a.h_even; // pushes of this step
        if (r < a.gtasks) {
            // ghost-row task: from global memory, no slab
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[L % NS]);
            ++L;
            wave_ghost_rows<PHYS>(e, u, sf, pb, d, (s & 1) ? a.h_odd : a.h_even, r, a.gtasks, tid,
                            nthreads);
            asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
            if (tid == 0) {
                __threadfence();
                asm volatile("fence.proxy.async.global;" ::: "memory");
                atomicAdd(a.ghost_done, 1);
                wave_item_done(a, s, per_step);
            }
            continue;
        }
        const int unit = r - a.gtasks;
        const int ch = unit / a.nstrips, st = unit % a.nstrips;
        const int ja = ch * a.chunk + 1, jb = min(d.ny, ja + a.chunk - 1);
        const int i0 = 1 + st * TX;
        const bool active = c < min(TX, d.nx - i0 + 1) && kl <= kh;
        const bool down = wave_rows_down(a, unit);
        for (int m = 0; m <= jb - ja; ++m) {
            // slabs l0, l1, l2 hold rows j-1, j, j+1 (upwards) or j+1, j, j-1 (downwards)
            const int j = down ? jb - m : ja + m;
            const uint32_t l0 = L + m, l1 = l0 + 1, l2 = l0 + 2;
            if (m == 0) mbar_wait(&full[l1 % NS], (l1 / NS) & 1);
            mbar_wait(&full[l2 % NS], (l2 / NS) & 1);
            if (active) {
                const unsigned char* stm = smem + (size_t)((down ? l2 : l0) % NS) * G.stage;
                const unsigned char* st0 = smem + (size_t)(l1 % NS) * G.stage;
                const unsigned char* stp = smem + (size_t)((down ? l0 : l2) % NS) * G.stage;
                const double* em = reinterpret_cast<const double*>(stm) + cc;
                const double* e0 = reinterpret_cast<const double*>(st0) + cc;
                const double* ep = reinterpret_cast<const double*>(stp) + cc;
                const double* Sm = reinterpret_cast<const double*>(stm + G.e_bytes) + cc;
                const double* S0 = reinterpret_cast<const double*>(st0 + G.e_bytes) + cc;
                const double* Sp = reinterpret_cast<const double*>(stp + G.e_bytes) + cc;
                const double* Bm = reinterpret_cast<const double*>(stm + G.e_bytes + G.r_bytes) + cc;
                const double* B0 = reinterpret_cast<const double*>(st0 + G.e_bytes + G.r_bytes) + cc;
                const double* Bp = reinterpret_cast<const double*>(stp + G.e_bytes + G.r_bytes) + cc;
                double* up = u + (long long)(i0 + c) * d.si + (long long)j * d.sj +
                             (long long)(kl - 1) * d.sk;
                const ColumnRow row{em, e0, ep, Sm, S0, Sp, Bm, B0, Bp, up, d.sk,
                                    w, 1, kl, kh, nz, ri, tv, dv, c5, c6, i0 + c, j};
                column_row<PHYS>(row);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[l0 % NS]);
        }
        const uint32_t lend = L + (jb - ja + 1);
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&empty[lend % NS]);
            mbar_arrive(&empty[(lend + 1) % NS]);
        }
        L = lend + 2;
        // decomposed rim unit: its cells near a face go to the neighbours
        if (hs.active && rim_unit(d, i0, TX, ja, jb)) {
            asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
            push_box(hs, d, u, i0, min(i0 + TX - 1, d.nx), ja, jb, tid, nthreads);
        }
        // the i-ghost columns of these rows (their partners are in the same rows)
        const bool west = st == 0 && d.own_w, east = st == a.nstrips - 1 && d.own_e;
        if (west || east) wave_ghost_cols<PHYS>(e, u, sf, pb, d, hs, ja, jb, west, east, tid, nthreads);
        // publish: every consumer's stores of this unit precede the count
        asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
        if (tid == 0) {
            __threadfence();
            asm volatile("fence.proxy.async.global;" ::: "memory");
            atomicAdd(&a.chunk_done[ch], 1);
            wave_item_done(a, s, per_step);
        }
    }
}

// PHYS = false: diffusion-only sweeps of an already post-physics field
// (hftw_diffuse_steps), the same schedule.
template <int TX, int NCW, bool PHYS>
__global__ void __launch_bounds__((NCW + 1) * 32, 1)
    step_wave_kernel(const __grid_constant__ CUtensorMap tm_e0,
                     const __grid_constant__ CUtensorMap tm_e1,
                     const __grid_constant__ CUtensorMap tm_sf,
                     const __grid_constant__ CUtensorMap tm_pb, const double* __restrict__ sf,
                     const double* __restrict__ pb, Dom d,
                     const __grid_constant__ WaveArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const SlabGeom G = slab_geom(TX, d.nz);
    const int NS = a.ns;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NS * G.stage);
    uint64_t* empty = full + NS;
    int* slot_item = reinterpret_cast<int*>(empty + NS); // work item of each slot (-1: stop)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int units = a.nstrips * a.nchunks;
    const int per_step = a.gtasks + units;
    const long long total = (long long)per_step * a.nsteps;
    const int last = a.nchunks - 1;

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
        // ---------------- producer: work list, dependency waits, TMA ----------------
        if (lane == 0) {
            uint32_t L = 0;
            long long seen = -1; // the step whose neighbour flags this producer has seen
            for (;;) {
                const int item = atomicAdd(&a.sched[0], 1);
                const bool stop = item >= total;
                int s = 0, r = 0;
                if (!stop) {
                    s = item / per_step;
                    r = item % per_step;
                }
                // ghost-row task of step s: rows 0, 1, ny, ny+1 of step s-1 done
                // (and, decomposed, the neighbours' step s-1: far slots, corners)
                if (!stop && r < a.gtasks) {
                    if (s > 0) {
                        wait_geq(&a.chunk_done[0], s * a.nstrips);
                        wait_geq(&a.chunk_done[last], s * a.nstrips);
                        wait_geq(a.ghost_done, s * a.gtasks);
                    }
                    const Halo& hs = (s & 1) ? a.h_odd : a.h_even;
                    if (hs.active) {
                        Halo hw = hs;
                        hw.step = hs.step + s;
                        halo_wait(hw, 0xF);
                    }
                }
                int ja = 0, jb = -1, ic = 0;
                if (!stop && r >= a.gtasks) {
                    const int unit = r - a.gtasks;
                    const int ch = unit / a.nstrips, st = unit % a.nstrips;
                    ja = ch * a.chunk + 1;
                    jb = min(d.ny, ja + a.chunk - 1);
                    ic = a.fp + 1 + st * TX - 2;
                    if (s > 0) {
                        if (ch > 0) wait_geq(&a.chunk_done[ch - 1], s * a.nstrips);
                        wait_geq(&a.chunk_done[ch], s * a.nstrips);
                        if (ch < last) wait_geq(&a.chunk_done[ch + 1], s * a.nstrips);
                        if (ch == 0 || ch == last) wait_geq(a.ghost_done, s * a.gtasks);
                    }
                    // decomposed: a unit on the subdomain rim reads halo slots the
                    // neighbour pushed in its step s-1 and pushes into slots it read
                    // then -- wait until that neighbour has finished step s-1
                    const Halo& hs = (s & 1) ? a.h_odd : a.h_even;
                    const int mask = rim_unit(d, 1 + st * TX, TX, ja, jb);
                    if (hs.active && mask) {
                        Halo hw = hs;
                        hw.step = hs.step + s;
                        halo_wait_once(hw, mask, seen);
                    }
                    // generic-proxy writes of other CTAs -> this CTA's TMA reads
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                }
                const bool cmd = stop || r < a.gtasks; // a slot without data
                const CUtensorMap* tm = (s & 1) ? &tm_e1 : &tm_e0;
                // odd chunks load (and compute) their rows bottom-up: the rows two
                // neighbouring chunks share are then read by both at about the same
                // time (both units' starts, or both ends), while L2 still holds them
                const bool down = !cmd && wave_rows_down(a, r - a.gtasks);
                for (int t = 0; cmd ? t == 0 : t <= jb - ja + 2; ++t, ++L) {
                    const int jj = down ? jb + 1 - t : ja - 1 + t;
                    const uint32_t slot = L % NS;
                    if (L >= (uint32_t)NS) mbar_wait(&empty[slot], ((L / NS) - 1) & 1);
                    slot_item[slot] = stop ? -1 : item;
                    if (cmd) {
                        mbar_arrive(&full[slot]); // no bytes: a command slot
                        ++L;
                        break;
                    }
                    unsigned char* stg = smem + (size_t)slot * G.stage;
                    mbar_expect_tx(&full[slot], G.tx_bytes);
                    tma_load_3d(stg, tm, &full[slot], ic, a.jrow0 + jj, 0);
                    tma_load_2d(stg + G.e_bytes, &tm_sf, &full[slot], ic, a.jrow0 + jj);
                    tma_load_2d(stg + G.e_bytes + G.r_bytes, &tm_pb, &full[slot], ic, a.jrow0 + jj);
                }
                if (stop) break;
            }
        }
        __syncwarp();
    } else {
        wave_consumers<TX, NCW, PHYS>(smem, G, full, empty, slot_item, sf, pb, d, a);
    }
    // every warp of this CTA is done (consumers have published their units):
    // the last CTA to finish re-arms the scheduler and the counters
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&a.sched[1], 1) == (int)gridDim.x - 1) {
            for (int c = 0; c < a.nchunks; ++c) a.chunk_done[c] = 0;
            *a.ghost_done = 0;
            if (a.h_even.active)
                for (int t = 0; t < a.nsteps; ++t) a.step_done[t] = 0;
            a.sched[0] = 0;
            a.sched[1] = 0;
            __threadfence();
        }
    }
}

} // namespace hftw
