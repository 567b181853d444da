/* include/hftw.h -- C ABI of the B200-native minimal-weather timestep.
 *
 * This is the drop-in boundary for the reference's native weather simulator
 * (/root/reference/proj/include/hft/weather.hpp).  Each entry point names the
 * reference interface it replaces.  Plain pointers and sizes only: no torch,
 * no C++ types.  Exported from paper_1802_05839_b200/libhftw.so (nvcc, sm_100a).
 *
 * Conventions:
 *  - Every function returns 0 on success, a nonzero HFTW_E* code otherwise;
 *    hftw_last_error(ctx) (or hftw_last_error(NULL) for create failures)
 *    returns the message.  No exceptions cross the ABI.
 *  - Host buffers use the reference's unpadded LOGICAL column-major layout of
 *    hft::ArrayObject::data (interpreter.hpp:25-36): 3D fields over
 *    (0..nx+1, 0..ny+1, 1..nz), 2D fields over (0..nx+1, 0..ny+1)
 *    (weather.cpp:71,77).  One memcpy fills SimState::field.data.  Pinned host
 *    memory makes transfers run at full PCIe rate but is not required.
 *  - The library owns device memory, streams, tensor maps and graphs; the
 *    caller owns host buffers.  One host thread per context.
 *  - Arithmetic is bitwise identical to hft::reference_step: every kernel
 *    uses explicitly rounded IEEE double ops (__dadd_rn/__dmul_rn), i.e. no
 *    FMA contraction, and the reference's association order.
 */
#ifndef HFTW_H
#define HFTW_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HFTW_ABI_VERSION 1

/* Mirrors hft::GridConfig field for field (weather.hpp:26-35). */
typedef struct hftw_grid {
    int64_t nx, ny, nz;
    double timestep;
    double output_timestep;
    double diffusion_velocity;
    double radiation_intensity;
    double transfer_velocity;
    double surf_energy;
    double pbl_energy;
} hftw_grid;

/* The four SimState members (weather.hpp:39-46). */
enum hftw_field {
    HFTW_ENERGY = 0,
    HFTW_ENERGY_U = 1,
    HFTW_ENERGY_SURF = 2,
    HFTW_ENERGY_PBL = 3
};

/* Device storage order of 3D fields (BuildConfig::storage_order, config.hpp:41-43;
 * permutation semantics of unpermute_storage, weather.cpp:306-338):
 *   IJK = {1,2,3}: i fastest (the reference GPU default).
 *   KIJ = {3,1,2}: raw tuple (k,i,j), k fastest (the paper's CPU-friendly order). */
enum hftw_layout { HFTW_IJK = 0, HFTW_KIJ = 1 };

/* Step kernel selection (hftw_set_kernel).  AUTO picks the fastest valid one. */
enum hftw_kernel {
    HFTW_KERNEL_AUTO = 0,
    HFTW_KERNEL_FUSED_TMA = 1, /* fused physics+diffusion, TMA row-slab pipeline */
    HFTW_KERNEL_FUSED_CELL = 2, /* fused physics+diffusion, one cell per thread */
    HFTW_KERNEL_SPLIT = 3,      /* reference structure: physics pass, then diffusion pass */
    HFTW_KERNEL_FUSED_PAIR = 4  /* two fused steps per pass over HBM (the intermediate field
                                   stays on chip), single-step TMA launches for the rest */
};

enum hftw_error {
    HFTW_OK = 0,
    HFTW_EINVAL = 1,   /* invalid argument or grid (validate() failed) */
    HFTW_ECUDA = 2,    /* CUDA runtime/driver error */
    HFTW_ENOMEM = 3,   /* device allocation failed */
    HFTW_ESTATE = 4,   /* call not valid in the current context state */
    HFTW_EUNSUP = 5    /* unsupported combination (e.g. TMA kernel with nz > 256) */
};

typedef struct hftw_ctx hftw_ctx;

/* ABI version of the loaded library (HFTW_ABI_VERSION). */
int hftw_abi_version(void);

/* hft::validate (weather.hpp:37, weather.cpp:24-41).  Returns 0 when valid,
 * HFTW_EINVAL otherwise with the reference's diagnostics, one per line, in
 * msg (truncated to cap). */
int hftw_validate(const hftw_grid* grid, char* msg, size_t cap);

/* Create a context for `grid` on CUDA device `device` with the given storage
 * layout.  Fields are allocated but undefined until hftw_init/hftw_upload. */
int hftw_create(const hftw_grid* grid, int layout, int device, hftw_ctx** out);

/* Release everything the context owns. NULL is accepted. */
void hftw_destroy(hftw_ctx* ctx);

/* hft::reference_init (weather.hpp:48-51, weather.cpp:67-99), on the device. */
int hftw_init(hftw_ctx* ctx);

/* Host -> device copy of one field from its logical column-major buffer. */
int hftw_upload(hftw_ctx* ctx, int field, const double* host);

/* Device -> host copy of one field into its logical column-major buffer.
 * Synchronous with respect to the context stream. */
int hftw_download(hftw_ctx* ctx, int field, double* host);

/* nsteps x hft::reference_step (weather.hpp:53-55, weather.cpp:101-171),
 * asynchronous on the context stream.  After the call ENERGY holds the new
 * field and ENERGY_U the post-physics, pre-diffusion field of the last step,
 * exactly as after the reference's buffer swap (weather.cpp:170). */
int hftw_step(hftw_ctx* ctx, int64_t nsteps);

/* hft::reference_step (weather.hpp:53-55) on a HOST SimState, end to end:
 * energy/energy_surf/energy_pbl are the state before the step (logical
 * column-major host arrays); energy_out and energy_u_out receive SimState's
 * energy and energy_u after it.  energy_out may alias energy (in-place, as
 * the reference mutates its SimState); energy_u_out must not alias the inputs.
 * Equivalent to upload x3 + hftw_step(1) + download x2, but pipelined in
 * row blocks so that PCIe H2D, the step kernels and PCIe D2H overlap.
 * Synchronous; afterwards the context holds the stepped state.  If it fails
 * part-way, all copies have stopped when it returns and the device state is
 * undefined: later calls fail with HFTW_ESTATE until hftw_init or an upload of
 * all four fields.  A group context runs the same calls in sequence. */
int hftw_step_host(hftw_ctx* ctx, const double* energy, const double* energy_surf,
                   const double* energy_pbl, double* energy_out, double* energy_u_out);

/* Page-lock (and unlock) host memory the caller owns, e.g. the four
 * std::vector buffers of a SimState, so that hftw_step_host / upload /
 * download move it at PCIe speed: pageable buffers go through the driver's
 * bounce buffer (ASUCA reference_step: ~185 ms against ~41 ms pinned).  The
 * range must stay allocated until hftw_host_unregister. */
int hftw_host_register(void* ptr, size_t bytes);
int hftw_host_unregister(void* ptr);

/* Wait for all work queued on the context stream. */
int hftw_sync(hftw_ctx* ctx);

/* Error text of the last failing call (ctx may be NULL). */
const char* hftw_last_error(const hftw_ctx* ctx);

/* hft::run_reference (weather.hpp:57-59, weather.cpp:173-178) in one call:
 * create on `device`, init, steps, download the four fields into the caller's
 * buffers (any may be NULL), destroy. */
int hftw_run_reference(const hftw_grid* grid, int64_t steps, int device, double* energy,
                       double* energy_u, double* energy_surf, double* energy_pbl);

/* ---- measurement / configuration hooks (not part of the reference API) ---- */

/* Run the context's work on an external cudaStream_t (NULL = own stream). */
int hftw_set_stream(hftw_ctx* ctx, void* cuda_stream);
/* The cudaStream_t kernels are launched on. */
void* hftw_stream(hftw_ctx* ctx);
/* Select the step kernel (enum hftw_kernel). */
int hftw_set_kernel(hftw_ctx* ctx, int kernel);
/* Kernel actually used by hftw_step (resolves AUTO). */
int hftw_get_kernel(const hftw_ctx* ctx);

/* Scheduling options of hftw_step (results are bitwise the same for every
 * value; only the launch schedule changes).  The library reads no environment
 * variables: kernel choice and tiling depend on the grid, the device and these
 * calls only. */
enum hftw_option {
    HFTW_OPT_MULTISTEP = 1, /* single-step kernel, n >= 2 steps in ONE persistent launch:
                               -1 never, 0 where a step is short (default), 1 always */
    HFTW_OPT_PAIR = 2,      /* AUTO may use two-step passes: 1 (default) or 0 */
    HFTW_OPT_EXCHANGE = 3,  /* group contexts: 0 the step kernels push the halos (default);
                               1 the un-overlapped baseline -- steps without the halo
                               protocol, then a separate face-copy kernel per rank and
                               event waits (single-step kernels only; measurement) */
    HFTW_OPT_REVERSE = 4    /* 1: the pair and single-step kernels hand out their work
                               units in reverse order (last chunk first) -- the analogue
                               of the reference emulator's launch-order reversal
                               (interpreter.hpp:38-45), a race check: results must not
                               change.  0 (default): the j-major order */
};
int hftw_set_option(hftw_ctx* ctx, int option, int64_t value);

/* Measurement hook: when on, every step launch is bracketed by CUDA events on
 * the context stream.  hftw_get_timing returns the summed device time (ms)
 * and the number of launches of one launch kind since timing was switched
 * on: kind 0 = single-step kernels, 1 = two-step (pair) passes (one launch per
 * pass), 2 = multi-step (wavefront) launches of the single-step kernel's
 * tiling. */
int hftw_set_timing(hftw_ctx* ctx, int on);
/* steps (may be NULL): the timesteps those launches computed. */
int hftw_get_timing(hftw_ctx* ctx, int kind, double* ms, int64_t* launches, int64_t* steps);

/* Phase 1 alone (weather.cpp:118-128): in-place column physics on ENERGY.
 * mode 0 = one column per thread with the k loop in registers (the
 * reference's emitted GPU mapping, emit_cuda.cpp:159-214; coalesced in IJK,
 * strided in KIJ), 1 = layout-aware mapping (IJK: i across threads along
 * each (j,k) row; KIJ: one column per warp, lanes along k).  Leaves
 * ENERGY_U untouched. */
int hftw_physics(hftw_ctx* ctx, int mode);
/* Phases 2-5 alone (weather.cpp:130-168): ENERGY <- diffusion(ENERGY), with
 * ENERGY_U receiving the previous ENERGY (the swap of weather.cpp:170). */
int hftw_diffuse(hftw_ctx* ctx);
/* n diffusion-only sweeps (n x hftw_diffuse, bitwise): one persistent launch
 * whose sweeps overlap as a wavefront (the multi-step schedule of hftw_step). */
int hftw_diffuse_steps(hftw_ctx* ctx, int64_t n);

/* Measurement hook: overwrite `bytes` of scratch device memory on the context
 * stream (evicts the L2 between timed sweeps) with the same shared-memory
 * configuration as the step kernel, so no carveout change is timed. */
int hftw_flush_l2(hftw_ctx* ctx, size_t bytes);

/* Algorithmic HBM bytes of one call: what = 0 full step, 1 physics, 2 diffusion
 * (16 B per stored cell + 16 B per column for a step). */
double hftw_algorithmic_bytes(const hftw_ctx* ctx, int what);
/* Number of kernel launches one hftw_step(ctx, 1) enqueues. */
int hftw_launches_per_step(const hftw_ctx* ctx);

/* Raw device view of a field for zero-copy interop: base pointer of logical
 * (i=0, j=0, k=1) and element strides (si, sj, sk); sk = 0 for 2D fields.
 * The view is writable: any request first materialises ENERGY_U (so writes to
 * ENERGY_SURF / ENERGY_PBL through a view cannot change it) and, for a
 * decomposed rank, marks the halos stale (refilled by hftw_exchange).  The
 * ENERGY and ENERGY_U pointers swap after every step (ping-pong store): take
 * a fresh view after hftw_step. */
int hftw_field_view(hftw_ctx* ctx, int field, void** dptr, int64_t strides[3]);

/* ---- output path ----------------------------------
 * The corpus driver's time loop (fixtures/corpus/simple_weather.h90:74-108,
 * driven by weather.cpp:364-376): time = start; loop { if modulo(time +
 * 0.001, output_timestep) < 0.01 then write_data(energy, "energy", time);
 * step; time = time + timestep; if time > end_time: stop }.  modulo is
 * a - floor(a/p)*p (interpreter.cpp:109).  Each output is snapshotted on the
 * device and copied to a pinned host ring on a separate stream while the
 * following steps run; `write` receives the field as a logical column-major
 * buffer that is valid only during the call (interpreter.hpp:68-69
 * on_write_data).  Single-domain contexts only. */
typedef void (*hftw_write_fn)(void* user, const char* tag, double time, const double* field);
int hftw_simulate(hftw_ctx* ctx, double start_time, double end_time, double timestep,
                  double output_timestep, hftw_write_fn write, void* user, int64_t* steps_done,
                  int64_t* writes_done);

/* ---- multi-GPU: 2D horizontal (I x J) decomposition, one process per GPU ----
 *
 * The paper's ASUCA decomposition, not implemented by the
 * reference: full k columns per rank, px x py ranks, rank =
 * ry * px + rx.  Rank r of p owns inner indices 1 + floor(r*n/p) ..
 * floor((r+1)*n/p); rank 0 also owns ghost 0 and rank p-1 ghost n+1.  The
 * cyclic ghost rules (weather.cpp:152-168) become a torus: each rank pushes its
 * first/last inner column and row of every new field into the neighbours'
 * halo slots (pre-physics values; physics of halo cells is recomputed from
 * static sf/pb halos), and a per-direction step flag orders the pushes.  The
 * result is bitwise identical to the single-domain run. */
enum hftw_dir { HFTW_W = 0, HFTW_E = 1, HFTW_S = 2, HFTW_N = 3 };
enum hftw_diag { HFTW_SW = 0, HFTW_SE = 1, HFTW_NW = 2, HFTW_NE = 3 };

typedef struct hftw_plan {
    int32_t px, py, rx, ry, rank;
    int64_t gi0, gj0;            /* global index of local i = 0 / j = 0 */
    int64_t lnx, lny;            /* owned inner extents */
    int32_t own_w, own_e, own_s, own_n; /* owns the global ghost column / row */
    int32_t wfar, efar, sfar, nfar;     /* local index of a ghost cell's cyclic partner */
    int32_t nbr[4];              /* neighbour rank per hftw_dir, -1 = cyclic partner is local */
    int32_t send_slot[4];        /* my face lands in the neighbour at this local column (W/E) or row (S/N) */
    int64_t face_lo[4], face_hi[4]; /* local range along each face (j for W/E, i for S/N) */
    /* two-step (pair) passes read 2-deep halos: */
    int32_t depth[4];            /* layers my face sends (and receives): 2 to an interior
                                    neighbour, 1 to a wrap partner (its far slot), 0 none */
    int32_t diag[4];             /* diagonal neighbour SW, SE, NW, NE (-1: none); it gets my
                                    corner cell (1,1) / (nx,1) / (1,ny) / (nx,ny) column */
    int32_t diag_slot[4][2];     /* (i, j) where that corner column lands in it */
} hftw_plan;

/* Host-only (no GPU needed): the plan of `rank` in a px x py decomposition. */
int hftw_plan_rank(const hftw_grid* grid, int px, int py, int rank, hftw_plan* out);

/* Create the context of one rank's subdomain on `device`.  Host buffers of
 * upload/download stay GLOBAL logical arrays; a rank reads/writes only the
 * cells it owns.  Peers must be connected before init/upload/step. */
int hftw_create_dist(const hftw_grid* grid, int layout, int device, int px, int py, int rank,
                     hftw_ctx** out);
/* Bytes of this rank's exported peer descriptor (CUDA IPC handles + geometry). */
size_t hftw_peer_desc_size(void);
/* Export this rank's descriptor into `desc` (hftw_peer_desc_size() bytes). */
int hftw_peer_export(hftw_ctx* ctx, void* desc);
/* Map the neighbours: `all` holds every rank's descriptor back to back in rank order. */
int hftw_peer_connect(hftw_ctx* ctx, const void* all, int world);
/* Push the current energy and the static sf/pb faces to the neighbours'
 * halo slots and wait for completion.  The caller brackets it with a
 * process barrier (after every rank's upload/init, before the next step). */
int hftw_exchange(hftw_ctx* ctx);
/* This rank's plan. */
int hftw_get_plan(const hftw_ctx* ctx, hftw_plan* out);

/* ---- multi-GPU from ONE host process ("multi-GPU fan-out is
 * internal") ------------------------------------------------------------------
 * A group context owns px*py rank subdomains, rank r on CUDA device
 * devices[r] (devices == NULL: rank r on device r).  The ranks exchange halos
 * exactly as above (in-kernel pushes + step flags) through plain device
 * pointers: peer access is enabled between distinct devices (NVLink /
 * NVSwitch); ranks that share a device run on one stream, one launch per step
 * in rank order (that is how a single GPU can run -- and test -- any
 * decomposition).  The handle works with every function of this header:
 * init/upload/download take GLOBAL logical host arrays, hftw_step runs all
 * ranks (halos are refilled automatically after init/upload), hftw_sync waits
 * for every device.  Results are bitwise identical to the single-domain run.
 * hftw_create_multi(grid, layout, 1, 1, devices, &ctx) is a one-rank group. */
int hftw_create_multi(const hftw_grid* grid, int layout, int px, int py, const int* devices,
                      hftw_ctx** out);
/* Ranks of a group context (1 for any other context). */
int hftw_group_size(const hftw_ctx* ctx);
/* Rank r's own context (owned by the group: valid until hftw_destroy(group);
 * for per-rank plans, timing and field views).  A plain context returns itself
 * for r = 0. */
int hftw_group_rank(hftw_ctx* ctx, int r, hftw_ctx** out);

#ifdef __cplusplus
}
#endif
#endif /* HFTW_H */
