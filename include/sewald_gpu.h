/*
 * sewald_gpu.h — C-ABI of the B200-native Spectral Ewald engine.
 *
 * Plain C: pointers, sizes, POD structs. No torch/CUDA types in signatures
 * (streams are passed as void*). Every entry point returns an int status
 * (SEWALD_OK = 0) and leaves a message in sewald_gpu_last_error(ctx) or
 * sewald_last_error() for the context-free calls.
 *
 * Each entry point replaces one function of the reference C++ library
 * (/root/reference/proj/include/sewald/...); the mapping is cited per call.
 * Coordinates and strengths are AoS fp64, 3 doubles per point — exactly
 * reinterpret_cast<const double*>(std::vector<std::array<double,3>>::data())
 * of the reference's Vec3 vectors (domain.h:11, :52-70), so a C++ caller
 * passes its vectors zero-copy.
 */
#ifndef SEWALD_GPU_H
#define SEWALD_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. The drop-in C++ layer rethrows them as the reference's
 * exception types (std::invalid_argument / std::domain_error /
 * std::runtime_error), throw sites in /root/reference/proj/src. */
enum {
    SEWALD_OK = 0,
    SEWALD_EINVAL = 1,   /* std::invalid_argument */
    SEWALD_EDOMAIN = 2,  /* std::domain_error */
    SEWALD_ERUNTIME = 3, /* std::runtime_error */
    SEWALD_ECUDA = 4,
    SEWALD_ECUFFT = 5,
    SEWALD_ENOMEM = 6
};

/* enum class Kernel (domain.h:26) */
enum { SEWALD_STOKESLET = 0, SEWALD_STRESSLET = 1, SEWALD_ROTLET = 2 };
/* enum class WindowKind (window.h:9) */
enum { SEWALD_WIN_KB = 0, SEWALD_WIN_PKB = 1, SEWALD_WIN_TG = 2 };

/* POD mirror of EwaldParams (estimates.h:62-71) flattened with its
 * GridSpec (grid.h:13-24), WindowSpec (window.h:15-29) and UpsamplingPlan
 * (grid.h:29-35). */
typedef struct sewald_params_c {
    int32_t kind;
    int32_t d;
    double xi;
    double rc;
    double R;
    /* GridSpec */
    double h;
    int32_t M[3];
    int32_t M_ext[3];
    double L[3];
    double L_ext[3];
    double pad[3];
    int32_t f_m;
    /* WindowSpec */
    int32_t win_kind;
    int32_t P;
    double win_h;
    double beta;
    int32_t nu;
    double alpha;
    /* UpsamplingPlan */
    double s0;
    double s_star;
    int32_t k_star[3];
    double s0_raw;
    double s_star_raw;
} sewald_params_c;

/* POD mirror of EstimateReport (estimates.h:73-90). */
typedef struct sewald_report_c {
    double tau_abs, U, kinf, fourier_trunc, realspace_trunc, window_err, h_estimate;
    int32_t P_estimate;
    double h_target;
    int32_t P_target;
    int32_t rc_clamped, kinf_clamped, window_saturated, tg_support_from_pkb;
} sewald_report_c;

/* Per-call stage timings (CUDA events, milliseconds) of the last pipeline run. */
typedef struct sewald_timings_c {
    double h2d_ms, sort_ms, spread_ms, fft_fwd_ms, scale_ms, fft_inv_ms, gather_ms,
        realspace_ms, assemble_ms, d2h_ms, total_ms;
    int64_t kernel_launches;
    int64_t realspace_pairs;     /* accepted pairs (if counted), else -1 */
} sewald_timings_c;

typedef struct sewald_gpu_ctx sewald_gpu_ctx;

/* ---- host-side parameter layer (no GPU needed) ---------------------- */

/* select_parameters (estimates.h:106-107, estimates.cpp:211-268). */
int sewald_select_parameters(int kind, int d, const double L[3], double Q, double xi,
                             double tol_value, int tol_relative, int f_m, int window_kind,
                             int pollution_fix, sewald_params_c* out, sewald_report_c* report);

/* WindowSpec::make (window.cpp:76-86) into p->win_* fields. */
int sewald_window_make(int window_kind, int P, double h, sewald_params_c* p);

/* build_grid (grid.h:38, grid.cpp:35-77) into p's grid fields. */
int sewald_build_grid(const double L[3], int d, double h_target, int P, int kind, int f_m,
                      sewald_params_c* p);

/* pkb_build (window.cpp:112-138): P*(nu+1) coefficients, row l+P/2. */
int sewald_pkb_coefficients(const sewald_params_c* p, double* coef_out);

/* Window::eval1d / hat1d (window.cpp:171-182), host evaluation for tests. */
int sewald_window_eval(const sewald_params_c* p, const double* r, int64_t n, double* out);
int sewald_window_hat(const sewald_params_c* p, const double* k, int64_t n, double* out);

/* Q = source_quantity (domain.cpp:53-62). */
double sewald_source_quantity(int kind, const double* f, const double* nu, int64_t N);

const char* sewald_last_error(void);

/* ---- device context -------------------------------------------------- */

int sewald_gpu_create(int device, sewald_gpu_ctx** out);
void sewald_gpu_destroy(sewald_gpu_ctx* ctx);
const char* sewald_gpu_last_error(const sewald_gpu_ctx* ctx);
/* Run all work on this cudaStream_t (NULL = the legacy default stream). A new
 * context uses its own non-blocking stream until this is called. */
int sewald_gpu_set_stream(sewald_gpu_ctx* ctx, void* stream);
int sewald_gpu_get_timings(const sewald_gpu_ctx* ctx, sewald_timings_c* out);
/* 1 = record per-stage CUDA events (adds event overhead), 0 = off. */
int sewald_gpu_set_profiling(sewald_gpu_ctx* ctx, int enabled);

/* Pinned host memory of the context (>= bytes, valid until the next call
 * with a larger size or sewald_gpu_destroy): passed as the u_out of the
 * host-buffer entry points it receives the result by DMA without staging.
 * The C++ drop-in uses it to overlap the allocation of its returned vector
 * with the device work. */
int sewald_gpu_host_buffer(sewald_gpu_ctx* ctx, size_t bytes, void** out);

/* Cumulative number of engine kernels launched on this context. */
int64_t sewald_gpu_launch_count(const sewald_gpu_ctx* ctx);

/* Measured fp64 FMA-pipe throughput of this device in TFLOP/s (DFMA
 * microbenchmark; roofline denominator for the fp64-bound kernels). */
int sewald_gpu_fp64_peak(sewald_gpu_ctx* ctx, double* tflops);

/* ---- kernel-choice switches (process-wide; diagnostics and tests) ------
 * Defaults are the measured best and come from the SEWALD_* environment
 * variables DESIGN.md §6b lists; setting one makes later calls on every
 * context use it (sessions rebuild their orderings). Not part of the
 * reference API: the reference has one CPU code path per stage. */
enum {
    SEWALD_OPT_RS_SYM = 0,        /* real space, targets == sources: 0 never pair-symmetric,
                                     1 auto (large target sets), 2 always */
    SEWALD_OPT_GATHER = 1,        /* -1 auto, 0 warp per target, 1 z-sweep, 2 tiles */
    SEWALD_OPT_GATHER_MMA = 2,    /* tiled gather: 1 tensor-core form (P <= 16), 0 CUDA-core form */
    SEWALD_OPT_GATHER_L = 3,      /* tiled gather region edge: 0 auto, 15, 19, 23 or 31 */
    SEWALD_OPT_SPREAD_SWEEP = 4,  /* -1 auto (P <= 24), 0 off, 1 on */
    SEWALD_OPT_SPREAD_MMA = 5,    /* 1 tensor-core spread for 15 <= P <= 32, 0 off */
    SEWALD_OPT_SPREAD_MMA_L = 6,  /* tensor-core spread region edge for P <= 20: 23 or 19 */
    SEWALD_OPT_SPREAD_CACHED = 7, /* tensor-core spread: 1 staged tables per chunk, 0 per group */
    SEWALD_OPT_SPREAD_ROWSWEEP = 8, /* tensor-core spread, P <= 20: 1 row-sweep CTAs (several per SM) */
    SEWALD_OPT_SPREAD_FUSED = 9,  /* tensor-core spread tiles (3 components): 1 taps evaluated in the
                                     kernel, 0 read from a taps array written by a separate kernel */
    SEWALD_OPT_GATHER_WIDE = 10,  /* tensor-core gather tiles with the A fragments read from the grid into
                                     registers: 2 every width (default), 1 only 20 < P <= 32, 0 never
                                     (shared-memory region tiles for P <= 20, z-sweep above) */
    SEWALD_OPT_GATHER_FUSED = 11, /* register-A gather tiles: 1 taps evaluated in the kernel, 0 taps array */
    SEWALD_OPT_SPREAD_SORT = 12,  /* tensor-core spread tiles (P <= 20): 1 points of a tile ordered by their
                                     (x, y) stencil offset and MMA steps that cannot reach a row block
                                     skipped, 0 tile order only */
    SEWALD_OPT_GATHER_SORT = 13,  /* register-A gather tiles: the same ordering and skipping for targets */
    SEWALD_OPT_D0_YFUSED = 14,    /* D = 0 solve: 1 x transforms over the data rows only and the y transform,
                                     scale and inverse y transform fused in one kernel (padded y a power of
                                     two, 256..1024; default), 0 batched 2-D transforms + scale kernel; read
                                     when a session builds its D = 0 plan */
    SEWALD_OPT_COUNT = 15
};
int sewald_gpu_set_option(int which, int value);
int sewald_gpu_get_option(int which, int* value);

/* ---- multi-GPU context (one process, several GPUs of one node) --------
 * Replaces the reference's only parallel knob (realspace_potential's
 * n_threads, realspace.h:40-41) for callers without MPI/torch: the sources
 * are spread in 1/W slices, the grids summed over NVLink peer memory, and
 * each GPU evaluates 1/W of the targets. dev_ids may repeat a
 * device (tests on one GPU); distinct devices need peer access (ECUDA
 * otherwise). Arguments and results as sewald_gpu_full_potential. */
typedef struct sewald_gpu_multi sewald_gpu_multi;
int sewald_gpu_multi_create(int n_gpus, const int* dev_ids, sewald_gpu_multi** out);
void sewald_gpu_multi_destroy(sewald_gpu_multi* m);
const char* sewald_gpu_multi_last_error(const sewald_gpu_multi* m);
int sewald_gpu_multi_size(const sewald_gpu_multi* m);
/* The single-device context of member d (e.g. for sewald_gpu_set_table0p). */
sewald_gpu_ctx* sewald_gpu_multi_context(sewald_gpu_multi* m, int d);
int sewald_gpu_multi_full_potential(sewald_gpu_multi* m, const sewald_params_c* p, const double* x,
                                    const double* f, const double* nu, int64_t N, const double* xt, int64_t Nt,
                                    int same_as_sources, int precompute_0p, double* u_out);
int sewald_gpu_multi_fourier_potential(sewald_gpu_multi* m, const sewald_params_c* p, const double* x,
                                       const double* f, const double* nu, int64_t N, const double* xt, int64_t Nt,
                                       int same_as_sources, int precompute_0p, double* u_out);

/* ---- host-buffer entry points (drop-in path) ------------------------- */
/* x, f: N*3 doubles; nu: N*3 (stresslet) or NULL; xt: Nt*3. When
 * same_as_sources != 0 the targets are the sources (xt may be NULL or x).
 * u_out: Nt*3 doubles (host). */

/* full_potential (realspace.h:46-47, realspace.cpp:205-219). */
int sewald_gpu_full_potential(sewald_gpu_ctx* ctx, const sewald_params_c* p, const double* x,
                              const double* f, const double* nu, int64_t N, const double* xt,
                              int64_t Nt, int same_as_sources, int precompute_0p, double* u_out);

/* se_fourier_potential (fourier.h:81-82, fourier.cpp:805-852). */
int sewald_gpu_fourier_potential(sewald_gpu_ctx* ctx, const sewald_params_c* p,
                                 const double* x, const double* f, const double* nu, int64_t N,
                                 const double* xt, int64_t Nt, int same_as_sources,
                                 int precompute_0p, double* u_out);

/* realspace_potential (realspace.h:40-41, realspace.cpp:166-203). */
int sewald_gpu_realspace_potential(sewald_gpu_ctx* ctx, int kind, int d, const double L[3],
                                   const double* x, const double* f, const double* nu, int64_t N,
                                   const double* xt, int64_t Nt, int same_as_sources, double xi,
                                   double rc, int starred, double* u_out);

/* spread (fourier.h:59, fourier.cpp:237-274): grid_out = C * prod(M_ext)
 * doubles, component-major, last axis fastest (RealField layout, fourier.h:15-28). */
int sewald_gpu_spread(sewald_gpu_ctx* ctx, const sewald_params_c* p, const double* x,
                      const double* f, const double* nu, int64_t N, double* grid_out);

/* gather (fourier.h:71-72, fourier.cpp:276-309): grid = 3 * prod(M_ext). */
int sewald_gpu_gather(sewald_gpu_ctx* ctx, const sewald_params_c* p, const double* grid,
                      const double* xt, int64_t Nt, double* u_out);

/* ---- reference stage functions (fourier.h:59-74) -------------------- */
/* FourierField (fourier.h:30-46) travels as this geometry plus three complex
 * arrays of interleaved (re, im) doubles — the memory of the reference's
 * std::vector<std::complex<double>> far / near / zero, so a C++ caller
 * passes them zero-copy:
 *   far  [comps][prod M_ext]                        (d = 1, 2, 3)
 *   zero [comps][n_zero block]                      (d = 0: the whole s0-padded box)
 *   near [comps][n_near_rows][n_near block]         (d = 1, 2)
 * The per-row blocks are n_zero[1]*n_zero[2] (d = 1) or n_zero[2] (d = 2),
 * likewise for near. *_len are complex element counts over all comps. */
typedef struct sewald_fourier_geom_c {
    int32_t d, comps;
    int32_t n_per[3], n_far[3], n_near[3], n_zero[3];
    int32_t n_near_rows;
    int64_t far_len, near_len, zero_len;
} sewald_fourier_geom_c;

/* POD mirror of ModifiedKernelSpec (modified_kernels.h:10-21). */
typedef struct sewald_modspec_c {
    int32_t kind, d;
    double R, a_B, b_B, ell_H, ell_B, c_B;
} sewald_modspec_c;

/* ModifiedKernelSpec::optimal (modified_kernels.cpp:52-63). */
int sewald_modspec_optimal(int kind, int d, double R, sewald_modspec_c* out);

/* Geometry aft_forward produces for a comps-component field on p's grid and
 * upsampling plan (p->s0, p->s_star, p->k_star; the D = 0 precomputed-kernel
 * pipeline sets p->s0 = 2, fourier.cpp:819-821). near_rows_out (may be NULL)
 * receives n_near_rows ints: classify_rows (fourier.cpp:101-125). Host only. */
int sewald_aft_geometry(const sewald_params_c* p, int comps, sewald_fourier_geom_c* g,
                        int32_t* near_rows_out);

/* aft_forward (fourier.h:61, fourier.cpp:311-416): field = g->comps *
 * prod(M_ext) doubles (RealField layout); g must equal sewald_aft_geometry's.
 * Unused arrays (e.g. near / zero for d = 3) may be NULL. */
int sewald_gpu_aft_forward(sewald_gpu_ctx* ctx, const sewald_params_c* p, const double* field,
                           const sewald_fourier_geom_c* g, double* far, double* near, double* zero);

/* aft_inverse (fourier.h:62, fourier.cpp:418-520): field_out = g->comps *
 * prod(M_ext) doubles. near_rows: g->n_near_rows ints (the field's own). */
int sewald_gpu_aft_inverse(sewald_gpu_ctx* ctx, const sewald_params_c* p,
                           const sewald_fourier_geom_c* g, const int32_t* near_rows,
                           const double* far, const double* near, const double* zero,
                           double* field_out);

/* scale (fourier.h:66-67, fourier.cpp:522-666): the output field has the
 * geometry g with comps = 3 (the stresslet contracts nine to three). The
 * window is p's (its h must equal the grid's, fourier.cpp:155-158). */
int sewald_gpu_scale(sewald_gpu_ctx* ctx, const sewald_params_c* p, const sewald_modspec_c* spec,
                     double xi, const sewald_fourier_geom_c* g, const int32_t* near_rows,
                     const double* far, const double* near, const double* zero, double* far_out,
                     double* near_out, double* zero_out);

/* scale with a PrecomputedKernel0P (fourier.h:68-69, fourier.cpp:668-720):
 * table = prod(table_n) complex (interleaved); d = 0 only. */
int sewald_gpu_scale_table(sewald_gpu_ctx* ctx, const sewald_params_c* p, int kind,
                           const int32_t table_n[3], const double* table, double xi,
                           const sewald_fourier_geom_c* g, const double* zero, double* zero_out);

/* precompute_0p (fourier.h:74, fourier.cpp:722-803): n_out = 2 M_ext;
 * table_out = prod(n_out) complex (interleaved), or NULL to query n_out. */
int sewald_gpu_precompute_0p(sewald_gpu_ctx* ctx, const sewald_params_c* p, int kind, double R,
                             int32_t n_out[3], double* table_out);

/* SePipelineOptions::table (fourier.h:76-79): install a caller-built D = 0
 * kernel table (precompute_0p layout, prod(n) interleaved complex, host or
 * device memory) for the pipelines run with parameters p on this context;
 * table == NULL goes back to the engine's own table. n must be 2 M_ext
 * (the table path pads with s0 = 2). Passing the same pointer again skips
 * the upload. */
int sewald_gpu_set_table0p(sewald_gpu_ctx* ctx, const sewald_params_c* p, const int32_t n[3],
                           const double* table);

/* ---- device-resident session (time stepping / multi-GPU plumbing) ---- */
/* A session keeps sources, targets, sort permutations, grids and cuFFT plans
 * resident in HBM between calls. All pointers given to *_dev calls are
 * device pointers on the context's device; work is ordered on the context
 * stream. This is the layer bench.py times as `value` and the multi-GPU
 * driver composes with torch.distributed collectives. */
typedef struct sewald_gpu_session sewald_gpu_session;

int sewald_gpu_session_create(sewald_gpu_ctx* ctx, const sewald_params_c* p,
                              sewald_gpu_session** out);
void sewald_gpu_session_destroy(sewald_gpu_session* s);
/* Sources: device AoS arrays (N*3). Copied into session-owned sorted storage. */
int sewald_gpu_session_set_sources(sewald_gpu_session* s, const double* x_dev,
                                   const double* f_dev, const double* nu_dev, int64_t N);
/* Targets: device AoS (Nt*3); same_as_sources uses the sources. */
int sewald_gpu_session_set_targets(sewald_gpu_session* s, const double* xt_dev, int64_t Nt,
                                   int same_as_sources);
/* Number of doubles of the spread grid (C * prod M_ext). */
int64_t sewald_gpu_session_grid_size(const sewald_gpu_session* s);
/* Spread sources [i0, i1) (in the caller's original order) into grid_dev
 * (zeroed first). grid_dev may be NULL to use the session's own grid. */
int sewald_gpu_session_spread(sewald_gpu_session* s, int64_t i0, int64_t i1, double* grid_dev);
/* Forward transform, k-space scaling, inverse transform: grid_dev (C comps)
 * -> session flow field (3 comps). precompute_0p selects the D=0 table path. */
int sewald_gpu_session_solve(sewald_gpu_session* s, const double* grid_dev, int precompute_0p);
/* Evaluate the targets of part `part` of `nparts` cluster-aligned contiguous
 * slices of the session's internal (cell-sorted, hence spatially compact)
 * target order. u_dev holds Nt*3 doubles in the caller's original target
 * order. With nparts == 1 it receives the full result. With nparts > 1 (or
 * when the pair-symmetric real-space sum is used, targets == sources) the
 * whole array is zeroed first and this part's contributions are
 * accumulated, so per-rank outputs combine with a sum all-reduce. `parts` bit mask:
 * 1 = Fourier (gather of the solved flow), 2 = real space, 4 = self /
 * zero-mode / gauge terms. */
int sewald_gpu_session_evaluate(sewald_gpu_session* s, int part, int nparts, int parts,
                                double* u_dev);
/* ---- slab-distributed D = 0 / D = 3 solve (one rank of `world`) -
 * D = 3 runs the same stages on the unpadded periodic box (n = M) with the
 * periodic operator (G(0) = 0) in place of the free-space one. */
/* ---- (D = 0 details) ------------------------------------------------------
 * Replaces se_fourier_potential's single-box transform (fourier.cpp:311-520,
 * :668-720) by x-slabs of the M_ext box for the z transforms and kz-slabs of
 * the half spectrum for the (x, y) transforms and the scale, with two
 * all-to-all exchanges done by the caller (NCCL). Bounds arrays hold world+1
 * split points (x over m[0], kz over h2). Buffer layouts (complex doubles):
 *   forward send chunk q: [C][xb-xa][m1][kz in q]     (sum over q = C*(xb-xa)*m1*h2)
 *   middle  recv chunk p: [C][x in p][m1][kb-ka]     -> send chunk q: [3][kb-ka][x in q][m1]
 *   inverse recv chunk p: [3][kz in p][xb-xa][m1]    -> flow slab [3][xb-xa][m1][m2] (real)
 * The grid slab passed to forward is [C][xb-xa][m1][m2] (real). */
int sewald_gpu_session_d0_geometry(sewald_gpu_session* s, int precompute_0p, int m[3], int n[3], int* h2,
                                   int* C);
int sewald_gpu_session_d0_forward(sewald_gpu_session* s, int precompute_0p, const double* grid_slab, int xa,
                                  int xb, int world, const int* kz_bounds, void* send_dev);
int sewald_gpu_session_d0_middle(sewald_gpu_session* s, int precompute_0p, const void* recv_dev, int world,
                                 const int* x_bounds, int ka, int kb, void* send_dev);
int sewald_gpu_session_d0_inverse(sewald_gpu_session* s, int precompute_0p, const void* recv_dev, int xa, int xb,
                                  int world, const int* kz_bounds, double* flow_slab_dev);
/* Session form of sewald_gpu_set_table0p. */
int sewald_gpu_session_set_table0p(sewald_gpu_session* s, const int32_t n[3], const double* table);
/* Install a full flow field (3 comps, M_ext, device) for evaluate()'s gather. */
int sewald_gpu_session_set_flow(sewald_gpu_session* s, const double* flow_dev);
/* Accepted real-space pairs counted since the last reset (synchronises). */
int64_t sewald_gpu_session_pair_count(sewald_gpu_session* s, int reset);
/* Whole pipeline on one GPU: spread all, solve, evaluate all (parts = 7). */
int sewald_gpu_session_run(sewald_gpu_session* s, int precompute_0p, double* u_dev);

/* ---- analytic oracles (SPEC.md module `reference`) ----
 * Slow, independently derived sums for validating the fast path (the
 * reference ships this module as a stub, proj/src/reference.cpp:1). Host
 * buffers in and out; sizes meant for validation (N * Nt * modes work).
 * Periodic sums run over k_i = 2 pi j / L_i, -kmax_i <= j <= kmax_i - 1
 * (PAPER.md:1117-1130), real part kept. */

/* direct_sum_0p: plain O(N Nt) bare-kernel
 * sum; starred skips n == t (Nt == N). A target on a source otherwise ->
 * SEWALD_EDOMAIN. */
int sewald_gpu_direct_sum_0p(sewald_gpu_ctx* ctx, int kind, const double* x, const double* f, const double* nu,
                             int64_t N, const double* xt, int64_t Nt, int starred, double* u_out);
/* direct_ewald_fourier_3p: the k != 0 Fourier
 * sum over the (2 kmax)^3 cube plus the stresslet zero mode. */
int sewald_gpu_ewald_fourier_3p(sewald_gpu_ctx* ctx, int kind, const double L[3], double xi, const int kmax[3],
                                const double* x, const double* f, const double* nu, int64_t N, const double* xt,
                                int64_t Nt, double* u_out);
/* fourier_reference_potential: d = 2
 * Appendix-A q-sums, d = 1 Appendix-B q-sums (gauge constants ell = 1), d = 3
 * forwards to sewald_gpu_ewald_fourier_3p. kmax has d entries. */
int sewald_gpu_fourier_reference_potential(sewald_gpu_ctx* ctx, int kind, int d, const double L[3], double xi,
                                           const int* kmax, const double* x, const double* f, const double* nu,
                                           int64_t N, const double* xt, int64_t Nt, double* u_out);
/* q2p / q2p_zero / q1p / q1p_zero pointwise: args = 3 per
 * point, (k1, k2, r3) for d = 2 or (k1, r2, r3) for d = 1; out = per point
 * 3 x C complex (re, im) entries [j][c], c = l (C = 3) or 3 l + m (stresslet,
 * C = 9). */
int sewald_gpu_qtensor(sewald_gpu_ctx* ctx, int kind, int d, int zero_mode, int64_t n, const double* args,
                       double xi, double* out);
/* Incomplete Bessel K_nu(a, b), nu = -1, 0, 1, 2 (PAPER.md Knu-def), device
 * quadrature used by the d = 1 oracle: out = 4 values per (a, b). */
int sewald_gpu_incomplete_bessel_k4(sewald_gpu_ctx* ctx, int64_t n, const double* a, const double* b,
                                    double* out);
/* rms_error / rel_rms_error: n targets, 3 doubles each;
 * SEWALD_EDOMAIN when rel_err is requested and u_ref is zero. */
int sewald_rms_error(const double* u, const double* u_ref, int64_t n, double* abs_err, double* rel_err);

#ifdef __cplusplus
}
#endif

#endif /* SEWALD_GPU_H */
