// Device context, resident session and pipeline orchestration.
//
// Pipeline (fourier.cpp:805-852 + realspace.cpp:205-219), all on one stream:
//   sources -> [bucket by stencil tile, sort] -> spread (tiles)      -> grid
//   grid    -> cuFFT D2Z -> k-space scale (fused operator) -> Z2D    -> flow
//   targets -> [fold, cell sort] -> real space (cell rows) -> u  (=)
//   flow    -> gather (warp per target)                    -> u  (+=)
//   self / stresslet zero mode / gauge epilogue            -> u  (+=)
// Everything stays resident in HBM between calls; host-buffer entry points
// wrap a cached session with one H2D and one D2H copy.
#include "engine.h"
#include "host_params.h"
#include "aft_d0.h"
#include "options.h"

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <thread>

namespace sewald_b200 {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw EngineError(SEWALD_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void cufft_check(cufftResult r, const char* what) {
    if (r != CUFFT_SUCCESS)
        throw EngineError(SEWALD_ECUFFT, std::string(what) + ": cuFFT error " + std::to_string((int)r));
}

PinnedBuf::~PinnedBuf() {
    if (ptr) cudaFreeHost(ptr);
}

void* PinnedBuf::ensure(size_t n) {
    if (n <= bytes) return ptr;
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    bytes = 0;
    cuda_check(cudaMallocHost(&ptr, n), "pinned staging");
    bytes = n;
    return ptr;
}

namespace {

// memcpy on up to 8 host threads (pageable <-> pinned staging: one thread
// copies ~5-10 GB/s; a 1e6-point input array is 24 MB).
void parallel_memcpy(void* dst, const void* src, size_t n) {
    const size_t chunk = size_t(4) << 20;
    unsigned t = (unsigned)std::min<size_t>(8, (n + chunk - 1) / chunk);
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    t = std::max(1u, std::min(t, hw));
    if (t <= 1) {
        std::memcpy(dst, src, n);
        return;
    }
    std::vector<std::thread> th;
    for (unsigned k = 1; k < t; ++k)
        th.emplace_back([=] {
            const size_t a = n * k / t, b = n * (k + 1) / t;
            std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
        });
    std::memcpy(dst, src, n / t);
    for (auto& x : th) x.join();
}

bool is_pageable(const void* p) {
    cudaPointerAttributes a{};
    const cudaError_t e = cudaPointerGetAttributes(&a, p);
    cudaGetLastError();
    return e != cudaSuccess || a.type == cudaMemoryTypeUnregistered;
}

// A pageable host array is staged into pinned memory with parallel host
// copies so its H2D copy runs asynchronously at full link speed; pinned and
// device arrays are used as they are.
const double* stage_in(PinnedBuf& buf, const double* src, size_t count) {
    if (!src || count == 0 || !is_pageable(src)) return src;
    double* dst = static_cast<double*>(buf.ensure(sizeof(double) * count));
    parallel_memcpy(dst, src, sizeof(double) * count);
    return dst;
}

}  // namespace

HostFlags::~HostFlags() {
    if (p) cudaFreeHost(p);
}

int* HostFlags::get() {
    if (!p) {
        cuda_check(cudaMallocHost(reinterpret_cast<void**>(&p), sizeof(int) * 16), "pinned flags");
        std::memset(p, 0, sizeof(int) * 16);
    }
    return p;
}

DevBuf::~DevBuf() {
    if (ptr) cudaFree(ptr);
}

void* DevBuf::ensure(size_t n) {
    if (n <= bytes && ptr) return ptr;
    if (ptr) {
        cuda_check(cudaDeviceSynchronize(), "sync before realloc");
        cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
    }
    const size_t alloc = std::max<size_t>(n, 256);
    cudaError_t e = cudaMalloc(&ptr, alloc);
    if (e != cudaSuccess) {
        ptr = nullptr;
        throw EngineError(SEWALD_ENOMEM, std::string("cudaMalloc failed: ") + cudaGetErrorString(e));
    }
    bytes = alloc;
    return ptr;
}

struct FourierPlanD3 {
    int n[3];
    int C;
    cufftHandle fwd = 0, inv = 0;
    DevBuf spec;
    DevBuf tables;  // k0,k1,k2 (n0+n1+nh), what0, what1, what2
    KspaceTables kt{};
    ~FourierPlanD3() {
        if (fwd) cufftDestroy(fwd);
        if (inv) cufftDestroy(inv);
    }
};

namespace {

// ---- small kernels -------------------------------------------------------

__global__ void finite_check_kernel(const double* __restrict__ x, int64_t n, int* __restrict__ bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && !isfinite(x[i])) atomicExch(bad, 1);
}

constexpr int RED_BLOCKS = 256;
constexpr int RED_THREADS = 256;

// Per-block min/max of each coordinate (free-axis cell-list bounds).
__global__ void minmax_kernel(const double* __restrict__ x, int64_t N, double* __restrict__ part) {
    __shared__ double s[6][RED_THREADS];
    double v[6] = {1e300, 1e300, 1e300, -1e300, -1e300, -1e300};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x)
        for (int a = 0; a < 3; ++a) {
            v[a] = fmin(v[a], x[3 * i + a]);
            v[3 + a] = fmax(v[3 + a], x[3 * i + a]);
        }
    for (int a = 0; a < 6; ++a) s[a][threadIdx.x] = v[a];
    __syncthreads();
    for (int st = RED_THREADS / 2; st > 0; st >>= 1) {
        if ((int)threadIdx.x < st)
            for (int a = 0; a < 6; ++a)
                s[a][threadIdx.x] = a < 3 ? fmin(s[a][threadIdx.x], s[a][threadIdx.x + st])
                                          : fmax(s[a][threadIdx.x], s[a][threadIdx.x + st]);
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int a = 0; a < 6; ++a) part[blockIdx.x * 6 + a] = s[a][0];
}

// Per-block partial sums: sum f (3), sum q.nu (1), sum x (q.nu) (3).
__global__ void sums_partial_kernel(const double* __restrict__ x, const double* __restrict__ f,
                                    const double* __restrict__ nu, int64_t N,
                                    double* __restrict__ part) {
    __shared__ double s[7][RED_THREADS];
    double v[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x) {
        v[0] += f[3 * i];
        v[1] += f[3 * i + 1];
        v[2] += f[3 * i + 2];
        if (nu) {
            const double qn = f[3 * i] * nu[3 * i] + f[3 * i + 1] * nu[3 * i + 1] + f[3 * i + 2] * nu[3 * i + 2];
            v[3] += qn;
            v[4] += qn * x[3 * i];
            v[5] += qn * x[3 * i + 1];
            v[6] += qn * x[3 * i + 2];
        }
    }
    for (int a = 0; a < 7; ++a) s[a][threadIdx.x] = v[a];
    __syncthreads();
    for (int st = RED_THREADS / 2; st > 0; st >>= 1) {
        if ((int)threadIdx.x < st)
            for (int a = 0; a < 7; ++a) s[a][threadIdx.x] += s[a][threadIdx.x + st];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int a = 0; a < 7; ++a) part[blockIdx.x * 7 + a] = s[a][0];
}

__global__ void sums_final_kernel(const double* __restrict__ part, int nblocks, double* __restrict__ out) {
    const int a = threadIdx.x;
    if (a >= 7) return;
    double acc = 0.0;
    for (int b = 0; b < nblocks; ++b) acc += part[b * 7 + a];
    out[a] = acc;
}

struct EpilogueArgs {
    int kind, d, same, fourier;
    double self_coef;   // -4 xi / sqrt(pi) (stokeslet, same points)
    double zm_scale;    // -8 pi / V (stresslet, d = 3)
    double gauge[3];    // per-component multipliers of sum f (d <= 1 stokeslet)
};

// u += self term + stresslet zero mode - gauge shift (realspace.cpp:211-217,
// kernels.cpp:169-187, modified_kernels.cpp:272-281).
__global__ void epilogue_kernel(EpilogueArgs e, const double* __restrict__ f,
                                const double* __restrict__ xt, const double* __restrict__ sums,
                                const uint32_t* __restrict__ torder, int64_t t0, int64_t t1,
                                int accumulate, double* __restrict__ u) {
    const int64_t t = t0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= t1) return;
    const int64_t ti = torder[t];
    double v[3] = {0.0, 0.0, 0.0};
    if (e.fourier) {
        for (int c = 0; c < 3; ++c) v[c] -= e.gauge[c] * sums[c];
    }
    if (e.same && e.kind == SEWALD_STOKESLET)
        for (int c = 0; c < 3; ++c) v[c] += e.self_coef * f[3 * ti + c];
    if (e.kind == SEWALD_STRESSLET && e.d == 3)
        for (int c = 0; c < 3; ++c) v[c] += e.zm_scale * (sums[3] * xt[3 * ti + c] - sums[4 + c]);
    for (int c = 0; c < 3; ++c) {
        if (accumulate)
            u[3 * ti + c] += v[c];
        else
            u[3 * ti + c] = v[c];
    }
}

int bits_for(uint64_t nkeys) {
    int b = 1;
    while ((1ull << b) < nkeys) ++b;
    return b;
}

void sort_pairs(sewald_gpu_session* s, const uint32_t* kin, uint32_t* kout, const uint32_t* vin,
                uint32_t* vout, int64_t n, int bits) {
    size_t tmp = 0;
    cuda_check(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin, kout, vin, vout, (int)n, 0, bits,
                                               s->ctx->stream),
               "cub sort size");
    void* t = s->cub_tmp.ensure(tmp);
    cuda_check(cub::DeviceRadixSort::SortPairs(t, tmp, kin, kout, vin, vout, (int)n, 0, bits,
                                               s->ctx->stream),
               "cub sort");
    s->ctx->launches += 3;
}

void check_flag(sewald_gpu_session* s, int which, int code, const char* msg) {
    int h = 0;
    cuda_check(cudaMemcpyAsync(&h, s->flags.as<int>() + which, sizeof(int), cudaMemcpyDeviceToHost,
                               s->ctx->stream),
               "flag read");
    cuda_check(cudaStreamSynchronize(s->ctx->stream), "flag sync");
    if (h) {
        cuda_check(cudaMemsetAsync(s->flags.as<int>() + which, 0, sizeof(int), s->ctx->stream), "flag reset");
        throw EngineError(code, msg);
    }
}

enum { FLAG_SRC_NONFINITE = 0, FLAG_TGT_NONFINITE = 1, FLAG_SPREAD_BOX = 2, FLAG_GATHER_BOX = 3,
       FLAG_SINGULAR = 4, NFLAGS = 8 };

// The input checks of one call (non-finite sources and targets) are read
// together, once, by the first stage that consumes the inputs: one D2H and
// one stream synchronisation instead of one per stage.
void check_inputs(sewald_gpu_session* s) {
    if (s->inputs_checked) return;
    int* h = s->hflags.get();
    cuda_check(cudaMemcpyAsync(h, s->flags.as<int>(), sizeof(int) * 2, cudaMemcpyDeviceToHost, s->ctx->stream),
               "flag read");
    cuda_check(cudaStreamSynchronize(s->ctx->stream), "flag sync");
    if (h[FLAG_SRC_NONFINITE] || h[FLAG_TGT_NONFINITE]) {
        cuda_check(cudaMemsetAsync(s->flags.as<int>(), 0, sizeof(int) * 2, s->ctx->stream), "flag reset");
        if (h[FLAG_SRC_NONFINITE]) throw EngineError(SEWALD_EINVAL, "non-finite source position");
        throw EngineError(SEWALD_EINVAL, "target coordinates must be finite");
    }
    s->inputs_checked = true;
}

void build_cell_grid(sewald_gpu_session* s) {
    const sewald_params_c& p = s->p;
    CellGrid cg{};
    cg.d = p.d;
    for (int a = 0; a < 3; ++a) cg.L[a] = p.L[a];
    // Free axes: span of the (unwrapped) source coordinates.
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    if (p.d < 3 && s->N > 0) {
        const int nb = (int)std::min<int64_t>(RED_BLOCKS, (s->N + RED_THREADS - 1) / RED_THREADS);
        double* part = static_cast<double*>(s->partials.ensure(sizeof(double) * 6 * RED_BLOCKS));
        minmax_kernel<<<nb, RED_THREADS, 0, s->ctx->stream>>>(s->x.as<double>(), s->N, part);
        ++s->ctx->launches;
        std::vector<double> h(6 * nb);
        cuda_check(cudaMemcpyAsync(h.data(), part, sizeof(double) * 6 * nb, cudaMemcpyDeviceToHost,
                                   s->ctx->stream),
                   "minmax copy");
        cuda_check(cudaStreamSynchronize(s->ctx->stream), "minmax sync");
        for (int a = 0; a < 3; ++a) {
            lo[a] = h[a];
            hi[a] = h[3 + a];
            for (int b = 1; b < nb; ++b) {
                lo[a] = std::min(lo[a], h[6 * b + a]);
                hi[a] = std::max(hi[a], h[6 * b + 3 + a]);
            }
        }
    }
    // Cell width: about PPC = 28 particles per cell, so that an i-cluster of
    // 32 sorted particles spans about one cell (measured: c2 flat between 28
    // and 40, c5 80 vs 85 ms against the fixed rc/4 = 9/cell, c3 127 vs 133),
    // clamped to [rc/8, rc/2].
    // SEWALD_RS_REFINE=r forces rc/r; SEWALD_RS_PPC sets the target.
    static const double refine = [] {
        const char* e = getenv("SEWALD_RS_REFINE");
        return e ? atof(e) : 0.0;
    }();
    static const double ppc_env = [] {
        const char* e = getenv("SEWALD_RS_PPC");
        return e ? atof(e) : 0.0;
    }();
    const bool sym_on = option(SEWALD_OPT_RS_SYM) != 0;
    double target_w;
    if (refine > 0.0) {
        target_w = p.rc / refine;
    } else {
        double vol = 1.0;
        for (int a = 0; a < 3; ++a) vol *= std::max(a < p.d ? p.L[a] : hi[a] - lo[a], 1e-300);
        const double dens = s->N > 0 ? (double)s->N / vol : 1.0;
        // pair-symmetric kernel (targets == sources): 28, or 40 with more than
        // 5000 neighbours in the rc ball (c2 10.7k: 50.9 -> 50.3 ms, c3 19.7k:
        // 102.3 -> 101.4; c5 2.5k: 51.5 vs 52.0 at 40); separate targets: 40 (c4:
        // 47.6 vs 49.3 ms)
        const double nbrs = dens * 4.18879020478639 * p.rc * p.rc * p.rc;
        const double ppc = ppc_env > 0.0 ? ppc_env : (s->same && sym_on ? (nbrs > 5000.0 ? 40.0 : 28.0) : 40.0);
        target_w = std::cbrt(ppc / dens);
        target_w = std::min(std::max(target_w, p.rc / 8.0), p.rc / 2.0);
    }
    for (int a = 0; a < 3; ++a) {
        const double span = a < p.d ? p.L[a] : hi[a] - lo[a];
        cg.origin[a] = a < p.d ? 0.0 : lo[a];
        cg.n[a] = std::max(1, (int)std::floor(span / target_w));
        if (cg.n[a] > 4096) cg.n[a] = 4096;
    }
    while ((int64_t)cg.n[0] * cg.n[1] * cg.n[2] > (int64_t(1) << 22)) {
        int a = 0;
        for (int b = 1; b < 3; ++b)
            if (cg.n[b] > cg.n[a]) a = b;
        cg.n[a] = (cg.n[a] + 1) / 2;
    }
    for (int a = 0; a < 3; ++a) {
        const double span = a < p.d ? p.L[a] : hi[a] - lo[a];
        cg.w[a] = span > 0.0 ? span / cg.n[a] : target_w;
    }
    static const int sub_env = [] {
        const char* e = getenv("SEWALD_RS_SUB");
        return e ? atoi(e) : 8;
    }();
    const int64_t ncell = (int64_t)cg.n[0] * cg.n[1] * cg.n[2];
    cg.sub = std::max(0, std::min(sub_env, 32 - bits_for((uint64_t)ncell)));
    s->cg = cg;
}

void ensure_sums(sewald_gpu_session* s) {
    if (s->sums_ready) return;
    double* out = static_cast<double*>(s->sums.ensure(sizeof(double) * 8));
    double* part = static_cast<double*>(s->partials.ensure(sizeof(double) * 7 * RED_BLOCKS));
    const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(RED_BLOCKS, (s->N + RED_THREADS - 1) / RED_THREADS));
    if (s->N > 0) {
        sums_partial_kernel<<<nb, RED_THREADS, 0, s->ctx->stream>>>(
            s->x.as<double>(), s->f.as<double>(), s->stresslet ? s->nu.as<double>() : nullptr, s->N, part);
        sums_final_kernel<<<1, 32, 0, s->ctx->stream>>>(part, nb, out);
        s->ctx->launches += 2;
    } else {
        cuda_check(cudaMemsetAsync(out, 0, sizeof(double) * 8, s->ctx->stream), "sums zero");
    }
    s->sums_ready = true;
}

// Orderings built under other kernel-choice switches are dropped (options.h).
void sync_options(sewald_gpu_session* s) {
    const int e = options_epoch();
    if (s->opt_epoch == e) return;
    s->opt_epoch = e;
    s->sp_i0 = s->sp_i1 = -1;
    s->cells_ready = false;
    s->tg_ready = false;
    s->tg_wpart = -1;
}

void ensure_spread_order(sewald_gpu_session* s, int64_t i0, int64_t i1) {
    sync_options(s);
    if (s->sp_i0 == i0 && s->sp_i1 == i1) return;
    const int64_t n = i1 - i0;
    cudaStream_t st = s->ctx->stream;
    s->shape = spread_plan_shape(s->g, s->p.P);
    s->sweep = sweep_shape(s->g, s->p.P);
    // z-sweep for P <= 24 (c1-c3, c5); the 8x8x16 tile kernel wins for the
    // widest windows (c4, P = 32: 25 ms vs 42 ms). SEWALD_SPREAD_SWEEP=0/1 forces.
    const int sweep_mode = option(SEWALD_OPT_SPREAD_SWEEP);
    if (sweep_mode == 0 || (sweep_mode < 0 && s->p.P > 24)) s->sweep.ok = false;
    // tensor-core tiles for P <= 16 (SEWALD_SPREAD_MMA=0 disables)
    const bool mma_enabled = option(SEWALD_OPT_SPREAD_MMA) != 0;
    s->sm_shape = spread_mma_shape(s->g, s->p.P);
    s->sp_mode = (mma_enabled && s->sm_shape.ok) ? 2 : (s->sweep.ok ? 1 : 0);
    const int64_t nb = s->sp_mode == 2 ? s->sm_shape.ntiles
                       : s->sweep.ok   ? s->sweep.nkeys
                                       : (int64_t)s->shape.nb[0] * s->shape.nb[1] * s->shape.nb[2];
    s->sp_keys.ensure(sizeof(uint32_t) * std::max<int64_t>(n, 1));
    s->sp_keys2.ensure(sizeof(uint32_t) * std::max<int64_t>(n, 1));
    s->sp_vals.ensure(sizeof(uint32_t) * std::max<int64_t>(n, 1));
    s->sp_order.ensure(sizeof(uint32_t) * std::max<int64_t>(n, 1));
    s->sp_off.ensure(sizeof(int64_t) * (nb + 1));
    int* bad = s->flags.as<int>() + FLAG_SPREAD_BOX;
    const int sub = s->sp_mode == 2 ? s->sm_shape.sub : 0;
    if (s->sp_mode == 2)
        launch_spread_mma_bucket(s->g, s->p.P, s->sm_shape, s->x.as<double>() + 3 * i0, n, s->sp_keys.as<uint32_t>(),
                                 s->sp_vals.as<uint32_t>(), bad, st);
    else if (s->sweep.ok)
        launch_sweep_bucket(s->g, s->p.P, s->x.as<double>() + 3 * i0, n, s->sweep, s->sp_keys.as<uint32_t>(),
                            s->sp_vals.as<uint32_t>(), bad, st);
    else
        launch_spread_bucket(s->g, s->p.P, s->x.as<double>() + 3 * i0, n, s->shape,
                             s->sp_keys.as<uint32_t>(), s->sp_vals.as<uint32_t>(), bad, st);
    ++s->ctx->launches;
    // a finite point always has an in-range stencil on a periodic axis
    if (s->p.d < 3)
        check_flag(s, FLAG_SPREAD_BOX, SEWALD_EINVAL,
                   "point too close to the extended box boundary; free-direction padding is too small");
    if (n > 0) {
        sort_pairs(s, s->sp_keys.as<uint32_t>(), s->sp_keys2.as<uint32_t>(), s->sp_vals.as<uint32_t>(),
                   s->sp_order.as<uint32_t>(), n, bits_for((uint64_t)nb + 1) + sub);
    }
    launch_bucket_offsets(s->sp_keys2.as<uint32_t>(), n, (int)nb, s->sp_off.as<int64_t>(), st, sub);
    ++s->ctx->launches;
    s->sp_i0 = i0;
    s->sp_i1 = i1;
}

void ensure_cells(sewald_gpu_session* s) {
    sync_options(s);
    if (s->cells_ready) return;
    cudaStream_t st = s->ctx->stream;
    build_cell_grid(s);
    const int64_t N = s->N;
    const int64_t ncell = (int64_t)s->cg.n[0] * s->cg.n[1] * s->cg.n[2];
    s->s_folded.ensure(sizeof(double) * 3 * std::max<int64_t>(N, 1));
    s->c_keys.ensure(sizeof(uint32_t) * std::max<int64_t>(N, 1));
    s->c_keys2.ensure(sizeof(uint32_t) * std::max<int64_t>(N, 1));
    s->c_vals.ensure(sizeof(uint32_t) * std::max<int64_t>(N, 1));
    s->c_order.ensure(sizeof(uint32_t) * std::max<int64_t>(N, 1));
    s->c_off.ensure(sizeof(int64_t) * (ncell + 1));
    const int S = s->stresslet ? 12 : 8;
    s->packed.ensure(sizeof(double) * S * std::max<int64_t>(N, 1));
    s->packedf.ensure(sizeof(float4) * std::max<int64_t>(N, 1));
    launch_fold_and_key(s->cg, s->x.as<double>(), N, s->s_folded.as<double>(), s->c_keys.as<uint32_t>(),
                        s->c_vals.as<uint32_t>(), st);
    if (N > 0) {
        ++s->ctx->launches;
        sort_pairs(s, s->c_keys.as<uint32_t>(), s->c_keys2.as<uint32_t>(), s->c_vals.as<uint32_t>(),
                   s->c_order.as<uint32_t>(), N, bits_for((uint64_t)ncell << s->cg.sub));
    }
    launch_bucket_offsets(s->c_keys2.as<uint32_t>(), N, (int)ncell, s->c_off.as<int64_t>(), st, s->cg.sub);
    launch_pack_sources(s->s_folded.as<double>(), s->f.as<double>(), s->nu.as<double>(), s->stresslet,
                        s->c_order.as<uint32_t>(), N, s->packed.as<double>(), s->packedf.as<float4>(), st);
    s->ctx->launches += 2;
    s->cells_ready = true;
}

void ensure_target_order(sewald_gpu_session* s) {
    ensure_cells(s);
    if (s->same) return;  // targets reuse the source cell order
    cudaStream_t st = s->ctx->stream;
    const int64_t Nt = s->Nt;
    const int64_t ncell = (int64_t)s->cg.n[0] * s->cg.n[1] * s->cg.n[2];
    if (Nt == 0) return;
    s->t_folded.ensure(sizeof(double) * 3 * Nt);
    s->t_keys.ensure(sizeof(uint32_t) * Nt);
    s->t_keys2.ensure(sizeof(uint32_t) * Nt);
    s->t_vals.ensure(sizeof(uint32_t) * Nt);
    s->t_order.ensure(sizeof(uint32_t) * Nt);
    launch_fold_and_key(s->cg, s->xt.as<double>(), Nt, s->t_folded.as<double>(), s->t_keys.as<uint32_t>(),
                        s->t_vals.as<uint32_t>(), st);
    ++s->ctx->launches;
    sort_pairs(s, s->t_keys.as<uint32_t>(), s->t_keys2.as<uint32_t>(), s->t_vals.as<uint32_t>(),
               s->t_order.as<uint32_t>(), Nt, bits_for((uint64_t)ncell << s->cg.sub));
}

const double* target_positions(sewald_gpu_session* s) {
    return s->same ? s->x.as<double>() : s->xt.as<double>();
}
const double* target_folded(sewald_gpu_session* s) {
    return s->same ? s->s_folded.as<double>() : s->t_folded.as<double>();
}
const uint32_t* target_order(sewald_gpu_session* s) {
    return s->same ? s->c_order.as<uint32_t>() : s->t_order.as<uint32_t>();
}

// Targets bucketed / sorted for the tiled gather (P <= 20) or the z-sweep
// gather (P > 20), with their window taps. Returns 0 (warp-per-target
// gather), 1 (sweep) or 2 (tiles). SEWALD_GATHER=warp|sweep|tile forces one.
// Window taps of the targets in the tiles of part `part` of `nparts` (the tile
// range evaluate() gathers); the sorted-index window is read on the device.
void ensure_gather_weights(sewald_gpu_session* s, int mode, int part, int nparts) {
    const int key = nparts == 1 ? 0 : part * 4096 + nparts;
    if (s->tg_wpart == key) return;
    // the fused tensor-core tiles evaluate their taps themselves
    if (mode == 2 && gather_tile_fused_ok(tile_shape(s->g, s->p.P, s->Nt))) return;
    const SweepShape sh = sweep_shape(s->g, s->p.P);
    const TileShape ts = tile_shape(s->g, s->p.P, s->Nt);
    const int64_t nt = mode == 1 ? (int64_t)sh.nbx * sh.nby : ts.ntiles;
    // the sweep buckets tile (x, y) patches over all z starts; the tile path tiles
    const int64_t per = mode == 1 ? (int64_t)s->g.n[2] : 1;
    const int64_t t0 = nt * part / nparts, t1 = nt * (part + 1) / nparts;
    const int64_t* off = s->tg_off.as<int64_t>();
    const double* xt = s->same ? s->x.as<double>() : s->xt.as<double>();
    launch_sweep_weights(s->g, s->w, xt, nullptr, nullptr, 0, s->tg_order.as<uint32_t>(), s->Nt, s->tg_w.as<double>(),
                         s->tg_sw.as<int4>(), nullptr, s->ctx->stream, nparts == 1 ? nullptr : off + t0 * per,
                         nparts == 1 ? nullptr : off + t1 * per);
    ++s->ctx->launches;
    s->tg_wpart = key;
}

int ensure_gather_order(sewald_gpu_session* s, int part, int nparts) {
    sync_options(s);
    const int forced = option(SEWALD_OPT_GATHER);
    const SweepShape sh = sweep_shape(s->g, s->p.P);
    const TileShape ts = tile_shape(s->g, s->p.P, s->Nt);
    // tiles up to P = 32 (P > 20: gather_wide_mma_kernel; c4 17.3 -> 9.1 ms vs the z-sweep)
    int mode = forced >= 0 ? forced : 2;
    if (mode == 2 && !ts.ok) mode = sh.ok ? 1 : 0;
    if (mode == 1 && !sh.ok) mode = 0;
    if (mode == 0) return 0;
    if (s->tg_ready && s->tg_mode == mode) {
        ensure_gather_weights(s, mode, part, nparts);
        return mode;
    }
    cudaStream_t st = s->ctx->stream;
    const int64_t Nt = s->Nt;
    const double* xt = s->same ? s->x.as<double>() : s->xt.as<double>();
    const int64_t n = std::max<int64_t>(Nt, 1);
    const int64_t nkeys = mode == 1 ? sh.nkeys : ts.ntiles;
    s->tg_keys.ensure(sizeof(uint32_t) * n);
    s->tg_keys2.ensure(sizeof(uint32_t) * n);
    s->tg_vals.ensure(sizeof(uint32_t) * n);
    s->tg_order.ensure(sizeof(uint32_t) * n);
    s->tg_off.ensure(sizeof(int64_t) * (nkeys + 1));
    s->tg_w.ensure(sizeof(double) * 3 * s->p.P * n);
    s->tg_sw.ensure(sizeof(int4) * n);
    int* bad = s->flags.as<int>() + FLAG_GATHER_BOX;
    // register-A tiles: a tile's targets ordered by their x stencil offset (n-blocks skip rows they cannot reach)
    const int sub = (mode == 2 && gather_tile_regA(ts) && option(SEWALD_OPT_GATHER_SORT) != 0 &&
                     ts.ntiles < (int64_t(1) << 26))
                        ? 6
                        : 0;
    if (mode == 1)
        launch_sweep_bucket(s->g, s->p.P, xt, Nt, sh, s->tg_keys.as<uint32_t>(), s->tg_vals.as<uint32_t>(), bad, st);
    else
        launch_tile_bucket(s->g, s->p.P, ts, xt, Nt, s->tg_keys.as<uint32_t>(), s->tg_vals.as<uint32_t>(), bad, st,
                           sub);
    check_flag(s, FLAG_GATHER_BOX, SEWALD_EINVAL,
               "point too close to the extended box boundary; free-direction padding is too small");
    if (Nt > 0)
        sort_pairs(s, s->tg_keys.as<uint32_t>(), s->tg_keys2.as<uint32_t>(), s->tg_vals.as<uint32_t>(),
                   s->tg_order.as<uint32_t>(), Nt, bits_for((uint64_t)nkeys + 1) + sub);
    launch_bucket_offsets(s->tg_keys2.as<uint32_t>(), Nt, (int)nkeys, s->tg_off.as<int64_t>(), st, sub);
    s->ctx->launches += 2;
    s->tg_ready = true;
    s->tg_mode = mode;
    s->tg_wpart = -1;
    ensure_gather_weights(s, mode, part, nparts);
    return mode;
}

void d3_prepare(sewald_gpu_session* s) {
    if (s->d3) return;
    auto P = std::make_unique<FourierPlanD3>();
    const sewald_params_c& p = s->p;
    P->C = s->C;
    for (int a = 0; a < 3; ++a) P->n[a] = p.M_ext[a];
    const int n0 = P->n[0], n1 = P->n[1], n2 = P->n[2], nh = n2 / 2 + 1;
    const int64_t vol = (int64_t)n0 * n1 * n2, hvol = (int64_t)n0 * n1 * nh;
    // Tables: wavenumbers on the periodic grid M with spacing h and the
    // window transform at each (fourier.cpp:543-548).
    std::vector<double> hostt;
    std::vector<double> kx[3], wx[3];
    for (int a = 0; a < 3; ++a) {
        kx[a] = wavenumbers(p.M[a], p.h);
        wx[a] = window_hat_table(p, kx[a]);
    }
    kx[2].resize(nh);
    wx[2].resize(nh);
    for (int a = 0; a < 3; ++a) hostt.insert(hostt.end(), kx[a].begin(), kx[a].end());
    for (int a = 0; a < 3; ++a) hostt.insert(hostt.end(), wx[a].begin(), wx[a].end());
    double* dt = static_cast<double*>(P->tables.ensure(sizeof(double) * hostt.size()));
    cuda_check(cudaMemcpyAsync(dt, hostt.data(), sizeof(double) * hostt.size(), cudaMemcpyHostToDevice,
                               s->ctx->stream),
               "k tables");
    const int len[3] = {n0, n1, nh};
    size_t o = 0;
    for (int a = 0; a < 3; ++a) { P->kt.k[a] = dt + o; o += len[a]; }
    for (int a = 0; a < 3; ++a) { P->kt.what[a] = dt + o; o += len[a]; }
    P->spec.ensure(sizeof(cuDoubleComplex) * hvol * s->C);
    int n[3] = {n0, n1, n2};
    int nemb_r[3] = {n0, n1, n2}, nemb_c[3] = {n0, n1, nh};
    cufft_check(cufftPlanMany(&P->fwd, 3, n, nemb_r, 1, (int)vol, nemb_c, 1, (int)hvol, CUFFT_D2Z, s->C),
                "plan D2Z");
    cufft_check(cufftPlanMany(&P->inv, 3, n, nemb_c, 1, (int)hvol, nemb_r, 1, (int)vol, CUFFT_Z2D, 3),
                "plan Z2D");
    cufft_check(cufftSetStream(P->fwd, s->ctx->stream), "fft stream");
    cufft_check(cufftSetStream(P->inv, s->ctx->stream), "fft stream");
    cuda_check(cudaStreamSynchronize(s->ctx->stream), "tables sync");
    s->d3 = std::move(P);
}

struct StageTimer {
    sewald_gpu_ctx* ctx;
    cudaEvent_t ev[12];
    int n = 0;
    explicit StageTimer(sewald_gpu_ctx* c) : ctx(c) {
        if (ctx->profiling)
            for (auto& e : ev) cudaEventCreate(&e);
    }
    void mark() {
        if (ctx->profiling && n < 12) cudaEventRecord(ev[n++], ctx->stream);
    }
    double ms(int a, int b) {
        float t = 0;
        if (!ctx->profiling || b >= n) return 0.0;
        cudaEventElapsedTime(&t, ev[a], ev[b]);
        return t;
    }
    ~StageTimer() {
        if (ctx->profiling)
            for (auto& e : ev) cudaEventDestroy(e);
    }
};

}  // namespace

DevGrid make_dev_grid(const sewald_params_c& p) {
    DevGrid g{};
    g.d = p.d;
    g.h = p.h;
    for (int a = 0; a < 3; ++a) {
        g.n[a] = p.M_ext[a];
        g.x0[a] = a < p.d ? 0.0 : -0.5 * p.pad[a];
        g.L[a] = p.L[a];
    }
    return g;
}

DevWindow make_dev_window(const sewald_params_c& p) {
    validate_window(p);
    if (p.P > kMaxP) throw EngineError(SEWALD_EINVAL, "window support P exceeds the device limit");
    DevWindow w{};
    w.kind = p.win_kind;
    w.P = p.P;
    w.nu = p.nu;
    w.h = p.win_h;
    w.half_width = 0.5 * p.win_h * static_cast<double>(p.P);
    w.beta = p.beta;
    w.i0_beta = bessel_i0(p.beta);
    w.alpha = p.alpha;
    if (p.win_kind == SEWALD_WIN_PKB) {
        if (p.nu > kMaxNu) throw EngineError(SEWALD_EINVAL, "PKB degree exceeds the device limit");
        const std::vector<double> c = pkb_coefficients(p);
        std::copy(c.begin(), c.end(), w.coef);
    }
    return w;
}

void session_init(sewald_gpu_session* s, sewald_gpu_ctx* ctx, const sewald_params_c& p) {
    if (p.d < 0 || p.d > 3) throw EngineError(SEWALD_EINVAL, "periodicity d must be in 0..3");
    if (p.kind < 0 || p.kind > 2) throw EngineError(SEWALD_EINVAL, "unknown kernel");
    for (int a = 0; a < 3; ++a)
        if (!(p.L[a] > 0.0)) throw EngineError(SEWALD_EINVAL, "cell lengths must be positive");
    if (std::fabs(p.win_h - p.h) > 1e-12 * p.h)
        throw EngineError(SEWALD_EINVAL, "window was built for a different grid spacing");
    s->ctx = ctx;
    s->p = p;
    s->g = make_dev_grid(p);
    s->w = make_dev_window(p);
    s->stresslet = p.kind == SEWALD_STRESSLET;
    s->C = s->stresslet ? 9 : 3;
    s->flags.ensure(sizeof(int) * NFLAGS);
    cuda_check(cudaMemsetAsync(s->flags.ptr, 0, sizeof(int) * NFLAGS, ctx->stream), "flags");
    s->pair_counter.ensure(sizeof(unsigned long long));
    cuda_check(cudaMemsetAsync(s->pair_counter.ptr, 0, sizeof(unsigned long long), ctx->stream), "pairs");
}

void session_set_sources(sewald_gpu_session* s, const double* x, const double* f, const double* nu,
                         int64_t N) {
    cudaStream_t st = s->ctx->stream;
    if (s->stresslet && N > 0 && !nu) throw EngineError(SEWALD_EINVAL, "stresslet needs one orientation per source");
    if (!s->stresslet && nu) throw EngineError(SEWALD_EINVAL, "orientations only apply to the stresslet");
    s->N = N;
    const size_t b = sizeof(double) * 3 * std::max<int64_t>(N, 1);
    s->x.ensure(b);
    s->f.ensure(b);
    if (N > 0) {
        cuda_check(cudaMemcpyAsync(s->x.ptr, x, sizeof(double) * 3 * N, cudaMemcpyDefault, st), "x copy");
        cuda_check(cudaMemcpyAsync(s->f.ptr, f, sizeof(double) * 3 * N, cudaMemcpyDefault, st), "f copy");
    }
    if (s->stresslet) {
        s->nu.ensure(b);
        if (N > 0)
            cuda_check(cudaMemcpyAsync(s->nu.ptr, nu, sizeof(double) * 3 * N, cudaMemcpyDefault, st), "nu copy");
    }
    if (N > 0) {
        finite_check_kernel<<<(unsigned)((3 * N + 255) / 256), 256, 0, st>>>(
            s->x.as<double>(), 3 * N, s->flags.as<int>() + FLAG_SRC_NONFINITE);
        ++s->ctx->launches;
    }
    s->sp_i0 = s->sp_i1 = -1;
    s->cells_ready = false;
    s->sums_ready = false;
    s->tg_ready = false;
    s->inputs_checked = false;
    if (s->same) s->Nt = N;
}

void session_set_targets(sewald_gpu_session* s, const double* xt, int64_t Nt, bool same) {
    if (s->same != same) s->cells_ready = false;  // the cell width depends on the kernel (build_cell_grid)
    s->same = same;
    s->tg_ready = false;
    s->inputs_checked = false;
    if (same) {
        s->Nt = s->N;
        return;
    }
    s->Nt = Nt;
    cudaStream_t st = s->ctx->stream;
    s->xt.ensure(sizeof(double) * 3 * std::max<int64_t>(Nt, 1));
    if (Nt > 0) {
        cuda_check(cudaMemcpyAsync(s->xt.ptr, xt, sizeof(double) * 3 * Nt, cudaMemcpyDefault, st), "xt copy");
        finite_check_kernel<<<(unsigned)((3 * Nt + 255) / 256), 256, 0, st>>>(
            s->xt.as<double>(), 3 * Nt, s->flags.as<int>() + FLAG_TGT_NONFINITE);
        ++s->ctx->launches;
    }
}

void session_spread(sewald_gpu_session* s, int64_t i0, int64_t i1, double* grid) {
    if (i0 < 0 || i1 > s->N || i0 > i1) throw EngineError(SEWALD_EINVAL, "bad source range");
    check_inputs(s);
    ensure_spread_order(s, i0, i1);
    cudaStream_t st = s->ctx->stream;
    const int64_t vol = (int64_t)s->g.n[0] * s->g.n[1] * s->g.n[2];
    if (s->sp_mode == 2 && spread_mma_fused_ok(s->sm_shape, s->C)) {
        void* fsrc = s->fused_arg.ensure(fused_src_bytes());
        s->ctx->launches += launch_spread_mma_fused(s->g, s->w, s->p.P, s->sm_shape, s->x.as<double>() + 3 * i0,
                                                    s->f.as<double>() + 3 * i0,
                                                    s->stresslet ? s->nu.as<double>() + 3 * i0 : nullptr,
                                                    s->sp_order.as<uint32_t>(), s->C, s->sp_off.as<int64_t>(), grid,
                                                    fsrc, st);
        cuda_check(cudaGetLastError(), "spread launch");
        return;
    }
    if (s->sp_mode == 2 || s->sweep.ok) {
        const int64_t n = i1 - i0;
        const int P = s->p.P;
        double* W = static_cast<double*>(s->sp_w.ensure(sizeof(double) * 3 * P * std::max<int64_t>(n, 1)));
        int4* SW = static_cast<int4*>(s->sp_sw.ensure(sizeof(int4) * std::max<int64_t>(n, 1)));
        double* STR = static_cast<double*>(s->sp_str.ensure(sizeof(double) * s->C * std::max<int64_t>(n, 1)));
        launch_sweep_weights(s->g, s->w, s->x.as<double>() + 3 * i0, s->f.as<double>() + 3 * i0,
                             s->stresslet ? s->nu.as<double>() + 3 * i0 : nullptr, s->stresslet,
                             s->sp_order.as<uint32_t>(), n, W, SW, STR, st);
        if (s->sp_mode == 2)
            s->ctx->launches += 1 + launch_spread_mma(s->g, P, s->sm_shape, W, SW, STR, s->C,
                                                      s->sp_off.as<int64_t>(), grid, st);
        else
            s->ctx->launches += 1 + launch_spread_sweep(s->g, P, W, SW, STR, s->C, s->sp_off.as<int64_t>(),
                                                        s->sweep, grid, st);
        cuda_check(cudaGetLastError(), "spread sweep launch");
        return;
    }
    if (!s->shape.tiled) {
        cuda_check(cudaMemsetAsync(grid, 0, sizeof(double) * s->C * vol, st), "grid zero");
        launch_spread_atomic(s->g, s->w, s->x.as<double>() + 3 * i0, s->f.as<double>() + 3 * i0,
                             s->stresslet ? s->nu.as<double>() + 3 * i0 : nullptr, s->stresslet,
                             i1 - i0, grid, st);
        ++s->ctx->launches;
        return;
    }
    launch_spread_tiles(s->g, s->w, s->x.as<double>() + 3 * i0, s->f.as<double>() + 3 * i0,
                        s->stresslet ? s->nu.as<double>() + 3 * i0 : nullptr, s->stresslet,
                        s->sp_order.as<uint32_t>(), s->sp_off.as<int64_t>(), s->shape, grid, st);
    s->ctx->launches += s->stresslet ? 3 : 1;
    cuda_check(cudaGetLastError(), "spread launch");
}

void session_solve(sewald_gpu_session* s, const double* grid, bool precompute_0p) {
    if (!(s->p.xi > 0.0)) throw EngineError(SEWALD_EINVAL, "xi must be positive");
    const int64_t vol = (int64_t)s->g.n[0] * s->g.n[1] * s->g.n[2];
    s->flow.ensure(sizeof(double) * 3 * vol);
    if (s->p.d < 3) {
        aft_solve(s, grid, precompute_0p);
        return;
    }
    d3_prepare(s);
    FourierPlanD3& P = *s->d3;
    cudaStream_t st = s->ctx->stream;
    cuDoubleComplex* spec = P.spec.as<cuDoubleComplex>();
    // cuFFT plans keep the stream they were last given; the context's stream
    // can change between calls (Session follows torch's current stream), so
    // every execution sets it (here and in aft.cu / aft_d0.cu)
    cufftSetStream(P.fwd, st);
    cufft_check(cufftExecD2Z(P.fwd, const_cast<double*>(grid), spec), "exec D2Z");
    const int64_t hvol = (int64_t)P.n[0] * P.n[1] * (P.n[2] / 2 + 1);
    launch_scale_periodic(s->p.kind, P.n[0], P.n[1], P.n[2], s->p.xi, 1.0 / (double)vol, P.kt, spec,
                          hvol, st);
    ++s->ctx->launches;
    cufftSetStream(P.inv, st);
    cufft_check(cufftExecZ2D(P.inv, spec, s->flow.as<double>()), "exec Z2D");
    cuda_check(cudaGetLastError(), "solve launch");
}

void session_evaluate(sewald_gpu_session* s, int part, int nparts, int parts, double* u) {
    if (nparts < 1 || part < 0 || part >= nparts) throw EngineError(SEWALD_EINVAL, "bad target partition");
    check_inputs(s);
    cudaStream_t st = s->ctx->stream;
    ensure_target_order(s);
    const int64_t Nt = s->Nt;
    // Cluster-aligned partition of the cell-ordered targets (32 per cluster).
    const int64_t ncl = (Nt + 31) / 32;
    const int64_t c0 = ncl * part / nparts, c1 = ncl * (part + 1) / nparts;
    const int64_t t0 = std::min<int64_t>(32 * c0, Nt), t1 = std::min<int64_t>(32 * c1, Nt);
    // A part may own no 32-target cluster (more parts than clusters) and still
    // own gather tiles (the tiled / swept gathers split the tiles, not the
    // clusters): it then contributes its gather share only.
    const bool has_targets = t1 > t0;
    if (Nt == 0) return;
    const uint32_t* torder = target_order(s);
    // SEWALD_RS_SYM: 0 = never the pair-symmetric kernel, "force" = always
    // when targets are the sources (tests pin it at small N), else automatic.
    const int sym_mode = option(SEWALD_OPT_RS_SYM);
    // Small target sets (fewer 32-target groups than resident warps) take the
    // non-symmetric kernel with each group's rows split over several warps and
    // a fixed-order combination: the whole GPU works on them and the result is
    // independent of scheduling (no reactions, no atomics).
    // The choice is made once for the whole partition (from the smallest part,
    // ncl / nparts clusters), so every part and rank runs the same kernel: the
    // symmetric kernel's half rule assigns each pair to the part holding its
    // lower index, which is only complete when all parts use it.
    const int rs_split = realspace_split(32 * std::max<int64_t>(1, ncl / nparts));
    const bool use_sym = (parts & 2) && s->same && sym_mode != 0 && (rs_split == 1 || sym_mode == 2);
    // The pair-symmetric real-space sum adds reactions to any particle, and
    // multi-part evaluation is combined by summing the per-part outputs: in
    // both cases the whole output is zeroed here and every stage accumulates.
    bool first = true;
    if (use_sym || nparts > 1) {
        cuda_check(cudaMemsetAsync(u, 0, sizeof(double) * 3 * Nt, st), "u zero");
        first = false;
    }
    // the pair-symmetric kernel takes interleaved clusters (below): part p has
    // work iff p < ncl; the other kernels take the contiguous target range
    const bool rs_work = use_sym ? (int64_t)part < ncl : has_targets;
    if ((parts & 2) && rs_work) {
        if (!(s->p.xi > 0.0)) throw EngineError(SEWALD_EINVAL, "split parameter must be positive");
        if (!(s->p.rc > 0.0)) throw EngineError(SEWALD_EINVAL, "cell list cutoff must be positive");
        RealspaceArgs a{};
        a.kind = s->p.kind;
        a.xi = s->p.xi;
        a.rc = s->p.rc;
        a.xi2 = a.xi * a.xi;
        a.rc2 = a.rc * a.rc;
        a.skip_self = s->same ? 1 : 0;
        // fp32 candidate bound: coordinates (targets folded or inside the
        // free-axis span, +-shift) are O(ext); fp32 differences carry at
        // most a few ulp(ext) error per axis, so pad rc by 2^-18 ext.
        double ext = a.rc;
        for (int ax = 0; ax < 3; ++ax)
            ext = std::max(ext, std::fabs(s->cg.origin[ax]) + s->cg.n[ax] * s->cg.w[ax] + s->cg.L[ax] + 2.0 * a.rc);
        const double rpad = a.rc + std::ldexp(ext, -18);
        a.thresh_f = (float)(rpad * rpad * (1.0 + std::ldexp(1.0, -16)));
        if (use_sym) {
            // Parts take every nparts-th cluster (not a contiguous range): the half
            // rule gives the clusters near the start of the cell order (low z)
            // the periodic-wrap pairs of both ends, so contiguous ranges would
            // load the first part with up to ~1.5x the average (measured 55 / 45 %
            // of the pairs for two parts at c2); interleaved parts sample every
            // z layer. The epilogue keeps the contiguous target range: each is a
            // partition of its own work and the outputs are summed.
            launch_realspace_sym(s->cg, a, s->packed.as<double>(), Nt, s->c_off.as<int64_t>(),
                                 nparts > 1 ? part : 0, ncl, nparts, u,
                                 s->pair_counter.as<unsigned long long>(), s->flags.as<int>() + FLAG_SINGULAR,
                                 static_cast<unsigned long long*>(s->work_counter.ensure(sizeof(unsigned long long))),
                                 st);
        } else {
            double* scratch = rs_split > 1 ? static_cast<double*>(s->rs_scratch.ensure(
                                                  sizeof(double) * 3 * (size_t)rs_split * (size_t)(t1 - t0)))
                                            : nullptr;
            launch_realspace(s->cg, a, s->packed.as<double>(), s->packedf.as<float4>(), s->stresslet,
                             s->c_off.as<int64_t>(), target_folded(s), torder + t0, t1 - t0, u, first ? 0 : 1,
                             s->pair_counter.as<unsigned long long>(), s->flags.as<int>() + FLAG_SINGULAR, rs_split,
                             scratch, st);
        }
        ++s->ctx->launches;
        first = false;
    }
    if (parts & 1) {
        const double h3 = s->p.h * s->p.h * s->p.h;
        const int gmode = ensure_gather_order(s, part, nparts);
        if (gmode == 1) {
            if (first) cuda_check(cudaMemsetAsync(u, 0, sizeof(double) * 3 * Nt, st), "u zero");
            launch_gather_sweep(s->g, s->p.P, s->tg_w.as<double>(), s->tg_sw.as<int4>(), s->tg_off.as<int64_t>(),
                                sweep_shape(s->g, s->p.P), part, nparts, s->flow.as<double>(), h3, u, st);
        } else if (gmode == 2) {
            const TileShape ts = tile_shape(s->g, s->p.P, s->Nt);
            if (gather_tile_fused_ok(ts))
                launch_gather_tile_fused(s->g, s->w, s->p.P, ts, target_positions(s), s->tg_order.as<uint32_t>(),
                                         s->tg_off.as<int64_t>(), part, nparts, s->flow.as<double>(), h3,
                                         first ? 0 : 1, u, s->fused_garg.ensure(fused_tgt_bytes()), st);
            else
                launch_gather_tile(s->g, s->p.P, ts, s->tg_w.as<double>(), s->tg_sw.as<int4>(), s->tg_off.as<int64_t>(),
                                   part, nparts, s->flow.as<double>(), h3, first ? 0 : 1, u, st);
        } else if (has_targets) {
            launch_gather(s->g, s->w, s->flow.as<double>(), target_positions(s), torder + t0, t1 - t0, h3,
                          first ? 0 : 1, u, st);
        }
        ++s->ctx->launches;
        first = false;
    }
    if ((parts & 4 || (parts & 1)) && has_targets) {
        ensure_sums(s);
        EpilogueArgs e{};
        e.kind = s->p.kind;
        e.d = s->p.d;
        e.same = (parts & 4) && s->same;
        e.fourier = (parts & 1) ? 1 : 0;
        e.self_coef = -4.0 * s->p.xi / 1.7724538509055160273;
        e.zm_scale = (parts & 4) ? -8.0 * kPi / (s->p.L[0] * s->p.L[1] * s->p.L[2]) : 0.0;
        // gauge_flow_correction (modified_kernels.cpp:272-281) with the
        // optimal gauge constants (modified_kernels.cpp:52-63).
        if (s->p.kind == SEWALD_STOKESLET && s->p.d <= 1) {
            const double R = s->p.R;
            if (s->p.d == 0) {
                const double bB = -0.5 / R;
                e.gauge[0] = e.gauge[1] = e.gauge[2] = 4.0 * bB;
            } else {
                const double ellH = R, ellB = R * std::sqrt(M_E);
                const double c1 = std::log(ellH * M_E) * 4.0;
                const double c23 = std::log(ellB) * 2.0;
                const double inv = 1.0 / s->p.L[0];
                e.gauge[0] = c1 * inv;
                e.gauge[1] = c23 * inv;
                e.gauge[2] = c23 * inv;
            }
        }
        const int64_t n = t1 - t0;
        epilogue_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
            e, s->f.as<double>(), target_positions(s), s->sums.as<double>(), torder, t0, t1, first ? 0 : 1, u);
        ++s->ctx->launches;
    }
    cuda_check(cudaGetLastError(), "evaluate launch");
}

// The context's host-buffer session, rebuilt when the parameters change.
sewald_gpu_session* cached_session(sewald_gpu_ctx* ctx, const sewald_params_c& p) {
    if (ctx->cached && std::memcmp(&ctx->cached_params, &p, sizeof(p)) == 0) return ctx->cached.get();
    ctx->cached.reset();
    auto s = std::make_unique<sewald_gpu_session>();
    session_init(s.get(), ctx, p);
    ctx->cached = std::move(s);
    ctx->cached_params = p;
    return ctx->cached.get();
}

// Free-axis stencil bound of the targets (the reference's gather check,
// fourier.cpp:176-181), d < 3 only: one flag read.
void session_check_target_box(sewald_gpu_session* s) {
    if (s->p.d >= 3 || s->Nt == 0) return;
    launch_stencil_bounds(s->g, s->p.P, target_positions(s), s->Nt, s->flags.as<int>() + FLAG_GATHER_BOX,
                          s->ctx->stream);
    check_flag(s, FLAG_GATHER_BOX, SEWALD_EINVAL,
               "point too close to the extended box boundary; free-direction padding is too small");
}

// Starts the read of the real-space singularity flag (r = 0 between distinct
// points) into pinned memory; session_finish_singular throws after the
// caller's stream synchronisation if it was set.
void session_read_singular(sewald_gpu_session* s) {
    int* hf = s->hflags.get();
    cuda_check(cudaMemcpyAsync(hf + FLAG_SINGULAR, s->flags.as<int>() + FLAG_SINGULAR, sizeof(int),
                               cudaMemcpyDeviceToHost, s->ctx->stream), "flag read");
}

void session_finish_singular(sewald_gpu_session* s) {
    int* hf = s->hflags.get();
    if (hf[FLAG_SINGULAR]) {
        hf[FLAG_SINGULAR] = 0;
        cuda_check(cudaMemsetAsync(s->flags.as<int>() + FLAG_SINGULAR, 0, sizeof(int), s->ctx->stream), "flag reset");
        throw EngineError(SEWALD_EDOMAIN, "real-space kernel is singular at the origin");
    }
}

}  // namespace sewald_b200


// ===========================================================================
// C-ABI (device part)
// ===========================================================================

using namespace sewald_b200;

namespace {

template <class F>
int ctx_guard(sewald_gpu_ctx* ctx, F&& fn) {
    try {
        if (ctx) cudaSetDevice(ctx->device);
        fn();
        return SEWALD_OK;
    } catch (const EngineError& e) {
        if (ctx) ctx->err = e.what();
        return e.code;
    } catch (const std::invalid_argument& e) {
        if (ctx) ctx->err = e.what();
        return SEWALD_EINVAL;
    } catch (const std::domain_error& e) {
        if (ctx) ctx->err = e.what();
        return SEWALD_EDOMAIN;
    } catch (const std::exception& e) {
        if (ctx) ctx->err = e.what();
        return SEWALD_ERUNTIME;
    }
}

void host_pipeline(sewald_gpu_ctx* ctx, const sewald_params_c* p, const double* x, const double* f,
                   const double* nu, int64_t N, const double* xt, int64_t Nt, int same, int use_table,
                   int parts, double* u_out) {
    if (!p) throw EngineError(SEWALD_EINVAL, "null parameters");
    if (N < 0 || Nt < 0) throw EngineError(SEWALD_EINVAL, "negative sizes");
    if (same && Nt != N && Nt != 0 && xt) throw EngineError(SEWALD_EINVAL, "starred evaluation needs one target per source");
    sewald_gpu_session* s = cached_session(ctx, *p);
    StageTimer tm(ctx);
    const int64_t launches0 = ctx->launches;
    tm.mark();
    x = stage_in(ctx->px, x, 3 * (size_t)N);
    f = stage_in(ctx->pf, f, 3 * (size_t)N);
    nu = stage_in(ctx->pnu, nu, 3 * (size_t)N);
    if (!same) xt = stage_in(ctx->pxt, xt, 3 * (size_t)Nt);
    session_set_targets(s, xt, Nt, same != 0);
    session_set_sources(s, x, f, nu, N);
    if (!same) session_set_targets(s, xt, Nt, false);
    tm.mark();  // 1: after H2D
    const int64_t nt = s->Nt;
    double* du = static_cast<double*>(ctx->hu.ensure(sizeof(double) * 3 * std::max<int64_t>(nt, 1)));
    double* out_stage = nullptr;
    if (parts & 1) {
        const int64_t vol = (int64_t)s->g.n[0] * s->g.n[1] * s->g.n[2];
        double* grid = static_cast<double*>(s->grid.ensure(sizeof(double) * s->C * vol));
        session_spread(s, 0, N, grid);
        tm.mark();  // 2
        session_solve(s, grid, use_table != 0);
        tm.mark();  // 3
    } else {
        tm.mark();
        tm.mark();
    }
    if (nt > 0) {
        ensure_target_order(s);
        if (parts & 1) session_check_target_box(s);
        tm.mark();  // 4
        session_evaluate(s, 0, 1, parts, du);
        tm.mark();  // 5
        if (is_pageable(u_out)) {  // through pinned staging, copied out after the synchronisation
            out_stage = static_cast<double*>(ctx->pu.ensure(sizeof(double) * 3 * nt));
            cuda_check(cudaMemcpyAsync(out_stage, du, sizeof(double) * 3 * nt, cudaMemcpyDeviceToHost, ctx->stream),
                       "u copy");
        } else {
            cuda_check(cudaMemcpyAsync(u_out, du, sizeof(double) * 3 * nt, cudaMemcpyDefault, ctx->stream), "u copy");
        }
    } else {
        tm.mark();
        tm.mark();
    }
    tm.mark();  // 6
    session_read_singular(s);  // read with the result: no extra synchronisation
    cuda_check(cudaStreamSynchronize(ctx->stream), "pipeline sync");
    session_finish_singular(s);
    if (out_stage) parallel_memcpy(u_out, out_stage, sizeof(double) * 3 * nt);
    sewald_timings_c& T = ctx->timings;
    T = sewald_timings_c{};
    T.h2d_ms = tm.ms(0, 1);
    T.spread_ms = tm.ms(1, 2);
    T.fft_fwd_ms = tm.ms(2, 3);
    T.realspace_ms = tm.ms(4, 5);
    T.d2h_ms = tm.ms(5, 6);
    T.total_ms = tm.ms(0, 6);
    T.kernel_launches = ctx->launches - launches0;
    T.realspace_pairs = -1;
}

}  // namespace

extern "C" {

int sewald_gpu_create(int device, sewald_gpu_ctx** out) {
    if (!out) return SEWALD_EINVAL;
    *out = nullptr;
    auto* ctx = new sewald_gpu_ctx();
    ctx->device = device;
    int rc = ctx_guard(ctx, [&] {
        cuda_check(cudaSetDevice(device), "cudaSetDevice");
        cuda_check(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking), "stream");
        ctx->stream = ctx->own_stream;
    });
    if (rc != SEWALD_OK) {
        delete ctx;
        return rc;
    }
    *out = ctx;
    return SEWALD_OK;
}

void sewald_gpu_destroy(sewald_gpu_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    ctx->cached.reset();
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
}

const char* sewald_gpu_last_error(const sewald_gpu_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int sewald_gpu_set_stream(sewald_gpu_ctx* ctx, void* stream) {
    if (!ctx) return SEWALD_EINVAL;
    // The value is used as is: NULL is the legacy default stream (what
    // torch.cuda.current_stream().cuda_stream returns for the default).
    ctx->stream = static_cast<cudaStream_t>(stream);
    return SEWALD_OK;
}

int sewald_gpu_get_timings(const sewald_gpu_ctx* ctx, sewald_timings_c* out) {
    if (!ctx || !out) return SEWALD_EINVAL;
    *out = ctx->timings;
    return SEWALD_OK;
}

int sewald_gpu_host_buffer(sewald_gpu_ctx* ctx, size_t bytes, void** out) {
    if (!ctx || !out) return SEWALD_EINVAL;
    try {
        cuda_check(cudaSetDevice(ctx->device), "set device");
        *out = ctx->pout.ensure(std::max<size_t>(bytes, 1));
        return SEWALD_OK;
    } catch (const std::exception& e) {
        ctx->err = e.what();
        return SEWALD_ECUDA;
    }
}

int sewald_gpu_set_profiling(sewald_gpu_ctx* ctx, int enabled) {
    if (!ctx) return SEWALD_EINVAL;
    ctx->profiling = enabled != 0;
    return SEWALD_OK;
}

int sewald_gpu_full_potential(sewald_gpu_ctx* ctx, const sewald_params_c* p, const double* x,
                              const double* f, const double* nu, int64_t N, const double* xt,
                              int64_t Nt, int same_as_sources, int precompute_0p, double* u_out) {
    if (!ctx) return SEWALD_EINVAL;
    return ctx_guard(ctx, [&] {
        host_pipeline(ctx, p, x, f, nu, N, xt, Nt, same_as_sources, precompute_0p, 7, u_out);
    });
}

int sewald_gpu_fourier_potential(sewald_gpu_ctx* ctx, const sewald_params_c* p, const double* x,
                                 const double* f, const double* nu, int64_t N, const double* xt,
                                 int64_t Nt, int same_as_sources, int precompute_0p, double* u_out) {
    if (!ctx) return SEWALD_EINVAL;
    return ctx_guard(ctx, [&] {
        host_pipeline(ctx, p, x, f, nu, N, xt, Nt, same_as_sources, precompute_0p, 1, u_out);
    });
}

int sewald_gpu_realspace_potential(sewald_gpu_ctx* ctx, int kind, int d, const double L[3],
                                   const double* x, const double* f, const double* nu, int64_t N,
                                   const double* xt, int64_t Nt, int same_as_sources, double xi,
                                   double rc, int starred, double* u_out) {
    if (!ctx) return SEWALD_EINVAL;
    return ctx_guard(ctx, [&] {
        if (!(xi > 0.0)) throw EngineError(SEWALD_EINVAL, "split parameter must be positive");
        if (!(rc > 0.0)) throw EngineError(SEWALD_EINVAL, "cell list cutoff must be positive");
        const bool skip_self = starred && same_as_sources;
        if (skip_self && Nt != N) throw EngineError(SEWALD_EINVAL, "starred evaluation needs one target per source");
        // A minimal parameter set: real space needs kind, d, cell, xi, rc.
        sewald_params_c p{};
        p.kind = kind;
        p.d = d;
        p.xi = xi;
        p.rc = rc;
        for (int a = 0; a < 3; ++a) {
            p.L[a] = L[a];
            p.M[a] = p.M_ext[a] = 8;
            p.L_ext[a] = L[a];
        }
        p.h = L[0] / 8;
        p.f_m = 4;
        window_make(SEWALD_WIN_TG, 2, p.h, p);
        // Unstarred sums over coincident points must see them as distinct
        // targets (so r = 0 is reported), which the session does by
        // treating targets as separate when skip_self is false.
        const bool same = skip_self;
        const double* tx = same ? x : (same_as_sources ? x : xt);
        host_pipeline(ctx, &p, x, f, nu, N, tx, same ? N : Nt, same ? 1 : 0, 0, 2, u_out);
    });
}

int sewald_gpu_spread(sewald_gpu_ctx* ctx, const sewald_params_c* p, const double* x,
                      const double* f, const double* nu, int64_t N, double* grid_out) {
    if (!ctx) return SEWALD_EINVAL;
    return ctx_guard(ctx, [&] {
        sewald_gpu_session* s = cached_session(ctx, *p);
        session_set_sources(s, x, f, nu, N);
        const int64_t vol = (int64_t)s->g.n[0] * s->g.n[1] * s->g.n[2];
        double* grid = static_cast<double*>(s->grid.ensure(sizeof(double) * s->C * vol));
        session_spread(s, 0, N, grid);
        cuda_check(cudaMemcpyAsync(grid_out, grid, sizeof(double) * s->C * vol, cudaMemcpyDefault, ctx->stream),
                   "grid copy");
        cuda_check(cudaStreamSynchronize(ctx->stream), "spread sync");
    });
}

int sewald_gpu_gather(sewald_gpu_ctx* ctx, const sewald_params_c* p, const double* grid,
                      const double* xt, int64_t Nt, double* u_out) {
    if (!ctx) return SEWALD_EINVAL;
    return ctx_guard(ctx, [&] {
        // The stage function runs the same gather kernel the pipeline picks
        // (tiles / tensor-core tiles / z-sweep / warp per target, options.h),
        // on the caller's grid and targets, without the epilogue terms.
        sewald_gpu_session* s = cached_session(ctx, *p);
        const int64_t vol = (int64_t)s->g.n[0] * s->g.n[1] * s->g.n[2];
        double* flow = static_cast<double*>(s->flow.ensure(sizeof(double) * 3 * vol));
        cuda_check(cudaMemcpyAsync(flow, grid, sizeof(double) * 3 * vol, cudaMemcpyDefault, ctx->stream), "grid in");
        double* du = static_cast<double*>(ctx->hu.ensure(sizeof(double) * 3 * std::max<int64_t>(Nt, 1)));
        // the cached session's sources stay; its targets become xt
        session_set_targets(s, xt, Nt, false);
        if (Nt > 0) {
            check_inputs(s);
            launch_stencil_bounds(s->g, s->p.P, s->xt.as<double>(), Nt, s->flags.as<int>() + FLAG_GATHER_BOX,
                                  ctx->stream);
            check_flag(s, FLAG_GATHER_BOX, SEWALD_EINVAL,
                       "point too close to the extended box boundary; free-direction padding is too small");
            const double h3 = s->p.h * s->p.h * s->p.h;
            const int gmode = ensure_gather_order(s, 0, 1);
            if (gmode == 1) {
                cuda_check(cudaMemsetAsync(du, 0, sizeof(double) * 3 * Nt, ctx->stream), "u zero");
                launch_gather_sweep(s->g, s->p.P, s->tg_w.as<double>(), s->tg_sw.as<int4>(), s->tg_off.as<int64_t>(),
                                    sweep_shape(s->g, s->p.P), 0, 1, flow, h3, du, ctx->stream);
            } else if (gmode == 2) {
                const TileShape ts = tile_shape(s->g, s->p.P, Nt);
                if (gather_tile_fused_ok(ts))
                    launch_gather_tile_fused(s->g, s->w, s->p.P, ts, s->xt.as<double>(), s->tg_order.as<uint32_t>(),
                                             s->tg_off.as<int64_t>(), 0, 1, flow, h3, 0, du,
                                             s->fused_garg.ensure(fused_tgt_bytes()), ctx->stream);
                else
                    launch_gather_tile(s->g, s->p.P, ts, s->tg_w.as<double>(), s->tg_sw.as<int4>(),
                                       s->tg_off.as<int64_t>(), 0, 1, flow, h3, 0, du, ctx->stream);
            } else {
                launch_gather(s->g, s->w, flow, s->xt.as<double>(), nullptr, Nt, h3, 0, du, ctx->stream);
            }
            ++ctx->launches;
            cuda_check(cudaGetLastError(), "gather launch");
            cuda_check(cudaMemcpyAsync(u_out, du, sizeof(double) * 3 * Nt, cudaMemcpyDefault, ctx->stream), "u out");
        }
        cuda_check(cudaStreamSynchronize(ctx->stream), "gather sync");
    });
}

int sewald_gpu_aft_forward(sewald_gpu_ctx* ctx, const sewald_params_c* p, const double* field,
                           const sewald_fourier_geom_c* g, double* far, double* near, double* zero) {
    if (!ctx || !p || !g) return SEWALD_EINVAL;
    return ctx_guard(ctx, [&] { stage_aft_forward(ctx, *p, field, *g, far, near, zero); });
}

int sewald_gpu_aft_inverse(sewald_gpu_ctx* ctx, const sewald_params_c* p, const sewald_fourier_geom_c* g,
                           const int32_t* near_rows, const double* far, const double* near, const double* zero,
                           double* field_out) {
    if (!ctx || !p || !g) return SEWALD_EINVAL;
    return ctx_guard(ctx, [&] { stage_aft_inverse(ctx, *p, *g, near_rows, far, near, zero, field_out); });
}

int sewald_gpu_scale(sewald_gpu_ctx* ctx, const sewald_params_c* p, const sewald_modspec_c* spec, double xi,
                     const sewald_fourier_geom_c* g, const int32_t* near_rows, const double* far,
                     const double* near, const double* zero, double* far_out, double* near_out,
                     double* zero_out) {
    if (!ctx || !p || !spec || !g) return SEWALD_EINVAL;
    return ctx_guard(ctx, [&] {
        if (spec->kind < 0 || spec->kind > 2) throw EngineError(SEWALD_EINVAL, "unknown kernel");
        stage_scale(ctx, *p, spec->kind, spec, nullptr, nullptr, xi, *g, near_rows, far, near, zero, far_out,
                    near_out, zero_out);
    });
}

int sewald_gpu_scale_table(sewald_gpu_ctx* ctx, const sewald_params_c* p, int kind, const int32_t table_n[3],
                           const double* table, double xi, const sewald_fourier_geom_c* g, const double* zero,
                           double* zero_out) {
    if (!ctx || !p || !table_n || !table || !g) return SEWALD_EINVAL;
    return ctx_guard(ctx, [&] {
        if (kind < 0 || kind > 2) throw EngineError(SEWALD_EINVAL, "unknown kernel");
        stage_scale(ctx, *p, kind, nullptr, table_n, table, xi, *g, nullptr, nullptr, nullptr, zero, nullptr,
                    nullptr, zero_out);
    });
}

int sewald_gpu_precompute_0p(sewald_gpu_ctx* ctx, const sewald_params_c* p, int kind, double R, int32_t n_out[3],
                             double* table_out) {
    if (!ctx || !p || !n_out) return SEWALD_EINVAL;
    return ctx_guard(ctx, [&] {
        if (kind < 0 || kind > 2) throw EngineError(SEWALD_EINVAL, "unknown kernel");
        stage_precompute_0p(ctx, *p, kind, R, n_out, table_out);
    });
}

int sewald_gpu_set_table0p(sewald_gpu_ctx* ctx, const sewald_params_c* p, const int32_t n[3],
                           const double* table) {
    if (!ctx || !p || (table && !n)) return SEWALD_EINVAL;
    return ctx_guard(ctx, [&] { session_set_table0p(cached_session(ctx, *p), n, table); });
}

int sewald_gpu_session_set_table0p(sewald_gpu_session* s, const int32_t n[3], const double* table) {
    if (!s || (table && !n)) return SEWALD_EINVAL;
    return ctx_guard(s->ctx, [&] { session_set_table0p(s, n, table); });
}

int sewald_gpu_session_create(sewald_gpu_ctx* ctx, const sewald_params_c* p, sewald_gpu_session** out) {
    if (!ctx || !p || !out) return SEWALD_EINVAL;
    *out = nullptr;
    return ctx_guard(ctx, [&] {
        auto s = std::make_unique<sewald_gpu_session>();
        session_init(s.get(), ctx, *p);
        *out = s.release();
    });
}

void sewald_gpu_session_destroy(sewald_gpu_session* s) {
    if (!s) return;
    cudaSetDevice(s->ctx->device);
    cudaStreamSynchronize(s->ctx->stream);
    delete s;
}

int sewald_gpu_session_set_sources(sewald_gpu_session* s, const double* x, const double* f,
                                   const double* nu, int64_t N) {
    if (!s) return SEWALD_EINVAL;
    return ctx_guard(s->ctx, [&] { session_set_sources(s, x, f, nu, N); });
}

int sewald_gpu_session_set_targets(sewald_gpu_session* s, const double* xt, int64_t Nt, int same) {
    if (!s) return SEWALD_EINVAL;
    return ctx_guard(s->ctx, [&] { session_set_targets(s, xt, Nt, same != 0); });
}

int64_t sewald_gpu_session_grid_size(const sewald_gpu_session* s) {
    if (!s) return -1;
    return (int64_t)s->C * s->g.n[0] * s->g.n[1] * s->g.n[2];
}

int sewald_gpu_session_spread(sewald_gpu_session* s, int64_t i0, int64_t i1, double* grid) {
    if (!s) return SEWALD_EINVAL;
    return ctx_guard(s->ctx, [&] {
        double* g = grid;
        if (!g) g = static_cast<double*>(s->grid.ensure(sizeof(double) * sewald_gpu_session_grid_size(s)));
        session_spread(s, i0, i1, g);
    });
}

int sewald_gpu_session_solve(sewald_gpu_session* s, const double* grid, int precompute_0p) {
    if (!s) return SEWALD_EINVAL;
    return ctx_guard(s->ctx, [&] { session_solve(s, grid ? grid : s->grid.as<double>(), precompute_0p != 0); });
}

int sewald_gpu_session_evaluate(sewald_gpu_session* s, int part, int nparts, int parts, double* u) {
    if (!s) return SEWALD_EINVAL;
    return ctx_guard(s->ctx, [&] { session_evaluate(s, part, nparts, parts, u); });
}

static sewald_b200::SlabBounds slab_bounds_from(int world, const int* b) {
    if (world < 1 || world > sewald_b200::kMaxWorld || !b)
        throw sewald_b200::EngineError(SEWALD_EINVAL, "bad slab bounds");
    sewald_b200::SlabBounds sb{};
    sb.world = world;
    for (int r = 0; r <= world; ++r) {
        sb.b[r] = b[r];
        if (r > 0 && b[r] < b[r - 1]) throw sewald_b200::EngineError(SEWALD_EINVAL, "slab bounds must be sorted");
    }
    return sb;
}

int sewald_gpu_session_d0_geometry(sewald_gpu_session* s, int precompute_0p, int m[3], int n[3], int* h2,
                                   int* C) {
    if (!s || !m || !n || !h2 || !C) return SEWALD_EINVAL;
    return ctx_guard(s->ctx, [&] { aft_d0_geometry(s, precompute_0p != 0, m, n, h2, C); });
}

int sewald_gpu_session_d0_forward(sewald_gpu_session* s, int precompute_0p, const double* grid_slab, int xa,
                                  int xb, int world, const int* kz_bounds, void* send) {
    if (!s) return SEWALD_EINVAL;
    return ctx_guard(s->ctx, [&] {
        aft_d0_slab_forward(s, precompute_0p != 0, grid_slab, xa, xb, slab_bounds_from(world, kz_bounds), send);
    });
}

int sewald_gpu_session_d0_middle(sewald_gpu_session* s, int precompute_0p, const void* recv, int world,
                                 const int* x_bounds, int ka, int kb, void* send) {
    if (!s) return SEWALD_EINVAL;
    return ctx_guard(s->ctx, [&] {
        aft_d0_slab_middle(s, precompute_0p != 0, recv, slab_bounds_from(world, x_bounds), ka, kb, send);
    });
}

int sewald_gpu_session_d0_inverse(sewald_gpu_session* s, int precompute_0p, const void* recv, int xa, int xb,
                                  int world, const int* kz_bounds, double* flow_slab) {
    if (!s) return SEWALD_EINVAL;
    return ctx_guard(s->ctx, [&] {
        aft_d0_slab_inverse(s, precompute_0p != 0, recv, xa, xb, slab_bounds_from(world, kz_bounds), flow_slab);
    });
}

int sewald_gpu_session_set_flow(sewald_gpu_session* s, const double* flow_dev) {
    if (!s || !flow_dev) return SEWALD_EINVAL;
    return ctx_guard(s->ctx, [&] {
        const int64_t vol = (int64_t)s->g.n[0] * s->g.n[1] * s->g.n[2];
        double* f = static_cast<double*>(s->flow.ensure(sizeof(double) * 3 * vol));
        cuda_check(cudaMemcpyAsync(f, flow_dev, sizeof(double) * 3 * vol, cudaMemcpyDeviceToDevice, s->ctx->stream),
                   "set flow");
    });
}

int64_t sewald_gpu_launch_count(const sewald_gpu_ctx* ctx) { return ctx ? ctx->launches : -1; }

int64_t sewald_gpu_session_pair_count(sewald_gpu_session* s, int reset) {
    if (!s) return -1;
    unsigned long long h = 0;
    int rc = ctx_guard(s->ctx, [&] {
        cuda_check(cudaMemcpyAsync(&h, s->pair_counter.ptr, sizeof(h), cudaMemcpyDeviceToHost, s->ctx->stream),
                   "pair count");
        cuda_check(cudaStreamSynchronize(s->ctx->stream), "pair sync");
        if (reset) cuda_check(cudaMemsetAsync(s->pair_counter.ptr, 0, sizeof(h), s->ctx->stream), "pair reset");
    });
    return rc == SEWALD_OK ? (int64_t)h : -1;
}

int sewald_gpu_session_run(sewald_gpu_session* s, int precompute_0p, double* u) {
    if (!s) return SEWALD_EINVAL;
    return ctx_guard(s->ctx, [&] {
        double* g = static_cast<double*>(s->grid.ensure(sizeof(double) * sewald_gpu_session_grid_size(s)));
        session_spread(s, 0, s->N, g);
        session_solve(s, g, precompute_0p != 0);
        session_evaluate(s, 0, 1, 7, u);
    });
}

}  // extern "C"
