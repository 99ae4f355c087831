// Spread (point strengths -> grid) and gather (grid -> targets) in fp64.
//
// Reference: spread  /root/reference/proj/src/fourier.cpp:237-274
//            gather  /root/reference/proj/src/fourier.cpp:276-309
//            stencil /root/reference/proj/src/fourier.cpp:168-188
//
// Spread is OUTPUT-STATIONARY: one CTA owns a TX x TY x TZ block of the
// grid; each thread owns one (x, y) column of TZ values per component in
// registers. Points are bucketed by the grid tile of their stencil START
// index; a CTA streams the buckets whose stencils reach its block through
// shared memory (tile-local weights computed once per staging), and every
// grid value is written exactly once — no atomics, no zero-fill pass.
//
// Gather is WARP-PER-TARGET: lanes cover (two stencil rows) x (16 z taps), so
// each warp load is two coalesced 128 B row segments of the L2-resident grid.
#include "device_common.cuh"
#include "sg_kernels.h"

namespace sewald_b200 {

namespace {

constexpr int TX = 8, TY = 8, TZ = 16;
constexpr int SPREAD_THREADS = TX * TY;  // one thread per (x,y) column
constexpr int CHUNK = SPREAD_THREADS;    // points staged per round

struct StagedPoint {
    double wx[TX];
    double wy[TY];
    double wz[TZ];
    double s[3];        // strength components of this pass
    int dx, dy;         // tile-relative stencil offsets (X0 - sx, Y0 - sy)
};

__device__ __forceinline__ int tile_delta(int T0, int s, int n, bool periodic, int P) {
    // Representative of T0 - s in [-(T-1), P-1] (periodic axes wrap).
    int d = T0 - s;
    if (periodic) {
        d %= n;
        if (d < 0) d += n;
        if (d > P - 1) d -= n;
    }
    return d;
}

// Per-point bucket key: tile coordinates of the stencil start, wrapped on
// periodic axes. Sets *bad if a free-axis stencil leaves the extended box.
__global__ void spread_bucket_kernel(DevGrid g, int P, const double* __restrict__ x, int64_t N,
                                     int nbx, int nby, int nbz, uint32_t* __restrict__ keys,
                                     uint32_t* __restrict__ vals, int* __restrict__ bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    int b[3];
    const int T[3] = {TX, TY, TZ};
    for (int ax = 0; ax < 3; ++ax) {
        int j0;
        double rel;
        stencil_origin(g, P, ax, x[3 * i + ax], j0, rel);
        const int n = g.n[ax];
        if (ax < g.d) {
            j0 = wrap_index(j0, n);
        } else if (j0 < 0 || j0 + P > n) {
            atomicExch(bad, 1);
            j0 = 0;
        }
        b[ax] = j0 / T[ax];
    }
    keys[i] = (uint32_t)((b[0] * nby + b[1]) * nbz + b[2]);
    vals[i] = (uint32_t)i;
}

// off[b] = first sorted position with key >= b (b in [0, nb]).
__global__ void bucket_offsets_kernel(const uint32_t* __restrict__ keys, int64_t N, int nb,
                                      int64_t* __restrict__ off, int shift) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b > nb) return;
    int64_t lo = 0, hi = N;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((keys[mid] >> shift) < (uint32_t)b) lo = mid + 1; else hi = mid;
    }
    off[b] = lo;
}

// Range of bucket indices along one axis whose stencil starts can reach the
// tile [T0, T0+T). Up to two linear pieces (periodic wrap).
struct AxisBuckets {
    int lo[2], hi[2], pieces;
};

__device__ __forceinline__ AxisBuckets axis_buckets(int T0, int T, int n, int P, bool periodic,
                                                    int nbk) {
    AxisBuckets a;
    int s_lo = T0 - P + 1, s_hi = T0 + T - 1;
    if (s_hi > n - 1 && !periodic) s_hi = n - 1;
    if (!periodic) {
        if (s_lo < 0) s_lo = 0;
        a.pieces = 1;
        a.lo[0] = s_lo / T;
        a.hi[0] = s_hi / T;
        return a;
    }
    if (s_hi > n - 1) s_hi = n - 1;  // partial last tile: starts stop at n-1
    if (s_lo >= 0) {
        a.pieces = 1;
        a.lo[0] = s_lo / T;
        a.hi[0] = s_hi / T;
    } else {
        a.pieces = 2;
        a.lo[0] = 0;
        a.hi[0] = s_hi / T;
        a.lo[1] = (s_lo + n) / T;
        a.hi[1] = nbk - 1;
        if (a.lo[1] <= a.hi[0]) {  // pieces meet: whole axis once
            a.pieces = 1;
            a.lo[0] = 0;
            a.hi[0] = nbk - 1;
        }
    }
    return a;
}

// kind: 0 vector strengths f (3 comps), 1 stresslet outer product q_l nu_m
// with l = pass (comps 3l..3l+2).
__global__ void __launch_bounds__(SPREAD_THREADS)
spread_tile_kernel(DevGrid g, DevWindow win, const double* __restrict__ x,
                   const double* __restrict__ f, const double* __restrict__ nu, int stresslet,
                   int pass, const uint32_t* __restrict__ order, const int64_t* __restrict__ off,
                   int nbx, int nby, int nbz, double* __restrict__ out) {
    __shared__ StagedPoint sp[CHUNK];
    const int P = win.P;
    const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
    const int tbx = blockIdx.x, tby = blockIdx.y, tbz = blockIdx.z;
    const int X0 = tbx * TX, Y0 = tby * TY, Z0 = tbz * TZ;

    double acc[TZ][3];
#pragma unroll
    for (int z = 0; z < TZ; ++z)
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[z][c] = 0.0;

    const AxisBuckets ax = axis_buckets(X0, TX, g.n[0], P, g.d > 0, nbx);
    const AxisBuckets ay = axis_buckets(Y0, TY, g.n[1], P, g.d > 1, nby);
    const AxisBuckets az = axis_buckets(Z0, TZ, g.n[2], P, g.d > 2, nbz);

    for (int pxi = 0; pxi < ax.pieces; ++pxi)
    for (int bx = ax.lo[pxi]; bx <= ax.hi[pxi]; ++bx)
    for (int pyi = 0; pyi < ay.pieces; ++pyi)
    for (int by = ay.lo[pyi]; by <= ay.hi[pyi]; ++by)
    for (int pzi = 0; pzi < az.pieces; ++pzi) {
        // buckets (bx, by, az.lo..az.hi) are contiguous in key order
        const int kb0 = (bx * nby + by) * nbz + az.lo[pzi];
        const int kb1 = (bx * nby + by) * nbz + az.hi[pzi];
        const int64_t p0 = off[kb0], p1 = off[kb1 + 1];
        for (int64_t base = p0; base < p1; base += CHUNK) {
            const int cnt = (int)min((int64_t)CHUNK, p1 - base);
            if ((int)threadIdx.x < cnt) {
                const int64_t i = order[base + threadIdx.x];
                StagedPoint& q = sp[threadIdx.x];
                int s0[3], delta[3];
                double rel[3];
                for (int a = 0; a < 3; ++a) {
                    stencil_origin(g, P, a, x[3 * i + a], s0[a], rel[a]);
                }
                const int Tt[3] = {X0, Y0, Z0};
                for (int a = 0; a < 3; ++a) {
                    const bool per = a < g.d;
                    const int sw = per ? wrap_index(s0[a], g.n[a]) : s0[a];
                    delta[a] = tile_delta(Tt[a], sw, g.n[a], per, P);
                }
                // tile-local weights: tap p = delta + t (zero outside [0,P))
#pragma unroll
                for (int t = 0; t < TX; ++t) {
                    const int p = delta[0] + t;
                    q.wx[t] = (p >= 0 && p < P) ? window_eval(win, ((double)(s0[0] + p) - rel[0]) * g.h) : 0.0;
                }
#pragma unroll
                for (int t = 0; t < TY; ++t) {
                    const int p = delta[1] + t;
                    q.wy[t] = (p >= 0 && p < P) ? window_eval(win, ((double)(s0[1] + p) - rel[1]) * g.h) : 0.0;
                }
#pragma unroll
                for (int t = 0; t < TZ; ++t) {
                    const int p = delta[2] + t;
                    q.wz[t] = (p >= 0 && p < P) ? window_eval(win, ((double)(s0[2] + p) - rel[2]) * g.h) : 0.0;
                }
                q.dx = delta[0];
                q.dy = delta[1];
                if (!stresslet) {
                    q.s[0] = f[3 * i];
                    q.s[1] = f[3 * i + 1];
                    q.s[2] = f[3 * i + 2];
                } else {
                    const double ql = f[3 * i + pass];
                    q.s[0] = ql * nu[3 * i];
                    q.s[1] = ql * nu[3 * i + 1];
                    q.s[2] = ql * nu[3 * i + 2];
                }
            }
            __syncthreads();
            for (int k = 0; k < cnt; ++k) {
                const StagedPoint& q = sp[k];
                const int ox = q.dx + tx, oy = q.dy + ty;
                if (ox < 0 || ox >= P || oy < 0 || oy >= P) continue;
                const double wxy = q.wx[tx] * q.wy[ty];
                const double s0 = wxy * q.s[0], s1 = wxy * q.s[1], s2 = wxy * q.s[2];
#pragma unroll
                for (int z = 0; z < TZ; ++z) {
                    const double wz = q.wz[z];
                    acc[z][0] = fma(s0, wz, acc[z][0]);
                    acc[z][1] = fma(s1, wz, acc[z][1]);
                    acc[z][2] = fma(s2, wz, acc[z][2]);
                }
            }
            __syncthreads();
        }
    }

    const int gx = X0 + tx, gy = Y0 + ty;
    if (gx >= g.n[0] || gy >= g.n[1]) return;
    const int64_t cs = (int64_t)g.n[0] * g.n[1] * g.n[2];
    const int comp0 = stresslet ? 3 * pass : 0;
    double* col = out + ((int64_t)gx * g.n[1] + gy) * g.n[2];
#pragma unroll
    for (int z = 0; z < TZ; ++z) {
        if (Z0 + z < g.n[2]) {
            col[(comp0 + 0) * cs + Z0 + z] = acc[z][0];
            col[(comp0 + 1) * cs + Z0 + z] = acc[z][1];
            col[(comp0 + 2) * cs + Z0 + z] = acc[z][2];
        }
    }
}

// Fallback for tiny periodic grids (P + T - 1 > n): one thread per point,
// fp64 atomics. Exact same stencil rule; only used by small test grids.
__global__ void spread_atomic_kernel(DevGrid g, DevWindow win, const double* __restrict__ x,
                                     const double* __restrict__ f, const double* __restrict__ nu,
                                     int stresslet, int64_t N, double* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int P = win.P;
    double w[3][kMaxP];
    int idx[3][kMaxP];
    for (int a = 0; a < 3; ++a) {
        int j0;
        double rel;
        stencil_origin(g, P, a, x[3 * i + a], j0, rel);
        for (int p = 0; p < P; ++p) {
            const int j = j0 + p;
            w[a][p] = window_eval(win, ((double)j - rel) * g.h);
            idx[a][p] = a < g.d ? wrap_index(j, g.n[a]) : j;
        }
    }
    double fc[9];
    const int C = stresslet ? 9 : 3;
    if (!stresslet) {
        for (int c = 0; c < 3; ++c) fc[c] = f[3 * i + c];
    } else {
        for (int l = 0; l < 3; ++l)
            for (int m = 0; m < 3; ++m) fc[3 * l + m] = f[3 * i + l] * nu[3 * i + m];
    }
    const int64_t cs = (int64_t)g.n[0] * g.n[1] * g.n[2];
    for (int p1 = 0; p1 < P; ++p1)
        for (int p2 = 0; p2 < P; ++p2) {
            const double w12 = w[0][p1] * w[1][p2];
            const int64_t o2 = ((int64_t)idx[0][p1] * g.n[1] + idx[1][p2]) * g.n[2];
            for (int p3 = 0; p3 < P; ++p3) {
                const double ww = w12 * w[2][p3];
                for (int c = 0; c < C; ++c) atomicAdd(out + c * cs + o2 + idx[2][p3], ww * fc[c]);
            }
        }
}

// Warp per target. mode 0: u = h^3 acc (overwrite), 1: u += h^3 acc.
__global__ void __launch_bounds__(128)
gather_warp_kernel(DevGrid g, DevWindow win, const double* __restrict__ grid,
                   const double* __restrict__ xt, const uint32_t* __restrict__ order, int64_t Nt,
                   double h3, int accumulate, double* __restrict__ u) {
    __shared__ double sw[4][3][kMaxP];
    __shared__ int sidx[4][3][kMaxP];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t = (int64_t)blockIdx.x * 4 + warp;
    if (t >= Nt) return;
    const int64_t ti = order ? (int64_t)order[t] : t;
    const int P = win.P;
    for (int a = 0; a < 3; ++a) {
        int j0;
        double rel;
        stencil_origin(g, P, a, xt[3 * ti + a], j0, rel);
        for (int p = lane; p < P; p += 32) {
            const int j = j0 + p;
            sw[warp][a][p] = window_eval(win, ((double)j - rel) * g.h);
            int jj = a < g.d ? wrap_index(j, g.n[a]) : j;
            if (jj < 0 || jj >= g.n[a]) jj = 0;  // out-of-box rejected on host
            sidx[warp][a][p] = jj;
        }
    }
    __syncwarp();
    const int64_t cs = (int64_t)g.n[0] * g.n[1] * g.n[2];
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    const int half = lane >> 4, zl = lane & 15;
    for (int zc = 0; zc < P; zc += 16) {
        const int p3 = zc + zl;
        const bool v3 = p3 < P;
        const double w3 = v3 ? sw[warp][2][p3] : 0.0;
        const int i3 = v3 ? sidx[warp][2][p3] : 0;
        for (int p1 = 0; p1 < P; ++p1) {
            const double w1 = sw[warp][0][p1];
            const int64_t o1 = (int64_t)sidx[warp][0][p1] * g.n[1];
            for (int p2 = half; p2 < P; p2 += 2) {
                if (!v3) continue;
                const double ww = (w1 * sw[warp][1][p2]) * w3;
                const int64_t o = (o1 + sidx[warp][1][p2]) * g.n[2] + i3;
                a0 = fma(ww, __ldg(grid + o), a0);
                a1 = fma(ww, __ldg(grid + cs + o), a1);
                a2 = fma(ww, __ldg(grid + 2 * cs + o), a2);
            }
        }
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, s);
        a1 += __shfl_xor_sync(0xffffffffu, a1, s);
        a2 += __shfl_xor_sync(0xffffffffu, a2, s);
    }
    if (lane == 0) {
        if (accumulate) {
            u[3 * ti] += h3 * a0;
            u[3 * ti + 1] += h3 * a1;
            u[3 * ti + 2] += h3 * a2;
        } else {
            u[3 * ti] = h3 * a0;
            u[3 * ti + 1] = h3 * a1;
            u[3 * ti + 2] = h3 * a2;
        }
    }
}

// Free-axis bounds check for targets (fourier.cpp:178-180).
__global__ void stencil_bounds_kernel(DevGrid g, int P, const double* __restrict__ x, int64_t N,
                                      int* __restrict__ bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    for (int ax = g.d; ax < 3; ++ax) {
        int j0;
        double rel;
        stencil_origin(g, P, ax, x[3 * i + ax], j0, rel);
        if (j0 < 0 || j0 + P > g.n[ax]) atomicExch(bad, 1);
    }
}

}  // namespace

SpreadPlanShape spread_plan_shape(const DevGrid& g, int P) {
    SpreadPlanShape s;
    s.nb[0] = (g.n[0] + TX - 1) / TX;
    s.nb[1] = (g.n[1] + TY - 1) / TY;
    s.nb[2] = (g.n[2] + TZ - 1) / TZ;
    const int T[3] = {TX, TY, TZ};
    s.tiled = true;
    for (int a = 0; a < 3; ++a)
        if (a < g.d && P + T[a] - 1 > g.n[a]) s.tiled = false;
    return s;
}

void launch_spread_bucket(const DevGrid& g, int P, const double* x, int64_t N,
                          const SpreadPlanShape& s, uint32_t* keys, uint32_t* vals, int* bad,
                          cudaStream_t st) {
    if (N == 0) return;
    spread_bucket_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(g, P, x, N, s.nb[0], s.nb[1],
                                                                       s.nb[2], keys, vals, bad);
}

void launch_bucket_offsets(const uint32_t* keys, int64_t N, int nb, int64_t* off, cudaStream_t st,
                           int shift) {
    bucket_offsets_kernel<<<(nb + 1 + 255) / 256, 256, 0, st>>>(keys, N, nb, off, shift);
}

void launch_spread_tiles(const DevGrid& g, const DevWindow& w, const double* x, const double* f,
                         const double* nu, int stresslet, const uint32_t* order,
                         const int64_t* off, const SpreadPlanShape& s, double* out,
                         cudaStream_t st) {
    dim3 grid(s.nb[0], s.nb[1], s.nb[2]);
    const int passes = stresslet ? 3 : 1;
    for (int pass = 0; pass < passes; ++pass)
        spread_tile_kernel<<<grid, SPREAD_THREADS, 0, st>>>(g, w, x, f, nu, stresslet, pass, order,
                                                            off, s.nb[0], s.nb[1], s.nb[2], out);
}

void launch_spread_atomic(const DevGrid& g, const DevWindow& w, const double* x, const double* f,
                          const double* nu, int stresslet, int64_t N, double* out,
                          cudaStream_t st) {
    if (N == 0) return;
    spread_atomic_kernel<<<(unsigned)((N + 127) / 128), 128, 0, st>>>(g, w, x, f, nu, stresslet, N,
                                                                       out);
}

void launch_gather(const DevGrid& g, const DevWindow& w, const double* grid, const double* xt,
                   const uint32_t* order, int64_t Nt, double h3, int accumulate, double* u,
                   cudaStream_t st) {
    if (Nt == 0) return;
    gather_warp_kernel<<<(unsigned)((Nt + 3) / 4), 128, 0, st>>>(g, w, grid, xt, order, Nt, h3,
                                                                  accumulate, u);
}

void launch_stencil_bounds(const DevGrid& g, int P, const double* x, int64_t N, int* bad,
                           cudaStream_t st) {
    if (N == 0 || g.d == 3) return;
    stencil_bounds_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(g, P, x, N, bad);
}

}  // namespace sewald_b200
