// Spread on the fp64 tensor cores (15 <= P <= 20): source-stationary tiles.
//
// Reference: spread /root/reference/proj/src/fourier.cpp:237-274 (stencil
// :168-188). Same taps, stencil origins and wrap; only the summation order
// differs (the north_star allows atomic spreading order).
//
// Sources are bucketed by the B^3 block of their (wrapped) stencil start, so
// every stencil of a block lies in its L^3 region (L = B + P - 1). For one
// component the region is the GEMM
//   R[(a,b), z] = sum_t F[(a,b), t] Z[t, z],   F = f_t wx_t(a) wy_t(b),  Z = wz_t(z)
// ((L^2 x T) . (T x L), each source's taps placed at its offset, zero
// elsewhere), computed with mma.sync.m8n8k4.f64 (256 FMAs per warp
// instruction) and added to the grid with fp64 RED. The grid is zeroed first.
#include "device_common.cuh"
#include "sg_kernels.h"
#include "options.h"

#include <algorithm>
#include <cstdlib>

namespace sewald_b200 {

namespace {

#ifndef SEWALD_SPREAD_MMA_WARPS
#define SEWALD_SPREAD_MMA_WARPS 16
#endif
constexpr int SM_WARPS = SEWALD_SPREAD_MMA_WARPS;
constexpr int SM_THREADS = 32 * SM_WARPS;
#ifndef SEWALD_SPREAD_MMA_PMIN
#define SEWALD_SPREAD_MMA_PMIN 15
#endif
#ifndef SEWALD_SPREAD_MMA_PMAX
#define SEWALD_SPREAD_MMA_PMAX 20
#endif
constexpr int SM_TG = 32;  // sources per table group (8 k-steps of 4)
constexpr int SM_LS = 24;  // padded table width (z: 3 n-blocks of 8)
// Row stride of the cached kernel's tables: 28 doubles (= 12 mod 16) puts the
// four source rows a half warp reads 24 banks apart; at 24 (= 8 mod 16) rows
// t and t + 2 shared banks and every table load conflicted 2-way.
#ifndef SEWALD_SM_LSP
#define SEWALD_SM_LSP 28
#endif
constexpr int SM_LSP = SEWALD_SM_LSP;

// v >= 0 reduced mod n by subtraction (a region coordinate exceeds the grid
// by less than the region edge): replaces an integer division per flushed row
__device__ __forceinline__ int wrap_up(int v, int n) {
    while (v >= n) v -= n;
    return v;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int L>
__global__ void __launch_bounds__(SM_THREADS)
spread_tile_mma_kernel(DevGrid g, int P, int B, int ntx, int nty, int ntz, int64_t tile0, const double* __restrict__ W,
                       const int4* __restrict__ SW, const double* __restrict__ STR, int C,
                       const int64_t* __restrict__ off, double* __restrict__ out) {
    constexpr int ROWS = L * L;
    constexpr int RB = (ROWS + 7) / 8;
    constexpr int RBW = (RB + SM_WARPS - 1) / SM_WARPS;  // row blocks per warp
    __shared__ __align__(16) double wxf[SM_TG][SM_LS];    // f_t wx_t(a), zero padded
    __shared__ __align__(16) double wy[SM_TG][SM_LS];
    __shared__ __align__(16) double wz[SM_TG][SM_LS];

    const int64_t tile = tile0 + blockIdx.x;
    const int64_t p0 = off[tile], p1 = off[tile + 1];
    if (p0 >= p1) return;
    const int tz = (int)(tile % ntz);
    const int ty = (int)((tile / ntz) % nty);
    const int tx = (int)(tile / ((int64_t)ntz * nty));
    const int X0 = tx * B, Y0 = ty * B, Z0 = tz * B;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t cs = (int64_t)g.n[0] * g.n[1] * g.n[2];
    const int ngroups = (int)((p1 - p0 + SM_TG - 1) / SM_TG);

    for (int c = 0; c < C; ++c) {
        double acc[RBW][3][2];
#pragma unroll
        for (int j = 0; j < RBW; ++j)
#pragma unroll
            for (int nb = 0; nb < 3; ++nb) acc[j][nb][0] = acc[j][nb][1] = 0.0;
        for (int grp = 0; grp < ngroups; ++grp) {
            const int64_t q0 = p0 + (int64_t)grp * SM_TG;
            const int T = (int)min((int64_t)SM_TG, p1 - q0);
            __syncthreads();
            // tables: warp per source, lane = region index
            for (int t = warp; t < SM_TG; t += SM_WARPS) {
                int4 sw = make_int4(0, 0, 0, 0);
                double f = 0.0;
                if (t < T) {
                    sw = SW[q0 + t];
                    f = STR[(q0 + t) * C + c];
                }
                if (lane < SM_LS) {
                    const int k = lane;
                    double vx = 0.0, vy = 0.0, vz = 0.0;
                    if (t < T && k < L) {
                        const double* w = W + (q0 + t) * 3 * P;
                        const int kx = k - (sw.x - X0), ky = k - (sw.y - Y0), kz = k - (sw.z - Z0);
                        if (kx >= 0 && kx < P) vx = __ldg(w + kx);
                        if (ky >= 0 && ky < P) vy = __ldg(w + P + ky);
                        if (kz >= 0 && kz < P) vz = __ldg(w + 2 * P + kz);
                    }
                    wxf[t][k] = f * vx;
                    wy[t][k] = vy;
                    wz[t][k] = vz;
                }
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < RBW; ++j) {
                const int rb = warp + j * SM_WARPS;
                if (rb < RB) {
                    const int row = rb * 8 + (lane >> 2);  // A / C row of this lane
                    const int a = row / L, b = row - a * L;
#pragma unroll
                    for (int ks = 0; ks < SM_TG / 4; ++ks) {
                        const int t = ks * 4 + (lane & 3);
                        const double af = wxf[t][a] * wy[t][b];
                        const int tb = ks * 4 + (lane & 3);
#pragma unroll
                        for (int nb = 0; nb < 3; ++nb) dmma(acc[j][nb][0], acc[j][nb][1], af, wz[tb][nb * 8 + (lane >> 2)]);
                    }
                }
            }
        }
        // add the region to the grid
        double* oc = out + (int64_t)c * cs;
#pragma unroll
        for (int j = 0; j < RBW; ++j) {
            const int rb = warp + j * SM_WARPS;
            if (rb >= RB) continue;
            const int row = rb * 8 + (lane >> 2);
            if (row >= ROWS) continue;
            const int a = row / L, b = row - a * L;
            int gx = X0 + a, gy = Y0 + b;
            if (g.d > 0) gx = wrap_up(gx, g.n[0]); else if (gx >= g.n[0]) continue;
            if (g.d > 1) gy = wrap_up(gy, g.n[1]); else if (gy >= g.n[1]) continue;
            double* col = oc + ((int64_t)gx * g.n[1] + gy) * g.n[2];
#pragma unroll
            for (int nb = 0; nb < 3; ++nb)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int z = nb * 8 + 2 * (lane & 3) + h;
                    if (z >= L) continue;
                    int gz = Z0 + z;
                    if (g.d > 2) gz = wrap_up(gz, g.n[2]); else if (gz >= g.n[2]) continue;
                    const double v = acc[j][nb][h];
                    if (v != 0.0) atomicAdd(col + gz, v);
                }
        }
    }
}

// Same contraction with every source table of a tile chunk (up to CT_TMAX
// sources) staged once in shared memory and reused by all components: the
// per-group table rebuild (global tap loads + two block barriers per group
// and component) of the kernel above leaves the tensor pipe waiting on memory.
// Each warp owns consecutive row blocks (so its rows span ~2 region x rows)
// and visits only the k-steps whose points' x windows reach those rows: with
// the points of a tile ordered by their x offset (SEWALD_OPT_SPREAD_SORT)
// that is a contiguous k range, ~3/4 of the chunk instead of all of it; the
// point's z taps and strength are loaded once per k-step for all the warp's
// row blocks. c2 4.31 -> 3.77 ms, c3 12.18 -> 10.42 ms (unsorted 4.52 /
// 11.84: the k range is then the whole chunk).
constexpr int CT_TMAX = 256;
constexpr int CT_CMAX = 9;

// + per-point x offsets and per-row k-step ranges
size_t cached_smem_bytes() {
    return sizeof(double) * (size_t)CT_TMAX * (3 * SM_LSP + CT_CMAX) + sizeof(int) * (CT_TMAX + 2 * SM_LS);
}

// Fused taps (FUSED = true): the chunk's window taps are evaluated here from
// the positions (fourier.cpp:168-188, same expression as the taps kernel)
// instead of being read from a taps array written by a separate kernel: no
// 3 P doubles per source through HBM and one launch less per spread. One
// thread per (axis, source), axis-major, so a warp's PKB coefficient reads
// are uniform. Measured at c2 (C = 3): 4.31 vs 4.40 ms with the taps kernel;
// c3 (C = 9): 12.7 vs 12.2 ms, so it is the default for 3 components only.
// With the taps evaluated four at a time (window_taps) the staging got
// cheaper: c2 3.52 -> 3.26 ms, xi = 63 5.57 -> 4.96; c3 fused (option 2)
// 10.22 vs 10.01 ms unfused, still off for C = 9.
struct FusedSrc {
    const double* x;        // positions of the spread slice (AoS)
    const double* f;        // strengths
    const double* nu;       // stresslet orientations or null
    const uint32_t* order;  // bucket-sorted -> slice index
    DevWindow win;
};

template <int L, bool FUSED = false>
__global__ void __launch_bounds__(SM_THREADS)
spread_tile_mma_cached_kernel(DevGrid g, int P, int B, int ntx, int nty, int ntz, int64_t tile0,
                              const double* __restrict__ W, const int4* __restrict__ SW,
                              const double* __restrict__ STR, int C, const int64_t* __restrict__ off,
                              double* __restrict__ out, const FusedSrc* __restrict__ fsrc) {
    constexpr int ROWS = L * L;
    constexpr int RB = (ROWS + 7) / 8;
    constexpr int RBW = (RB + SM_WARPS - 1) / SM_WARPS;  // row blocks per warp
    extern __shared__ __align__(16) double csm[];
    double(*wx)[SM_LSP] = reinterpret_cast<double(*)[SM_LSP]>(csm);
    double(*wy)[SM_LSP] = reinterpret_cast<double(*)[SM_LSP]>(csm + CT_TMAX * SM_LSP);
    double(*wz)[SM_LSP] = reinterpret_cast<double(*)[SM_LSP]>(csm + 2 * CT_TMAX * SM_LSP);
    double* fs = csm + 3 * CT_TMAX * SM_LSP;  // [CT_TMAX][C]
    int* ox = reinterpret_cast<int*>(fs + CT_TMAX * CT_CMAX);  // [CT_TMAX] x offset of each point in the region
    int* kmin = ox + CT_TMAX;                                  // [SM_LS] first / last k-step reaching row a
    int* kmax = kmin + SM_LS;

    const int64_t tile = tile0 + blockIdx.x;
    const int64_t p0 = off[tile], p1 = off[tile + 1];
    if (p0 >= p1) return;
    const int tz = (int)(tile % ntz);
    const int ty = (int)((tile / ntz) % nty);
    const int tx = (int)(tile / ((int64_t)ntz * nty));
    const int X0 = tx * B, Y0 = ty * B, Z0 = tz * B;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t cs = (int64_t)g.n[0] * g.n[1] * g.n[2];
    // consecutive row blocks per warp (4 or 5 for L = 23), so that a warp's rows
    // cover few region x rows and few k-steps
    const int nrb = RB / SM_WARPS + (warp < RB % SM_WARPS ? 1 : 0);
    const int rb0 = warp * (RB / SM_WARPS) + min(warp, RB % SM_WARPS);
    const int a_first = (rb0 * 8) / L, a_last = nrb ? min((rb0 + nrb) * 8 - 1, ROWS - 1) / L : -1;

    for (int64_t q0 = p0; q0 < p1; q0 += CT_TMAX) {
        const int T = (int)min((int64_t)CT_TMAX, p1 - q0);
        const int ngroups = (T + SM_TG - 1) / SM_TG;
        __syncthreads();
        if (threadIdx.x < SM_LS) {
            kmin[threadIdx.x] = 1 << 20;
            kmax[threadIdx.x] = -1;
        }
        if (FUSED) {
            // zero the padding rows of the chunk's tables; the (axis, source,
            // half) items below write whole rows (taps and the zeros around them)
            const int rows = ngroups * SM_TG;
            for (int e = T * SM_LSP + threadIdx.x; e < rows * SM_LSP; e += SM_THREADS) {
                (&wx[0][0])[e] = 0.0;
                (&wy[0][0])[e] = 0.0;
                (&wz[0][0])[e] = 0.0;
            }
            for (int e = threadIdx.x; e < rows * C; e += SM_THREADS) {
                const int t = e / C, c = e - t * C;
                double v = 0.0;
                if (t < T) {
                    const int64_t i = fsrc->order[q0 + t];
                    if (C == 3) {
                        v = fsrc->f[3 * i + c];
                    } else {  // stresslet: q_l nu_m (fourier.cpp:253-258)
                        const int l = c / 3, m = c - 3 * l;
                        v = fsrc->f[3 * i + l] * fsrc->nu[3 * i + m];
                    }
                }
                fs[e] = v;
            }
            // work item = (axis, source, half of the taps): more independent
            // items than threads per chunk (c2: 1464 for 512 threads)
            const int half = ((P + 1) / 2 + 3) & ~3;
            for (int e = threadIdx.x; e < 6 * T; e += SM_THREADS) {
                const int hh = e / (3 * T), e2 = e - hh * 3 * T;
                const int ax = e2 / T, t = e2 - ax * T;
                const int64_t i = fsrc->order[q0 + t];
                int j0;
                double rel;
                stencil_origin(g, P, ax, fsrc->x[3 * i + ax], j0, rel);
                const int sw = ax < g.d ? wrap_index(j0, g.n[ax]) : j0;
                const int o = sw - (ax == 0 ? X0 : (ax == 1 ? Y0 : Z0));
                if (ax == 0 && hh == 0) ox[t] = o;
                double* row = ax == 0 ? wx[t] : (ax == 1 ? wy[t] : wz[t]);
                const int pb = hh ? min(half, P) : 0, pe = hh ? P : min(half, P);
                window_taps(fsrc->win, j0, rel, g.h, row + o, 1, pb, pe);
                // zeros of this half's side of the row: [0, o) / [o + P, SM_LS)
                if (hh == 0) for (int k = 0; k < o; ++k) row[k] = 0.0;
                else for (int k = o + P; k < SM_LS; ++k) row[k] = 0.0;
            }
        } else {
            // tables of the chunk: warp per source, lane = region index
            for (int t = warp; t < ngroups * SM_TG; t += SM_WARPS) {
                int4 sw = make_int4(0, 0, 0, 0);
                if (t < T) sw = SW[q0 + t];
                if (lane == 0 && t < T) ox[t] = sw.x - X0;
                if (lane < SM_LS) {
                    const int k = lane;
                    double vx = 0.0, vy = 0.0, vz = 0.0;
                    if (t < T && k < L) {
                        const double* w = W + (q0 + t) * 3 * P;
                        const int kx = k - (sw.x - X0), ky = k - (sw.y - Y0), kz = k - (sw.z - Z0);
                        if (kx >= 0 && kx < P) vx = __ldg(w + kx);
                        if (ky >= 0 && ky < P) vy = __ldg(w + P + ky);
                        if (kz >= 0 && kz < P) vz = __ldg(w + 2 * P + kz);
                    }
                    wx[t][k] = vx;
                    wy[t][k] = vy;
                    wz[t][k] = vz;
                }
                if (lane < C) fs[t * C + lane] = t < T ? STR[(q0 + t) * C + lane] : 0.0;
            }
        }
        __syncthreads();
        // k-steps (4 points each) whose x windows reach region row a: a
        // contiguous range [kmin[a], kmax[a]] when the points are ordered by
        // their x offset (SEWALD_OPT_SPREAD_SORT), a conservative cover otherwise
        for (int k = threadIdx.x; k < ngroups * (SM_TG / 4); k += SM_THREADS) {
            int lo = 1 << 20, hi = -(1 << 20);
            for (int q = 4 * k; q < min(4 * k + 4, T); ++q) {
                lo = min(lo, ox[q]);
                hi = max(hi, ox[q] + P - 1);
            }
            for (int a = max(lo, 0); a <= min(hi, L - 1); ++a) {
                atomicMin(&kmin[a], k);
                atomicMax(&kmax[a], k);
            }
        }
        __syncthreads();
        for (int c = 0; c < C; ++c) {
            double acc[RBW][3][2];
#pragma unroll
            for (int j = 0; j < RBW; ++j)
#pragma unroll
                for (int nb = 0; nb < 3; ++nb) acc[j][nb][0] = acc[j][nb][1] = 0.0;
            // this warp's consecutive row blocks rb0 .. rb0 + nrb - 1 span region
            // rows a_first..a_last; only k-steps reaching them are visited
            int ra[RBW], rbv[RBW];
#pragma unroll
            for (int j = 0; j < RBW; ++j) {
                const int row = (rb0 + j) * 8 + (lane >> 2);  // A / C row of this lane
                ra[j] = row / L;
                rbv[j] = row - ra[j] * L;
            }
            int kb = 1 << 20, ke = -1;
            for (int a = a_first; a <= a_last; ++a) {
                kb = min(kb, kmin[a]);
                ke = max(ke, kmax[a]);
            }
            for (int k = kb; k <= ke; ++k) {
                const int t = k * 4 + (lane & 3);
                const double f = fs[t * C + c];
                double bz[3];
#pragma unroll
                for (int nb = 0; nb < 3; ++nb) bz[nb] = wz[t][nb * 8 + (lane >> 2)];
#pragma unroll
                for (int j = 0; j < RBW; ++j) {
                    if (j < nrb) {
                        const double af = (f * wx[t][ra[j]]) * wy[t][rbv[j]];
#pragma unroll
                        for (int nb = 0; nb < 3; ++nb) dmma(acc[j][nb][0], acc[j][nb][1], af, bz[nb]);
                    }
                }
            }
            // add the region to the grid
            double* oc = out + (int64_t)c * cs;
#pragma unroll
            for (int j = 0; j < RBW; ++j) {
                const int rb = rb0 + j;
                if (j >= nrb) continue;
                const int row = rb * 8 + (lane >> 2);
                if (row >= ROWS) continue;
                const int a = row / L, b = row - a * L;
                int gx = X0 + a, gy = Y0 + b;
                if (gx >= g.n[0]) {
                    if (g.d <= 0) continue;
                    gx = wrap_up(gx, g.n[0]);
                }
                if (gy >= g.n[1]) {
                    if (g.d <= 1) continue;
                    gy = wrap_up(gy, g.n[1]);
                }
                double* col = oc + ((int64_t)gx * g.n[1] + gy) * g.n[2];
#pragma unroll
                for (int nb = 0; nb < 3; ++nb)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int z = nb * 8 + 2 * (lane & 3) + h;
                        if (z >= L) continue;
                        int gz = Z0 + z;
                        if (gz >= g.n[2]) {  // rare: the region crosses the grid's end
                            if (g.d <= 2) continue;
                            gz = wrap_up(gz, g.n[2]);
                        }
                        const double v = acc[j][nb][h];
                        if (v != 0.0) atomicAdd(col + gz, v);
                    }
            }
        }
    }
}

// Wide windows (20 < P <= 32, e.g. the Gaussian window of c4 at P = 32;
// with SEWALD_OPT_SPREAD_SORT each row block visits only the k-steps that
// reach it, c4 9.55 -> 8.50 ms):
// B = 8, region L = P + 7 <= 39, z padded to LS = 40 (5 n-blocks). The whole
// tile's source tables stay in shared memory (up to WT_TMAX sources per pass),
// each warp owns whole row blocks and sweeps all sources for them with every
// n-block in flight, then flushes the row block with fp64 RED. Sources beyond
// WT_TMAX per tile are handled in further passes (more RED, same result).
constexpr int WT_TMAX = 128;
constexpr int WT_LS = 40;
#ifndef SEWALD_WT_PAD
#define SEWALD_WT_PAD 1
#endif
__host__ __device__ constexpr int wide_table_stride(int LS) {
    return (!SEWALD_WT_PAD || LS % 16 == 4 || LS % 16 == 12) ? LS : LS + 4;
}
constexpr int WT_WARPS = 16;
#ifndef SEWALD_SPREAD_RS_WARPS
#define SEWALD_SPREAD_RS_WARPS 8
#endif
#ifndef SEWALD_SPREAD_RS_MINB
#define SEWALD_SPREAD_RS_MINB 2
#endif

// Also used for 15 <= P <= 20 (L = 23 / 19, LS = 24) as the row-sweep form
// (SEWALD_OPT_SPREAD_ROWSWEEP): few registers per warp, so several tile
// CTAs share an SM and one's table staging overlaps another's MMAs.
template <int L, int LS = WT_LS, int NW = WT_WARPS, int MINB = 1>
__global__ void __launch_bounds__(32 * NW, MINB)
spread_tile_mma_wide_kernel(DevGrid g, int P, int B, int ntx, int nty, int ntz, int64_t tile0,
                            const double* __restrict__ W, const int4* __restrict__ SW,
                            const double* __restrict__ STR, int C, const int64_t* __restrict__ off,
                            double* __restrict__ out) {
    constexpr int WT_LS = LS;
    constexpr int WT_WARPS = NW;
    constexpr int ROWS = L * L;
    constexpr int RB = (ROWS + 7) / 8;
    constexpr int NB = WT_LS / 8;
    // table row stride: 4 or 12 mod 16 doubles, so the four source rows a half
    // warp reads lie on distinct banks (at LS = 40 / 24 rows t and t + 2 collide)
    constexpr int LSP = wide_table_stride(LS);
    extern __shared__ __align__(16) double wsm[];
    double(*wxf)[LSP] = reinterpret_cast<double(*)[LSP]>(wsm);                     // f_t wx_t(a)
    double(*wx)[LSP] = reinterpret_cast<double(*)[LSP]>(wsm + WT_TMAX * LSP);      // wx_t(a)
    double(*wy)[LSP] = reinterpret_cast<double(*)[LSP]>(wsm + 2 * WT_TMAX * LSP);  // wy_t(b)
    double(*wz)[LSP] = reinterpret_cast<double(*)[LSP]>(wsm + 3 * WT_TMAX * LSP);  // wz_t(z)
    int* ox = reinterpret_cast<int*>(wsm + 4 * WT_TMAX * LSP);  // [WT_TMAX] x offset of each point
    int* kmin = ox + WT_TMAX;                                      // [WT_LS] first / last k-step reaching row a
    int* kmax = kmin + WT_LS;

    const int64_t tile = tile0 + blockIdx.x;
    const int64_t p0 = off[tile], p1 = off[tile + 1];
    if (p0 >= p1) return;
    const int tz = (int)(tile % ntz);
    const int ty = (int)((tile / ntz) % nty);
    const int tx = (int)(tile / ((int64_t)ntz * nty));
    const int X0 = tx * B, Y0 = ty * B, Z0 = tz * B;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t cs = (int64_t)g.n[0] * g.n[1] * g.n[2];

    for (int64_t q0 = p0; q0 < p1; q0 += WT_TMAX) {
        const int T = (int)min((int64_t)WT_TMAX, p1 - q0);
        const int T4 = (T + 3) & ~3;
        __syncthreads();
        if (threadIdx.x < WT_LS) {
            kmin[threadIdx.x] = 1 << 20;
            kmax[threadIdx.x] = -1;
        }
        for (int t = warp; t < T4; t += WT_WARPS) {
            int4 sw = make_int4(0, 0, 0, 0);
            if (t < T) sw = SW[q0 + t];
            if (lane == 0 && t < T) ox[t] = sw.x - X0;
            for (int k = lane; k < WT_LS; k += 32) {
                double vx = 0.0, vy = 0.0, vz = 0.0;
                if (t < T && k < L) {
                    const double* w = W + (q0 + t) * 3 * P;
                    const int kx = k - (sw.x - X0), ky = k - (sw.y - Y0), kz = k - (sw.z - Z0);
                    if (kx >= 0 && kx < P) vx = __ldg(w + kx);
                    if (ky >= 0 && ky < P) vy = __ldg(w + P + ky);
                    if (kz >= 0 && kz < P) vz = __ldg(w + 2 * P + kz);
                }
                wx[t][k] = vx;
                wy[t][k] = vy;
                wz[t][k] = vz;
            }
        }
        __syncthreads();
        // k-steps whose points' x windows reach region row a (contiguous when the
        // points are ordered by x offset, SEWALD_OPT_SPREAD_SORT)
        for (int k = threadIdx.x; k < T4 / 4; k += 32 * WT_WARPS) {
            int lo = 1 << 20, hi = -(1 << 20);
            for (int q = 4 * k; q < min(4 * k + 4, T); ++q) {
                lo = min(lo, ox[q]);
                hi = max(hi, ox[q] + P - 1);
            }
            for (int a = max(lo, 0); a <= min(hi, L - 1); ++a) {
                atomicMin(&kmin[a], k);
                atomicMax(&kmax[a], k);
            }
        }
        for (int c = 0; c < C; ++c) {
            __syncthreads();
            for (int e = threadIdx.x; e < T4 * WT_LS; e += 32 * WT_WARPS) {
                const int t = e / WT_LS, k = e - t * WT_LS;
                wxf[t][k] = t < T ? STR[(q0 + t) * C + c] * wx[t][k] : 0.0;
            }
            __syncthreads();
            double* oc = out + (int64_t)c * cs;
            for (int rb = warp; rb < RB; rb += WT_WARPS) {
                const int row = rb * 8 + (lane >> 2);
                const int a = row / L, b = row - a * L;
                double acc[NB][2];
#pragma unroll
                for (int nb = 0; nb < NB; ++nb) acc[nb][0] = acc[nb][1] = 0.0;
                const int a_lo = (rb * 8) / L, a_hi = min(rb * 8 + 7, ROWS - 1) / L;
                const int kb = min(kmin[a_lo], kmin[a_hi]), ke = max(kmax[a_lo], kmax[a_hi]);
                for (int ks = kb; ks <= ke; ++ks) {
                    const int t = ks * 4 + (lane & 3);
                    const double af = wxf[t][a] * wy[t][b];
#pragma unroll
                    for (int nb = 0; nb < NB; ++nb) dmma(acc[nb][0], acc[nb][1], af, wz[t][nb * 8 + (lane >> 2)]);
                }
                if (row >= ROWS) continue;
                int gx = X0 + a, gy = Y0 + b;
                if (g.d > 0) gx = wrap_up(gx, g.n[0]); else if (gx >= g.n[0]) continue;
                if (g.d > 1) gy = wrap_up(gy, g.n[1]); else if (gy >= g.n[1]) continue;
                double* col = oc + ((int64_t)gx * g.n[1] + gy) * g.n[2];
#pragma unroll
                for (int nb = 0; nb < NB; ++nb)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int z = nb * 8 + 2 * (lane & 3) + h;
                        if (z >= L) continue;
                        int gz = Z0 + z;
                        if (g.d > 2) gz = wrap_up(gz, g.n[2]); else if (gz >= g.n[2]) continue;
                        const double v = acc[nb][h];
                        if (v != 0.0) atomicAdd(col + gz, v);
                    }
            }
        }
    }
}

}  // namespace

SpreadMmaShape spread_mma_shape(const DevGrid& g, int P) {
    SpreadMmaShape s{};
    const int Lenv = option(SEWALD_OPT_SPREAD_MMA_L);
    s.L = (Lenv == 19 && P <= 19) ? 19 : 23;  // the region must hold a P-wide stencil (B >= 1)
    if (P > 20 && P <= 32) {  // wide windows: B = 8, L = P + 7 (spread_tile_mma_wide_kernel)
        s.ok = (int64_t)g.n[0] * g.n[1] * g.n[2] < (int64_t(1) << 31);
        s.B = 8;
        s.L = P + 7;
        for (int ax = 0; ax < 3; ++ax) s.nt[ax] = (g.n[ax] + s.B - 1) / s.B;
        s.ntiles = (int64_t)s.nt[0] * s.nt[1] * s.nt[2];
        if (s.ntiles >= (int64_t(1) << 31)) s.ok = false;
        s.sub = (option(SEWALD_OPT_SPREAD_SORT) != 0 && s.ntiles < (int64_t(1) << 26)) ? 6 : 0;
        return s;
    }
    // The region work is fixed by L (L^2 x 24 per 32 sources) while the sweep's
    // shrinks as P^3: measured, the tensor-core form wins at P = 16 (c2: 4.9
    // vs 7.1 ms) and P = 18 (c3: 15.1 vs 23.2 ms) and loses at P = 14 (c5:
    // 22.5 vs 14.0 ms).
    s.ok = P >= SEWALD_SPREAD_MMA_PMIN && P <= SEWALD_SPREAD_MMA_PMAX;
    s.B = std::max(1, s.L + 1 - P);
    for (int ax = 0; ax < 3; ++ax) s.nt[ax] = (g.n[ax] + s.B - 1) / s.B;
    s.ntiles = (int64_t)s.nt[0] * s.nt[1] * s.nt[2];
    if (s.ntiles >= (int64_t(1) << 31) || (int64_t)g.n[0] * g.n[1] * g.n[2] >= (int64_t(1) << 31)) s.ok = false;
    // points of a tile ordered by their (x, y) stencil offset: the cached tile
    // kernel then skips k-steps that cannot reach a row block
    s.sub = (option(SEWALD_OPT_SPREAD_SORT) != 0 && s.ntiles < (int64_t(1) << 26)) ? 6 : 0;
    return s;
}

void launch_spread_mma_bucket(const DevGrid& g, int P, const SpreadMmaShape& s, const double* x, int64_t N,
                              uint32_t* keys, uint32_t* vals, int* bad, cudaStream_t st) {
    TileShape ts{};
    ts.B = s.B;
    ts.L = s.L;
    for (int ax = 0; ax < 3; ++ax) ts.nt[ax] = s.nt[ax];
    ts.ntiles = s.ntiles;
    launch_tile_bucket(g, P, ts, x, N, keys, vals, bad, st, s.sub);
}

bool spread_mma_fused_ok(const SpreadMmaShape& s, int C) {
    // 1: three-component strengths only; 2: also the stresslet's nine
    return s.ok && s.L <= 23 && (C == 3 || option(SEWALD_OPT_SPREAD_FUSED) == 2) &&
           option(SEWALD_OPT_SPREAD_CACHED) != 0 && !option(SEWALD_OPT_SPREAD_ROWSWEEP) &&
           option(SEWALD_OPT_SPREAD_FUSED) != 0;
}

int launch_spread_mma_fused(const DevGrid& g, const DevWindow& w, int P, const SpreadMmaShape& s, const double* x,
                            const double* f, const double* nu, const uint32_t* order, int C, const int64_t* off,
                            double* out, void* fsrc_dev, cudaStream_t st) {
    cudaMemsetAsync(out, 0, sizeof(double) * C * (size_t)g.n[0] * g.n[1] * g.n[2], st);
    FusedSrc h{x, f, nu, order, w};
    cudaMemcpyAsync(fsrc_dev, &h, sizeof(FusedSrc), cudaMemcpyHostToDevice, st);
    const size_t sm = cached_smem_bytes();
    auto kern = s.L == 23 ? spread_tile_mma_cached_kernel<23, true> : spread_tile_mma_cached_kernel<19, true>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    for (int64_t a = 0; a < s.ntiles; a += (int64_t)1 << 30) {
        const int64_t n = std::min<int64_t>(s.ntiles - a, (int64_t)1 << 30);
        kern<<<(unsigned)n, SM_THREADS, sm, st>>>(g, P, s.B, s.nt[0], s.nt[1], s.nt[2], a, nullptr, nullptr, nullptr, C,
                                                  off, out, static_cast<const FusedSrc*>(fsrc_dev));
    }
    return 1;
}

size_t fused_src_bytes() { return sizeof(FusedSrc); }

int launch_spread_mma(const DevGrid& g, int P, const SpreadMmaShape& s, const double* W, const int4* SW,
                      const double* STR, int C, const int64_t* off, double* out, cudaStream_t st) {
    cudaMemsetAsync(out, 0, sizeof(double) * C * (size_t)g.n[0] * g.n[1] * g.n[2], st);
    const bool cached = option(SEWALD_OPT_SPREAD_CACHED) != 0;  // 0: per-group tables (A/B)
    for (int64_t a = 0; a < s.ntiles; a += (int64_t)1 << 30) {
        const int64_t n = std::min<int64_t>(s.ntiles - a, (int64_t)1 << 30);
        if (s.L > 23) {
            const size_t sm = sizeof(double) * 4 * WT_TMAX * wide_table_stride(WT_LS) + sizeof(int) * (WT_TMAX + 2 * WT_LS);
            auto kern = s.L <= 31 ? spread_tile_mma_wide_kernel<31>
                                  : (s.L <= 35 ? spread_tile_mma_wide_kernel<35> : spread_tile_mma_wide_kernel<39>);
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            kern<<<(unsigned)n, 32 * WT_WARPS, sm, st>>>(g, P, s.B, s.nt[0], s.nt[1], s.nt[2], a, W, SW, STR, C, off,
                                                        out);
        } else if (option(SEWALD_OPT_SPREAD_ROWSWEEP)) {
            const size_t sm = sizeof(double) * 4 * WT_TMAX * wide_table_stride(24) + sizeof(int) * (WT_TMAX + 2 * 24);
            auto kern = s.L == 23 ? spread_tile_mma_wide_kernel<23, 24, SEWALD_SPREAD_RS_WARPS, SEWALD_SPREAD_RS_MINB>
                                  : spread_tile_mma_wide_kernel<19, 24, SEWALD_SPREAD_RS_WARPS, SEWALD_SPREAD_RS_MINB>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            kern<<<(unsigned)n, 32 * SEWALD_SPREAD_RS_WARPS, sm, st>>>(g, P, s.B, s.nt[0], s.nt[1], s.nt[2], a, W, SW,
                                                                      STR, C, off, out);
        } else if (cached && C <= CT_CMAX) {
            const size_t sm = cached_smem_bytes();
            auto kern = s.L == 23 ? spread_tile_mma_cached_kernel<23> : spread_tile_mma_cached_kernel<19>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            kern<<<(unsigned)n, SM_THREADS, sm, st>>>(g, P, s.B, s.nt[0], s.nt[1], s.nt[2], a, W, SW, STR, C, off, out,
                                                      nullptr);
        } else if (s.L == 23)
            spread_tile_mma_kernel<23><<<(unsigned)n, SM_THREADS, 0, st>>>(g, P, s.B, s.nt[0], s.nt[1], s.nt[2], a, W,
                                                                           SW, STR, C, off, out);
        else
            spread_tile_mma_kernel<19><<<(unsigned)n, SM_THREADS, 0, st>>>(g, P, s.B, s.nt[0], s.nt[1], s.nt[2], a, W,
                                                                           SW, STR, C, off, out);
    }
    return 1;
}

}  // namespace sewald_b200
