// Gather through shared-memory grid tiles (P <= 16).
//
// Reference: gather /root/reference/proj/src/fourier.cpp:276-309 (stencil
// :168-188). Same taps, stencil origins and wrap; only the summation order
// differs.
//
// Targets are bucketed by the B x B x B block of their (wrapped) stencil
// start. One CTA owns one block: it stages the L^3 region (L = B + P - 1)
// that every stencil of the block lies in, one flow component at a time,
// into shared memory, then each warp evaluates whole targets from it (lanes
// = 16 z taps x 2 y rows, warp reduction). The L2 stream per target drops
// from P^3 x 3 values (warp-per-target gather) to the region share, and the
// tap loop reads shared memory only. Every target is owned by one block, so
// results are written without atomics.
#include "device_common.cuh"
#include "sg_kernels.h"
#include "options.h"

#include <algorithm>
#include <cstdlib>

namespace sewald_b200 {

namespace {

constexpr int GT_WARPS = 8;
constexpr int GT_THREADS = 32 * GT_WARPS;
constexpr int GT_PMAX = 16;

__global__ void tile_bucket_kernel(DevGrid g, int P, int B, int ntx, int nty, int ntz, const double* __restrict__ x,
                                   int64_t N, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                   int* __restrict__ bad, int sub) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    int t[3], l[3];
    const int nt[3] = {ntx, nty, ntz};
    for (int ax = 0; ax < 3; ++ax) {
        int j0;
        double rel;
        stencil_origin(g, P, ax, x[3 * i + ax], j0, rel);
        if (ax < g.d) {
            j0 = wrap_index(j0, g.n[ax]);
        } else if (j0 < 0 || j0 + P > g.n[ax]) {
            atomicExch(bad, 1);
            j0 = 0;
        }
        t[ax] = min(j0 / B, nt[ax] - 1);
        l[ax] = min(j0 - t[ax] * B, 7);
    }
    // sub = 6: the low bits order a tile's points by the (x, y) offset of their
    // stencil start inside the tile (the spread skips MMA steps whose points
    // cannot reach a row block)
    const uint32_t lo = sub ? (uint32_t)((l[0] << 3) | l[1]) : 0u;
    keys[i] = ((uint32_t)(((int64_t)t[0] * nty + t[1]) * ntz + t[2]) << sub) | lo;
    vals[i] = (uint32_t)i;
}

__global__ void __launch_bounds__(GT_THREADS)
gather_tile_kernel(DevGrid g, int P, int B, int L, int ntx, int nty, int ntz, int64_t tile0,
                   const double* __restrict__ W, const int4* __restrict__ SW, const int64_t* __restrict__ off,
                   const double* __restrict__ grid, double h3, int accumulate, double* __restrict__ u) {
    extern __shared__ double sm[];
    const int64_t tile = tile0 + blockIdx.x;
    const int64_t p0 = off[tile], p1 = off[tile + 1];
    if (p0 >= p1) return;
    const int tz = (int)(tile % ntz);
    const int ty = (int)((tile / ntz) % nty);
    const int tx = (int)(tile / ((int64_t)ntz * nty));
    const int X0 = tx * B, Y0 = ty * B, Z0 = tz * B;
    const int L2 = L * L, L3 = L2 * L;
    // region + zero pad (lanes past the stencil read it with zero weight)
    const int pad = 2 * GT_PMAX * L + 2 * GT_PMAX;
    double* region = sm;
    double* wsm = sm + L3 + pad;  // per warp: 3 * P taps
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* wt_s = wsm + warp * 3 * GT_PMAX;
    int* rowoff = reinterpret_cast<int*>(wsm + GT_WARPS * 3 * GT_PMAX);  // L^2 row offsets (-1: outside)
    int* zoff = rowoff + L2;                                            // L z offsets (-1: outside)
    for (int e = threadIdx.x; e < pad; e += GT_THREADS) region[L3 + e] = 0.0;
    for (int row = threadIdx.x; row < L2; row += GT_THREADS) {
        const int i = row / L, j = row - i * L;
        int gx = X0 + i, gy = Y0 + j;
        bool ok = true;
        if (g.d > 0) gx %= g.n[0]; else ok = gx < g.n[0];
        if (g.d > 1) gy %= g.n[1]; else ok = ok && gy < g.n[1];
        rowoff[row] = ok ? (gx * g.n[1] + gy) * g.n[2] : -1;
    }
    if (threadIdx.x < L) {
        int gz = Z0 + threadIdx.x;
        bool ok = true;
        if (g.d > 2) gz %= g.n[2]; else ok = gz < g.n[2];
        zoff[threadIdx.x] = ok ? gz : -1;
    }

    const int64_t cs = (int64_t)g.n[0] * g.n[1] * g.n[2];
    const int z = lane & 15, half = lane >> 4;
    for (int c = 0; c < 3; ++c) {
        __syncthreads();
        const double* gc = grid + c * cs;
        // cp.async row copies: L z-values per (x, y) row, offsets precomputed
        for (int row = warp; row < L2; row += GT_WARPS) {
            const int ro = rowoff[row];
            if (lane < L) {
                double* dst = region + row * L + lane;
                const int zo = zoff[lane];
                if (ro >= 0 && zo >= 0) {
                    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gc + ro + zo));
                } else {
                    *dst = 0.0;
                }
            }
        }
        asm volatile("cp.async.wait_all;\n" ::);
        __syncthreads();
        for (int64_t t = p0 + warp; t < p1; t += GT_WARPS) {
            __syncwarp();
            const double* wt = W + t * 3 * P;
            for (int q = lane; q < 3 * P; q += 32) wt_s[(q / P) * GT_PMAX + q % P] = __ldg(wt + q);
            const int4 sw = SW[t];
            __syncwarp();
            const double wz = z < P ? wt_s[2 * GT_PMAX + z] : 0.0;
            double cy[GT_PMAX / 2];
#pragma unroll
            for (int m = 0; m < GT_PMAX / 2; ++m) {
                const int b = half + 2 * m;
                cy[m] = b < P ? wt_s[GT_PMAX + b] * wz : 0.0;
            }
            const int ox = sw.x - X0, oy = sw.y - Y0, oz = sw.z - Z0;
            const double* rp = region + (ox * L + oy + half) * L + oz + z;
            double acc = 0.0, acc2 = 0.0;
            for (int a = 0; a < P; ++a) {
                const double wx = wt_s[a];
#pragma unroll
                for (int m = 0; m < GT_PMAX / 2; m += 2) {
                    acc = fma(wx * cy[m], rp[2 * m * L], acc);
                    acc2 = fma(wx * cy[m + 1], rp[2 * (m + 1) * L], acc2);
                }
                rp += L2;
            }
            acc += acc2;
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
            if (lane == 0) {
                double* dst = u + 3 * (int64_t)sw.w + c;
                *dst = accumulate ? *dst + h3 * acc : h3 * acc;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// FP64 tensor-core variant (DMMA m8n8k4). With L = B + P - 1 = 19 for every
// P <= 19, the tile contraction is
//   H[(a,b), t] = sum_c G[a][b][c] Wz'[c][t]     (GEMM: 361 x 20 x T, zero-padded)
//   u_t         = sum_(a,b) H[(a,b), t] Wx'[a][t] Wy'[b][t]
// where Wx', Wy', Wz' are each target's taps placed at its offset in the
// region (zero elsewhere). The GEMM runs on the fp64 tensor cores (one DMMA
// = 256 FMAs per warp instruction), the second contraction in the fragment
// epilogue. Shared-memory traffic per tile drops ~15x against the per-target
// tap loop.
constexpr int MM_TG = 32;            // targets per group (4 n-blocks of 8)
// targets whose taps are staged per tile chunk: 64, or 128 for dense tiles
// (>= 64 targets on average; c3: 8.1 -> 6.6 -> 5.6 ms for 32 / 64 / 128,
// c2 / c5 prefer 64 for occupancy)
constexpr int MM_WARPS = 8;
constexpr int MM_THREADS = 32 * MM_WARPS;

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int MM_L, int MM_TMAX>  // region edge: 15 (B = 16 - P), 19 (B = 20 - P, P <= 16) or 23 (B = 24 - P, P <= 20)
__global__ void __launch_bounds__(MM_THREADS)
gather_tile_mma_kernel(DevGrid g, int P, int B, int ntx, int nty, int ntz, int64_t tile0,
                       const double* __restrict__ W, const int4* __restrict__ SW, const int64_t* __restrict__ off,
                       const double* __restrict__ grid, double h3, int accumulate, double* __restrict__ u) {
    constexpr int MM_LS = (MM_L + 4) & ~3;         // padded row: K = MM_LS = 4 x KS
    constexpr int KS = MM_LS / 4;
    constexpr int MM_ROWS = MM_L * MM_L;            // GEMM rows (a, b)
    constexpr int MM_RB = (MM_ROWS + 7) / 8;        // row blocks
    extern __shared__ __align__(16) double sm[];
    const int64_t tile = tile0 + blockIdx.x;
    const int64_t p0 = off[tile], p1 = off[tile + 1];
    if (p0 >= p1) return;
    const int tz = (int)(tile % ntz);
    const int ty = (int)((tile / ntz) % nty);
    const int tx = (int)(tile / ((int64_t)ntz * nty));
    const int X0 = tx * B, Y0 = ty * B, Z0 = tz * B;

    // Target taps of up to MM_TMAX targets (MM_TMAX / 32 groups) are staged once
    // per tile chunk; each component's region is then loaded once and serves
    // every group of the chunk.
    double* region = sm;                                   // [MM_RB*8][MM_LS] (rows >= L*L zero)
    double* wz = region + MM_RB * 8 * MM_LS;               // [MM_TMAX][MM_LS]   Wz'[t][c]
    double* wx = wz + MM_TMAX * MM_LS;                     // [MM_LS][MM_TMAX]   Wx'[a][t] (a = L zero)
    double* wy = wx + MM_LS * MM_TMAX;                     // [MM_LS][MM_TMAX]   Wy'[b][t]
    double* part = wy + MM_LS * MM_TMAX;                   // [MM_WARPS][MM_TMAX]
    int* rowoff = reinterpret_cast<int*>(part + MM_WARPS * MM_TMAX);  // [L*L]
    int* zoff = rowoff + MM_ROWS;                                    // [L]
    int* tid = zoff + MM_L;                                          // [MM_TMAX] target ids
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // zero padding only: column c = L of every row and the rows >= L*L (never loaded)
    for (int e = threadIdx.x; e < MM_ROWS; e += MM_THREADS) region[e * MM_LS + MM_L] = 0.0;
    for (int e = threadIdx.x; e < (MM_RB * 8 - MM_ROWS) * MM_LS; e += MM_THREADS) region[MM_ROWS * MM_LS + e] = 0.0;
    for (int row = threadIdx.x; row < MM_ROWS; row += MM_THREADS) {
        const int i = row / MM_L, j = row - i * MM_L;
        int gx = X0 + i, gy = Y0 + j;
        bool ok = true;
        if (g.d > 0) gx %= g.n[0]; else ok = gx < g.n[0];
        if (g.d > 1) gy %= g.n[1]; else ok = ok && gy < g.n[1];
        rowoff[row] = ok ? (gx * g.n[1] + gy) * g.n[2] : -1;
    }
    if (threadIdx.x < MM_L) {
        int gz = Z0 + threadIdx.x;
        bool ok = true;
        if (g.d > 2) gz %= g.n[2]; else ok = gz < g.n[2];
        zoff[threadIdx.x] = ok ? gz : -1;
    }
    const int64_t cs = (int64_t)g.n[0] * g.n[1] * g.n[2];

    for (int64_t q0 = p0; q0 < p1; q0 += MM_TMAX) {
        const int T = (int)min((int64_t)MM_TMAX, p1 - q0);
        const int ngroups = (T + MM_TG - 1) / MM_TG;
        __syncthreads();
        // per-target taps placed at the target's offset in the region (warp per
        // target, lane = region index k)
        for (int t = warp; t < ngroups * MM_TG; t += MM_WARPS) {
            int4 sw = make_int4(0, 0, 0, -1);
            if (t < T) sw = SW[q0 + t];
            if (lane < MM_LS) {
                const int k = lane;
                double vz = 0.0, vx = 0.0, vy = 0.0;
                if (t < T && k < MM_L) {
                    const double* wt = W + (q0 + t) * 3 * P;
                    const int kx = k - (sw.x - X0), ky = k - (sw.y - Y0), kz = k - (sw.z - Z0);
                    if (kx >= 0 && kx < P) vx = __ldg(wt + kx);
                    if (ky >= 0 && ky < P) vy = __ldg(wt + P + ky);
                    if (kz >= 0 && kz < P) vz = __ldg(wt + 2 * P + kz);
                }
                wz[t * MM_LS + k] = vz;
                wx[k * MM_TMAX + t] = vx;
                wy[k * MM_TMAX + t] = vy;
            }
            if (lane == 0) tid[t] = sw.w;
        }
        for (int c = 0; c < 3; ++c) {
            __syncthreads();
            const double* gc = grid + c * cs;
            {
                const int zo = lane < MM_L ? zoff[lane] : -1;
                const unsigned sbase = (unsigned)__cvta_generic_to_shared(region + lane);
#pragma unroll 4
                for (int row = warp; row < MM_ROWS; row += MM_WARPS) {
                    const int ro = rowoff[row];
                    if (lane < MM_L) {
                        if (ro >= 0 && zo >= 0)
                            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sbase + row * MM_LS * 8),
                                         "l"(gc + ro + zo));
                        else
                            region[row * MM_LS + lane] = 0.0;
                    }
                }
            }
            asm volatile("cp.async.wait_all;\n" ::);
            __syncthreads();
            for (int grp = 0; grp < ngroups; ++grp) {
                const int tg0 = grp * MM_TG;
                const int nblk = (min(T - tg0, MM_TG) + 7) / 8;
                // B fragments (k-steps x n-blocks): lane holds Wz'[k0 + lane%4][n0 + lane/4]
                double bf[KS][4];
#pragma unroll
                for (int ks = 0; ks < KS; ++ks)
#pragma unroll
                    for (int nb = 0; nb < 4; ++nb)
                        bf[ks][nb] = wz[(tg0 + nb * 8 + (lane >> 2)) * MM_LS + ks * 4 + (lane & 3)];
                double acc[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
                const int tc = tg0 + 2 * (lane & 3);  // this lane's two target columns within an n-block
                for (int rb = warp; rb < MM_RB; rb += MM_WARPS) {
                    const int row_a = rb * 8 + (lane >> 2);  // A-fragment row of this lane
                    double af[KS];
#pragma unroll
                    for (int ks = 0; ks < KS; ++ks) af[ks] = region[row_a * MM_LS + ks * 4 + (lane & 3)];
                    const int a = row_a / MM_L, b = row_a - a * MM_L;  // C rows = A rows (groupID)
#pragma unroll
                    for (int nb = 0; nb < 4; ++nb) {
                        if (nb < nblk) {
                            double d0 = 0.0, d1 = 0.0;
#pragma unroll
                            for (int ks = 0; ks < KS; ++ks) dmma_8x8x4(d0, d1, af[ks], bf[ks][nb]);
                            const int t = nb * 8 + tc;
                            const double2 vx = *reinterpret_cast<const double2*>(wx + a * MM_TMAX + t);
                            const double2 vy = *reinterpret_cast<const double2*>(wy + b * MM_TMAX + t);
                            acc[nb][0] = fma(d0, vx.x * vy.x, acc[nb][0]);
                            acc[nb][1] = fma(d1, vx.y * vy.y, acc[nb][1]);
                        }
                    }
                }
                // reduce over the 8 lanes sharing a column pair (lane % 4)
#pragma unroll
                for (int nb = 0; nb < 4; ++nb)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
#pragma unroll
                        for (int s2 = 4; s2 < 32; s2 <<= 1) acc[nb][h] += __shfl_xor_sync(0xffffffffu, acc[nb][h], s2);
                if (lane < 4) {
#pragma unroll
                    for (int nb = 0; nb < 4; ++nb) {
                        part[warp * MM_TMAX + tg0 + nb * 8 + 2 * lane] = acc[nb][0];
                        part[warp * MM_TMAX + tg0 + nb * 8 + 2 * lane + 1] = acc[nb][1];
                    }
                }
            }
            __syncthreads();
            for (int t = threadIdx.x; t < T; t += MM_THREADS) {
                double v = 0.0;
#pragma unroll
                for (int w = 0; w < MM_WARPS; ++w) v += part[w * MM_TMAX + t];
                double* dst = u + 3 * (int64_t)tid[t] + c;
                *dst = accumulate ? *dst + h3 * v : h3 * v;
            }
        }
    }
}

// Register-A form (default for every width): the A fragments (grid values
// G[(a,b)][c]) are read straight from the L2-resident grid per row block and
// every n-block of the chunk's targets consumes them from registers; the B
// fragments (z taps) and the epilogue tables stay in shared memory. No region
// staging, no cp.async phase between barriers. Wide windows (20 < P <= 32,
// c4's Gaussian window at P = 32: B = L - P + 1, L = 31 / 35 / 39) need it, as
// the L^3 region does not fit in shared memory: c4 17.3 -> 9.1 ms against the
// z-sweep; for L = 19 / 23 it beats the shared-region kernel above too
// (c2 3.68 -> 3.24 ms, c3 5.62 -> 4.50, c5 13.8 -> 11.9).
// With a tile's targets ordered by their x stencil offset
// (SEWALD_OPT_GATHER_SORT) each row block visits only the n-blocks whose x
// windows reach it (and loads no A fragments when none does): c2 2.90 ->
// 2.84 ms, c3 4.35 -> 3.71, c4 9.12 -> 7.94, c5 10.62 -> 9.81.
#ifndef SEWALD_WG_TMAX
#define SEWALD_WG_TMAX 64
#endif
#ifndef SEWALD_WG_MINB
#define SEWALD_WG_MINB 3
#endif
#ifndef SEWALD_WG_PAIR
#define SEWALD_WG_PAIR 1
#endif
constexpr int WG_TMAX = SEWALD_WG_TMAX;
// Row stride of the Wx' / Wy' epilogue tables: WG_TMAX + 8 doubles puts the
// two rows (b, b + 1) a quarter warp reads 16 banks apart (with a stride of
// WG_TMAX = 64 doubles every row starts on the same bank: 2-way conflicts on
// every epilogue load)
#ifndef SEWALD_WG_PAD
#define SEWALD_WG_PAD 8
#endif
constexpr int WXS = WG_TMAX + SEWALD_WG_PAD;
// Row stride of the Wz' (B-fragment) table: the 8 rows a fragment load reads
// must spread over the banks (stride = 4 or 12 mod 16 doubles); the GEMM K
// stays LS. LS = 24 (L = 23) had every other row on the same banks.
__host__ __device__ constexpr int wz_stride(int LS) {
    return SEWALD_WG_PAD == 0 ? LS : ((LS % 16 == 4 || LS % 16 == 12) ? LS : LS + 4);
}

// Targets' taps evaluated in the kernel (FUSED): positions + bucket order
// instead of the taps array of a separate kernel.
struct FusedTgt {
    const double* x;        // target positions (AoS)
    const uint32_t* order;  // bucket-sorted -> target index
    DevWindow win;
};

template <int MM_L, bool FUSED = false>
__global__ void __launch_bounds__(MM_THREADS, SEWALD_WG_MINB)
gather_wide_mma_kernel(DevGrid g, int P, int B, int ntx, int nty, int ntz, int64_t tile0,
                       const double* __restrict__ W, const int4* __restrict__ SW, const int64_t* __restrict__ off,
                       const double* __restrict__ grid, double h3, int accumulate, double* __restrict__ u,
                       const FusedTgt* __restrict__ ftg) {
    constexpr int LS = (MM_L + 4) & ~3;  // K = LS = 4 x KS (columns >= L are zero taps)
    constexpr int WZS = wz_stride(LS);   // row stride of the B-fragment table
    constexpr int KS = LS / 4;
    constexpr int ROWS = MM_L * MM_L;
    constexpr int RB = (ROWS + 7) / 8;
    constexpr int NBMAX = WG_TMAX / 8;
    extern __shared__ __align__(16) double sm[];
    const int64_t tile = tile0 + blockIdx.x;
    const int64_t p0 = off[tile], p1 = off[tile + 1];
    if (p0 >= p1) return;
    const int tz = (int)(tile % ntz);
    const int ty = (int)((tile / ntz) % nty);
    const int tx = (int)(tile / ((int64_t)ntz * nty));
    const int X0 = tx * B, Y0 = ty * B, Z0 = tz * B;
    double* wz = sm;                                   // [WG_TMAX][LS]   Wz'[t][c]
    double* wx = wz + WG_TMAX * WZS;                   // [LS][WXS]       Wx'[a][t]
    double* wy = wx + LS * WXS;                        // [LS][WXS]       Wy'[b][t]
    double* part = wy + LS * WXS;                      // [MM_WARPS][WG_TMAX]
    int* rowoff = reinterpret_cast<int*>(part + MM_WARPS * WG_TMAX);  // [ROWS]
    int* zoff = rowoff + ROWS;                                      // [LS]
    int* tid = zoff + LS;                                           // [WG_TMAX]
    int* ox = tid + WG_TMAX;                                        // [WG_TMAX] x offset of each target
    int* nbmin = ox + WG_TMAX;                                      // [LS] first / last n-block reaching row a
    int* nbmax = nbmin + LS;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    for (int row = threadIdx.x; row < ROWS; row += MM_THREADS) {
        const int i = row / MM_L, j = row - i * MM_L;
        int gx = X0 + i, gy = Y0 + j;
        bool ok = true;
        if (g.d > 0) gx %= g.n[0]; else ok = gx < g.n[0];
        if (g.d > 1) gy %= g.n[1]; else ok = ok && gy < g.n[1];
        rowoff[row] = ok ? (gx * g.n[1] + gy) * g.n[2] : -1;
    }
    for (int k = threadIdx.x; k < LS; k += MM_THREADS) {
        int gz = Z0 + k;
        bool ok = k < MM_L;
        if (g.d > 2) gz %= g.n[2]; else ok = ok && gz < g.n[2];
        zoff[k] = ok ? gz : -1;
    }
    const int64_t cs = (int64_t)g.n[0] * g.n[1] * g.n[2];

    for (int64_t q0 = p0; q0 < p1; q0 += WG_TMAX) {
        const int T = (int)min((int64_t)WG_TMAX, p1 - q0);
        const int nblk = (T + 7) / 8;
        __syncthreads();
        if (threadIdx.x < LS) {
            nbmin[threadIdx.x] = 1 << 20;
            nbmax[threadIdx.x] = -1;
        }
        if (FUSED) {
            for (int e = threadIdx.x; e < nblk * 8 * WZS; e += MM_THREADS) wz[e] = 0.0;
            for (int e = threadIdx.x; e < LS * WXS; e += MM_THREADS) {
                wx[e] = 0.0;
                wy[e] = 0.0;
            }
            for (int t = threadIdx.x; t < nblk * 8; t += MM_THREADS) tid[t] = t < T ? (int)ftg->order[q0 + t] : -1;
            __syncthreads();
            for (int e = threadIdx.x; e < 3 * T; e += MM_THREADS) {
                const int ax = e / T, t = e - ax * T;
                const int64_t i = ftg->order[q0 + t];
                int j0;
                double rel;
                stencil_origin(g, P, ax, ftg->x[3 * i + ax], j0, rel);
                const int sw = ax < g.d ? wrap_index(j0, g.n[ax]) : j0;
                const int o = sw - (ax == 0 ? X0 : (ax == 1 ? Y0 : Z0));
                if (ax == 0) ox[t] = o;
                if (ax == 2) window_taps(ftg->win, j0, rel, g.h, wz + t * WZS + o);
                else window_taps(ftg->win, j0, rel, g.h, (ax == 0 ? wx : wy) + o * WXS + t, WXS);
            }
        } else
        for (int t = warp; t < nblk * 8; t += MM_WARPS) {
            int4 sw = make_int4(0, 0, 0, -1);
            if (t < T) sw = SW[q0 + t];
            for (int k = lane; k < LS; k += 32) {
                double vz = 0.0, vx = 0.0, vy = 0.0;
                if (t < T && k < MM_L) {
                    const double* wt = W + (q0 + t) * 3 * P;
                    const int kx = k - (sw.x - X0), ky = k - (sw.y - Y0), kz = k - (sw.z - Z0);
                    if (kx >= 0 && kx < P) vx = __ldg(wt + kx);
                    if (ky >= 0 && ky < P) vy = __ldg(wt + P + ky);
                    if (kz >= 0 && kz < P) vz = __ldg(wt + 2 * P + kz);
                }
                wz[t * WZS + k] = vz;
                wx[k * WXS + t] = vx;
                wy[k * WXS + t] = vy;
            }
            if (lane == 0) {
                tid[t] = sw.w;
                if (t < T) ox[t] = sw.x - X0;
            }
        }
        __syncthreads();
        // n-blocks (8 targets) whose x windows reach region row a: a contiguous
        // range when the targets are ordered by x offset (SEWALD_OPT_GATHER_SORT),
        // a conservative cover otherwise
        for (int nb = threadIdx.x; nb < nblk; nb += MM_THREADS) {
            int lo = 1 << 20, hi = -(1 << 20);
            for (int t = 8 * nb; t < min(8 * nb + 8, T); ++t) {
                lo = min(lo, ox[t]);
                hi = max(hi, ox[t] + P - 1);
            }
            for (int a = max(lo, 0); a <= min(hi, MM_L - 1); ++a) {
                atomicMin(&nbmin[a], nb);
                atomicMax(&nbmax[a], nb);
            }
        }
        __syncthreads();
        for (int c = 0; c < 3; ++c) {
            const double* gc = grid + c * cs;
            double acc[NBMAX][2];
#pragma unroll
            for (int nb = 0; nb < NBMAX; ++nb) acc[nb][0] = acc[nb][1] = 0.0;
            const int tcol = 2 * (lane & 3);
            // two row blocks per pass for L = 23: each B fragment (z taps) read from
            // shared memory feeds two DMMAs (the kernel is bound by the L1 / shared
            // path): xi = 63 3.71 -> 3.55 ms; for L = 19 (46 row blocks over 8
            // warps) it loses (c2 2.84 -> 3.10 ms)
            if (SEWALD_WG_PAIR && MM_L == 23) {
            for (int rb = warp; rb < RB; rb += 2 * MM_WARPS) {
                const int rbq[2] = {rb, rb + MM_WARPS};
                int lo[2], hi[2], aa[2], bb[2];
                double af[2][KS];
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    lo[q] = 1 << 20;
                    hi[q] = -1;
                    const int r = rbq[q];
                    if (r < RB) {
                        const int a_lo = (r * 8) / MM_L, a_hi = min(r * 8 + 7, ROWS - 1) / MM_L;
                        lo[q] = min(nbmin[a_lo], nbmin[a_hi]);
                        hi[q] = max(nbmax[a_lo], nbmax[a_hi]);
                    }
                    const int row_a = r * 8 + (lane >> 2);
                    const int ro = (lo[q] <= hi[q] && row_a < ROWS) ? rowoff[row_a] : -1;
#pragma unroll
                    for (int ks = 0; ks < KS; ++ks) {
                        const int zo = zoff[ks * 4 + (lane & 3)];
                        af[q][ks] = (ro >= 0 && zo >= 0) ? __ldg(gc + ro + zo) : 0.0;
                    }
                    aa[q] = row_a / MM_L;
                    bb[q] = row_a - aa[q] * MM_L;
                }
                if (lo[0] > hi[0] && lo[1] > hi[1]) continue;
#pragma unroll
                for (int nb = 0; nb < NBMAX; ++nb) {
                    const bool in0 = nb >= lo[0] && nb <= hi[0], in1 = nb >= lo[1] && nb <= hi[1];
                    if (in0 || in1) {
                        double d[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
                        for (int ks = 0; ks < KS; ++ks) {
                            const double bz = wz[(nb * 8 + (lane >> 2)) * WZS + ks * 4 + (lane & 3)];
                            if (in0) dmma_8x8x4(d[0][0], d[0][1], af[0][ks], bz);
                            if (in1) dmma_8x8x4(d[1][0], d[1][1], af[1][ks], bz);
                        }
                        const int t = nb * 8 + tcol;
#pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            if ((q ? in1 : in0) && aa[q] < LS) {
                                const double2 vx = *reinterpret_cast<const double2*>(wx + aa[q] * WXS + t);
                                const double2 vy = *reinterpret_cast<const double2*>(wy + bb[q] * WXS + t);
                                acc[nb][0] = fma(d[q][0], vx.x * vy.x, acc[nb][0]);
                                acc[nb][1] = fma(d[q][1], vx.y * vy.y, acc[nb][1]);
                            }
                        }
                    }
                }
            }
            } else {
            for (int rb = warp; rb < RB; rb += MM_WARPS) {
                const int a_lo = (rb * 8) / MM_L, a_hi = min(rb * 8 + 7, ROWS - 1) / MM_L;
                const int nb_lo = min(nbmin[a_lo], nbmin[a_hi]), nb_hi = max(nbmax[a_lo], nbmax[a_hi]);
                if (nb_lo > nb_hi) continue;  // no target of the chunk reaches these rows
                const int row_a = rb * 8 + (lane >> 2);
                const int ro = row_a < ROWS ? rowoff[row_a] : -1;
                double af[KS];
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) {
                    const int zo = zoff[ks * 4 + (lane & 3)];
                    af[ks] = (ro >= 0 && zo >= 0) ? __ldg(gc + ro + zo) : 0.0;
                }
                const int a = row_a / MM_L, b = row_a - a * MM_L;  // rows >= L*L: a >= L (zero taps)
#pragma unroll
                for (int nb = 0; nb < NBMAX; ++nb) {
                    if (nb >= nb_lo && nb <= nb_hi) {
                        double d0 = 0.0, d1 = 0.0;
#pragma unroll
                        for (int ks = 0; ks < KS; ++ks)
                            dmma_8x8x4(d0, d1, af[ks], wz[(nb * 8 + (lane >> 2)) * WZS + ks * 4 + (lane & 3)]);
                        if (a < LS) {
                            const int t = nb * 8 + tcol;
                            const double2 vx = *reinterpret_cast<const double2*>(wx + a * WXS + t);
                            const double2 vy = *reinterpret_cast<const double2*>(wy + b * WXS + t);
                            acc[nb][0] = fma(d0, vx.x * vy.x, acc[nb][0]);
                            acc[nb][1] = fma(d1, vx.y * vy.y, acc[nb][1]);
                        }
                    }
                }
            }
            }
#pragma unroll
            for (int nb = 0; nb < NBMAX; ++nb)
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int s2 = 4; s2 < 32; s2 <<= 1) acc[nb][h] += __shfl_xor_sync(0xffffffffu, acc[nb][h], s2);
            if (lane < 4) {
#pragma unroll
                for (int nb = 0; nb < NBMAX; ++nb) {
                    part[warp * WG_TMAX + nb * 8 + 2 * lane] = acc[nb][0];
                    part[warp * WG_TMAX + nb * 8 + 2 * lane + 1] = acc[nb][1];
                }
            }
            __syncthreads();
            for (int t = threadIdx.x; t < T; t += MM_THREADS) {
                double v = 0.0;
#pragma unroll
                for (int w = 0; w < MM_WARPS; ++w) v += part[w * WG_TMAX + t];
                double* dst = u + 3 * (int64_t)tid[t] + c;
                *dst = accumulate ? *dst + h3 * v : h3 * v;
            }
            __syncthreads();
        }
    }
}

size_t wide_smem_bytes(int L);

template <int L>
void launch_wide_fused(const DevGrid& g, int P, const TileShape& s, int64_t t0, int64_t t1, const int64_t* off,
                       const double* grid, double h3, int accumulate, double* u, const FusedTgt* arg,
                       cudaStream_t st) {
    auto kern = gather_wide_mma_kernel<L, true>;
    const size_t smw = wide_smem_bytes(L);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smw);
    for (int64_t a = t0; a < t1; a += (int64_t)1 << 30) {
        const int64_t n = std::min<int64_t>(t1 - a, (int64_t)1 << 30);
        kern<<<(unsigned)n, MM_THREADS, smw, st>>>(g, P, s.B, s.nt[0], s.nt[1], s.nt[2], a, nullptr, nullptr, off,
                                                   grid, h3, accumulate, u, arg);
    }
}

size_t wide_smem_bytes(int L) {
    const int LS = (L + 4) & ~3;
    return sizeof(double) * ((size_t)WG_TMAX * wz_stride(LS) + 2 * (size_t)WXS * LS + MM_WARPS * WG_TMAX) +
           sizeof(int) * ((size_t)L * L + 3 * LS + 2 * WG_TMAX);
}

size_t mma_smem_bytes(int L, int MM_TMAX) {
    const int LS = (L + 4) & ~3, rows = L * L, rb = (rows + 7) / 8;
    return sizeof(double) * ((size_t)rb * 8 * LS + MM_TMAX * LS + 2 * LS * MM_TMAX + MM_WARPS * MM_TMAX) +
           sizeof(int) * (rows + L + MM_TMAX);
}

}  // namespace

TileShape tile_shape(const DevGrid& g, int P, int64_t Nt) {
    TileShape s{};
    // P <= 16: B = 20 - P (L = 19; CUDA-core or tensor-core kernel);
    // 16 < P <= 20: B = 24 - P (L = 23; tensor-core kernel only).
    // Dense targets and P <= 15: L = 15 (B = 16 - P) when a tile still holds
    // >= 12 targets on average: the GEMM does (15/19)^2 * 16/20 = 0.5x the work
    // per target and a tile's region is loaded once per component.
    s.ok = P <= 20;
    s.B = P <= GT_PMAX ? std::max(1, 20 - P) : std::max(1, 24 - P);
    if (P > 20 && P <= 32) {  // wide-window tensor-core tiles (gather_wide_mma_kernel)
        s.L = P <= 24 ? 31 : (P <= 28 ? 35 : 39);
        s.B = s.L - P + 1;
        for (int ax = 0; ax < 3; ++ax) s.nt[ax] = (g.n[ax] + s.B - 1) / s.B;
        s.ntiles = (int64_t)s.nt[0] * s.nt[1] * s.nt[2];
        s.tpt = s.ntiles > 0 ? (double)Nt / (double)s.ntiles : 0.0;
        s.smem = wide_smem_bytes(s.L);
        s.ok = option(SEWALD_OPT_GATHER_WIDE) != 0 && s.ntiles < (int64_t(1) << 31) &&
               (int64_t)g.n[0] * g.n[1] * g.n[2] < (int64_t(1) << 31);
        return s;
    }
    const int forced_l = option(SEWALD_OPT_GATHER_L);
    if (P <= 15) {
        const double cells = (double)g.n[0] * g.n[1] * g.n[2];
        const int b15 = 16 - P;
        const double tpt = cells > 0 ? (double)Nt / cells * b15 * b15 * b15 : 0.0;
        if (forced_l == 15 || (forced_l == 0 && tpt >= 12.0)) s.B = b15;
    }
    // Sparse targets (register-A kernel): L = 23 tiles (B = 24 - P) when an L = 19
    // tile would hold fewer than 24 targets on average - every chunk loads its
    // whole region, so small chunks are load-bound. c2 workload at xi = 60
    // (M = 204, 7.5 targets per L = 19 tile): 6.73 -> 3.63 ms; xi = 70: 10.8 ->
    // 4.3 ms; xi = 45 (16.9 per tile) 3.76 -> 3.38 ms; at xi = 37 (30 per tile)
    // L = 19 stays ahead (2.84 vs 3.38 ms).
    // L = 31 (B = 32 - P, forced only) measured slower in all three.
    if (P <= 16 && s.B == 20 - P && forced_l == 0 && option(SEWALD_OPT_GATHER_WIDE) == 2) {
        const double b = s.B;
        const double tpt19 = (double)Nt * b * b * b / ((double)g.n[0] * g.n[1] * g.n[2]);
        if (tpt19 < 24.0) s.B = 24 - P;
    }
    if ((forced_l == 23 || forced_l == 31) && P <= 20 && option(SEWALD_OPT_GATHER_WIDE) == 2) s.B = forced_l + 1 - P;
    s.L = s.B + P - 1;
    for (int ax = 0; ax < 3; ++ax) s.nt[ax] = (g.n[ax] + s.B - 1) / s.B;
    s.ntiles = (int64_t)s.nt[0] * s.nt[1] * s.nt[2];
    s.tpt = s.ntiles > 0 ? (double)Nt / (double)s.ntiles : 0.0;
    if (s.ntiles >= (int64_t(1) << 31)) s.ok = false;
    if (s.L == 31) {  // register-A tiles only (the L^3 region does not fit in shared memory)
        s.smem = wide_smem_bytes(s.L);
        if ((int64_t)g.n[0] * g.n[1] * g.n[2] >= (int64_t(1) << 31)) s.ok = false;
        return s;
    }
    const int pad = 2 * GT_PMAX * s.L + 2 * GT_PMAX;
    s.smem = sizeof(double) * ((size_t)s.L * s.L * s.L + pad + GT_WARPS * 3 * GT_PMAX) +
             sizeof(int) * ((size_t)s.L * s.L + s.L);
    if ((int64_t)g.n[0] * g.n[1] * g.n[2] >= (int64_t(1) << 31)) s.ok = false;  // int offsets
    if (s.smem > 200 * 1024 || s.L > 32) s.ok = false;
    return s;
}

void launch_tile_bucket(const DevGrid& g, int P, const TileShape& s, const double* x, int64_t N, uint32_t* keys,
                        uint32_t* vals, int* bad, cudaStream_t st, int sub) {
    if (N == 0) return;
    tile_bucket_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(g, P, s.B, s.nt[0], s.nt[1], s.nt[2], x, N,
                                                                     keys, vals, bad, sub);
}

bool gather_tile_regA(const TileShape& s) {
    return s.ok && (s.L >= 31 || (option(SEWALD_OPT_GATHER_WIDE) == 2 && (s.L == 15 || s.L == 19 || s.L == 23)));
}

bool gather_tile_fused_ok(const TileShape& s) {
    return s.ok && option(SEWALD_OPT_GATHER_FUSED) != 0 &&
           (s.L >= 31 || (option(SEWALD_OPT_GATHER_WIDE) == 2 && (s.L == 15 || s.L == 19 || s.L == 23)));
}

size_t fused_tgt_bytes() { return sizeof(FusedTgt); }

void launch_gather_tile_fused(const DevGrid& g, const DevWindow& w, int P, const TileShape& s, const double* xt,
                              const uint32_t* order, const int64_t* off, int part, int nparts, const double* grid,
                              double h3, int accumulate, double* u, void* arg_dev, cudaStream_t st) {
    const int64_t t0 = s.ntiles * part / nparts, t1 = s.ntiles * (part + 1) / nparts;
    if (t1 <= t0) return;
    FusedTgt h{xt, order, w};
    cudaMemcpyAsync(arg_dev, &h, sizeof(FusedTgt), cudaMemcpyHostToDevice, st);
    const FusedTgt* a = static_cast<const FusedTgt*>(arg_dev);
    switch (s.L) {
        case 15: launch_wide_fused<15>(g, P, s, t0, t1, off, grid, h3, accumulate, u, a, st); break;
        case 19: launch_wide_fused<19>(g, P, s, t0, t1, off, grid, h3, accumulate, u, a, st); break;
        case 23: launch_wide_fused<23>(g, P, s, t0, t1, off, grid, h3, accumulate, u, a, st); break;
        case 31: launch_wide_fused<31>(g, P, s, t0, t1, off, grid, h3, accumulate, u, a, st); break;
        case 35: launch_wide_fused<35>(g, P, s, t0, t1, off, grid, h3, accumulate, u, a, st); break;
        default: launch_wide_fused<39>(g, P, s, t0, t1, off, grid, h3, accumulate, u, a, st); break;
    }
}

void launch_gather_tile(const DevGrid& g, int P, const TileShape& s, const double* W, const int4* SW,
                        const int64_t* off, int part, int nparts, const double* grid, double h3, int accumulate,
                        double* u, cudaStream_t st) {
    const int64_t t0 = s.ntiles * part / nparts, t1 = s.ntiles * (part + 1) / nparts;
    if (t1 <= t0) return;
    const bool use_mma = option(SEWALD_OPT_GATHER_MMA) != 0;
    const bool wide_all = option(SEWALD_OPT_GATHER_WIDE) == 2 && (s.L == 15 || s.L == 19 || s.L == 23);
    if (s.L >= 31 || wide_all) {
        auto kern = s.L == 31 ? gather_wide_mma_kernel<31>
                              : (s.L == 35 ? gather_wide_mma_kernel<35>
                                           : (s.L == 39 ? gather_wide_mma_kernel<39>
                                                        : (s.L == 15 ? gather_wide_mma_kernel<15>
                                                                     : (s.L == 19 ? gather_wide_mma_kernel<19>
                                                                                  : gather_wide_mma_kernel<23>))));
        const size_t smw = wide_smem_bytes(s.L);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smw);
        const FusedTgt* ftg_null = nullptr;
        for (int64_t a = t0; a < t1; a += (int64_t)1 << 30) {
            const int64_t n = std::min<int64_t>(t1 - a, (int64_t)1 << 30);
            kern<<<(unsigned)n, MM_THREADS, smw, st>>>(g, P, s.B, s.nt[0], s.nt[1], s.nt[2], a, W, SW, off, grid,
                                                       h3, accumulate, u, ftg_null);
        }
        return;
    }
    if ((use_mma || P > GT_PMAX || s.L == 15) && (s.L == 15 || s.L == 19 || s.L == 23)) {
        const bool wide = s.tpt >= 64.0;
        const size_t sm = mma_smem_bytes(s.L, wide ? 128 : 64);
        auto kern = wide ? (s.L == 15 ? gather_tile_mma_kernel<15, 128>
                                      : (s.L == 19 ? gather_tile_mma_kernel<19, 128> : gather_tile_mma_kernel<23, 128>))
                         : (s.L == 15 ? gather_tile_mma_kernel<15, 64>
                                      : (s.L == 19 ? gather_tile_mma_kernel<19, 64> : gather_tile_mma_kernel<23, 64>));
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        for (int64_t a = t0; a < t1; a += (int64_t)1 << 30) {
            const int64_t n = std::min<int64_t>(t1 - a, (int64_t)1 << 30);
            kern<<<(unsigned)n, MM_THREADS, sm, st>>>(g, P, s.B, s.nt[0], s.nt[1], s.nt[2], a, W, SW, off, grid, h3,
                                                      accumulate, u);
        }
        return;
    }
    cudaFuncSetAttribute(gather_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s.smem);
    // grid.x limit is 2^31 - 1: launch in chunks
    for (int64_t a = t0; a < t1; a += (int64_t)1 << 30) {
        const int64_t n = std::min<int64_t>(t1 - a, (int64_t)1 << 30);
        gather_tile_kernel<<<(unsigned)n, GT_THREADS, s.smem, st>>>(g, P, s.B, s.L, s.nt[0], s.nt[1], s.nt[2], a, W,
                                                                     SW, off, grid, h3, accumulate, u);
    }
}

}  // namespace sewald_b200
