// Short-range (real-space) Ewald sum over a cell list, fp64.
//
// Reference: accumulate_rows  /root/reference/proj/src/realspace.cpp:30-93
//            build_cell_list  /root/reference/proj/src/realspace.cpp:97-164
//            realspace_kernel /root/reference/proj/src/kernels.cpp:71-116
//            apply            /root/reference/proj/src/kernels.cpp:189-202
//
// B200 layout: sources folded into the cell and sorted by a fine cell grid
// (cell width ~ rc/4, x fastest) and packed as 64/96-byte records. One CTA
// takes 128 consecutive targets in the same cell order; their bounding box
// selects the cell rows whose distance is below rc, and each row's x range is
// trimmed to the ball. Every row piece is one contiguous source range, staged
// through shared memory and read as warp broadcasts. Per chunk, each lane
// first tests all staged sources and records accepted ones in a 128-bit
// register mask, then evaluates the erfc/exp kernel only on accepted pairs,
// so the expensive fp64 path runs with converged lanes.
//
// The accepted set is the reference's: r = (x_t - x_s) - shift computed in
// the same order, |r|^2 formed without FMA contraction and compared with
// rc*rc, and the self pair skipped only on the primary image.
#include "device_common.cuh"

#include <algorithm>
#include "sg_kernels.h"
#include "../../include/sewald_gpu.h"
#include "screened_math.cuh"

namespace sewald_b200 {

namespace {

constexpr int RS_THREADS = 128;
constexpr int RS_WARPS = 4;
#ifndef SEWALD_RS_CHUNK
#define SEWALD_RS_CHUNK 64
#endif
constexpr int WCHUNK = SEWALD_RS_CHUNK;  // 64 or 128 (mask path)
// candidate sources of a chunk as a per-lane 64-bit mask (1) or a per-lane
// byte queue in shared memory (0): c4 47.9 -> 43.2 ms (no per-candidate
// stores in the fp32 pass, no queue reads in the fp64 pass; same pair order).
// 128-source chunks (two masks) measured slower: 56.9 ms.
// rows / chunks no target of the warp can reach are skipped before staging
// (c4 43.3 -> 40.6 ms)
#ifndef SEWALD_RS_BLOCKTEST
#define SEWALD_RS_BLOCKTEST 1
#endif
#ifndef SEWALD_RS_MASK
#define SEWALD_RS_MASK 1
#endif

__device__ __forceinline__ int floor_div(int a, int b) {
    int q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
    return q;
}

__device__ __forceinline__ int cell_of(const CellGrid& cg, int ax, double v) {
    int c = (int)floor((v - cg.origin[ax]) / cg.w[ax]);
    return c < 0 ? 0 : (c > cg.n[ax] - 1 ? cg.n[ax] - 1 : c);
}

__global__ void fold_key_kernel(CellGrid cg, const double* __restrict__ x, int64_t N,
                                double* __restrict__ folded, uint32_t* __restrict__ keys,
                                uint32_t* __restrict__ vals) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    double y[3];
    for (int ax = 0; ax < 3; ++ax) {
        double v = x[3 * i + ax];
        if (ax < cg.d) {  // wrap_position (domain.cpp:64-71): fmod is exact
            v = fmod(v, cg.L[ax]);
            if (v < 0.0) v += cg.L[ax];
        }
        y[ax] = v;
        folded[3 * i + ax] = v;
    }
    const int cx = cell_of(cg, 0, y[0]), cy = cell_of(cg, 1, y[1]), cz = cell_of(cg, 2, y[2]);
    // low `sub` bits: x position inside the cell, so that consecutive particles
    // of a cell row (i-clusters, j-blocks) are compact along x as well
    const int ns = 1 << cg.sub;
    int sx = (int)floor(((y[0] - cg.origin[0]) / cg.w[0] - cx) * ns);
    sx = sx < 0 ? 0 : (sx > ns - 1 ? ns - 1 : sx);
    keys[i] = ((uint32_t)((cz * cg.n[1] + cy) * cg.n[0] + cx) << cg.sub) | (uint32_t)sx;
    vals[i] = (uint32_t)i;
}

__global__ void pack_kernel(const double* __restrict__ folded, const double* __restrict__ f,
                            const double* __restrict__ nu, int stresslet,
                            const uint32_t* __restrict__ order, int64_t N,
                            double* __restrict__ packed, float4* __restrict__ packedf) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= N) return;
    const int64_t i = order[k];
    const int S = stresslet ? 12 : 8;
    double* o = packed + k * S;
    const double x0 = folded[3 * i], x1 = folded[3 * i + 1], x2 = folded[3 * i + 2];
    o[0] = x0;
    o[1] = x1;
    o[2] = x2;
    o[3] = __longlong_as_double((long long)i);
    o[4] = f[3 * i];
    o[5] = f[3 * i + 1];
    o[6] = f[3 * i + 2];
    if (stresslet) {
        o[7] = nu[3 * i];
        o[8] = nu[3 * i + 1];
        o[9] = nu[3 * i + 2];
        o[10] = fma(f[3 * i + 2], nu[3 * i + 2], fma(f[3 * i + 1], nu[3 * i + 1], f[3 * i] * nu[3 * i]));  // q.nu
        o[11] = 0.0;
    } else {
        o[7] = 0.0;
    }
    packedf[k] = make_float4((float)x0, (float)x1, (float)x2, 0.0f);
}

// Pair contribution given the shared screened factors (kernels.cpp:71-116
// contracted with apply, kernels.cpp:189-202). s points at the strength
// block of the packed record: f (3) or q (3) followed by nu (3).
template <int KIND>
__device__ __forceinline__ void pair_accumulate(const Screened& sc, double xi2, double n2, double r0,
                                                double r1, double r2, const double* s, double& u0,
                                                double& u1, double& u2) {
    if (KIND == SEWALD_STOKESLET) {
        // m_jl = (d_jl + r_j r_l / r^2)(erfc/r + g) - 2 g d_jl
        const double a = sc.Ey * (sc.R - sc.cx);
        const double b = sc.Ey * (sc.iy * sc.iy) * (sc.R + sc.cx);
        const double rf = r0 * s[0] + r1 * s[1] + r2 * s[2];
        const double brf = b * rf;
        u0 = fma(a, s[0], fma(brf, r0, u0));
        u1 = fma(a, s[1], fma(brf, r1, u1));
        u2 = fma(a, s[2], fma(brf, r2, u2));
    } else if (KIND == SEWALD_ROTLET) {
        // m_jl = eps_jlm r_m (erfc/r + g) / r^2  ->  c (f x r)
        const double c = sc.Ey * (sc.iy * sc.iy) * (sc.R + sc.cx);
        u0 = fma(c, s[1] * r2 - s[2] * r1, u0);
        u1 = fma(c, s[2] * r0 - s[0] * r2, u1);
        u2 = fma(c, s[0] * r1 - s[1] * r0, u2);
    } else {
        // t_jlm = c1 r_j r_l r_m + c2 (d_jl r_m + d_mj r_l + d_lm r_j)
        const double iy2 = sc.iy * sc.iy;
        const double x2 = xi2 * n2;
        const double c1 = -2.0 * sc.Ey * (iy2 * iy2) * (3.0 * sc.R + (3.0 + 2.0 * x2) * sc.cx);
        const double c2 = 2.0 * xi2 * sc.Ey * sc.cx;
        const double* q = s;
        const double* v = s + 3;
        const double rq = r0 * q[0] + r1 * q[1] + r2 * q[2];
        const double rv = r0 * v[0] + r1 * v[1] + r2 * v[2];
        const double qv = q[0] * v[0] + q[1] * v[1] + q[2] * v[2];
        const double t = c1 * rq * rv + c2 * qv;
        u0 += t * r0 + c2 * (q[0] * rv + v[0] * rq);
        u1 += t * r1 + c2 * (q[1] * rv + v[1] * rq);
        u2 += t * r2 + c2 * (q[2] * rv + v[2] * rq);
    }
}

// One WARP = one independent work unit: 32 consecutive targets in cell
// order (spatially compact), their bounding box, the cell rows within rc of
// it, and a private shared-memory staging area. No block-wide barriers.
#ifndef SEWALD_RS_F2
#define SEWALD_RS_F2 1
#endif

template <int KIND, int S, bool SHORT>
__global__ void __launch_bounds__(RS_THREADS, 4)
realspace_kernel(CellGrid cg, RealspaceArgs a, const double* __restrict__ packed,
                 const float4* __restrict__ packedf, const int64_t* __restrict__ cell_off,
                 const double* __restrict__ tfolded, const uint32_t* __restrict__ torder, int64_t Nt,
                 double* __restrict__ u, int accumulate, unsigned long long* __restrict__ pair_count,
                 int* __restrict__ err, int split, double* __restrict__ scratch) {
    constexpr int CH = S > 8 ? 64 : WCHUNK;  // stresslet records: 64 (static shared-memory limit)
    __shared__ __align__(16) double src_all[RS_WARPS][CH * S];
    __shared__ float4 srcf_all[RS_WARPS][CH];
#if SEWALD_RS_F2
    // negated fp32 positions in pairs for the packed fp32x2 candidate pass:
    // [-x_2p, -x_2p+1, -y_2p, -y_2p+1] and [-z_2p, -z_2p+1]
    __shared__ float4 srcq_all[RS_WARPS][CH / 2];
    __shared__ float2 srcz_all[RS_WARPS][CH / 2];
#endif
#if !SEWALD_RS_MASK
    __shared__ uint8_t queue_all[RS_WARPS][CH][32];
#endif
    __shared__ double exp_tab[32];
    if (threadIdx.x < 32) exp_tab[threadIdx.x] = exp_tab_entry<SHORT>(threadIdx.x);
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* src = src_all[warp];
    float4* srcf = srcf_all[warp];
#if !SEWALD_RS_MASK
    uint8_t(*queue)[32] = queue_all[warp];
#endif

    // work item = (32-target group, row part): small target sets split each
    // group's neighbour rows over `split` warps; the parts' sums are added in
    // a fixed order afterwards (realspace_sum_parts), so results do not
    // depend on scheduling
    const int64_t witem = (int64_t)blockIdx.x * RS_WARPS + warp;
    const int64_t group = witem / split;
    const int part = (int)(witem % split);
    const int64_t t = group * 32 + lane;
    if (group * 32 >= Nt) return;  // whole warp idle
    const bool valid = t < Nt;
    double xt0 = 0, xt1 = 0, xt2 = 0;
    int64_t tori = -1;
    if (valid) {
        tori = torder[t];
        xt0 = tfolded[3 * tori];
        xt1 = tfolded[3 * tori + 1];
        xt2 = tfolded[3 * tori + 2];
    }

    // Bounding box of this warp's targets.
    double lo[3] = {valid ? xt0 : 1e300, valid ? xt1 : 1e300, valid ? xt2 : 1e300};
    double hi[3] = {valid ? xt0 : -1e300, valid ? xt1 : -1e300, valid ? xt2 : -1e300};
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) {
            lo[ax] = fmin(lo[ax], __shfl_xor_sync(0xffffffffu, lo[ax], s));
            hi[ax] = fmax(hi[ax], __shfl_xor_sync(0xffffffffu, hi[ax], s));
        }
    }

    const double rc2 = a.rc2;  // kernel-parameter operands
    const double xi2 = a.xi2;
    const double rcm = a.rc * (1.0 + 1e-10) + 1e-12 * fmax(fmax(cg.L[0], cg.L[1]), cg.L[2]);
    const double rcm2 = rcm * rcm;

    int clo[3], chi[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        clo[ax] = (int)floor((lo[ax] - rcm - cg.origin[ax]) / cg.w[ax]);
        chi[ax] = (int)floor((hi[ax] + rcm - cg.origin[ax]) / cg.w[ax]);
        if (ax >= cg.d) {
            clo[ax] = max(clo[ax], 0);
            chi[ax] = min(chi[ax], cg.n[ax] - 1);
        }
    }

    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    // per-target pair count in 32 bits inside the pair loop (one instruction
    // instead of a 64-bit add pair; a target's pairs <= 27 N fit for
    // N < 1.5e8), widened to 64 bits for the warp sum below
    unsigned npairs32 = 0;
    int row_id = -1;

    for (int cz = clo[2]; cz <= chi[2]; ++cz) {
        const int sz = 2 < cg.d ? floor_div(cz, cg.n[2]) : 0;
        const int jz = cz - sz * cg.n[2];
        const double zlo = cg.origin[2] + cz * cg.w[2], zhi = zlo + cg.w[2];
        const double dz = fmax(0.0, fmax(zlo - hi[2], lo[2] - zhi));
        const double shz = (double)sz * cg.L[2];
        for (int cy = clo[1]; cy <= chi[1]; ++cy) {
            if (split > 1 && (++row_id) % split != part) continue;
            const int sy = 1 < cg.d ? floor_div(cy, cg.n[1]) : 0;
            const int jy = cy - sy * cg.n[1];
            const double ylo = cg.origin[1] + cy * cg.w[1], yhi = ylo + cg.w[1];
            const double dy = fmax(0.0, fmax(ylo - hi[1], lo[1] - yhi));
            const double lat2 = dy * dy + dz * dz;
            if (lat2 >= rcm2) continue;
            const double ext = sqrt(rcm2 - lat2);
            int cxl = (int)floor((lo[0] - ext - cg.origin[0]) / cg.w[0]);
            int cxh = (int)floor((hi[0] + ext - cg.origin[0]) / cg.w[0]);
            cxl = max(cxl, clo[0]);
            cxh = min(cxh, chi[0]);
            if (cxl > cxh) continue;
            const double shy = (double)sy * cg.L[1];
            const int64_t rowbase = ((int64_t)jz * cg.n[1] + jy) * cg.n[0];
            const int sxa = 0 < cg.d ? floor_div(cxl, cg.n[0]) : 0;
            const int sxb = 0 < cg.d ? floor_div(cxh, cg.n[0]) : 0;
            for (int sx = sxa; sx <= sxb; ++sx) {
                const int jlo = max(cxl - sx * cg.n[0], 0);
                const int jhi = min(cxh - sx * cg.n[0], cg.n[0] - 1);
                const int64_t b0 = cell_off[rowbase + jlo], b1 = cell_off[rowbase + jhi + 1];
                if (b0 >= b1) continue;
                const double shx = (double)sx * cg.L[0];
                const bool primary = (sx == 0) && (sy == 0) && (sz == 0);
                // fp32 image of this target relative to the row piece's shift
                const float tf0 = (float)(xt0 - shx), tf1 = (float)(xt1 - shy), tf2 = (float)(xt2 - shz);
#if SEWALD_RS_BLOCKTEST
                // per-target distance to the row's (y, z) slab and to each chunk's
                // x range: rows and chunks no target of the warp can reach are
                // skipped before staging (the bounding box reaches more)
                const double ylo_f = cg.origin[1] + jy * cg.w[1], zlo_f = cg.origin[2] + jz * cg.w[2];
                const double ys = xt1 - shy, zs = xt2 - shz, xsx = xt0 - shx;
                const double ey = fmax(0.0, fmax(ylo_f - ys, ys - (ylo_f + cg.w[1])));
                const double ez = fmax(0.0, fmax(zlo_f - zs, zs - (zlo_f + cg.w[2])));
                const double lat_l = ey * ey + ez * ez;
                const bool row_near = valid && lat_l < rcm2;
                if (!__any_sync(0xffffffffu, row_near)) continue;
                const double subw = cg.w[0] / (double)(1 << cg.sub);  // x order holds up to a sub-cell
#endif
                for (int64_t base = b0; base < b1; base += CH) {
                    const int cnt = (int)min((int64_t)CH, b1 - base);
#if SEWALD_RS_BLOCKTEST
                    {
                        const double xb0 = __ldg(packed + base * S) - subw;
                        const double xb1 = __ldg(packed + (base + cnt - 1) * S) + subw;
                        const double ex = fmax(0.0, fmax(xb0 - xsx, xsx - xb1));
                        if (!__any_sync(0xffffffffu, row_near && fma(ex, ex, lat_l) < rcm2)) continue;
                    }
#endif
                    __syncwarp();
                    {
                        const double2* g2 = reinterpret_cast<const double2*>(packed + base * S);
                        double2* s2 = reinterpret_cast<double2*>(src);
                        for (int e = lane; e < cnt * (S / 2); e += 32) s2[e] = __ldg(g2 + e);
#if SEWALD_RS_MASK
                        // slots past the chunk: far away in fp32 (never candidates)
                        for (int e = lane; e < CH; e += 32) {
                            const float4 v = e < cnt ? __ldg(packedf + base + e) : make_float4(1e30f, 1e30f, 1e30f, 0.0f);
                            srcf[e] = v;
#if SEWALD_RS_F2
                            float* sq = reinterpret_cast<float*>(srcq_all[warp]) + (e >> 1) * 4 + (e & 1);
                            sq[0] = -v.x;
                            sq[2] = -v.y;
                            reinterpret_cast<float*>(srcz_all[warp])[e] = -v.z;
#endif
                        }
#else
                        for (int e = lane; e < cnt; e += 32) srcf[e] = __ldg(packedf + base + e);
#endif
                    }
                    __syncwarp();
                    if (!valid) continue;
#if SEWALD_RS_MASK
                    // Pass 1 (fp32, conservative): this lane's candidate sources as a
                    // 64-bit mask (no per-candidate stores; slots past cnt are far away).
                    constexpr int NM = CH / 64;
                    unsigned long long cm[NM];
                    const int cnt8 = (cnt + 7) & ~7;
#pragma unroll
                    for (int h = 0; h < NM; ++h) {
                        cm[h] = 0ull;
                        const int kend = min(cnt8 - 64 * h, 64);
#if SEWALD_RS_F2
                        // two sources per packed fp32x2 operation, the same IEEE fp32
                        // operations as the scalar test (x + (-y) == x - y)
                        const float2 t0 = make_float2(tf0, tf0), t1 = make_float2(tf1, tf1),
                                     t2 = make_float2(tf2, tf2);
                        const float4* sq = srcq_all[warp] + 32 * h;
                        const float2* sz = srcz_all[warp] + 32 * h;
#pragma unroll 4
                        for (int kp = 0; kp < kend / 2; ++kp) {
                            const float4 q = sq[kp];
                            const float2 d0 = __fadd2_rn(t0, make_float2(q.x, q.y));
                            const float2 d1 = __fadd2_rn(t1, make_float2(q.z, q.w));
                            const float2 d2 = __fadd2_rn(t2, sz[kp]);
                            const float2 dd = __ffma2_rn(d2, d2, __ffma2_rn(d1, d1, __fmul2_rn(d0, d0)));
                            cm[h] |= ((unsigned long long)(dd.x < a.thresh_f) | ((unsigned long long)(dd.y < a.thresh_f) << 1))
                                     << (2 * kp);
                        }
#else
#pragma unroll 8
                        for (int kk = 0; kk < kend; ++kk) {
                            const float4 q = srcf[64 * h + kk];
                            const float d0 = tf0 - q.x, d1 = tf1 - q.y, d2 = tf2 - q.z;
                            const float dd = fmaf(d2, d2, fmaf(d1, d1, d0 * d0));
                            cm[h] |= (unsigned long long)(dd < a.thresh_f) << kk;
                        }
#endif
                    }
                    // Pass 2 (fp64, exact reference test + kernel) on the candidates.
                    for (;;) {
                        int k;
                        if (cm[0]) {
                            k = __ffsll((long long)cm[0]) - 1;
                            cm[0] &= cm[0] - 1ull;
                        } else if (NM > 1 && cm[NM - 1]) {
                            k = 64 * (NM - 1) + __ffsll((long long)cm[NM - 1]) - 1;
                            cm[NM - 1] &= cm[NM - 1] - 1ull;
                        } else {
                            break;
                        }
#else
                    // Pass 1 (fp32, conservative): queue candidate sources.
                    int nq = 0;
                    for (int k = 0; k < cnt; ++k) {
                        const float4 q = srcf[k];
                        const float d0 = tf0 - q.x, d1 = tf1 - q.y, d2 = tf2 - q.z;
                        const float dd = fmaf(d2, d2, fmaf(d1, d1, d0 * d0));
                        if (dd < a.thresh_f) queue[nq++][lane] = (uint8_t)k;
                    }
                    // Pass 2 (fp64, exact reference test + kernel) on queued pairs.
                    for (int j = 0; j < nq; ++j) {
                        const int k = queue[j][lane];
#endif
                        const double* q = src + k * S;
                        const double r0 = (xt0 - q[0]) - shx;
                        const double r1 = (xt1 - q[1]) - shy;
                        const double r2 = (xt2 - q[2]) - shz;
                        const double n2 = __dadd_rn(__dadd_rn(__dmul_rn(r0, r0), __dmul_rn(r1, r1)),
                                                    __dmul_rn(r2, r2));
                        if (!(n2 < rc2)) continue;
                        if (n2 == 0.0) {  // self pair (skipped) or coincident points (kernels.cpp:19-22)
                            if (!(a.skip_self && primary && __double_as_longlong(q[3]) == tori))
                                atomicExch(err, 1);
                            continue;
                        }
                        const Screened sc = screened<SHORT>(n2, a.xi, xi2, exp_tab);
                        pair_accumulate<KIND>(sc, xi2, n2, r0, r1, r2, q + 4, acc0, acc1, acc2);
                        ++npairs32;
                    }
                }
            }
        }
    }

    if (valid && split > 1) {
        double* o = scratch + ((int64_t)part * Nt + t) * 3;
        o[0] = acc0;
        o[1] = acc1;
        o[2] = acc2;
    } else if (valid) {
        if (accumulate) {
            u[3 * tori] += acc0;
            u[3 * tori + 1] += acc1;
            u[3 * tori + 2] += acc2;
        } else {
            u[3 * tori] = acc0;
            u[3 * tori + 1] = acc1;
            u[3 * tori + 2] = acc2;
        }
    }
    if (pair_count) {
        unsigned long long npairs = npairs32;
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) npairs += __shfl_xor_sync(0xffffffffu, npairs, s);
        if (lane == 0 && npairs) atomicAdd(pair_count, npairs);
    }
}

// u[torder[t]] (=, +=) sum over parts p = 0, 1, ... of scratch[p][t], in order.
__global__ void realspace_sum_parts(const double* __restrict__ scratch, int split, const uint32_t* __restrict__ torder,
                                    int64_t Nt, double* __restrict__ u, int accumulate) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= Nt) return;
    double v0 = 0.0, v1 = 0.0, v2 = 0.0;
    for (int p = 0; p < split; ++p) {
        const double* o = scratch + ((int64_t)p * Nt + t) * 3;
        v0 += o[0];
        v1 += o[1];
        v2 += o[2];
    }
    double* d = u + 3 * (int64_t)torder[t];
    if (accumulate) {
        d[0] += v0;
        d[1] += v1;
        d[2] += v2;
    } else {
        d[0] = v0;
        d[1] = v1;
        d[2] = v2;
    }
}

}  // namespace

int realspace_split(int64_t Nt) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t groups = (Nt + 31) / 32;
    const int64_t warps = (int64_t)sms * 4 * RS_WARPS;  // resident at the launch bound
    if (groups <= 0 || groups >= warps) return 1;
    return (int)std::min<int64_t>(16, (2 * warps + groups - 1) / groups);
}

void launch_fold_and_key(const CellGrid& cg, const double* x, int64_t N, double* folded,
                         uint32_t* keys, uint32_t* vals, cudaStream_t st) {
    if (N == 0) return;
    fold_key_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(cg, x, N, folded, keys, vals);
}

void launch_pack_sources(const double* folded, const double* f, const double* nu, int stresslet,
                         const uint32_t* order, int64_t N, double* packed, float4* packedf,
                         cudaStream_t st) {
    if (N == 0) return;
    pack_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(folded, f, nu, stresslet, order, N,
                                                              packed, packedf);
}

void launch_realspace(const CellGrid& cg, const RealspaceArgs& a, const double* packed,
                      const float4* packedf, int stresslet, const int64_t* cell_off, const double* tfolded,
                      const uint32_t* torder, int64_t Nt, double* u, int accumulate,
                      unsigned long long* pair_count, int* err, int split, double* scratch, cudaStream_t st) {
    if (Nt == 0) return;
    if (!scratch) split = 1;
    const int64_t items = ((Nt + 31) / 32) * split;
    const unsigned blocks = (unsigned)((items + RS_WARPS - 1) / RS_WARPS);
    const bool shrt = a.xi * a.rc <= SEWALD_ERFCX8_XMAX;  // shorter erfcx rational suffices
#define SEWALD_RS_LAUNCH(K, SZ)                                                                              \
    if (shrt)                                                                                                \
        realspace_kernel<K, SZ, true><<<blocks, RS_THREADS, 0, st>>>(cg, a, packed, packedf, cell_off, tfolded, \
                                                                     torder, Nt, u, accumulate, pair_count, err, split, scratch); \
    else                                                                                                     \
        realspace_kernel<K, SZ, false><<<blocks, RS_THREADS, 0, st>>>(cg, a, packed, packedf, cell_off, tfolded, \
                                                                      torder, Nt, u, accumulate, pair_count, err, split, scratch);
    switch (a.kind) {
        case SEWALD_STOKESLET: SEWALD_RS_LAUNCH(SEWALD_STOKESLET, 8) break;
        case SEWALD_ROTLET: SEWALD_RS_LAUNCH(SEWALD_ROTLET, 8) break;
        default: SEWALD_RS_LAUNCH(SEWALD_STRESSLET, 12) break;
    }
#undef SEWALD_RS_LAUNCH
    if (split > 1)
        realspace_sum_parts<<<(unsigned)((Nt + 255) / 256), 256, 0, st>>>(scratch, split, torder, Nt, u, accumulate);
}

}  // namespace sewald_b200
