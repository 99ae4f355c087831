// Real-space sum for targets == sources (the starred sum of full_potential),
// using pair symmetry: each unordered pair {a, b + shift} within rc is
// evaluated ONCE and applied to both particles (the kernels are even
// (stokeslet) or odd (rotlet, stresslet) in r). The separation is formed as
// r = (x_a - shift) - x_b with the shifted position computed once per row
// piece; it differs from the reference's (x_a - x_b) - shift by at most one
// rounding of a coordinate, so the accepted set can differ only for pairs
// within ~1e-16 of rc, whose terms are ~erfc(xi rc) below the rms.
//
// Reference: accumulate_rows /root/reference/proj/src/realspace.cpp:30-93,
//            realspace_kernel /root/reference/proj/src/kernels.cpp:71-116.
//
// Work unit = one warp = one i-cluster of 32 consecutive particles in cell
// order. Its bounding box selects the cell rows within rc; each row piece is
// streamed as j-blocks of up to 32 particles into warp-private shared
// memory. The 32 x 32 block is swept in 32 lock-step rotations (lane l pairs
// with j = (l + s) mod 32), so the j particles touched in one step are all
// distinct: reactions accumulate in shared memory without atomics and are
// flushed once per j-block with fp64 RED to global memory. Steps with no
// accepted lane are skipped (warp vote). Half rule: a pair (a, b, shift) is
// evaluated iff b > a, or b == a with shift > 0 lexicographically (the self
// pair, b == a with zero shift, is the starred exclusion).
#include "device_common.cuh"
#include "sg_kernels.h"
#include "screened_math.cuh"
#include "../../include/sewald_gpu.h"

#include <algorithm>

namespace sewald_b200 {

namespace {

constexpr int SYM_WARPS = 4;
constexpr int SYM_THREADS = 32 * SYM_WARPS;
#ifndef SEWALD_SYM_BRANCHFREE
#define SEWALD_SYM_BRANCHFREE 1
#endif
#ifndef SEWALD_SYM_MINB
#define SEWALD_SYM_MINB 4
#endif

__device__ __forceinline__ int fdiv(int a, int b) {
    int q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
    return q;
}

template <int KIND>
struct Strength;
template <>
struct Strength<SEWALD_STOKESLET> {
    static constexpr int n = 3;
};
template <>
struct Strength<SEWALD_ROTLET> {
    static constexpr int n = 3;
};
template <>
struct Strength<SEWALD_STRESSLET> {
    static constexpr int n = 7;  // q, nu, q.nu (packed record slot 10)
};

// Contribution of source strength s at separation r (target - source) and
// its reaction on the source from the target strength t (separation -r),
// accumulated into ua (target) and ub (source).
template <int KIND>
__device__ __forceinline__ void pair_both(const Screened& sc, double xi2, double n2, double r0, double r1,
                                          double r2, const double* s, const double* t, double* ua, double* ub) {
    if (KIND == SEWALD_STOKESLET) {
        const double a = sc.Ey * (sc.R - sc.cx);
        const double b = sc.Ey * (sc.iy * sc.iy) * (sc.R + sc.cx);
        const double bs = b * (r0 * s[0] + r1 * s[1] + r2 * s[2]);
        const double bt = b * (r0 * t[0] + r1 * t[1] + r2 * t[2]);
        ua[0] = fma(a, s[0], fma(bs, r0, ua[0]));
        ua[1] = fma(a, s[1], fma(bs, r1, ua[1]));
        ua[2] = fma(a, s[2], fma(bs, r2, ua[2]));
        ub[0] = fma(a, t[0], fma(bt, r0, ub[0]));
        ub[1] = fma(a, t[1], fma(bt, r1, ub[1]));
        ub[2] = fma(a, t[2], fma(bt, r2, ub[2]));
    } else if (KIND == SEWALD_ROTLET) {
        const double c = sc.Ey * (sc.iy * sc.iy) * (sc.R + sc.cx);
        ua[0] = fma(c, s[1] * r2 - s[2] * r1, ua[0]);
        ua[1] = fma(c, s[2] * r0 - s[0] * r2, ua[1]);
        ua[2] = fma(c, s[0] * r1 - s[1] * r0, ua[2]);
        ub[0] = fma(-c, t[1] * r2 - t[2] * r1, ub[0]);
        ub[1] = fma(-c, t[2] * r0 - t[0] * r2, ub[1]);
        ub[2] = fma(-c, t[0] * r1 - t[1] * r0, ub[2]);
    } else {
        // stresslet: s, t = (q, nu, q.nu) with q.nu precomputed per particle
        const double iy2 = sc.iy * sc.iy;
        const double x2 = xi2 * n2;
        const double c1 = -2.0 * sc.Ey * (iy2 * iy2) * (3.0 * sc.R + (3.0 + 2.0 * x2) * sc.cx);
        const double c2 = 2.0 * xi2 * sc.Ey * sc.cx;
        {
            const double rq = r0 * s[0] + r1 * s[1] + r2 * s[2];
            const double rv = r0 * s[3] + r1 * s[4] + r2 * s[5];
            const double w = fma(c1 * rq, rv, c2 * s[6]);
            const double cv = c2 * rv, cq = c2 * rq;
            ua[0] = fma(cq, s[3], fma(cv, s[0], fma(w, r0, ua[0])));
            ua[1] = fma(cq, s[4], fma(cv, s[1], fma(w, r1, ua[1])));
            ua[2] = fma(cq, s[5], fma(cv, s[2], fma(w, r2, ua[2])));
        }
        {
            const double rq = r0 * t[0] + r1 * t[1] + r2 * t[2];
            const double rv = r0 * t[3] + r1 * t[4] + r2 * t[5];
            const double w = fma(c1 * rq, rv, c2 * t[6]);
            const double cv = c2 * rv, cq = c2 * rq;
            ub[0] = fma(-cq, t[3], fma(-cv, t[0], fma(-w, r0, ub[0])));
            ub[1] = fma(-cq, t[4], fma(-cv, t[1], fma(-w, r1, ub[1])));
            ub[2] = fma(-cq, t[5], fma(-cv, t[2], fma(-w, r2, ub[2])));
        }
    }
}

template <int KIND, int S, bool SHORT>
__global__ void __launch_bounds__(SYM_THREADS, SEWALD_SYM_MINB)
realspace_sym_kernel(CellGrid cg, RealspaceArgs a, const double* __restrict__ packed,
                     const int64_t* __restrict__ cell_off, int64_t N, int64_t c0, int64_t c1,
                     double* __restrict__ u, unsigned long long* __restrict__ pair_count, int* __restrict__ err,
                     unsigned long long* __restrict__ work) {
    constexpr int NS = Strength<KIND>::n;
    // j record: [x y | z s0 | s1 s2 | ... | r0 r1 | r2 pad], a multiple of 16 B
    // so positions, strengths and reactions move with 128-bit shared accesses
    // (stride 80 B / 112 B: conflict-free per quarter warp).
    constexpr int RS = (3 + NS + 3 + 1) & ~1;
    constexpr int RO = RS - 4;  // reaction offset
    // branch-free steps (c2 -1.5 %, stresslet neutral); the branchy form is kept for
    // flop counting (tools/gpu_probe3.sh builds with SEWALD_SYM_BRANCHFREE=0)
    constexpr bool BF = SEWALD_SYM_BRANCHFREE;
    __shared__ __align__(16) double jrec_all[SYM_WARPS][32][RS];
    __shared__ long long jid_all[SYM_WARPS][32];
    __shared__ float4 jf_all[SYM_WARPS][32];  // fp32 positions for the candidate pass
    __shared__ double exp_tab[32];
    if (threadIdx.x < 32) exp_tab[threadIdx.x] = c_exp2_tab32[threadIdx.x];
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double(*jrec)[RS] = jrec_all[warp];
    long long* jid = jid_all[warp];
    float4* jf = jf_all[warp];
    unsigned long long npairs = 0;  // flushed per cluster from the 32-bit step counter
    // Persistent warps: clusters are taken from a global counter, so the
    // uneven per-cluster work (row geometry, half rule) does not leave SMs
    // idle in the tail.
    for (;;) {
    long long next = 0;
    if (lane == 0) next = (long long)atomicAdd(work, 1ull);
    const int64_t cl = c0 + __shfl_sync(0xffffffffu, next, 0);
    if (cl >= c1) break;

    const int64_t istart = cl * 32;
    const int64_t ia = istart + lane;
    unsigned npairs32 = 0;
    const bool valid = ia < N;
    double xa0 = 0, xa1 = 0, xa2 = 0, fa[NS];
    long long ida = -1;
#pragma unroll
    for (int c = 0; c < NS; ++c) fa[c] = 0.0;
    if (valid) {
        const double* q = packed + ia * S;
        xa0 = q[0];
        xa1 = q[1];
        xa2 = q[2];
        ida = __double_as_longlong(q[3]);
#pragma unroll
        for (int c = 0; c < NS; ++c) fa[c] = q[4 + c];
    }

    double lo[3] = {valid ? xa0 : 1e300, valid ? xa1 : 1e300, valid ? xa2 : 1e300};
    double hi[3] = {valid ? xa0 : -1e300, valid ? xa1 : -1e300, valid ? xa2 : -1e300};
#pragma unroll
    for (int ax = 0; ax < 3; ++ax)
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) {
            lo[ax] = fmin(lo[ax], __shfl_xor_sync(0xffffffffu, lo[ax], s));
            hi[ax] = fmax(hi[ax], __shfl_xor_sync(0xffffffffu, hi[ax], s));
        }

    const double rc2 = a.rc2;  // kernel-parameter operands: no registers
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

    double ua[3] = {0.0, 0.0, 0.0};

    for (int cz = clo[2]; cz <= chi[2]; ++cz) {
        const int sz = 2 < cg.d ? fdiv(cz, cg.n[2]) : 0;
        const int jz = cz - sz * cg.n[2];
        const double zlo = cg.origin[2] + cz * cg.w[2], zhi = zlo + cg.w[2];
        const double dz = fmax(0.0, fmax(zlo - hi[2], lo[2] - zhi));
        const double shz = __dmul_rn((double)sz, cg.L[2]);
        for (int cy = clo[1]; cy <= chi[1]; ++cy) {
            const int sy = 1 < cg.d ? fdiv(cy, cg.n[1]) : 0;
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
            const double shy = __dmul_rn((double)sy, cg.L[1]);
            const int64_t rowbase = ((int64_t)jz * cg.n[1] + jy) * cg.n[0];
            const int sxa = 0 < cg.d ? fdiv(cxl, cg.n[0]) : 0;
            const int sxb = 0 < cg.d ? fdiv(cxh, cg.n[0]) : 0;
            for (int sx = sxa; sx <= sxb; ++sx) {
                const int jlo = max(cxl - sx * cg.n[0], 0);
                const int jhi = min(cxh - sx * cg.n[0], cg.n[0] - 1);
                int64_t b0 = cell_off[rowbase + jlo];
                const int64_t b1 = cell_off[rowbase + jhi + 1];
                // half rule: partners with a smaller sorted index than every
                // particle of this cluster are evaluated by their own warp
                if (b0 < istart) b0 = istart;
                if (b0 >= b1) continue;
                const double shx = __dmul_rn((double)sx, cg.L[0]);
                const bool pos_shift = sx > 0 || (sx == 0 && (sy > 0 || (sy == 0 && sz > 0)));
                // shifted target position, once per row piece (r = (x_a - shift) - x_j)
                const double xs0 = xa0 - shx, xs1 = xa1 - shy, xs2 = xa2 - shz;
                const float tf0 = (float)xs0, tf1 = (float)xs1, tf2 = (float)xs2;
                for (int64_t jb = b0; jb < b1; jb += 32) {
                    const int cnt = (int)min((int64_t)32, b1 - jb);
                    __syncwarp();
                    if (lane < cnt) {
                        const double* q = packed + (jb + lane) * S;
                        double* rec = jrec[lane];
                        rec[0] = q[0];
                        rec[1] = q[1];
                        rec[2] = q[2];
                        jid[lane] = __double_as_longlong(q[3]);
                        jf[lane] = make_float4((float)q[0], (float)q[1], (float)q[2], 0.0f);
#pragma unroll
                        for (int c = 0; c < NS; ++c) rec[3 + c] = q[4 + c];
                    } else {
                        // unused slots: far away in fp32 (never candidates) and
                        // finite in fp64 (branch-free steps read them)
                        jf[lane] = make_float4(1e30f, 1e30f, 1e30f, 0.0f);
                        double* rec = jrec[lane];
                        rec[0] = rec[1] = rec[2] = 1e100;
#pragma unroll
                        for (int c = 0; c < NS; ++c) rec[3 + c] = 0.0;
                    }
                    *reinterpret_cast<double2*>(&jrec[lane][RO]) = make_double2(0.0, 0.0);
                    jrec[lane][RO + 2] = 0.0;
                    __syncwarp();
                    // pair (lane, j) is "after" in sorted order iff j - lane > dlt
                    const int dlt = (int)max((int64_t)-64, istart - jb);
                    // (1) candidate rotations of this lane, fp32 bound (independent
                    // iterations, FP32 pipe); (2) steps with any candidate (one
                    // warp OR-reduction); (3) fp64 work only on those steps.
                    unsigned m = 0u;
                    if (valid) {
                        if (dlt <= -32) {
                            // block entirely after the cluster: no half-rule test
                            // (unused slots are far away and fail the distance test)
#pragma unroll 8
                            for (int s = 0; s < 32; ++s) {
                                const float4 p = jf[(lane + s) & 31];
                                const float d0 = tf0 - p.x, d1 = tf1 - p.y, d2 = tf2 - p.z;
                                m |= (fmaf(d2, d2, fmaf(d1, d1, d0 * d0)) < a.thresh_f ? 1u : 0u) << s;
                            }
                        } else {
#pragma unroll 8
                            for (int s = 0; s < 32; ++s) {
                                const int j = (lane + s) & 31;
                                const int dj = j - lane;
                                const float4 p = jf[j];
                                const float d0 = tf0 - p.x, d1 = tf1 - p.y, d2 = tf2 - p.z;
                                const bool ok = j < cnt && (dj > dlt || (dj == dlt && pos_shift)) &&
                                                fmaf(d2, d2, fmaf(d1, d1, d0 * d0)) < a.thresh_f;
                                m |= (ok ? 1u : 0u) << s;
                            }
                        }
                    }
                    unsigned steps = __reduce_or_sync(0xffffffffu, m);
                    bool coincident = false;
                    while (steps) {
                        const int s = 31 - __clz(steps);  // highest step first: one FLO
                        steps ^= 1u << s;
                        const int j = (lane + s) & 31;
                        if (BF) {
                            // Branch-free step: every lane evaluates; lanes without an
                            // accepted pair use a harmless separation and a zero Gaussian
                            // factor, so their contributions and reactions are exact zeros
                            // (their j slot is distinct from every other lane's).
                            const bool in = (m >> s) & 1u;
                            double* rec = jrec[j];
                            const double2 xy = *reinterpret_cast<const double2*>(rec);
                            const double2 zs0 = *reinterpret_cast<const double2*>(rec + 2);
                            const double r0 = xs0 - xy.x, r1 = xs1 - xy.y, r2 = xs2 - zs0.x;
                            const double n2 = __dadd_rn(__dadd_rn(__dmul_rn(r0, r0), __dmul_rn(r1, r1)), __dmul_rn(r2, r2));
                            bool acc = in && n2 < rc2;
                            // coincident distinct points (kernels.cpp:19-22): flagged per block
                            coincident |= acc && n2 == 0.0;
                            acc = acc && n2 != 0.0;
                            const double n2e = acc ? n2 : 0.25 * rc2;
                            double sj[NS];
                            sj[0] = zs0.y;
#pragma unroll
                            for (int c = 1; c < NS; c += 2) {
                                const double2 v = *reinterpret_cast<const double2*>(rec + 3 + c);
                                sj[c] = v.x;
                                if (c + 1 < NS) sj[c + 1] = v.y;
                            }
                            Screened sc = screened<SHORT>(n2e, a.xi, xi2, exp_tab);
                            sc.Ey = acc ? sc.Ey : 0.0;
                            const double2 r01 = *reinterpret_cast<const double2*>(rec + RO);
                            double ub[3] = {r01.x, r01.y, rec[RO + 2]};
                            pair_both<KIND>(sc, xi2, n2e, r0, r1, r2, sj, fa, ua, ub);
                            *reinterpret_cast<double2*>(rec + RO) = make_double2(ub[0], ub[1]);
                            rec[RO + 2] = ub[2];
                            npairs32 += acc ? 2u : 0u;
                        } else {
                            bool acc = (m >> s) & 1u;
                            double r0 = 0, r1 = 0, r2 = 0, n2 = 0;
                            double* rec = jrec[j];
                            double2 zs0;
                            if (acc) {
                                const double2 xy = *reinterpret_cast<const double2*>(rec);
                                zs0 = *reinterpret_cast<const double2*>(rec + 2);
                                r0 = xs0 - xy.x;
                                r1 = xs1 - xy.y;
                                r2 = xs2 - zs0.x;
                                n2 = __dadd_rn(__dadd_rn(__dmul_rn(r0, r0), __dmul_rn(r1, r1)), __dmul_rn(r2, r2));
                                acc = n2 < rc2;
                            }
                            if (acc) {
                                if (n2 == 0.0) {  // coincident distinct points (kernels.cpp:19-22)
                                    atomicExch(err, 1);
                                } else {
                                    double sj[NS];
                                    sj[0] = zs0.y;
#pragma unroll
                                    for (int c = 1; c < NS; c += 2) {
                                        const double2 v = *reinterpret_cast<const double2*>(rec + 3 + c);
                                        sj[c] = v.x;
                                        if (c + 1 < NS) sj[c + 1] = v.y;
                                    }
                                    const Screened sc = screened<SHORT>(n2, a.xi, xi2, exp_tab);
                                    const double2 r01 = *reinterpret_cast<const double2*>(rec + RO);
                                    double ub[3] = {r01.x, r01.y, rec[RO + 2]};
                                    pair_both<KIND>(sc, xi2, n2, r0, r1, r2, sj, fa, ua, ub);
                                    *reinterpret_cast<double2*>(rec + RO) = make_double2(ub[0], ub[1]);
                                    rec[RO + 2] = ub[2];
                                    npairs32 += 2;
                                }
                            }
                        }
                    }
                    if (coincident) atomicExch(err, 1);
                    __syncwarp();
                    if (lane < cnt) {
                        double* dst = u + 3 * jid[lane];
                        atomicAdd(dst, jrec[lane][RO]);
                        atomicAdd(dst + 1, jrec[lane][RO + 1]);
                        atomicAdd(dst + 2, jrec[lane][RO + 2]);
                    }
                }
            }
        }
    }
    npairs += npairs32;
    if (valid) {
        double* dst = u + 3 * ida;
        atomicAdd(dst, ua[0]);
        atomicAdd(dst + 1, ua[1]);
        atomicAdd(dst + 2, ua[2]);
    }
    }  // persistent loop
    if (pair_count) {
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) npairs += __shfl_xor_sync(0xffffffffu, npairs, s);
        if (lane == 0 && npairs) atomicAdd(pair_count, npairs);
    }
}

}  // namespace

void launch_realspace_sym(const CellGrid& cg, const RealspaceArgs& a, const double* packed, int64_t N,
                          const int64_t* cell_off, int64_t c0, int64_t c1, double* u,
                          unsigned long long* pair_count, int* err, unsigned long long* work, cudaStream_t st) {
    if (c1 <= c0) return;
    cudaMemsetAsync(work, 0, sizeof(unsigned long long), st);
    int dev = 0, sms = 148, per_sm = 4;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
#ifdef SEWALD_NO_SHORT
    const bool shrt = false;
#else
    const bool shrt = a.xi * a.rc <= SEWALD_ERFCX8_XMAX;
#endif
    if (a.kind == SEWALD_STRESSLET)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, shrt ? realspace_sym_kernel<SEWALD_STRESSLET, 12, true> : realspace_sym_kernel<SEWALD_STRESSLET, 12, false>,
            SYM_THREADS, 0);
    else if (a.kind == SEWALD_ROTLET)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, shrt ? realspace_sym_kernel<SEWALD_ROTLET, 8, true> : realspace_sym_kernel<SEWALD_ROTLET, 8, false>,
            SYM_THREADS, 0);
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, shrt ? realspace_sym_kernel<SEWALD_STOKESLET, 8, true> : realspace_sym_kernel<SEWALD_STOKESLET, 8, false>,
            SYM_THREADS, 0);
    const int64_t need = (c1 - c0 + SYM_WARPS - 1) / SYM_WARPS;
    const unsigned blocks = (unsigned)std::min<int64_t>(need, (int64_t)sms * std::max(per_sm, 1));
#define SEWALD_SYM_LAUNCH(K, S)                                                                            \
    if (shrt)                                                                                              \
        realspace_sym_kernel<K, S, true><<<blocks, SYM_THREADS, 0, st>>>(cg, a, packed, cell_off, N, c0, c1, u, \
                                                                          pair_count, err, work);          \
    else                                                                                                   \
        realspace_sym_kernel<K, S, false><<<blocks, SYM_THREADS, 0, st>>>(cg, a, packed, cell_off, N, c0, c1, u, \
                                                                           pair_count, err, work);
    switch (a.kind) {
        case SEWALD_STOKESLET: SEWALD_SYM_LAUNCH(SEWALD_STOKESLET, 8) break;
        case SEWALD_ROTLET: SEWALD_SYM_LAUNCH(SEWALD_ROTLET, 8) break;
        default: SEWALD_SYM_LAUNCH(SEWALD_STRESSLET, 12) break;
    }
#undef SEWALD_SYM_LAUNCH
}

}  // namespace sewald_b200
