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
#ifndef SEWALD_SYM_BCAST
#define SEWALD_SYM_BCAST 1
#endif
// packed fp32x2 candidate pass (needs SEWALD_SYM_BCAST)
#ifndef SEWALD_SYM_F2
#define SEWALD_SYM_F2 1
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

// The same pair split in two halves so that two pairs can be in flight per
// lane (SEWALD_SYM_ILP = 2): the scalar coefficients of a pair, then its
// contribution to one side. sign = +1 for the target (separation r), -1 for
// the source's reaction (separation -r: the odd kernels change sign).
template <int KIND>
struct PairCoef {
    double a, b;
};

template <int KIND>
__device__ __forceinline__ PairCoef<KIND> pair_coef(const Screened& sc, double xi2, double n2) {
    PairCoef<KIND> c;
    if (KIND == SEWALD_STOKESLET) {
        c.a = sc.Ey * (sc.R - sc.cx);
        c.b = sc.Ey * (sc.iy * sc.iy) * (sc.R + sc.cx);
    } else if (KIND == SEWALD_ROTLET) {
        c.a = sc.Ey * (sc.iy * sc.iy) * (sc.R + sc.cx);
        c.b = 0.0;
    } else {
        const double iy2 = sc.iy * sc.iy;
        const double x2 = xi2 * n2;
        c.a = -2.0 * sc.Ey * (iy2 * iy2) * (3.0 * sc.R + (3.0 + 2.0 * x2) * sc.cx);
        c.b = 2.0 * xi2 * sc.Ey * sc.cx;
    }
    return c;
}

template <int KIND, bool REACTION>
__device__ __forceinline__ void pair_apply(const PairCoef<KIND>& c, double r0, double r1, double r2,
                                           const double* s, double* u) {
    if (KIND == SEWALD_STOKESLET) {
        const double bs = c.b * (r0 * s[0] + r1 * s[1] + r2 * s[2]);
        u[0] = fma(c.a, s[0], fma(bs, r0, u[0]));
        u[1] = fma(c.a, s[1], fma(bs, r1, u[1]));
        u[2] = fma(c.a, s[2], fma(bs, r2, u[2]));
    } else if (KIND == SEWALD_ROTLET) {
        const double cc = REACTION ? -c.a : c.a;
        u[0] = fma(cc, s[1] * r2 - s[2] * r1, u[0]);
        u[1] = fma(cc, s[2] * r0 - s[0] * r2, u[1]);
        u[2] = fma(cc, s[0] * r1 - s[1] * r0, u[2]);
    } else {
        const double rq = r0 * s[0] + r1 * s[1] + r2 * s[2];
        const double rv = r0 * s[3] + r1 * s[4] + r2 * s[5];
        const double w = fma(c.a * rq, rv, c.b * s[6]);
        const double cv = c.b * rv, cq = c.b * rq;
        if (REACTION) {
            u[0] = fma(-cq, s[3], fma(-cv, s[0], fma(-w, r0, u[0])));
            u[1] = fma(-cq, s[4], fma(-cv, s[1], fma(-w, r1, u[1])));
            u[2] = fma(-cq, s[5], fma(-cv, s[2], fma(-w, r2, u[2])));
        } else {
            u[0] = fma(cq, s[3], fma(cv, s[0], fma(w, r0, u[0])));
            u[1] = fma(cq, s[4], fma(cv, s[1], fma(w, r1, u[1])));
            u[2] = fma(cq, s[5], fma(cv, s[2], fma(w, r2, u[2])));
        }
    }
}

#ifndef SEWALD_SYM_ILP
#define SEWALD_SYM_ILP 1
#endif
// Blocks with fewer candidate pairs than this go through the pooled path
// (0 = rotation steps only). c2: rotation only 67.6 ms; pooled below
// 192 / 256 / 384 pairs (mode 2): 63.3 / 62.7-63.0 / 63.5 ms; mode 3 at
// 256 / 384 / 512: c2 59.1 / 58.3 / 59.0, c3 116.0 / 112.3 / 112.5,
// c5 67.0 / 66.3 / 68.0.
#ifndef SEWALD_SYM_POOL
#define SEWALD_SYM_POOL 384
#endif
// Rotation steps of denser blocks with fewer than SEWALD_SYM_SPLIT active
// lanes are pooled too (0 = off): 6 / 9 / 12 lanes measured c2 58.2 / 58.3 /
// 58.4, c3 108.7 / 108.4 / 107.9, c5 66.0 / 65.7 / 65.6 against 56.7 / 108.2 /
// 64.4 ms without (4 more registers, and the pooled pair costs ~2.5 lane-slots).
// pooled pairs' i side: 0 segmented sum into the cluster's pool, 1 global RED
// (c2 53.1 -> 52.9, c3 103.8 -> 101.8, c5 60.2 -> 61.0 ms: kept at 0)
#ifndef SEWALD_SYM_POOL_IRED
#define SEWALD_SYM_POOL_IRED 0
#endif
// Row pieces and j-blocks that no particle of the cluster can reach (per-lane
// distance to the row slab / the block's x range, one vote) are skipped before
// staging: c2 53.5 -> 50.8 ms, c3 103.8 -> 102.4, c5 60.1 -> 51.4.
#ifndef SEWALD_SYM_BLOCKTEST
#define SEWALD_SYM_BLOCKTEST 1
#endif
#ifndef SEWALD_SYM_SPLIT
#define SEWALD_SYM_SPLIT 0
#endif
#define SEWALD_SYM_QMAX (SEWALD_SYM_POOL > 32 * SEWALD_SYM_SPLIT ? SEWALD_SYM_POOL : 32 * SEWALD_SYM_SPLIT)
// Pooled pairs: history at c2 (pool threshold 256). Both sides with shared
// fp64 atomics (CAS loops; j side in the block's reaction slots) 67.0 ms; both
// sides with global fp64 RED 63.4; i side shared CAS, j side global RED 63.0
// (61.4 with the 16-byte record loads) — there the CAS loops retried ~5 times
// per batch (rotation-major batches of a sparse block repeat the few busy i
// particles) and drew 16 % of the kernel's stall samples; lane-major queue
// with the segmented i-side sum (below) 58.9 (c3 117.9 -> 115.6, c5 70.8 ->
// 66.8). Pooling whole blocks whose rotation steps would be < 40 / 55 / 70 %
// occupied: c2 58.4 / 59.8 / 63.3 against 58.2 ms (threshold only).
// j-block records loaded with 16-byte loads (c2 62.9 -> 61.3 ms, c3 118.9 ->
// 117.9, c5 72.4 -> 71.1 against 8-byte loads). A fully coalesced block load
// (lane l reading chunks l, l + 32, ... and scattering the fields) measured
// 74.6 ms: the per-lane field selection diverges four ways.
#ifndef SEWALD_SYM_VEC
#define SEWALD_SYM_VEC 1
#endif

// exp table copies (lane-interleaved, conflict-free lookups): 16 copies
// measured slower at c2 (69.0 vs 67.6 ms), so one copy.
#ifndef SEWALD_EXP_REP
#define SEWALD_EXP_REP 1
#endif

// One branch-free pair slot of a step: separation, acceptance, screened
// coefficients (zero for lanes without an accepted pair).
template <int KIND, int NS, bool SHORT>
struct SlotEval {
    double r0, r1, r2;
    PairCoef<KIND> c;
    double sj[NS];
    bool acc;
};

template <int KIND, int RS, int NS, bool SHORT>
__device__ __forceinline__ void slot_eval(SlotEval<KIND, NS, SHORT>& e, const double* rec, double xs0, double xs1,
                                          double xs2, bool in, double rc2, double xi, double xi2,
                                          const double* exp_tab, bool& coincident) {
    const double2 xy = *reinterpret_cast<const double2*>(rec);
    const double2 zs0 = *reinterpret_cast<const double2*>(rec + 2);
    e.r0 = xs0 - xy.x;
    e.r1 = xs1 - xy.y;
    e.r2 = xs2 - zs0.x;
    const double n2 = __dadd_rn(__dadd_rn(__dmul_rn(e.r0, e.r0), __dmul_rn(e.r1, e.r1)), __dmul_rn(e.r2, e.r2));
    bool acc = in && n2 < rc2;
    coincident |= acc && n2 == 0.0;
    acc = acc && n2 != 0.0;
    e.acc = acc;
    const double n2e = acc ? n2 : 0.25 * rc2;
    e.sj[0] = zs0.y;
#pragma unroll
    for (int c = 1; c < NS; c += 2) {
        const double2 v = *reinterpret_cast<const double2*>(rec + 3 + c);
        e.sj[c] = v.x;
        if (c + 1 < NS) e.sj[c + 1] = v.y;
    }
    Screened sc = screened<SHORT, SEWALD_EXP_REP>(n2e, xi, xi2, exp_tab);
    sc.Ey = acc ? sc.Ey : 0.0;
    e.c = pair_coef<KIND>(sc, xi2, n2e);
}

template <int KIND, int S, bool SHORT>
__global__ void __launch_bounds__(SYM_THREADS, SEWALD_SYM_MINB)
realspace_sym_kernel(CellGrid cg, RealspaceArgs a, const double* __restrict__ packed,
                     const int64_t* __restrict__ cell_off, int64_t N, int64_t c0, int64_t c1, int64_t cstride,
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
    // fp32 positions for the candidate pass, stored twice (slot k and k + 32) so
    // that rotation s reads jf[lane + s] at a constant offset (no wrap); with the
    // 32 rotations fully unrolled a candidate test is 9 instructions instead of
    // 14 (the kernel is issue-bound: c2 56.5 -> 53.2 ms, c3 108.0 -> 103.8, c5
    // 64.1 -> 59.8)
    __shared__ float4 jf_all[SYM_WARPS][64];
#if SEWALD_SYM_F2
    // the same fp32 positions negated and packed in pairs for the f32x2
    // candidate pass: [-x_2p, -x_2p+1, -y_2p, -y_2p+1] and [-z_2p, -z_2p+1]
    __shared__ float4 jq_all[SYM_WARPS][16];
    __shared__ float2 jz_all[SYM_WARPS][16];
#endif
    // 2^(j/32) table, replicated SEWALD_EXP_REP times (lane-interleaved: conflict-free lookups)
    __shared__ double exp_tab_rep[32 * SEWALD_EXP_REP];
#if SEWALD_SYM_POOL > 0
    // sparse-block pool (see below): the cluster's records, its pooled
    // i-side sums and the block's candidate queue, per warp
    constexpr int IS = (3 + NS) | 1;  // odd stride (in doubles): random il hit distinct banks
    __shared__ double irec_all[SYM_WARPS][32][IS];
    __shared__ double ipool_all[SYM_WARPS][32][3];
    __shared__ unsigned short queue_all[SYM_WARPS][SEWALD_SYM_QMAX];
#endif
    for (int t = threadIdx.x; t < 32 * SEWALD_EXP_REP; t += SYM_THREADS) exp_tab_rep[t] = exp_tab_entry<SHORT>(t / SEWALD_EXP_REP);
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double* exp_tab = exp_tab_rep + (lane % SEWALD_EXP_REP);
    double(*jrec)[RS] = jrec_all[warp];
    long long* jid = jid_all[warp];
    float4* jf = jf_all[warp];
#if SEWALD_SYM_F2
    float* jqf = reinterpret_cast<float*>(jq_all[warp]);
    float* jzf = reinterpret_cast<float*>(jz_all[warp]);
    // this lane's slots in the pair tables
    const int qx = (lane >> 1) * 4 + (lane & 1), qz = lane;
#define SYM_F2_STORE(X, Y, Z) { jqf[qx] = -(X); jqf[qx + 2] = -(Y); jzf[qz] = -(Z); }
#else
#define SYM_F2_STORE(X, Y, Z) {}
#endif
#if SEWALD_SYM_POOL > 0
    double(*irec)[IS] = irec_all[warp];
    double(*ipool)[3] = ipool_all[warp];
    unsigned short* queue = queue_all[warp];
#endif
    unsigned long long npairs = 0;  // flushed per cluster from the 32-bit step counter
    // Persistent warps: clusters are taken from a global counter, so the
    // uneven per-cluster work (row geometry, half rule) does not leave SMs
    // idle in the tail.
    for (;;) {
    long long next = 0;
    if (lane == 0) next = (long long)atomicAdd(work, 1ull);
    const int64_t cl = c0 + cstride * __shfl_sync(0xffffffffu, next, 0);
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

#if SEWALD_SYM_POOL > 0
    __syncwarp();
    irec[lane][0] = xa0;
    irec[lane][1] = xa1;
    irec[lane][2] = xa2;
#pragma unroll
    for (int c = 0; c < NS; ++c) irec[lane][3 + c] = fa[c];
    irec[lane][IS - 1] = __longlong_as_double(valid ? ida : 0);  // index (pad slot)
    ipool[lane][0] = ipool[lane][1] = ipool[lane][2] = 0.0;
    __syncwarp();
#endif
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
#if SEWALD_SYM_BLOCKTEST
                // per-particle distance to the row's (y, z) slab: a row piece (and
                // below, a j-block) that no particle of the cluster can reach is
                // skipped before it is staged (the cluster's bounding box reaches
                // more rows and blocks than the union of its particles' balls)
                const double ylo_f = cg.origin[1] + jy * cg.w[1], zlo_f = cg.origin[2] + jz * cg.w[2];
                const double ey = fmax(0.0, fmax(ylo_f - xs1, xs1 - (ylo_f + cg.w[1])));
                const double ez = fmax(0.0, fmax(zlo_f - xs2, xs2 - (zlo_f + cg.w[2])));
                const double lat_l = ey * ey + ez * ez;
                const bool row_near = valid && lat_l < rcm2;
                if (!__any_sync(0xffffffffu, row_near)) continue;
                const double subw = cg.w[0] / (double)(1 << cg.sub);  // x order holds up to a sub-cell
#endif
                for (int64_t jb = b0; jb < b1; jb += 32) {
                    const int cnt = (int)min((int64_t)32, b1 - jb);
#if SEWALD_SYM_BLOCKTEST
                    {
                        // x range of the block: a row piece is sorted by x up to the sub-cell width
                        const double xb0 = __ldg(packed + jb * S) - subw;
                        const double xb1 = __ldg(packed + (jb + cnt - 1) * S) + subw;
                        const double ex = fmax(0.0, fmax(xb0 - xs0, xs0 - xb1));
                        if (!__any_sync(0xffffffffu, row_near && fma(ex, ex, lat_l) < rcm2)) continue;
                    }
#endif
                    __syncwarp();
#if SEWALD_SYM_VEC
                    if (lane < cnt) {
                        // 16-byte loads of the lane's record (S doubles, 16-byte aligned):
                        // half the load instructions and L1 sectors of 8-byte loads
                        const double2* q2 = reinterpret_cast<const double2*>(packed + (jb + lane) * S);
                        double* rec = jrec[lane];
                        const double2 xy = __ldg(q2), zi = __ldg(q2 + 1);
                        rec[0] = xy.x;
                        rec[1] = xy.y;
                        rec[2] = zi.x;
                        jid[lane] = __double_as_longlong(zi.y);
                        jf[lane] = make_float4((float)xy.x, (float)xy.y, (float)zi.x, 0.0f);
                        SYM_F2_STORE((float)xy.x, (float)xy.y, (float)zi.x)
                        if (!SEWALD_SYM_BCAST) jf[lane + 32] = jf[lane];
#pragma unroll
                        for (int c = 0; c < NS; c += 2) {
                            const double2 v = __ldg(q2 + 2 + c / 2);
                            rec[3 + c] = v.x;
                            if (c + 1 < NS) rec[4 + c] = v.y;
                        }
                    } else {
#else
                    if (lane < cnt) {
                        const double* q = packed + (jb + lane) * S;
                        double* rec = jrec[lane];
                        rec[0] = q[0];
                        rec[1] = q[1];
                        rec[2] = q[2];
                        jid[lane] = __double_as_longlong(q[3]);
                        jf[lane] = make_float4((float)q[0], (float)q[1], (float)q[2], 0.0f);
                        SYM_F2_STORE((float)q[0], (float)q[1], (float)q[2])
                        if (!SEWALD_SYM_BCAST) jf[lane + 32] = jf[lane];
#pragma unroll
                        for (int c = 0; c < NS; ++c) rec[3 + c] = q[4 + c];
                    } else {
#endif
                        // unused slots: far away in fp32 (never candidates) and
                        // finite in fp64 (branch-free steps read them)
                        jf[lane] = make_float4(1e30f, 1e30f, 1e30f, 0.0f);
                        SYM_F2_STORE(1e30f, 1e30f, 1e30f)
                        if (!SEWALD_SYM_BCAST) jf[lane + 32] = jf[lane];
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
#if SEWALD_SYM_BCAST
                    // Candidate pass in j order with broadcast reads: every lane reads
                    // the same jf[j] (one shared-memory wavefront instead of four for
                    // a 16-byte access per lane at a different j), the lane's bits are
                    // collected by j and rotated into step order at the end (bit s of
                    // m <-> j = (lane + s) mod 32).
                    if (valid) {
                        unsigned mj = 0u;
                        if (dlt <= -32) {
#if SEWALD_SYM_F2
                            // two j per packed fp32x2 operation (FADD2 / FMUL2 / FFMA2):
                            // the same IEEE fp32 operations as the scalar test, so the
                            // same mask (x + (-y) == x - y exactly)
                            const float2 t0 = make_float2(tf0, tf0), t1 = make_float2(tf1, tf1),
                                         t2 = make_float2(tf2, tf2);
                            const float4* jq = jq_all[warp];
                            const float2* jz = jz_all[warp];
#pragma unroll
                            for (int jp = 0; jp < 16; ++jp) {
                                const float4 q = jq[jp];
                                const float2 d0 = __fadd2_rn(t0, make_float2(q.x, q.y));
                                const float2 d1 = __fadd2_rn(t1, make_float2(q.z, q.w));
                                const float2 d2 = __fadd2_rn(t2, jz[jp]);
                                const float2 ss = __ffma2_rn(d2, d2, __ffma2_rn(d1, d1, __fmul2_rn(d0, d0)));
                                if (ss.x < a.thresh_f) mj |= 1u << (2 * jp);
                                if (ss.y < a.thresh_f) mj |= 2u << (2 * jp);
                            }
#else
#pragma unroll
                            for (int j = 0; j < 32; ++j) {
                                const float4 p = jf[j];
                                const float d0 = tf0 - p.x, d1 = tf1 - p.y, d2 = tf2 - p.z;
                                if (fmaf(d2, d2, fmaf(d1, d1, d0 * d0)) < a.thresh_f) mj |= 1u << j;
                            }
#endif
                        } else {
#pragma unroll 8
                            for (int j = 0; j < 32; ++j) {
                                const int dj = j - lane;
                                const float4 p = jf[j];
                                const float d0 = tf0 - p.x, d1 = tf1 - p.y, d2 = tf2 - p.z;
                                const bool ok = j < cnt && (dj > dlt || (dj == dlt && pos_shift)) &&
                                                fmaf(d2, d2, fmaf(d1, d1, d0 * d0)) < a.thresh_f;
                                mj |= (ok ? 1u : 0u) << j;
                            }
                        }
                        m = __funnelshift_r(mj, mj, lane);
                    }
#else
                    if (valid) {
                        if (dlt <= -32) {
                            // block entirely after the cluster: no half-rule test
                            // (unused slots are far away and fail the distance test)
                            // fully unrolled: constant shared offsets and mask bits
                            const float4* jl = jf + lane;
#pragma unroll
                            for (int s = 0; s < 32; ++s) {
                                const float4 p = jl[s];
                                const float d0 = tf0 - p.x, d1 = tf1 - p.y, d2 = tf2 - p.z;
                                if (fmaf(d2, d2, fmaf(d1, d1, d0 * d0)) < a.thresh_f) m |= 1u << s;
                            }
                        } else {
#pragma unroll 8
                            for (int s = 0; s < 32; ++s) {
                                const int j = (lane + s) & 31;
                                const int dj = j - lane;
                                const float4 p = jf[lane + s];
                                const float d0 = tf0 - p.x, d1 = tf1 - p.y, d2 = tf2 - p.z;
                                const bool ok = j < cnt && (dj > dlt || (dj == dlt && pos_shift)) &&
                                                fmaf(d2, d2, fmaf(d1, d1, d0 * d0)) < a.thresh_f;
                                m |= (ok ? 1u : 0u) << s;
                            }
                        }
                    }
#endif
                    unsigned steps = __reduce_or_sync(0xffffffffu, m);
                    bool coincident = false;
#if SEWALD_SYM_POOL > 0
                    // Pooled pairs: every pair of a sparse block (fewer than
                    // SEWALD_SYM_POOL candidates, spread over many rotations) and, in
                    // denser blocks, the pairs of rotation steps with fewer than
                    // SEWALD_SYM_SPLIT active lanes: those steps would run mostly
                    // idle lanes. The pairs are queued lane-major (each i particle's
                    // pairs consecutive) and evaluated 32 at a time, one pair per
                    // lane: the i side is summed over each batch's runs of equal i
                    // particle (one plain shared add per run into the cluster's pool,
                    // added to the lane sums at the end), the j side goes to global
                    // memory with fp64 RED.
                    unsigned mp = m;
                    int np = __reduce_add_sync(0xffffffffu, __popc(m));
                    if (np >= SEWALD_SYM_POOL) {
#if SEWALD_SYM_SPLIT > 0
                        // active lanes per rotation step: 32 x 32 bit transpose of the
                        // masks (lane k ends up with the lane bits of step 31 - k)
                        unsigned x = m, msk = 0x0000FFFFu;
#pragma unroll
                        for (int jj = 16; jj > 0; jj >>= 1, msk ^= msk << jj) {
                            const unsigned y = __shfl_xor_sync(0xffffffffu, x, jj);
                            if (lane & jj)
                                x ^= ((y ^ (x >> jj)) & msk) << jj;
                            else
                                x ^= (x ^ (y >> jj)) & msk;
                        }
                        const unsigned sparse =
                            __brev(__ballot_sync(0xffffffffu, __popc(x) < SEWALD_SYM_SPLIT)) & steps;
                        mp = m & sparse;
                        np = sparse ? __reduce_add_sync(0xffffffffu, __popc(mp)) : 0;
                        steps &= ~sparse;
#else
                        np = 0;
#endif
                    } else {
                        steps = 0u;  // the rotation loop below has nothing left
                    }
                    if (np > 0) {
                        {
                            const int cntm = __popc(mp);
                            int off = cntm;
#pragma unroll
                            for (int d = 1; d < 32; d <<= 1) {
                                const int t = __shfl_up_sync(0xffffffffu, off, d);
                                if (lane >= d) off += t;
                            }
                            off -= cntm;
                            unsigned mm = mp;
                            while (mm) {
                                const int s = __ffs(mm) - 1;
                                mm &= mm - 1u;
                                queue[off++] = (unsigned short)((lane << 5) | ((lane + s) & 31));
                            }
                        }
                        __syncwarp();
                        for (int k0 = 0; k0 < np; k0 += 32) {
                            const int k = k0 + lane;
                            const bool in = k < np;
                            const int e = in ? queue[k] : 0;
                            const int il = e >> 5, j = e & 31;
                            const double* ir = irec[il];
                            const double ys0 = ir[0] - shx, ys1 = ir[1] - shy, ys2 = ir[2] - shz;
                            double fi[NS];
#pragma unroll
                            for (int c = 0; c < NS; ++c) fi[c] = ir[3 + c];
                            SlotEval<KIND, NS, SHORT> ev;
                            slot_eval<KIND, RS, NS, SHORT>(ev, jrec[j], ys0, ys1, ys2, in, rc2, a.xi, xi2, exp_tab,
                                                          coincident);
                            double ui[3] = {0.0, 0.0, 0.0};
                            if (ev.acc) {
                                double uj[3] = {0.0, 0.0, 0.0};
                                pair_apply<KIND, false>(ev.c, ev.r0, ev.r1, ev.r2, ev.sj, ui);
                                pair_apply<KIND, true>(ev.c, ev.r0, ev.r1, ev.r2, fi, uj);
                                double* dj = u + 3 * jid[j];
#pragma unroll
                                for (int c = 0; c < 3; ++c) atomicAdd(dj + c, uj[c]);
                                npairs32 += 2u;
                            }
#if SEWALD_SYM_POOL_IRED
                            if (ev.acc) {  // i side with global fp64 RED as well (no scan)
                                double* di = u + 3 * __double_as_longlong(irec[il][IS - 1]);
#pragma unroll
                                for (int c = 0; c < 3; ++c) atomicAdd(di + c, ui[c]);
                            }
#else
                            const unsigned same = __match_any_sync(0xffffffffu, in ? il : 32 + lane);
                            const int first = __ffs(same) - 1;
                            const int runmax = __reduce_max_sync(0xffffffffu, __popc(same));
                            for (int d = 1; d < runmax; d <<= 1) {
#pragma unroll
                                for (int c = 0; c < 3; ++c) {
                                    const double t = __shfl_up_sync(0xffffffffu, ui[c], d);
                                    if (lane - d >= first) ui[c] += t;
                                }
                            }
                            if (in && lane == 31 - __clz(same)) {
#pragma unroll
                                for (int c = 0; c < 3; ++c) ipool[il][c] += ui[c];
                            }
                            __syncwarp();
#endif
                        }
                    }
#endif
                    const bool rotated = steps != 0u;  // reaction slots written: flush below
#if SEWALD_SYM_ILP == 2
                    // Two steps in flight per lane: their scalar math is independent
                    // (hides the fp64 dependency latency); the reactions are applied
                    // one step after the other with a warp barrier between, since
                    // lane l's slot in the second step can be another lane's slot in
                    // the first.
                    while (BF && steps) {
                        const int s1 = 31 - __clz(steps);
                        steps ^= 1u << s1;
                        const int j1 = (lane + s1) & 31;
                        if (steps == 0u) {
                            SlotEval<KIND, NS, SHORT> e;
                            double* rec = jrec[j1];
                            slot_eval<KIND, RS, NS, SHORT>(e, rec, xs0, xs1, xs2, (m >> s1) & 1u, rc2, a.xi, xi2,
                                                          exp_tab, coincident);
                            pair_apply<KIND, false>(e.c, e.r0, e.r1, e.r2, e.sj, ua);
                            const double2 r01 = *reinterpret_cast<const double2*>(rec + RO);
                            double ub[3] = {r01.x, r01.y, rec[RO + 2]};
                            pair_apply<KIND, true>(e.c, e.r0, e.r1, e.r2, fa, ub);
                            *reinterpret_cast<double2*>(rec + RO) = make_double2(ub[0], ub[1]);
                            rec[RO + 2] = ub[2];
                            npairs32 += e.acc ? 2u : 0u;
                            break;
                        }
                        const int s2 = 31 - __clz(steps);
                        steps ^= 1u << s2;
                        const int j2 = (lane + s2) & 31;
                        SlotEval<KIND, NS, SHORT> e1, e2;
                        double* rec1 = jrec[j1];
                        double* rec2 = jrec[j2];
                        slot_eval<KIND, RS, NS, SHORT>(e1, rec1, xs0, xs1, xs2, (m >> s1) & 1u, rc2, a.xi, xi2,
                                                      exp_tab, coincident);
                        slot_eval<KIND, RS, NS, SHORT>(e2, rec2, xs0, xs1, xs2, (m >> s2) & 1u, rc2, a.xi, xi2,
                                                      exp_tab, coincident);
                        pair_apply<KIND, false>(e1.c, e1.r0, e1.r1, e1.r2, e1.sj, ua);
                        pair_apply<KIND, false>(e2.c, e2.r0, e2.r1, e2.r2, e2.sj, ua);
                        {
                            const double2 r01 = *reinterpret_cast<const double2*>(rec1 + RO);
                            double ub[3] = {r01.x, r01.y, rec1[RO + 2]};
                            pair_apply<KIND, true>(e1.c, e1.r0, e1.r1, e1.r2, fa, ub);
                            *reinterpret_cast<double2*>(rec1 + RO) = make_double2(ub[0], ub[1]);
                            rec1[RO + 2] = ub[2];
                        }
                        __syncwarp();
                        {
                            const double2 r01 = *reinterpret_cast<const double2*>(rec2 + RO);
                            double ub[3] = {r01.x, r01.y, rec2[RO + 2]};
                            pair_apply<KIND, true>(e2.c, e2.r0, e2.r1, e2.r2, fa, ub);
                            *reinterpret_cast<double2*>(rec2 + RO) = make_double2(ub[0], ub[1]);
                            rec2[RO + 2] = ub[2];
                        }
                        __syncwarp();
                        npairs32 += (e1.acc ? 2u : 0u) + (e2.acc ? 2u : 0u);
                    }
#endif
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
                            // (predicated stores: one instruction each on the rare path)
                            if (acc && n2 == 0.0) coincident = true;
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
                            Screened sc = screened<SHORT, SEWALD_EXP_REP>(n2e, a.xi, xi2, exp_tab);
                            sc.Ey = acc ? sc.Ey : 0.0;
#if defined(SEWALD_PROBE_NOREACT)  // timing probes only (wrong results)
                            {
                                const PairCoef<KIND> pc = pair_coef<KIND>(sc, xi2, n2e);
                                pair_apply<KIND, false>(pc, r0, r1, r2, sj, ua);
                            }
#elif defined(SEWALD_PROBE_WONLY)
                            double ub[3] = {0.0, 0.0, 0.0};
                            pair_both<KIND>(sc, xi2, n2e, r0, r1, r2, sj, fa, ua, ub);
                            *reinterpret_cast<double2*>(rec + RO) = make_double2(ub[0], ub[1]);
                            rec[RO + 2] = ub[2];
#else
                            const double2 r01 = *reinterpret_cast<const double2*>(rec + RO);
                            double ub[3] = {r01.x, r01.y, rec[RO + 2]};
                            pair_both<KIND>(sc, xi2, n2e, r0, r1, r2, sj, fa, ua, ub);
                            *reinterpret_cast<double2*>(rec + RO) = make_double2(ub[0], ub[1]);
                            rec[RO + 2] = ub[2];
#endif
                            if (acc) npairs32 += 2u;
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
                                    const Screened sc = screened<SHORT, SEWALD_EXP_REP>(n2, a.xi, xi2, exp_tab);
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
                    if (rotated && lane < cnt) {
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
#if SEWALD_SYM_POOL > 0
    __syncwarp();
    ua[0] += ipool[lane][0];
    ua[1] += ipool[lane][1];
    ua[2] += ipool[lane][2];
#endif
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
                          const int64_t* cell_off, int64_t c0, int64_t c1, int64_t cstride, double* u,
                          unsigned long long* pair_count, int* err, unsigned long long* work, cudaStream_t st) {
    if (c1 <= c0 || cstride < 1) return;
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
    const int64_t count = (c1 - c0 + cstride - 1) / cstride;
    const int64_t need = (count + SYM_WARPS - 1) / SYM_WARPS;
    const unsigned blocks = (unsigned)std::min<int64_t>(need, (int64_t)sms * std::max(per_sm, 1));
#define SEWALD_SYM_LAUNCH(K, S)                                                                            \
    if (shrt)                                                                                              \
        realspace_sym_kernel<K, S, true><<<blocks, SYM_THREADS, 0, st>>>(cg, a, packed, cell_off, N, c0, c1, cstride, u, \
                                                                          pair_count, err, work);          \
    else                                                                                                   \
        realspace_sym_kernel<K, S, false><<<blocks, SYM_THREADS, 0, st>>>(cg, a, packed, cell_off, N, c0, c1, cstride, u, \
                                                                           pair_count, err, work);
    switch (a.kind) {
        case SEWALD_STOKESLET: SEWALD_SYM_LAUNCH(SEWALD_STOKESLET, 8) break;
        case SEWALD_ROTLET: SEWALD_SYM_LAUNCH(SEWALD_ROTLET, 8) break;
        default: SEWALD_SYM_LAUNCH(SEWALD_STRESSLET, 12) break;
    }
#undef SEWALD_SYM_LAUNCH
}

}  // namespace sewald_b200
