// fp64 building blocks of the real-space (Hasimoto / Ewald screened) kernels,
// written for the B200 fp64 pipe instead of the general libdevice routines:
//
//   erfc(x) / r  and  (2 xi / sqrt(pi)) e^{-x^2},  x = xi r
//
// both share E = e^{-x^2}: erfc(x) = E * erfcx(x), and erfcx is smooth on
// [0, inf) so one branch-free rational P9/Q9 (tools/fit_erfcx.py, max rel.
// error 7e-16 on [0,10]) covers every pair; beyond x = 10 the product with
// E (< 4e-44) is negligible. exp uses a Cody-Waite reduction, a 2^(j/32)
// table and a degree-6 polynomial; 1/r and 1/Q start from the MUFU
// approximations and take one third-order correction step. Together ~45
// fp64 instructions per pair instead of ~600 for erfc() + exp() + sqrt() +
// two divisions from libdevice.
//
// Reference formulas: /root/reference/proj/src/kernels.cpp:71-116.
#pragma once

#include "erfcx_coeffs.h"
#include "exp2_table.h"

namespace sewald_b200 {

// Polynomial coefficients live in the constant bank so DFMA takes them as
// c[][] operands (as literals they are rebuilt with UMOVs on every use).
__constant__ double c_erfcx_p[10] = SEWALD_ERFCX_P;
__constant__ double c_erfcx_q[10] = SEWALD_ERFCX_Q;
__constant__ double c_erfcx8_p[9] = SEWALD_ERFCX8_P;
__constant__ double c_erfcx8_q[9] = SEWALD_ERFCX8_Q;

// The hot path evaluates the same rational and exponential in scaled form, so
// that no Horner chain starts from two constant operands (ptxas ran out of
// uniform registers for ~35 loop constants and reloaded 7 of them from the
// constant bank in every rotation step):
//   erfcx(x) = K P^(x) / Q^(x), P^ = P / p_n, Q^ = Q / q_n monic (K = p_n / q_n),
//   e^f = (f^6 + 6 f^5 + 30 f^4 + 120 f^3 + 360 f^2 + 720 f + 720) / 720
// (integer coefficients are instruction immediates). The factors K / 720 are
// folded into the 2^(j/32) table and 1/K into the Gaussian coefficient, so
// Screened carries Ey * K, R / K and cx / K: every kernel formula uses Ey
// times a linear combination of R and cx, which is unchanged.
namespace screened_detail {
constexpr double P9[10] = SEWALD_ERFCX_P, Q9[10] = SEWALD_ERFCX_Q;
constexpr double P8[9] = SEWALD_ERFCX8_P, Q8[9] = SEWALD_ERFCX8_Q;
constexpr double K9 = P9[9] / Q9[9], K8 = P8[8] / Q8[8];
}  // namespace screened_detail
#define SEWALD_MONIC8(A) {A[0] / A[8], A[1] / A[8], A[2] / A[8], A[3] / A[8], A[4] / A[8], A[5] / A[8], A[6] / A[8], A[7] / A[8]}
#define SEWALD_MONIC9(A) {A[0] / A[9], A[1] / A[9], A[2] / A[9], A[3] / A[9], A[4] / A[9], A[5] / A[9], A[6] / A[9], A[7] / A[9], A[8] / A[9]}
__constant__ double c_erfcx_pm[9] = SEWALD_MONIC9(screened_detail::P9);
__constant__ double c_erfcx_qm[9] = SEWALD_MONIC9(screened_detail::Q9);
__constant__ double c_erfcx8_pm[8] = SEWALD_MONIC8(screened_detail::P8);
__constant__ double c_erfcx8_qm[8] = SEWALD_MONIC8(screened_detail::Q8);
#undef SEWALD_MONIC8
#undef SEWALD_MONIC9
// [0]: P9/Q9 (x <= 10), [1]: P8/Q8 (SHORT): K, K / 720 (table scale), (2/sqrt(pi)) / K
__constant__ double c_rat_k[2] = {screened_detail::K9, screened_detail::K8};
__constant__ double c_tab_scale[2] = {screened_detail::K9 / 720.0, screened_detail::K8 / 720.0};
__constant__ double c_cx_k[2] = {1.12837916709551257390 / screened_detail::K9, 1.12837916709551257390 / screened_detail::K8};
// 2^(j/32), j < 32 (copied to shared memory by the kernels: per-lane index)
__constant__ double c_exp2_tab32[32] = SEWALD_EXP2_TAB32;
// e^f on |f| <= ln2/64: Taylor degree 6 (truncation < 4e-18)
__constant__ double c_exp6[7] = {1.0, 1.0, 0.5, 1.6666666666666666667e-01, 4.1666666666666666667e-02,
                                 8.3333333333333333333e-03, 1.3888888888888888889e-03};
__constant__ double c_exp_tab_k[3] = {SEWALD_INV_LN2_32, -SEWALD_LN2_32_HI, -SEWALD_LN2_32_LO};
__constant__ double c_exp_poly[14] = {
    1.0, 1.0, 0.5, 1.6666666666666666667e-01, 4.1666666666666666667e-02, 8.3333333333333333333e-03,
    1.3888888888888888889e-03, 1.9841269841269841270e-04, 2.4801587301587301587e-05,
    2.7557319223985890653e-06, 2.7557319223985890653e-07, 2.5052108385441718775e-08,
    2.0876756987868098979e-09, 1.6059043836821614599e-10};

// exp reduction constants: shifter (1.5 * 2^52), log2(e), -ln2 hi/lo, 2/sqrt(pi)
__constant__ double c_misc[5] = {6755399441055744.0, 1.4426950408889634074, -6.93147180559945286227e-01,
                                 -2.31904681384629955842e-17, 1.12837916709551257390};

__device__ __forceinline__ double rcp_approx(double a) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
    return r;
}

__device__ __forceinline__ double rsqrt_approx(double a) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
    return r;
}

// 1/sqrt(a), a > 0 normal: MUFU seed y0 = (1 + d)/sqrt(a), |d| < 2^-22, and
// one third-order step y0 (1 + e/2 + 3e^2/8), e = 1 - a y0^2 (truncation
// 2.5 d^3 < 2^-64): 5 fp64 ops instead of 8 for two Newton steps.
__device__ __forceinline__ double rsqrt_nr(double a) {
    const double y = rsqrt_approx(a);
    const double e = fma(-a * y, y, 1.0);
    return fma(y * e, fma(0.375, e, 0.5), y);
}

// e^{-y} for y >= 0 (clamped at 708 where the result is < 1e-307).
__device__ __forceinline__ double exp_neg(double y) {
    y = fmin(y, 708.0);
    const double shifter = c_misc[0];
    const double t = fma(-y, c_misc[1], shifter);
    const int n = __double2loint(t);
    const double dn = t - shifter;
    double f = fma(dn, c_misc[2], -y);
    f = fma(dn, c_misc[3], f);
    double p = c_exp_poly[13];
#pragma unroll
    for (int i = 12; i >= 0; --i) p = fma(p, f, c_exp_poly[i]);
    return p * __hiloint2double((n + 1023) << 20, 0);
}

// Entry j of the shared-memory exponential table used by screened<SHORT>:
// 2^(j/32) * K / 720 (see above).
template <bool SHORT>
__device__ __forceinline__ double exp_tab_entry(int j) {
    return c_exp2_tab32[j] * c_tab_scale[SHORT ? 1 : 0];
}

// e^{-y} * K for y >= 0 via the scaled 2^(j/32) table (tab: exp_tab_entry
// values) and the monic degree-6 polynomial: 9 fp64 FMAs instead of 16.
// STRIDE > 1: the table is replicated STRIDE times, interleaved, and `tab`
// points at the calling lane's copy (lane % STRIDE), so a warp's random
// indices fall in distinct shared-memory banks.
template <bool CLAMP = true, int STRIDE = 1>
__device__ __forceinline__ double exp_neg_tab(double y, const double* tab) {
    // callers that guarantee y <= 49 (x <= 7, the SHORT real-space kernels) skip the
    // clamp; 600 keeps K e^{-y} (|K| >= 1.6e-10) normal for the exponent-field scaling
    if (CLAMP) y = fmin(y, 600.0);
    const double shifter = c_misc[0];
    const double t = fma(-y, c_exp_tab_k[0], shifter);
    const int n = __double2loint(t);
    const double dn = t - shifter;
    double f = fma(dn, c_exp_tab_k[1], -y);
    f = fma(dn, c_exp_tab_k[2], f);
    double p = f + 6.0;
    p = fma(p, f, 30.0);
    p = fma(p, f, 120.0);
    p = fma(p, f, 360.0);
    p = fma(p, f, 720.0);
    p = fma(p, f, 720.0);
    const int m = n >> 5;  // n = 32 m + j, n <= 0
    // scale by 2^m in the exponent field (y <= 600 keeps the result normal)
    const double v = p * tab[(n & 31) * STRIDE];
    return __hiloint2double(__double2hiint(v) + (m << 20), __double2loint(v));
}

// p/q = p y0 (1 + e + e^2), e = 1 - q y0, y0 = MUFU 1/q (|e| < 2^-22)
__device__ __forceinline__ double div_rat(double p, double q) {
    const double y = rcp_approx(q);
    const double e = fma(-q, y, 1.0);
    const double r = p * y;
    return fma(r, fma(e, e, e), r);
}

// erfcx(x) = e^{x^2} erfc(x) for x >= 0: rational P9/Q9 on [0,10], or the
// shorter P8/Q8 valid on [0,7] (SHORT, when xi * rc <= 7).
template <bool SHORT = false>
__device__ __forceinline__ double erfcx_rat(double x) {
    double p, q;
    if (SHORT) {
        p = c_erfcx8_p[8];
        q = c_erfcx8_q[8];
#pragma unroll
        for (int i = 7; i >= 0; --i) {
            p = fma(p, x, c_erfcx8_p[i]);
            q = fma(q, x, c_erfcx8_q[i]);
        }
    } else {
        p = c_erfcx_p[9];
        q = c_erfcx_q[9];
#pragma unroll
        for (int i = 8; i >= 0; --i) {
            p = fma(p, x, c_erfcx_p[i]);
            q = fma(q, x, c_erfcx_q[i]);
        }
    }
    return div_rat(p, q);
}

// erfcx(x) / K from the monic polynomials (scaled form, see above)
template <bool SHORT = false>
__device__ __forceinline__ double erfcx_rat_monic(double x) {
    double p, q;
    if (SHORT) {
        p = x + c_erfcx8_pm[7];
        q = x + c_erfcx8_qm[7];
#pragma unroll
        for (int i = 6; i >= 0; --i) {
            p = fma(p, x, c_erfcx8_pm[i]);
            q = fma(q, x, c_erfcx8_qm[i]);
        }
    } else {
        p = x + c_erfcx_pm[8];
        q = x + c_erfcx_qm[8];
#pragma unroll
        for (int i = 7; i >= 0; --i) {
            p = fma(p, x, c_erfcx_pm[i]);
            q = fma(q, x, c_erfcx_qm[i]);
        }
    }
    return div_rat(p, q);
}

// Shared screened factors for one pair at squared distance n2:
//   iy   = 1/r
//   Ey   = K e^{-x^2} / r
//   R    = erfcx(x) / K, cx = (2/sqrt(pi)) x / K
// so that erfc(x)/r = Ey R and the Gaussian term g = (2 xi/sqrt(pi)) e^{-x^2} = Ey cx
// (K: the scale of the monic erfcx rational, see above; E = K e^{-x^2}).
struct Screened {
    double iy, Ey, R, cx, E;
};

template <bool SHORT = false, int STRIDE = 1>
__device__ __forceinline__ Screened screened(double n2, double xi, double xi2, const double* exp_tab = nullptr) {
    Screened s;
    s.iy = rsqrt_nr(n2);
    const double r = n2 * s.iy;
    const double x = xi * r;
#ifdef SEWALD_PROBE_NOEXP  // timing probe builds only (wrong results)
    s.E = 1.0 / (1.0 + 0.0 * n2);
#else
    s.E = exp_tab ? exp_neg_tab<!SHORT, STRIDE>(xi2 * n2, exp_tab) : exp_neg(xi2 * n2) * c_rat_k[SHORT ? 1 : 0];
#endif
    s.Ey = s.E * s.iy;
#ifdef SEWALD_PROBE_NOERFCX
    s.R = x;
#else
    s.R = erfcx_rat_monic<SHORT>(x);
#endif
    s.cx = c_cx_k[SHORT ? 1 : 0] * x;
    return s;
}

}  // namespace sewald_b200
