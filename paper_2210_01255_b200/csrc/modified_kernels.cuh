// Device restatement of the k-space kernels with the k = 0 singularity
// regularised for free directions (truncated "modified" kernels):
//
//   modified_kernel_hat   /root/reference/proj/src/modified_kernels.cpp:248-270
//   modified_1p_branch    :175-217   (d = 1, k_0 = 0: J0/J1-based H and B)
//   modified_2p_branch    :219-244   (d = 2, k_0 = k_1 = 0: H2p, Z)
//   *_hat_trunc_0p/1p/2p  :74-145
//   plain_kernel_hat      :162-167, diffop_hat kernels.cpp:118-149
//   screening_hat         kernels.cpp:65-69
//
// The power-series coefficients used below |R kappa| < 1 depend only on the
// gauge constants; they are assembled on the host exactly as the reference
// does (modified_kernels.cpp:22-36, :85-94, :104-108, :117-124) and passed
// in ModSpec.
#pragma once

#include <cuComplex.h>

#include <cmath>

// Host and device: the same restatement also backs the host modified_kernel_hat
// of the drop-in API (host_api.cu), so both sides share one implementation.
#define SEWALD_HD __host__ __device__ __forceinline__

namespace sewald_b200 {

constexpr int kSeries = 13;

struct ModSpec {
    int kind;     // SEWALD_STOKESLET / STRESSLET / ROTLET
    int d;        // 0, 1, 2, 3
    double R, a_B, b_B, ell_H, ell_B, c_B;
    double g_h1, g_b1, ch_b1;          // log(R/ell_H), log(R/ell_B), (c_B - R^2 g_b1)/R^2
    double bR3, p0, q0;                // 0P biharmonic constants
    double ser_b0[kSeries];            // 0P biharmonic series (n >= 2)
    double ser_h1[kSeries];            // 1P harmonic series (n >= 1)
    double ser_b1[kSeries];            // 1P biharmonic series (n >= 2)
};

constexpr double kPiM = 3.14159265358979323846;

SEWALD_HD double series_eval(const double* c, int first, int count, double x2) {
    double acc = 0.0;
    for (int n = first + count - 1; n >= first; --n) acc = c[n] + acc * x2;
    return acc;
}

SEWALD_HD double harmonic_trunc_0p(double kappa, double R) {
    if (kappa == 0.0) return 2.0 * kPiM * R * R;
    const double s = sin(0.5 * R * kappa);
    return 8.0 * kPiM * s * s / (kappa * kappa);
}

SEWALD_HD double biharmonic_trunc_0p(const ModSpec& m, double kappa) {
    const double x = m.R * kappa;
    if (fabs(x) < 1.0) {
        const double R2 = m.R * m.R;
        return -8.0 * kPiM * R2 * R2 * series_eval(m.ser_b0, 2, kSeries - 2, x * x);
    }
    const double bracket = 1.0 - (1.0 + m.bR3 - m.p0 * x * x) * cos(x) + (m.bR3 - m.q0 * x * x) * sin(x) / x;
    const double k2 = kappa * kappa;
    return -8.0 * kPiM / (k2 * k2) * bracket;
}

SEWALD_HD double harmonic_trunc_1p(const ModSpec& m, double kappa) {
    const double x = m.R * kappa;
    if (fabs(x) < 1.0) return 4.0 * kPiM * m.R * m.R * series_eval(m.ser_h1, 1, kSeries - 1, x * x);
    const double bracket = 1.0 - j0(x) - m.g_h1 * x * j1(x);
    return 4.0 * kPiM / (kappa * kappa) * bracket;
}

SEWALD_HD double biharmonic_trunc_1p(const ModSpec& m, double kappa) {
    const double x = m.R * kappa;
    if (fabs(x) < 1.0) {
        const double R2 = m.R * m.R;
        return -8.0 * kPiM * R2 * R2 * series_eval(m.ser_b1, 2, kSeries - 2, x * x);
    }
    const double J0 = j0(x), J1 = j1(x);
    const double g = m.g_b1;
    const double bracket = 1.0 - J0 - x * (1.0 + g) * J1 + 0.25 * x * x * (1.0 + 2.0 * g) * J0 -
                           0.25 * x * x * x * m.ch_b1 * J1;
    const double k2 = kappa * kappa;
    return -8.0 * kPiM / (k2 * k2) * bracket;
}

SEWALD_HD double Z_trunc_2p_im(double k3, double R) {
    if (k3 == 0.0) return 0.0;
    const double s = sin(0.5 * R * k3);
    return -8.0 * kPiM * s * s / k3;
}

SEWALD_HD double H2p_trunc(double k3, double R) {
    if (k3 == 0.0) return -2.0 * kPiM * R * R;
    const double x = R * k3;
    const double s = sin(0.5 * x);
    const double bracket = 2.0 * s * s - x * sin(x);
    return 4.0 * kPiM / (k3 * k3) * bracket;
}

// Kernel tensor G(k) = re + i im, rank 2 (9 entries, [3j+l]) or rank 3
// (27 entries, [9j+3l+m]). diffop only (the scalar factor is applied by
// the caller): stokeslet real, rotlet / stresslet purely imaginary.
template <int KIND>
SEWALD_HD void diffop_coeffs(double k0, double k1, double k2, double* re, double* im) {
    const double kk = k0 * k0 + k1 * k1 + k2 * k2;
    const double kv[3] = {k0, k1, k2};
    if (KIND == SEWALD_STOKESLET) {
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int l = 0; l < 3; ++l) {
                re[3 * j + l] = (j == l ? -kk : 0.0) + kv[j] * kv[l];
                im[3 * j + l] = 0.0;
            }
    } else if (KIND == SEWALD_ROTLET) {
        const double e[9] = {0.0, k2, -k1, -k2, 0.0, k0, k1, -k0, 0.0};  // eps_jlm k_m
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            re[q] = 0.0;
            im[q] = -e[q];
        }
    } else {
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int l = 0; l < 3; ++l)
#pragma unroll
                for (int m = 0; m < 3; ++m) {
                    const double deltas = (j == l ? kv[m] : 0.0) + (m == j ? kv[l] : 0.0) + (l == m ? kv[j] : 0.0);
                    re[9 * j + 3 * l + m] = 0.0;
                    im[9 * j + 3 * l + m] = -deltas * kk + 2.0 * kv[j] * kv[l] * kv[m];
                }
    }
}

// modified_kernel_hat(spec, k) for d in {0,1,2,3} (the d = 3 solve itself uses kspace.cu).
template <int KIND>
SEWALD_HD void modified_coeffs(const ModSpec& m, double k0, double k1, double k2,
                                                double* re, double* im) {
    constexpr int NG = KIND == SEWALD_STRESSLET ? 27 : 9;
    const bool plain = (m.d == 2 && (k0 != 0.0 || k1 != 0.0)) || (m.d == 1 && k0 != 0.0) || m.d == 3;
    if (plain || m.d == 0) {
        const double kk = k0 * k0 + k1 * k1 + k2 * k2;
        if ((m.d == 0 || m.d == 3) && kk == 0.0) {  // d = 3: G(0) = 0 (modified_kernels.cpp:250-252)
#pragma unroll
            for (int q = 0; q < NG; ++q) re[q] = im[q] = 0.0;
            return;
        }
        double base;
        if (m.d == 0) {
            const double kappa = sqrt(kk);
            base = KIND == SEWALD_ROTLET ? harmonic_trunc_0p(kappa, m.R) : biharmonic_trunc_0p(m, kappa);
        } else {
            base = KIND == SEWALD_ROTLET ? 4.0 * kPiM / kk : -8.0 * kPiM / (kk * kk);
        }
        diffop_coeffs<KIND>(k0, k1, k2, re, im);
#pragma unroll
        for (int q = 0; q < NG; ++q) {
            re[q] *= base;
            im[q] *= base;
        }
        return;
    }
#pragma unroll
    for (int q = 0; q < NG; ++q) re[q] = im[q] = 0.0;
    if (m.d == 2) {  // k0 = k1 = 0 (modified_2p_branch)
        if (KIND == SEWALD_STOKESLET) {
            const double H = H2p_trunc(k2, m.R);
            re[0] = 2.0 * H;
            re[4] = 2.0 * H;
        } else if (KIND == SEWALD_ROTLET) {
            const double Z = Z_trunc_2p_im(k2, m.R);
            im[1] = Z;
            im[3] = -Z;
        } else {
            const double m2 = -2.0 * Z_trunc_2p_im(k2, m.R);
            // t[0][0][2], t[0][2][0], t[1][1][2], t[1][2][1], t[2][0][0], t[2][1][1], t[2][2][2]
            im[2] = im[6] = m2;
            im[9 + 3 + 2] = im[9 + 6 + 1] = m2;
            im[18 + 0] = im[18 + 4] = im[18 + 8] = m2;
        }
        return;
    }
    // d = 1, k0 = 0 (modified_1p_branch) with (k2, k3) -> (k1, k2) here
    const double kappa = sqrt(k1 * k1 + k2 * k2);
    const double H = harmonic_trunc_1p(m, kappa);
    if (KIND == SEWALD_ROTLET) {
        diffop_coeffs<KIND>(0.0, k1, k2, re, im);
#pragma unroll
        for (int q = 0; q < 9; ++q) im[q] *= H;
        return;
    }
    const double B = biharmonic_trunc_1p(m, kappa);
    if (KIND == SEWALD_STOKESLET) {
        re[0] = 2.0 * H;
        re[4] = -k2 * k2 * B;
        re[5] = k1 * k2 * B;
        re[7] = k1 * k2 * B;
        re[8] = -k1 * k1 * B;
        return;
    }
    // stresslet: cth (H part) and ctb (B part), modified_kernels.cpp:464-484
    const double kk = kappa * kappa;
    double cth[27], ctb[27];
#pragma unroll
    for (int q = 0; q < 27; ++q) cth[q] = ctb[q] = 0.0;
    cth[0 * 9 + 0 * 3 + 1] = cth[0 * 9 + 1 * 3 + 0] = k1;
    cth[0 * 9 + 0 * 3 + 2] = cth[0 * 9 + 2 * 3 + 0] = k2;
    cth[1 * 9 + 0 * 3 + 0] = k1;
    cth[2 * 9 + 0 * 3 + 0] = k2;
    ctb[1 * 9 + 1 * 3 + 1] = k1 * (3.0 * kk - 2.0 * k1 * k1);
    ctb[1 * 9 + 1 * 3 + 2] = ctb[1 * 9 + 2 * 3 + 1] = k2 * (kk - 2.0 * k1 * k1);
    ctb[1 * 9 + 2 * 3 + 2] = k1 * (kk - 2.0 * k2 * k2);
    ctb[2 * 9 + 1 * 3 + 1] = k2 * (kk - 2.0 * k1 * k1);
    ctb[2 * 9 + 1 * 3 + 2] = ctb[2 * 9 + 2 * 3 + 1] = k1 * (kk - 2.0 * k2 * k2);
    ctb[2 * 9 + 2 * 3 + 2] = k2 * (3.0 * kk - 2.0 * k2 * k2);
#pragma unroll
    for (int q = 0; q < 27; ++q) im[q] = 2.0 * cth[q] * H - ctb[q] * B;
}

// ModifiedKernelSpec fields (any gauge) -> ModSpec with the series blocks
// (aft.cu), and the optimal gauge (modified_kernels.cpp:52-63).
ModSpec make_modspec_full(int kind, int d, double R, double a_B, double b_B, double ell_H, double ell_B,
                          double c_B);
ModSpec make_modspec(int kind, int d, double R);

}  // namespace sewald_b200
