// k-space scaling: multiply each retained mode by the screened, window-
// deconvolved Green's function and contract the strength components.
//
// Reference: scale       /root/reference/proj/src/fourier.cpp:522-666
//            apply_mode  /root/reference/proj/src/fourier.cpp:190-216
//            diffop_hat  /root/reference/proj/src/kernels.cpp:118-149
//            plain_kernel_hat / modified_kernel_hat
//                        /root/reference/proj/src/modified_kernels.cpp:162-167, :248-270
//            screening   /root/reference/proj/src/kernels.cpp:65-69
//
// The reference transforms real data with complex-to-complex FFTs and keeps
// the real part of the inverse (fourier.cpp:336, :434). Here the fully
// periodic path uses R2C/C2R (half the bytes). Taking the real part is the
// same as applying the Hermitian part of the operator,
//     H(m) = 1/2 [G(k(m)) + conj G(k(-m))],
// and since the Nyquist index maps to -pi/h on both m and -m, k(-m) = -k~
// where k~ flips the Nyquist components of k(m). With G(-k) = conj G(k) this
// is H(m) = 1/2 [G(k) + G(k~)], evaluated below on the Nyquist planes only.
// Normalisation: h^3 before the forward and 1/(h^3 vol) after the inverse
// fold into one factor 1/vol applied here.
#include "device_common.cuh"
#include "sg_kernels.h"
#include "../../include/sewald_gpu.h"

#include <cuComplex.h>

namespace sewald_b200 {

namespace {

constexpr double kPiD = 3.14159265358979323846;

// Real coefficients g of G = g (stokeslet, real) or G = i g (rotlet,
// stresslet), including the k-space base kernel A(k) (Hasimoto -8 pi/k^4,
// Ewald 4 pi/k^2). Rank 2: g[3][3]; rank 3: g[3][9] with (l,m) -> 3l+m.
template <int KIND>
__device__ __forceinline__ void operator_coeffs(double k0, double k1, double k2, double* g) {
    const double kk = k0 * k0 + k1 * k1 + k2 * k2;
    const double kv[3] = {k0, k1, k2};
    if (KIND == SEWALD_STOKESLET) {
        const double base = -8.0 * kPiD / (kk * kk);
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int l = 0; l < 3; ++l) g[3 * j + l] = ((j == l ? -kk : 0.0) + kv[j] * kv[l]) * base;
    } else if (KIND == SEWALD_ROTLET) {
        const double base = 4.0 * kPiD / kk;
        // diffop = -i eps_jlm k_m: coefficient of i is -(eps_jlm k_m)
        g[0] = 0.0;            g[1] = -k2 * base;      g[2] = k1 * base;
        g[3] = k2 * base;      g[4] = 0.0;             g[5] = -k0 * base;
        g[6] = -k1 * base;     g[7] = k0 * base;       g[8] = 0.0;
    } else {
        const double base = -8.0 * kPiD / (kk * kk);
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int l = 0; l < 3; ++l)
#pragma unroll
                for (int m = 0; m < 3; ++m) {
                    const double deltas = (j == l ? kv[m] : 0.0) + (m == j ? kv[l] : 0.0) +
                                          (l == m ? kv[j] : 0.0);
                    g[9 * j + 3 * l + m] = (-deltas * kk + 2.0 * kv[j] * kv[l] * kv[m]) * base;
                }
    }
}

template <int KIND>
__global__ void scale_periodic_kernel(int n0, int n1, int n2, double xi, double norm, KspaceTables t,
                                      cuDoubleComplex* __restrict__ data, int64_t cstride) {
    constexpr int NC = KIND == SEWALD_STRESSLET ? 9 : 3;  // input components
    constexpr int NG = 3 * NC;
    const int nh = n2 / 2 + 1;
    const int64_t nmodes = (int64_t)n0 * n1 * nh;
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= nmodes) return;
    const int m = (int)(idx % nh);
    const int64_t ij = idx / nh;
    const int j = (int)(ij % n1);
    const int i = (int)(ij / n1);

    const double k0 = t.k[0][i], k1 = t.k[1][j], k2 = t.k[2][m];
    const double kk = k0 * k0 + k1 * k1 + k2 * k2;
    if (kk == 0.0) {  // G(0) = 0 for d = 3 (modified_kernels.cpp:250-252)
#pragma unroll
        for (int c = 0; c < 3; ++c) data[c * cstride + idx] = make_cuDoubleComplex(0.0, 0.0);
        return;
    }
    const double wp = t.what[0][i] * t.what[1][j] * t.what[2][m];
    const double q = kk / (4.0 * xi * xi);
    const double gscr = exp(-q);
    const double scr = KIND == SEWALD_ROTLET ? gscr : gscr * (1.0 + q);
    const double fac = scr / (wp * wp) * norm;

    double g[NG];
    operator_coeffs<KIND>(k0, k1, k2, g);
    const bool ny0 = (n0 % 2 == 0) && (i == n0 / 2);
    const bool ny1 = (n1 % 2 == 0) && (j == n1 / 2);
    const bool ny2 = (n2 % 2 == 0) && (m == n2 / 2);
    if (ny0 || ny1 || ny2) {
        double gt[NG];
        operator_coeffs<KIND>(ny0 ? -k0 : k0, ny1 ? -k1 : k1, ny2 ? -k2 : k2, gt);
#pragma unroll
        for (int e = 0; e < NG; ++e) g[e] = 0.5 * (g[e] + gt[e]);
    }

    cuDoubleComplex in[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) in[c] = data[c * cstride + idx];
#pragma unroll
    for (int jj = 0; jj < 3; ++jj) {
        double re = 0.0, im = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            re += g[NC * jj + c] * in[c].x;
            im += g[NC * jj + c] * in[c].y;
        }
        if (KIND == SEWALD_STOKESLET)
            data[jj * cstride + idx] = make_cuDoubleComplex(fac * re, fac * im);
        else  // i * (re + i im) = -im + i re
            data[jj * cstride + idx] = make_cuDoubleComplex(-fac * im, fac * re);
    }
}

}  // namespace

void launch_scale_periodic(int kind, int n0, int n1, int n2, double xi, double norm,
                           const KspaceTables& t, cuDoubleComplex* data, int64_t cstride,
                           cudaStream_t st) {
    const int64_t nmodes = (int64_t)n0 * n1 * (n2 / 2 + 1);
    const unsigned blocks = (unsigned)((nmodes + 255) / 256);
    switch (kind) {
        case SEWALD_STOKESLET:
            scale_periodic_kernel<SEWALD_STOKESLET><<<blocks, 256, 0, st>>>(n0, n1, n2, xi, norm, t, data, cstride);
            break;
        case SEWALD_ROTLET:
            scale_periodic_kernel<SEWALD_ROTLET><<<blocks, 256, 0, st>>>(n0, n1, n2, xi, norm, t, data, cstride);
            break;
        default:
            scale_periodic_kernel<SEWALD_STRESSLET><<<blocks, 256, 0, st>>>(n0, n1, n2, xi, norm, t, data, cstride);
            break;
    }
}

}  // namespace sewald_b200
