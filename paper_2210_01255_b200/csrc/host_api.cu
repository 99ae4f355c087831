// Host evaluation layer of the drop-in API (include/sewald/sewald_b200.hpp):
// kernel tensors, screening, the truncated (modified) kernels, the gauge
// correction, the stresslet mean-flow term and the real-space cell list, for
// callers and for the reference's own unit tests compiled against this
// library. None of it is on the measured path (the device kernels evaluate
// the same formulas inline); the modified kernels share their implementation
// with the device through modified_kernels.cuh (__host__ __device__).
//
// Reference formulas:
//   bare_kernel / realspace_kernel   kernels.cpp:27-116
//   screening_hat                    kernels.cpp:65-69
//   diffop_hat / fourier_kernel_hat  kernels.cpp:118-167
//   self_term / stresslet_zero_mode  kernels.cpp:169-187
//   apply                            kernels.cpp:189-221
//   *_hat_trunc_*, modified_kernel_hat, gauge_flow_correction
//                                    modified_kernels.cpp:65-281
//   build_cell_list                  realspace.cpp:16-20, :97-164
#include "../../include/sewald/sewald_b200.hpp"
#include "../../include/sewald_gpu.h"
#include "modified_kernels.cuh"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>
#include <string>

namespace sewald {

namespace {

constexpr double kPiH = 3.14159265358979323846;
constexpr double kTwoOverSqrtPi = 1.1283791670955125739;

// eps_{jlm} v_m for fixed (j, l)
double cross_entry(int j, int l, const Vec3& v) {
    if (j == l) return 0.0;
    const int m = 3 - j - l;
    const double sign = ((l - j + 3) % 3 == 1) ? 1.0 : -1.0;  // (j, l, m) cyclic -> +1
    return sign * v[m];
}

void nonzero_or_throw(const Vec3& r, const char* what) {
    if (r[0] == 0.0 && r[1] == 0.0 && r[2] == 0.0)
        throw std::domain_error(std::string(what) + " is singular at the origin");
}

int kid(Kernel k) {
    return k == Kernel::stokeslet ? SEWALD_STOKESLET : (k == Kernel::stresslet ? SEWALD_STRESSLET : SEWALD_ROTLET);
}

sewald_b200::ModSpec modspec(const ModifiedKernelSpec& s) {
    return sewald_b200::make_modspec_full(kid(s.kind), s.d, s.R, s.a_B, s.b_B, s.ell_H, s.ell_B, s.c_B);
}

template <int KIND>
KernelTensor modified_tensor(const sewald_b200::ModSpec& m, const Vec3& k) {
    constexpr int NG = KIND == SEWALD_STRESSLET ? 27 : 9;
    double re[NG], im[NG];
    sewald_b200::modified_coeffs<KIND>(m, k[0], k[1], k[2], re, im);
    KernelTensor out;
    out.rank = KIND == SEWALD_STRESSLET ? 3 : 2;
    for (int q = 0; q < NG; ++q) {
        const cplx v(re[q], im[q]);
        if (NG == 9)
            out.m[q / 3][q % 3] = v;
        else
            out.t[q / 9][(q / 3) % 3][q % 3] = v;
    }
    return out;
}

}  // namespace

// ---- kernels.h ------------------------------------------------------------------
KernelTensorR bare_kernel(Kernel kind, const Vec3& r) {
    nonzero_or_throw(r, "bare kernel");
    const double r2 = norm2(r), rn = std::sqrt(r2);
    KernelTensorR K;
    if (kind == Kernel::stresslet) {
        K.rank = 3;
        const double c = -6.0 / (r2 * r2 * rn);
        for (int j = 0; j < 3; ++j)
            for (int l = 0; l < 3; ++l)
                for (int m = 0; m < 3; ++m) K.t[j][l][m] = c * r[j] * r[l] * r[m];
        return K;
    }
    K.rank = 2;
    for (int j = 0; j < 3; ++j)
        for (int l = 0; l < 3; ++l)
            K.m[j][l] = kind == Kernel::stokeslet ? (j == l ? 1.0 / rn : 0.0) + r[j] * r[l] / (r2 * rn)
                                                  : cross_entry(j, l, r) / (r2 * rn);
    return K;
}

double screening_hat(Screening skind, const Vec3& k, double xi) {
    const double q = norm2(k) / (4.0 * xi * xi);
    const double e = std::exp(-q);
    return skind == Screening::ewald ? e : e * (1.0 + q);
}

KernelTensorR realspace_kernel(Kernel kind, const Vec3& r, double xi) {
    nonzero_or_throw(r, "real-space kernel");
    const double r2 = norm2(r), rn = std::sqrt(r2);
    const double x = xi * rn;
    const double erfc_r = std::erfc(x) / rn;
    const double g = kTwoOverSqrtPi * xi * std::exp(-x * x);
    KernelTensorR K;
    if (kind == Kernel::stresslet) {
        K.rank = 3;
        const double a = -2.0 / (r2 * r2) * (3.0 * erfc_r + (3.0 + 2.0 * x * x) * g);
        const double b = 2.0 * xi * xi * g;
        for (int j = 0; j < 3; ++j)
            for (int l = 0; l < 3; ++l)
                for (int m = 0; m < 3; ++m) {
                    const double d = (j == l ? r[m] : 0.0) + (m == j ? r[l] : 0.0) + (l == m ? r[j] : 0.0);
                    K.t[j][l][m] = a * r[j] * r[l] * r[m] + b * d;
                }
        return K;
    }
    K.rank = 2;
    const double s = erfc_r + g;
    for (int j = 0; j < 3; ++j)
        for (int l = 0; l < 3; ++l) {
            if (kind == Kernel::stokeslet) {
                const double delta = j == l ? 1.0 : 0.0;
                K.m[j][l] = (delta + r[j] * r[l] / r2) * s - 2.0 * g * delta;
            } else {
                K.m[j][l] = cross_entry(j, l, r) * (s / r2);
            }
        }
    return K;
}

KernelTensor diffop_hat(Kernel kind, const Vec3& k) {
    KernelTensor K;
    const double kk = norm2(k);
    if (kind == Kernel::stresslet) {
        K.rank = 3;
        for (int j = 0; j < 3; ++j)
            for (int l = 0; l < 3; ++l)
                for (int m = 0; m < 3; ++m) {
                    const double d = (j == l ? k[m] : 0.0) + (m == j ? k[l] : 0.0) + (l == m ? k[j] : 0.0);
                    K.t[j][l][m] = cplx(0.0, 2.0 * k[j] * k[l] * k[m] - d * kk);
                }
        return K;
    }
    K.rank = 2;
    for (int j = 0; j < 3; ++j)
        for (int l = 0; l < 3; ++l)
            K.m[j][l] = kind == Kernel::stokeslet ? cplx(k[j] * k[l] - (j == l ? kk : 0.0), 0.0)
                                                  : cplx(0.0, -cross_entry(j, l, k));
    return K;
}

KernelTensor fourier_kernel_hat(Kernel kind, const Vec3& k, double xi) {
    const double kk = norm2(k);
    if (kk == 0.0) throw std::domain_error("long-range kernel is singular at k=0");
    const Screening sc = screening_of(kind);
    const double base = sc == Screening::ewald ? 4.0 * kPiH / kk : -8.0 * kPiH / (kk * kk);
    const double f = base * screening_hat(sc, k, xi);
    KernelTensor K = diffop_hat(kind, k);
    for (auto& row : K.m)
        for (auto& v : row) v *= f;
    for (auto& mat : K.t)
        for (auto& row : mat)
            for (auto& v : row) v *= f;
    return K;
}

Vec3 self_term(Kernel kind, double xi, const Vec3& strength) {
    if (kind != Kernel::stokeslet) return {0.0, 0.0, 0.0};
    return (-2.0 * kTwoOverSqrtPi * xi) * strength;
}

std::vector<Vec3> stresslet_zero_mode_3p(const TargetSet& targets, const SourceSystem& system) {
    // u(x) = -(8 pi / V) [x sum_n c_n - sum_n c_n x_n],  c_n = q_n . nu_n
    double c_sum = 0.0;
    Vec3 cx{0.0, 0.0, 0.0};
    for (std::size_t n = 0; n < system.size(); ++n) {
        const double c = dot(system.f[n], system.nu[n]);
        c_sum += c;
        cx += c * system.x[n];
    }
    const double pref = -8.0 * kPiH / system.cell.volume();
    std::vector<Vec3> u;
    u.reserve(targets.x.size());
    for (const Vec3& xm : targets.x) u.push_back(pref * (c_sum * xm - cx));
    return u;
}

Vec3 apply(const KernelTensorR& K, const Vec3& f) {
    Vec3 u{0.0, 0.0, 0.0};
    for (int j = 0; j < 3; ++j)
        for (int l = 0; l < 3; ++l) u[j] += K.m[j][l] * f[l];
    return u;
}

Vec3 apply(const KernelTensorR& K, const Vec3& q, const Vec3& nu) {
    Vec3 u{0.0, 0.0, 0.0};
    for (int j = 0; j < 3; ++j)
        for (int l = 0; l < 3; ++l)
            for (int m = 0; m < 3; ++m) u[j] += K.t[j][l][m] * q[l] * nu[m];
    return u;
}

CVec3 apply(const KernelTensor& K, const Vec3& f) {
    CVec3 u{};
    for (int j = 0; j < 3; ++j)
        for (int l = 0; l < 3; ++l) u[j] += K.m[j][l] * f[l];
    return u;
}

CVec3 apply(const KernelTensor& K, const Vec3& q, const Vec3& nu) {
    CVec3 u{};
    for (int j = 0; j < 3; ++j)
        for (int l = 0; l < 3; ++l)
            for (int m = 0; m < 3; ++m) u[j] += K.t[j][l][m] * (q[l] * nu[m]);
    return u;
}

// ---- modified_kernels.h ----------------------------------------------------------
double harmonic_hat_trunc_0p(double kappa, double R) { return sewald_b200::harmonic_trunc_0p(kappa, R); }

double biharmonic_hat_trunc_0p(double kappa, double R, double a_B, double b_B) {
    const sewald_b200::ModSpec m = sewald_b200::make_modspec_full(SEWALD_STOKESLET, 0, R, a_B, b_B, R, R, 0.0);
    return sewald_b200::biharmonic_trunc_0p(m, kappa);
}

double harmonic_hat_trunc_1p(double kappa, double R, double ell_H) {
    const sewald_b200::ModSpec m = sewald_b200::make_modspec_full(SEWALD_ROTLET, 1, R, 0.0, 0.0, ell_H, R, 0.0);
    return sewald_b200::harmonic_trunc_1p(m, kappa);
}

double biharmonic_hat_trunc_1p(double kappa, double R, double ell_B, double c_B) {
    const sewald_b200::ModSpec m = sewald_b200::make_modspec_full(SEWALD_STOKESLET, 1, R, 0.0, 0.0, R, ell_B, c_B);
    return sewald_b200::biharmonic_trunc_1p(m, kappa);
}

cplx Z_hat_trunc_2p(double kappa3, double R) { return cplx(0.0, sewald_b200::Z_trunc_2p_im(kappa3, R)); }

double H2p_hat_trunc(double kappa3, double R) { return sewald_b200::H2p_trunc(kappa3, R); }

KernelTensor modified_kernel_hat(const ModifiedKernelSpec& spec, const Vec3& k) {
    if (spec.d < 0 || spec.d > 3) throw std::invalid_argument("periodicity must be in 0..3");
    const sewald_b200::ModSpec m = modspec(spec);
    switch (spec.kind) {
        case Kernel::stokeslet: return modified_tensor<SEWALD_STOKESLET>(m, k);
        case Kernel::rotlet: return modified_tensor<SEWALD_ROTLET>(m, k);
        default: return modified_tensor<SEWALD_STRESSLET>(m, k);
    }
}

Vec3 gauge_flow_correction(const ModifiedKernelSpec& spec, const SourceSystem& system) {
    if (spec.kind != Kernel::stokeslet || spec.d > 1) return {0.0, 0.0, 0.0};
    Vec3 F{0.0, 0.0, 0.0};
    for (const Vec3& f : system.f) F += f;
    if (spec.d == 0) return (4.0 * spec.b_B) * F;
    const double inv_L = 1.0 / system.cell.L[0];
    const double a = 4.0 * std::log(spec.ell_H * M_E) * inv_L;
    const double b = 2.0 * std::log(spec.ell_B) * inv_L;
    return {a * F[0], b * F[1], b * F[2]};
}

namespace detail {
double mollifier_taper(double t) {
    const double a2 = 4.0 * std::log(100.0) / 49.0;
    return std::exp(-a2 * t * t) + std::exp(-a2 * (t - 7.0) * (t - 7.0));
}
}  // namespace detail

// ---- realspace.h: host cell list -----------------------------------------------------
CellList build_cell_list(const SourceSystem& system, double rc) {
    if (!(rc > 0.0)) throw std::invalid_argument("cell list cutoff must be positive");
    validate_system(system);
    CellList cl;
    cl.rc = rc;
    cl.d = system.d;
    cl.cell = system.cell;
    const std::size_t N = system.size();
    cl.folded.reserve(N);
    for (const Vec3& x : system.x) cl.folded.push_back(wrap_position(x, system.cell, system.d));

    // periodic axes span the cell from 0; free axes the sources' bounding slab
    std::array<double, 3> span{};
    for (int ax = 0; ax < 3; ++ax) {
        if (ax < system.d) {
            span[ax] = system.cell.L[ax];
            cl.origin[ax] = 0.0;
        } else {
            double lo = N ? cl.folded[0][ax] : 0.0, hi = lo;
            for (const Vec3& p : cl.folded) {
                lo = std::min(lo, p[ax]);
                hi = std::max(hi, p[ax]);
            }
            span[ax] = hi - lo;
            cl.origin[ax] = lo;
        }
        cl.n[ax] = std::max(1, static_cast<int>(std::floor(span[ax] / rc)));
    }
    // at most 2^22 buckets: halve the longest axis (first of equals) until it fits
    while (static_cast<std::size_t>(cl.n[0]) * cl.n[1] * cl.n[2] > (std::size_t{1} << 22)) {
        int ax = 0;
        for (int a = 1; a < 3; ++a)
            if (cl.n[a] > cl.n[ax]) ax = a;
        cl.n[ax] = (cl.n[ax] + 1) / 2;
    }
    for (int ax = 0; ax < 3; ++ax) {
        cl.width[ax] = ax < system.d ? system.cell.L[ax] / cl.n[ax] : std::max(span[ax] / cl.n[ax], rc);
        int reach = static_cast<int>(std::ceil(rc / cl.width[ax]));
        while (reach * cl.width[ax] < rc) ++reach;
        cl.reach[ax] = reach;
    }
    // counting sort by bucket, x fastest
    const std::size_t nb = static_cast<std::size_t>(cl.n[0]) * cl.n[1] * cl.n[2];
    std::vector<std::size_t> bucket(N);
    cl.offset.assign(nb + 1, 0);
    for (std::size_t i = 0; i < N; ++i) {
        std::size_t id = 0;
        for (int ax = 2; ax >= 0; --ax) {
            const int c = std::clamp(
                static_cast<int>(std::floor((cl.folded[i][ax] - cl.origin[ax]) / cl.width[ax])), 0, cl.n[ax] - 1);
            id = id * static_cast<std::size_t>(cl.n[ax]) + static_cast<std::size_t>(c);
        }
        bucket[i] = id;
        ++cl.offset[id + 1];
    }
    std::partial_sum(cl.offset.begin(), cl.offset.end(), cl.offset.begin());
    std::vector<std::size_t> fill(cl.offset.begin(), cl.offset.end() - 1);
    cl.index.resize(N);
    for (std::size_t i = 0; i < N; ++i) cl.index[fill[bucket[i]]++] = i;
    return cl;
}

}  // namespace sewald
