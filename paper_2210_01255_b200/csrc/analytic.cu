// GPU analytic oracles (SURVEY §8 f row 3; SPEC.md module `reference`,
// SPEC.md:704-798). The reference ships this module as a stub
// (proj/src/reference.cpp:1); SPEC.md specifies it and PAPER.md gives the
// formulas. These are slow, independently derived sums used to validate the
// fast path, not part of it: they share no code with the Spectral Ewald
// kernels (own kernel tensors, own special functions: CUDA libdevice erf /
// erfcx / exp, a Gauss-Legendre incomplete Bessel K, a series / continued
// fraction E1).
//
//   direct_sum_0p              PAPER.md:355 (periodic-potential, D = 0): the bare
//                              kernel summed over all pairs, star-respecting
//   ewald_fourier_3p           PAPER.md:673 (fourier-space-potential-3p) with the
//                              stresslet zero mode PAPER.md:775 (k0-stresslet-3p)
//   fourier_reference (d=2)    PAPER.md:1051-1066 with Q^{2P}
//                              and Q^{2P,(0)}
//   fourier_reference (d=1)    PAPER.md:1087-1100 with Q^{1P}
//                              and Q^{1P,(0)}
//   incomplete Bessel K        K_nu(a, b) = int_1^inf t^{-nu-1} e^{-a t - b/t} dt
//                              (Knu-def), nu = -1, 0, 1, 2 at once
//
// Periodic sums are truncated at k_i = 2 pi j / L_i, -kmax_i <= j <= kmax_i - 1
// and the real part is kept, which averages the unpaired
// j = -kmax mode with its mirror exactly as the Spectral Ewald grid's
// Hermitian Nyquist treatment does.
#include "engine.h"

#include <cmath>
#include <string>
#include <vector>

using namespace sewald_b200;

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kSqrtPi = 1.77245385090551602730;
constexpr double kEulerGamma = 0.57721566490153286061;

template <class F>
int oracle_guard(sewald_gpu_ctx* ctx, F&& fn) {
    try {
        if (!ctx) return SEWALD_EINVAL;
        cudaSetDevice(ctx->device);
        fn();
        return SEWALD_OK;
    } catch (const EngineError& e) {
        ctx->err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        ctx->err = e.what();
        return SEWALD_ERUNTIME;
    }
}

// ---------------------------------------------------------------- helpers

struct cplx {
    double re, im;
};
__device__ __forceinline__ cplx cmul(cplx a, cplx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }

// e^{i 2 pi t} with t reduced to [-1/2, 1/2] first (argument rounding stays
// at the ulp of t, not of 2 pi t).
__device__ __forceinline__ cplx phase(double t) {
    t -= rint(t);
    double s, c;
    sincospi(2.0 * t, &s, &c);
    return {c, s};
}

// Strengths of one source: C = 3 (f) or 9 (q_l nu_m, row-major l, m).
struct Strength {
    double s[9];
};
__device__ __forceinline__ int ncomp(int kind) { return kind == SEWALD_STRESSLET ? 9 : 3; }
__device__ __forceinline__ void load_strength(int kind, const double* f, const double* nu, int64_t n, Strength& s) {
    if (kind == SEWALD_STRESSLET) {
        for (int l = 0; l < 3; ++l)
            for (int m = 0; m < 3; ++m) s.s[3 * l + m] = f[3 * n + l] * nu[3 * n + m];
    } else {
        for (int l = 0; l < 3; ++l) s.s[l] = f[3 * n + l];
    }
}

// u_j += Re[ sum_c Q_{j,c} s_c e^{i phi} ] for a complex tensor Q stored as
// [j][c] (c = l for rank 2, c = 3 l + m for rank 3).
__device__ __forceinline__ void contract_re(int C, const cplx* Q, const Strength& s, cplx e, double u[3]) {
    for (int j = 0; j < 3; ++j) {
        double re = 0.0, im = 0.0;
        for (int c = 0; c < C; ++c) {
            re += Q[j * C + c].re * s.s[c];
            im += Q[j * C + c].im * s.s[c];
        }
        u[j] += re * e.re - im * e.im;
    }
}

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide sum of three values; thread 0 gets the result.
__device__ void block_sum3(double u[3]) {
    __shared__ double red[3][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    for (int j = 0; j < 3; ++j) {
        const double v = warp_sum(u[j]);
        if (lane == 0) red[j][w] = v;
    }
    __syncthreads();
    if (w == 0)
        for (int j = 0; j < 3; ++j) {
            double v = lane < nw ? red[j][lane] : 0.0;
            v = warp_sum(v);
            u[j] = v;
        }
}

// ------------------------------------------------- special functions (oracle)

// E1(v) + ln(v), v > 0 (no cancellation as v -> 0):
// v <= 1: -gamma - sum_{k>=1} (-v)^k / (k k!); v > 1: E1 by its continued
// fraction (modified Lentz) plus ln v.
__device__ double e1_plus_log(double v) {
    if (v <= 1.0) {
        double term = 1.0, sum = 0.0;
        for (int k = 1; k < 60; ++k) {
            term *= -v / k;
            const double d = term / k;
            sum += d;
            if (fabs(d) < 1e-18 * fabs(sum) + 1e-300) break;
        }
        return -kEulerGamma - sum;
    }
    const double tiny = 1e-300;
    double b = v + 1.0, c = 1.0 / tiny, d = 1.0 / b, h = d;
    for (int i = 1; i < 500; ++i) {
        const double an = -(double)i * i;
        b += 2.0;
        d = 1.0 / (an * d + b);
        c = b + an / c;
        const double del = c * d;
        h *= del;
        if (fabs(del - 1.0) < 1e-17) break;
    }
    return h * exp(-v) + log(v);
}

__constant__ double c_gl16_x[8] = {0.0950125098376374401853193, 0.2816035507792589132304605,
                                   0.4580167776572273863424194, 0.6178762444026437484466718,
                                   0.7554044083550030338951012, 0.8656312023878317438804679,
                                   0.9445750230732325760779884, 0.9894009349916499325961542};
__constant__ double c_gl16_w[8] = {0.1894506104550684962853967, 0.1826034150449235888667637,
                                   0.1691565193950025381893121, 0.1495959888165767320815017,
                                   0.1246289712555338720524763, 0.0951585116824927848099251,
                                   0.0622535239386478928628438, 0.0271524594117540948517806};

// K_nu(a, b) for nu = -1, 0, 1, 2 (a > 0, b >= 0). In s = ln t the integrand
// is exp(-psi(s) - q s), psi(s) = a e^s + b e^{-s} - s, q = nu + 1: a convex
// exponent, so the integral is taken over the interval where psi_{-1} (right)
// and psi_2 (left) lie within 46 of their minima (e^{-46} ~ 1e-20 relative),
// with 16-point Gauss-Legendre panels no wider than 1 / sqrt(psi'') (the
// integrand's local Gaussian width) and 1.
__device__ double kb_psi(double a, double b, double s, double lin) { return a * exp(s) + b * exp(-s) + lin * s; }

__device__ double kb_edge(double a, double b, double lin, double s0, double dir, double target) {
    // first s = s0 + dir * t (t >= 0) with psi_lin(s) >= target, by doubling + bisection
    double t_lo = 0.0, t_hi = 0.5;
    for (int i = 0; i < 80; ++i) {
        const double s = s0 + dir * t_hi;
        if (dir < 0 && s <= 0.0) return 0.0;
        if (kb_psi(a, b, s, lin) >= target) break;
        t_lo = t_hi;
        t_hi *= 2.0;
    }
    for (int i = 0; i < 60; ++i) {
        const double tm = 0.5 * (t_lo + t_hi);
        if (kb_psi(a, b, s0 + dir * tm, lin) >= target) t_hi = tm; else t_lo = tm;
    }
    return fmax(0.0, s0 + dir * t_hi);
}

__device__ void incomplete_bessel_k4(double a, double b, double out[4]) {
    const double ab = a * b;
    // minimum of psi_{-1} = a e^s + b e^-s - s: a e^s - b e^-s = 1
    const double sm1 = fmax(0.0, log((1.0 + sqrt(1.0 + 4.0 * ab)) / (2.0 * a)));
    const double pm1 = kb_psi(a, b, sm1, -1.0);
    // minimum of psi_2 = a e^s + b e^-s + 2 s: a e^s - b e^-s = -2
    const double e2 = (-1.0 + sqrt(1.0 + ab)) / a;
    const double s2 = e2 > 1.0 ? log(e2) : 0.0;
    const double p2 = kb_psi(a, b, s2, 2.0);
    const double s_hi = kb_edge(a, b, -1.0, sm1, 1.0, pm1 + 46.0);
    const double s_lo = s2 > 0.0 ? kb_edge(a, b, 2.0, s2, -1.0, p2 + 46.0) : 0.0;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    double s = s_lo;
    while (s_hi - s > 1e-13) {
        const double c0 = a * exp(s) + b * exp(-s);
        double w = fmin(1.0, 1.0 / sqrt(c0));
        const double c1 = a * exp(s + w) + b * exp(-(s + w));
        w = fmin(w, 1.0 / sqrt(c1));
        w = fmin(w, s_hi - s);
        const double mid = s + 0.5 * w, hw = 0.5 * w;
        for (int i = 0; i < 16; ++i) {
            const double xi = (i < 8) ? -c_gl16_x[7 - i] : c_gl16_x[i - 8];
            const double wi = (i < 8) ? c_gl16_w[7 - i] : c_gl16_w[i - 8];
            const double si = mid + hw * xi;
            const double et = exp(si);
            const double g = wi * hw * exp(-(a * et + b / et - si - pm1));
            const double em = 1.0 / et;
            acc[0] += g;
            acc[1] += g * em;
            acc[2] += g * em * em;
            acc[3] += g * em * em * em;
        }
        s += w;
    }
    const double scale = exp(-pm1);
    for (int q = 0; q < 4; ++q) out[q] = acc[q] * scale;
}

// ------------------------------------------------------ kernel tensors

// Bare free-space kernels (PAPER.md eqs. for S, Omega, T; kernels.cpp:26-62):
// u += G(r) . s for one pair.
__device__ __forceinline__ void bare_apply(int kind, double r0, double r1, double r2, const Strength& s, double u[3]) {
    const double rr = r0 * r0 + r1 * r1 + r2 * r2;
    const double inv = 1.0 / sqrt(rr);
    const double r[3] = {r0, r1, r2};
    if (kind == SEWALD_STOKESLET) {
        const double rf = r0 * s.s[0] + r1 * s.s[1] + r2 * s.s[2];
        const double i3 = inv * inv * inv;
        for (int j = 0; j < 3; ++j) u[j] += s.s[j] * inv + r[j] * rf * i3;
    } else if (kind == SEWALD_ROTLET) {
        const double i3 = inv * inv * inv;
        // u = (f x r) / r^3
        u[0] += (s.s[1] * r2 - s.s[2] * r1) * i3;
        u[1] += (s.s[2] * r0 - s.s[0] * r2) * i3;
        u[2] += (s.s[0] * r1 - s.s[1] * r0) * i3;
    } else {
        double rqn = 0.0;  // r_l r_m q_l nu_m
        for (int l = 0; l < 3; ++l)
            for (int m = 0; m < 3; ++m) rqn += r[l] * r[m] * s.s[3 * l + m];
        const double i5 = inv * inv * inv * inv * inv;
        for (int j = 0; j < 3; ++j) u[j] += -6.0 * r[j] * rqn * i5;
    }
}

// Fourier-space long-range kernel G^F(k): diffop * scalar
// base * screening, stored as Q[j][c].
__device__ void gf_hat(int kind, const double k[3], double xi, cplx* Q) {
    const double k2 = k[0] * k[0] + k[1] * k[1] + k[2] * k[2];
    const double q = k2 / (4.0 * xi * xi);
    const double g = exp(-q);
    if (kind == SEWALD_ROTLET) {
        const double sc = 4.0 * kPi / k2 * g;
        // -i eps_jlm k_m
        const double eps_k[3][3] = {{0.0, k[2], -k[1]}, {-k[2], 0.0, k[0]}, {k[1], -k[0], 0.0}};
        for (int j = 0; j < 3; ++j)
            for (int l = 0; l < 3; ++l) Q[3 * j + l] = {0.0, -eps_k[j][l] * sc};
        return;
    }
    const double sc = -8.0 * kPi / (k2 * k2) * g * (1.0 + q);
    if (kind == SEWALD_STOKESLET) {
        for (int j = 0; j < 3; ++j)
            for (int l = 0; l < 3; ++l) Q[3 * j + l] = {((j == l) ? -k2 : 0.0) * sc + k[j] * k[l] * sc, 0.0};
        return;
    }
    for (int j = 0; j < 3; ++j)
        for (int l = 0; l < 3; ++l)
            for (int m = 0; m < 3; ++m) {
                const double dl = (j == l ? k[m] : 0.0) + (m == j ? k[l] : 0.0) + (l == m ? k[j] : 0.0);
                Q[9 * j + 3 * l + m] = {0.0, (-dl * k2 + 2.0 * k[j] * k[l] * k[m]) * sc};
            }
}

// Fill a fully symmetric rank-3 tensor from its 10 distinct entries
// e = {111,112,113,122,123,133,222,223,233,333} (1-based indices).
__device__ void sym3(const cplx e[10], cplx* Q) {
    const int idx[3][3][3] = {{{0, 1, 2}, {1, 3, 4}, {2, 4, 5}},
                              {{1, 3, 4}, {3, 6, 7}, {4, 7, 8}},
                              {{2, 4, 5}, {4, 7, 8}, {5, 8, 9}}};
    for (int j = 0; j < 3; ++j)
        for (int l = 0; l < 3; ++l)
            for (int m = 0; m < 3; ++m) Q[9 * j + 3 * l + m] = e[idx[j][l][m]];
}

// theta = e^{sgn alpha r3} erfc(alpha/(2 xi) + sgn xi r3) without overflow:
// for z >= 0 it equals exp(-alpha^2/(4 xi^2) - xi^2 r3^2) erfcx(z).
__device__ double theta_pm(double alpha, double r3, double xi, double sgn, double G) {
    const double z = alpha / (2.0 * xi) + sgn * xi * r3;
    if (z >= 0.0) return G * erfcx(z);
    return exp(sgn * alpha * r3) * 2.0 - G * erfcx(-z);
}

// Q^{2P}(k1, k2, r3; xi), (k1, k2) != 0: PAPER.md eq. (2p-aux), (2p-rotlet-Q),
// (2p-stokeslet-Q), (2p-stresslet-Q). The entries 113, 223, 333 of
// (2p-stresslet-Q) are printed with a factor 2 on the r3 alpha beta+ and beta-
// terms; applying K^T (k3 -> -i d/dr3) to Q^B = -pi Lambda / alpha^2 with the
// paper's own derivative rules gives -2 pi (xi^2 r3 lambda - k~1^2 r3 alpha
// beta+ - beta-) etc., which is what the defining integral (Qtilde-2p-def)
// evaluates to numerically (tests/test_gpu_analytic.py, Fourier quadrature).
__device__ void q2p(int kind, double k1, double k2, double r3, double xi, cplx* Q) {
    const double alpha = sqrt(k1 * k1 + k2 * k2);
    const double t1 = k1 / alpha, t2 = k2 / alpha;
    const double G = exp(-alpha * alpha / (4.0 * xi * xi) - xi * xi * r3 * r3);
    const double thp = theta_pm(alpha, r3, xi, 1.0, G);
    const double thm = theta_pm(alpha, r3, xi, -1.0, G);
    const double bp = thp + thm, bm = thp - thm;
    const double lam = 2.0 / (kSqrtPi * xi) * G;
    const double Lam = lam + bp / alpha - r3 * bm;
    const double Psi = -bp / alpha - r3 * bm;
    if (kind == SEWALD_ROTLET) {
        Q[0] = {0, 0};
        Q[1] = {-kPi * bm, 0};
        Q[2] = {0, kPi * t2 * bp};
        Q[3] = {kPi * bm, 0};
        Q[4] = {0, 0};
        Q[5] = {0, -kPi * t1 * bp};
        Q[6] = {0, -kPi * t2 * bp};
        Q[7] = {0, kPi * t1 * bp};
        Q[8] = {0, 0};
        return;
    }
    if (kind == SEWALD_STOKESLET) {
        Q[0] = {kPi * (t2 * t2 * Lam - Psi), 0};
        Q[1] = {-kPi * t1 * t2 * Lam, 0};
        Q[2] = {0, -kPi * t1 * r3 * bp};
        Q[3] = Q[1];
        Q[4] = {kPi * (t1 * t1 * Lam - Psi), 0};
        Q[5] = {0, -kPi * t2 * r3 * bp};
        Q[6] = Q[2];
        Q[7] = Q[5];
        Q[8] = {kPi * Lam, 0};
        return;
    }
    const double x2r = xi * xi * r3 * lam;
    cplx e[10];
    e[0] = {0, kPi * t1 * alpha * ((2 * t2 * t2 + 1) * Lam - 3 * Psi)};     // 111
    e[1] = {0, kPi * t2 * alpha * ((2 * t2 * t2 - 1) * Lam - Psi)};         // 112
    e[2] = {-2 * kPi * (x2r - t1 * t1 * r3 * alpha * bp - bm), 0};          // 113
    e[3] = {0, kPi * t1 * alpha * ((2 * t1 * t1 - 1) * Lam - Psi)};         // 122
    e[4] = {2 * kPi * t1 * t2 * r3 * alpha * bp, 0};                        // 123
    e[5] = {0, kPi * t1 * alpha * (Lam + Psi)};                             // 133
    e[6] = {0, kPi * t2 * alpha * ((2 * t1 * t1 + 1) * Lam - 3 * Psi)};     // 222
    e[7] = {-2 * kPi * (x2r - t2 * t2 * r3 * alpha * bp - bm), 0};          // 223
    e[8] = {0, kPi * t2 * alpha * (Lam + Psi)};                             // 233
    e[9] = {-2 * kPi * (x2r + r3 * alpha * bp - bm), 0};                    // 333
    sym3(e, Q);
}

// Q^{2P,(0)}(r3; xi): PAPER.md eqs. (2p-rotlet-Q0), (2p-stokeslet-Q0), (2p-stresslet-Q0).
__device__ void q2p_zero(int kind, double r3, double xi, cplx* Q) {
    const double er = erf(xi * r3), ga = exp(-xi * xi * r3 * r3);
    const int C = kind == SEWALD_STRESSLET ? 9 : 3;
    for (int i = 0; i < 3 * C; ++i) Q[i] = {0, 0};
    if (kind == SEWALD_ROTLET) {
        Q[1] = {2 * kPi * er, 0};
        Q[3] = {-2 * kPi * er, 0};
        return;
    }
    if (kind == SEWALD_STOKESLET) {
        const double v = -2 * kPi * (2 * r3 * er + ga / (kSqrtPi * xi));
        Q[0] = {v, 0};
        Q[4] = {v, 0};
        return;
    }
    const double v = -4 * kPi * (er + xi * r3 / kSqrtPi * ga);
    // C_1lm: (1,3),(3,1); C_2lm: (2,3),(3,2); C_3lm: identity
    Q[9 * 0 + 3 * 0 + 2] = {v, 0};
    Q[9 * 0 + 3 * 2 + 0] = {v, 0};
    Q[9 * 1 + 3 * 1 + 2] = {v, 0};
    Q[9 * 1 + 3 * 2 + 1] = {v, 0};
    Q[9 * 2 + 3 * 0 + 0] = {v, 0};
    Q[9 * 2 + 3 * 1 + 1] = {v, 0};
    Q[9 * 2 + 3 * 2 + 2] = {v, 0};
}

// Q^{1P}(k1, r2, r3; xi), k1 != 0, from K_nu(U, V), nu = -1..2 (Km[nu + 1]):
// PAPER.md eqs. (1p-aux), (1p-rotlet-Q), (1p-stokeslet-Q), (1p-stresslet-Q).
__device__ void q1p_from_k(int kind, double k1, double r2, double r3, double xi, const double Km[4], cplx* Q) {
    const double U = k1 * k1 / (4.0 * xi * xi), V = xi * xi * (r2 * r2 + r3 * r3);
    const double Kn1 = Km[0], K0 = Km[1], K1 = Km[2], K2 = Km[3];
    const double x2 = xi * xi;
    if (kind == SEWALD_ROTLET) {
        Q[0] = {0, 0};
        Q[1] = {2 * x2 * r3 * K1, 0};
        Q[2] = {-2 * x2 * r2 * K1, 0};
        Q[3] = {-2 * x2 * r3 * K1, 0};
        Q[4] = {0, 0};
        Q[5] = {0, -k1 * K0};
        Q[6] = {2 * x2 * r2 * K1, 0};
        Q[7] = {0, k1 * K0};
        Q[8] = {0, 0};
        return;
    }
    if (kind == SEWALD_STOKESLET) {
        Q[0] = {2 * K0 - 2 * V * K1, 0};
        Q[1] = {0, -k1 * r2 * K0};
        Q[2] = {0, -k1 * r3 * K0};
        Q[3] = Q[1];
        Q[4] = {2 * U * Kn1 + K0 - 2 * x2 * r3 * r3 * K1, 0};
        Q[5] = {2 * x2 * r2 * r3 * K1, 0};
        Q[6] = Q[2];
        Q[7] = Q[5];
        Q[8] = {2 * U * Kn1 + K0 - 2 * x2 * r2 * r2 * K1, 0};
        return;
    }
    cplx e[10];
    e[0] = {0, 2 * k1 * (U * Kn1 + 3 * K0 - 3 * V * K1)};                              // 111
    e[1] = {4 * x2 * r2 * (U * K0 - 2 * K1 + V * K2), 0};                              // 112
    e[2] = {4 * x2 * r3 * (U * K0 - 2 * K1 + V * K2), 0};                              // 113
    e[3] = {0, 2 * k1 * (U * Kn1 + x2 * (r2 * r2 - r3 * r3) * K1)};                    // 122
    e[4] = {0, 4 * x2 * k1 * r2 * r3 * K1};                                            // 123
    e[5] = {0, 2 * k1 * (U * Kn1 + x2 * (r3 * r3 - r2 * r2) * K1)};                    // 133
    e[6] = {-4 * x2 * r2 * (3 * U * K0 + 3 * K1 - x2 * (r2 * r2 + 3 * r3 * r3) * K2), 0};  // 222
    e[7] = {-4 * x2 * r3 * (U * K0 + K1 + x2 * (r2 * r2 - r3 * r3) * K2), 0};          // 223
    e[8] = {-4 * x2 * r2 * (U * K0 + K1 + x2 * (r3 * r3 - r2 * r2) * K2), 0};          // 233
    e[9] = {-4 * x2 * r3 * (3 * U * K0 + 3 * K1 - x2 * (3 * r2 * r2 + r3 * r3) * K2), 0};  // 333
    sym3(e, Q);
}

// Q^{1P,(0)}(r2, r3; xi) with gauge constants ell_H = ell_B = 1:
// PAPER.md eqs. (1p-aux-zero), (1p-rotlet-Q0), (1p-stokeslet-Q0) and its limit,
// (1p-stresslet-Q0) and its limit.
__device__ void q1p_zero(int kind, double r2, double r3, double xi, cplx* Q) {
    const int C = kind == SEWALD_STRESSLET ? 9 : 3;
    for (int i = 0; i < 3 * C; ++i) Q[i] = {0, 0};
    const double rho2 = r2 * r2 + r3 * r3;
    const double V = xi * xi * rho2;
    // phi1 / rho^2 and phi2 / rho^2 (finite as rho -> 0)
    double p1, p2;
    if (V < 1e-3) {  // series: phi1 = V - V^2/2 + V^3/6 ..., phi2 = V^2/2 - V^3/3 + V^4/8 ...
        p1 = xi * xi * (1.0 - V / 2.0 + V * V / 6.0 - V * V * V / 24.0 + V * V * V * V / 120.0);
        p2 = xi * xi * V * (0.5 - V / 3.0 + V * V / 8.0 - V * V * V / 30.0 + V * V * V * V / 144.0);
    } else {
        const double ph1 = -expm1(-V);
        p1 = ph1 / rho2;
        p2 = (ph1 - V * exp(-V)) / rho2;
    }
    if (kind == SEWALD_ROTLET) {
        // (2 phi1 / rho) [[0, r3~, -r2~], [-r3~, 0, 0], [r2~, 0, 0]] = 2 (phi1/rho^2) [r3, -r2 ...]
        Q[1] = {2 * p1 * r3, 0};
        Q[2] = {-2 * p1 * r2, 0};
        Q[3] = {-2 * p1 * r3, 0};
        Q[6] = {2 * p1 * r2, 0};
        return;
    }
    if (kind == SEWALD_STOKESLET) {
        // phi0 = E1(V) + log(rho^2) + 1 = (E1(V) + ln V) - ln xi^2 + 1
        const double phi0 = (V > 0.0 ? e1_plus_log(V) : -kEulerGamma) - log(xi * xi) + 1.0;
        const double phi1 = p1 * rho2;
        Q[0] = {-2 * (phi0 + phi1), 0};
        Q[4] = {-(phi0 + 2 * r3 * r3 * p1), 0};
        Q[5] = {2 * r2 * r3 * p1, 0};
        Q[7] = Q[5];
        Q[8] = {-(phi0 + 2 * r2 * r2 * p1), 0};
        return;
    }
    // R r~_a (c1 phi1 - c2 phi2) with R = -4/rho: -4 r_a (c1 phi1 - c2 phi2)/rho^2,
    // and the rho^-2-weighted squares r~_b^2 phi2 = r_b^2 (phi2/rho^2)
    cplx e[10];
    for (int i = 0; i < 10; ++i) e[i] = {0, 0};
    const double r22 = r2 * r2, r33 = r3 * r3;
    const double q2 = rho2 > 0.0 ? p2 / rho2 : 0.0;  // phi2 / rho^4 (-> xi^4/2 as rho -> 0)
    e[1] = {-4 * r2 * (2 * p1 - p2), 0};                                 // 112
    e[2] = {-4 * r3 * (2 * p1 - p2), 0};                                 // 113
    e[6] = {-4 * r2 * (3 * p1 - (r22 + 3 * r33) * q2), 0};               // 222
    e[7] = {-4 * r3 * (p1 - (r33 - r22) * q2), 0};                       // 223
    e[8] = {-4 * r2 * (p1 - (r22 - r33) * q2), 0};                       // 233
    e[9] = {-4 * r3 * (3 * p1 - (3 * r22 + r33) * q2), 0};               // 333
    sym3(e, Q);
}

// ------------------------------------------------------------ kernels

__global__ void direct_0p_kernel(int kind, const double* __restrict__ x, const double* __restrict__ f,
                                 const double* __restrict__ nu, int64_t N, const double* __restrict__ xt,
                                 int64_t Nt, int starred, double* __restrict__ u, int* flag) {
    const int64_t t = blockIdx.x;
    if (t >= Nt) return;
    const double p0 = xt[3 * t], p1 = xt[3 * t + 1], p2 = xt[3 * t + 2];
    double acc[3] = {0.0, 0.0, 0.0};
    for (int64_t n = threadIdx.x; n < N; n += blockDim.x) {
        if (starred && n == t) continue;
        const double r0 = p0 - x[3 * n], r1 = p1 - x[3 * n + 1], r2 = p2 - x[3 * n + 2];
        if (r0 == 0.0 && r1 == 0.0 && r2 == 0.0) {
            atomicOr(flag, 1);
            continue;
        }
        Strength s;
        load_strength(kind, f, nu, n, s);
        bare_apply(kind, r0, r1, r2, s, acc);
    }
    block_sum3(acc);
    if (threadIdx.x == 0)
        for (int j = 0; j < 3; ++j) u[3 * t + j] = acc[j];
}

// Structure factors S_c(k) = sum_n s_{n,c} e^{-i k.x_n} for the truncated
// cube of modes, one thread per mode.
__global__ void structure_factor_kernel(int kind, const double* __restrict__ x, const double* __restrict__ f,
                                        const double* __restrict__ nu, int64_t N, int K0, int K1, int K2,
                                        double L0, double L1, double L2, double* __restrict__ S) {
    const int64_t nm = (int64_t)(2 * K0) * (2 * K1) * (2 * K2);
    const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (m >= nm) return;
    const int j2 = (int)(m % (2 * K2)) - K2;
    const int j1 = (int)((m / (2 * K2)) % (2 * K1)) - K1;
    const int j0 = (int)(m / ((int64_t)(2 * K2) * (2 * K1))) - K0;
    const int C = ncomp(kind);
    double sr[9] = {0}, si[9] = {0};
    for (int64_t n = 0; n < N; ++n) {
        const double t = -(j0 * x[3 * n] / L0 + j1 * x[3 * n + 1] / L1 + j2 * x[3 * n + 2] / L2);
        const cplx e = phase(t);
        Strength s;
        load_strength(kind, f, nu, n, s);
        for (int c = 0; c < C; ++c) {
            sr[c] += s.s[c] * e.re;
            si[c] += s.s[c] * e.im;
        }
    }
    for (int c = 0; c < C; ++c) {
        S[(m * C + c) * 2] = sr[c];
        S[(m * C + c) * 2 + 1] = si[c];
    }
}

// u(x_t) = (1/V) sum_{k != 0} Re[ G^F(k) S(k) e^{i k.x_t} ] (+ the stresslet
// zero mode -(8 pi / V) (s0 x_t - s1), sums[0..3] = {s0, s1}).
__global__ void ewald_fourier_3p_kernel(int kind, const double* __restrict__ S, int K0, int K1, int K2,
                                        double L0, double L1, double L2, double xi,
                                        const double* __restrict__ xt, int64_t Nt, const double* __restrict__ sums,
                                        double* __restrict__ u) {
    const int64_t t = blockIdx.x;
    if (t >= Nt) return;
    const int64_t nm = (int64_t)(2 * K0) * (2 * K1) * (2 * K2);
    const int C = ncomp(kind);
    const double p0 = xt[3 * t], p1 = xt[3 * t + 1], p2 = xt[3 * t + 2];
    double acc[3] = {0.0, 0.0, 0.0};
    cplx Q[27];
    for (int64_t m = threadIdx.x; m < nm; m += blockDim.x) {
        const int j2 = (int)(m % (2 * K2)) - K2;
        const int j1 = (int)((m / (2 * K2)) % (2 * K1)) - K1;
        const int j0 = (int)(m / ((int64_t)(2 * K2) * (2 * K1))) - K0;
        if (j0 == 0 && j1 == 0 && j2 == 0) continue;
        const double k[3] = {2 * kPi * j0 / L0, 2 * kPi * j1 / L1, 2 * kPi * j2 / L2};
        gf_hat(kind, k, xi, Q);
        Strength s;  // S(k) as a complex strength: contract real and imaginary parts separately
        const cplx e = phase(j0 * p0 / L0 + j1 * p1 / L1 + j2 * p2 / L2);
        double ur[3] = {0, 0, 0}, ui[3] = {0, 0, 0};
        for (int c = 0; c < C; ++c) s.s[c] = S[(m * C + c) * 2];
        contract_re(C, Q, s, e, ur);
        for (int c = 0; c < C; ++c) s.s[c] = S[(m * C + c) * 2 + 1];
        contract_re(C, Q, s, cmul(e, cplx{0.0, 1.0}), ui);
        for (int j = 0; j < 3; ++j) acc[j] += ur[j] + ui[j];
    }
    block_sum3(acc);
    if (threadIdx.x == 0) {
        const double vol = L0 * L1 * L2;
        for (int j = 0; j < 3; ++j) {
            double v = acc[j] / vol;
            if (kind == SEWALD_STRESSLET) v += -8.0 * kPi / vol * (sums[0] * xt[3 * t + j] - sums[1 + j]);
            u[3 * t + j] = v;
        }
    }
}

// s0 = sum_n q_n . nu_n, s1 = sum_n (q_n . nu_n) x_n (one block).
__global__ void stresslet_moments_kernel(const double* __restrict__ x, const double* __restrict__ f,
                                         const double* __restrict__ nu, int64_t N, double* sums) {
    double a = 0.0, b[3] = {0.0, 0.0, 0.0};
    for (int64_t n = threadIdx.x; n < N; n += blockDim.x) {
        const double qn = f[3 * n] * nu[3 * n] + f[3 * n + 1] * nu[3 * n + 1] + f[3 * n + 2] * nu[3 * n + 2];
        a += qn;
        for (int j = 0; j < 3; ++j) b[j] += qn * x[3 * n + j];
    }
    __shared__ double red[4][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double v[4] = {warp_sum(a), warp_sum(b[0]), warp_sum(b[1]), warp_sum(b[2])};
    if (lane == 0)
        for (int i = 0; i < 4; ++i) red[i][w] = v[i];
    __syncthreads();
    if (threadIdx.x == 0)
        for (int i = 0; i < 4; ++i) {
            double s = 0.0;
            for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[i][k];
            sums[i] = s;
        }
}

// Doubly periodic q-sum (periodic x, y; free z), one block per target.
__global__ void qsum_2p_kernel(int kind, const double* __restrict__ x, const double* __restrict__ f,
                               const double* __restrict__ nu, int64_t N, const double* __restrict__ xt,
                               int64_t Nt, int K0, int K1, double L0, double L1, double xi,
                               double* __restrict__ u) {
    const int64_t t = blockIdx.x;
    if (t >= Nt) return;
    const int C = ncomp(kind);
    const int64_t nmode = (int64_t)(2 * K0) * (2 * K1);
    const int64_t work = N * nmode;
    double acc[3] = {0.0, 0.0, 0.0};
    cplx Q[27];
    const double p0 = xt[3 * t], p1 = xt[3 * t + 1], p2 = xt[3 * t + 2];
    for (int64_t w = threadIdx.x; w < work; w += blockDim.x) {
        const int64_t n = w / nmode, m = w % nmode;
        const int j0 = (int)(m / (2 * K1)) - K0, j1 = (int)(m % (2 * K1)) - K1;
        Strength s;
        load_strength(kind, f, nu, n, s);
        const double r3 = p2 - x[3 * n + 2];
        if (j0 == 0 && j1 == 0) {
            q2p_zero(kind, r3, xi, Q);
            contract_re(C, Q, s, cplx{1.0, 0.0}, acc);
        } else {
            q2p(kind, 2 * kPi * j0 / L0, 2 * kPi * j1 / L1, r3, xi, Q);
            const cplx e = phase(j0 * (p0 - x[3 * n]) / L0 + j1 * (p1 - x[3 * n + 1]) / L1);
            contract_re(C, Q, s, e, acc);
        }
    }
    block_sum3(acc);
    if (threadIdx.x == 0)
        for (int j = 0; j < 3; ++j) u[3 * t + j] = acc[j] / (L0 * L1);
}

// Singly periodic q-sum (periodic x; free y, z), one block per target; the
// incomplete Bessel K of |j| serves both k1 = +-2 pi |j| / L0.
__global__ void qsum_1p_kernel(int kind, const double* __restrict__ x, const double* __restrict__ f,
                               const double* __restrict__ nu, int64_t N, const double* __restrict__ xt,
                               int64_t Nt, int K0, double L0, double xi, double* __restrict__ u) {
    const int64_t t = blockIdx.x;
    if (t >= Nt) return;
    const int C = ncomp(kind);
    const int64_t work = N * (int64_t)(K0 + 1);  // |j| = 0 (zero mode) .. K0
    double acc[3] = {0.0, 0.0, 0.0};
    cplx Q[27];
    const double p0 = xt[3 * t], p1 = xt[3 * t + 1], p2 = xt[3 * t + 2];
    for (int64_t w = threadIdx.x; w < work; w += blockDim.x) {
        const int64_t n = w / (K0 + 1);
        const int aj = (int)(w % (K0 + 1));
        Strength s;
        load_strength(kind, f, nu, n, s);
        const double r2 = p1 - x[3 * n + 1], r3 = p2 - x[3 * n + 2];
        if (aj == 0) {
            q1p_zero(kind, r2, r3, xi, Q);
            contract_re(C, Q, s, cplx{1.0, 0.0}, acc);
            continue;
        }
        const double k1 = 2 * kPi * aj / L0;
        double Km[4];
        incomplete_bessel_k4(k1 * k1 / (4.0 * xi * xi), xi * xi * (r2 * r2 + r3 * r3), Km);
        const double dx = (p0 - x[3 * n]) / L0;
        // j = -aj always in range; j = +aj only below K0
        q1p_from_k(kind, -k1, r2, r3, xi, Km, Q);
        contract_re(C, Q, s, phase(-aj * dx), acc);
        if (aj < K0) {
            q1p_from_k(kind, k1, r2, r3, xi, Km, Q);
            contract_re(C, Q, s, phase(aj * dx), acc);
        }
    }
    block_sum3(acc);
    if (threadIdx.x == 0)
        for (int j = 0; j < 3; ++j) u[3 * t + j] = acc[j] / L0;
}

__global__ void kbatch_kernel(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                              double* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double k[4];
    incomplete_bessel_k4(a[i], b[i], k);
    for (int q = 0; q < 4; ++q) out[4 * i + q] = k[q];
}

// Pointwise tensors for tests: args (3 per point) = (k1, k2, r3) for d = 2,
// (k1, r2, r3) for d = 1; zero_mode selects Q^{(0)} (k arguments ignored).
__global__ void qtensor_kernel(int kind, int d, int zero_mode, int64_t n, const double* __restrict__ args,
                               double xi, double* __restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int C = ncomp(kind);
    cplx Q[27];
    const double a0 = args[3 * i], a1 = args[3 * i + 1], a2 = args[3 * i + 2];
    if (d == 2) {
        if (zero_mode) q2p_zero(kind, a2, xi, Q); else q2p(kind, a0, a1, a2, xi, Q);
    } else {
        if (zero_mode) {
            q1p_zero(kind, a1, a2, xi, Q);
        } else {
            double Km[4];
            incomplete_bessel_k4(a0 * a0 / (4.0 * xi * xi), xi * xi * (a1 * a1 + a2 * a2), Km);
            q1p_from_k(kind, a0, a1, a2, xi, Km, Q);
        }
    }
    for (int c = 0; c < 3 * C; ++c) {
        out[(i * 3 * C + c) * 2] = Q[c].re;
        out[(i * 3 * C + c) * 2 + 1] = Q[c].im;
    }
}

// ------------------------------------------------------------ host side

struct Staged {
    DevBuf x, f, nu, xt, u, S, sums, flag;
};

void check_inputs(int kind, const double* x, const double* f, const double* nu, int64_t N, const double* xt,
                  int64_t Nt) {
    if (kind < 0 || kind > 2) throw EngineError(SEWALD_EINVAL, "unknown kernel");
    if (N < 0 || Nt < 0) throw EngineError(SEWALD_EINVAL, "negative size");
    if (N > 0 && (!x || !f)) throw EngineError(SEWALD_EINVAL, "null source arrays");
    if (N > 0 && kind == SEWALD_STRESSLET && !nu) throw EngineError(SEWALD_EINVAL, "stresslet needs orientations");
    if (Nt > 0 && !xt) throw EngineError(SEWALD_EINVAL, "null target array");
}

void upload(DevBuf& b, const double* h, int64_t n, cudaStream_t st) {
    double* d = static_cast<double*>(b.ensure(sizeof(double) * std::max<int64_t>(n, 1)));
    if (n > 0) cuda_check(cudaMemcpyAsync(d, h, sizeof(double) * n, cudaMemcpyHostToDevice, st), "H2D");
}

void stage_sources(Staged& g, int kind, const double* x, const double* f, const double* nu, int64_t N,
                   const double* xt, int64_t Nt, cudaStream_t st) {
    upload(g.x, x, 3 * N, st);
    upload(g.f, f, 3 * N, st);
    upload(g.nu, kind == SEWALD_STRESSLET ? nu : nullptr, kind == SEWALD_STRESSLET ? 3 * N : 0, st);
    upload(g.xt, xt, 3 * Nt, st);
    g.u.ensure(sizeof(double) * std::max<int64_t>(3 * Nt, 1));
}

void finish(sewald_gpu_ctx* ctx, Staged& g, int64_t Nt, double* u_out) {
    cuda_check(cudaGetLastError(), "oracle kernel launch");
    if (Nt > 0)
        cuda_check(cudaMemcpyAsync(u_out, g.u.as<double>(), sizeof(double) * 3 * Nt, cudaMemcpyDeviceToHost,
                                   ctx->stream), "D2H");
    cuda_check(cudaStreamSynchronize(ctx->stream), "oracle sync");
}

int check_kmax(const int* kmax, int n) {
    for (int a = 0; a < n; ++a)
        if (kmax[a] < 1 || kmax[a] > 4096) throw EngineError(SEWALD_EINVAL, "kmax must be in 1..4096");
    return 0;
}

}  // namespace

extern "C" {

int sewald_gpu_direct_sum_0p(sewald_gpu_ctx* ctx, int kind, const double* x, const double* f, const double* nu,
                             int64_t N, const double* xt, int64_t Nt, int starred, double* u_out) {
    return oracle_guard(ctx, [&] {
        check_inputs(kind, x, f, nu, N, xt, Nt);
        if (starred && Nt != N) throw EngineError(SEWALD_EINVAL, "starred evaluation needs one target per source");
        Staged g;
        stage_sources(g, kind, x, f, nu, N, xt, Nt, ctx->stream);
        int* flag = static_cast<int*>(g.flag.ensure(sizeof(int)));
        cuda_check(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream), "memset");
        if (Nt > 0)
            direct_0p_kernel<<<(unsigned)Nt, 256, 0, ctx->stream>>>(kind, g.x.as<double>(), g.f.as<double>(),
                                                                    g.nu.as<double>(), N, g.xt.as<double>(), Nt,
                                                                    starred, g.u.as<double>(), flag);
        ++ctx->launches;
        int hflag = 0;
        cuda_check(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream), "flag");
        finish(ctx, g, Nt, u_out);
        if (hflag) throw EngineError(SEWALD_EDOMAIN, "direct sum: target coincides with a source (singular kernel)");
    });
}

int sewald_gpu_ewald_fourier_3p(sewald_gpu_ctx* ctx, int kind, const double L[3], double xi, const int kmax[3],
                                const double* x, const double* f, const double* nu, int64_t N, const double* xt,
                                int64_t Nt, double* u_out) {
    return oracle_guard(ctx, [&] {
        check_inputs(kind, x, f, nu, N, xt, Nt);
        if (!(xi > 0.0)) throw EngineError(SEWALD_EINVAL, "xi must be positive");
        for (int a = 0; a < 3; ++a)
            if (!(L[a] > 0.0)) throw EngineError(SEWALD_EINVAL, "cell lengths must be positive");
        check_kmax(kmax, 3);
        Staged g;
        stage_sources(g, kind, x, f, nu, N, xt, Nt, ctx->stream);
        const int C = kind == SEWALD_STRESSLET ? 9 : 3;
        const int64_t nm = (int64_t)(2 * kmax[0]) * (2 * kmax[1]) * (2 * kmax[2]);
        double* S = static_cast<double*>(g.S.ensure(sizeof(double) * 2 * C * nm));
        double* sums = static_cast<double*>(g.sums.ensure(sizeof(double) * 4));
        cuda_check(cudaMemsetAsync(sums, 0, sizeof(double) * 4, ctx->stream), "memset");
        structure_factor_kernel<<<(unsigned)((nm + 127) / 128), 128, 0, ctx->stream>>>(
            kind, g.x.as<double>(), g.f.as<double>(), g.nu.as<double>(), N, kmax[0], kmax[1], kmax[2], L[0], L[1],
            L[2], S);
        if (kind == SEWALD_STRESSLET && N > 0)
            stresslet_moments_kernel<<<1, 1024, 0, ctx->stream>>>(g.x.as<double>(), g.f.as<double>(),
                                                                  g.nu.as<double>(), N, sums);
        if (Nt > 0)
            ewald_fourier_3p_kernel<<<(unsigned)Nt, 256, 0, ctx->stream>>>(
                kind, S, kmax[0], kmax[1], kmax[2], L[0], L[1], L[2], xi, g.xt.as<double>(), Nt, sums,
                g.u.as<double>());
        ctx->launches += 3;
        finish(ctx, g, Nt, u_out);
    });
}

int sewald_gpu_fourier_reference_potential(sewald_gpu_ctx* ctx, int kind, int d, const double L[3], double xi,
                                           const int* kmax, const double* x, const double* f, const double* nu,
                                           int64_t N, const double* xt, int64_t Nt, double* u_out) {
    if (d == 3) return sewald_gpu_ewald_fourier_3p(ctx, kind, L, xi, kmax, x, f, nu, N, xt, Nt, u_out);
    return oracle_guard(ctx, [&] {
        if (d != 1 && d != 2) throw EngineError(SEWALD_EINVAL, "fourier_reference_potential needs d in 1..3");
        check_inputs(kind, x, f, nu, N, xt, Nt);
        if (!(xi > 0.0)) throw EngineError(SEWALD_EINVAL, "xi must be positive");
        for (int a = 0; a < d; ++a)
            if (!(L[a] > 0.0)) throw EngineError(SEWALD_EINVAL, "periodic cell lengths must be positive");
        check_kmax(kmax, d);
        Staged g;
        stage_sources(g, kind, x, f, nu, N, xt, Nt, ctx->stream);
        if (Nt > 0) {
            if (d == 2)
                qsum_2p_kernel<<<(unsigned)Nt, 256, 0, ctx->stream>>>(kind, g.x.as<double>(), g.f.as<double>(),
                                                                      g.nu.as<double>(), N, g.xt.as<double>(), Nt,
                                                                      kmax[0], kmax[1], L[0], L[1], xi,
                                                                      g.u.as<double>());
            else
                qsum_1p_kernel<<<(unsigned)Nt, 256, 0, ctx->stream>>>(kind, g.x.as<double>(), g.f.as<double>(),
                                                                      g.nu.as<double>(), N, g.xt.as<double>(), Nt,
                                                                      kmax[0], L[0], xi, g.u.as<double>());
            ++ctx->launches;
        }
        finish(ctx, g, Nt, u_out);
    });
}

int sewald_gpu_incomplete_bessel_k4(sewald_gpu_ctx* ctx, int64_t n, const double* a, const double* b,
                                    double* out) {
    return oracle_guard(ctx, [&] {
        if (n < 0 || (n > 0 && (!a || !b || !out))) throw EngineError(SEWALD_EINVAL, "bad arguments");
        for (int64_t i = 0; i < n; ++i)
            if (!(a[i] > 0.0) || !(b[i] >= 0.0))
                throw EngineError(SEWALD_EDOMAIN, "incomplete Bessel K oracle requires a > 0, b >= 0");
        if (n == 0) return;
        DevBuf da, db, dout;
        upload(da, a, n, ctx->stream);
        upload(db, b, n, ctx->stream);
        double* o = static_cast<double*>(dout.ensure(sizeof(double) * 4 * n));
        kbatch_kernel<<<(unsigned)((n + 127) / 128), 128, 0, ctx->stream>>>(n, da.as<double>(), db.as<double>(), o);
        ++ctx->launches;
        cuda_check(cudaGetLastError(), "launch");
        cuda_check(cudaMemcpyAsync(out, o, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        cuda_check(cudaStreamSynchronize(ctx->stream), "sync");
    });
}

int sewald_gpu_qtensor(sewald_gpu_ctx* ctx, int kind, int d, int zero_mode, int64_t n, const double* args,
                       double xi, double* out) {
    return oracle_guard(ctx, [&] {
        if (kind < 0 || kind > 2 || (d != 1 && d != 2)) throw EngineError(SEWALD_EINVAL, "kind / d");
        if (!(xi > 0.0)) throw EngineError(SEWALD_EINVAL, "xi must be positive");
        if (n < 0 || (n > 0 && (!args || !out))) throw EngineError(SEWALD_EINVAL, "bad arguments");
        if (!zero_mode)
            for (int64_t i = 0; i < n; ++i) {
                const bool kzero = d == 2 ? (args[3 * i] == 0.0 && args[3 * i + 1] == 0.0) : args[3 * i] == 0.0;
                if (kzero) throw EngineError(SEWALD_EDOMAIN, "q-tensor of the zero mode: use zero_mode = 1");
            }
        if (n == 0) return;
        const int C = kind == SEWALD_STRESSLET ? 9 : 3;
        DevBuf da, dout;
        upload(da, args, 3 * n, ctx->stream);
        double* o = static_cast<double*>(dout.ensure(sizeof(double) * 2 * 3 * C * n));
        qtensor_kernel<<<(unsigned)((n + 63) / 64), 64, 0, ctx->stream>>>(kind, d, zero_mode, n, da.as<double>(),
                                                                         xi, o);
        ++ctx->launches;
        cuda_check(cudaGetLastError(), "launch");
        cuda_check(cudaMemcpyAsync(out, o, sizeof(double) * 2 * 3 * C * n, cudaMemcpyDeviceToHost, ctx->stream),
                   "D2H");
        cuda_check(cudaStreamSynchronize(ctx->stream), "sync");
    });
}

int sewald_rms_error(const double* u, const double* u_ref, int64_t n, double* abs_err, double* rel_err) {
    // SPEC.md:758-764 (abs-rms-error / rel-rms-error, PAPER.md): sqrt(mean |u - u_ref|^2)
    // and that divided by sqrt(mean |u_ref|^2).
    if (n <= 0 || !u || !u_ref) return SEWALD_EINVAL;
    double se = 0.0, sr = 0.0;
    for (int64_t i = 0; i < 3 * n; ++i) {
        const double dlt = u[i] - u_ref[i];
        se += dlt * dlt;
        sr += u_ref[i] * u_ref[i];
    }
    const double a = std::sqrt(se / (double)n);
    if (abs_err) *abs_err = a;
    if (rel_err) {
        if (sr == 0.0) return SEWALD_EDOMAIN;
        *rel_err = a / std::sqrt(sr / (double)n);
    }
    return SEWALD_OK;
}

}  // extern "C"
