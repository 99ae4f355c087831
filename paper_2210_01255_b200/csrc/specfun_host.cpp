// Host special functions of the drop-in API that the hot path does not use:
// the reference's analytic-module helpers declared in sewald/specfun.h
// (/root/reference/proj/include/sewald/specfun.h:18-45). Standard published
// algorithms, written here:
//   erf / erfc rational form   erfc(x) = e^{-x^2} erfcx(x), erfcx from the
//                              P9/Q9 fit of tools/fit_erfcx.py (x <= 10) and its
//                              asymptotic series beyond; erf by its Taylor
//                              series for |x| < 1/2
//   exp_integral_E(n, a)       series about 0 (a <= 1) / modified-Lentz
//                              continued fraction (a > 1)
//   incomplete_bessel_K        int_1^inf e^{-a t - b/t} t^{-(nu+1)} dt with
//                              t = e^s: adaptive Gauss-Kronrod (7/15) on the
//                              double-exponentially decaying integrand; a = 0
//                              in closed form b^{-nu} gamma(nu, b)
//   exp_times_erfc(L, z)       e^{L - z^2} erfcx(z) (no separate over/underflow)
#include "../../include/sewald/specfun.h"

#include "erfcx_coeffs.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <stdexcept>
#include <vector>

namespace sewald {

namespace {

constexpr double kSqrtPi = 1.7724538509055160273;
constexpr double kEuler = 0.57721566490153286061;

// e^{x^2} erfc(x) for x >= 0
double erfcx_pos(double x) {
    if (x <= 10.0) {
        static const double P[] = SEWALD_ERFCX_P;
        static const double Q[] = SEWALD_ERFCX_Q;
        double p = P[9], q = Q[9];
        for (int i = 8; i >= 0; --i) {
            p = p * x + P[i];
            q = q * x + Q[i];
        }
        return p / q;
    }
    // asymptotic: 1/(x sqrt(pi)) sum_k (-1)^k (2k-1)!! / (2 x^2)^k
    const double r = 1.0 / (2.0 * x * x);
    double term = 1.0, sum = 1.0;
    for (int k = 1; k < 60; ++k) {
        term *= -(2.0 * k - 1.0) * r;
        sum += term;
        if (std::fabs(term) < 1e-17 * std::fabs(sum)) break;
    }
    return sum / (x * kSqrtPi);
}

double erf_series(double x) {  // |x| < 1/2
    const double x2 = x * x;
    double term = x, sum = x;
    for (int n = 1; n < 40; ++n) {
        term *= -x2 / n;
        const double add = term / (2.0 * n + 1.0);
        sum += add;
        if (std::fabs(add) < 1e-18 * std::fabs(sum)) break;
    }
    return 2.0 / kSqrtPi * sum;
}

// 15-point Kronrod / 7-point Gauss on [-1, 1]
const double kXgk[8] = {0.991455371120812639206854697526329, 0.949107912342758524526189684047851,
                        0.864864423359769072789712788640926, 0.741531185599394439863864773280788,
                        0.586087235467691130294144845693013, 0.405845151377397166906606412076961,
                        0.207784955007898467600689403773245, 0.0};
const double kWgk[8] = {0.022935322010529224963732008058970, 0.063092092629978553290700663189204,
                        0.104790010322250183839876322541518, 0.140653259715525918745189590510238,
                        0.169004726639267902826583426598550, 0.190350578064785409913256402421014,
                        0.204432940075298892414161999234649, 0.209482141084727828012999174891714};
const double kWg[4] = {0.129484966168869693270611432679082, 0.279705391489276667901467771423780,
                       0.381830050505118944950369775488975, 0.417959183673469387755102040816327};

// Integrand of K_nu(a, b) in s = ln t for the orders nu0..nu0+3 at once:
// exp(-a e^s - b e^{-s} - nu s).
void kb_integrand(int nu0, double a, double b, double s, double out[4]) {
    const double es = std::exp(s);
    const double ems = 1.0 / es;
    out[0] = std::exp(-a * es - b * ems - nu0 * s);
    for (int q = 1; q < 4; ++q) out[q] = out[q - 1] * ems;
}

void gk15(int nu0, double a, double b, double lo, double hi, double res[4], double err[4]) {
    const double c = 0.5 * (lo + hi), h = 0.5 * (hi - lo);
    double fc[4];
    kb_integrand(nu0, a, b, c, fc);
    double rk[4], rg[4];
    for (int q = 0; q < 4; ++q) {
        rk[q] = fc[q] * kWgk[7];
        rg[q] = fc[q] * kWg[3];
    }
    for (int j = 0; j < 7; ++j) {
        double f1[4], f2[4];
        kb_integrand(nu0, a, b, c - h * kXgk[j], f1);
        kb_integrand(nu0, a, b, c + h * kXgk[j], f2);
        for (int q = 0; q < 4; ++q) {
            rk[q] += kWgk[j] * (f1[q] + f2[q]);
            if (j & 1) rg[q] += kWg[j / 2] * (f1[q] + f2[q]);
        }
    }
    for (int q = 0; q < 4; ++q) {
        res[q] = rk[q] * h;
        err[q] = std::fabs((rk[q] - rg[q]) * h);
    }
}

// Adaptive GK15 over [0, S] for all four orders; the subdivision stops when
// the estimated error of every order is below rel_tol of its value.
std::array<double, 4> kb_quadrature(int nu0, double a, double b, const QuadratureConfig& cfg) {
    // beyond S the integrand is below e^{-745} (a > 0: a e^S >= 745 + max(0, S))
    double S = 1.0;
    while (a * std::exp(S) < 745.0 + std::fabs((double)nu0) * S + S) S += 1.0;
    struct Seg {
        double lo, hi, r[4], e[4];
    };
    std::vector<Seg> segs;
    const int n0 = std::max(8, (int)std::ceil(S));
    for (int k = 0; k < n0; ++k) {
        Seg g{S * k / n0, S * (k + 1) / n0, {}, {}};
        gk15(nu0, a, b, g.lo, g.hi, g.r, g.e);
        segs.push_back(g);
    }
    const int max_seg = std::max(cfg.max_subdivisions, n0) * 8;
    for (;;) {
        double tot[4] = {0, 0, 0, 0}, et[4] = {0, 0, 0, 0};
        for (const Seg& g : segs)
            for (int q = 0; q < 4; ++q) {
                tot[q] += g.r[q];
                et[q] += g.e[q];
            }
        bool done = true;
        for (int q = 0; q < 4; ++q)
            if (et[q] > cfg.rel_tol * std::fabs(tot[q]) && et[q] > 1e-300) done = false;
        if (done || (int)segs.size() >= max_seg) return {tot[0], tot[1], tot[2], tot[3]};
        // split the segment with the largest relative error contribution
        size_t worst = 0;
        double wv = -1.0;
        for (size_t i = 0; i < segs.size(); ++i) {
            double v = 0.0;
            for (int q = 0; q < 4; ++q) v = std::max(v, segs[i].e[q] / std::max(std::fabs(tot[q]), 1e-300));
            if (v > wv) {
                wv = v;
                worst = i;
            }
        }
        const Seg g = segs[worst];
        const double mid = 0.5 * (g.lo + g.hi);
        Seg l{g.lo, mid, {}, {}}, r{mid, g.hi, {}, {}};
        gk15(nu0, a, b, l.lo, l.hi, l.r, l.e);
        gk15(nu0, a, b, r.lo, r.hi, r.r, r.e);
        segs[worst] = l;
        segs.push_back(r);
    }
}

// a = 0 (nu >= 1): int_1^inf e^{-b/t} t^{-nu-1} dt = b^{-nu} gamma(nu, b),
// gamma(n, b) = b^n e^{-b} sum_k b^k / (n (n+1) ... (n+k)).
double kb_a0(int nu, double b) {
    double term = 1.0 / nu, sum = term;
    for (int k = 1; k < 2000; ++k) {
        term *= b / (nu + k);
        sum += term;
        if (term < 1e-17 * sum) break;
    }
    return std::exp(-b) * sum;
}

void kb_domain(int order, double a, double b) {
    if (!(a >= 0.0) || !(b >= 0.0)) throw std::domain_error("incomplete Bessel K requires a, b >= 0");
    if (a == 0.0 && b == 0.0) throw std::domain_error("incomplete Bessel K requires a or b positive");
    if (a == 0.0 && order <= 0) throw std::domain_error("incomplete Bessel K with a = 0 requires nu > 0");
}

}  // namespace

namespace detail {

double erfc_rational(double x) {
    if (std::isnan(x)) return x;
    if (x < 0.0) return 2.0 - erfc_rational(-x);
    if (x > 27.3) return 0.0;
    return std::exp(-x * x) * erfcx_pos(x);
}

double erf_rational(double x) {
    if (std::isnan(x)) return x;
    if (std::fabs(x) < 0.5) return erf_series(x);
    const double c = erfc_rational(std::fabs(x));
    return x < 0.0 ? c - 1.0 : 1.0 - c;
}

}  // namespace detail

double exp_integral_E(int order, double a) {
    if (order < 1) throw std::invalid_argument("exp_integral_E requires order >= 1");
    if (!(a > 0.0)) throw std::domain_error("exp_integral_E requires a > 0");
    const int n = order;
    if (a > 1.0) {  // continued fraction, modified Lentz
        const double tiny = 1e-300;
        double b = a + n, c = 1.0 / tiny, d = 1.0 / b, h = d;
        for (int i = 1; i < 10000; ++i) {
            const double an = -(double)i * (n - 1 + i);
            b += 2.0;
            d = 1.0 / (an * d + b);
            c = b + an / c;
            const double del = c * d;
            h *= del;
            if (std::fabs(del - 1.0) < 1e-16) break;
        }
        return h * std::exp(-a);
    }
    // series about a = 0
    double ans = (n - 1 != 0) ? 1.0 / (n - 1) : -std::log(a) - kEuler;
    double fact = 1.0;
    for (int i = 1; i < 10000; ++i) {
        fact *= -a / i;
        double del;
        if (i != n - 1) {
            del = -fact / (i - n + 1);
        } else {
            double psi = -kEuler;
            for (int k = 1; k <= n - 1; ++k) psi += 1.0 / k;
            del = fact * (-std::log(a) + psi);
        }
        ans += del;
        if (std::fabs(del) < std::fabs(ans) * 1e-17) break;
    }
    return ans;
}

double incomplete_bessel_K(int order, double a, double b, const QuadratureConfig& cfg) {
    kb_domain(order, a, b);
    if (a == 0.0) return kb_a0(order, b);
    if (b == 0.0) {
        if (order >= 0) return exp_integral_E(order + 1, a);  // int_1^inf e^{-a t} t^{-(nu+1)} dt
        if (order == -1) return std::exp(-a) / a;
    }
    return kb_quadrature(order, a, b, cfg)[0];
}

std::array<double, 4> incomplete_bessel_K_batch(double a, double b, const QuadratureConfig& cfg) {
    kb_domain(-1, a, b);
    if (b == 0.0)
        return {incomplete_bessel_K(-1, a, 0.0, cfg), incomplete_bessel_K(0, a, 0.0, cfg),
                incomplete_bessel_K(1, a, 0.0, cfg), incomplete_bessel_K(2, a, 0.0, cfg)};
    return kb_quadrature(-1, a, b, cfg);
}

double exp_times_erfc(double log_scale, double z) {
    if (z < 0.5) return std::exp(log_scale) * detail::erfc_rational(z);
    return std::exp(log_scale - z * z) * erfcx_pos(z);
}

}  // namespace sewald
