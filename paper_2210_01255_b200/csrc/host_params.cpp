// Host parameter layer. See host_params.h for the reference functions each
// routine restates. Compiled with the same host flags as the oracle build so
// the scalar results are bit-identical to the reference's (checked by
// tests/test_host_params.py against oracle/_ref).
#include "host_params.h"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>
#include <string>

namespace sewald_b200 {

namespace {

void must_be_positive(double v, const char* name) {
    if (!(v > 0.0)) throw std::invalid_argument(std::string(name) + " must be positive");
}

// Truncation-error model c * x^a * exp(-b x^2) (estimates.cpp:24-53).
struct ErrorModel {
    double c, a, b;
    double at(double x) const { return c * std::pow(x, a) * std::exp(-b * x * x); }
    double log_excess(double x, double log_tau) const {
        return std::log(c) + a * std::log(x) - b * x * x - log_tau;
    }
};

ErrorModel kspace_model(int kernel, double xi, double L, double Q) {
    const double b = 1.0 / (4.0 * xi * xi);
    if (kernel == SEWALD_STOKESLET) return {4.0 / (kPi * L) * std::sqrt(Q / 3.0), 0.0, b};
    if (kernel == SEWALD_STRESSLET) return {4.0 / (3.0 * kPi * L) * std::sqrt(3.5 * Q), 1.0, b};
    if (kernel == SEWALD_ROTLET)
        return {std::sqrt(8.0 * xi * xi * Q / (3.0 * kPi * L * L * L)), -0.5, b};
    throw std::invalid_argument("unknown kernel");
}

ErrorModel rspace_model(int kernel, double xi, double L, double Q) {
    const double b = xi * xi;
    const double L3 = L * L * L;
    if (kernel == SEWALD_STOKESLET) return {std::sqrt(4.0 * Q / L3), 0.5, b};
    if (kernel == SEWALD_STRESSLET) return {std::sqrt(112.0 * Q * b * b / (9.0 * L3)), 1.5, b};
    if (kernel == SEWALD_ROTLET) return {std::sqrt(8.0 * Q / (3.0 * L3)), -0.5, b};
    throw std::invalid_argument("unknown kernel");
}

struct Cutoff {
    double value;
    bool clamped;
};

// Smallest cutoff on the decaying branch meeting tau (estimates.cpp:57-87):
// bracket, then safeguarded Newton on the log residual.
Cutoff invert_model(const ErrorModel& m, double tau, double floor_value) {
    const double log_tau = std::log(tau);
    double lo;
    if (m.a > 0.0) {
        lo = std::sqrt(m.a / (2.0 * m.b));
        if (m.at(lo) <= tau) return {lo, true};
    } else if (m.a == 0.0) {
        if (m.c <= tau) return {floor_value, true};
        return {std::sqrt(std::log(m.c / tau) / m.b), false};
    } else {
        lo = 1e-14;
        if (m.log_excess(lo, log_tau) <= 0.0) return {lo, true};
    }
    double hi = std::max(2.0 * lo, 1.0 / std::sqrt(m.b));
    for (int n = 0; m.log_excess(hi, log_tau) > 0.0; ++n) {
        hi *= 2.0;
        if (n > 200) throw std::runtime_error("cutoff bracket expansion failed");
    }
    double x = 0.5 * (lo + hi);
    for (int it = 0; it < 200; ++it) {
        const double g = m.log_excess(x, log_tau);
        if (std::abs(g) < 1e-14) break;
        if (g > 0.0)
            lo = x;
        else
            hi = x;
        const double slope = m.a / x - 2.0 * m.b * x;
        const double newton = x - g / slope;
        x = (newton > lo && newton < hi) ? newton : 0.5 * (lo + hi);
    }
    return {x, false};
}

double lambert_w0_impl(double t) {
    // Principal branch of w e^w = t (specfun.cpp:259-284 semantics): initial
    // guess by region, then Halley iterations.
    static const double inv_e = std::exp(-1.0);
    if (t < -inv_e - 1e-15) throw std::domain_error("lambert_w0 requires t >= -1/e");
    if (t == 0.0) return 0.0;
    double w;
    if (t < -0.32) {
        const double p = std::sqrt(std::max(2.0 * (std::exp(1.0) * t + 1.0), 0.0));
        w = -1.0 + p * (1.0 + p * (-1.0 / 3.0 + p * (11.0 / 72.0)));
        if (p < 1e-4) return w;
    } else if (t < 1.0) {
        w = t * (1.0 - t * (1.0 - 1.5 * t));
    } else {
        w = std::log(t);
        if (w > 1.0) w -= std::log(w);
    }
    for (int it = 0; it < 60; ++it) {
        const double ew = std::exp(w);
        const double f = w * ew - t;
        const double fp = ew * (w + 1.0);
        if (fp == 0.0) break;
        const double step = f / (fp - f * (w + 2.0) / (2.0 * (w + 1.0)));
        w -= step;
        if (std::fabs(step) <= 1e-16 * (1.0 + std::fabs(w))) break;
    }
    return w;
}

Cutoff kinf_for(int kernel, double xi, double tau, double L, double Q) {
    const ErrorModel m = kspace_model(kernel, xi, L, Q);
    if (kernel == SEWALD_ROTLET) {
        const double c2 = m.c * m.c;
        return {xi * std::sqrt(lambert_w0_impl(c2 * c2 / (xi * xi * std::pow(tau, 4.0)))), false};
    }
    return invert_model(m, tau, 2.0 * kPi / L);
}

double fitted_rms(int kernel, double L, double Q, double xi) {
    const double t = xi * L;
    if (kernel == SEWALD_STOKESLET) {
        const double fit = (1.0 + 1.323e-2 * t + 2.469e-4 * t * t) * std::exp(-5.205 / (t * t));
        return 1.8 * std::sqrt(Q) * fit / L;
    }
    if (kernel == SEWALD_STRESSLET) return 7.2 * std::sqrt(Q) * std::sqrt(t) / (L * L);
    if (kernel == SEWALD_ROTLET)
        return 2.4 * std::sqrt(Q) * std::sqrt(t) * std::exp(-11.60 / (t * t)) / (L * L);
    throw std::invalid_argument("unknown kernel");
}

int round_up_to(double x, int f) {
    const double q = std::ceil(x / f - 1e-9);
    return f * static_cast<int>(q < 1.0 ? 1.0 : q);
}

// Smallest factor >= s making every free padded length a multiple of f_m
// (estimates.cpp:91-101).
double grid_compatible_factor(double s, const sewald_params_c& g) {
    long common = 0;
    for (int i = g.d; i < 3; ++i) {
        if (g.M_ext[i] % g.f_m != 0)
            throw std::invalid_argument("extended grid sizes must be multiples of f_m");
        common = std::gcd(common, static_cast<long>(g.M_ext[i] / g.f_m));
    }
    if (common == 0) return std::max(s, 1.0);
    const double up = std::ceil(s * static_cast<double>(common) - 1e-9) / static_cast<double>(common);
    return std::max(up, 1.0);
}

// Upsampling factors and near-mode thresholds (estimates.cpp:180-209).
void upsampling_for(sewald_params_c& g, double tau, double U) {
    if (g.d < 0 || g.d > 2)
        throw std::invalid_argument("upsampling applies only to grids with free directions");
    must_be_positive(tau, "tau");
    must_be_positive(U, "U");
    const double R = free_truncation_radius(g);
    double Lmin = g.L_ext[g.d];
    for (int i = g.d + 1; i < 3; ++i) Lmin = std::min(Lmin, g.L_ext[i]);
    g.s0_raw = 1.0 + R / Lmin;
    g.s0 = grid_compatible_factor(std::ceil(10.0 * g.s0_raw - 1e-9) / 10.0, g);
    g.s_star = 1.0;
    g.s_star_raw = 1.0;
    g.k_star[0] = g.k_star[1] = g.k_star[2] = 0;
    if (g.d >= 1) {
        int Mext_min = g.M_ext[g.d];
        for (int i = g.d + 1; i < 3; ++i) Mext_min = std::min(Mext_min, g.M_ext[i]);
        const double lr = std::log(U / (2.0 * tau));
        int Mmax = 0;
        for (int i = 0; i < g.d; ++i) Mmax = std::max(Mmax, g.M[i]);
        if (Mext_min <= Mmax)
            throw std::runtime_error(
                "grid has no free-direction padding; near-axis upsampling is undefined");
        g.s_star_raw = static_cast<double>(Mmax) / Mext_min * (1.0 + lr / (2.0 * kPi));
        g.s_star = grid_compatible_factor(std::max(g.s_star_raw, 1.0), g);
        for (int i = 0; i < g.d; ++i) {
            const double v =
                static_cast<double>(g.M[i]) / (Mext_min - g.M[i]) * lr / (2.0 * kPi) - 1.0;
            g.k_star[i] = std::max(0, static_cast<int>(std::ceil(v - 1e-9)));
        }
    }
}

// (nu+1)x(nu+1) Vandermonde solve in long double with partial pivoting
// (window.cpp:21-56).
void vandermonde_solve(int n, const long double* x, long double* rhs, double* c) {
    std::vector<long double> A(static_cast<std::size_t>(n) * n);
    for (int r = 0; r < n; ++r) {
        long double pw = 1.0L;
        for (int k = 0; k < n; ++k) {
            A[static_cast<std::size_t>(r) * n + k] = pw;
            pw *= x[r];
        }
    }
    auto at = [&](int r, int k) -> long double& { return A[static_cast<std::size_t>(r) * n + k]; };
    for (int k = 0; k < n; ++k) {
        int best = k;
        for (int r = k + 1; r < n; ++r)
            if (std::fabs(static_cast<double>(at(r, k))) > std::fabs(static_cast<double>(at(best, k))))
                best = r;
        if (best != k) {
            for (int q = k; q < n; ++q) std::swap(at(k, q), at(best, q));
            std::swap(rhs[k], rhs[best]);
        }
        for (int r = k + 1; r < n; ++r) {
            const long double f = at(r, k) / at(k, k);
            for (int q = k; q < n; ++q) at(r, q) -= f * at(k, q);
            rhs[r] -= f * rhs[k];
        }
    }
    for (int r = n - 1; r >= 0; --r) {
        long double s = rhs[r];
        for (int q = r + 1; q < n; ++q) s -= at(r, q) * static_cast<long double>(c[q]);
        c[r] = static_cast<double>(s / at(r, r));
    }
}

}  // namespace

double bessel_i0(double t) { return std::cyl_bessel_i(0.0, std::fabs(t)); }

double lambert_w0(double t) { return lambert_w0_impl(t); }

void validate_window(const sewald_params_c& p) {
    if (p.P < 2 || p.P % 2 != 0)
        throw std::invalid_argument("window size P must be an even integer >= 2");
    if (!(p.win_h > 0.0)) throw std::invalid_argument("grid spacing must be positive");
    if (!(p.beta > 0.0)) throw std::invalid_argument("window shape beta must be positive");
    if (p.win_kind == SEWALD_WIN_TG && !(p.alpha > 0.0))
        throw std::invalid_argument("window shape alpha must be positive");
    if (p.win_kind == SEWALD_WIN_PKB && p.nu < 1)
        throw std::invalid_argument("polynomial degree must be at least 1");
    if (p.win_kind < 0 || p.win_kind > 2) throw std::invalid_argument("unknown window kind");
}

double kb_value(const sewald_params_c& p, double r) {
    const double aw = 0.5 * p.win_h * static_cast<double>(p.P);
    if (std::fabs(r) > aw) return 0.0;
    const double t = r / aw;
    const double arg = std::max(1.0 - t * t, 0.0);
    return bessel_i0(p.beta * std::sqrt(arg)) / bessel_i0(p.beta);
}

double kb_transform(const sewald_params_c& p, double k) {
    const double aw = 0.5 * p.win_h * static_cast<double>(p.P);
    const double s = p.beta * p.beta - k * k * aw * aw;
    const double front = 2.0 * aw / bessel_i0(p.beta);
    if (s > 1e-6) {
        const double q = std::sqrt(s);
        return front * std::sinh(q) / q;
    }
    if (s < -1e-6) {
        const double q = std::sqrt(-s);
        return front * std::sin(q) / q;
    }
    return front * (1.0 + s / 6.0 + s * s / 120.0);
}

double ug_transform(const sewald_params_c& p, double k) {
    const double aw = 0.5 * p.win_h * static_cast<double>(p.P);
    return std::sqrt(kPi / p.alpha) * aw * std::exp(-k * k * aw * aw / (4.0 * p.alpha));
}

std::vector<double> pkb_coefficients(const sewald_params_c& p) {
    validate_window(p);
    const int nu = p.nu;
    if (nu < 1) throw std::invalid_argument("polynomial degree must be at least 1");
    const int n = nu + 1;
    std::vector<double> coef(static_cast<std::size_t>(p.P) * n);
    std::vector<long double> x(n), y(n);
    for (int j = 0; j < n; ++j) x[j] = std::cos(static_cast<long double>(j) * kPi / nu);
    for (int l = -p.P / 2; l < p.P / 2; ++l) {
        const double left = l * p.win_h;
        const double mid = left + 0.5 * p.win_h;
        for (int j = 0; j < n; ++j) y[j] = kb_value(p, mid + 0.5 * p.win_h * static_cast<double>(x[j]));
        vandermonde_solve(n, x.data(), y.data(),
                          coef.data() + static_cast<std::size_t>(l + p.P / 2) * n);
    }
    return coef;
}

double window_value(const sewald_params_c& p, const std::vector<double>& pkb, double r) {
    const double aw = 0.5 * p.win_h * static_cast<double>(p.P);
    switch (p.win_kind) {
        case SEWALD_WIN_KB: return kb_value(p, r);
        case SEWALD_WIN_TG: {
            if (std::fabs(r) > aw) return 0.0;
            const double t = r / aw;
            return std::exp(-p.alpha * t * t);
        }
        default: {
            if (std::fabs(r) > 0.5 * p.win_h * p.P) return 0.0;
            int l = static_cast<int>(std::floor(r / p.win_h));
            l = std::clamp(l, -p.P / 2, p.P / 2 - 1);
            const double u = 2.0 * (r - l * p.win_h) / p.win_h - 1.0;
            const double* c = pkb.data() + static_cast<std::size_t>(l + p.P / 2) * (p.nu + 1);
            double acc = 0.0;
            for (int i = p.nu; i >= 0; --i) acc = c[i] + acc * u;
            return acc;
        }
    }
}

double window_transform(const sewald_params_c& p, double k) {
    return p.win_kind == SEWALD_WIN_TG ? ug_transform(p, k) : kb_transform(p, k);
}

void window_make(int kind, int P, double h, sewald_params_c& p) {
    p.win_kind = kind;
    p.P = P;
    p.win_h = h;
    p.beta = 2.5 * P;
    p.nu = std::min(P / 2 + 2, 10);
    p.alpha = 0.91 * 0.5 * kPi * P;
    validate_window(p);
}

void grid_build(const std::array<double, 3>& L, int d, double h_target, int P, int kernel, int f_m,
                sewald_params_c& g) {
    if (d < 0 || d > 3) throw std::invalid_argument("periodicity must be 0, 1, 2 or 3");
    if (!(h_target > 0.0)) throw std::invalid_argument("grid spacing must be positive");
    if (P < 2 || P % 2 != 0) throw std::invalid_argument("window size must be a positive even integer");
    if (f_m < 2 || f_m % 2 != 0)
        throw std::invalid_argument("grid granularity must be a positive even integer");
    for (double Li : L)
        if (!(Li > 0.0)) throw std::invalid_argument("cell lengths must be positive");
    g.d = d;
    g.f_m = f_m;
    for (int i = 0; i < 3; ++i) g.L[i] = L[i];
    g.M[0] = round_up_to(L[0] / h_target, f_m);
    g.h = L[0] / g.M[0];
    for (int i = 1; i < 3; ++i) {
        const double ratio = L[i] / g.h;
        if (i < d) {
            const int Mi = static_cast<int>(std::llround(ratio));
            if (Mi < 2 || Mi % 2 != 0 || std::abs(ratio - Mi) > 1e-9 * ratio)
                throw std::invalid_argument(
                    "periodic cell length must be an even multiple of the grid spacing");
            g.M[i] = Mi;
        } else {
            g.M[i] = round_up_to(ratio, f_m);
        }
    }
    // Free-axis padding: window support plus the screening tail, scaled by a
    // kernel- and periodicity-dependent factor (grid.cpp:11-24, :250-263).
    double lambda = 2.4;
    if (d == 0) lambda = kernel == SEWALD_STOKESLET ? 2.2 : (kernel == SEWALD_STRESSLET ? 2.4 : 1.5);
    const double theta = kernel == SEWALD_ROTLET ? 0 : 8;
    for (int i = 0; i < 3; ++i) {
        if (i < d) {
            g.M_ext[i] = g.M[i];
            g.L_ext[i] = L[i];
            g.pad[i] = 0.0;
        } else {
            const double raw = L[i] / g.h + P + (lambda - 1.0) * std::max<double>(P, theta);
            g.M_ext[i] = round_up_to(raw, f_m);
            g.L_ext[i] = g.h * g.M_ext[i];
            g.pad[i] = g.L_ext[i] - L[i];
        }
    }
}

double free_truncation_radius(const sewald_params_c& g) {
    switch (g.d) {
        case 0:
            return std::sqrt(g.L_ext[0] * g.L_ext[0] + g.L_ext[1] * g.L_ext[1] + g.L_ext[2] * g.L_ext[2]);
        case 1: return std::sqrt(g.L_ext[1] * g.L_ext[1] + g.L_ext[2] * g.L_ext[2]);
        case 2: return g.L_ext[2];
        default: throw std::invalid_argument("truncation radius applies to d in {0,1,2}");
    }
}

void select_parameters(int kernel, int d, const std::array<double, 3>& Lc, double Q, double xi,
                       double tol, bool relative, int f_m, int window, bool pollution_fix,
                       sewald_params_c& out, sewald_report_c* report) {
    if (d < 0 || d > 3) throw std::invalid_argument("periodicity must be 0, 1, 2 or 3");
    if (kernel < 0 || kernel > 2) throw std::invalid_argument("unknown kernel");
    must_be_positive(xi, "xi");
    must_be_positive(Q, "Q");
    const double L = std::cbrt(Lc[0] * Lc[1] * Lc[2]);

    sewald_report_c rep{};
    rep.U = fitted_rms(kernel, L, Q, xi);
    rep.tau_abs = relative ? tol * rep.U : tol;
    must_be_positive(rep.tau_abs, "tolerance");
    const double tau = rep.tau_abs;

    must_be_positive(tau, "tau");
    must_be_positive(L, "L");
    const Cutoff rc = invert_model(rspace_model(kernel, xi, L, Q), tau, 0.0);
    rep.rc_clamped = rc.clamped;

    const Cutoff kf = kinf_for(kernel, xi, tau, L, Q);
    rep.kinf = kf.value;
    rep.kinf_clamped = kf.clamped;
    rep.h_estimate = kPi / kf.value;

    // Window support from the gridding-error model 10 U e^{-2.5 P}
    // (estimates.cpp:158-171), reduced for the truncated Gaussian.
    int P_est;
    if (tau >= 10.0 * rep.U) {
        P_est = 2;
        rep.window_saturated = 1;
    } else {
        const double P_real = std::log(10.0 * rep.U / tau) / 2.5;
        P_est = std::max(2 * static_cast<int>(std::ceil(0.5 * P_real - 1e-9)), 2);
    }
    if (window == SEWALD_WIN_TG) {
        P_est = 2 * static_cast<int>(std::ceil(P_est / 1.2 - 1e-9));
        rep.tg_support_from_pkb = 1;
    }
    rep.P_estimate = P_est;

    double h_target = rep.h_estimate;
    int P_target = P_est;
    if (pollution_fix) {
        must_be_positive(h_target, "h");
        if (d == 0) {
            h_target = h_target / 1.1;
            P_target = P_target + 2;
        } else {
            h_target = h_target / 1.05;
            P_target = P_target + 4;
        }
    }
    rep.h_target = h_target;
    rep.P_target = P_target;
    const int P = 2 * ((P_target + 1) / 2);

    sewald_params_c p{};
    p.kind = kernel;
    p.d = d;
    p.xi = xi;
    p.rc = rc.value;
    grid_build(Lc, d, h_target, P, kernel, f_m, p);
    window_make(window, P, p.h, p);

    rep.fourier_trunc = kspace_model(kernel, xi, L, Q).at(kPi / p.h);
    rep.realspace_trunc = rspace_model(kernel, xi, L, Q).at(rc.value);
    const double P_eff = window == SEWALD_WIN_TG ? 0.6 * P : static_cast<double>(P);
    rep.window_err = 10.0 * rep.U * std::exp(-2.5 * P_eff);

    p.s0 = 1.0;
    p.s_star = 1.0;
    p.s0_raw = 1.0;
    p.s_star_raw = 1.0;
    if (d < 3) {
        p.R = free_truncation_radius(p);
        upsampling_for(p, tau, rep.U);
    }
    out = p;
    if (report) *report = rep;
}

static void positive_args(double xi, double x, double L, double Q, const char* xname) {
    must_be_positive(xi, "xi");
    must_be_positive(x, xname);
    must_be_positive(L, "L");
    must_be_positive(Q, "Q");
}

double fourier_trunc_error(int kernel, double xi, double kinf, double L, double Q) {
    positive_args(xi, kinf, L, Q, "kinf");
    return kspace_model(kernel, xi, L, Q).at(kinf);
}

double realspace_trunc_error(int kernel, double xi, double rc, double L, double Q) {
    positive_args(xi, rc, L, Q, "rc");
    return rspace_model(kernel, xi, L, Q).at(rc);
}

CutoffValue solve_kinf(int kernel, double xi, double tau, double L, double Q) {
    positive_args(xi, tau, L, Q, "tau");
    const Cutoff c = kinf_for(kernel, xi, tau, L, Q);
    return {c.value, c.clamped};
}

CutoffValue solve_rc(int kernel, double xi, double tau, double L, double Q) {
    positive_args(xi, tau, L, Q, "tau");
    const Cutoff c = invert_model(rspace_model(kernel, xi, L, Q), tau, 0.0);
    return {c.value, c.clamped};
}

double potential_rms(int kernel, double L, double Q, double xi) {
    must_be_positive(L, "L");
    must_be_positive(Q, "Q");
    must_be_positive(xi, "xi");
    return fitted_rms(kernel, L, Q, xi);
}

double window_error(double P, double U) {
    must_be_positive(U, "U");
    if (P < 0.0) throw std::invalid_argument("P must be nonnegative");
    return 10.0 * U * std::exp(-2.5 * P);
}

void solve_P(double tau, double U, int& P, bool& saturated) {
    must_be_positive(tau, "tau");
    must_be_positive(U, "U");
    saturated = tau >= 10.0 * U;
    if (saturated) {
        P = 2;
        return;
    }
    const double P_real = std::log(10.0 * U / tau) / 2.5;
    P = std::max(2 * static_cast<int>(std::ceil(0.5 * P_real - 1e-9)), 2);
}

void pollution_adjust(double h, int P, int d, double& h_out, int& P_out) {
    if (d < 0 || d > 3) throw std::invalid_argument("periodicity must be 0, 1, 2 or 3");
    must_be_positive(h, "h");
    h_out = d == 0 ? h / 1.1 : h / 1.05;
    P_out = d == 0 ? P + 2 : P + 4;
}

void upsampling_params(sewald_params_c& g, double tau, double U) { upsampling_for(g, tau, U); }

std::vector<double> wavenumbers(int n, double h) {
    std::vector<double> k(n);
    const double dk = 2.0 * kPi / (n * h);
    for (int m = 0; m < n; ++m) k[m] = dk * signed_mode(m, n);
    return k;
}

std::vector<double> window_hat_table(const sewald_params_c& p, const std::vector<double>& k) {
    const double w0 = window_transform(p, 0.0);
    std::vector<double> w(k.size());
    for (std::size_t m = 0; m < k.size(); ++m) {
        w[m] = window_transform(p, k[m]);
        if (!(std::isfinite(w[m]) && std::fabs(w[m]) > 1e-14 * std::fabs(w0)))
            throw std::runtime_error(
                "window transform vanishes at a retained mode; the window is too narrow for this grid");
    }
    return w;
}

int padded_length(double s, int m_ext) {
    const double v = s * m_ext;
    const long r = std::lround(v);
    if (std::fabs(v - static_cast<double>(r)) > 1e-6 || r < m_ext)
        throw std::invalid_argument("upsampling factor does not yield an integer grid size");
    return static_cast<int>(r);
}

}  // namespace sewald_b200
