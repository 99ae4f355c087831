// C-ABI of the host parameter layer (no GPU needed). Each call restates a
// reference host function; see host_params.h for the citations.
#include "host_params.h"

#include <array>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>

using namespace sewald_b200;

namespace {

thread_local std::string g_err;

template <class F>
int host_guard(F&& fn) {
    try {
        fn();
        return SEWALD_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return SEWALD_EINVAL;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return SEWALD_EDOMAIN;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SEWALD_ERUNTIME;
    }
}

}  // namespace

extern "C" {

const char* sewald_last_error(void) { return g_err.c_str(); }

int sewald_select_parameters(int kind, int d, const double L[3], double Q, double xi,
                             double tol_value, int tol_relative, int f_m, int window_kind,
                             int pollution_fix, sewald_params_c* out, sewald_report_c* report) {
    if (!out || !L) return SEWALD_EINVAL;
    return host_guard([&] {
        select_parameters(kind, d, {L[0], L[1], L[2]}, Q, xi, tol_value, tol_relative != 0, f_m,
                          window_kind, pollution_fix != 0, *out, report);
    });
}

int sewald_window_make(int window_kind, int P, double h, sewald_params_c* p) {
    if (!p) return SEWALD_EINVAL;
    return host_guard([&] { window_make(window_kind, P, h, *p); });
}

int sewald_build_grid(const double L[3], int d, double h_target, int P, int kind, int f_m,
                      sewald_params_c* p) {
    if (!p || !L) return SEWALD_EINVAL;
    return host_guard([&] { grid_build({L[0], L[1], L[2]}, d, h_target, P, kind, f_m, *p); });
}

int sewald_pkb_coefficients(const sewald_params_c* p, double* coef_out) {
    if (!p || !coef_out) return SEWALD_EINVAL;
    return host_guard([&] {
        const std::vector<double> c = pkb_coefficients(*p);
        std::memcpy(coef_out, c.data(), sizeof(double) * c.size());
    });
}

int sewald_window_eval(const sewald_params_c* p, const double* r, int64_t n, double* out) {
    if (!p) return SEWALD_EINVAL;
    return host_guard([&] {
        validate_window(*p);
        std::vector<double> pkb;
        if (p->win_kind == SEWALD_WIN_PKB) pkb = pkb_coefficients(*p);
        for (int64_t i = 0; i < n; ++i) out[i] = window_value(*p, pkb, r[i]);
    });
}

int sewald_window_hat(const sewald_params_c* p, const double* k, int64_t n, double* out) {
    if (!p) return SEWALD_EINVAL;
    return host_guard([&] {
        validate_window(*p);
        for (int64_t i = 0; i < n; ++i) out[i] = window_transform(*p, k[i]);
    });
}

int sewald_modspec_optimal(int kind, int d, double R, sewald_modspec_c* out) {
    if (!out) return SEWALD_EINVAL;
    return host_guard([&] {
        if (kind < 0 || kind > 2) throw std::invalid_argument("unknown kernel");
        *out = sewald_modspec_c{kind, d, R, -0.5 * R, -0.5 / R, R, R * std::sqrt(M_E), -0.5 * R * R};
    });
}

int sewald_aft_geometry(const sewald_params_c* p, int comps, sewald_fourier_geom_c* g, int32_t* near_rows_out) {
    if (!p || !g) return SEWALD_EINVAL;
    return host_guard([&] {
        std::vector<int> rows;
        aft_geometry(*p, comps, *g, &rows);
        if (near_rows_out)
            for (size_t i = 0; i < rows.size(); ++i) near_rows_out[i] = rows[i];
    });
}

double sewald_source_quantity(int kind, const double* f, const double* nu, int64_t N) {
    double q = 0.0;
    for (int64_t n = 0; n < N; ++n) {
        const double* a = f + 3 * n;
        const double fa = a[0] * a[0] + a[1] * a[1] + a[2] * a[2];
        if (kind == SEWALD_STRESSLET) {
            const double* b = nu + 3 * n;
            q += fa * (b[0] * b[0] + b[1] * b[1] + b[2] * b[2]);
        } else {
            q += fa;
        }
    }
    return q;
}

}  // extern "C"
