// ORACLE TEST INFRASTRUCTURE — GSL subset shim (GSL is not installed here).
// Fixed-order Gauss-Legendre table, used only by the reference test
// /root/reference/proj/tests/test_realspace.cpp:196-219. Nodes by Newton
// iteration on the Legendre recurrence.
#pragma once
#include <cmath>
#include <cstddef>
#include <vector>
struct gsl_integration_glfixed_table { std::vector<double> x, w; };
inline gsl_integration_glfixed_table* gsl_integration_glfixed_table_alloc(std::size_t n) {
    auto* t = new gsl_integration_glfixed_table;
    t->x.resize(n);
    t->w.resize(n);
    for (std::size_t i = 0; i < n; ++i) {
        long double z = std::cos(M_PI * (i + 0.75) / (n + 0.5)), dp = 0;
        for (int it = 0; it < 100; ++it) {
            long double p1 = 1, p0 = 0;
            for (std::size_t j = 1; j <= n; ++j) {
                long double pm = p0;
                p0 = p1;
                p1 = ((2.0L * j - 1) * z * p0 - (j - 1.0L) * pm) / j;
            }
            dp = n * (z * p1 - p0) / (z * z - 1);
            long double dz = p1 / dp;
            z -= dz;
            if (std::fabs(static_cast<double>(dz)) < 1e-19) break;
        }
        t->x[i] = static_cast<double>(z);
        t->w[i] = static_cast<double>(2 / ((1 - z * z) * dp * dp));
    }
    return t;
}
inline int gsl_integration_glfixed_point(double a, double b, std::size_t i, double* xi, double* wi,
                                         const gsl_integration_glfixed_table* t) {
    *xi = 0.5 * (a + b) + 0.5 * (b - a) * t->x[i];
    *wi = 0.5 * (b - a) * t->w[i];
    return 0;
}
inline void gsl_integration_glfixed_table_free(gsl_integration_glfixed_table* t) { delete t; }
