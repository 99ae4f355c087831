// ORACLE TEST INFRASTRUCTURE — GSL subset shim (GSL is not installed here).
// E_n(x) = int_1^inf e^{-xt} t^{-n} dt, used at /root/reference/proj/src/specfun.cpp:118-122.
// E_1 from libstdc++ (E_1(x) = -Ei(-x)); higher orders by the upward recurrence
// E_{n+1}(x) = (e^{-x} - x E_n(x)) / n for moderate x, and by a continued
// fraction (Lentz) for x > 1 where the recurrence loses digits.
#pragma once
#include <cmath>
inline double gsl_sf_expint_En(int n, double x) {
    if (n == 0) return std::exp(-x) / x;
    if (x > 1.0) {
        // Continued fraction for E_n (modified Lentz), valid for x > 0.
        const double tiny = 1e-300;
        double b = x + n, c = 1.0 / tiny, d = 1.0 / b, h = d;
        for (int i = 1; i < 1000; ++i) {
            const double an = -static_cast<double>(i) * (n - 1 + i);
            b += 2.0;
            d = 1.0 / (an * d + b);
            c = b + an / c;
            const double del = c * d;
            h *= del;
            if (std::fabs(del - 1.0) < 1e-17) break;
        }
        return h * std::exp(-x);
    }
    double e = -std::expint(-x);
    for (int k = 1; k < n; ++k) e = (std::exp(-x) - x * e) / k;
    return e;
}
