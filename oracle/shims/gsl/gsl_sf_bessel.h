// ORACLE TEST INFRASTRUCTURE — GSL subset shim (GSL is not installed here).
// Bessel functions used at /root/reference/proj/src/specfun.cpp:100-116, mapped
// onto the C++17 special functions of libstdc++ (same published definitions:
// J_n, I_n, K_n of real argument). Pinned by the reference's own boundary
// tests /root/reference/proj/tests/test_specfun.cpp:31-72.
#pragma once
#include <cmath>
inline double gsl_sf_bessel_J0(double x) { return std::cyl_bessel_j(0.0, std::fabs(x)); }
inline double gsl_sf_bessel_J1(double x) {
    return x < 0.0 ? -std::cyl_bessel_j(1.0, -x) : std::cyl_bessel_j(1.0, x);
}
inline double gsl_sf_bessel_I0(double x) { return std::cyl_bessel_i(0.0, std::fabs(x)); }
inline double gsl_sf_bessel_K1(double x) { return std::cyl_bessel_k(1.0, x); }
inline double gsl_sf_bessel_Kn(int n, double x) { return std::cyl_bessel_k(static_cast<double>(n < 0 ? -n : n), x); }
