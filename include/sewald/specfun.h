// sewald/specfun.h of the drop-in API: only the special functions the hot
// path's host layer needs (Lambert W for the rotlet cutoff, the Bessel
// functions behind the windows and the 1P kernels, the error functions).
// The incomplete Bessel quadratures of the reference's analytic module are
// not part of this library.
#pragma once

namespace sewald {

// principal branch of w e^w = y (y >= -1/e)
double lambert_w0(double y);

// modified Bessel K_n (x > 0), K_1, I_0 and Bessel J_n for n = 0, 1
double bessel_Kn(int n, double x);
double bessel_K1(double x);
double bessel_I0(double x);
double bessel_J(int n, double x);

double erfc(double z);
double erf(double z);

// Quadrature controls, kept for source compatibility of callers that pass them.
struct QuadratureConfig {
    double rel_tol = 1e-13;
    int max_subdivisions = 200;
};

}  // namespace sewald
