// Special functions of the drop-in API (the subset of the reference's
// sewald/specfun.h that the hot path's host layer uses: error function,
// Bessel J0/J1/I0/K1/Kn and the principal Lambert W). The incomplete Bessel
// quadratures of the reference's analytic module are out of scope.
#pragma once

namespace sewald {

struct QuadratureConfig {
    double rel_tol = 1e-13;
    int max_subdivisions = 200;
};

double erf(double x);
double erfc(double x);
double bessel_J(int order, double t);
double bessel_I0(double t);
double bessel_K1(double t);
double bessel_Kn(int order, double t);
double lambert_w0(double t);

}  // namespace sewald
