// sewald/specfun.h of the drop-in API (/root/reference/proj/include/sewald/specfun.h):
// the special functions of the host layer (Lambert W for the rotlet cutoff,
// the Bessel functions behind the windows and the 1P kernels, the error
// functions) and the analytic-module helpers (exponential integral,
// incomplete Bessel K, scaled erfc; csrc/specfun_host.cpp).
#pragma once

#include <array>

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

// adaptive quadrature controls of incomplete_bessel_K
struct QuadratureConfig {
    double rel_tol = 1e-13;
    int max_subdivisions = 200;
};

namespace detail {
// rational-form error functions (erfc = e^{-x^2} erfcx(x), erfcx rational)
double erf_rational(double x);
double erfc_rational(double x);
}  // namespace detail

// E_n(a) = int_1^inf e^{-a t} t^{-n} dt, n >= 1, a > 0
double exp_integral_E(int order, double a);

// K_nu(a, b) = int_1^inf e^{-a t - b/t} t^{-(nu+1)} dt; a, b >= 0 not both
// zero, a > 0 when nu <= 0
double incomplete_bessel_K(int order, double a, double b, const QuadratureConfig& cfg = {});

// {K_-1, K_0, K_1, K_2}(a, b) from one set of integrand evaluations
std::array<double, 4> incomplete_bessel_K_batch(double a, double b, const QuadratureConfig& cfg = {});

// e^{log_scale} erfc(z) without separate over/underflow of the factors
double exp_times_erfc(double log_scale, double z);

}  // namespace sewald
