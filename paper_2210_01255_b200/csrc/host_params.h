// Host-side parameter layer of the B200 Spectral Ewald engine.
//
// Restates, operation for operation, the reference's host arithmetic so the
// parameters the GPU path consumes are bit-identical to the reference's:
//   select_parameters   /root/reference/proj/src/estimates.cpp:211-268
//   build_grid          /root/reference/proj/src/grid.cpp:35-77
//   WindowSpec::make    /root/reference/proj/src/window.cpp:76-86
//   pkb_build           /root/reference/proj/src/window.cpp:112-138
//   kb_eval / kb_hat    /root/reference/proj/src/window.cpp:88-110
//   tg_eval / ug_hat    /root/reference/proj/src/window.cpp:152-162
//   truncation_radius   /root/reference/proj/src/modified_kernels.cpp:65-72
// Errors are thrown as the reference's std exception types; the C-ABI layer
// maps them to status codes.
#pragma once

#include "../../include/sewald_gpu.h"

#include <array>
#include <vector>

namespace sewald_b200 {

constexpr double kPi = 3.14159265358979323846;

double bessel_i0(double t);
double lambert_w0(double t);  // principal branch (specfun.cpp:259-284)

// Window shape functions on the host (tables, PKB fitting, tests).
double kb_value(const sewald_params_c& p, double r);
double kb_transform(const sewald_params_c& p, double k);
double ug_transform(const sewald_params_c& p, double k);
double window_value(const sewald_params_c& p, const std::vector<double>& pkb, double r);
double window_transform(const sewald_params_c& p, double k);

std::vector<double> pkb_coefficients(const sewald_params_c& p);

void window_make(int kind, int P, double h, sewald_params_c& p);
void grid_build(const std::array<double, 3>& L, int d, double h_target, int P, int kernel,
                int f_m, sewald_params_c& p);
double free_truncation_radius(const sewald_params_c& p);

void select_parameters(int kernel, int d, const std::array<double, 3>& L, double Q, double xi,
                       double tol, bool relative, int f_m, int window, bool pollution_fix,
                       sewald_params_c& out, sewald_report_c* report);

// Signed DFT mode of index m on an axis of n points (fourier.cpp:28-30).
inline int signed_mode(int m, int n) { return m < (n + 1) / 2 ? m : m - n; }

// Wavenumbers 2 pi m/(n h) in DFT order (fourier.cpp:64-69).
std::vector<double> wavenumbers(int n, double h);
// w_hat at each wavenumber; throws runtime_error where it vanishes (fourier.cpp:71-81).
std::vector<double> window_hat_table(const sewald_params_c& p, const std::vector<double>& k);

// Integer padded length s * m_ext (fourier.cpp:92-98).
int padded_length(double s, int m_ext);

// FourierField geometry aft_forward produces (fourier.cpp:317-328) and the
// near rows of classify_rows (fourier.cpp:101-125); defined in aft.cu.
void aft_geometry(const sewald_params_c& p, int comps, sewald_fourier_geom_c& g, std::vector<int>* near_rows);

void validate_window(const sewald_params_c& p);

// Error-estimate layer of the reference (estimates.h:28-55), same checks and
// arithmetic as used inside select_parameters.
struct CutoffValue {
    double value;
    bool clamped;
};
double fourier_trunc_error(int kernel, double xi, double kinf, double L, double Q);
double realspace_trunc_error(int kernel, double xi, double rc, double L, double Q);
CutoffValue solve_kinf(int kernel, double xi, double tau, double L, double Q);
CutoffValue solve_rc(int kernel, double xi, double tau, double L, double Q);
double potential_rms(int kernel, double L, double Q, double xi);
double window_error(double P, double U);
void solve_P(double tau, double U, int& P, bool& saturated);
void pollution_adjust(double h, int P, int d, double& h_out, int& P_out);
// upsampling_params (estimates.cpp:180-209): fills g's s0 / s_star / k_star.
void upsampling_params(sewald_params_c& g, double tau, double U);

}  // namespace sewald_b200
