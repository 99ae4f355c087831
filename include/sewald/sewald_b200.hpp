// Drop-in C++ host API of the B200 Spectral Ewald engine.
//
// Source-compatible with the hot-path subset of the reference library's
// public API (namespace sewald; /root/reference/proj/include/sewald/*.h):
// the same type names, members and function signatures, so user code that
// selects parameters and evaluates the velocity compiles unchanged against
// this header and links libsewald_gpu.so instead. The numeric work runs in the
// sm_100a kernels behind include/sewald_gpu.h; errors surface as the
// reference's exception types (std::invalid_argument, std::domain_error,
// std::runtime_error).
//
// The per-file headers sewald/domain.h, estimates.h, grid.h, window.h,
// modified_kernels.h, fourier.h and realspace.h forward here.
#pragma once

#include <array>
#include <complex>
#include <cstddef>
#include <string>
#include <utility>
#include <vector>

namespace sewald {

// ---- value types (domain.h) ------------------------------------------------
using Vec3 = std::array<double, 3>;
using Mat3 = std::array<std::array<double, 3>, 3>;
using Ten3 = std::array<Mat3, 3>;  // t[j][l][m]
using cplx = std::complex<double>;
using CVec3 = std::array<cplx, 3>;
using CMat3 = std::array<CVec3, 3>;
using CTen3 = std::array<CMat3, 3>;

inline Vec3 operator+(const Vec3& a, const Vec3& b) { return {a[0] + b[0], a[1] + b[1], a[2] + b[2]}; }
inline Vec3 operator-(const Vec3& a, const Vec3& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
inline Vec3 operator*(double s, const Vec3& a) { return {s * a[0], s * a[1], s * a[2]}; }
inline Vec3& operator+=(Vec3& a, const Vec3& b) {
    for (int i = 0; i < 3; ++i) a[i] += b[i];
    return a;
}
inline double dot(const Vec3& a, const Vec3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
inline double norm2(const Vec3& a) { return dot(a, a); }

enum class Kernel { stokeslet, stresslet, rotlet };
enum class Screening { ewald, hasimoto };

Screening screening_of(Kernel kind);
const char* kernel_name(Kernel kind);
int strength_components(Kernel kind);
bool kernel_from_name(const std::string& name, Kernel& out);

struct Cell {
    std::array<double, 3> L{1.0, 1.0, 1.0};
    double volume() const { return L[0] * L[1] * L[2]; }
};

struct Periodicity {
    int d = 3;
    bool periodic(int axis) const { return axis < d; }
};

struct SourceSystem {
    Kernel kind = Kernel::stokeslet;
    Cell cell;
    int d = 3;
    std::vector<Vec3> x;   // positions
    std::vector<Vec3> f;   // strengths (stresslet: q)
    std::vector<Vec3> nu;  // stresslet orientations, empty otherwise
    std::size_t size() const { return x.size(); }
};

struct TargetSet {
    std::vector<Vec3> x;
    bool same_as_sources = false;
    static TargetSet from_sources(const SourceSystem& s) { return TargetSet{s.x, true}; }
};

void validate_system(const SourceSystem& s);
double source_quantity(const SourceSystem& s);
Vec3 wrap_position(const Vec3& x, const Cell& cell, int d);
Vec3 minimum_image(const Vec3& r, const Cell& cell, int d);

// ---- kernels (kernels.h): host evaluation of the kernel tensors ---------------
struct KernelTensor {
    int rank = 2;
    CMat3 m{};
    CTen3 t{};
};

struct KernelTensorR {
    int rank = 2;
    Mat3 m{};
    Ten3 t{};
};

KernelTensorR bare_kernel(Kernel kind, const Vec3& r);
double screening_hat(Screening skind, const Vec3& k, double xi);
KernelTensorR realspace_kernel(Kernel kind, const Vec3& r, double xi);
KernelTensor diffop_hat(Kernel kind, const Vec3& k);
KernelTensor fourier_kernel_hat(Kernel kind, const Vec3& k, double xi);
Vec3 self_term(Kernel kind, double xi, const Vec3& strength);
std::vector<Vec3> stresslet_zero_mode_3p(const TargetSet& targets, const SourceSystem& system);
Vec3 apply(const KernelTensorR& K, const Vec3& f);
Vec3 apply(const KernelTensorR& K, const Vec3& q, const Vec3& nu);
CVec3 apply(const KernelTensor& K, const Vec3& f);
CVec3 apply(const KernelTensor& K, const Vec3& q, const Vec3& nu);

// ---- window (window.h) -------------------------------------------------------
enum class WindowKind { kb, pkb, tg };
std::string window_kind_name(WindowKind kind);
WindowKind window_kind_from_name(const std::string& name);

struct WindowSpec {
    WindowKind kind = WindowKind::pkb;
    int P = 8;
    double h = 1.0;
    double beta = 20.0;
    int nu = 6;
    double alpha = 0.0;
    double half_width() const { return 0.5 * h * static_cast<double>(P); }
    static WindowSpec make(WindowKind kind, int P, double h);
};

struct PiecewisePolyWindow {
    int P = 0;
    int nu = 0;
    double h = 1.0;
    std::vector<double> coef;
};

double kb_eval(const WindowSpec& spec, double r);
double kb_hat(const WindowSpec& spec, double k);
PiecewisePolyWindow pkb_build(const WindowSpec& spec);
double pkb_eval(const PiecewisePolyWindow& win, double r);
double tg_eval(const WindowSpec& spec, double r);
double ug_hat(const WindowSpec& spec, double k);

class Window {
  public:
    explicit Window(const WindowSpec& spec);
    const WindowSpec& spec() const { return spec_; }
    double eval1d(double r) const;
    double hat1d(double k) const;

  private:
    WindowSpec spec_;
    std::vector<double> coef_;  // PKB table (P x (nu+1))
};

double tensor_window_eval(const Window& win, const Vec3& r);

// ---- grid (grid.h) -------------------------------------------------------------
struct GridSpec {
    int d = 3;
    double h = 0.0;
    std::array<int, 3> M{};
    std::array<int, 3> M_ext{};
    Vec3 L{};
    Vec3 L_ext{};
    Vec3 pad{};
    int f_m = 4;
    double kinf() const;
};

struct UpsamplingPlan {
    double s0 = 1.0;
    double s_star = 1.0;
    std::array<int, 3> k_star{};
    double s0_raw = 1.0;
    double s_star_raw = 1.0;
};

GridSpec build_grid(const Cell& cell, int d, double h_target, int P, Kernel kind, int f_m);

// ---- parameter selection (estimates.h) -------------------------------------------
struct ToleranceSpec {
    double value = 1e-8;
    bool relative = false;
    double absolute(double U) const { return relative ? value * U : value; }
};

struct CutoffResult {
    double value = 0.0;
    bool clamped = false;
};

struct WindowSizeResult {
    int P = 2;
    bool saturated = false;
};

double fourier_trunc_error(Kernel kind, double xi, double kinf, double L, double Q);
double realspace_trunc_error(Kernel kind, double xi, double rc, double L, double Q);
CutoffResult solve_kinf(Kernel kind, double xi, double tau, double L, double Q);
CutoffResult solve_rc(Kernel kind, double xi, double tau, double L, double Q);
double potential_rms(Kernel kind, double L, double Q, double xi);
double window_error(double P, double U);
WindowSizeResult solve_P(double tau, double U);
std::pair<double, int> pollution_adjust(double h, int P, int d);
UpsamplingPlan upsampling_params(const GridSpec& grid, double tau, double U);

struct EwaldParams {
    Kernel kind = Kernel::stokeslet;
    int d = 3;
    double xi = 1.0;
    double rc = 0.0;
    double R = 0.0;
    GridSpec grid;
    WindowSpec window;
    UpsamplingPlan upsampling;
};

struct EstimateReport {
    double tau_abs = 0.0;
    double U = 0.0;
    double kinf = 0.0;
    double fourier_trunc = 0.0;
    double realspace_trunc = 0.0;
    double window_err = 0.0;
    double h_estimate = 0.0;
    int P_estimate = 0;
    double h_target = 0.0;
    int P_target = 0;
    bool rc_clamped = false;
    bool kinf_clamped = false;
    bool window_saturated = false;
    bool tg_support_from_pkb = false;
};

struct SelectionOptions {
    int f_m = 4;
    WindowKind window = WindowKind::pkb;
    bool pollution_fix = true;
};

struct ParameterSelection {
    EwaldParams params;
    EstimateReport report;
};

ParameterSelection select_parameters(Kernel kind, int d, const Cell& cell, double Q, double xi,
                                     const ToleranceSpec& tol, const SelectionOptions& opt = {});

// ---- modified kernels (modified_kernels.h) ----------------------------------------
struct ModifiedKernelSpec {
    Kernel kind = Kernel::stokeslet;
    int d = 0;
    double R = 1.0;
    double a_B = 0.0;
    double b_B = 0.0;
    double ell_H = 1.0;
    double ell_B = 1.0;
    double c_B = 0.0;
    static ModifiedKernelSpec optimal(Kernel kind, int d, double R);
};

double truncation_radius(const std::array<double, 3>& L_ext, int d);
double harmonic_hat_trunc_0p(double kappa, double R);
double biharmonic_hat_trunc_0p(double kappa, double R, double a_B, double b_B);
double harmonic_hat_trunc_1p(double kappa, double R, double ell_H);
double biharmonic_hat_trunc_1p(double kappa, double R, double ell_B, double c_B);
cplx Z_hat_trunc_2p(double kappa3, double R);
double H2p_hat_trunc(double kappa3, double R);
KernelTensor modified_kernel_hat(const ModifiedKernelSpec& spec, const Vec3& k);
Vec3 gauge_flow_correction(const ModifiedKernelSpec& spec, const SourceSystem& system);

// ---- Fourier part (fourier.h) ----------------------------------------------------
struct RealField {
    std::array<int, 3> n{};
    int comps = 0;
    std::vector<double> v;
    static RealField zeros(const std::array<int, 3>& n, int comps);
    double& at(int c, int i, int j, int k) {
        return v[((static_cast<long>(c) * n[0] + i) * n[1] + j) * n[2] + k];
    }
    double at(int c, int i, int j, int k) const {
        return v[((static_cast<long>(c) * n[0] + i) * n[1] + j) * n[2] + k];
    }
};

// Mixed-space coefficients (fourier.h:30-46): far / near / zero per mode class.
struct FourierField {
    int d = 3;
    int comps = 0;
    std::array<int, 3> n_per{1, 1, 1};
    std::array<int, 3> n_far{1, 1, 1};
    std::array<int, 3> n_near{1, 1, 1};
    std::array<int, 3> n_zero{1, 1, 1};
    std::vector<cplx> far;
    std::vector<int> near_rows;
    std::vector<cplx> near;
    std::vector<cplx> zero;
};

// D = 0 kernel table (fourier.h:52-57). se_fourier_potential builds and caches
// it on the device per parameter set unless SePipelineOptions::table supplies
// one (then that table is used, as in the reference); precompute_0p() returns
// it on the host.
struct PrecomputedKernel0P {
    Kernel kind = Kernel::stokeslet;
    std::array<int, 3> n{};
    double R = 0.0;
    std::vector<cplx> table;
};

struct SePipelineOptions {
    bool precompute_0p = true;
    const PrecomputedKernel0P* table = nullptr;
};

RealField spread(const SourceSystem& system, const GridSpec& grid, const Window& window);
FourierField aft_forward(const RealField& field, const GridSpec& grid, const UpsamplingPlan& plan);
RealField aft_inverse(const FourierField& field, const GridSpec& grid, const UpsamplingPlan& plan);
FourierField scale(const FourierField& field, const ModifiedKernelSpec& spec, double xi, const Window& window,
                   const GridSpec& grid);
FourierField scale(const FourierField& field, const PrecomputedKernel0P& pre, double xi, const Window& window,
                   const GridSpec& grid);
PrecomputedKernel0P precompute_0p(Kernel kind, const GridSpec& grid, double R);

namespace detail {
double mollifier_taper(double t);  // fourier.cpp:222-225
}  // namespace detail
std::vector<Vec3> gather(const RealField& field, const GridSpec& grid, const Window& window,
                         const TargetSet& targets);
std::vector<Vec3> se_fourier_potential(const SourceSystem& system, const TargetSet& targets,
                                       const EwaldParams& params, const SePipelineOptions& opt = {});

// ---- real space and full potential (realspace.h) -----------------------------------
// Host cell list of the reference's real-space sum (realspace.cpp:97-164); the
// device path builds its own finer grid, this one serves callers and tests.
struct CellList {
    double rc = 0.0;
    int d = 3;
    Cell cell;
    std::array<int, 3> n{1, 1, 1};
    std::array<double, 3> width{};
    std::array<double, 3> origin{};
    std::array<int, 3> reach{1, 1, 1};
    std::vector<std::size_t> offset;
    std::vector<std::size_t> index;
    std::vector<Vec3> folded;
    std::size_t bucket_count() const { return offset.empty() ? 0 : offset.size() - 1; }
};

CellList build_cell_list(const SourceSystem& system, double rc);
std::vector<Vec3> realspace_potential(const SourceSystem& system, const TargetSet& targets,
                                      double xi, double rc, bool starred, int n_threads = 1);
std::vector<Vec3> full_potential(const SourceSystem& system, const TargetSet& targets,
                                 const EwaldParams& params, const SePipelineOptions& opt = {});

// ---- B200 extension (not in the reference API) -------------------------------------

// ---- analytic oracles (SPEC.md module `reference`; the
// reference ships it as a stub, proj/src/reference.cpp:1). Slow direct sums
// on the GPU for validating the fast path (include/sewald_gpu.h "analytic
// oracles"); periodic sums over -kmax_i <= j <= kmax_i - 1 per periodic axis.
std::vector<Vec3> direct_sum_0p(const SourceSystem& system, const TargetSet& targets, bool starred);
std::vector<Vec3> direct_ewald_fourier_3p(const SourceSystem& system, const TargetSet& targets, double xi,
                                          const std::array<int, 3>& kmax);
std::vector<Vec3> fourier_reference_potential(const SourceSystem& system, const TargetSet& targets, double xi,
                                              const std::array<int, 3>& kmax);
// kmax per axis with the omitted modes below e^{-39} of the largest.
std::array<int, 3> oracle_kmax(double xi, const Cell& cell);
double rms_error(const std::vector<Vec3>& u, const std::vector<Vec3>& u_ref);
double rel_rms_error(const std::vector<Vec3>& u, const std::vector<Vec3>& u_ref);

namespace b200 {
// full_potential / se_fourier_potential on these GPUs of this node (one
// process, NVLink peer memory; include/sewald_gpu.h sewald_gpu_multi_*).
// Fewer than two entries: one GPU (the default; SEWALD_DEVICES="0,1,..."
// sets the initial list).
void use_devices(const std::vector<int>& devices);
}  // namespace b200

}  // namespace sewald
