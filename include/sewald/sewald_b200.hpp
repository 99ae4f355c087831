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
using cplx = std::complex<double>;

enum class Kernel { stokeslet, stresslet, rotlet };
enum class Screening { ewald, hasimoto };

Screening screening_of(Kernel kind);
const char* kernel_name(Kernel kind);
int strength_components(Kernel kind);

struct Cell {
    std::array<double, 3> L{1.0, 1.0, 1.0};
    double volume() const { return L[0] * L[1] * L[2]; }
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

// ---- window (window.h) -------------------------------------------------------
enum class WindowKind { kb, pkb, tg };

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
// it on the device per parameter set; precompute_0p() returns it on the host
// for the stage API.
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
std::vector<Vec3> gather(const RealField& field, const GridSpec& grid, const Window& window,
                         const TargetSet& targets);
std::vector<Vec3> se_fourier_potential(const SourceSystem& system, const TargetSet& targets,
                                       const EwaldParams& params, const SePipelineOptions& opt = {});

// ---- real space and full potential (realspace.h) -----------------------------------
std::vector<Vec3> realspace_potential(const SourceSystem& system, const TargetSet& targets,
                                      double xi, double rc, bool starred, int n_threads = 1);
std::vector<Vec3> full_potential(const SourceSystem& system, const TargetSet& targets,
                                 const EwaldParams& params, const SePipelineOptions& opt = {});

}  // namespace sewald
