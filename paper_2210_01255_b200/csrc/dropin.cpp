// Drop-in C++ host API (include/sewald/sewald_b200.hpp) on top of the C-ABI.
// Each function keeps the reference signature and semantics
// (/root/reference/proj/include/sewald/*.h) and forwards the numeric work to
// the device engine through sewald_gpu.h; status codes are rethrown as the
// reference's exception types.
#include "../../include/sewald/sewald_b200.hpp"
#include "../../include/sewald/specfun.h"

#include "../../include/sewald_gpu.h"
#include "host_params.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <future>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>

namespace sewald {

namespace {

std::mutex g_mu;

sewald_gpu_ctx* context() {
    static sewald_gpu_ctx* ctx = [] {
        sewald_gpu_ctx* c = nullptr;
        if (sewald_gpu_create(0, &c) != SEWALD_OK)
            throw std::runtime_error("sewald: no usable CUDA device for the B200 engine");
        return c;
    }();
    return ctx;
}

// Several GPUs for full_potential / se_fourier_potential: sewald::b200::use_devices
// or SEWALD_DEVICES="0,1,2,3" (read once); one device otherwise.
std::vector<int> g_devices;
bool g_devices_set = false;
sewald_gpu_multi* g_multi = nullptr;

std::vector<int> env_devices() {
    std::vector<int> d;
    const char* e = getenv("SEWALD_DEVICES");
    if (!e) return d;
    std::string s(e);
    size_t pos = 0;
    while (pos < s.size()) {
        size_t q = s.find(',', pos);
        if (q == std::string::npos) q = s.size();
        if (q > pos) d.push_back(std::atoi(s.substr(pos, q - pos).c_str()));
        pos = q + 1;
    }
    return d;
}

sewald_gpu_multi* multi_context() {
    if (!g_devices_set) {
        g_devices = env_devices();
        g_devices_set = true;
    }
    if (g_devices.size() < 2) return nullptr;
    if (!g_multi) {
        if (sewald_gpu_multi_create(static_cast<int>(g_devices.size()), g_devices.data(), &g_multi) != SEWALD_OK)
            throw std::runtime_error("sewald: cannot open the multi-GPU context (peer access between the devices?)");
    }
    return g_multi;
}

void rethrow(int rc, const char* msg) {
    switch (rc) {
        case SEWALD_OK: return;
        case SEWALD_EINVAL: throw std::invalid_argument(msg);
        case SEWALD_EDOMAIN: throw std::domain_error(msg);
        default: throw std::runtime_error(msg);
    }
}

void check_ctx(int rc) { rethrow(rc, sewald_gpu_last_error(context())); }
void check_host(int rc) { rethrow(rc, sewald_last_error()); }

int kernel_id(Kernel k) {
    return k == Kernel::stokeslet ? SEWALD_STOKESLET : (k == Kernel::stresslet ? SEWALD_STRESSLET : SEWALD_ROTLET);
}
Kernel kernel_of(int k) {
    return k == SEWALD_STOKESLET ? Kernel::stokeslet : (k == SEWALD_STRESSLET ? Kernel::stresslet : Kernel::rotlet);
}
int window_id(WindowKind w) { return w == WindowKind::kb ? SEWALD_WIN_KB : (w == WindowKind::pkb ? SEWALD_WIN_PKB : SEWALD_WIN_TG); }
WindowKind window_of(int w) {
    return w == SEWALD_WIN_KB ? WindowKind::kb : (w == SEWALD_WIN_PKB ? WindowKind::pkb : WindowKind::tg);
}

void put_window(const WindowSpec& w, sewald_params_c& p) {
    p.win_kind = window_id(w.kind);
    p.P = w.P;
    p.win_h = w.h;
    p.beta = w.beta;
    p.nu = w.nu;
    p.alpha = w.alpha;
}

void put_grid(const GridSpec& g, sewald_params_c& p) {
    p.h = g.h;
    p.f_m = g.f_m;
    for (int i = 0; i < 3; ++i) {
        p.M[i] = g.M[i];
        p.M_ext[i] = g.M_ext[i];
        p.L[i] = g.L[i];
        p.L_ext[i] = g.L_ext[i];
        p.pad[i] = g.pad[i];
    }
}

sewald_params_c to_c(const EwaldParams& e) {
    sewald_params_c p{};
    p.kind = kernel_id(e.kind);
    p.d = e.d;
    p.xi = e.xi;
    p.rc = e.rc;
    p.R = e.R;
    put_grid(e.grid, p);
    put_window(e.window, p);
    p.s0 = e.upsampling.s0;
    p.s_star = e.upsampling.s_star;
    p.s0_raw = e.upsampling.s0_raw;
    p.s_star_raw = e.upsampling.s_star_raw;
    for (int i = 0; i < 3; ++i) p.k_star[i] = e.upsampling.k_star[i];
    return p;
}

EwaldParams from_c(const sewald_params_c& p) {
    EwaldParams e;
    e.kind = kernel_of(p.kind);
    e.d = p.d;
    e.xi = p.xi;
    e.rc = p.rc;
    e.R = p.R;
    e.grid.d = p.d;
    e.grid.h = p.h;
    e.grid.f_m = p.f_m;
    for (int i = 0; i < 3; ++i) {
        e.grid.M[i] = p.M[i];
        e.grid.M_ext[i] = p.M_ext[i];
        e.grid.L[i] = p.L[i];
        e.grid.L_ext[i] = p.L_ext[i];
        e.grid.pad[i] = p.pad[i];
        e.upsampling.k_star[i] = p.k_star[i];
    }
    e.window.kind = window_of(p.win_kind);
    e.window.P = p.P;
    e.window.h = p.win_h;
    e.window.beta = p.beta;
    e.window.nu = p.nu;
    e.window.alpha = p.alpha;
    e.upsampling.s0 = p.s0;
    e.upsampling.s_star = p.s_star;
    e.upsampling.s0_raw = p.s0_raw;
    e.upsampling.s_star_raw = p.s_star_raw;
    return e;
}

const double* D(const std::vector<Vec3>& v) { return v.empty() ? nullptr : reinterpret_cast<const double*>(v.data()); }

}  // namespace

// ---- domain ---------------------------------------------------------------------
Screening screening_of(Kernel kind) { return kind == Kernel::rotlet ? Screening::ewald : Screening::hasimoto; }

const char* kernel_name(Kernel kind) {
    return kind == Kernel::stokeslet ? "stokeslet" : (kind == Kernel::stresslet ? "stresslet" : "rotlet");
}

int strength_components(Kernel kind) { return kind == Kernel::stresslet ? 9 : 3; }

void validate_system(const SourceSystem& s) {
    if (s.d < 0 || s.d > 3) throw std::invalid_argument("periodicity d must be in 0..3");
    for (double Li : s.cell.L)
        if (!(Li > 0.0)) throw std::invalid_argument("cell lengths must be positive");
    if (s.f.size() != s.x.size()) throw std::invalid_argument("strength count does not match position count");
    if (s.kind == Kernel::stresslet) {
        if (s.nu.size() != s.x.size()) throw std::invalid_argument("stresslet needs one orientation per source");
    } else if (!s.nu.empty()) {
        throw std::invalid_argument("orientations only apply to the stresslet");
    }
    // non-finite positions: checked on the device by the first stage that
    // reads them (finite_check_kernel), same std::invalid_argument message
}

double source_quantity(const SourceSystem& s) {
    return sewald_source_quantity(kernel_id(s.kind), D(s.f), s.kind == Kernel::stresslet ? D(s.nu) : nullptr,
                                  static_cast<int64_t>(s.f.size()));
}

Vec3 wrap_position(const Vec3& x, const Cell& cell, int d) {
    Vec3 y = x;
    for (int i = 0; i < d; ++i) {
        y[i] = std::fmod(y[i], cell.L[i]);
        if (y[i] < 0.0) y[i] += cell.L[i];
    }
    return y;
}

// ---- special functions (specfun.h subset) ------------------------------------------------
double erf(double x) { return std::erf(x); }
double erfc(double x) { return std::erfc(x); }

double bessel_J(int order, double t) {
    if (order == 0) return ::j0(t);
    if (order == 1) return ::j1(t);
    throw std::invalid_argument("bessel_J supports orders 0 and 1");
}

double bessel_I0(double t) { return sewald_b200::bessel_i0(t); }

double bessel_K1(double t) {
    if (!(t > 0.0)) throw std::domain_error("bessel_K1 requires t > 0");
    return std::cyl_bessel_k(1.0, t);
}

double bessel_Kn(int order, double t) {
    if (!(t > 0.0)) throw std::domain_error("bessel_Kn requires t > 0");
    return std::cyl_bessel_k(static_cast<double>(order < 0 ? -order : order), t);
}

double lambert_w0(double t) { return sewald_b200::lambert_w0(t); }

bool kernel_from_name(const std::string& name, Kernel& out) {
    for (Kernel k : {Kernel::stokeslet, Kernel::stresslet, Kernel::rotlet})
        if (name == kernel_name(k)) {
            out = k;
            return true;
        }
    return false;
}

Vec3 minimum_image(const Vec3& r, const Cell& cell, int d) {
    Vec3 y = r;
    for (int i = 0; i < d; ++i) y[i] -= cell.L[i] * std::floor(y[i] / cell.L[i] + 0.5);
    return y;
}

// ---- estimates (estimates.h:28-55) ----------------------------------------------------
double fourier_trunc_error(Kernel kind, double xi, double kinf, double L, double Q) {
    return sewald_b200::fourier_trunc_error(kernel_id(kind), xi, kinf, L, Q);
}

double realspace_trunc_error(Kernel kind, double xi, double rc, double L, double Q) {
    return sewald_b200::realspace_trunc_error(kernel_id(kind), xi, rc, L, Q);
}

CutoffResult solve_kinf(Kernel kind, double xi, double tau, double L, double Q) {
    const auto c = sewald_b200::solve_kinf(kernel_id(kind), xi, tau, L, Q);
    return {c.value, c.clamped};
}

CutoffResult solve_rc(Kernel kind, double xi, double tau, double L, double Q) {
    const auto c = sewald_b200::solve_rc(kernel_id(kind), xi, tau, L, Q);
    return {c.value, c.clamped};
}

double potential_rms(Kernel kind, double L, double Q, double xi) {
    return sewald_b200::potential_rms(kernel_id(kind), L, Q, xi);
}

double window_error(double P, double U) { return sewald_b200::window_error(P, U); }

WindowSizeResult solve_P(double tau, double U) {
    WindowSizeResult r;
    sewald_b200::solve_P(tau, U, r.P, r.saturated);
    return r;
}

std::pair<double, int> pollution_adjust(double h, int P, int d) {
    std::pair<double, int> r;
    sewald_b200::pollution_adjust(h, P, d, r.first, r.second);
    return r;
}

UpsamplingPlan upsampling_params(const GridSpec& grid, double tau, double U) {
    EwaldParams e;
    e.d = grid.d;
    e.grid = grid;
    sewald_params_c p = to_c(e);
    sewald_b200::upsampling_params(p, tau, U);
    return from_c(p).upsampling;
}

// ---- window / grid ------------------------------------------------------------------
std::string window_kind_name(WindowKind kind) {
    return kind == WindowKind::kb ? "kb" : (kind == WindowKind::tg ? "tg" : "pkb");
}

WindowKind window_kind_from_name(const std::string& name) {
    if (name == "kb") return WindowKind::kb;
    if (name == "pkb") return WindowKind::pkb;
    if (name == "tg") return WindowKind::tg;
    throw std::invalid_argument("unknown window kind: " + name);
}

double kb_eval(const WindowSpec& spec, double r) {
    sewald_params_c p{};
    put_window(spec, p);
    return sewald_b200::kb_value(p, r);
}

double kb_hat(const WindowSpec& spec, double k) {
    sewald_params_c p{};
    put_window(spec, p);
    return sewald_b200::kb_transform(p, k);
}

double ug_hat(const WindowSpec& spec, double k) {
    sewald_params_c p{};
    put_window(spec, p);
    return sewald_b200::ug_transform(p, k);
}

double tg_eval(const WindowSpec& spec, double r) {
    WindowSpec t = spec;
    t.kind = WindowKind::tg;
    sewald_params_c p{};
    put_window(t, p);
    return sewald_b200::window_value(p, {}, r);
}

PiecewisePolyWindow pkb_build(const WindowSpec& spec) {
    sewald_params_c p{};
    put_window(spec, p);
    sewald_b200::validate_window(p);
    if (spec.nu < 1) throw std::invalid_argument("polynomial degree must be at least 1");
    PiecewisePolyWindow w;
    w.P = spec.P;
    w.nu = spec.nu;
    w.h = spec.h;
    w.coef = sewald_b200::pkb_coefficients(p);
    return w;
}

double pkb_eval(const PiecewisePolyWindow& win, double r) {
    sewald_params_c p{};
    p.win_kind = SEWALD_WIN_PKB;
    p.P = win.P;
    p.nu = win.nu;
    p.win_h = win.h;
    return sewald_b200::window_value(p, win.coef, r);
}

double tensor_window_eval(const Window& win, const Vec3& r) {
    return win.eval1d(r[0]) * win.eval1d(r[1]) * win.eval1d(r[2]);
}

// ---- window / grid ------------------------------------------------------------------
WindowSpec WindowSpec::make(WindowKind kind, int P, double h) {
    sewald_params_c p{};
    check_host(sewald_window_make(window_id(kind), P, h, &p));
    return from_c(p).window;
}

Window::Window(const WindowSpec& spec) : spec_(spec) {
    sewald_params_c p{};
    put_window(spec, p);
    sewald_b200::validate_window(p);
    if (spec.kind == WindowKind::pkb) coef_ = sewald_b200::pkb_coefficients(p);
}

double Window::eval1d(double r) const {
    sewald_params_c p{};
    put_window(spec_, p);
    return sewald_b200::window_value(p, coef_, r);
}

double Window::hat1d(double k) const {
    sewald_params_c p{};
    put_window(spec_, p);
    return sewald_b200::window_transform(p, k);
}

double GridSpec::kinf() const { return sewald_b200::kPi / h; }

GridSpec build_grid(const Cell& cell, int d, double h_target, int P, Kernel kind, int f_m) {
    sewald_params_c p{};
    check_host(sewald_build_grid(cell.L.data(), d, h_target, P, kernel_id(kind), f_m, &p));
    return from_c(p).grid;
}

ParameterSelection select_parameters(Kernel kind, int d, const Cell& cell, double Q, double xi,
                                     const ToleranceSpec& tol, const SelectionOptions& opt) {
    sewald_params_c p{};
    sewald_report_c r{};
    check_host(sewald_select_parameters(kernel_id(kind), d, cell.L.data(), Q, xi, tol.value, tol.relative ? 1 : 0,
                                        opt.f_m, window_id(opt.window), opt.pollution_fix ? 1 : 0, &p, &r));
    ParameterSelection out;
    out.params = from_c(p);
    EstimateReport& e = out.report;
    e.tau_abs = r.tau_abs;
    e.U = r.U;
    e.kinf = r.kinf;
    e.fourier_trunc = r.fourier_trunc;
    e.realspace_trunc = r.realspace_trunc;
    e.window_err = r.window_err;
    e.h_estimate = r.h_estimate;
    e.P_estimate = r.P_estimate;
    e.h_target = r.h_target;
    e.P_target = r.P_target;
    e.rc_clamped = r.rc_clamped != 0;
    e.kinf_clamped = r.kinf_clamped != 0;
    e.window_saturated = r.window_saturated != 0;
    e.tg_support_from_pkb = r.tg_support_from_pkb != 0;
    return out;
}

// ---- Fourier / real space / full ---------------------------------------------------------
RealField RealField::zeros(const std::array<int, 3>& n, int comps) {
    RealField f;
    f.n = n;
    f.comps = comps;
    f.v.assign(static_cast<std::size_t>(comps) * n[0] * n[1] * n[2], 0.0);
    return f;
}

RealField spread(const SourceSystem& system, const GridSpec& grid, const Window& window) {
    validate_system(system);
    if (std::fabs(window.spec().h - grid.h) > 1e-12 * grid.h)
        throw std::invalid_argument("window was built for a different grid spacing");
    if (system.d != grid.d) throw std::invalid_argument("system and grid periodicity differ");
    EwaldParams e;
    e.kind = system.kind;
    e.d = system.d;
    e.grid = grid;
    e.window = window.spec();
    sewald_params_c p = to_c(e);
    RealField out = RealField::zeros(grid.M_ext, strength_components(system.kind));
    std::lock_guard<std::mutex> lk(g_mu);
    check_ctx(sewald_gpu_spread(context(), &p, D(system.x), D(system.f),
                                system.kind == Kernel::stresslet ? D(system.nu) : nullptr,
                                static_cast<int64_t>(system.size()), out.v.data()));
    return out;
}

std::vector<Vec3> gather(const RealField& field, const GridSpec& grid, const Window& window,
                         const TargetSet& targets) {
    if (field.n != grid.M_ext) throw std::invalid_argument("field shape does not match the extended grid");
    if (field.comps != 3) throw std::invalid_argument("gather expects a 3-component field");
    if (std::fabs(window.spec().h - grid.h) > 1e-12 * grid.h)
        throw std::invalid_argument("window was built for a different grid spacing");
    EwaldParams e;
    e.d = grid.d;
    e.grid = grid;
    e.window = window.spec();
    sewald_params_c p = to_c(e);
    std::vector<Vec3> u(targets.x.size());
    std::lock_guard<std::mutex> lk(g_mu);
    check_ctx(sewald_gpu_gather(context(), &p, field.v.data(), D(targets.x), static_cast<int64_t>(targets.x.size()),
                                reinterpret_cast<double*>(u.data())));
    return u;
}

// ---- modified kernels / stage functions ---------------------------------------------
ModifiedKernelSpec ModifiedKernelSpec::optimal(Kernel kind, int d, double R) {
    sewald_modspec_c m{};
    check_host(sewald_modspec_optimal(kernel_id(kind), d, R, &m));
    ModifiedKernelSpec s;
    s.kind = kind;
    s.d = m.d;
    s.R = m.R;
    s.a_B = m.a_B;
    s.b_B = m.b_B;
    s.ell_H = m.ell_H;
    s.ell_B = m.ell_B;
    s.c_B = m.c_B;
    return s;
}

double truncation_radius(const std::array<double, 3>& L, int d) {  // modified_kernels.cpp:65-73
    switch (d) {
        case 0: return std::sqrt(L[0] * L[0] + L[1] * L[1] + L[2] * L[2]);
        case 1: return std::sqrt(L[1] * L[1] + L[2] * L[2]);
        case 2: return L[2];
        default: throw std::invalid_argument("truncation radius applies to d in {0,1,2}");
    }
}

namespace {

sewald_params_c stage_params(const GridSpec& grid, const UpsamplingPlan* plan, const WindowSpec* win) {
    EwaldParams e;
    e.d = grid.d;
    e.grid = grid;
    if (plan) e.upsampling = *plan;
    if (win)
        e.window = *win;
    else
        e.window.h = grid.h;
    return to_c(e);
}

sewald_fourier_geom_c geom_of(const FourierField& F) {
    sewald_fourier_geom_c g{};
    g.d = F.d;
    g.comps = F.comps;
    for (int i = 0; i < 3; ++i) {
        g.n_per[i] = F.n_per[i];
        g.n_far[i] = F.n_far[i];
        g.n_near[i] = F.n_near[i];
        g.n_zero[i] = F.n_zero[i];
    }
    g.n_near_rows = static_cast<int32_t>(F.near_rows.size());
    g.far_len = static_cast<int64_t>(F.far.size());
    g.near_len = static_cast<int64_t>(F.near.size());
    g.zero_len = static_cast<int64_t>(F.zero.size());
    return g;
}

FourierField field_of(const sewald_fourier_geom_c& g, int comps) {
    FourierField F;
    F.d = g.d;
    F.comps = comps;
    for (int i = 0; i < 3; ++i) {
        F.n_per[i] = g.n_per[i];
        F.n_far[i] = g.n_far[i];
        F.n_near[i] = g.n_near[i];
        F.n_zero[i] = g.n_zero[i];
    }
    const int c0 = std::max(g.comps, 1);
    F.far.resize(static_cast<std::size_t>(g.far_len / c0 * comps));
    F.near.resize(static_cast<std::size_t>(g.near_len / c0 * comps));
    F.zero.resize(static_cast<std::size_t>(g.zero_len / c0 * comps));
    return F;
}

double* Z(std::vector<cplx>& v) { return v.empty() ? nullptr : reinterpret_cast<double*>(v.data()); }
const double* Z(const std::vector<cplx>& v) { return v.empty() ? nullptr : reinterpret_cast<const double*>(v.data()); }
const int32_t* rows_of(const std::vector<int>& r) {
    static_assert(sizeof(int) == sizeof(int32_t), "int is 32-bit");
    return r.empty() ? nullptr : reinterpret_cast<const int32_t*>(r.data());
}

}  // namespace

FourierField aft_forward(const RealField& field, const GridSpec& grid, const UpsamplingPlan& plan) {
    if (field.n != grid.M_ext) throw std::invalid_argument("field shape does not match the extended grid");
    if (field.comps < 1 || field.v.size() != static_cast<std::size_t>(field.comps) * field.n[0] * field.n[1] * field.n[2])
        throw std::invalid_argument("field storage is inconsistent");
    sewald_params_c p = stage_params(grid, &plan, nullptr);
    sewald_fourier_geom_c g{};
    std::vector<int32_t> rows(static_cast<std::size_t>(std::max(1, grid.d == 1 ? grid.M[0] : grid.M[0] * grid.M[1])));
    check_host(sewald_aft_geometry(&p, field.comps, &g, rows.data()));
    FourierField F = field_of(g, field.comps);
    F.near_rows.assign(rows.begin(), rows.begin() + g.n_near_rows);
    std::lock_guard<std::mutex> lk(g_mu);
    check_ctx(sewald_gpu_aft_forward(context(), &p, field.v.data(), &g, Z(F.far), Z(F.near), Z(F.zero)));
    return F;
}

RealField aft_inverse(const FourierField& field, const GridSpec& grid, const UpsamplingPlan& plan) {
    if (field.d != grid.d) throw std::invalid_argument("field and grid periodicity differ");
    sewald_params_c p = stage_params(grid, &plan, nullptr);
    const sewald_fourier_geom_c g = geom_of(field);
    RealField out = RealField::zeros(grid.M_ext, field.comps);
    std::lock_guard<std::mutex> lk(g_mu);
    check_ctx(sewald_gpu_aft_inverse(context(), &p, &g, rows_of(field.near_rows), Z(field.far), Z(field.near),
                                     Z(field.zero), out.v.data()));
    return out;
}

FourierField scale(const FourierField& field, const ModifiedKernelSpec& spec, double xi, const Window& window,
                   const GridSpec& grid) {
    sewald_params_c p = stage_params(grid, nullptr, &window.spec());
    const sewald_fourier_geom_c g = geom_of(field);
    const sewald_modspec_c m{kernel_id(spec.kind), spec.d, spec.R, spec.a_B, spec.b_B, spec.ell_H, spec.ell_B, spec.c_B};
    FourierField out = field_of(g, 3);
    out.near_rows = field.near_rows;
    std::lock_guard<std::mutex> lk(g_mu);
    check_ctx(sewald_gpu_scale(context(), &p, &m, xi, &g, rows_of(field.near_rows), Z(field.far), Z(field.near),
                               Z(field.zero), Z(out.far), Z(out.near), Z(out.zero)));
    return out;
}

FourierField scale(const FourierField& field, const PrecomputedKernel0P& pre, double xi, const Window& window,
                   const GridSpec& grid) {
    sewald_params_c p = stage_params(grid, nullptr, &window.spec());
    const sewald_fourier_geom_c g = geom_of(field);
    if (pre.table.size() != static_cast<std::size_t>(pre.n[0]) * pre.n[1] * pre.n[2])
        throw std::invalid_argument("kernel table storage is inconsistent");
    const int32_t tn[3] = {pre.n[0], pre.n[1], pre.n[2]};
    FourierField out;  // fourier.cpp:688-692: only d, comps and n_zero carried over
    out.d = 0;
    out.comps = 3;
    out.n_zero = field.n_zero;
    out.zero.resize(static_cast<std::size_t>(g.zero_len / std::max(g.comps, 1) * 3));
    std::lock_guard<std::mutex> lk(g_mu);
    check_ctx(sewald_gpu_scale_table(context(), &p, kernel_id(pre.kind), tn, Z(pre.table), xi, &g, Z(field.zero),
                                     Z(out.zero)));
    return out;
}

PrecomputedKernel0P precompute_0p(Kernel kind, const GridSpec& grid, double R) {
    sewald_params_c p = stage_params(grid, nullptr, nullptr);
    int32_t n[3];
    std::lock_guard<std::mutex> lk(g_mu);
    check_ctx(sewald_gpu_precompute_0p(context(), &p, kernel_id(kind), R, n, nullptr));
    PrecomputedKernel0P pre;
    pre.kind = kind;
    pre.R = R;
    pre.n = {n[0], n[1], n[2]};
    pre.table.resize(static_cast<std::size_t>(n[0]) * n[1] * n[2]);
    check_ctx(sewald_gpu_precompute_0p(context(), &p, kernel_id(kind), R, n, Z(pre.table)));
    return pre;
}

namespace {

// Host copy split over up to 8 threads (4 MB or more each).
void parallel_copy(void* dst, const void* src, std::size_t n) {
    const std::size_t chunk = std::size_t(4) << 20;
    unsigned k = static_cast<unsigned>(std::min<std::size_t>(8, (n + chunk - 1) / chunk));
    k = std::max(1u, std::min(k, std::max(1u, std::thread::hardware_concurrency())));
    std::vector<std::thread> th;
    for (unsigned i = 1; i < k; ++i)
        th.emplace_back([=] {
            const std::size_t a = n * i / k, b = n * (i + 1) / k;
            std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
        });
    std::memcpy(dst, src, n / k);
    for (auto& x : th) x.join();
}

std::vector<Vec3> pipeline(bool full, const SourceSystem& s, const TargetSet& t, const EwaldParams& e,
                           const SePipelineOptions& opt) {
    validate_system(s);
    if (s.kind != e.kind || s.d != e.d) throw std::invalid_argument("parameter set was built for a different system");
    if (!(e.xi > 0.0)) throw std::invalid_argument("xi must be positive");
    if (opt.table && opt.table->kind != e.kind)
        throw std::invalid_argument("kernel table was built for a different kernel");
    sewald_params_c p = to_c(e);
    for (int i = 0; i < 3; ++i) p.L[i] = s.cell.L[i];
    const std::size_t nt = t.same_as_sources ? s.size() : t.x.size();
    // The returned vector is allocated (and value-initialised: page faults and
    // a serial zero fill, ~5 ms for 1e6 targets) on a helper thread while the
    // device works; the engine writes the result into the context's pinned
    // buffer by DMA, and a parallel copy moves it into the vector at the end.
    std::future<std::vector<Vec3>> ufut =
        std::async(std::launch::async, [nt] { return std::vector<Vec3>(nt); });
    const double* nu = s.kind == Kernel::stresslet ? D(s.nu) : nullptr;
    std::lock_guard<std::mutex> lk(g_mu);
    // SePipelineOptions::table: the caller's table replaces the engine's own
    // (fourier.cpp:822-829); without one the engine builds / reuses its own.
    if (e.d == 0 && opt.precompute_0p) {
        const int32_t tn[3] = {opt.table ? opt.table->n[0] : 0, opt.table ? opt.table->n[1] : 0,
                               opt.table ? opt.table->n[2] : 0};
        if (opt.table && opt.table->table.size() != static_cast<std::size_t>(tn[0]) * tn[1] * tn[2])
            throw std::invalid_argument("kernel table storage is inconsistent");
        check_ctx(sewald_gpu_set_table0p(context(), &p, tn, opt.table ? Z(opt.table->table) : nullptr));
    }
    if (sewald_gpu_multi* m = multi_context()) {
        if (e.d == 0 && opt.precompute_0p) {
            const int32_t tn[3] = {opt.table ? opt.table->n[0] : 0, opt.table ? opt.table->n[1] : 0,
                                   opt.table ? opt.table->n[2] : 0};
            for (int d = 0; d < sewald_gpu_multi_size(m); ++d) {
                sewald_gpu_ctx* c = sewald_gpu_multi_context(m, d);
                rethrow(sewald_gpu_set_table0p(c, &p, tn, opt.table ? Z(opt.table->table) : nullptr),
                        sewald_gpu_last_error(c));
            }
        }
        void* pinned = nullptr;
        check_ctx(sewald_gpu_host_buffer(context(), sizeof(Vec3) * nt, &pinned));
        auto fm = full ? sewald_gpu_multi_full_potential : sewald_gpu_multi_fourier_potential;
        rethrow(fm(m, &p, D(s.x), D(s.f), nu, static_cast<int64_t>(s.size()), t.same_as_sources ? nullptr : D(t.x),
                   static_cast<int64_t>(nt), t.same_as_sources ? 1 : 0, opt.precompute_0p ? 1 : 0,
                   static_cast<double*>(pinned)),
                sewald_gpu_multi_last_error(m));
        std::vector<Vec3> u = ufut.get();
        parallel_copy(u.data(), pinned, sizeof(Vec3) * nt);
        return u;
    }
    void* pinned = nullptr;
    check_ctx(sewald_gpu_host_buffer(context(), sizeof(Vec3) * nt, &pinned));
    auto fn = full ? sewald_gpu_full_potential : sewald_gpu_fourier_potential;
    check_ctx(fn(context(), &p, D(s.x), D(s.f), nu, static_cast<int64_t>(s.size()),
                 t.same_as_sources ? nullptr : D(t.x), static_cast<int64_t>(nt), t.same_as_sources ? 1 : 0,
                 opt.precompute_0p ? 1 : 0, static_cast<double*>(pinned)));
    std::vector<Vec3> u = ufut.get();
    parallel_copy(u.data(), pinned, sizeof(Vec3) * nt);
    return u;
}

}  // namespace

namespace b200 {

void use_devices(const std::vector<int>& devices) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_multi) {
        sewald_gpu_multi_destroy(g_multi);
        g_multi = nullptr;
    }
    g_devices = devices;
    g_devices_set = true;
}

}  // namespace b200

std::vector<Vec3> se_fourier_potential(const SourceSystem& system, const TargetSet& targets,
                                       const EwaldParams& params, const SePipelineOptions& opt) {
    return pipeline(false, system, targets, params, opt);
}

std::vector<Vec3> full_potential(const SourceSystem& system, const TargetSet& targets, const EwaldParams& params,
                                 const SePipelineOptions& opt) {
    return pipeline(true, system, targets, params, opt);
}

std::vector<Vec3> realspace_potential(const SourceSystem& system, const TargetSet& targets, double xi, double rc,
                                      bool starred, int n_threads) {
    (void)n_threads;  // accepted for compatibility; the sum runs on the GPU
    if (!(xi > 0.0)) throw std::invalid_argument("split parameter must be positive");
    const bool skip_self = starred && targets.same_as_sources;
    if (skip_self && targets.x.size() != system.size())
        throw std::invalid_argument("starred evaluation needs one target per source");
    validate_system(system);
    for (const Vec3& p : targets.x)
        for (double c : p)
            if (!std::isfinite(c)) throw std::invalid_argument("target coordinates must be finite");
    std::vector<Vec3> u(targets.x.size());
    std::lock_guard<std::mutex> lk(g_mu);
    check_ctx(sewald_gpu_realspace_potential(
        context(), kernel_id(system.kind), system.d, system.cell.L.data(), D(system.x), D(system.f),
        system.kind == Kernel::stresslet ? D(system.nu) : nullptr, static_cast<int64_t>(system.size()),
        D(targets.x), static_cast<int64_t>(targets.x.size()), targets.same_as_sources ? 1 : 0, xi, rc,
        starred ? 1 : 0, reinterpret_cast<double*>(u.data())));
    return u;
}

// ---- analytic oracles (C-ABI sewald_gpu_direct_sum_0p / _ewald_fourier_3p /
// _fourier_reference_potential, csrc/analytic.cu)

namespace {
TargetSet oracle_targets(const SourceSystem& system, const TargetSet& targets) {
    validate_system(system);
    for (const Vec3& p : targets.x)
        for (double c : p)
            if (!std::isfinite(c)) throw std::invalid_argument("target coordinates must be finite");
    return targets.same_as_sources ? TargetSet{system.x, true} : targets;
}
}  // namespace

std::vector<Vec3> direct_sum_0p(const SourceSystem& system, const TargetSet& targets, bool starred) {
    if (system.d != 0) throw std::invalid_argument("direct_sum_0p needs d = 0");
    const TargetSet t = oracle_targets(system, targets);
    if (starred && t.x.size() != system.size())
        throw std::invalid_argument("starred evaluation needs one target per source");
    std::vector<Vec3> u(t.x.size());
    std::lock_guard<std::mutex> lk(g_mu);
    check_ctx(sewald_gpu_direct_sum_0p(context(), kernel_id(system.kind), D(system.x), D(system.f),
                                       system.kind == Kernel::stresslet ? D(system.nu) : nullptr,
                                       static_cast<int64_t>(system.size()), D(t.x), static_cast<int64_t>(t.x.size()),
                                       starred ? 1 : 0, reinterpret_cast<double*>(u.data())));
    return u;
}

std::vector<Vec3> fourier_reference_potential(const SourceSystem& system, const TargetSet& targets, double xi,
                                              const std::array<int, 3>& kmax) {
    const TargetSet t = oracle_targets(system, targets);
    std::vector<Vec3> u(t.x.size());
    std::lock_guard<std::mutex> lk(g_mu);
    check_ctx(sewald_gpu_fourier_reference_potential(
        context(), kernel_id(system.kind), system.d, system.cell.L.data(), xi, kmax.data(), D(system.x),
        D(system.f), system.kind == Kernel::stresslet ? D(system.nu) : nullptr, static_cast<int64_t>(system.size()),
        D(t.x), static_cast<int64_t>(t.x.size()), reinterpret_cast<double*>(u.data())));
    return u;
}

std::vector<Vec3> direct_ewald_fourier_3p(const SourceSystem& system, const TargetSet& targets, double xi,
                                          const std::array<int, 3>& kmax) {
    if (system.d != 3) throw std::invalid_argument("direct_ewald_fourier_3p needs d = 3");
    return fourier_reference_potential(system, targets, xi, kmax);
}

std::array<int, 3> oracle_kmax(double xi, const Cell& cell) {
    const double kc = 2.0 * xi * std::sqrt(39.0);
    std::array<int, 3> k{};
    for (int a = 0; a < 3; ++a) k[a] = static_cast<int>(std::ceil(kc * cell.L[a] / (2.0 * M_PI))) + 1;
    return k;
}

double rms_error(const std::vector<Vec3>& u, const std::vector<Vec3>& u_ref) {
    if (u.size() != u_ref.size()) throw std::invalid_argument("rms error needs equal lengths");
    if (u.empty()) throw std::invalid_argument("rms error of an empty set");
    double a = 0.0;
    rethrow(sewald_rms_error(D(u), D(u_ref), static_cast<int64_t>(u.size()), &a, nullptr), "rms error");
    return a;
}

double rel_rms_error(const std::vector<Vec3>& u, const std::vector<Vec3>& u_ref) {
    if (u.size() != u_ref.size()) throw std::invalid_argument("rms error needs equal lengths");
    if (u.empty()) throw std::invalid_argument("rms error of an empty set");
    double a = 0.0, r = 0.0;
    rethrow(sewald_rms_error(D(u), D(u_ref), static_cast<int64_t>(u.size()), &a, &r),
            "relative rms error of a zero reference");
    return r;
}

}  // namespace sewald
