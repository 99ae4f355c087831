// ORACLE TEST INFRASTRUCTURE — not product code. Only tests/, smoke() and
// bench.py's reference/cpu_baseline legs load the library built from this
// file (oracle/_ref/libsewald_ref.so).
//
// extern "C" wrapper over the UNMODIFIED reference C++ library
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile with the
// shims in oracle/shims/). It lets Python tests call the reference itself
// through ctypes with the same POD parameter struct the product C-ABI uses
// (include/sewald_gpu.h), so parity is checked against the reference's own
// arithmetic, not a re-derivation.
#include "sewald/domain.h"
#include "sewald/estimates.h"
#include "sewald/fourier.h"
#include "sewald/grid.h"
#include "sewald/kernels.h"
#include "sewald/modified_kernels.h"
#include "sewald/realspace.h"
#include "sewald/window.h"

#include "../include/sewald_gpu.h"

#include <chrono>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

using namespace sewald;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& fn) {
    try {
        fn();
        return SEWALD_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return SEWALD_EINVAL;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return SEWALD_EDOMAIN;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SEWALD_ERUNTIME;
    }
}

Kernel to_kernel(int k) {
    switch (k) {
        case SEWALD_STOKESLET: return Kernel::stokeslet;
        case SEWALD_STRESSLET: return Kernel::stresslet;
        case SEWALD_ROTLET: return Kernel::rotlet;
    }
    throw std::invalid_argument("bad kernel id");
}

WindowKind to_window(int w) {
    switch (w) {
        case SEWALD_WIN_KB: return WindowKind::kb;
        case SEWALD_WIN_PKB: return WindowKind::pkb;
        case SEWALD_WIN_TG: return WindowKind::tg;
    }
    throw std::invalid_argument("bad window id");
}

int from_window(WindowKind w) {
    return w == WindowKind::kb ? SEWALD_WIN_KB : (w == WindowKind::pkb ? SEWALD_WIN_PKB : SEWALD_WIN_TG);
}

void to_c(const EwaldParams& e, sewald_params_c* p) {
    std::memset(p, 0, sizeof(*p));
    p->kind = static_cast<int>(e.kind == Kernel::stokeslet ? SEWALD_STOKESLET
                               : e.kind == Kernel::stresslet ? SEWALD_STRESSLET
                                                             : SEWALD_ROTLET);
    p->d = e.d;
    p->xi = e.xi;
    p->rc = e.rc;
    p->R = e.R;
    p->h = e.grid.h;
    for (int i = 0; i < 3; ++i) {
        p->M[i] = e.grid.M[i];
        p->M_ext[i] = e.grid.M_ext[i];
        p->L[i] = e.grid.L[i];
        p->L_ext[i] = e.grid.L_ext[i];
        p->pad[i] = e.grid.pad[i];
        p->k_star[i] = e.upsampling.k_star[i];
    }
    p->f_m = e.grid.f_m;
    p->win_kind = from_window(e.window.kind);
    p->P = e.window.P;
    p->win_h = e.window.h;
    p->beta = e.window.beta;
    p->nu = e.window.nu;
    p->alpha = e.window.alpha;
    p->s0 = e.upsampling.s0;
    p->s_star = e.upsampling.s_star;
    p->s0_raw = e.upsampling.s0_raw;
    p->s_star_raw = e.upsampling.s_star_raw;
}

EwaldParams from_c(const sewald_params_c* p) {
    EwaldParams e;
    e.kind = to_kernel(p->kind);
    e.d = p->d;
    e.xi = p->xi;
    e.rc = p->rc;
    e.R = p->R;
    e.grid.d = p->d;
    e.grid.h = p->h;
    for (int i = 0; i < 3; ++i) {
        e.grid.M[i] = p->M[i];
        e.grid.M_ext[i] = p->M_ext[i];
        e.grid.L[i] = p->L[i];
        e.grid.L_ext[i] = p->L_ext[i];
        e.grid.pad[i] = p->pad[i];
        e.upsampling.k_star[i] = p->k_star[i];
    }
    e.grid.f_m = p->f_m;
    e.window.kind = to_window(p->win_kind);
    e.window.P = p->P;
    e.window.h = p->win_h;
    e.window.beta = p->beta;
    e.window.nu = p->nu;
    e.window.alpha = p->alpha;
    e.upsampling.s0 = p->s0;
    e.upsampling.s_star = p->s_star;
    e.upsampling.s0_raw = p->s0_raw;
    e.upsampling.s_star_raw = p->s_star_raw;
    return e;
}

std::vector<Vec3> vec3(const double* a, int64_t n) {
    std::vector<Vec3> v(static_cast<std::size_t>(n));
    if (n) std::memcpy(v.data(), a, sizeof(double) * 3 * n);
    return v;
}

SourceSystem make_system(int kind, int d, const double L[3], const double* x, const double* f,
                         const double* nu, int64_t N) {
    SourceSystem s;
    s.kind = to_kernel(kind);
    s.d = d;
    s.cell.L = {L[0], L[1], L[2]};
    s.x = vec3(x, N);
    s.f = vec3(f, N);
    if (s.kind == Kernel::stresslet) s.nu = vec3(nu, N);
    return s;
}

TargetSet make_targets(const SourceSystem& s, const double* xt, int64_t Nt, int same) {
    if (same) return TargetSet::from_sources(s);
    TargetSet t;
    t.x = vec3(xt, Nt);
    return t;
}

void out3(const std::vector<Vec3>& u, double* out) {
    if (!u.empty()) std::memcpy(out, u.data(), sizeof(double) * 3 * u.size());
}

double g_last_seconds[4] = {0, 0, 0, 0};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// Wall seconds of the last ref_full_split call: [fourier, realspace, terms, total].
void ref_last_seconds(double* out) { std::memcpy(out, g_last_seconds, sizeof(g_last_seconds)); }

int ref_select_parameters(int kind, int d, const double L[3], double Q, double xi, double tol,
                          int relative, int f_m, int window_kind, int pollution_fix,
                          sewald_params_c* out, sewald_report_c* rep) {
    return guarded([&] {
        SelectionOptions opt;
        opt.f_m = f_m;
        opt.window = to_window(window_kind);
        opt.pollution_fix = pollution_fix != 0;
        Cell cell;
        cell.L = {L[0], L[1], L[2]};
        ParameterSelection sel =
            select_parameters(to_kernel(kind), d, cell, Q, xi, ToleranceSpec{tol, relative != 0}, opt);
        to_c(sel.params, out);
        if (rep) {
            const EstimateReport& r = sel.report;
            rep->tau_abs = r.tau_abs;
            rep->U = r.U;
            rep->kinf = r.kinf;
            rep->fourier_trunc = r.fourier_trunc;
            rep->realspace_trunc = r.realspace_trunc;
            rep->window_err = r.window_err;
            rep->h_estimate = r.h_estimate;
            rep->P_estimate = r.P_estimate;
            rep->h_target = r.h_target;
            rep->P_target = r.P_target;
            rep->rc_clamped = r.rc_clamped;
            rep->kinf_clamped = r.kinf_clamped;
            rep->window_saturated = r.window_saturated;
            rep->tg_support_from_pkb = r.tg_support_from_pkb;
        }
    });
}

int ref_pkb_coefficients(const sewald_params_c* p, double* coef) {
    return guarded([&] {
        PiecewisePolyWindow w = pkb_build(from_c(p).window);
        std::memcpy(coef, w.coef.data(), sizeof(double) * w.coef.size());
    });
}

int ref_window_eval(const sewald_params_c* p, const double* r, int64_t n, double* out) {
    return guarded([&] {
        Window w(from_c(p).window);
        for (int64_t i = 0; i < n; ++i) out[i] = w.eval1d(r[i]);
    });
}

int ref_window_hat(const sewald_params_c* p, const double* k, int64_t n, double* out) {
    return guarded([&] {
        Window w(from_c(p).window);
        for (int64_t i = 0; i < n; ++i) out[i] = w.hat1d(k[i]);
    });
}

int ref_build_grid(const double L[3], int d, double h_target, int P, int kind, int f_m,
                   sewald_params_c* out) {
    return guarded([&] {
        Cell cell;
        cell.L = {L[0], L[1], L[2]};
        EwaldParams e;
        e.kind = to_kernel(kind);
        e.d = d;
        e.grid = build_grid(cell, d, h_target, P, e.kind, f_m);
        to_c(e, out);
    });
}

int ref_spread(const sewald_params_c* p, const double* x, const double* f, const double* nu,
               int64_t N, double* grid_out) {
    return guarded([&] {
        EwaldParams e = from_c(p);
        SourceSystem s = make_system(p->kind, p->d, p->L, x, f, nu, N);
        RealField phi = spread(s, e.grid, Window(e.window));
        std::memcpy(grid_out, phi.v.data(), sizeof(double) * phi.v.size());
    });
}

int ref_gather(const sewald_params_c* p, const double* grid, const double* xt, int64_t Nt,
               double* u_out) {
    return guarded([&] {
        EwaldParams e = from_c(p);
        RealField fld = RealField::zeros(e.grid.M_ext, 3);
        std::memcpy(fld.v.data(), grid, sizeof(double) * fld.v.size());
        TargetSet t;
        t.x = vec3(xt, Nt);
        out3(gather(fld, e.grid, Window(e.window), t), u_out);
    });
}

// Spread -> forward -> scale -> inverse; returns the 3-component flow field
// on the extended grid (the RealField gather consumes).
int ref_flow_field(const sewald_params_c* p, const double* x, const double* f, const double* nu,
                   int64_t N, int use_table, double* flow_out) {
    return guarded([&] {
        EwaldParams e = from_c(p);
        SourceSystem s = make_system(p->kind, p->d, p->L, x, f, nu, N);
        const Window window(e.window);
        const ModifiedKernelSpec spec = ModifiedKernelSpec::optimal(e.kind, e.d, e.d == 3 ? 1.0 : e.R);
        RealField phi = spread(s, e.grid, window);
        UpsamplingPlan plan = e.upsampling;
        FourierField scaled;
        if (e.d == 0 && use_table) {
            plan.s0 = 2.0;
            FourierField modes = aft_forward(phi, e.grid, plan);
            PrecomputedKernel0P table = precompute_0p(e.kind, e.grid, e.R);
            scaled = scale(modes, table, e.xi, window, e.grid);
        } else {
            FourierField modes = aft_forward(phi, e.grid, plan);
            scaled = scale(modes, spec, e.xi, window, e.grid);
        }
        RealField flow = aft_inverse(scaled, e.grid, plan);
        std::memcpy(flow_out, flow.v.data(), sizeof(double) * flow.v.size());
    });
}

// aft_forward -> scale -> aft_inverse on a given spread grid (C comps) ->
// 3-component flow field (the stage sequence of se_fourier_potential,
// fourier.cpp:816-840, starting from an existing RealField).
int ref_solve_grid(const sewald_params_c* p, const double* grid, int use_table, double* flow_out) {
    return guarded([&] {
        EwaldParams e = from_c(p);
        const Window window(e.window);
        const ModifiedKernelSpec spec = ModifiedKernelSpec::optimal(e.kind, e.d, e.d == 3 ? 1.0 : e.R);
        RealField phi = RealField::zeros(e.grid.M_ext, strength_components(e.kind));
        std::memcpy(phi.v.data(), grid, sizeof(double) * phi.v.size());
        UpsamplingPlan plan = e.upsampling;
        FourierField scaled;
        if (e.d == 0 && use_table) {
            plan.s0 = 2.0;
            FourierField modes = aft_forward(phi, e.grid, plan);
            PrecomputedKernel0P table = precompute_0p(e.kind, e.grid, e.R);
            scaled = scale(modes, table, e.xi, window, e.grid);
        } else {
            FourierField modes = aft_forward(phi, e.grid, plan);
            scaled = scale(modes, spec, e.xi, window, e.grid);
        }
        RealField flow = aft_inverse(scaled, e.grid, plan);
        std::memcpy(flow_out, flow.v.data(), sizeof(double) * flow.v.size());
    });
}

int ref_fourier_potential(const sewald_params_c* p, const double* x, const double* f,
                          const double* nu, int64_t N, const double* xt, int64_t Nt, int same,
                          int precompute_0p, double* u_out) {
    return guarded([&] {
        EwaldParams e = from_c(p);
        SourceSystem s = make_system(p->kind, p->d, p->L, x, f, nu, N);
        TargetSet t = make_targets(s, xt, Nt, same);
        SePipelineOptions opt;
        opt.precompute_0p = precompute_0p != 0;
        out3(se_fourier_potential(s, t, e, opt), u_out);
    });
}

int ref_realspace_potential(int kind, int d, const double L[3], const double* x, const double* f,
                            const double* nu, int64_t N, const double* xt, int64_t Nt, int same,
                            double xi, double rc, int starred, int n_threads, double* u_out) {
    return guarded([&] {
        SourceSystem s = make_system(kind, d, L, x, f, nu, N);
        TargetSet t = make_targets(s, xt, Nt, same);
        out3(realspace_potential(s, t, xi, rc, starred != 0, n_threads), u_out);
    });
}

int ref_full_potential(const sewald_params_c* p, const double* x, const double* f,
                       const double* nu, int64_t N, const double* xt, int64_t Nt, int same,
                       int precompute_0p, double* u_out) {
    return guarded([&] {
        EwaldParams e = from_c(p);
        SourceSystem s = make_system(p->kind, p->d, p->L, x, f, nu, N);
        TargetSet t = make_targets(s, xt, Nt, same);
        SePipelineOptions opt;
        opt.precompute_0p = precompute_0p != 0;
        out3(full_potential(s, t, e, opt), u_out);
    });
}

// full_potential assembled exactly as realspace.cpp:205-219 but with the
// real-space sum on n_threads workers (the reference's only parallel knob,
// realspace.h:40-41). Used as the CPU baseline; stage wall times are kept
// for ref_last_seconds.
int ref_full_parts(const sewald_params_c* p, const double* x, const double* f, const double* nu,
                   int64_t N, const double* xt, int64_t Nt, int same, int precompute_0p,
                   int n_threads, double* u_out, double* uf_out, double* ur_out) {
    return guarded([&] {
        using clk = std::chrono::steady_clock;
        EwaldParams e = from_c(p);
        SourceSystem s = make_system(p->kind, p->d, p->L, x, f, nu, N);
        TargetSet t = make_targets(s, xt, Nt, same);
        SePipelineOptions opt;
        opt.precompute_0p = precompute_0p != 0;
        auto t0 = clk::now();
        std::vector<Vec3> u = realspace_potential(s, t, e.xi, e.rc, t.same_as_sources, n_threads);
        auto t1 = clk::now();
        const std::vector<Vec3> far = se_fourier_potential(s, t, e, opt);
        auto t2 = clk::now();
        if (ur_out) out3(u, ur_out);
        if (uf_out) out3(far, uf_out);
        for (std::size_t i = 0; i < u.size(); ++i) u[i] += far[i];
        if (t.same_as_sources)
            for (std::size_t i = 0; i < u.size(); ++i) u[i] += self_term(s.kind, e.xi, s.f[i]);
        if (s.kind == Kernel::stresslet && e.d == 3) {
            const std::vector<Vec3> mean = stresslet_zero_mode_3p(t, s);
            for (std::size_t i = 0; i < u.size(); ++i) u[i] += mean[i];
        }
        auto t3 = clk::now();
        g_last_seconds[0] = std::chrono::duration<double>(t2 - t1).count();
        g_last_seconds[1] = std::chrono::duration<double>(t1 - t0).count();
        g_last_seconds[2] = std::chrono::duration<double>(t3 - t2).count();
        g_last_seconds[3] = std::chrono::duration<double>(t3 - t0).count();
        out3(u, u_out);
    });
}

// full_potential assembled as realspace.cpp:205-219 (u only).
int ref_full_split(const sewald_params_c* p, const double* x, const double* f, const double* nu,
                   int64_t N, const double* xt, int64_t Nt, int same, int precompute_0p,
                   int n_threads, double* u_out) {
    return ref_full_parts(p, x, f, nu, N, xt, Nt, same, precompute_0p, n_threads, u_out, nullptr,
                          nullptr);
}

// precompute_0p (fourier.cpp:722-803): table of (2 M_ext)^3 complex values,
// written as interleaved (re, im) doubles.
int ref_precompute_0p(const sewald_params_c* p, double* table_out, int32_t* n_out) {
    return guarded([&] {
        EwaldParams e = from_c(p);
        PrecomputedKernel0P t = precompute_0p(e.kind, e.grid, e.R);
        for (int i = 0; i < 3; ++i) n_out[i] = t.n[i];
        if (table_out) std::memcpy(table_out, t.table.data(), sizeof(double) * 2 * t.table.size());
    });
}

// ---- stage functions (fourier.h:61-74) on one held FourierField ----------
// ref_aft_forward / ref_field_set load it, ref_scale / ref_scale_table
// replace it by its scaled copy, ref_field_get / ref_aft_inverse read it.
// Arrays cross as interleaved (re, im) doubles with the geometry of
// sewald_fourier_geom_c (include/sewald_gpu.h).
namespace {
FourierField g_field;

void field_geom(const FourierField& F, sewald_fourier_geom_c* g) {
    std::memset(g, 0, sizeof(*g));
    g->d = F.d;
    g->comps = F.comps;
    for (int i = 0; i < 3; ++i) {
        g->n_per[i] = F.n_per[i];
        g->n_far[i] = F.n_far[i];
        g->n_near[i] = F.n_near[i];
        g->n_zero[i] = F.n_zero[i];
    }
    g->n_near_rows = static_cast<int32_t>(F.near_rows.size());
    g->far_len = static_cast<int64_t>(F.far.size());
    g->near_len = static_cast<int64_t>(F.near.size());
    g->zero_len = static_cast<int64_t>(F.zero.size());
}

void copy_in(std::vector<cplx>& v, const double* a, int64_t n) {
    v.assign(static_cast<std::size_t>(n), cplx{});
    if (n) std::memcpy(v.data(), a, sizeof(double) * 2 * n);
}
void copy_out(const std::vector<cplx>& v, double* a) {
    if (a && !v.empty()) std::memcpy(a, v.data(), sizeof(double) * 2 * v.size());
}
}  // namespace

int ref_aft_forward(const sewald_params_c* p, const double* field, int comps, sewald_fourier_geom_c* g) {
    return guarded([&] {
        EwaldParams e = from_c(p);
        RealField phi = RealField::zeros(e.grid.M_ext, comps);
        std::memcpy(phi.v.data(), field, sizeof(double) * phi.v.size());
        g_field = aft_forward(phi, e.grid, e.upsampling);
        field_geom(g_field, g);
    });
}

int ref_field_get(sewald_fourier_geom_c* g, int32_t* near_rows, double* far, double* near, double* zero) {
    return guarded([&] {
        field_geom(g_field, g);
        if (near_rows)
            for (std::size_t i = 0; i < g_field.near_rows.size(); ++i) near_rows[i] = g_field.near_rows[i];
        copy_out(g_field.far, far);
        copy_out(g_field.near, near);
        copy_out(g_field.zero, zero);
    });
}

int ref_field_set(const sewald_fourier_geom_c* g, const int32_t* near_rows, const double* far, const double* near,
                  const double* zero) {
    return guarded([&] {
        FourierField F;
        F.d = g->d;
        F.comps = g->comps;
        for (int i = 0; i < 3; ++i) {
            F.n_per[i] = g->n_per[i];
            F.n_far[i] = g->n_far[i];
            F.n_near[i] = g->n_near[i];
            F.n_zero[i] = g->n_zero[i];
        }
        F.near_rows.assign(near_rows, near_rows + g->n_near_rows);
        copy_in(F.far, far, g->far_len);
        copy_in(F.near, near, g->near_len);
        copy_in(F.zero, zero, g->zero_len);
        g_field = std::move(F);
    });
}

int ref_scale(const sewald_params_c* p, const sewald_modspec_c* m, double xi, sewald_fourier_geom_c* g) {
    return guarded([&] {
        EwaldParams e = from_c(p);
        ModifiedKernelSpec spec;
        spec.kind = to_kernel(m->kind);
        spec.d = m->d;
        spec.R = m->R;
        spec.a_B = m->a_B;
        spec.b_B = m->b_B;
        spec.ell_H = m->ell_H;
        spec.ell_B = m->ell_B;
        spec.c_B = m->c_B;
        const Window window(e.window);
        g_field = scale(g_field, spec, xi, window, e.grid);
        field_geom(g_field, g);
    });
}

// scale with precompute_0p(kind, grid, R) (fourier.cpp:668-720, :722-803).
int ref_scale_table(const sewald_params_c* p, int kind, double R, double xi, sewald_fourier_geom_c* g) {
    return guarded([&] {
        EwaldParams e = from_c(p);
        const Window window(e.window);
        PrecomputedKernel0P t = precompute_0p(to_kernel(kind), e.grid, R);
        g_field = scale(g_field, t, xi, window, e.grid);
        field_geom(g_field, g);
    });
}

int ref_aft_inverse(const sewald_params_c* p, double* field_out) {
    return guarded([&] {
        EwaldParams e = from_c(p);
        RealField out = aft_inverse(g_field, e.grid, e.upsampling);
        std::memcpy(field_out, out.v.data(), sizeof(double) * out.v.size());
    });
}

// Scalar kernel probes for restatement pinning.
int ref_realspace_kernel(int kind, const double r[3], double xi, double* out27) {
    return guarded([&] {
        KernelTensorR K = realspace_kernel(to_kernel(kind), {r[0], r[1], r[2]}, xi);
        if (K.rank == 2)
            for (int j = 0; j < 3; ++j)
                for (int l = 0; l < 3; ++l) out27[3 * j + l] = K.m[j][l];
        else
            for (int j = 0; j < 3; ++j)
                for (int l = 0; l < 3; ++l)
                    for (int m = 0; m < 3; ++m) out27[9 * j + 3 * l + m] = K.t[j][l][m];
    });
}

int ref_modified_kernel_hat(int kind, int d, double R, const double k[3], double* out54) {
    return guarded([&] {
        ModifiedKernelSpec spec = ModifiedKernelSpec::optimal(to_kernel(kind), d, R);
        KernelTensor K = modified_kernel_hat(spec, {k[0], k[1], k[2]});
        if (K.rank == 2)
            for (int j = 0; j < 3; ++j)
                for (int l = 0; l < 3; ++l) {
                    out54[2 * (3 * j + l)] = K.m[j][l].real();
                    out54[2 * (3 * j + l) + 1] = K.m[j][l].imag();
                }
        else
            for (int j = 0; j < 3; ++j)
                for (int l = 0; l < 3; ++l)
                    for (int m = 0; m < 3; ++m) {
                        out54[2 * (9 * j + 3 * l + m)] = K.t[j][l][m].real();
                        out54[2 * (9 * j + 3 * l + m) + 1] = K.t[j][l][m].imag();
                    }
    });
}

}  // extern "C"
