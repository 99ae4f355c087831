// Drop-in C++ API test: user code written against the reference headers
// (#include "sewald/realspace.h", namespace sewald) compiled against this
// repo's include/ and linked with libsewald_gpu.so. The checks restate the
// reference's own physics tests:
//   free-space potential = bare kernel sum      test_realspace.cpp:469-514
//   full potential invariant under xi            test_realspace.cpp:516-540
//   unstarred evaluation on a source is singular test_realspace.cpp:429-435
// and composes the stage functions spread -> aft_forward -> scale ->
// aft_inverse -> gather exactly as se_fourier_potential (fourier.cpp:805-852).
#include "sewald/estimates.h"
#include "sewald/fourier.h"
#include "sewald/modified_kernels.h"
#include "sewald/realspace.h"

#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>

using namespace sewald;

static int failures = 0;
#define EXPECT(c)                                                          \
    do {                                                                   \
        if (!(c)) {                                                        \
            ++failures;                                                    \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);        \
        }                                                                  \
    } while (0)

static Vec3 bare(Kernel kind, const Vec3& r, const Vec3& f, const Vec3& nu) {
    const double r2 = r[0] * r[0] + r[1] * r[1] + r[2] * r[2], rn = std::sqrt(r2);
    Vec3 u{0, 0, 0};
    if (kind == Kernel::stokeslet) {
        const double rf = r[0] * f[0] + r[1] * f[1] + r[2] * f[2];
        for (int j = 0; j < 3; ++j) u[j] = f[j] / rn + r[j] * rf / (r2 * rn);
    } else if (kind == Kernel::rotlet) {
        const double c = 1.0 / (r2 * rn);
        u = {c * (f[1] * r[2] - f[2] * r[1]), c * (f[2] * r[0] - f[0] * r[2]), c * (f[0] * r[1] - f[1] * r[0])};
    } else {
        const double rq = r[0] * f[0] + r[1] * f[1] + r[2] * f[2];
        const double rv = r[0] * nu[0] + r[1] * nu[1] + r[2] * nu[2];
        for (int j = 0; j < 3; ++j) u[j] = -6.0 * r[j] * rq * rv / (r2 * r2 * rn);
    }
    return u;
}

static SourceSystem random_system(Kernel kind, int d, int n, std::mt19937& rng) {
    std::uniform_real_distribution<double> up(0.0, 1.0), uf(0.1, 0.9), us(-1.0, 1.0);
    SourceSystem s;
    s.kind = kind;
    s.d = d;
    for (int i = 0; i < n; ++i) {
        Vec3 x{};
        for (int a = 0; a < 3; ++a) x[a] = a < d ? up(rng) : uf(rng);
        s.x.push_back(x);
        s.f.push_back({us(rng), us(rng), us(rng)});
        if (kind == Kernel::stresslet) s.nu.push_back({us(rng), us(rng), us(rng)});
    }
    return s;
}

int main() {
    // free space: two sources, full potential equals the bare sum
    for (Kernel kind : {Kernel::stokeslet, Kernel::rotlet, Kernel::stresslet}) {
        for (double xi : {4.0, 7.0}) {
            SourceSystem s;
            s.kind = kind;
            s.d = 0;
            s.x = {{0.25, 0.3, 0.35}, {0.6, 0.55, 0.7}};
            s.f = {{1.0, -0.5, 0.75}, {-0.25, 1.25, 0.5}};
            if (kind == Kernel::stresslet) s.nu = {{0.3, 0.8, -0.5}, {-0.6, 0.2, 0.9}};
            const EwaldParams p =
                select_parameters(kind, 0, s.cell, source_quantity(s), xi, ToleranceSpec{1e-9, false}).params;
            const auto u = full_potential(s, TargetSet::from_sources(s), p);
            const Vec3 nu0 = s.nu.empty() ? Vec3{} : s.nu[0], nu1 = s.nu.empty() ? Vec3{} : s.nu[1];
            const Vec3 e0 = bare(kind, {s.x[0][0] - s.x[1][0], s.x[0][1] - s.x[1][1], s.x[0][2] - s.x[1][2]}, s.f[1], nu1);
            const Vec3 e1 = bare(kind, {s.x[1][0] - s.x[0][0], s.x[1][1] - s.x[0][1], s.x[1][2] - s.x[0][2]}, s.f[0], nu0);
            double err = 0.0;
            for (int c = 0; c < 3; ++c) err = std::fmax(err, std::fmax(std::fabs(u[0][c] - e0[c]), std::fabs(u[1][c] - e1[c])));
            std::printf("free space %-9s xi=%.0f max|u - bare| = %.3e\n", kernel_name(kind), xi, err);
            EXPECT(err <= 1e-8);
        }
    }
    // xi invariance of the full potential, rms <= 10 (tau + tau)
    std::mt19937 rng(57120848);
    struct Case { Kernel kind; int d; double xa, xb; };
    for (const Case c : {Case{Kernel::stokeslet, 3, 8.0, 12.0}, Case{Kernel::stresslet, 3, 8.0, 12.0},
                         Case{Kernel::stresslet, 2, 6.0, 9.0}, Case{Kernel::rotlet, 1, 6.0, 9.0}}) {
        SourceSystem s = random_system(c.kind, c.d, 40, rng);
        const double tau = 1e-10, Q = source_quantity(s);
        const auto ua = full_potential(s, TargetSet::from_sources(s),
                                       select_parameters(c.kind, c.d, s.cell, Q, c.xa, ToleranceSpec{tau, false}).params);
        const auto ub = full_potential(s, TargetSet::from_sources(s),
                                       select_parameters(c.kind, c.d, s.cell, Q, c.xb, ToleranceSpec{tau, false}).params);
        double acc = 0.0;
        for (std::size_t t = 0; t < ua.size(); ++t)
            for (int k = 0; k < 3; ++k) acc += (ua[t][k] - ub[t][k]) * (ua[t][k] - ub[t][k]);
        const double rms = std::sqrt(acc / ua.size());
        std::printf("xi invariance %-9s d=%d rms = %.3e\n", kernel_name(c.kind), c.d, rms);
        EXPECT(rms <= 10.0 * (tau + tau));
    }
    // stage composition == se_fourier_potential (no gauge correction for
    // these kinds: gauge_flow_correction is stokeslet, d <= 1 only)
    struct StageCase { Kernel kind; int d; bool table; };
    for (const StageCase c : {StageCase{Kernel::stokeslet, 3, false}, StageCase{Kernel::stresslet, 2, false},
                              StageCase{Kernel::rotlet, 1, false}, StageCase{Kernel::stokeslet, 2, false},
                              StageCase{Kernel::rotlet, 0, false}, StageCase{Kernel::stresslet, 0, true}}) {
        SourceSystem s = random_system(c.kind, c.d, 60, rng);
        const EwaldParams p =
            select_parameters(c.kind, c.d, s.cell, source_quantity(s), 7.0, ToleranceSpec{1e-9, false}).params;
        const Window window(p.window);
        RealField phi = spread(s, p.grid, window);
        UpsamplingPlan plan = p.upsampling;
        FourierField scaled;
        if (c.table) {
            plan.s0 = 2.0;
            const PrecomputedKernel0P pre = precompute_0p(c.kind, p.grid, p.R);
            scaled = scale(aft_forward(phi, p.grid, plan), pre, p.xi, window, p.grid);
        } else {
            const ModifiedKernelSpec spec = ModifiedKernelSpec::optimal(c.kind, c.d, c.d == 3 ? 1.0 : p.R);
            scaled = scale(aft_forward(phi, p.grid, plan), spec, p.xi, window, p.grid);
        }
        const RealField flow = aft_inverse(scaled, p.grid, plan);
        const TargetSet t = TargetSet::from_sources(s);
        const auto us = gather(flow, p.grid, window, t);
        SePipelineOptions opt;
        opt.precompute_0p = c.table;
        const auto ur = se_fourier_potential(s, t, p, opt);
        double num = 0.0, den = 0.0;
        for (std::size_t i = 0; i < ur.size(); ++i)
            for (int k = 0; k < 3; ++k) {
                num += (us[i][k] - ur[i][k]) * (us[i][k] - ur[i][k]);
                den += ur[i][k] * ur[i][k];
            }
        const double rel = std::sqrt(num / den);
        std::printf("stages %-9s d=%d table=%d rel = %.3e\n", kernel_name(c.kind), c.d, c.table ? 1 : 0, rel);
        EXPECT(rel <= 1e-12);
    }
    // error behaviour
    {
        SourceSystem s = random_system(Kernel::stokeslet, 3, 5, rng);
        bool threw = false;
        try {
            (void)realspace_potential(s, TargetSet::from_sources(s), 3.0, 0.3, false);
        } catch (const std::domain_error&) {
            threw = true;
        }
        EXPECT(threw);
        threw = false;
        try {
            (void)realspace_potential(s, TargetSet::from_sources(s), 0.0, 0.3, true);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        EXPECT(threw);
    }
    std::printf("dropin: %s (%d failures)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
