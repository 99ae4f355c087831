// End-to-end timing of the C++ drop-in path (what a reference user's code
// calls): sewald::full_potential with pageable std::vector inputs and output,
// linked against libsewald_gpu.so. The workload is BASELINE config 2 (N = 1e6
// uniform triply periodic stokeslets, forces N(0,1), tol 1e-8, xi pinned at 37:
// M = 128^3, P = 16), drawn with std::mt19937_64 (the timing does not depend
// on the particular draw). Prints one JSON line; bench.py reports it as
// e2e_cpp beside the Python pinned-buffer figure.
//
//   bench_dropin [N] [calls]
#include "sewald/estimates.h"
#include "sewald/realspace.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

using namespace sewald;

int main(int argc, char** argv) {
    const int N = argc > 1 ? std::atoi(argv[1]) : 1000000;
    const int calls = argc > 2 ? std::atoi(argv[2]) : 5;
    std::mt19937_64 rng(1002);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    std::normal_distribution<double> G(0.0, 1.0);
    SourceSystem s;
    s.kind = Kernel::stokeslet;
    s.d = 3;
    s.cell.L = {1.0, 1.0, 1.0};
    s.x.resize(N);
    s.f.resize(N);
    for (auto& p : s.x) p = {U(rng), U(rng), U(rng)};
    for (auto& p : s.f) p = {G(rng), G(rng), G(rng)};
    const double Q = source_quantity(s);
    const ParameterSelection sel = select_parameters(Kernel::stokeslet, 3, s.cell, Q, 37.0, ToleranceSpec{1e-8, false});
    const TargetSet t = TargetSet::from_sources(s);
    std::vector<Vec3> u = full_potential(s, t, sel.params);  // warm: plans, buffers
    std::vector<double> ms;
    for (int k = 0; k < calls; ++k) {
        const auto t0 = std::chrono::steady_clock::now();
        u = full_potential(s, t, sel.params);  // pageable vectors in, a new vector out
        const auto t1 = std::chrono::steady_clock::now();
        ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
    }
    std::sort(ms.begin(), ms.end());
    const double med = ms[ms.size() / 2];
    double rms = 0.0;
    for (const auto& v : u) rms += v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
    std::printf("{\"api\": \"sewald::full_potential (C++ drop-in, pageable std::vector in/out)\", \"N\": %d, "
                "\"M\": %d, \"P\": %d, \"calls\": %d, \"ms_per_call\": %.4f, \"value\": %.6g, \"unit\": \"targets/s\", "
                "\"h2d_bytes_per_step\": %lld, \"d2h_bytes_per_step\": %lld, \"u_rms\": %.10g}\n",
                N, sel.params.grid.M[0], sel.params.window.P, calls, med, N / (med * 1e-3),
                (long long)N * 48, (long long)N * 24, std::sqrt(rms / N));
    return 0;
}
