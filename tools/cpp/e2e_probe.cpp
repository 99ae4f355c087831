// Host-buffer pipeline timing breakdown (diagnostic): sewald_gpu_full_potential
// with pageable vs pinned buffers, per-stage CUDA-event times from the context.
#include "../../include/sewald_gpu.h"
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <random>
#include <vector>

int main() {
    const int N = 1000000;
    std::mt19937_64 rng(1);
    std::uniform_real_distribution<double> U(0, 1);
    std::normal_distribution<double> G(0, 1);
    std::vector<double> x(3 * N), f(3 * N), u(3 * N);
    for (auto& v : x) v = U(rng);
    for (auto& v : f) v = G(rng);
    double L[3] = {1, 1, 1};
    sewald_params_c p;
    sewald_report_c rep;
    double Q = 0;
    for (double v : f) Q += v * v;
    sewald_select_parameters(SEWALD_STOKESLET, 3, L, Q, 37.0, 1e-8, 0, 4, SEWALD_WIN_PKB, 1, &p, &rep);
    sewald_gpu_ctx* ctx;
    sewald_gpu_create(0, &ctx);
    sewald_gpu_set_profiling(ctx, 1);
    double *px, *pf, *pu;
    cudaMallocHost((void**)&px, 24e6);
    cudaMallocHost((void**)&pf, 24e6);
    cudaMallocHost((void**)&pu, 24e6);
    std::copy(x.begin(), x.end(), px);
    std::copy(f.begin(), f.end(), pf);
    for (int mode = 0; mode < 2; ++mode)
        for (int k = 0; k < 4; ++k) {
            auto t0 = std::chrono::steady_clock::now();
            int rc = mode == 0 ? sewald_gpu_full_potential(ctx, &p, x.data(), f.data(), nullptr, N, nullptr, N, 1, 1, u.data())
                               : sewald_gpu_full_potential(ctx, &p, px, pf, nullptr, N, nullptr, N, 1, 1, pu);
            auto t1 = std::chrono::steady_clock::now();
            sewald_timings_c T;
            sewald_gpu_get_timings(ctx, &T);
            std::printf("%s rc=%d wall %.2f ms | h2d %.2f spread %.2f fft %.2f rs+gather %.2f d2h %.2f total %.2f\n",
                        mode == 0 ? "pageable" : "pinned  ", rc,
                        std::chrono::duration<double, std::milli>(t1 - t0).count(), T.h2d_ms, T.spread_ms,
                        T.fft_fwd_ms, T.realspace_ms, T.d2h_ms, T.total_ms);
        }
    return 0;
}
