// Device-side shared definitions of the B200 Spectral Ewald engine: grid and
// window descriptors passed BY VALUE as kernel parameters (they live in the
// constant bank, so warp-uniform reads are broadcasts), and the per-axis
// stencil rule of the reference.
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

namespace sewald_b200 {

constexpr int kMaxP = 40;        // largest window support handled on device
constexpr int kMaxNu = 10;       // PKB degree cap (window.cpp:82)

// Grid geometry: periodic axes wrap with origin 0, free axes start at
// -pad/2 (fourier.cpp:174-185).
struct DevGrid {
    int d;
    int n[3];          // M_ext
    double h;
    double inv_h_unused;
    double x0[3];      // 0 on periodic axes, -pad/2 on free axes
    double L[3];       // primary cell
};

// Window: exact KB, PKB (piecewise polynomial) or truncated Gaussian
// (window.cpp:88-157). coef holds the PKB table row-major (P rows of nu+1).
struct DevWindow {
    int kind;
    int P;
    int nu;
    double h;
    double half_width;
    double beta;
    double i0_beta;
    double alpha;
    double coef[kMaxP * (kMaxNu + 1)];
};

// Window value at offset r (window.cpp:140-157, :88-94). Arithmetic follows
// the reference expression order.
__device__ __forceinline__ double window_eval(const DevWindow& w, double r) {
    if (fabs(r) > w.half_width) return 0.0;
    if (w.kind == 1) {  // PKB
        int l = (int)floor(r / w.h);
        l = l < -w.P / 2 ? -w.P / 2 : (l > w.P / 2 - 1 ? w.P / 2 - 1 : l);
        const double u = 2.0 * (r - l * w.h) / w.h - 1.0;
        const double* c = w.coef + (l + w.P / 2) * (w.nu + 1);
        double acc = 0.0;
        for (int i = w.nu; i >= 0; --i) acc = c[i] + acc * u;
        return acc;
    }
    const double t = r / w.half_width;
    if (w.kind == 2) return exp(-w.alpha * t * t);  // TG
    const double arg = fmax(1.0 - t * t, 0.0);      // exact KB
    return cyl_bessel_i0(w.beta * sqrt(arg)) / w.i0_beta;
}

// The P taps window_eval(w, ((j0 + p) - rel) * h), p < P, into out[0..P):
// the same per-tap arithmetic (bit-identical values), four taps interleaved
// so their division and Horner chains overlap (a thread evaluating its taps
// one after another is latency-bound: the taps kernel of the c2 gather took
// 0.41 ms for 1e6 targets).
__device__ __forceinline__ void window_taps(const DevWindow& w, int j0, double rel, double h, double* out,
                                            int stride = 1, int p_begin = 0, int p_end = -1) {
    const int P = p_end < 0 ? w.P : p_end;
    int p = p_begin;
    if (w.kind == 1) {
        for (; p + 4 <= P; p += 4) {
            double r[4], u[4], acc[4];
            const double* c[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                r[q] = ((double)(j0 + p + q) - rel) * h;
                int l = (int)floor(r[q] / w.h);
                l = l < -w.P / 2 ? -w.P / 2 : (l > w.P / 2 - 1 ? w.P / 2 - 1 : l);
                u[q] = 2.0 * (r[q] - l * w.h) / w.h - 1.0;
                c[q] = w.coef + (l + w.P / 2) * (w.nu + 1);
                acc[q] = 0.0;
            }
            for (int i = w.nu; i >= 0; --i)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[q] = c[q][i] + acc[q] * u[q];
#pragma unroll
            for (int q = 0; q < 4; ++q) out[(p + q) * stride] = fabs(r[q]) > w.half_width ? 0.0 : acc[q];
        }
    }
    for (; p < P; ++p) out[p * stride] = window_eval(w, ((double)(j0 + p) - rel) * h);
}

// Stencil start index and relative coordinate along one axis
// (fourier.cpp:174-176): rel = (x - x0)/h, j0 = ceil(rel - P/2).
__device__ __forceinline__ void stencil_origin(const DevGrid& g, int P, int ax, double x,
                                               int& j0, double& rel) {
    rel = (x - g.x0[ax]) / g.h;
    j0 = (int)ceil(rel - 0.5 * P);
}

__device__ __forceinline__ int wrap_index(int j, int n) {
    j %= n;
    return j < 0 ? j + n : j;
}

}  // namespace sewald_b200
