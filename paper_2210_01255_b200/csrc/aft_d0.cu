// D = 0 (free space) Fourier solve on the zero-padded box with real
// transforms and pruned passes.
//
// Reference: aft_forward / aft_inverse for d = 0 /root/reference/proj/src/fourier.cpp:311-520,
//            scale with the precomputed table :668-720, direct modified kernels :522-666.
//
// The reference transforms the whole padded box (2 M_ext per axis with the
// table, s0 M_ext without) complex-to-complex and keeps the real part. Here:
//   z: D2Z of the M_ext(0) x M_ext(1) input lines only (zero-padded in z),
//   transpose to [c][kz][y][x] (x, y zero-padded: a resident zero block of
//   the out-of-place input buffer, never written),
//   (x, y): one batched 2-D Z2Z over all (c, kz) slices, out of place,
// scale, then the mirror passes (2-D inverse in place, transpose back of the
// x < M_ext(0), y < M_ext(1) corner, Z2D, crop). The strided 1-D pass along x
// that a [x][kz][y] layout needs runs at half the bandwidth of the 2-D plan
// on B200 (tools/cpp/fft_plans.cu), hence the kz-major layout; with x (960 at
// c5) the contiguous axis the 2-D plan runs 1.94 ms vs 2.55 ms per component
// (tools/fft_probe4.py). Keeping Re of
// the C2C inverse equals applying the Hermitian part of the operator,
// H(m) = (G(m) + conj G(-m)) / 2; with the table's Hermitian part Th and
// k(-m) = -k~(m) (Nyquist components keep their sign) this is
// H = fac (D(k) + D(k~)) / 2 Th(m) for the table path and (G(k) + G(k~)) / 2
// for the analytic kernels - both Hermitian, so the C2R inverse reproduces
// the reference's real part.
//
// Layouts: input/output grid [c][x][y][z] (M_ext); R [c][x][y][n2] real;
// Z [c][x][y][h2]; Tin/Tout [c][kz][y][x] with kz < h2, y < n1, x < n0 (x fastest).
#include "engine.h"
#include "aft_d0.h"
#include "modified_kernels.cuh"
#include "options.h"

#include <cmath>
#include <vector>

#include <algorithm>

namespace sewald_b200 {

namespace {

unsigned blocks_for(int64_t n) { return (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 64); }

__global__ void d0_pad_z_kernel(const double* __restrict__ grid, int64_t lines, int m2, int n2,
                                double* __restrict__ R) {
    const int64_t tot = lines * n2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t line = i / n2;
        const int z = (int)(i - line * n2);
        R[i] = z < m2 ? grid[line * m2 + z] : 0.0;
    }
}

__global__ void d0_extract_kernel(const double* __restrict__ R, int64_t lines, int m2, int n2,
                                  double* __restrict__ out) {
    const int64_t tot = lines * m2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t line = i / m2;
        const int z = (int)(i - line * m2);
        out[i] = R[line * n2 + z];
    }
}

// Per (c, y) pair: Z[x][kz] (x < m0, stride m1 h2) <-> T[kz][y][x] (x fastest,
// plane n1 n0). grid (ceil(h2/32), ceil(m0/32), C*m1), block (32, 8).
// rows: y rows of a T plane (n1, or m1 for the compact layout of the fused y path)
template <bool FWD>
__global__ void d0_transpose_kernel(cuDoubleComplex* __restrict__ Z, cuDoubleComplex* __restrict__ T, int m0, int m1,
                                    int n0, int rows, int h2) {
    __shared__ cuDoubleComplex tile[32][33];
    const int cy = blockIdx.z;
    const int c = cy / m1, y = cy - c * m1;
    const int64_t zrow = (int64_t)m1 * h2;  // Z stride between x
    cuDoubleComplex* zs = Z + ((int64_t)c * m0 * m1 + y) * h2;
    const int64_t plane = (int64_t)n0 * rows;
    cuDoubleComplex* ts = T + (int64_t)c * h2 * plane + (int64_t)y * n0;
    const int kz0 = blockIdx.x * 32, x0 = blockIdx.y * 32;
    if (FWD) {
        for (int i = threadIdx.y; i < 32; i += 8) {
            const int x = x0 + i, kz = kz0 + threadIdx.x;
            if (x < m0 && kz < h2) tile[i][threadIdx.x] = zs[x * zrow + kz];
        }
        __syncthreads();
        for (int i = threadIdx.y; i < 32; i += 8) {
            const int kz = kz0 + i, x = x0 + threadIdx.x;
            if (kz < h2 && x < m0) ts[kz * plane + x] = tile[threadIdx.x][i];
        }
    } else {
        for (int i = threadIdx.y; i < 32; i += 8) {
            const int kz = kz0 + i, x = x0 + threadIdx.x;
            if (kz < h2 && x < m0) tile[threadIdx.x][i] = ts[kz * plane + x];
        }
        __syncthreads();
        for (int i = threadIdx.y; i < 32; i += 8) {
            const int x = x0 + i, kz = kz0 + threadIdx.x;
            if (x < m0 && kz < h2) zs[x * zrow + kz] = tile[i][threadIdx.x];
        }
    }
}

// Th[kz][ky][kx] = (T(m) + conj T(-m)) / 2 from the full table [kx][ky][kz].
__global__ void d0_herm_table_kernel(const cuDoubleComplex* __restrict__ T, int n0, int n1, int n2, int h2,
                                     cuDoubleComplex* __restrict__ Th) {
    const int64_t tot = (int64_t)n0 * h2 * n1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        const int kx = (int)(i % n0);
        const int64_t t = i / n0;
        const int ky = (int)(t % n1);
        const int kz = (int)(t / n1);
        const int mx = kx == 0 ? 0 : n0 - kx, my = ky == 0 ? 0 : n1 - ky, mz = kz == 0 ? 0 : n2 - kz;
        const cuDoubleComplex a = T[((int64_t)kx * n1 + ky) * n2 + kz];
        const cuDoubleComplex b = T[((int64_t)mx * n1 + my) * n2 + mz];
        Th[i] = make_cuDoubleComplex(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
    }
}

template <int KIND>
__device__ __forceinline__ void d0_operator(const ModSpec& spec, bool table, double k0, double k1, double k2,
                                            double* re, double* im) {
    if (table)
        diffop_coeffs<KIND>(k0, k1, k2, re, im);
    else
        modified_coeffs<KIND>(spec, k0, k1, k2, re, im);
}

template <int KIND>
__global__ void d0_scale_kernel(ModSpec spec, D0ScaleArgs a, double xi, cuDoubleComplex* __restrict__ data,
                                const cuDoubleComplex* __restrict__ Th) {
    constexpr int NC = KIND == SEWALD_STRESSLET ? 9 : 3;
    constexpr int NG = 3 * NC;
    const int64_t n = (int64_t)a.n0 * a.h2 * a.n1;
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= n) return;
    const int kx = (int)(idx % a.n0);
    const int64_t t = idx / a.n0;
    const int ky = (int)(t % a.n1);
    const int kz = a.kz0 + (int)(t / a.n1);  // a.h2 = kz count of this launch
    const double k0 = a.k0[kx], k1 = a.k1[ky], k2 = a.k2[kz];
    const double wp = a.w0[kx] * a.w1[ky] * a.w2[kz];
    const double kk = k0 * k0 + k1 * k1 + k2 * k2;
    const double q = kk / (4.0 * xi * xi);
    const double g = exp(-q);
    const double scr = KIND == SEWALD_ROTLET ? g : g * (1.0 + q);
    const double fac = scr / (wp * wp) * a.norm;
    const bool table = Th != nullptr;
    double re[NG], im[NG];
    d0_operator<KIND>(spec, table, k0, k1, k2, re, im);
    // Nyquist indices: k(-m) = -k~(m) with the Nyquist components unflipped
    const bool nx = (a.n0 % 2 == 0) && kx == a.n0 / 2;
    const bool ny = (a.n1 % 2 == 0) && ky == a.n1 / 2;
    const bool nz = (a.n2 % 2 == 0) && kz == a.n2 / 2;
    if (nx || ny || nz) {
        double re2[NG], im2[NG];
        d0_operator<KIND>(spec, table, nx ? -k0 : k0, ny ? -k1 : k1, nz ? -k2 : k2, re2, im2);
#pragma unroll
        for (int e = 0; e < NG; ++e) {
            re[e] = 0.5 * (re[e] + re2[e]);
            im[e] = 0.5 * (im[e] + im2[e]);
        }
    }
    if (table) {
        const cuDoubleComplex tv = Th[idx + (int64_t)a.kz0 * a.n0 * a.n1];
#pragma unroll
        for (int e = 0; e < NG; ++e) {
            const double x = re[e], y = im[e];
            re[e] = x * tv.x - y * tv.y;
            im[e] = x * tv.y + y * tv.x;
        }
    }
    cuDoubleComplex in[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) in[c] = data[c * a.cstride + idx];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        double ar = 0.0, ai = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            ar += re[NC * j + c] * in[c].x - im[NC * j + c] * in[c].y;
            ai += re[NC * j + c] * in[c].y + im[NC * j + c] * in[c].x;
        }
        data[j * a.cstride + idx] = make_cuDoubleComplex(fac * ar, fac * ai);
    }
}

// ---------------------------------------------------------------------------
// Fused y path (SEWALD_OPT_D0_YFUSED, default; c5: solve 17.6 -> 12.8 ms,
// the kernel 5.9 ms, shared-memory and barrier bound): per (kz, pair of x
// columns) block, the m1 data rows of every
// input component are loaded (rows m1..N-1 are the zero padding), transformed
// along y (length N, radix-8/4/2 Stockham in shared memory), scaled exactly
// as d0_scale_kernel does, transformed back for the 3 flow components and the
// m1 rows the inverse z pass needs are stored. Replaces the forward y pass,
// the scale kernel and the inverse y pass (three HBM round trips of the
// padded slices) by one; the x passes then run over the m1 data rows only.

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ double2 cmi(double2 a) {
    return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

template <bool INV>
__device__ __forceinline__ void dft4(double2& a0, double2& a1, double2& a2, double2& a3) {
    const double2 t0 = cadd(a0, a2), t1 = csub(a0, a2), t2 = cadd(a1, a3), t3 = cmi<INV>(csub(a1, a3));
    a0 = cadd(t0, t2);
    a2 = csub(t0, t2);
    a1 = cadd(t1, t3);
    a3 = csub(t1, t3);
}

template <int R, bool INV>
__device__ __forceinline__ void dft(double2* a) {
    if (R == 2) {
        const double2 t = a[0];
        a[0] = cadd(t, a[1]);
        a[1] = csub(t, a[1]);
    } else if (R == 4) {
        dft4<INV>(a[0], a[1], a[2], a[3]);
    } else {
        constexpr double h = 0.70710678118654752440;
        double2 e0 = a[0], e1 = a[2], e2 = a[4], e3 = a[6];
        double2 o0 = a[1], o1 = a[3], o2 = a[5], o3 = a[7];
        dft4<INV>(e0, e1, e2, e3);
        dft4<INV>(o0, o1, o2, o3);
        // o_k *= W8^(+-k)
        o1 = cmul(o1, make_double2(h, INV ? h : -h));
        o2 = cmi<INV>(o2);
        o3 = cmul(o3, make_double2(-h, INV ? h : -h));
        a[0] = cadd(e0, o0);
        a[4] = csub(e0, o0);
        a[1] = cadd(e1, o1);
        a[5] = csub(e1, o1);
        a[2] = cadd(e2, o2);
        a[6] = csub(e2, o2);
        a[3] = cadd(e3, o3);
        a[7] = csub(e3, o3);
    }
}

// Shared-memory position of element a of a sequence: one pad slot per 8
// elements, so the stride-8 (NS = 1) and strided-group writes of the Stockham
// stages and the contiguous reads stay free of bank conflicts (16-byte
// elements: 8 lanes per wavefront).
__device__ __forceinline__ int ypad(int a) { return a + (a >> 3); }
template <int N>
constexpr int yseq() { return N + N / 8; }

// Radix of the Stockham stage that starts at subsequence length NS (8 while
// it divides, then 4 / 2), and the offset of that stage's twiddle table in the
// per-stage tables [r - 1][j] = W_N^(j r N / (NS R)) (r-major: the lanes of a
// warp read consecutive j, free of bank conflicts).
constexpr int stage_radix(int N, int NS) { return (N / NS) % 8 == 0 ? 8 : ((N / NS) % 4 == 0 ? 4 : 2); }
constexpr int tw_offset(int N, int NS) {
    int off = 0;
    for (int ns = 1; ns < NS; ns *= stage_radix(N, ns))
        if (ns > 1) off += (stage_radix(N, ns) - 1) * ns;
    return off;
}

// One Stockham stage (radix R, input subsequence length NS) on S sequences of
// length N in shared memory, in place: every thread loads its butterflies,
// the block synchronises, then writes them back.
template <int N, int R, int NS, bool INV, int THREADS, int SMAX>
__device__ __forceinline__ void fft_stage(double2* buf, int S, const double2* tw) {
    constexpr int NB = N / R;                                 // butterflies per sequence
    constexpr int BPT = (SMAX * NB + THREADS - 1) / THREADS;  // per thread (upper bound)
    const int total = S * NB;
    double2 a[BPT][R];
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
        const int b = threadIdx.x + q * THREADS;
        if (b < total) {
            const int s = b / NB, i = b - s * NB;
            const double2* x = buf + s * yseq<N>();
#pragma unroll
            for (int r = 0; r < R; ++r) a[q][r] = x[ypad(i + r * NB)];
        }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
        const int b = threadIdx.x + q * THREADS;
        if (b < total) {
            const int s = b / NB, i = b - s * NB;
            const int j = i % NS;
            if (NS > 1) {
                const double2* tws = tw + tw_offset(N, NS) + j;
#pragma unroll
                for (int r = 1; r < R; ++r) {
                    double2 w = tws[(r - 1) * NS];
                    if (INV) w.y = -w.y;
                    a[q][r] = cmul(a[q][r], w);
                }
            }
            dft<R, INV>(a[q]);
            double2* y = buf + s * yseq<N>();
            const int o = (i / NS) * NS * R + j;
#pragma unroll
            for (int r = 0; r < R; ++r) y[ypad(o + r * NS)] = a[q][r];
        }
    }
    __syncthreads();
}

template <int N, int NS, bool INV, int THREADS, int SMAX>
__device__ __forceinline__ void fft_all(double2* buf, int S, const double2* tw) {
    if constexpr (NS < N) {
        constexpr int R = stage_radix(N, NS);
        fft_stage<N, R, NS, INV, THREADS, SMAX>(buf, S, tw);
        fft_all<N, NS * R, INV, THREADS, SMAX>(buf, S, tw);
    }
}

#ifndef SEWALD_YF_COLS
#define SEWALD_YF_COLS 2
#endif
constexpr int YF_COLS = SEWALD_YF_COLS;  // x columns per block (2: 32-byte row segments, full sectors)

template <int KIND, int N>
struct YFusedCfg {
    static constexpr int NC = KIND == SEWALD_STRESSLET ? 9 : 3;
    static constexpr int SIN = NC * YF_COLS;                      // input sequences
    // one radix-8 butterfly per thread and stage, two above 512 threads
    static constexpr int THREADS = SIN * (N / 8) <= 512 ? SIN * (N / 8) : SIN * (N / 16);
    // + twiddles + the table values of the block's (col, ky) points
    static constexpr size_t SMEM = sizeof(double2) * ((size_t)SIN * (N + N / 8) + N + YF_COLS * N);
};

template <int KIND, int N>
__global__ void __launch_bounds__(YFusedCfg<KIND, N>::THREADS, YFusedCfg<KIND, N>::THREADS <= 384 ? 2 : 1)
d0_yfused_kernel(ModSpec spec, D0ScaleArgs a, double xi, int m1, cuDoubleComplex* __restrict__ data,
                 const cuDoubleComplex* __restrict__ Th, const double2* __restrict__ tw) {
    using Cfg = YFusedCfg<KIND, N>;
    constexpr int NC = Cfg::NC, SIN = Cfg::SIN, THREADS = Cfg::THREADS;
    constexpr int NG = 3 * NC;
    extern __shared__ double2 yb[];  // [c][col][y] (padded), twiddles, table values [col][ky]
    double2* tws = yb + SIN * yseq<N>();
    double2* ths = tws + N;
    const int kx0 = blockIdx.x * YF_COLS;
    const int kzl = blockIdx.y;  // kz of this launch (a.kz0 + kzl globally)
    const int kz = a.kz0 + kzl;
    const int64_t rowbase = (int64_t)kzl * m1;
    // every global read of the block as asynchronous copies into shared memory
    // (all in flight at once), the zero padding with plain stores
    auto cp16 = [](void* dst, const void* src) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src));
    };
    for (int k = threadIdx.x; k < N; k += THREADS) cp16(tws + k, tw + k);
    if (Th)
        for (int e = threadIdx.x; e < YF_COLS * N; e += THREADS) {
            const int col = e % YF_COLS, ky = e / YF_COLS;
            if (kx0 + col < a.n0) cp16(ths + col * N + ky, Th + ((int64_t)kz * a.n1 + ky) * a.n0 + kx0 + col);
        }
    for (int e = threadIdx.x; e < SIN * N; e += THREADS) {
        const int col = e % YF_COLS;
        const int t = e / YF_COLS;
        const int y = t % N, c = t / N;
        double2* dst = yb + (c * YF_COLS + col) * yseq<N>() + ypad(y);
        if (y < m1 && kx0 + col < a.n0)
            cp16(dst, data + c * a.cstride + (rowbase + y) * a.n0 + kx0 + col);
        else
            *dst = make_double2(0.0, 0.0);
    }
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
    fft_all<N, 1, false, THREADS, SIN>(yb, SIN, tws);
    // scale (d0_scale_kernel per (col, ky)): 3 outputs into sequences 0..2
    for (int e = threadIdx.x; e < YF_COLS * N; e += THREADS) {
        const int col = e / N, ky = e - col * N;
        const int kx = kx0 + col;
        if (kx >= a.n0) continue;
        const double k0 = a.k0[kx], k1 = a.k1[ky], k2 = a.k2[kz];
        const double wp = a.w0[kx] * a.w1[ky] * a.w2[kz];
        const double kk = k0 * k0 + k1 * k1 + k2 * k2;
        const double q = kk / (4.0 * xi * xi);
        const double g = exp(-q);
        const double scr = KIND == SEWALD_ROTLET ? g : g * (1.0 + q);
        const double fac = scr / (wp * wp) * a.norm;
        const bool table = Th != nullptr;
        double re[NG], im[NG];
        d0_operator<KIND>(spec, table, k0, k1, k2, re, im);
        const bool nx = (a.n0 % 2 == 0) && kx == a.n0 / 2;
        const bool ny = (a.n1 % 2 == 0) && ky == a.n1 / 2;
        const bool nz = (a.n2 % 2 == 0) && kz == a.n2 / 2;
        if (nx || ny || nz) {
            double re2[NG], im2[NG];
            d0_operator<KIND>(spec, table, nx ? -k0 : k0, ny ? -k1 : k1, nz ? -k2 : k2, re2, im2);
#pragma unroll
            for (int q2 = 0; q2 < NG; ++q2) {
                re[q2] = 0.5 * (re[q2] + re2[q2]);
                im[q2] = 0.5 * (im[q2] + im2[q2]);
            }
        }
        if (table) {
            const double2 tv = ths[col * N + ky];
#pragma unroll
            for (int q2 = 0; q2 < NG; ++q2) {
                const double x = re[q2], y = im[q2];
                re[q2] = x * tv.x - y * tv.y;
                im[q2] = x * tv.y + y * tv.x;
            }
        }
        double2 in[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) in[c] = yb[(c * YF_COLS + col) * yseq<N>() + ypad(ky)];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            double ar = 0.0, ai = 0.0;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                ar += re[NC * j + c] * in[c].x - im[NC * j + c] * in[c].y;
                ai += re[NC * j + c] * in[c].y + im[NC * j + c] * in[c].x;
            }
            yb[(j * YF_COLS + col) * yseq<N>() + ypad(ky)] = make_double2(fac * ar, fac * ai);
        }
    }
    __syncthreads();
    fft_all<N, 1, true, THREADS, SIN>(yb, 3 * YF_COLS, tws);
    for (int e = threadIdx.x; e < 3 * YF_COLS * m1; e += THREADS) {
        const int col = e % YF_COLS;
        const int t = e / YF_COLS;
        const int y = t % m1, j = t / m1;
        if (kx0 + col >= a.n0) continue;
        const double2 v = yb[(j * YF_COLS + col) * yseq<N>() + ypad(y)];
        data[j * a.cstride + (rowbase + y) * a.n0 + kx0 + col] = make_cuDoubleComplex(v.x, v.y);
    }
}

template <int KIND, int N>
void launch_yfused(const ModSpec& spec, const D0ScaleArgs& sa, double xi, int m1, int nkz, cuDoubleComplex* data,
                   const cuDoubleComplex* th, const double2* tw, cudaStream_t st) {
    using Cfg = YFusedCfg<KIND, N>;
    auto kern = d0_yfused_kernel<KIND, N>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
    const dim3 grid((unsigned)((sa.n0 + YF_COLS - 1) / YF_COLS), (unsigned)nkz);
    kern<<<grid, Cfg::THREADS, Cfg::SMEM, st>>>(spec, sa, xi, m1, data, th, tw);
}

template <int KIND>
void launch_yfused_n(int N, const ModSpec& spec, const D0ScaleArgs& sa, double xi, int m1, int nkz,
                     cuDoubleComplex* data, const cuDoubleComplex* th, const double2* tw, cudaStream_t st) {
    switch (N) {
        case 256: launch_yfused<KIND, 256>(spec, sa, xi, m1, nkz, data, th, tw, st); break;
        case 512: launch_yfused<KIND, 512>(spec, sa, xi, m1, nkz, data, th, tw, st); break;
        default: launch_yfused<KIND, 1024>(spec, sa, xi, m1, nkz, data, th, tw, st); break;
    }
}

bool yfused_ok(int n1, int C) {
    if (!(n1 == 256 || n1 == 512 || n1 == 1024)) return false;
    // shared memory: C x 2 columns x n1 complex
    return ((size_t)C * YF_COLS * (n1 + n1 / 8) + n1 + YF_COLS * n1) * sizeof(double2) <= 200 * 1024;
}

void fft_check(cufftResult r, const char* what) {
    if (r != CUFFT_SUCCESS) throw EngineError(SEWALD_ECUFFT, std::string("cuFFT: ") + what);
}

}  // namespace

D0Real::~D0Real() {
    for (auto h : plans) cufftDestroy(h);
}

void D0Real::setup(const int m_[3], const int n_[3], int C_, cudaStream_t st) {
    for (int ax = 0; ax < 3; ++ax) {
        m[ax] = m_[ax];
        n[ax] = n_[ax];
    }
    C = C_;
    h2 = n[2] / 2 + 1;
    yfused = option(SEWALD_OPT_D0_YFUSED) != 0 && yfused_ok(n[1], C);
    const int64_t lines_in = (int64_t)C * m[0] * m[1], lines_out = (int64_t)3 * m[0] * m[1];
    R.ensure(sizeof(double) * lines_in * n[2]);
    Z.ensure(sizeof(cuDoubleComplex) * lines_in * h2);
    // [c][kz][y][x] planes: all n1 rows, or the m1 data rows for the fused y path
    const int64_t slab = (int64_t)h2 * n[0] * (yfused ? m[1] : n[1]);
    Tin.ensure(sizeof(cuDoubleComplex) * C * slab);
    Tout.ensure(sizeof(cuDoubleComplex) * C * slab);
    cuda_check(cudaMemsetAsync(Tin.ptr, 0, sizeof(cuDoubleComplex) * C * slab, st), "d0 Tin zero");
    if (yfused) {  // per-stage twiddle tables (stage_radix / tw_offset order), padded to n1 entries
        const int N = n[1];
        std::vector<double2> h;
        for (int ns = 1; ns < N; ns *= stage_radix(N, ns)) {
            const int R = stage_radix(N, ns);
            if (ns == 1) continue;
            for (int r = 1; r < R; ++r)
                for (int j = 0; j < ns; ++j) {
                    const long double ang =
                        -2.0L * 3.14159265358979323846264338327950288L * ((long long)j * r * (N / (ns * R))) / N;
                    h.push_back(make_double2((double)cosl(ang), (double)sinl(ang)));
                }
        }
        h.resize(N, make_double2(0.0, 0.0));
        tw.ensure(sizeof(double2) * n[1]);
        cuda_check(cudaMemcpyAsync(tw.ptr, h.data(), sizeof(double2) * n[1], cudaMemcpyHostToDevice, st), "d0 tw");
        cuda_check(cudaStreamSynchronize(st), "d0 tw");
    }

    size_t ws = 0, w = 0;
    auto mk = [&](cufftHandle& h, int rank, const int* nl, const int* inem, long long is, long long id,
                  const int* onem, long long os, long long od, cufftType ty, long long batch) {
        fft_check(cufftCreate(&h), "create");
        plans.push_back(h);
        fft_check(cufftSetAutoAllocation(h, 0), "auto alloc");
        long long nn[2], ie[2], oe[2];
        for (int r = 0; r < rank; ++r) {
            nn[r] = nl[r];
            ie[r] = inem[r];
            oe[r] = onem[r];
        }
        fft_check(cufftMakePlanMany64(h, rank, nn, ie, is, id, oe, os, od, ty, batch, &w), "plan");
        fft_check(cufftSetStream(h, st), "stream");
        ws = std::max(ws, w);
    };
    int e_n2[1] = {n[2]}, e_h2[1] = {h2};
    mk(pz_f, 1, n + 2, e_n2, 1, n[2], e_h2, 1, h2, CUFFT_D2Z, lines_in);
    mk(pz_i, 1, n + 2, e_h2, 1, h2, e_n2, 1, n[2], CUFFT_Z2D, lines_out);
    if (yfused) {
        // x transforms of the m1 data rows of every (c, kz) plane (contiguous rows)
        const int e_n0[1] = {n[0]};
        mk(px_f, 1, n, e_n0, 1, n[0], e_n0, 1, n[0], CUFFT_Z2Z, (long long)C * h2 * m[1]);
        mk(px_i, 1, n, e_n0, 1, n[0], e_n0, 1, n[0], CUFFT_Z2Z, (long long)3 * h2 * m[1]);
    } else {
        const int64_t plane = (int64_t)n[0] * n[1];
        const int nyx[2] = {n[1], n[0]};  // [y][x] slices, x fastest
        mk(pxy_f, 2, nyx, nyx, 1, plane, nyx, 1, plane, CUFFT_Z2Z, (long long)C * h2);
        mk(pxy_i, 2, nyx, nyx, 1, plane, nyx, 1, plane, CUFFT_Z2Z, (long long)3 * h2);
    }
    work.ensure(std::max<size_t>(ws, 16));
    for (auto h : plans) fft_check(cufftSetWorkArea(h, work.ptr), "work area");
}

void D0Real::build_herm_table(const cuDoubleComplex* full, cudaStream_t st) {
    const int64_t tot = (int64_t)n[0] * h2 * n[1];
    Th.ensure(sizeof(cuDoubleComplex) * tot);
    d0_herm_table_kernel<<<blocks_for(tot), 256, 0, st>>>(full, n[0], n[1], n[2], h2, Th.as<cuDoubleComplex>());
    cuda_check(cudaGetLastError(), "d0 herm table");
}

int D0Real::solve(const double* grid, const ModSpec& spec, int kind, double xi, const D0ScaleArgs& sa_in, bool table,
                  double* flow, cudaStream_t st) {
    const int64_t lines_in = (int64_t)C * m[0] * m[1], lines_out = (int64_t)3 * m[0] * m[1];
    const int rows = yfused ? m[1] : n[1];  // y rows of a T plane
    const int64_t slab = (int64_t)h2 * n[0] * rows;
    double* r = R.as<double>();
    cuDoubleComplex* z = Z.as<cuDoubleComplex>();
    cuDoubleComplex* ti = Tin.as<cuDoubleComplex>();
    cuDoubleComplex* to = Tout.as<cuDoubleComplex>();
    int launches = 0;
    // forward
    d0_pad_z_kernel<<<blocks_for(lines_in * n[2]), 256, 0, st>>>(grid, lines_in, m[2], n[2], r);
    cufftSetStream(pz_f, st);
    fft_check(cufftExecD2Z(pz_f, r, z), "d0 z forward");
    const dim3 tb(32, 8), tg((h2 + 31) / 32, (m[0] + 31) / 32, C * m[1]);
    d0_transpose_kernel<true><<<tg, tb, 0, st>>>(z, ti, m[0], m[1], n[0], rows, h2);
    D0ScaleArgs sa = sa_in;
    sa.n0 = n[0];
    sa.n1 = n[1];
    sa.n2 = n[2];
    sa.h2 = h2;
    sa.kz0 = 0;
    sa.cstride = slab;
    const cuDoubleComplex* th = table ? Th.as<cuDoubleComplex>() : nullptr;
    if (yfused) {
        // x forward over the data rows, fused y transform / scale / inverse y, x inverse
        cufftSetStream(px_f, st);
        fft_check(cufftExecZ2Z(px_f, ti, to, CUFFT_FORWARD), "d0 x forward");
        const double2* twp = tw.as<double2>();
        switch (kind) {
            case SEWALD_STOKESLET:
                launch_yfused_n<SEWALD_STOKESLET>(n[1], spec, sa, xi, m[1], h2, to, th, twp, st);
                break;
            case SEWALD_ROTLET: launch_yfused_n<SEWALD_ROTLET>(n[1], spec, sa, xi, m[1], h2, to, th, twp, st); break;
            default: launch_yfused_n<SEWALD_STRESSLET>(n[1], spec, sa, xi, m[1], h2, to, th, twp, st); break;
        }
        cufftSetStream(px_i, st);
        fft_check(cufftExecZ2Z(px_i, to, to, CUFFT_INVERSE), "d0 x inverse");
        launches += 3;  // own kernels only (cuFFT launches are library work)
    } else {
        cufftSetStream(pxy_f, st);
        fft_check(cufftExecZ2Z(pxy_f, ti, to, CUFFT_FORWARD), "d0 xy forward");
        launches += 2;
        const unsigned sb = (unsigned)((slab + 127) / 128);
        switch (kind) {
            case SEWALD_STOKESLET: d0_scale_kernel<SEWALD_STOKESLET><<<sb, 128, 0, st>>>(spec, sa, xi, to, th); break;
            case SEWALD_ROTLET: d0_scale_kernel<SEWALD_ROTLET><<<sb, 128, 0, st>>>(spec, sa, xi, to, th); break;
            default: d0_scale_kernel<SEWALD_STRESSLET><<<sb, 128, 0, st>>>(spec, sa, xi, to, th); break;
        }
        ++launches;
        // inverse (3 flow components)
        cufftSetStream(pxy_i, st);
        fft_check(cufftExecZ2Z(pxy_i, to, to, CUFFT_INVERSE), "d0 xy inverse");
    }
    const dim3 tgi((h2 + 31) / 32, (m[0] + 31) / 32, 3 * m[1]);
    d0_transpose_kernel<false><<<tgi, tb, 0, st>>>(z, to, m[0], m[1], n[0], rows, h2);
    ++launches;
    cufftSetStream(pz_i, st);
    fft_check(cufftExecZ2D(pz_i, z, r), "d0 z inverse");
    d0_extract_kernel<<<blocks_for(lines_out * m[2]), 256, 0, st>>>(r, lines_out, m[2], n[2], flow);
    ++launches;
    cuda_check(cudaGetLastError(), "d0 solve");
    return launches;
}


// ---------------------------------------------------------------------------
// slab-distributed stages
// ---------------------------------------------------------------------------

namespace {

__device__ __forceinline__ int owner_of(const SlabBounds& b, int i) {
    int r = 0;
    while (r + 1 < b.world && b.b[r + 1] <= i) ++r;
    return r;
}

// Z slab [C][nxs][m1][h2] -> send chunks q: [C][nxs][m1][kz - ka_q]
__global__ void d0_pack_fwd_kernel(const cuDoubleComplex* __restrict__ Z, int C, int nxs, int m1, int h2,
                                   SlabBounds kzb, cuDoubleComplex* __restrict__ send) {
    const int64_t tot = (int64_t)C * nxs * m1 * h2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        const int kz = (int)(i % h2);
        const int64_t line = i / h2;  // (c, xs, y)
        const int q = owner_of(kzb, kz);
        const int ka = kzb.b[q], nk = kzb.b[q + 1] - ka;
        send[(int64_t)C * nxs * m1 * ka + line * nk + (kz - ka)] = Z[i];
    }
}

// recv chunks p: [C][nxs_p][m1][nk] -> Tin [C][nk][n1][n0] (x < m0, y < m1)
__global__ void d0_unpack_mid_kernel(const cuDoubleComplex* __restrict__ recv, int C, int m0, int m1, int n0,
                                     int n1, int nk, SlabBounds xbd, cuDoubleComplex* __restrict__ Tin) {
    const int64_t tot = (int64_t)C * nk * m1 * m0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(i % m0);
        int64_t t = i / m0;
        const int y = (int)(t % m1);
        t /= m1;
        const int kl = (int)(t % nk);
        const int c = (int)(t / nk);
        const int p = owner_of(xbd, x);
        const int xa = xbd.b[p], nxs = xbd.b[p + 1] - xa;
        const int64_t src = (int64_t)C * m1 * nk * xa + (((int64_t)c * nxs + (x - xa)) * m1 + y) * nk + kl;
        Tin[(((int64_t)c * nk + kl) * n1 + y) * n0 + x] = recv[src];
    }
}

// Tout [3][nk][n1][n0] (x < m0, y < m1) -> send chunks q: [3][nk][nxs_q][m1]
__global__ void d0_pack_mid_kernel(const cuDoubleComplex* __restrict__ Tout, int m0, int m1, int n0, int n1,
                                   int nk, SlabBounds xbd, cuDoubleComplex* __restrict__ send) {
    const int64_t tot = (int64_t)3 * nk * m0 * m1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        const int y = (int)(i % m1);
        int64_t t = i / m1;
        const int x = (int)(t % m0);
        const int64_t ck = t / m0;  // c * nk + kl
        const int q = owner_of(xbd, x);
        const int xa = xbd.b[q], nxs = xbd.b[q + 1] - xa;
        send[(int64_t)3 * nk * m1 * xa + (ck * nxs + (x - xa)) * m1 + y] = Tout[(ck * n1 + y) * n0 + x];
    }
}

// recv chunks p: [3][nk_p][nxs][m1] -> Z slab [3][nxs][m1][h2]
__global__ void d0_unpack_inv_kernel(const cuDoubleComplex* __restrict__ recv, int nxs, int m1, int h2,
                                     SlabBounds kzb, cuDoubleComplex* __restrict__ Z) {
    const int64_t tot = (int64_t)3 * nxs * m1 * h2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        const int kz = (int)(i % h2);
        int64_t t = i / h2;
        const int y = (int)(t % m1);
        t /= m1;
        const int xs = (int)(t % nxs);
        const int c = (int)(t / nxs);
        const int p = owner_of(kzb, kz);
        const int ka = kzb.b[p], nk = kzb.b[p + 1] - ka;
        Z[i] = recv[(int64_t)3 * nxs * m1 * ka + (((int64_t)c * nk + (kz - ka)) * nxs + xs) * m1 + y];
    }
}

}  // namespace

D0SlabPlan::~D0SlabPlan() {
    for (auto h : plans) cufftDestroy(h);
}

void D0Real::slab_plans(int nxs, int nk, cudaStream_t st) {
    D0SlabPlan& S = slab;
    if (S.nxs == nxs && S.nk == nk) return;
    for (auto h : S.plans) cufftDestroy(h);
    S.plans.clear();
    S.nxs = nxs;
    S.nk = nk;
    const int64_t lin = (int64_t)C * nxs * m[1], lout = (int64_t)3 * nxs * m[1];
    S.R.ensure(sizeof(double) * std::max<int64_t>(lin, 1) * n[2]);
    S.Z.ensure(sizeof(cuDoubleComplex) * std::max<int64_t>(lin, 1) * h2);
    const int64_t plane = (int64_t)n[0] * n[1];
    S.Tin.ensure(sizeof(cuDoubleComplex) * C * std::max(nk, 1) * plane);
    S.Tout.ensure(sizeof(cuDoubleComplex) * C * std::max(nk, 1) * plane);
    // the x >= m0 / y >= m1 parts of Tin are a resident zero block
    cuda_check(cudaMemsetAsync(S.Tin.ptr, 0, sizeof(cuDoubleComplex) * C * std::max(nk, 1) * plane, st),
               "slab Tin zero");
    size_t ws = 0, w = 0;
    auto mk = [&](cufftHandle& h, int rank, const int* nl, long long is, long long id, long long os, long long od,
                  cufftType ty, long long batch, const int* inem, const int* onem) {
        fft_check(cufftCreate(&h), "create");
        S.plans.push_back(h);
        fft_check(cufftSetAutoAllocation(h, 0), "auto alloc");
        long long nn[2], ie[2], oe[2];
        for (int r = 0; r < rank; ++r) {
            nn[r] = nl[r];
            ie[r] = inem[r];
            oe[r] = onem[r];
        }
        fft_check(cufftMakePlanMany64(h, rank, nn, ie, is, id, oe, os, od, ty, batch, &w), "slab plan");
        fft_check(cufftSetStream(h, st), "stream");
        ws = std::max(ws, w);
    };
    int e_n2[1] = {n[2]}, e_h2[1] = {h2};
    if (lin > 0) {
        mk(S.pz_f, 1, n + 2, 1, n[2], 1, h2, CUFFT_D2Z, lin, e_n2, e_h2);
        mk(S.pz_i, 1, n + 2, 1, h2, 1, n[2], CUFFT_Z2D, lout, e_h2, e_n2);
    }
    if (nk > 0) {
        const int nyx[2] = {n[1], n[0]};
        mk(S.pxy_f, 2, nyx, 1, plane, 1, plane, CUFFT_Z2Z, (long long)C * nk, nyx, nyx);
        mk(S.pxy_i, 2, nyx, 1, plane, 1, plane, CUFFT_Z2Z, (long long)3 * nk, nyx, nyx);
    }
    S.work.ensure(std::max<size_t>(ws, 16));
    for (auto h : S.plans) fft_check(cufftSetWorkArea(h, S.work.ptr), "work area");
}

int D0Real::slab_forward(const double* grid_slab, int xa, int xb, const SlabBounds& kzb, cuDoubleComplex* send,
                         cudaStream_t st) {
    const int nxs = xb - xa;
    const int nk = slab.nk < 0 ? 0 : slab.nk;
    slab_plans(nxs, std::max(slab.nk, 0), st);
    (void)nk;
    const int64_t lines = (int64_t)C * nxs * m[1];
    if (lines == 0) return 0;
    double* r = slab.R.as<double>();
    cuDoubleComplex* z = slab.Z.as<cuDoubleComplex>();
    d0_pad_z_kernel<<<blocks_for(lines * n[2]), 256, 0, st>>>(grid_slab, lines, m[2], n[2], r);
    cufftSetStream(slab.pz_f, st);
    fft_check(cufftExecD2Z(slab.pz_f, r, z), "slab z forward");
    d0_pack_fwd_kernel<<<blocks_for(lines * h2), 256, 0, st>>>(z, C, nxs, m[1], h2, kzb, send);
    cuda_check(cudaGetLastError(), "slab forward");
    return 2;
}

int D0Real::slab_middle(const cuDoubleComplex* recv, const SlabBounds& xbd, int ka, int kb, const ModSpec& spec,
                        int kind, double xi, const D0ScaleArgs& sa_in, bool table, cuDoubleComplex* send,
                        cudaStream_t st) {
    const int nk = kb - ka;
    slab_plans(std::max(slab.nxs, 0), nk, st);
    if (nk == 0) return 0;
    const int64_t plane = (int64_t)n[0] * n[1];
    cuDoubleComplex* ti = slab.Tin.as<cuDoubleComplex>();
    cuDoubleComplex* to = slab.Tout.as<cuDoubleComplex>();
    const int64_t nin = (int64_t)C * nk * m[0] * m[1];
    d0_unpack_mid_kernel<<<blocks_for(nin), 256, 0, st>>>(recv, C, m[0], m[1], n[0], n[1], nk, xbd, ti);
    cufftSetStream(slab.pxy_f, st);
    fft_check(cufftExecZ2Z(slab.pxy_f, ti, to, CUFFT_FORWARD), "slab xy forward");
    D0ScaleArgs sa = sa_in;
    sa.n0 = n[0];
    sa.n1 = n[1];
    sa.n2 = n[2];
    sa.h2 = nk;
    sa.kz0 = ka;
    sa.cstride = (int64_t)nk * plane;
    const cuDoubleComplex* th = table ? Th.as<cuDoubleComplex>() : nullptr;
    const unsigned sb = (unsigned)((sa.cstride + 127) / 128);
    switch (kind) {
        case SEWALD_STOKESLET: d0_scale_kernel<SEWALD_STOKESLET><<<sb, 128, 0, st>>>(spec, sa, xi, to, th); break;
        case SEWALD_ROTLET: d0_scale_kernel<SEWALD_ROTLET><<<sb, 128, 0, st>>>(spec, sa, xi, to, th); break;
        default: d0_scale_kernel<SEWALD_STRESSLET><<<sb, 128, 0, st>>>(spec, sa, xi, to, th); break;
    }
    cufftSetStream(slab.pxy_i, st);
    fft_check(cufftExecZ2Z(slab.pxy_i, to, to, CUFFT_INVERSE), "slab xy inverse");
    const int64_t nout = (int64_t)3 * nk * m[0] * m[1];
    d0_pack_mid_kernel<<<blocks_for(nout), 256, 0, st>>>(to, m[0], m[1], n[0], n[1], nk, xbd, send);
    cuda_check(cudaGetLastError(), "slab middle");
    return 3;
}

int D0Real::slab_inverse(const cuDoubleComplex* recv, int xa, int xb, const SlabBounds& kzb, double* flow_slab,
                         cudaStream_t st) {
    const int nxs = xb - xa;
    slab_plans(nxs, std::max(slab.nk, 0), st);
    const int64_t lines = (int64_t)3 * nxs * m[1];
    if (lines == 0) return 0;
    cuDoubleComplex* z = slab.Z.as<cuDoubleComplex>();
    double* r = slab.R.as<double>();
    d0_unpack_inv_kernel<<<blocks_for(lines * h2), 256, 0, st>>>(recv, nxs, m[1], h2, kzb, z);
    cufftSetStream(slab.pz_i, st);
    fft_check(cufftExecZ2D(slab.pz_i, z, r), "slab z inverse");
    d0_extract_kernel<<<blocks_for(lines * m[2]), 256, 0, st>>>(r, lines, m[2], n[2], flow_slab);
    cuda_check(cudaGetLastError(), "slab inverse");
    return 2;
}

}  // namespace sewald_b200
