// D = 0 (free space) Fourier solve on the zero-padded box with real
// transforms and pruned passes.
//
// Reference: aft_forward / aft_inverse for d = 0 /root/reference/proj/src/fourier.cpp:311-520,
//            scale with the precomputed table :668-720, direct modified kernels :522-666.
//
// The reference transforms the whole padded box (2 M_ext per axis with the
// table, s0 M_ext without) complex-to-complex and keeps the real part. Here:
//   z: D2Z of the M_ext(0) x M_ext(1) input lines only (zero-padded in z),
//   transpose to [c][kz][x][y] (x, y zero-padded: a resident zero block of
//   the out-of-place input buffer, never written),
//   (x, y): one batched 2-D Z2Z over all (c, kz) slices, out of place,
// scale, then the mirror passes (2-D inverse in place, transpose back of the
// x < M_ext(0), y < M_ext(1) corner, Z2D, crop). The strided 1-D pass along x
// that a [x][kz][y] layout needs runs at half the bandwidth of the 2-D plan
// on B200 (tools/cpp/fft_plans.cu), hence the kz-major layout. Keeping Re of
// the C2C inverse equals applying the Hermitian part of the operator,
// H(m) = (G(m) + conj G(-m)) / 2; with the table's Hermitian part Th and
// k(-m) = -k~(m) (Nyquist components keep their sign) this is
// H = fac (D(k) + D(k~)) / 2 Th(m) for the table path and (G(k) + G(k~)) / 2
// for the analytic kernels - both Hermitian, so the C2R inverse reproduces
// the reference's real part.
//
// Layouts: input/output grid [c][x][y][z] (M_ext); R [c][x][y][n2] real;
// Z [c][x][y][h2]; Tin/Tout [c][kz][x][y] with kz < h2, x < n0, y < n1.
#include "engine.h"
#include "aft_d0.h"
#include "modified_kernels.cuh"

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

// Per (c, x) slab: Z[y][kz] (m1 x h2) <-> T[kz][x][y] (row stride n0 n1),
// y < m1 only. grid (ceil(h2/32), ceil(m1/32), C*m0), block (32, 8).
template <bool FWD>
__global__ void d0_transpose_kernel(cuDoubleComplex* __restrict__ Z, cuDoubleComplex* __restrict__ T, int m0, int m1,
                                    int n0, int n1, int h2) {
    __shared__ cuDoubleComplex tile[32][33];
    const int cx = blockIdx.z;
    const int c = cx / m0, x = cx - c * m0;
    cuDoubleComplex* zs = Z + (int64_t)cx * m1 * h2;
    const int64_t plane = (int64_t)n0 * n1;
    cuDoubleComplex* ts = T + (int64_t)c * h2 * plane + (int64_t)x * n1;
    const int kz0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
    if (FWD) {
        for (int i = threadIdx.y; i < 32; i += 8) {
            const int y = y0 + i, kz = kz0 + threadIdx.x;
            if (y < m1 && kz < h2) tile[i][threadIdx.x] = zs[(int64_t)y * h2 + kz];
        }
        __syncthreads();
        for (int i = threadIdx.y; i < 32; i += 8) {
            const int kz = kz0 + i, y = y0 + threadIdx.x;
            if (kz < h2 && y < m1) ts[kz * plane + y] = tile[threadIdx.x][i];
        }
    } else {
        for (int i = threadIdx.y; i < 32; i += 8) {
            const int kz = kz0 + i, y = y0 + threadIdx.x;
            if (kz < h2 && y < m1) tile[threadIdx.x][i] = ts[kz * plane + y];
        }
        __syncthreads();
        for (int i = threadIdx.y; i < 32; i += 8) {
            const int y = y0 + i, kz = kz0 + threadIdx.x;
            if (y < m1 && kz < h2) zs[(int64_t)y * h2 + kz] = tile[i][threadIdx.x];
        }
    }
}

// Th[kz][kx][ky] = (T(m) + conj T(-m)) / 2 from the full table [kx][ky][kz].
__global__ void d0_herm_table_kernel(const cuDoubleComplex* __restrict__ T, int n0, int n1, int n2, int h2,
                                     cuDoubleComplex* __restrict__ Th) {
    const int64_t tot = (int64_t)n0 * h2 * n1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        const int ky = (int)(i % n1);
        const int64_t t = i / n1;
        const int kx = (int)(t % n0);
        const int kz = (int)(t / n0);
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
    const int ky = (int)(idx % a.n1);
    const int64_t t = idx / a.n1;
    const int kx = (int)(t % a.n0);
    const int kz = (int)(t / a.n0);
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
        const cuDoubleComplex tv = Th[idx];
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
    const int64_t lines_in = (int64_t)C * m[0] * m[1], lines_out = (int64_t)3 * m[0] * m[1];
    R.ensure(sizeof(double) * lines_in * n[2]);
    Z.ensure(sizeof(cuDoubleComplex) * lines_in * h2);
    const int64_t slab = (int64_t)h2 * n[0] * n[1];
    Tin.ensure(sizeof(cuDoubleComplex) * C * slab);
    Tout.ensure(sizeof(cuDoubleComplex) * C * slab);
    cuda_check(cudaMemsetAsync(Tin.ptr, 0, sizeof(cuDoubleComplex) * C * slab, st), "d0 Tin zero");

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
    const int64_t plane = (int64_t)n[0] * n[1];
    mk(pxy_f, 2, n, n, 1, plane, n, 1, plane, CUFFT_Z2Z, (long long)C * h2);
    mk(pxy_i, 2, n, n, 1, plane, n, 1, plane, CUFFT_Z2Z, (long long)3 * h2);
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
    const int64_t slab = (int64_t)h2 * n[0] * n[1];
    double* r = R.as<double>();
    cuDoubleComplex* z = Z.as<cuDoubleComplex>();
    cuDoubleComplex* ti = Tin.as<cuDoubleComplex>();
    cuDoubleComplex* to = Tout.as<cuDoubleComplex>();
    int launches = 0;
    // forward
    d0_pad_z_kernel<<<blocks_for(lines_in * n[2]), 256, 0, st>>>(grid, lines_in, m[2], n[2], r);
    fft_check(cufftExecD2Z(pz_f, r, z), "d0 z forward");
    const dim3 tb(32, 8), tg((h2 + 31) / 32, (m[1] + 31) / 32, C * m[0]);
    d0_transpose_kernel<true><<<tg, tb, 0, st>>>(z, ti, m[0], m[1], n[0], n[1], h2);
    fft_check(cufftExecZ2Z(pxy_f, ti, to, CUFFT_FORWARD), "d0 xy forward");
    launches += 2;  // own kernels only (cuFFT launches are library work)
    // scale
    D0ScaleArgs sa = sa_in;
    sa.n0 = n[0];
    sa.n1 = n[1];
    sa.n2 = n[2];
    sa.h2 = h2;
    sa.cstride = slab;
    const cuDoubleComplex* th = table ? Th.as<cuDoubleComplex>() : nullptr;
    const unsigned sb = (unsigned)((slab + 127) / 128);
    switch (kind) {
        case SEWALD_STOKESLET: d0_scale_kernel<SEWALD_STOKESLET><<<sb, 128, 0, st>>>(spec, sa, xi, to, th); break;
        case SEWALD_ROTLET: d0_scale_kernel<SEWALD_ROTLET><<<sb, 128, 0, st>>>(spec, sa, xi, to, th); break;
        default: d0_scale_kernel<SEWALD_STRESSLET><<<sb, 128, 0, st>>>(spec, sa, xi, to, th); break;
    }
    ++launches;
    // inverse (3 flow components)
    fft_check(cufftExecZ2Z(pxy_i, to, to, CUFFT_INVERSE), "d0 xy inverse");
    const dim3 tgi((h2 + 31) / 32, (m[1] + 31) / 32, 3 * m[0]);
    d0_transpose_kernel<false><<<tgi, tb, 0, st>>>(z, to, m[0], m[1], n[0], n[1], h2);
    ++launches;
    fft_check(cufftExecZ2D(pz_i, z, r), "d0 z inverse");
    d0_extract_kernel<<<blocks_for(lines_out * m[2]), 256, 0, st>>>(r, lines_out, m[2], n[2], flow);
    ++launches;
    cuda_check(cudaGetLastError(), "d0 solve");
    return launches;
}

}  // namespace sewald_b200
