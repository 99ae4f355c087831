// Fourier solve with free directions (d = 0, 1, 2): zero-padded and
// upsampled FFTs with the reference's mode classes, k-space scaling with
// the truncated (modified) kernels, and the D=0 precomputed-kernel path.
//
// Reference: aft_forward   /root/reference/proj/src/fourier.cpp:311-416
//            aft_inverse   /root/reference/proj/src/fourier.cpp:418-520
//            scale         /root/reference/proj/src/fourier.cpp:522-666
//            scale (table) /root/reference/proj/src/fourier.cpp:668-720
//            precompute_0p /root/reference/proj/src/fourier.cpp:722-803
//
// All free-direction transforms are complex-to-complex (cuFFT Z2Z), exactly
// the reference's structure: periodic axes first, the zero / near rows saved
// and re-transformed at their padded lengths, far rows transformed
// unpadded; inverse in the mirror order with the class rows overwritten.
// The three normalisations (h^3 before the forward, 1/n_class after the free
// inverse, 1/(prod M_per h^3) after the periodic inverse) are folded into a
// single per-class factor applied by the scale kernel.
#include "engine.h"
#include "host_params.h"
#include "modified_kernels.cuh"
#include "aft_d0.h"

#include <cufft.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

namespace sewald_b200 {

namespace {

// ---- host restatement of the series tables (modified_kernels.cpp:22-36) ----
struct Tabs {
    double cosc[kSeries], sinc[kSeries], j0[kSeries], xj1[kSeries];
};

Tabs make_tabs() {
    Tabs t{};
    t.cosc[0] = 1.0;
    t.sinc[0] = 1.0;
    t.j0[0] = 1.0;
    t.xj1[0] = 0.0;
    t.xj1[1] = 0.5;
    for (int n = 1; n < kSeries; ++n) {
        t.cosc[n] = -t.cosc[n - 1] / ((2.0 * n - 1.0) * (2.0 * n));
        t.sinc[n] = -t.sinc[n - 1] / ((2.0 * n) * (2.0 * n + 1.0));
        t.j0[n] = -t.j0[n - 1] / (4.0 * n * n);
        if (n >= 2) t.xj1[n] = -t.xj1[n - 1] / (4.0 * n * (n - 1.0));
    }
    return t;
}

}  // namespace

// ModifiedKernelSpec fields (modified_kernels.h:10-19, any gauge) plus the
// series coefficient blocks of the truncated kernels (modified_kernels.cpp:85-94,
// :104-108, :117-124).
ModSpec make_modspec_full(int kind, int d, double R, double a_B, double b_B, double ell_H, double ell_B,
                          double c_B) {
    const Tabs T = make_tabs();
    ModSpec m{};
    m.kind = kind;
    m.d = d;
    m.R = R;
    m.a_B = a_B;
    m.b_B = b_B;
    m.ell_H = ell_H;
    m.ell_B = ell_B;
    m.c_B = c_B;
    m.bR3 = 3.0 * m.b_B * R;
    m.p0 = (m.a_B + R + m.b_B * R * R) / (2.0 * R);
    m.q0 = (m.a_B + 2.0 * R + 3.0 * m.b_B * R * R) / (2.0 * R);
    for (int n = 2; n < kSeries; ++n)
        m.ser_b0[n] = -(1.0 + m.bR3) * T.cosc[n] + m.p0 * T.cosc[n - 1] - m.q0 * T.sinc[n - 1] + m.bR3 * T.sinc[n];
    m.g_h1 = std::log(R / m.ell_H);
    for (int n = 1; n < kSeries; ++n) m.ser_h1[n] = -T.j0[n] - m.g_h1 * T.xj1[n];
    m.g_b1 = std::log(R / m.ell_B);
    m.ch_b1 = (m.c_B - R * R * m.g_b1) / (R * R);
    for (int n = 2; n < kSeries; ++n)
        m.ser_b1[n] = -T.j0[n] - (1.0 + m.g_b1) * T.xj1[n] + 0.25 * (1.0 + 2.0 * m.g_b1) * T.j0[n - 1] -
                      0.25 * m.ch_b1 * T.xj1[n - 1];
    return m;
}

// ModifiedKernelSpec::optimal gauge constants (modified_kernels.cpp:52-63).
ModSpec make_modspec(int kind, int d, double R) {
    return make_modspec_full(kind, d, R, -0.5 * R, -0.5 / R, R, R * std::sqrt(M_E), -0.5 * R * R);
}

namespace {

double mollifier_taper(double t) {  // fourier.cpp:222-225
    const double a2 = 4.0 * std::log(100.0) / 49.0;
    return std::exp(-a2 * t * t) + std::exp(-a2 * (t - 7.0) * (t - 7.0));
}

// ---- device kernels ---------------------------------------------------------

// One class block: data[c][r][j][k], r < R rows, (nf1, nf2) free block.
// kv = (rk0[r], has_k1 ? rk1[r] : kf1[j], kf2[k]);  wp = rw[r] * (has_k1 ? 1 : wf1[j]) * wf2[k]
struct ClassBlock {
    int R, nf1, nf2, has_k1;
    const double* rk0;
    const double* rk1;
    const double* rw;
    const uint8_t* rmask;  // optional: rows with rmask[r] == 0 are skipped
    const double* kf1;
    const double* wf1;
    const double* kf2;
    const double* wf2;
    double norm;
    int64_t cstride;  // complex elements between components
    int zero_masked;  // masked rows: write zeros to the 3 output comps (stage scale)
};

template <int KIND>
__global__ void scale_class_kernel(ModSpec spec, ClassBlock b, double xi, cuDoubleComplex* __restrict__ data,
                                   const cuDoubleComplex* __restrict__ table) {
    constexpr int NC = KIND == SEWALD_STRESSLET ? 9 : 3;
    constexpr int NG = 3 * NC;
    const int64_t n = (int64_t)b.R * b.nf1 * b.nf2;
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= n) return;
    const int k = (int)(idx % b.nf2);
    const int64_t rj = idx / b.nf2;
    const int j = (int)(rj % b.nf1);
    const int r = (int)(rj / b.nf1);
    if (b.rmask && !b.rmask[r]) {
        if (b.zero_masked)
            for (int c = 0; c < 3; ++c) data[c * b.cstride + idx] = make_cuDoubleComplex(0.0, 0.0);
        return;
    }
    const double k0 = b.rk0[r];
    const double k1 = b.has_k1 ? b.rk1[r] : b.kf1[j];
    const double k2 = b.kf2[k];
    const double wp = b.rw[r] * (b.has_k1 ? 1.0 : b.wf1[j]) * b.wf2[k];
    const double kk = k0 * k0 + k1 * k1 + k2 * k2;
    const double q = kk / (4.0 * xi * xi);
    const double g = exp(-q);
    const double scr = KIND == SEWALD_ROTLET ? g : g * (1.0 + q);
    const double fac = scr / (wp * wp) * b.norm;
    double re[NG], im[NG];
    if (table) {
        // Precomputed 0P kernel: G = diffop(k) * table (fourier.cpp:699-701)
        diffop_coeffs<KIND>(k0, k1, k2, re, im);
        const cuDoubleComplex tv = table[idx];
#pragma unroll
        for (int e = 0; e < NG; ++e) {
            const double a = re[e], c = im[e];
            re[e] = a * tv.x - c * tv.y;
            im[e] = a * tv.y + c * tv.x;
        }
    } else {
        modified_coeffs<KIND>(spec, k0, k1, k2, re, im);
    }
    cuDoubleComplex in[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) in[c] = data[c * b.cstride + idx];
#pragma unroll
    for (int jj = 0; jj < 3; ++jj) {
        double ar = 0.0, ai = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            ar += re[NC * jj + c] * in[c].x - im[NC * jj + c] * in[c].y;
            ai += re[NC * jj + c] * in[c].y + im[NC * jj + c] * in[c].x;
        }
        data[jj * b.cstride + idx] = make_cuDoubleComplex(fac * ar, fac * ai);
    }
}

// real (C, n0, n1, n2) -> complex box (C, m0, m1, m2) corner times s, zero elsewhere.
__global__ void real_to_padded_kernel(const double* __restrict__ src, int C, int n0, int n1, int n2, int m0,
                                      int m1, int m2, cuDoubleComplex* __restrict__ dst, double s = 1.0) {
    const int64_t tot = (int64_t)C * m0 * m1 * m2;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(idx % m2);
        int64_t t = idx / m2;
        const int j = (int)(t % m1);
        t /= m1;
        const int i = (int)(t % m0);
        const int c = (int)(t / m0);
        double v = 0.0;
        if (i < n0 && j < n1 && k < n2) v = s * src[(((int64_t)c * n0 + i) * n1 + j) * n2 + k];
        dst[idx] = make_cuDoubleComplex(v, 0.0);
    }
}

// complex box (C, m0, m1, m2) corner -> real (C, n0, n1, n2), real part times s.
__global__ void padded_to_real_kernel(const cuDoubleComplex* __restrict__ src, int m0, int m1, int m2, int n0,
                                      int n1, int n2, int64_t cstride, double* __restrict__ dst, int C = 3,
                                      double s = 1.0) {
    const int64_t tot = (int64_t)C * n0 * n1 * n2;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(idx % n2);
        int64_t t = idx / n2;
        const int j = (int)(t % n1);
        t /= n1;
        const int i = (int)(t % n0);
        const int c = (int)(t / n0);
        dst[idx] = s * src[c * cstride + ((int64_t)i * m1 + j) * m2 + k].x;
    }
}

// Copy rows of free blocks between the far array and a padded class buffer.
// far:  [c][row][b1][b2]   (rows = prod n_per, block b1 x b2)
// cls:  [c][r][p1][p2]     (R rows of padded blocks)
// dir 0: far -> cls corner (zero-fill the rest); dir 1: cls corner -> far row.
__global__ void class_rows_kernel(cuDoubleComplex* __restrict__ far, int nrows, int b1, int b2,
                                  cuDoubleComplex* __restrict__ cls, int R, int p1, int p2,
                                  const int* __restrict__ rows, int C, int dir) {
    const int64_t tot = (int64_t)C * R * p1 * p2;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int q2 = (int)(idx % p2);
        int64_t t = idx / p2;
        const int q1 = (int)(t % p1);
        t /= p1;
        const int r = (int)(t % R);
        const int c = (int)(t / R);
        const bool inside = q1 < b1 && q2 < b2;
        const int64_t fidx = (((int64_t)c * nrows + rows[r]) * b1 + q1) * b2 + q2;
        if (dir == 0) {
            cls[idx] = inside ? far[fidx] : make_cuDoubleComplex(0.0, 0.0);
        } else if (inside) {
            far[fidx] = cls[idx];
        }
    }
}

// precompute_0p: box[i,j,k] = A_trunc(kappa) on the dense grid.
template <bool BIHARMONIC>
__global__ void table_box_kernel(ModSpec m, const double* __restrict__ k0t, const double* __restrict__ k1t,
                                 const double* __restrict__ k2t, int n0, int n1, int n2,
                                 cuDoubleComplex* __restrict__ box) {
    const int64_t tot = (int64_t)n0 * n1 * n2;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(idx % n2);
        const int64_t t = idx / n2;
        const int j = (int)(t % n1);
        const int i = (int)(t / n1);
        const double kappa = sqrt(k0t[i] * k0t[i] + k1t[j] * k1t[j] + k2t[k] * k2t[k]);
        const double v = BIHARMONIC ? biharmonic_trunc_0p(m, kappa) : harmonic_trunc_0p(kappa, m.R);
        box[idx] = make_cuDoubleComplex(v, 0.0);
    }
}

// Truncate the real-space kernel to the doubled box with the edge taper
// (fourier.cpp:769-799): table[dst(i,j,k)] = Re box[src(i,j,k)] * inv * taper.
__global__ void table_fold_kernel(const cuDoubleComplex* __restrict__ box, int d0, int d1, int d2,
                                  const int* __restrict__ src_idx, const int* __restrict__ dst_idx,
                                  const double* __restrict__ taper, int M0, int M1, int M2, double inv,
                                  cuDoubleComplex* __restrict__ table) {
    const int64_t tot = (int64_t)M0 * M1 * M2;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(idx % M2);
        const int64_t t = idx / M2;
        const int j = (int)(t % M1);
        const int i = (int)(t / M1);
        const int* s0 = src_idx;
        const int* s1 = src_idx + M0;
        const int* s2 = src_idx + M0 + M1;
        const int* q0 = dst_idx;
        const int* q1 = dst_idx + M0;
        const int* q2 = dst_idx + M0 + M1;
        const double tij = taper[i] * taper[M0 + j];
        const double a = box[((int64_t)s0[i] * d1 + s1[j]) * d2 + s2[k]].x * inv;
        table[((int64_t)q0[i] * M1 + q1[j]) * M2 + q2[k]] = make_cuDoubleComplex(a * tij * taper[M0 + M1 + k], 0.0);
    }
}

__global__ void scale_complex_kernel(cuDoubleComplex* __restrict__ a, int64_t n, double s) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = make_cuDoubleComplex(a[i].x * s, a[i].y * s);
}

unsigned grid_for(int64_t n) { return (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 64); }

template <class T>
T* upload(DevBuf& b, const std::vector<T>& v, cudaStream_t st) {
    T* p = static_cast<T*>(b.ensure(sizeof(T) * std::max<size_t>(v.size(), 1)));
    if (!v.empty()) cuda_check(cudaMemcpyAsync(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, st), "upload");
    return p;
}

}  // namespace

struct FourierPlanAFT {
    int d = 0, C = 3;
    bool table_path = false;
    int n[3]{};             // M_ext
    int nz[3]{1, 1, 1};     // zero-class free lengths (d=0: padded box)
    int nn[3]{1, 1, 1};     // near-class free lengths
    int nrows = 1, R = 0;   // periodic rows, near rows
    std::vector<cufftHandle> plans;
    cufftHandle p_per = 0, p_far = 0, p_zero = 0, p_near = 0, p_box = 0;
    DevBuf far, zero, near, rows_near, rows_zero, tables, mask, table0p;
    ClassBlock cb_far{}, cb_zero{}, cb_near{};
    ModSpec spec{};
    std::unique_ptr<D0Real> d0r;  // d = 0: real pruned transforms (aft_d0.cu)
    D0ScaleArgs d0sa{};
    ~FourierPlanAFT() {
        for (auto p : plans) cufftDestroy(p);
    }
    cufftHandle make(int rank, int* nn_, int* emb, int stride, int dist, int batch, cudaStream_t st) {
        cufftHandle h = 0;
        cufft_check(cufftPlanMany(&h, rank, nn_, emb, stride, dist, emb, stride, dist, CUFFT_Z2Z, batch), "plan Z2Z");
        cufft_check(cufftSetStream(h, st), "plan stream");
        plans.push_back(h);
        return h;
    }
};

void AftDeleter::operator()(FourierPlanAFT* p) const { delete p; }

// D=0 kernel table on the (2 M_ext)^3 mode grid (fourier.cpp:722-803) with
// cuFFT, into `out` ((2 M_ext)^3 complex, row-major). Returns kernel launches.
int build_table_0p(const sewald_params_c& p, int kind, double R, DevBuf& out, cudaStream_t st) {
    if (!(R > 0.0)) throw EngineError(SEWALD_EINVAL, "truncation radius must be positive");
    long g = 0;
    double Lmin = p.L_ext[0];
    for (int ax = 0; ax < 3; ++ax) {
        if (p.M_ext[ax] % p.f_m != 0)
            throw EngineError(SEWALD_EINVAL, "extended grid sizes must be multiples of f_m");
        g = std::gcd(g, static_cast<long>(p.M_ext[ax] / p.f_m));
        Lmin = std::min(Lmin, p.L_ext[ax]);
    }
    double s0 = std::ceil(10.0 * (1.0 + R / Lmin) - 1e-9) / 10.0;
    s0 = std::max(std::ceil(s0 * static_cast<double>(g) - 1e-9) / static_cast<double>(g), 1.0);
    int dense[3];
    for (int ax = 0; ax < 3; ++ax) dense[ax] = padded_length(s0, p.M_ext[ax]);
    const int64_t dvol = (int64_t)dense[0] * dense[1] * dense[2];
    const bool biharmonic = kind != SEWALD_ROTLET;
    const ModSpec m = make_modspec(kind, 0, R);

    std::vector<double> kt;
    for (int ax = 0; ax < 3; ++ax) {
        const std::vector<double> k = wavenumbers(dense[ax], p.h);
        kt.insert(kt.end(), k.begin(), k.end());
    }
    DevBuf dk, box, idxs, tap;
    double* dkt = upload(dk, kt, st);
    cuDoubleComplex* dbox = static_cast<cuDoubleComplex*>(box.ensure(sizeof(cuDoubleComplex) * dvol));
    if (biharmonic)
        table_box_kernel<true><<<grid_for(dvol), 256, 0, st>>>(m, dkt, dkt + dense[0], dkt + dense[0] + dense[1],
                                                               dense[0], dense[1], dense[2], dbox);
    else
        table_box_kernel<false><<<grid_for(dvol), 256, 0, st>>>(m, dkt, dkt + dense[0], dkt + dense[0] + dense[1],
                                                                dense[0], dense[1], dense[2], dbox);
    cufftHandle pd = 0;
    cufft_check(cufftPlan3d(&pd, dense[0], dense[1], dense[2], CUFFT_Z2Z), "plan dense");
    cufft_check(cufftSetStream(pd, st), "plan stream");
    cufft_check(cufftExecZ2Z(pd, dbox, dbox, CUFFT_INVERSE), "dense inverse");
    const double h3 = p.h * p.h * p.h;
    const double inv = 1.0 / (h3 * static_cast<double>(dvol));

    int M2[3];
    std::vector<int> src_idx, dst_idx;
    std::vector<double> taper;
    for (int ax = 0; ax < 3; ++ax) {
        M2[ax] = 2 * p.M_ext[ax];
        const int Me = p.M_ext[ax];
        std::vector<double> tp(M2[ax], 1.0);
        if (biharmonic)
            for (int t = 0; t < 4; ++t) {
                tp[t] = mollifier_taper(3.0 - t);
                tp[M2[ax] - 1 - t] = mollifier_taper(3.0 - t);
            }
        taper.insert(taper.end(), tp.begin(), tp.end());
        for (int t = 0; t < M2[ax]; ++t) {
            const int x = t - Me;
            src_idx.push_back((x % dense[ax] + dense[ax]) % dense[ax]);
            dst_idx.push_back((x + M2[ax]) % M2[ax]);
        }
    }
    DevBuf ds, dd;
    int* dsrc = upload(ds, src_idx, st);
    int* ddst = upload(dd, dst_idx, st);
    double* dtap = upload(tap, taper, st);
    const int64_t tvol = (int64_t)M2[0] * M2[1] * M2[2];
    cuDoubleComplex* table = static_cast<cuDoubleComplex*>(out.ensure(sizeof(cuDoubleComplex) * tvol));
    table_fold_kernel<<<grid_for(tvol), 256, 0, st>>>(dbox, dense[0], dense[1], dense[2], dsrc, ddst, dtap, M2[0],
                                                      M2[1], M2[2], inv, table);
    cufftHandle pt = 0;
    cufft_check(cufftPlan3d(&pt, M2[0], M2[1], M2[2], CUFFT_Z2Z), "plan table");
    cufft_check(cufftSetStream(pt, st), "plan stream");
    cufft_check(cufftExecZ2Z(pt, table, table, CUFFT_FORWARD), "table forward");
    scale_complex_kernel<<<grid_for(tvol), 256, 0, st>>>(table, tvol, h3);
    cuda_check(cudaStreamSynchronize(st), "table sync");
    cufftDestroy(pd);
    cufftDestroy(pt);
    return 4;
}

namespace {

void build_table_0p(sewald_gpu_session* s, FourierPlanAFT& A) {
    if (s->has_user_table) {  // SePipelineOptions::table: the caller's table is used as is
        const size_t bytes = sizeof(cuDoubleComplex) * 8 * (size_t)s->p.M_ext[0] * s->p.M_ext[1] * s->p.M_ext[2];
        A.table0p.ensure(bytes);
        cuda_check(cudaMemcpyAsync(A.table0p.ptr, s->user_table0p.ptr, bytes, cudaMemcpyDeviceToDevice,
                                   s->ctx->stream),
                   "user table");
        return;
    }
    s->ctx->launches += build_table_0p(s->p, s->p.kind, s->p.R, A.table0p, s->ctx->stream);
}

// classify_rows (fourier.cpp:101-125): flat periodic-mode rows inside K_star
// (excluding the zero row), in row order.
std::vector<int> near_rows_of(const sewald_params_c& p) {
    int nper[2] = {1, 1};
    for (int ax = 0; ax < p.d && ax < 2; ++ax) nper[ax] = p.M[ax];
    std::vector<int> near_rows;
    for (int i = 0; i < nper[0]; ++i)
        for (int j = 0; j < nper[1]; ++j) {
            const int m[2] = {i, j};
            bool zero = true, near = true;
            for (int ax = 0; ax < p.d; ++ax) {
                const int sm = signed_mode(m[ax], nper[ax]);
                if (sm != 0) zero = false;
                if (std::abs(sm) > p.k_star[ax]) near = false;
            }
            if (!zero && near) near_rows.push_back(i * nper[1] + j);
        }
    return near_rows;
}

// d = 1, 2: class buffers, cuFFT plans and k / window tables for the rows of
// A.nrows periodic modes; A.nz / A.nn (padded free lengths) are set by the
// caller. stage = true (reference stage functions): unit normalisation in
// scale and zero output on far rows of other classes (fourier.cpp:601-615);
// otherwise all normalisations are folded into the per-class scale.
void setup_classes(const sewald_params_c& p, FourierPlanAFT& A, const std::vector<int>& near_rows, bool stage,
                   cudaStream_t st) {
    const int d = A.d;
    const double h = p.h;
    int nper[3] = {1, 1, 1};
    for (int ax = 0; ax < d; ++ax) nper[ax] = p.M[ax];
    A.nrows = nper[0] * nper[1];
    std::vector<uint8_t> cls(A.nrows, 0);
    cls[0] = 2;
    for (int r : near_rows) {
        if (r <= 0 || r >= A.nrows) throw EngineError(SEWALD_EINVAL, "near row index out of range");
        cls[r] = 1;
    }
    A.R = static_cast<int>(near_rows.size());
    const int b1 = d == 1 ? p.M_ext[1] : 1, b2 = p.M_ext[2];          // free block (unpadded)
    const int z1 = d == 1 ? A.nz[1] : 1, z2 = A.nz[2];                   // zero block
    const int q1 = d == 1 ? A.nn[1] : 1, q2 = A.nn[2];                   // near block
    const int64_t vol = (int64_t)A.nrows * b1 * b2;
    A.far.ensure(sizeof(cuDoubleComplex) * vol * A.C);
    A.zero.ensure(sizeof(cuDoubleComplex) * (int64_t)z1 * z2 * A.C);
    A.near.ensure(sizeof(cuDoubleComplex) * std::max<int64_t>((int64_t)A.R * q1 * q2 * A.C, 1));
    std::vector<int> zr = {0};
    upload(A.rows_zero, zr, st);
    upload(A.rows_near, near_rows, st);
    std::vector<uint8_t> fmask(A.nrows);
    for (int r = 0; r < A.nrows; ++r) fmask[r] = cls[r] == 0;
    upload(A.mask, fmask, st);

    // plans
    if (d == 2) {
        int n2d[2] = {p.M[0], p.M[1]};
        A.p_per = A.make(2, n2d, n2d, b2, 1, b2, st);           // per component: stride Mz, batch Mz
        int nf[1] = {b2};
        A.p_far = A.make(1, nf, nf, 1, b2, A.C * A.nrows, st);
        int nzl[1] = {z2};
        A.p_zero = A.make(1, nzl, nzl, 1, z2, A.C, st);
        if (A.R > 0) {
            int nnl[1] = {q2};
            A.p_near = A.make(1, nnl, nnl, 1, q2, A.C * A.R, st);
        }
    } else {
        int n1d[1] = {p.M[0]};
        A.p_per = A.make(1, n1d, n1d, b1 * b2, 1, b1 * b2, st);  // per component
        int nf[2] = {b1, b2};
        A.p_far = A.make(2, nf, nf, 1, b1 * b2, A.C * A.nrows, st);
        int nzl[2] = {z1, z2};
        A.p_zero = A.make(2, nzl, nzl, 1, z1 * z2, A.C, st);
        if (A.R > 0) {
            int nnl[2] = {q1, q2};
            A.p_near = A.make(2, nnl, nnl, 1, q1 * q2, A.C * A.R, st);
        }
    }

    // tables (fourier.cpp:543-548, :595-599, :617-622, :640-645)
    std::vector<double> kper[2], wper[2];
    for (int ax = 0; ax < d; ++ax) {
        kper[ax] = wavenumbers(p.M[ax], h);
        wper[ax] = window_hat_table(p, kper[ax]);
    }
    auto kw = [&](int len) {
        std::vector<double> k = wavenumbers(len, h);
        return std::make_pair(k, window_hat_table(p, k));
    };
    // far rows: k0 = kper0[i], k1 = kper1[j] (d=2); weights wper0[i] * wper1[j]
    std::vector<double> fk0(A.nrows), fk1(A.nrows, 0.0), fw(A.nrows);
    for (int i = 0; i < nper[0]; ++i)
        for (int j = 0; j < nper[1]; ++j) {
            const int r = i * nper[1] + j;
            fk0[r] = kper[0][i];
            if (d == 2) fk1[r] = kper[1][j];
            fw[r] = d == 2 ? wper[0][i] * wper[1][j] : wper[0][i];
        }
    // zero row: k = 0 on periodic axes, weight prod wper[ax][0]
    double wper0 = 1.0;
    for (int ax = 0; ax < d; ++ax) wper0 *= wper[ax][0];
    std::vector<double> zk0 = {0.0}, zk1 = {0.0}, zw = {wper0};
    // near rows
    std::vector<double> nk0(std::max(A.R, 1)), nk1(std::max(A.R, 1), 0.0), nw(std::max(A.R, 1));
    for (int r = 0; r < A.R; ++r) {
        const int row = near_rows[r];
        const int m0 = d == 1 ? row : row / nper[1];
        const int m1 = d == 1 ? 0 : row % nper[1];
        nk0[r] = kper[0][m0];
        if (d == 2) nk1[r] = kper[1][m1];
        nw[r] = wper[0][m0] * (d == 2 ? wper[1][m1] : 1.0);
    }
    auto far1 = kw(p.M_ext[1]), far2 = kw(p.M_ext[2]);
    auto zer1 = kw(A.nz[1]), zer2 = kw(A.nz[2]);
    auto nea1 = kw(A.nn[1]), nea2 = kw(A.nn[2]);
    std::vector<const std::vector<double>*> parts = {&fk0, &fk1, &fw, &zk0, &zk1, &zw, &nk0, &nk1, &nw,
                                                     &far1.first, &far1.second, &far2.first, &far2.second,
                                                     &zer1.first, &zer1.second, &zer2.first, &zer2.second,
                                                     &nea1.first, &nea1.second, &nea2.first, &nea2.second};
    std::vector<double> tab;
    std::vector<size_t> off;
    for (auto* v : parts) {
        off.push_back(tab.size());
        tab.insert(tab.end(), v->begin(), v->end());
    }
    double* t = upload(A.tables, tab, st);
    auto P = [&](int i) { return static_cast<const double*>(t + off[i]); };
    // Per-class normalisation: h^3 (forward) * 1/n_class_free * 1/(prod M_per h^3).
    double inv_per = 1.0;
    for (int ax = 0; ax < d; ++ax) inv_per /= p.M[ax];
    double nf_far = 1.0, nf_zero = 1.0, nf_near = 1.0;
    for (int ax = d; ax < 3; ++ax) {
        nf_far /= p.M_ext[ax];
        nf_zero /= A.nz[ax];
        nf_near /= A.nn[ax];
    }
    const int has_k1 = d == 2 ? 1 : 0;
    if (stage) nf_far = nf_zero = nf_near = inv_per = 1.0;
    A.cb_far = ClassBlock{A.nrows, b1, b2, has_k1, P(0), P(1), P(2), A.mask.as<uint8_t>(), P(9), P(10), P(11),
                          P(12), nf_far * inv_per, vol, stage ? 1 : 0};
    A.cb_zero = ClassBlock{1, z1, z2, has_k1, P(3), P(4), P(5), nullptr, P(13), P(14), P(15), P(16),
                           nf_zero * inv_per, (int64_t)z1 * z2, 0};
    A.cb_near = ClassBlock{A.R, q1, q2, has_k1, P(6), P(7), P(8), nullptr, P(17), P(18), P(19), P(20),
                           nf_near * inv_per, (int64_t)A.R * q1 * q2, 0};
}

void prepare(sewald_gpu_session* s, bool use_table) {
    const sewald_params_c& p = s->p;
    if (s->aft && s->aft->table_path == (use_table && p.d == 0)) return;
    s->aft.reset(new FourierPlanAFT());
    FourierPlanAFT& A = *s->aft;
    cudaStream_t st = s->ctx->stream;
    A.d = p.d;
    A.C = s->C;
    A.table_path = use_table && p.d == 0;
    for (int ax = 0; ax < 3; ++ax) A.n[ax] = p.M_ext[ax];
    A.spec = make_modspec(p.kind, p.d, p.R);
    const int d = p.d;
    const double h = p.h;

    if (d == 0) {
        const double s0 = A.table_path ? 2.0 : p.s0;
        for (int ax = 0; ax < 3; ++ax) A.nz[ax] = padded_length(s0, p.M_ext[ax]);
        const int64_t zvol = (int64_t)A.nz[0] * A.nz[1] * A.nz[2];
        // SEWALD_D0_C2C=1: the reference's full complex box transform (A/B checks)
        static const bool c2c = [] {
            const char* e = getenv("SEWALD_D0_C2C");
            return e && e[0] == '1';
        }();
        if (c2c) {
            A.zero.ensure(sizeof(cuDoubleComplex) * zvol * A.C);
            int nn3[3] = {A.nz[0], A.nz[1], A.nz[2]};
            A.p_box = A.make(3, nn3, nn3, 1, (int)zvol, A.C, st);
        } else {
            A.d0r.reset(new D0Real());
            A.d0r->setup(A.n, A.nz, A.C, st);
        }
        // rows = axis 0 of the padded box (free), free block = axes 1, 2
        std::vector<double> k0 = wavenumbers(A.nz[0], h), k1 = wavenumbers(A.nz[1], h), k2 = wavenumbers(A.nz[2], h);
        std::vector<double> w0 = window_hat_table(p, k0), w1 = window_hat_table(p, k1), w2 = window_hat_table(p, k2);
        std::vector<double> tab;
        for (auto* v : {&k0, &w0, &k1, &w1, &k2, &w2}) tab.insert(tab.end(), v->begin(), v->end());
        double* t = upload(A.tables, tab, st);
        size_t o = 0;
        const double* dk0 = t + o; o += k0.size();
        const double* dw0 = t + o; o += w0.size();
        const double* dk1 = t + o; o += k1.size();
        const double* dw1 = t + o; o += w1.size();
        const double* dk2 = t + o; o += k2.size();
        const double* dw2 = t + o;
        A.cb_zero = ClassBlock{A.nz[0], A.nz[1], A.nz[2], 0, dk0, nullptr, dw0, nullptr, dk1, dw1, dk2, dw2,
                               1.0 / static_cast<double>(zvol), zvol};
        A.d0sa = D0ScaleArgs{0, 0, 0, 0, 0, dk0, dk1, dk2, dw0, dw1, dw2, 1.0 / static_cast<double>(zvol)};
        if (A.table_path) build_table_0p(s, A);
        if (A.table_path && A.d0r) A.d0r->build_herm_table(A.table0p.as<cuDoubleComplex>(), st);
        cuda_check(cudaStreamSynchronize(st), "aft prepare");
        return;
    }

    // d = 1, 2: periodic rows and the free block
    for (int ax = p.d; ax < 3; ++ax) {
        A.nz[ax] = padded_length(p.s0, p.M_ext[ax]);
        A.nn[ax] = padded_length(p.s_star, p.M_ext[ax]);
    }
    setup_classes(p, A, near_rows_of(p), false, st);
    cuda_check(cudaStreamSynchronize(st), "aft prepare");
}

void launch_scale_class(int kind, const ModSpec& m, const ClassBlock& b, double xi, cuDoubleComplex* data,
                        const cuDoubleComplex* table, cudaStream_t st) {
    const int64_t n = (int64_t)b.R * b.nf1 * b.nf2;
    if (n == 0) return;
    const unsigned blocks = (unsigned)((n + 127) / 128);
    switch (kind) {
        case SEWALD_STOKESLET: scale_class_kernel<SEWALD_STOKESLET><<<blocks, 128, 0, st>>>(m, b, xi, data, table); break;
        case SEWALD_ROTLET: scale_class_kernel<SEWALD_ROTLET><<<blocks, 128, 0, st>>>(m, b, xi, data, table); break;
        default: scale_class_kernel<SEWALD_STRESSLET><<<blocks, 128, 0, st>>>(m, b, xi, data, table); break;
    }
}

}  // namespace

void aft_solve(sewald_gpu_session* s, const double* grid, bool precompute_0p) {
    prepare(s, precompute_0p);
    FourierPlanAFT& A = *s->aft;
    const sewald_params_c& p = s->p;
    cudaStream_t st = s->ctx->stream;
    const int C = A.C;
    double* flow = s->flow.as<double>();

    if (p.d == 0 && A.d0r) {
        s->ctx->launches += A.d0r->solve(grid, A.spec, p.kind, p.xi, A.d0sa, A.table_path, flow, st);
        return;
    }
    if (p.d == 0) {
        const int64_t zvol = (int64_t)A.nz[0] * A.nz[1] * A.nz[2];
        cuDoubleComplex* z = A.zero.as<cuDoubleComplex>();
        real_to_padded_kernel<<<grid_for(C * zvol), 256, 0, st>>>(grid, C, A.n[0], A.n[1], A.n[2], A.nz[0], A.nz[1],
                                                                  A.nz[2], z);
        cufftSetStream(A.p_box, st);
        cufft_check(cufftExecZ2Z(A.p_box, z, z, CUFFT_FORWARD), "d0 forward");
        launch_scale_class(p.kind, A.spec, A.cb_zero, p.xi, z,
                           A.table_path ? A.table0p.as<cuDoubleComplex>() : nullptr, st);
        cufftSetStream(A.p_box, st);
        cufft_check(cufftExecZ2Z(A.p_box, z, z, CUFFT_INVERSE), "d0 inverse");
        padded_to_real_kernel<<<grid_for(3 * (int64_t)A.n[0] * A.n[1] * A.n[2]), 256, 0, st>>>(
            z, A.nz[0], A.nz[1], A.nz[2], A.n[0], A.n[1], A.n[2], zvol, flow);
        s->ctx->launches += 3;
        cuda_check(cudaGetLastError(), "aft d0");
        return;
    }

    const int d = p.d;
    const int b1 = d == 1 ? p.M_ext[1] : 1, b2 = p.M_ext[2];
    const int64_t vol = (int64_t)A.nrows * b1 * b2;
    const int z1 = d == 1 ? A.nz[1] : 1, z2 = A.nz[2];
    const int q1 = d == 1 ? A.nn[1] : 1, q2 = A.nn[2];
    cuDoubleComplex* far = A.far.as<cuDoubleComplex>();
    cuDoubleComplex* zero = A.zero.as<cuDoubleComplex>();
    cuDoubleComplex* near = A.near.as<cuDoubleComplex>();

    // forward: h^3 phi (normalisation folded into scale), periodic FFTs
    real_to_padded_kernel<<<grid_for(C * vol), 256, 0, st>>>(grid, C, A.n[0], A.n[1], A.n[2], A.n[0], A.n[1],
                                                             A.n[2], far);
    cufftSetStream(A.p_per, st);
    for (int c = 0; c < C; ++c)
        cufft_check(cufftExecZ2Z(A.p_per, far + c * vol, far + c * vol, CUFFT_FORWARD), "per forward");
    // save the zero / near rows' free blocks, zero padded
    class_rows_kernel<<<grid_for((int64_t)C * z1 * z2), 256, 0, st>>>(far, A.nrows, b1, b2, zero, 1, z1, z2,
                                                                       A.rows_zero.as<int>(), C, 0);
    if (A.R > 0)
        class_rows_kernel<<<grid_for((int64_t)C * A.R * q1 * q2), 256, 0, st>>>(far, A.nrows, b1, b2, near, A.R, q1,
                                                                                q2, A.rows_near.as<int>(), C, 0);
    // free transforms: all rows unpadded, zero and near rows padded
    cufftSetStream(A.p_far, st);
    cufft_check(cufftExecZ2Z(A.p_far, far, far, CUFFT_FORWARD), "far forward");
    cufftSetStream(A.p_zero, st);
    cufft_check(cufftExecZ2Z(A.p_zero, zero, zero, CUFFT_FORWARD), "zero forward");
    if (A.R > 0) cufftSetStream(A.p_near, st);
    if (A.R > 0) cufft_check(cufftExecZ2Z(A.p_near, near, near, CUFFT_FORWARD), "near forward");
    // scale each class (far rows of other classes are left unscaled and
    // overwritten on inversion, as in the reference)
    launch_scale_class(p.kind, A.spec, A.cb_far, p.xi, far, nullptr, st);
    launch_scale_class(p.kind, A.spec, A.cb_zero, p.xi, zero, nullptr, st);
    if (A.R > 0) launch_scale_class(p.kind, A.spec, A.cb_near, p.xi, near, nullptr, st);
    // inverse: free directions, class rows overwrite, periodic, real part
    cufftSetStream(A.p_far, st);
    cufft_check(cufftExecZ2Z(A.p_far, far, far, CUFFT_INVERSE), "far inverse");
    cufftSetStream(A.p_zero, st);
    cufft_check(cufftExecZ2Z(A.p_zero, zero, zero, CUFFT_INVERSE), "zero inverse");
    if (A.R > 0) cufftSetStream(A.p_near, st);
    if (A.R > 0) cufft_check(cufftExecZ2Z(A.p_near, near, near, CUFFT_INVERSE), "near inverse");
    class_rows_kernel<<<grid_for((int64_t)3 * z1 * z2), 256, 0, st>>>(far, A.nrows, b1, b2, zero, 1, z1, z2,
                                                                       A.rows_zero.as<int>(), 3, 1);
    if (A.R > 0)
        class_rows_kernel<<<grid_for((int64_t)3 * A.R * q1 * q2), 256, 0, st>>>(far, A.nrows, b1, b2, near, A.R, q1,
                                                                                q2, A.rows_near.as<int>(), 3, 1);
    cufftSetStream(A.p_per, st);
    for (int c = 0; c < 3; ++c)
        cufft_check(cufftExecZ2Z(A.p_per, far + c * vol, far + c * vol, CUFFT_INVERSE), "per inverse");
    padded_to_real_kernel<<<grid_for(3 * vol), 256, 0, st>>>(far, A.n[0], A.n[1], A.n[2], A.n[0], A.n[1], A.n[2], vol,
                                                             flow);
    s->ctx->launches += 10;
    cuda_check(cudaGetLastError(), "aft d12");
}

void session_set_table0p(sewald_gpu_session* s, const int32_t n[3], const double* table) {
    if (!table) {
        if (s->has_user_table) s->aft.reset();
        s->has_user_table = false;
        s->user_table_src = nullptr;
        return;
    }
    if (s->p.d != 0) throw EngineError(SEWALD_EINVAL, "precomputed kernels apply to d = 0 only");
    // Re-upload unless it is the same table: same address and size AND the
    // same values at 4096 sampled entries (a new table allocated at a freed
    // one's address differs there; the table can be GBs, so the full content
    // is not compared on every call).
    const int64_t cnt = (int64_t)n[0] * n[1] * n[2];
    uint64_t fp = 1469598103934665603ull ^ (uint64_t)cnt;
    cudaPointerAttributes attr{};
    const bool host_mem = cudaPointerGetAttributes(&attr, table) != cudaSuccess || attr.type == cudaMemoryTypeHost ||
                          attr.type == cudaMemoryTypeUnregistered;
    cudaGetLastError();
    if (!host_mem) fp = ~s->user_table_fp;  // device memory: always copied (device to device)
    for (int k = 0; k < 4096 && cnt > 0 && host_mem; ++k) {
        const int64_t i = (int64_t)((__int128)cnt * k / 4096);
        uint64_t w[2];
        std::memcpy(w, table + 2 * i, sizeof(w));
        fp = (fp ^ w[0]) * 1099511628211ull;
        fp = (fp ^ w[1]) * 1099511628211ull;
    }
    if (s->has_user_table && s->user_table_src == table && s->user_table_fp == fp) return;
    // the table path pads with s0 = 2 (fourier.cpp:819-821), so the table must
    // live on the (2 M_ext)^3 mode grid (fourier.cpp:672-673)
    for (int ax = 0; ax < 3; ++ax)
        if (n[ax] != 2 * s->p.M_ext[ax])
            throw EngineError(SEWALD_EINVAL, "kernel table was built for a different padded grid");
    const size_t bytes = sizeof(cuDoubleComplex) * (size_t)n[0] * n[1] * n[2];
    s->user_table0p.ensure(bytes);
    cuda_check(cudaMemcpyAsync(s->user_table0p.ptr, table, bytes, cudaMemcpyDefault, s->ctx->stream), "table in");
    cuda_check(cudaStreamSynchronize(s->ctx->stream), "table in");
    s->has_user_table = true;
    s->user_table_src = table;
    s->user_table_fp = fp;
    s->aft.reset();  // the next table-path solve rebuilds its plan with this table
}

// ---- slab-distributed solve: stage wrappers -------------------------
// D = 0: the padded-box real transforms of D0Real. D = 3: the same machinery on
// the unpadded periodic box (n = M, wavenumbers 2 pi m / L, Nyquist at -pi/h)
// with the plain periodic operator (modified_coeffs at d = 3: G(0) = 0,
// modified_kernels.cpp:250-252) and its Hermitian Nyquist part, i.e. the
// same per-mode operator as the single-GPU D = 3 solve (kspace.cu).

struct D3Slab {
    D0Real d;
    D0ScaleArgs sa{};
    DevBuf tables;
    ModSpec spec{};
};

void D3SlabDeleter::operator()(D3Slab* p) const { delete p; }

static D3Slab& d3_slab(sewald_gpu_session* s) {
    if (s->slab3) return *s->slab3;
    const sewald_params_c& p = s->p;
    cudaStream_t st = s->ctx->stream;
    std::unique_ptr<D3Slab, D3SlabDeleter> D(new D3Slab());
    int m[3];
    for (int ax = 0; ax < 3; ++ax) m[ax] = p.M_ext[ax];
    D->d.setup(m, m, s->C, st);
    D->spec = make_modspec(p.kind, 3, p.R);
    std::vector<double> k0 = wavenumbers(m[0], p.h), k1 = wavenumbers(m[1], p.h), k2 = wavenumbers(m[2], p.h);
    std::vector<double> w0 = window_hat_table(p, k0), w1 = window_hat_table(p, k1), w2 = window_hat_table(p, k2);
    std::vector<double> tab;
    for (auto* v : {&k0, &w0, &k1, &w1, &k2, &w2}) tab.insert(tab.end(), v->begin(), v->end());
    double* t = upload(D->tables, tab, st);
    size_t o = 0;
    const double* dk0 = t + o; o += k0.size();
    const double* dw0 = t + o; o += w0.size();
    const double* dk1 = t + o; o += k1.size();
    const double* dw1 = t + o; o += w1.size();
    const double* dk2 = t + o; o += k2.size();
    const double* dw2 = t + o;
    const int64_t vol = (int64_t)m[0] * m[1] * m[2];
    D->sa = D0ScaleArgs{0, 0, 0, 0, 0, dk0, dk1, dk2, dw0, dw1, dw2, 1.0 / static_cast<double>(vol)};
    cuda_check(cudaStreamSynchronize(st), "d3 slab prepare");
    s->slab3 = std::move(D);
    return *s->slab3;
}

static D0Real& d0_plan(sewald_gpu_session* s, bool use_table) {
    if (s->p.d == 3) return d3_slab(s).d;
    if (s->p.d != 0) throw EngineError(SEWALD_EINVAL, "the slab-distributed solve covers D = 0 and D = 3");
    prepare(s, use_table);
    FourierPlanAFT& A = *s->aft;
    if (!A.d0r) throw EngineError(SEWALD_EINVAL, "slab-distributed solve needs the real-transform D=0 path");
    return *A.d0r;
}

void aft_d0_geometry(sewald_gpu_session* s, bool use_table, int m[3], int n[3], int* h2, int* C) {
    D0Real& D = d0_plan(s, use_table);
    for (int a = 0; a < 3; ++a) {
        m[a] = D.m[a];
        n[a] = D.n[a];
    }
    *h2 = D.h2;
    *C = D.C;
}

void aft_d0_slab_forward(sewald_gpu_session* s, bool use_table, const double* grid_slab, int xa, int xb,
                         const SlabBounds& kzb, void* send) {
    D0Real& D = d0_plan(s, use_table);
    s->ctx->launches += D.slab_forward(grid_slab, xa, xb, kzb, static_cast<cuDoubleComplex*>(send), s->ctx->stream);
}

void aft_d0_slab_middle(sewald_gpu_session* s, bool use_table, const void* recv, const SlabBounds& xbd, int ka,
                        int kb, void* send) {
    D0Real& D = d0_plan(s, use_table);
    if (s->p.d == 3) {
        D3Slab& P = d3_slab(s);
        s->ctx->launches += D.slab_middle(static_cast<const cuDoubleComplex*>(recv), xbd, ka, kb, P.spec, s->p.kind,
                                          s->p.xi, P.sa, false, static_cast<cuDoubleComplex*>(send), s->ctx->stream);
        return;
    }
    FourierPlanAFT& A = *s->aft;
    s->ctx->launches += D.slab_middle(static_cast<const cuDoubleComplex*>(recv), xbd, ka, kb, A.spec, s->p.kind,
                                      s->p.xi, A.d0sa, A.table_path, static_cast<cuDoubleComplex*>(send),
                                      s->ctx->stream);
}

void aft_d0_slab_inverse(sewald_gpu_session* s, bool use_table, const void* recv, int xa, int xb,
                         const SlabBounds& kzb, double* flow_slab) {
    D0Real& D = d0_plan(s, use_table);
    s->ctx->launches += D.slab_inverse(static_cast<const cuDoubleComplex*>(recv), xa, xb, kzb, flow_slab,
                                       s->ctx->stream);
}

// ---- reference stage functions on host buffers -------------------
// aft_forward / scale / scale(table) / aft_inverse / precompute_0p with the
// reference's FourierField layout (fourier.h:30-46): complex arrays as
// interleaved (re, im) doubles, far [c][rows][free], zero [c][zero block],
// near [c][r][near block]. Same transforms and kernels as the fused solve,
// with the reference's per-stage normalisations instead of folded ones.

namespace {

int strength_comps(int kind) { return kind == SEWALD_STRESSLET ? 9 : 3; }

void check_window_h(const sewald_params_c& p) {  // fourier.cpp:155-158
    if (std::fabs(p.win_h - p.h) > 1e-12 * p.h)
        throw EngineError(SEWALD_EINVAL, "window was built for a different grid spacing");
}

int64_t cells3(const int32_t* n) { return (int64_t)n[0] * n[1] * n[2]; }

void fill_lengths(sewald_fourier_geom_c& g, const int32_t* M_ext) {
    const int C = g.comps, d = g.d;
    g.far_len = g.near_len = g.zero_len = 0;
    if (d == 3) {
        g.far_len = C * cells3(M_ext);
    } else if (d == 0) {
        g.zero_len = C * cells3(g.n_zero);
    } else {
        g.far_len = C * cells3(M_ext);
        g.zero_len = (int64_t)C * (d == 1 ? g.n_zero[1] * g.n_zero[2] : g.n_zero[2]);
        g.near_len = (int64_t)C * g.n_near_rows * (d == 1 ? g.n_near[1] * g.n_near[2] : g.n_near[2]);
    }
}

// FourierField geometry consistent with the grid (shapes only; the reference
// checks periodicity in aft_inverse / scale, fourier.cpp:421-422, :524-525).
void check_geometry(const sewald_params_c& p, const sewald_fourier_geom_c& g) {
    if (g.d != p.d) throw EngineError(SEWALD_EINVAL, "field and grid periodicity differ");
    if (g.comps < 1) throw EngineError(SEWALD_EINVAL, "field storage is inconsistent");
    // d = 3 reads only the grid, d = 0 only n_zero (a table-scaled field keeps
    // the default n_per / n_far, fourier.cpp:688-692); d = 1, 2 read them all.
    for (int ax = 0; ax < 3; ++ax) {
        const bool per = ax < p.d;
        const bool classes = p.d == 1 || p.d == 2;
        if ((classes && (g.n_per[ax] != (per ? p.M[ax] : 1) || g.n_far[ax] != (per ? 1 : p.M_ext[ax]))) ||
            g.n_near[ax] < 1 || g.n_zero[ax] < 1)
            throw EngineError(SEWALD_EINVAL, "field shape does not match the extended grid");
    }
    if (g.n_near_rows < 0) throw EngineError(SEWALD_EINVAL, "field storage is inconsistent");
    sewald_fourier_geom_c t = g;
    fill_lengths(t, p.M_ext);
    if (t.far_len != g.far_len || t.near_len != g.near_len || t.zero_len != g.zero_len)
        throw EngineError(SEWALD_EINVAL, "field storage is inconsistent");
}

// Transforms / tables for the field geometry g (box path for d = 3 and 0,
// class path for d = 1, 2 with the field's own near rows).
void stage_plan(const sewald_params_c& p, const sewald_fourier_geom_c& g, const int32_t* near_rows,
                bool tables, FourierPlanAFT& A, cudaStream_t st) {
    A.d = g.d;
    A.C = g.comps;
    for (int ax = 0; ax < 3; ++ax) A.n[ax] = p.M_ext[ax];
    if (g.d == 3 || g.d == 0) {
        for (int ax = 0; ax < 3; ++ax) A.nz[ax] = g.d == 3 ? p.M_ext[ax] : g.n_zero[ax];
        const int64_t bvol = cells3(A.nz);
        A.zero.ensure(sizeof(cuDoubleComplex) * bvol * A.C);
        int nn3[3] = {A.nz[0], A.nz[1], A.nz[2]};
        A.p_box = A.make(3, nn3, nn3, 1, (int)bvol, A.C, st);
        if (tables) {
            std::vector<double> tab, k[3], w[3];
            for (int ax = 0; ax < 3; ++ax) {
                k[ax] = wavenumbers(A.nz[ax], p.h);
                w[ax] = window_hat_table(p, k[ax]);
            }
            for (int ax = 0; ax < 3; ++ax) {
                tab.insert(tab.end(), k[ax].begin(), k[ax].end());
                tab.insert(tab.end(), w[ax].begin(), w[ax].end());
            }
            const double* t = upload(A.tables, tab, st);
            const double* k0 = t;
            const double* w0 = k0 + A.nz[0];
            const double* k1 = w0 + A.nz[0];
            const double* w1 = k1 + A.nz[1];
            const double* k2 = w1 + A.nz[1];
            const double* w2 = k2 + A.nz[2];
            A.cb_zero = ClassBlock{A.nz[0], A.nz[1], A.nz[2], 0, k0, nullptr, w0, nullptr, k1, w1, k2, w2, 1.0, bvol, 0};
        }
        return;
    }
    for (int ax = g.d; ax < 3; ++ax) {
        A.nz[ax] = g.n_zero[ax];
        A.nn[ax] = g.n_near[ax];
    }
    std::vector<int> rows(near_rows, near_rows + g.n_near_rows);
    setup_classes(p, A, rows, true, st);
}

void h2d(void* dst, const double* src, int64_t n, cudaStream_t st) {
    if (n > 0) cuda_check(cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDefault, st), "stage h2d");
}
void d2h(double* dst, const void* src, int64_t n, cudaStream_t st) {
    if (n > 0) cuda_check(cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDefault, st), "stage d2h");
}

}  // namespace

// Host only (no device calls): errors are std::invalid_argument.
void aft_geometry(const sewald_params_c& p, int comps, sewald_fourier_geom_c& g, std::vector<int>* near_rows) {
    if (comps < 1) throw std::invalid_argument("field storage is inconsistent");
    if (p.d < 0 || p.d > 3) throw std::invalid_argument("periodicity must be in 0..3");
    g = sewald_fourier_geom_c{};
    g.d = p.d;
    g.comps = comps;
    for (int ax = 0; ax < 3; ++ax) {
        g.n_per[ax] = g.n_far[ax] = g.n_near[ax] = g.n_zero[ax] = 1;
        if (ax < p.d) {
            g.n_per[ax] = p.M[ax];
        } else {
            g.n_far[ax] = p.M_ext[ax];
            g.n_near[ax] = padded_length(p.s_star, p.M_ext[ax]);
            g.n_zero[ax] = padded_length(p.s0, p.M_ext[ax]);
        }
    }
    std::vector<int> rows;
    if (p.d == 1 || p.d == 2) rows = near_rows_of(p);
    g.n_near_rows = static_cast<int32_t>(rows.size());
    fill_lengths(g, p.M_ext);
    if (near_rows) *near_rows = std::move(rows);
}

void stage_aft_forward(sewald_gpu_ctx* ctx, const sewald_params_c& p, const double* field,
                       const sewald_fourier_geom_c& g, double* far, double* near, double* zero) {
    sewald_fourier_geom_c want{};
    std::vector<int> rows;
    aft_geometry(p, g.comps, want, &rows);
    if (std::memcmp(&want, &g, sizeof(g)) != 0)
        throw EngineError(SEWALD_EINVAL, "field geometry does not match the grid and upsampling plan");
    cudaStream_t st = ctx->stream;
    FourierPlanAFT A;
    stage_plan(p, g, rows.data(), false, A, st);
    const int C = g.comps, d = g.d;
    const double h3 = p.h * p.h * p.h;
    const int64_t svol = cells3(p.M_ext);
    DevBuf dfield;
    double* df = static_cast<double*>(dfield.ensure(sizeof(double) * C * svol));
    h2d(df, field, C * svol, st);
    if (d == 3 || d == 0) {  // fourier.cpp:330-357
        const int64_t bvol = cells3(A.nz);
        cuDoubleComplex* z = A.zero.as<cuDoubleComplex>();
        real_to_padded_kernel<<<grid_for(C * bvol), 256, 0, st>>>(df, C, A.n[0], A.n[1], A.n[2], A.nz[0], A.nz[1],
                                                                  A.nz[2], z, h3);
        cufftSetStream(A.p_box, st);
        cufft_check(cufftExecZ2Z(A.p_box, z, z, CUFFT_FORWARD), "stage box forward");
        d2h(d == 3 ? far : zero, z, 2 * C * bvol, st);
        ctx->launches += 2;
    } else {  // fourier.cpp:359-415
        const int b1 = d == 1 ? p.M_ext[1] : 1, b2 = p.M_ext[2];
        const int z1 = d == 1 ? A.nz[1] : 1, z2 = A.nz[2];
        const int q1 = d == 1 ? A.nn[1] : 1, q2 = A.nn[2];
        const int64_t vol = svol;
        cuDoubleComplex* dfar = A.far.as<cuDoubleComplex>();
        cuDoubleComplex* dzero = A.zero.as<cuDoubleComplex>();
        cuDoubleComplex* dnear = A.near.as<cuDoubleComplex>();
        real_to_padded_kernel<<<grid_for(C * vol), 256, 0, st>>>(df, C, A.n[0], A.n[1], A.n[2], A.n[0], A.n[1],
                                                                 A.n[2], dfar, h3);
        cufftSetStream(A.p_per, st);
        for (int c = 0; c < C; ++c)
            cufft_check(cufftExecZ2Z(A.p_per, dfar + c * vol, dfar + c * vol, CUFFT_FORWARD), "stage per forward");
        class_rows_kernel<<<grid_for((int64_t)C * z1 * z2), 256, 0, st>>>(dfar, A.nrows, b1, b2, dzero, 1, z1, z2,
                                                                           A.rows_zero.as<int>(), C, 0);
        if (A.R > 0)
            class_rows_kernel<<<grid_for((int64_t)C * A.R * q1 * q2), 256, 0, st>>>(
                dfar, A.nrows, b1, b2, dnear, A.R, q1, q2, A.rows_near.as<int>(), C, 0);
        cufftSetStream(A.p_far, st);
        cufft_check(cufftExecZ2Z(A.p_far, dfar, dfar, CUFFT_FORWARD), "stage far forward");
        cufftSetStream(A.p_zero, st);
        cufft_check(cufftExecZ2Z(A.p_zero, dzero, dzero, CUFFT_FORWARD), "stage zero forward");
        if (A.R > 0) cufftSetStream(A.p_near, st);
        if (A.R > 0) cufft_check(cufftExecZ2Z(A.p_near, dnear, dnear, CUFFT_FORWARD), "stage near forward");
        d2h(far, dfar, 2 * g.far_len, st);
        d2h(zero, dzero, 2 * g.zero_len, st);
        d2h(near, dnear, 2 * g.near_len, st);
        ctx->launches += 3 + C + 2 + (A.R > 0 ? 2 : 0);
    }
    cuda_check(cudaStreamSynchronize(st), "stage aft_forward");
}

void stage_aft_inverse(sewald_gpu_ctx* ctx, const sewald_params_c& p, const sewald_fourier_geom_c& g,
                       const int32_t* near_rows, const double* far, const double* near, const double* zero,
                       double* field_out) {
    check_geometry(p, g);
    cudaStream_t st = ctx->stream;
    FourierPlanAFT A;
    stage_plan(p, g, near_rows, false, A, st);
    const int C = g.comps, d = g.d;
    const double h3 = p.h * p.h * p.h;
    const int64_t svol = cells3(p.M_ext);
    DevBuf dout;
    double* dfield = static_cast<double*>(dout.ensure(sizeof(double) * C * svol));
    if (d == 3 || d == 0) {  // fourier.cpp:425-456
        const int64_t bvol = cells3(A.nz);
        cuDoubleComplex* z = A.zero.as<cuDoubleComplex>();
        h2d(z, d == 3 ? far : zero, 2 * C * bvol, st);
        cufftSetStream(A.p_box, st);
        cufft_check(cufftExecZ2Z(A.p_box, z, z, CUFFT_INVERSE), "stage box inverse");
        padded_to_real_kernel<<<grid_for(C * svol), 256, 0, st>>>(z, A.nz[0], A.nz[1], A.nz[2], A.n[0], A.n[1],
                                                                  A.n[2], bvol, dfield, C,
                                                                  1.0 / (h3 * static_cast<double>(bvol)));
        ctx->launches += 2;
    } else {  // fourier.cpp:458-519
        const int b1 = d == 1 ? p.M_ext[1] : 1, b2 = p.M_ext[2];
        const int z1 = d == 1 ? A.nz[1] : 1, z2 = A.nz[2];
        const int q1 = d == 1 ? A.nn[1] : 1, q2 = A.nn[2];
        const int64_t vol = svol;
        cuDoubleComplex* dfar = A.far.as<cuDoubleComplex>();
        cuDoubleComplex* dzero = A.zero.as<cuDoubleComplex>();
        cuDoubleComplex* dnear = A.near.as<cuDoubleComplex>();
        h2d(dfar, far, 2 * g.far_len, st);
        h2d(dzero, zero, 2 * g.zero_len, st);
        h2d(dnear, near, 2 * g.near_len, st);
        double inv_free = 1.0, inv_zero = 1.0, inv_near = 1.0, inv_per = 1.0;
        for (int ax = d; ax < 3; ++ax) {
            inv_free /= g.n_far[ax];
            inv_zero /= g.n_zero[ax];
            inv_near /= g.n_near[ax];
        }
        for (int ax = 0; ax < d; ++ax) inv_per /= p.M[ax];
        cufftSetStream(A.p_far, st);
        cufft_check(cufftExecZ2Z(A.p_far, dfar, dfar, CUFFT_INVERSE), "stage far inverse");
        scale_complex_kernel<<<grid_for(C * vol), 256, 0, st>>>(dfar, C * vol, inv_free);
        cufftSetStream(A.p_zero, st);
        cufft_check(cufftExecZ2Z(A.p_zero, dzero, dzero, CUFFT_INVERSE), "stage zero inverse");
        scale_complex_kernel<<<grid_for(g.zero_len), 256, 0, st>>>(dzero, g.zero_len, inv_zero);
        class_rows_kernel<<<grid_for((int64_t)C * z1 * z2), 256, 0, st>>>(dfar, A.nrows, b1, b2, dzero, 1, z1, z2,
                                                                           A.rows_zero.as<int>(), C, 1);
        ctx->launches += 5;
        if (A.R > 0) {
            cufftSetStream(A.p_near, st);
            cufft_check(cufftExecZ2Z(A.p_near, dnear, dnear, CUFFT_INVERSE), "stage near inverse");
            scale_complex_kernel<<<grid_for(g.near_len), 256, 0, st>>>(dnear, g.near_len, inv_near);
            class_rows_kernel<<<grid_for((int64_t)C * A.R * q1 * q2), 256, 0, st>>>(
                dfar, A.nrows, b1, b2, dnear, A.R, q1, q2, A.rows_near.as<int>(), C, 1);
            ctx->launches += 3;
        }
        cufftSetStream(A.p_per, st);
        for (int c = 0; c < C; ++c)
            cufft_check(cufftExecZ2Z(A.p_per, dfar + c * vol, dfar + c * vol, CUFFT_INVERSE), "stage per inverse");
        padded_to_real_kernel<<<grid_for(C * vol), 256, 0, st>>>(dfar, A.n[0], A.n[1], A.n[2], A.n[0], A.n[1], A.n[2],
                                                                 vol, dfield, C, inv_per / h3);
        ctx->launches += C + 1;
    }
    d2h(field_out, dfield, C * svol, st);
    cuda_check(cudaStreamSynchronize(st), "stage aft_inverse");
}

// scale (fourier.cpp:522-666) with spec, or (fourier.cpp:668-720) with the
// 0P table when table != nullptr (table_n = its mode grid).
void stage_scale(sewald_gpu_ctx* ctx, const sewald_params_c& p, int kind, const sewald_modspec_c* spec,
                 const int32_t* table_n, const double* table, double xi, const sewald_fourier_geom_c& g,
                 const int32_t* near_rows, const double* far, const double* near, const double* zero,
                 double* far_out, double* near_out, double* zero_out) {
    if (table) {
        if (p.d != 0 || g.d != 0) throw EngineError(SEWALD_EINVAL, "precomputed kernels apply to d = 0 only");
        if (g.n_zero[0] != table_n[0] || g.n_zero[1] != table_n[1] || g.n_zero[2] != table_n[2])
            throw EngineError(SEWALD_EINVAL, "kernel table was built for a different padded grid");
    } else if (g.d != p.d || spec->d != p.d) {
        throw EngineError(SEWALD_EINVAL, "field, kernel and grid periodicity must agree");
    }
    if (g.comps != strength_comps(kind))
        throw EngineError(SEWALD_EINVAL, "field component count does not match the kernel");
    if (!(xi > 0.0)) throw EngineError(SEWALD_EINVAL, "xi must be positive");
    check_window_h(p);
    check_geometry(p, g);
    cudaStream_t st = ctx->stream;
    FourierPlanAFT A;
    stage_plan(p, g, near_rows, true, A, st);
    const ModSpec m = spec ? make_modspec_full(spec->kind, spec->d, spec->R, spec->a_B, spec->b_B, spec->ell_H,
                                               spec->ell_B, spec->c_B)
                           : make_modspec(kind, 0, 1.0);
    const int C = g.comps, d = g.d;
    if (d == 3 || d == 0) {
        const int64_t bvol = cells3(A.nz);
        cuDoubleComplex* z = A.zero.as<cuDoubleComplex>();
        h2d(z, d == 3 ? far : zero, 2 * C * bvol, st);
        DevBuf dt;
        const cuDoubleComplex* dtab = nullptr;
        if (table) {
            cuDoubleComplex* t = static_cast<cuDoubleComplex*>(dt.ensure(sizeof(cuDoubleComplex) * bvol));
            h2d(t, table, 2 * bvol, st);
            dtab = t;
        }
        launch_scale_class(kind, m, A.cb_zero, xi, z, dtab, st);
        d2h(d == 3 ? far_out : zero_out, z, 2 * 3 * bvol, st);
        ctx->launches += 1;
    } else {
        cuDoubleComplex* dfar = A.far.as<cuDoubleComplex>();
        cuDoubleComplex* dzero = A.zero.as<cuDoubleComplex>();
        cuDoubleComplex* dnear = A.near.as<cuDoubleComplex>();
        h2d(dfar, far, 2 * g.far_len, st);
        h2d(dzero, zero, 2 * g.zero_len, st);
        h2d(dnear, near, 2 * g.near_len, st);
        launch_scale_class(kind, m, A.cb_far, xi, dfar, nullptr, st);
        launch_scale_class(kind, m, A.cb_zero, xi, dzero, nullptr, st);
        if (A.R > 0) launch_scale_class(kind, m, A.cb_near, xi, dnear, nullptr, st);
        d2h(far_out, dfar, 2 * 3 * (g.far_len / C), st);
        d2h(zero_out, dzero, 2 * 3 * (g.zero_len / C), st);
        d2h(near_out, dnear, 2 * 3 * (g.near_len / C), st);
        ctx->launches += A.R > 0 ? 3 : 2;
    }
    cuda_check(cudaGetLastError(), "stage scale");
    cuda_check(cudaStreamSynchronize(st), "stage scale");
}

void stage_precompute_0p(sewald_gpu_ctx* ctx, const sewald_params_c& p, int kind, double R, int32_t n_out[3],
                         double* table_out) {
    if (p.d != 0) throw EngineError(SEWALD_EINVAL, "kernel precomputation applies to d = 0 only");
    if (!(R > 0.0)) throw EngineError(SEWALD_EINVAL, "truncation radius must be positive");
    for (int ax = 0; ax < 3; ++ax) n_out[ax] = 2 * p.M_ext[ax];
    if (!table_out) return;
    DevBuf t;
    ctx->launches += build_table_0p(p, kind, R, t, ctx->stream);
    d2h(table_out, t.ptr, 2 * cells3(n_out), ctx->stream);
    cuda_check(cudaStreamSynchronize(ctx->stream), "stage precompute_0p");
}

}  // namespace sewald_b200
