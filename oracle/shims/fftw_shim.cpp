// ORACLE TEST INFRASTRUCTURE — not product code.
//
// Implementation of the FFTW3 subset declared in fftw3.h. Each distinct
// (length, sign) pair gets a cached 1-D plan: a factorisation (radix 4 first,
// then 2, 3, 5, remaining primes) plus a long-double-accurate twiddle table.
// Prime factors above kBluesteinMin are transformed by Bluestein's chirp-z
// algorithm on a power-of-two length. Accuracy is ~1e-16 relative per
// butterfly level, which is what the reference's FFT-boundary tests
// (/root/reference/proj/tests/test_fourier.cpp:240-353, 1e-12) require.
#include "fftw3.h"

#include <cmath>
#include <complex>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

namespace {

using cd = std::complex<double>;
constexpr int kBluesteinMin = 67;

struct Plan1D {
    int n = 1;
    int sign = -1;
    std::vector<int> factors;
    std::vector<cd> tw;  // tw[j] = exp(sign * 2 pi i j / n)
    // Bluestein data when n itself is a large prime (leaf transform).
    int nb = 0;
    std::vector<cd> chirp;      // exp(sign * pi i j^2 / n), j < n
    std::vector<cd> chirp_hat;  // FFT_nb of the conjugate chirp, zero padded
    std::shared_ptr<const Plan1D> pow2_fwd, pow2_bwd;
};

std::shared_ptr<const Plan1D> get_plan(int n, int sign);

cd unit_root(long j, long n, int sign) {
    // exp(sign * 2 pi i j / n) evaluated in long double and rounded once.
    j %= n;
    if (j < 0) j += n;
    const long double ang = 2.0L * 3.141592653589793238462643383279502884L *
                            static_cast<long double>(j) / static_cast<long double>(n);
    return cd(static_cast<double>(std::cos(ang)), static_cast<double>(sign * std::sin(ang)));
}

std::vector<int> factorize(int n) {
    std::vector<int> f;
    while (n % 4 == 0) { f.push_back(4); n /= 4; }
    while (n % 2 == 0) { f.push_back(2); n /= 2; }
    for (int p = 3; static_cast<long>(p) * p <= n; p += 2)
        while (n % p == 0) { f.push_back(p); n /= p; }
    if (n > 1) f.push_back(n);
    return f;
}

void transform(const cd* in, long is, cd* out, int n, const Plan1D& P, std::size_t fi, long twstride);

void bluestein(const cd* in, long is, cd* out, const Plan1D& B) {
    const int n = B.n, nb = B.nb;
    std::vector<cd> a(nb, cd{}), A(nb);
    for (int j = 0; j < n; ++j) a[j] = in[j * is] * B.chirp[j];
    transform(a.data(), 1, A.data(), nb, *B.pow2_fwd, 0, 1);
    for (int j = 0; j < nb; ++j) A[j] *= B.chirp_hat[j];
    transform(A.data(), 1, a.data(), nb, *B.pow2_bwd, 0, 1);
    const double inv = 1.0 / nb;
    for (int k = 0; k < n; ++k) out[k] = a[k] * inv * B.chirp[k];
}

// Decimation in time: out[0..n) = DFT_n of in[0], in[is], in[2 is], ...
// Twiddles of this level are W_n^j = P.tw[j * twstride].
void transform(const cd* in, long is, cd* out, int n, const Plan1D& P, std::size_t fi, long twstride) {
    if (n == 1) { out[0] = in[0]; return; }
    const int p = P.factors[fi];
    if (p == n && p >= kBluesteinMin) {
        bluestein(in, is, out, *get_plan(p, P.sign));
        return;
    }
    const int m = n / p;
    for (int r = 0; r < p; ++r) transform(in + r * is, is * p, out + r * m, m, P, fi + 1, twstride * p);

    const cd* W = P.tw.data();
    const long wstep = twstride;          // W_n^1
    const long pstep = twstride * m;      // W_p^1 = W_n^m
    if (p == 2) {
        for (int k = 0; k < m; ++k) {
            const cd a = out[k];
            const cd b = out[m + k] * W[k * wstep];
            out[k] = a + b;
            out[m + k] = a - b;
        }
    } else if (p == 4) {
        const cd jsign(0.0, static_cast<double>(P.sign));  // W_4^1
        for (int k = 0; k < m; ++k) {
            const cd a0 = out[k];
            const cd a1 = out[m + k] * W[k * wstep];
            const cd a2 = out[2 * m + k] * W[2 * k * wstep];
            const cd a3 = out[3 * m + k] * W[3 * k * wstep];
            const cd s02 = a0 + a2, d02 = a0 - a2;
            const cd s13 = a1 + a3, d13 = (a1 - a3) * jsign;
            out[k] = s02 + s13;
            out[m + k] = d02 + d13;
            out[2 * m + k] = s02 - s13;
            out[3 * m + k] = d02 - d13;
        }
    } else {
        std::vector<cd> t(p);
        for (int k = 0; k < m; ++k) {
            t[0] = out[k];
            for (int r = 1; r < p; ++r) t[r] = out[r * m + k] * W[static_cast<long>(r) * k * wstep];
            for (int q = 0; q < p; ++q) {
                cd acc = t[0];
                for (int r = 1; r < p; ++r) acc += t[r] * W[((static_cast<long>(r) * q) % p) * pstep];
                out[q * m + k] = acc;
            }
        }
    }
}

std::shared_ptr<const Plan1D> build_plan(int n, int sign) {
    auto P = std::make_shared<Plan1D>();
    P->n = n;
    P->sign = sign;
    P->factors = factorize(n);
    P->tw.resize(n);
    for (int j = 0; j < n; ++j) P->tw[j] = unit_root(j, n, sign);
    const bool prime_leaf = P->factors.size() == 1 && n >= kBluesteinMin;
    if (prime_leaf) {
        int nb = 1;
        while (nb < 2 * n - 1) nb <<= 1;
        P->nb = nb;
        P->pow2_fwd = get_plan(nb, -1);
        P->pow2_bwd = get_plan(nb, +1);
        P->chirp.resize(n);
        // exp(sign * pi i j^2 / n) = unit_root(j^2, 2n)
        for (int j = 0; j < n; ++j)
            P->chirp[j] = unit_root((static_cast<long>(j) * j) % (2L * n), 2L * n, sign);
        std::vector<cd> b(nb, cd{});
        for (int j = 0; j < n; ++j) {
            b[j] = std::conj(P->chirp[j]);
            if (j) b[nb - j] = std::conj(P->chirp[j]);
        }
        P->chirp_hat.resize(nb);
        transform(b.data(), 1, P->chirp_hat.data(), nb, *P->pow2_fwd, 0, 1);
    }
    return P;
}

std::mutex g_mu;
std::map<std::pair<int, int>, std::shared_ptr<const Plan1D>> g_cache;

std::shared_ptr<const Plan1D> get_plan(int n, int sign) {
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_cache.find({n, sign});
        if (it != g_cache.end()) return it->second;
    }
    auto P = build_plan(n, sign);
    std::lock_guard<std::mutex> lk(g_mu);
    return g_cache.emplace(std::make_pair(n, sign), P).first->second;
}

}  // namespace

struct oracle_fftw_plan_s {
    int n, howmany, istride, idist, ostride, odist, sign;
    fftw_complex* in;
    fftw_complex* out;
    std::shared_ptr<const Plan1D> plan;
};

fftw_plan fftw_plan_many_dft(int rank, const int* n, int howmany, fftw_complex* in, const int*,
                             int istride, int idist, fftw_complex* out, const int*, int ostride,
                             int odist, int sign, unsigned) {
    if (rank != 1) return nullptr;
    auto* p = new oracle_fftw_plan_s{n[0], howmany, istride, idist, ostride, odist, sign, in, out,
                                     get_plan(n[0], sign)};
    return p;
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
    const int n = p->n;
    std::vector<cd> a(n), b(n);
    for (int h = 0; h < p->howmany; ++h) {
        const cd* src = reinterpret_cast<const cd*>(in) + static_cast<long>(h) * p->idist;
        cd* dst = reinterpret_cast<cd*>(out) + static_cast<long>(h) * p->odist;
        for (int i = 0; i < n; ++i) a[i] = src[static_cast<long>(i) * p->istride];
        transform(a.data(), 1, b.data(), n, *p->plan, 0, 1);
        for (int i = 0; i < n; ++i) dst[static_cast<long>(i) * p->ostride] = b[i];
    }
}

void fftw_execute(const fftw_plan p) { fftw_execute_dft(p, p->in, p->out); }

void fftw_destroy_plan(fftw_plan p) { delete p; }
