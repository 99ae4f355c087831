// Offline model: cluster-aligned j-blocks, classification of (cluster A, cluster B)
// combos into dense (symmetric rotation steps) and sparse (per-target pooled
// non-symmetric evaluation) by bbox-center distance, cost in fp64 lane-slots:
//   dense:  executed rotation steps x 32, one sym pair evaluation per slot (cost 1)
//   sparse: 2 directed evaluations per accepted pair at pooled utilisation u_n,
//           cost ratio 0.9 per slot (111.5 vs 124 flops)
// Build: g++ -O2 -std=c++17 rs_split_sim.cpp -o rs_split_sim
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <random>
#include <vector>

int main(int argc, char** argv) {
    const int N = argc > 1 ? atoi(argv[1]) : 1000000;
    const double rc = argc > 2 ? atof(argv[2]) : 0.1367;
    const double ppc = argc > 3 ? atof(argv[3]) : 28.0;
    const int nsample = argc > 4 ? atoi(argv[4]) : 200;
    const double un = argc > 5 ? atof(argv[5]) : 0.9;
    const double thr_sparse = argc > 6 ? atof(argv[6]) : 1.0;
    const int W = argc > 7 ? atoi(argv[7]) : 8;
    std::mt19937_64 rng(11);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    std::vector<double> x(3 * (size_t)N);
    for (auto& v : x) v = U(rng);
    int nc = std::max(1, (int)std::floor(std::cbrt(N / ppc)));
    const double w = 1.0 / nc;
    std::vector<uint64_t> key(N);
    std::vector<int> idx(N);
    for (int i = 0; i < N; ++i) {
        int c[3];
        for (int a = 0; a < 3; ++a) c[a] = std::min(nc - 1, (int)(x[3 * i + a] / w));
        int sub = std::min(255, (int)((x[3 * i] / w - c[0]) * 256));
        key[i] = ((((uint64_t)c[2] * nc + c[1]) * nc + c[0]) << 8) | sub;
        idx[i] = i;
    }
    std::sort(idx.begin(), idx.end(), [&](int a, int b) { return key[a] < key[b]; });
    std::vector<double> p(3 * (size_t)N);
    for (int k = 0; k < N; ++k)
        for (int a = 0; a < 3; ++a) p[3 * k + a] = x[3 * idx[k] + a];
    const int ncl = (N + 31) / 32;
    std::vector<double> cen(3 * (size_t)ncl), lo(3 * (size_t)ncl), hi(3 * (size_t)ncl);
    for (int c = 0; c < ncl; ++c)
        for (int a = 0; a < 3; ++a) {
            double l = 1e9, h = -1e9;
            for (int t = 32 * c; t < std::min(N, 32 * c + 32); ++t) {
                l = std::min(l, p[3 * t + a]);
                h = std::max(h, p[3 * t + a]);
            }
            lo[3 * c + a] = l; hi[3 * c + a] = h; cen[3 * c + a] = 0.5 * (l + h);
        }
    // cluster grid for neighbour search (uniform bins on the center)
    const int nb = std::max(1, (int)(1.0 / rc) * 2);
    std::vector<std::vector<int>> bins((size_t)nb * nb * nb);
    auto bidx = [&](double v) { return std::min(nb - 1, std::max(0, (int)(v * nb))); };
    for (int c = 0; c < ncl; ++c)
        bins[((size_t)bidx(cen[3 * c + 2]) * nb + bidx(cen[3 * c + 1])) * nb + bidx(cen[3 * c])].push_back(c);
    const double rc2 = rc * rc;
    const int NT = 24;  // thresholds on D / rc
    double dense_slots[NT] = {0}, sparse_pairs[NT] = {0}, Etot = 0, cur_slots = 0;
    std::uniform_int_distribution<int> pick(0, ncl - 1);
    double sp_pairs = 0, sp_slots = 0, sp_slots_nopool = 0;
    for (int t = 0; t < nsample; ++t) {
        int A;
        for (;;) {
            A = pick(rng);
            bool ok = true;
            for (int a = 0; a < 3; ++a) ok = ok && lo[3 * A + a] > 2 * rc && hi[3 * A + a] < 1 - 2 * rc;
            if (ok) break;
        }
        int b0[3], b1[3];
        for (int a = 0; a < 3; ++a) { b0[a] = bidx(lo[3 * A + a] - rc - 0.05); b1[a] = bidx(hi[3 * A + a] + rc + 0.05); }
        int lanecnt[32] = {0}, wn = 0;
        auto wflush = [&]() {
            int mx = 0, tot = 0;
            for (int l = 0; l < 32; ++l) { mx = std::max(mx, lanecnt[l]); tot += lanecnt[l]; lanecnt[l] = 0; }
            sp_pairs += tot;
            sp_slots += 32.0 * mx;
            wn = 0;
        };
        for (int bz = b0[2]; bz <= b1[2]; ++bz)
            for (int by = b0[1]; by <= b1[1]; ++by)
                for (int bx = b0[0]; bx <= b1[0]; ++bx)
                    for (int B : bins[((size_t)bz * nb + by) * nb + bx]) {
                        if (B != A) {  // sparse non-sym pass of A: all B, A-side counts only
                            double d2s = 0;
                            for (int a = 0; a < 3; ++a) {
                                double d = std::max(0.0, std::max(lo[3 * B + a] - hi[3 * A + a], lo[3 * A + a] - hi[3 * B + a]));
                                d2s += d * d;
                            }
                            double Dc = 0;
                            for (int a = 0; a < 3; ++a) { double d = cen[3 * A + a] - cen[3 * B + a]; Dc += d * d; }
                            if (d2s < rc2 && std::sqrt(Dc) / rc >= thr_sparse) {
                                int mxl = 0, tl = 0;
                                for (int l = 0; l < 32; ++l) {
                                    int c = 0;
                                    for (int j = 0; j < 32; ++j) {
                                        double r2 = 0;
                                        for (int a = 0; a < 3; ++a) { double d = p[3 * (32 * A + l) + a] - p[3 * (32 * B + j) + a]; r2 += d * d; }
                                        c += r2 < rc2;
                                    }
                                    lanecnt[l] += c;
                                    mxl = std::max(mxl, c);
                                    tl += c;
                                }
                                sp_slots_nopool += 32.0 * mxl;
                                if (tl && ++wn == W) wflush();
                            }
                        }
                        if (B < A) continue;  // half rule at cluster level (count each combo once)
                        // bbox distance prune (as the kernel's row scan would)
                        double d2 = 0;
                        for (int a = 0; a < 3; ++a) {
                            double d = std::max(0.0, std::max(lo[3 * B + a] - hi[3 * A + a], lo[3 * A + a] - hi[3 * B + a]));
                            d2 += d * d;
                        }
                        if (d2 >= rc2) continue;
                        uint32_t m[32];
                        int E = 0;
                        for (int l = 0; l < 32; ++l) {
                            m[l] = 0;
                            int ia = 32 * A + l;
                            for (int s = 0; s < 32; ++s) {
                                int jb = 32 * B + ((l + s) & 31);
                                if (B == A && jb <= ia) continue;
                                double r2 = 0;
                                for (int a = 0; a < 3; ++a) { double d = p[3 * ia + a] - p[3 * jb + a]; r2 += d * d; }
                                if (r2 < rc2) m[l] |= 1u << s;
                            }
                            E += __builtin_popcount(m[l]);
                        }
                        uint32_t OR = 0;
                        for (int l = 0; l < 32; ++l) OR |= m[l];
                        const int steps = __builtin_popcount(OR);
                        double D = 0;
                        for (int a = 0; a < 3; ++a) { double d = cen[3 * A + a] - cen[3 * B + a]; D += d * d; }
                        D = std::sqrt(D) / rc;
                        Etot += E;
                        cur_slots += 32.0 * steps;
                        for (int k = 0; k < NT; ++k) {
                            const double thr = 0.5 + 0.05 * k;  // dense iff D < thr
                            if (D < thr) dense_slots[k] += 32.0 * steps;
                            else sparse_pairs[k] += E;
                        }
                    }
        if (wn) wflush();
    }
    printf("sparse non-sym pass (thr %.2f): pooled W=%d util %.3f, per-block util %.3f\n", thr_sparse, W,
           sp_pairs / std::max(sp_slots, 1.0), sp_pairs / std::max(sp_slots_nopool, 1.0));
    printf("cluster-aligned blocks: util %.3f (pairs/cluster %.0f)\n", Etot / cur_slots, Etot / nsample);
    for (int k = 0; k < NT; ++k) {
        const double cost = dense_slots[k] + 0.9 * 2.0 * sparse_pairs[k] / un;
        printf("thr %.2f rc: sparse pairs %5.1f%%  dense util %.3f  cost vs current %.3f\n", 0.5 + 0.05 * k,
               100 * sparse_pairs[k] / Etot, (Etot - sparse_pairs[k]) / std::max(dense_slots[k], 1.0), cost / cur_slots);
    }
}
