// Offline model of the real-space sym kernel's lane utilisation (c2 geometry),
// plus pooling of sparse blocks (rs_pool_sim: per-block pair threshold):
// uniform points, the kernel's cell grid / sort / cluster / j-block scheme,
// and the fraction of fp64 lane-steps that carry an accepted pair under
// (a) the current rotation steps (one step per rotation with any pair) and
// (b) packed super-steps: rotations with disjoint lane sets AND disjoint
//     j sets merged into one step (greedy first-fit), lane picks its own s.
// Build: g++ -O2 -std=c++17 rs_pack_sim.cpp -o rs_pack_sim
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <random>
#include <vector>

static inline uint32_t rotl(uint32_t x, int s) { return s ? (x << s) | (x >> (32 - s)) : x; }

int main(int argc, char** argv) {
    const int N = argc > 1 ? atoi(argv[1]) : 1000000;
    const double rc = argc > 2 ? atof(argv[2]) : 0.1367;
    const double ppc = argc > 3 ? atof(argv[3]) : 28.0;
    const int nclusters = argc > 4 ? atoi(argv[4]) : 400;
    const int CS = argc > 5 ? atoi(argv[5]) : 32;  // i-cluster size; lanes l and l+CS.. share i
    const int W = argc > 6 ? atoi(argv[6]) : 4;    // blocks pooled by the windowed packer
    const double AX = argc > 7 ? atof(argv[7]) : 1.0;  // cell aspect w_x / w_yz (cell volume kept)
    const int JB = argc > 8 ? atoi(argv[8]) : 32;      // j-block size (16: lanes l, l+16 share slot j)
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    std::vector<double> x(3 * (size_t)N);
    for (auto& v : x) v = U(rng);
    const double nc0 = std::cbrt(N / ppc);
    const int ncx = std::max(1, (int)std::floor(nc0 / std::pow(AX, 2.0 / 3.0)));
    const int nc = std::max(1, (int)std::floor(nc0 * std::pow(AX, 1.0 / 3.0)));  // y, z
    const double w = 1.0 / nc, wx = 1.0 / ncx;
    std::vector<uint64_t> key(N);
    std::vector<int> idx(N);
    for (int i = 0; i < N; ++i) {
        int c[3];
        c[0] = std::min(ncx - 1, (int)(x[3 * i] / wx));
        for (int a = 1; a < 3; ++a) c[a] = std::min(nc - 1, (int)(x[3 * i + a] / w));
        int sub = std::min(255, (int)((x[3 * i] / wx - c[0]) * 256));
        key[i] = ((((uint64_t)c[2] * nc + c[1]) * ncx + c[0]) << 8) | sub;
        idx[i] = i;
    }
    std::sort(idx.begin(), idx.end(), [&](int a, int b) { return key[a] < key[b]; });
    std::vector<double> p(3 * (size_t)N);
    std::vector<int64_t> off((size_t)nc * nc * ncx + 1, 0);
    for (int k = 0; k < N; ++k) {
        for (int a = 0; a < 3; ++a) p[3 * k + a] = x[3 * idx[k] + a];
        off[(key[idx[k]] >> 8) + 1]++;
    }
    for (size_t c = 0; c + 1 < off.size(); ++c) off[c + 1] += off[c];
    const double rc2 = rc * rc;
    double E = 0, S_cur = 0, S_pack = 0, S_lb = 0, blocks = 0;
    double hE[11] = {0}, hS[11] = {0}, partialCnt = 0, sumCnt = 0;
    double S_win = 0;
    const int NTH = 9;
    const int TH[NTH] = {32, 64, 96, 128, 192, 256, 320, 410, 512};
    double Sd[NTH] = {0}, Ps[NTH] = {0}, Pb[NTH] = {0}, Pl[NTH] = {0};
    const int NK = 6;
    const int KT[NK] = {4, 8, 12, 16, 20, 24};
    double Sk[NK] = {0}, Pk[NK] = {0}, Bk[NK] = {0};  // steps kept, pooled pairs, pooled batches (per block)
    struct Ent { uint32_t a, v; int blk; };
    std::vector<Ent> win;
    int win_blocks = 0;
    auto flush = [&]() {
        // greedy first-fit, entries in descending popcount
        std::sort(win.begin(), win.end(), [](const Ent& x, const Ent& y) { return __builtin_popcount(x.a) > __builtin_popcount(y.a); });
        std::vector<uint32_t> Uo;
        std::vector<std::vector<uint32_t>> Vo;  // per superstep, per block j occupancy
        for (const Ent& e : win) {
            size_t k = 0;
            for (; k < Uo.size(); ++k) if (!(Uo[k] & e.a) && !(Vo[k][e.blk] & e.v)) break;
            if (k == Uo.size()) { Uo.push_back(0); Vo.emplace_back(W, 0u); }
            Uo[k] |= e.a;
            Vo[k][e.blk] |= e.v;
        }
        S_win += Uo.size();
        win.clear();
        win_blocks = 0;
    };
    const int ncl = (N + CS - 1) / CS;
    std::uniform_int_distribution<int> pick(0, ncl - 1);
    for (int t = 0; t < nclusters; ++t) {
        int cl;
        double lo[3], hi[3];
        // interior clusters only (no periodic images in the model)
        for (;;) {
            cl = pick(rng);
            for (int a = 0; a < 3; ++a) { lo[a] = 1e9; hi[a] = -1e9; }
            for (int l = 0; l < CS; ++l)
                for (int a = 0; a < 3; ++a) {
                    lo[a] = std::min(lo[a], p[3 * ((int64_t)CS * cl + l) + a]);
                    hi[a] = std::max(hi[a], p[3 * ((int64_t)CS * cl + l) + a]);
                }
            bool ok = true;
            for (int a = 0; a < 3; ++a) ok = ok && lo[a] - rc > 0.0 && hi[a] + rc < 1.0;
            if (ok) break;
        }
        const int64_t istart = CS * (int64_t)cl;
        int clo[3], chi[3];
        for (int a = 0; a < 3; ++a) {
            const double wa = a == 0 ? wx : w;
            clo[a] = (int)std::floor((lo[a] - rc) / wa);
            chi[a] = (int)std::floor((hi[a] + rc) / wa);
        }
        for (int cz = clo[2]; cz <= chi[2]; ++cz)
            for (int cy = clo[1]; cy <= chi[1]; ++cy) {
                double zlo = cz * w, zhi = zlo + w, ylo = cy * w, yhi = ylo + w;
                double dz = std::max(0.0, std::max(zlo - hi[2], lo[2] - zhi));
                double dy = std::max(0.0, std::max(ylo - hi[1], lo[1] - yhi));
                double lat2 = dy * dy + dz * dz;
                if (lat2 >= rc2) continue;
                double ext = std::sqrt(rc2 - lat2);
                double xl = lo[0] - ext, xh = hi[0] + ext;
                if (getenv("TRIM")) {  // per-particle union of the x-intervals
                    xl = 1e9; xh = -1e9;
                    for (int l = 0; l < CS; ++l) {
                        const double* pa = &p[3 * ((int64_t)CS * cl + l)];
                        double dy2 = std::max(0.0, std::max(ylo - pa[1], pa[1] - yhi));
                        double dz2 = std::max(0.0, std::max(zlo - pa[2], pa[2] - zhi));
                        double la = dy2 * dy2 + dz2 * dz2;
                        if (la >= rc2) continue;
                        double e = std::sqrt(rc2 - la);
                        xl = std::min(xl, pa[0] - e); xh = std::max(xh, pa[0] + e);
                    }
                    if (xl > xh) continue;
                }
                int cxl = std::max((int)std::floor(xl / wx), clo[0]);
                int cxh = std::min((int)std::floor(xh / wx), chi[0]);
                if (cxl > cxh) continue;
                int64_t rb = ((int64_t)cz * nc + cy) * ncx;
                int64_t b0 = off[rb + cxl], b1 = off[rb + cxh + 1];
                if (b0 < istart) b0 = istart;
                for (int64_t jb = b0; jb < b1; jb += JB) {
                    int cnt = (int)std::min<int64_t>(JB, b1 - jb);
                    uint32_t m[32], A[32];
                    int degj[32] = {0};
                    int Eb = 0, maxl = 0;
                    for (int l = 0; l < 32; ++l) {
                        m[l] = 0;
                        const int64_t ia = istart + (l % CS);
                        for (int s = 0; s < (JB < CS ? JB : CS); ++s) {
                            int j = JB == 32 ? ((l + s) & 31) : ((l + s) % JB);
                            if (j >= cnt) continue;
                            int64_t jg = jb + j;
                            if (jg <= ia) continue;
                            double d2 = 0;
                            for (int a = 0; a < 3; ++a) {
                                double d = p[3 * ia + a] - p[3 * jg + a];
                                d2 += d * d;
                            }
                            if (d2 < rc2) { m[l] |= 1u << s; degj[j]++; }
                        }
                        Eb += __builtin_popcount(m[l]);
                        maxl = std::max(maxl, __builtin_popcount(m[l]));
                    }
                    if (!Eb) { blocks += 1; continue; }
                    uint32_t OR = 0;
                    for (int s = 0; s < 32; ++s) {
                        A[s] = 0;
                        for (int l = 0; l < 32; ++l) A[s] |= ((m[l] >> s) & 1u) << l;
                        if (A[s]) OR |= 1u << s;
                    }
                    // greedy first-fit packing, rotations in descending popcount
                    int order[32], no = 0;
                    for (int s = 0; s < 32; ++s) if (A[s]) order[no++] = s;
                    std::sort(order, order + no, [&](int a, int b) { return __builtin_popcount(A[a]) > __builtin_popcount(A[b]); });
                    uint32_t Uo[32], Vo[32];
                    int K = 0;
                    for (int q = 0; q < no; ++q) {
                        int s = order[q];
                        uint32_t a = A[s], v = rotl(A[s], s);
                        int k = 0;
                        for (; k < K; ++k) if (!(Uo[k] & a) && !(Vo[k] & v)) break;
                        if (k == K) { Uo[K] = 0; Vo[K] = 0; ++K; }
                        Uo[k] |= a;
                        Vo[k] |= v;
                    }
                    for (int q = 0; q < no; ++q) win.push_back({A[order[q]], rotl(A[order[q]], order[q]), win_blocks});
                    if (++win_blocks == W) flush();
                    int maxj = 0;
                    for (int j = 0; j < 32; ++j) maxj = std::max(maxj, degj[j]);
                    E += Eb;
                    S_cur += __builtin_popcount(OR);
                    for (int q = 0; q < NK; ++q) {
                        int kept = 0, pp = 0;
                        for (int s2 = 0; s2 < 32; ++s2) {
                            const int c = __builtin_popcount(A[s2]);
                            if (!c) continue;
                            if (c >= KT[q]) ++kept; else pp += c;
                        }
                        Sk[q] += kept; Pk[q] += pp; Bk[q] += (pp + 31) / 32;
                    }
                    for (int q = 0; q < NTH; ++q) {
                        if (Eb < TH[q]) { Ps[q] += Eb; Pb[q] += (Eb + 31) / 32; Pl[q] += maxl; } else Sd[q] += __builtin_popcount(OR);
                    }
                    {
                        int bin = (int)(10.0 * Eb / (32.0 * CS));
                        if (bin > 10) bin = 10;
                        hE[bin] += Eb;
                        hS[bin] += __builtin_popcount(OR);
                        sumCnt += cnt;
                        if (cnt < 32) partialCnt += 1;
                    }
                    S_pack += K;
                    S_lb += std::max({maxl, maxj, (Eb + 31) / 32});
                    blocks += 1;
                }
            }
        if (win_blocks) flush();
    }
    printf("N=%d rc=%.4f ppc=%.1f cells/axis=%d  blocks=%.0f  pairs/cluster=%.0f\n", N, rc, ppc, nc, blocks, E / nclusters);
    printf("utilisation: current %.3f  packed %.3f  lower-bound %.3f  window(W=%d) %.3f\n", E / (32 * S_cur), E / (32 * S_pack), E / (32 * S_lb), W, E / (32 * S_win));
    for (int b = 0; b <= 10; ++b)
        printf("  acc %3d%%: pairs %5.1f%%  steps %5.1f%%  util %.2f\n", 10 * b, 100 * hE[b] / E, 100 * hS[b] / S_cur,
               hS[b] ? hE[b] / (32 * hS[b]) : 0.0);
    printf("avg cnt %.1f, short blocks %.1f%%\n", sumCnt / blocks, 100 * partialCnt / blocks);
    printf("steps per cluster: current %.1f packed %.1f lb %.1f\n", S_cur / nclusters, S_pack / nclusters, S_lb / nclusters);
    for (int q = 0; q < NTH; ++q)
        printf("pool blocks with < %3d pairs: dense steps %.3f of current, pooled pairs %.3f of all -> cost (ovh 1.0/1.5/2.0) %.3f %.3f %.3f\n",
               TH[q], Sd[q] / S_cur, Ps[q] / E, (Sd[q] + Ps[q] / 32.0) / S_cur, (Sd[q] + 1.5 * Ps[q] / 32.0) / S_cur,
               (Sd[q] + 2.0 * Ps[q] / 32.0) / S_cur);
    for (int q = 0; q < NTH; ++q)
        printf("per-block batches, < %3d pairs: cost (ovh 1.2/1.5) %.3f %.3f  (pooled batches/cluster %.1f)\n", TH[q],
               (Sd[q] + 1.2 * Pb[q]) / S_cur, (Sd[q] + 1.5 * Pb[q]) / S_cur, Pb[q] / nclusters);
    for (int q = 0; q < NK; ++q)
        printf("steps with < %2d lanes pooled (per block): kept steps %.3f, pooled pairs %.3f -> cost (ovh 1.2/1.5) %.3f %.3f\n",
               KT[q], Sk[q] / S_cur, Pk[q] / E, (Sk[q] + 1.2 * Bk[q]) / S_cur, (Sk[q] + 1.5 * Bk[q]) / S_cur);
    for (int q = 0; q < NTH; ++q)
        printf("per-lane candidate steps (max lane degree), < %3d pairs: cost (ovh 1.0/1.1/1.2) %.3f %.3f %.3f\n", TH[q],
               (Sd[q] + Pl[q]) / S_cur, (Sd[q] + 1.1 * Pl[q]) / S_cur, (Sd[q] + 1.2 * Pl[q]) / S_cur);
}
