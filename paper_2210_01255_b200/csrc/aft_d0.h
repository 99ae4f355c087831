// D = 0 Fourier solve with real, pruned transforms (aft_d0.cu), whole box on
// one GPU or slab-distributed over `world` ranks.
#pragma once

#include "engine.h"

#include <cufft.h>

#include <cstdint>
#include <vector>

namespace sewald_b200 {

struct ModSpec;

// Wavenumber / window-transform tables of the padded box and the combined
// normalisation; sizes and strides are filled in by the solve.
struct D0ScaleArgs {
    int n0, n1, n2, h2;
    int64_t cstride;
    const double *k0, *k1, *k2, *w0, *w1, *w2;
    double norm;
    int kz0;  // first kz of the slab (slab-distributed solve), 0 otherwise
};

// Balanced split points (world + 1 of them) of one axis over the ranks.
constexpr int kMaxWorld = 64;
struct SlabBounds {
    int world;
    int b[kMaxWorld + 1];
};

// Per-rank buffers and plans of the slab-distributed solve.
struct D0SlabPlan {
    int nxs = -1, nk = -1;
    std::vector<cufftHandle> plans;
    cufftHandle pz_f = 0, pz_i = 0, pxy_f = 0, pxy_i = 0;
    DevBuf R, Z, Tin, Tout, work;
    ~D0SlabPlan();
};

struct D0Real {
    int m[3]{}, n[3]{}, C = 3, h2 = 0;
    std::vector<cufftHandle> plans;
    cufftHandle pz_f = 0, pz_i = 0, pxy_f = 0, pxy_i = 0;
    // fused y path (n1 a power of two, 256..1024): x passes over the m1 data rows
    // only, y transform + scale + inverse y transform in one kernel per column set
    bool yfused = false;
    cufftHandle px_f = 0, px_i = 0;
    DevBuf R, Z, Tin, Tout, Th, work, tw;
    D0SlabPlan slab;
    ~D0Real();
    // m: input/output box (M_ext), n: padded transform box
    void setup(const int m[3], const int n[3], int C, cudaStream_t st);
    // Hermitian part of the full [n0][n1][n2] kernel table, half-spectrum layout
    void build_herm_table(const cuDoubleComplex* full, cudaStream_t st);
    // grid (C comps, M_ext) -> flow (3 comps, M_ext); returns own kernel launches
    int solve(const double* grid, const ModSpec& spec, int kind, double xi, const D0ScaleArgs& sa, bool table,
              double* flow, cudaStream_t st);

    // ---- slab-distributed stages (rank owns x in [xa, xb), kz in [ka, kb)) ----
    // grid slab [C][xb-xa][m1][m2] -> all-to-all send buffer, chunk q =
    // [C][xb-xa][m1][kz in slab q] (C (xb-xa) m1 (kz_q1 - kz_q0) complex)
    int slab_forward(const double* grid_slab, int xa, int xb, const SlabBounds& kzb, cuDoubleComplex* send,
                     cudaStream_t st);
    // received chunks p = [C][x in slab p][m1][kb-ka] -> 2-D transforms, scale,
    // inverse -> send buffer, chunk q = [3][kb-ka][x in slab q][m1]
    int slab_middle(const cuDoubleComplex* recv, const SlabBounds& xbd, int ka, int kb, const ModSpec& spec,
                    int kind, double xi, const D0ScaleArgs& sa, bool table, cuDoubleComplex* send,
                    cudaStream_t st);
    // received chunks p = [3][kz in slab p][xb-xa][m1] -> flow slab [3][xb-xa][m1][m2]
    int slab_inverse(const cuDoubleComplex* recv, int xa, int xb, const SlabBounds& kzb, double* flow_slab,
                     cudaStream_t st);

  private:
    void slab_plans(int nxs, int nk, cudaStream_t st);
};

}  // namespace sewald_b200
