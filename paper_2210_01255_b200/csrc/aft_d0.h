// D = 0 Fourier solve with real, pruned transforms (aft_d0.cu).
#pragma once

#include "engine.h"

#include <cufft.h>

#include <cstdint>
#include <vector>

namespace sewald_b200 {

struct ModSpec;

// Wavenumber / window-transform tables of the padded box and the combined
// normalisation; sizes and strides are filled in by D0Real::solve.
struct D0ScaleArgs {
    int n0, n1, n2, h2;
    int64_t cstride;
    const double *k0, *k1, *k2, *w0, *w1, *w2;
    double norm;
};

struct D0Real {
    int m[3]{}, n[3]{}, C = 3, h2 = 0;
    std::vector<cufftHandle> plans;
    cufftHandle pz_f = 0, pz_i = 0, pxy_f = 0, pxy_i = 0;
    DevBuf R, Z, Tin, Tout, Th, work;
    ~D0Real();
    // m: input/output box (M_ext), n: padded transform box
    void setup(const int m[3], const int n[3], int C, cudaStream_t st);
    // Hermitian part of the full [n0][n1][n2] kernel table, half-spectrum layout
    void build_herm_table(const cuDoubleComplex* full, cudaStream_t st);
    // grid (C comps, M_ext) -> flow (3 comps, M_ext); returns kernel launches
    int solve(const double* grid, const ModSpec& spec, int kind, double xi, const D0ScaleArgs& sa, bool table,
              double* flow, cudaStream_t st);
};

}  // namespace sewald_b200
