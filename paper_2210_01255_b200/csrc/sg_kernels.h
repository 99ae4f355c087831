// Launch wrappers for the device kernels (spread_gather.cu, realspace.cu,
// kspace.cu). Host code includes this; the kernels themselves stay private
// to their translation units.
#pragma once

#include "device_common.cuh"

#include <cuComplex.h>

namespace sewald_b200 {

// ---- spread / gather (spread_gather.cu) ----------------------------------
struct SpreadPlanShape {
    int nb[3];     // buckets (= output tiles) per axis
    bool tiled;    // false -> atomic fallback for tiny periodic grids
};

SpreadPlanShape spread_plan_shape(const DevGrid& g, int P);
void launch_spread_bucket(const DevGrid& g, int P, const double* x, int64_t N,
                          const SpreadPlanShape& s, uint32_t* keys, uint32_t* vals, int* bad,
                          cudaStream_t st);
void launch_bucket_offsets(const uint32_t* keys, int64_t N, int nb, int64_t* off, cudaStream_t st,
                           int shift = 0);
void launch_spread_tiles(const DevGrid& g, const DevWindow& w, const double* x, const double* f,
                         const double* nu, int stresslet, const uint32_t* order,
                         const int64_t* off, const SpreadPlanShape& s, double* out,
                         cudaStream_t st);
void launch_spread_atomic(const DevGrid& g, const DevWindow& w, const double* x, const double* f,
                          const double* nu, int stresslet, int64_t N, double* out,
                          cudaStream_t st);
void launch_gather(const DevGrid& g, const DevWindow& w, const double* grid, const double* xt,
                   const uint32_t* order, int64_t Nt, double h3, int accumulate, double* u,
                   cudaStream_t st);
void launch_stencil_bounds(const DevGrid& g, int P, const double* x, int64_t N, int* bad,
                           cudaStream_t st);

// z-sweep spread (spread_sweep.cu): buckets = 4x8 (x,y) patches x z start.
// Tiled gather (gather_tile.cu): targets bucketed by the B^3 block of their
// stencil start; one CTA stages the L^3 region (L = B + P - 1) in shared memory.
struct TileShape {
    int B, L;
    int nt[3];
    int64_t ntiles;
    size_t smem;
    bool ok;
    double tpt;  // mean targets per tile
};
// Nt: number of targets (tile size choice for dense targets)
TileShape tile_shape(const DevGrid& g, int P, int64_t Nt = 0);
void launch_tile_bucket(const DevGrid& g, int P, const TileShape& s, const double* x, int64_t N, uint32_t* keys,
                        uint32_t* vals, int* bad, cudaStream_t st, int sub = 0);
void launch_gather_tile(const DevGrid& g, int P, const TileShape& s, const double* W, const int4* SW,
                        const int64_t* off, int part, int nparts, const double* grid, double h3, int accumulate,
                        double* u, cudaStream_t st);
// Register-A tensor-core gather tiles with the taps evaluated in the kernel
// (no taps array); arg_dev: fused_tgt_bytes() of device scratch.
bool gather_tile_fused_ok(const TileShape& s);
// the tiles run the register-A tensor-core kernel (gather_wide_mma_kernel)
bool gather_tile_regA(const TileShape& s);
size_t fused_tgt_bytes();
void launch_gather_tile_fused(const DevGrid& g, const DevWindow& w, int P, const TileShape& s, const double* xt,
                              const uint32_t* order, const int64_t* off, int part, int nparts, const double* grid,
                              double h3, int accumulate, double* u, void* arg_dev, cudaStream_t st);

// Tensor-core spread (spread_mma.cu): sources bucketed by the B^3 block of
// their stencil start, region L^3 (L = B + P - 1) per block as a DMMA GEMM.
struct SpreadMmaShape {
    int B, L;
    int nt[3];
    int64_t ntiles;
    bool ok;
    int sub;  // low key bits ordering a tile's points by their (x, y) stencil offset (0 or 6)
};
SpreadMmaShape spread_mma_shape(const DevGrid& g, int P);
void launch_spread_mma_bucket(const DevGrid& g, int P, const SpreadMmaShape& s, const double* x, int64_t N,
                              uint32_t* keys, uint32_t* vals, int* bad, cudaStream_t st);
int launch_spread_mma(const DevGrid& g, int P, const SpreadMmaShape& s, const double* W, const int4* SW,
                      const double* STR, int C, const int64_t* off, double* out, cudaStream_t st);
// Same tiles with the taps evaluated in the kernel (no taps array); fsrc_dev:
// fused_src_bytes() of device scratch for the kernel's argument block.
bool spread_mma_fused_ok(const SpreadMmaShape& s, int C);
size_t fused_src_bytes();
int launch_spread_mma_fused(const DevGrid& g, const DevWindow& w, int P, const SpreadMmaShape& s, const double* x,
                            const double* f, const double* nu, const uint32_t* order, int C, const int64_t* off,
                            double* out, void* fsrc_dev, cudaStream_t st);

struct SweepShape {
    int nbx, nby, nseg;
    int64_t nkeys;
    bool ok;
};
SweepShape sweep_shape(const DevGrid& g, int P);
void launch_sweep_bucket(const DevGrid& g, int P, const double* x, int64_t N, const SweepShape& s, uint32_t* keys,
                         uint32_t* vals, int* bad, cudaStream_t st);
// Per-point taps / starts / strengths in bucket-sorted order (W: N*3*P,
// SW: N int4, STR: N*C).
void launch_sweep_weights(const DevGrid& g, const DevWindow& w, const double* x, const double* f, const double* nu,
                          int stresslet, const uint32_t* order, int64_t N, double* W, int4* SW, double* STR,
                          cudaStream_t st, const int64_t* klo = nullptr, const int64_t* khi = nullptr);
// Returns the number of kernel launches issued.
int launch_spread_sweep(const DevGrid& g, int P, const double* W, const int4* SW, const double* STR, int C,
                        const int64_t* off, const SweepShape& s, double* out, cudaStream_t st);

// z-sweep gather (spread_sweep.cu): tiles [part/nparts] of the (x,y) patches;
// u must be initialised (contributions are added with fp64 RED).
void launch_gather_sweep(const DevGrid& g, int P, const double* W, const int4* SW, const int64_t* off,
                         const SweepShape& s, int part, int nparts, const double* grid, double h3, double* u,
                         cudaStream_t st);

// ---- real space (realspace.cu) -------------------------------------------
struct CellGrid {
    int d;
    int n[3];
    double w[3];        // cell widths
    double origin[3];   // lower corner (0 on periodic axes)
    double L[3];
    int sub;            // x sub-cell key bits: particles sorted by x within a cell row
};

struct RealspaceArgs {
    int kind;           // SEWALD_STOKESLET / STRESSLET / ROTLET
    double xi;
    double rc;
    double xi2, rc2;    // xi^2, rc^2 (host-computed; kernels read them as parameters)
    int skip_self;      // starred && targets are the sources
    float thresh_f;     // conservative fp32 bound on rc^2 for the candidate pass
};

void launch_fold_and_key(const CellGrid& cg, const double* x, int64_t N, double* folded,
                         uint32_t* keys, uint32_t* vals, cudaStream_t st);
// Packs sorted sources: pos(3) + original index + strengths (3, or q(3)+nu(3)),
// plus an fp32 position copy for the candidate pass.
void launch_pack_sources(const double* folded, const double* f, const double* nu, int stresslet,
                         const uint32_t* order, int64_t N, double* packed, float4* packedf,
                         cudaStream_t st);
// Non-symmetric real-space sum for targets torder[0..Nt). split > 1 (small
// target sets, realspace_split) needs scratch of split * Nt * 3 doubles: the
// row parts' sums are combined in a fixed order (deterministic results).
void launch_realspace(const CellGrid& cg, const RealspaceArgs& a, const double* packed,
                      const float4* packedf, int stresslet, const int64_t* cell_off, const double* tfolded,
                      const uint32_t* torder, int64_t Nt, double* u, int accumulate,
                      unsigned long long* pair_count, int* err, int split, double* scratch, cudaStream_t st);
int realspace_split(int64_t Nt);

// Symmetric real-space sum for targets == sources (realspace_sym.cu):
// i-clusters c0, c0 + cstride, ... < c1 of 32 cell-ordered particles; u
// (original order) must be zeroed beforehand and receives contributions of
// every particle.
void launch_realspace_sym(const CellGrid& cg, const RealspaceArgs& a, const double* packed, int64_t N,
                          const int64_t* cell_off, int64_t c0, int64_t c1, int64_t cstride, double* u,
                          unsigned long long* pair_count, int* err, unsigned long long* work, cudaStream_t st);

// ---- k space (kspace.cu) ---------------------------------------------------
struct KspaceTables {
    const double* k[3];      // wavenumbers per axis (DFT order)
    const double* what[3];   // window transforms per axis
};

// D=3 half spectrum: modes (i, j, m) with m in [0, n2/2]; in: C comps
// (stride cstride complex), out: 3 comps written over comps 0..2.
void launch_scale_periodic(int kind, int n0, int n1, int n2, double xi, double norm,
                           const KspaceTables& t, cuDoubleComplex* data, int64_t cstride,
                           cudaStream_t st);

}  // namespace sewald_b200
