// Device context and resident session of the B200 Spectral Ewald engine.
#pragma once

#include "../../include/sewald_gpu.h"
#include "device_common.cuh"
#include "sg_kernels.h"

#include <cufft.h>

#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace sewald_b200 {

// Error carrying a C-ABI status code.
struct EngineError : std::runtime_error {
    int code;
    EngineError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what);
void cufft_check(cufftResult r, const char* what);

// Grow-only device allocation.
struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    ~DevBuf();
    void* ensure(size_t n);
    template <class T> T* as() const { return static_cast<T*>(ptr); }
};

// Pinned host copy of the session's device status flags (one D2H per check).
struct HostFlags {
    int* p = nullptr;
    ~HostFlags();
    int* get();
};

// Grow-only pinned host buffer (staging of pageable caller buffers).
struct PinnedBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    ~PinnedBuf();
    void* ensure(size_t n);
};

struct FourierPlanD3;   // cuFFT plans + k tables for the fully periodic path
struct FourierPlanAFT;  // zero-padded / upsampled free-direction path (d < 3)
struct AftDeleter {
    void operator()(FourierPlanAFT* p) const;
};
struct D3Slab;  // slab-distributed D = 3 solve (aft.cu)
struct D3SlabDeleter {
    void operator()(D3Slab* p) const;
};

}  // namespace sewald_b200

struct sewald_gpu_ctx {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    std::string err;
    bool profiling = false;
    sewald_timings_c timings{};
    int64_t launches = 0;
    // host-buffer entry points reuse one session while the parameters match
    std::unique_ptr<sewald_gpu_session> cached;
    sewald_params_c cached_params{};
    // staging for host-buffer entry points
    sewald_b200::DevBuf hx, hf, hnu, hxt, hu;
    // pinned staging of pageable host inputs / output (parallel host copies)
    sewald_b200::PinnedBuf px, pf, pnu, pxt, pu;
    sewald_b200::PinnedBuf pout;  // sewald_gpu_host_buffer
};

struct sewald_gpu_session {
    sewald_gpu_ctx* ctx = nullptr;
    sewald_params_c p{};
    sewald_b200::DevGrid g{};
    sewald_b200::DevWindow w{};
    int C = 3;
    bool stresslet = false;

    // sources (original order, device copies)
    int64_t N = 0;
    sewald_b200::DevBuf x, f, nu;
    // spread bucketing for source range [sp_i0, sp_i1)
    int64_t sp_i0 = -1, sp_i1 = -1;
    sewald_b200::SpreadPlanShape shape{};
    sewald_b200::SweepShape sweep{};
    sewald_b200::DevBuf sp_keys, sp_keys2, sp_vals, sp_order, sp_off, cub_tmp, sp_w, sp_sw, sp_str;
    // real-space cell list
    sewald_b200::CellGrid cg{};
    bool cells_ready = false;
    sewald_b200::DevBuf s_folded, c_keys, c_keys2, c_vals, c_order, c_off, packed, packedf;
    // targets
    int64_t Nt = 0;
    bool same = false;
    sewald_b200::DevBuf xt, t_folded, t_keys, t_keys2, t_vals, t_order;
    // gather sweep ordering of the targets
    int sp_mode = 0;  // spread: 0 tile kernel, 1 z-sweep, 2 tensor-core tiles
    sewald_b200::SpreadMmaShape sm_shape{};
    bool tg_ready = false;
    int tg_mode = 0;  // 1: z-sweep gather, 2: tiled gather
    int tg_wpart = -1;  // part of the targets whose taps are current (0: all)
    int opt_epoch = 0;  // options_epoch() the orderings were built under
    sewald_b200::DevBuf tg_keys, tg_keys2, tg_vals, tg_order, tg_off, tg_w, tg_sw;
    // grids
    sewald_b200::DevBuf grid, flow;
    // global sums: f (3), q.nu (1), x (q.nu) (3); partials
    sewald_b200::DevBuf sums, partials, flags, pair_counter, work_counter, rs_scratch;
    sewald_b200::DevBuf fused_arg, fused_garg;  // argument blocks of the fused-taps spread / gather kernels
    sewald_b200::HostFlags hflags;
    bool inputs_checked = false;  // non-finite source / target flags read since the last upload
    bool sums_ready = false;
    std::unique_ptr<sewald_b200::FourierPlanD3> d3;
    std::unique_ptr<sewald_b200::FourierPlanAFT, sewald_b200::AftDeleter> aft;
    std::unique_ptr<sewald_b200::D3Slab, sewald_b200::D3SlabDeleter> slab3;
    // D = 0 kernel table supplied by the caller (SePipelineOptions::table,
    // fourier.h:76-79); used instead of building one when set
    sewald_b200::DevBuf user_table0p;
    bool has_user_table = false;
    const void* user_table_src = nullptr;  // caller's pointer and sampled-content fingerprint:
    uint64_t user_table_fp = 0;            // the re-upload is skipped only when both are unchanged
};

namespace sewald_b200 {

DevGrid make_dev_grid(const sewald_params_c& p);
DevWindow make_dev_window(const sewald_params_c& p);

void session_init(sewald_gpu_session* s, sewald_gpu_ctx* ctx, const sewald_params_c& p);
void session_set_sources(sewald_gpu_session* s, const double* x, const double* f, const double* nu,
                         int64_t N);
void session_set_targets(sewald_gpu_session* s, const double* xt, int64_t Nt, bool same);
void session_spread(sewald_gpu_session* s, int64_t i0, int64_t i1, double* grid);
void session_solve(sewald_gpu_session* s, const double* grid, bool precompute_0p);
void session_evaluate(sewald_gpu_session* s, int part, int nparts, int parts, double* u);
sewald_gpu_session* cached_session(sewald_gpu_ctx* ctx, const sewald_params_c& p);
void session_check_target_box(sewald_gpu_session* s);
void session_read_singular(sewald_gpu_session* s);
void session_finish_singular(sewald_gpu_session* s);

// Fourier solve for d < 3 (aft.cu): grid (C comps, real) -> s->flow (3 comps).
void aft_solve(sewald_gpu_session* s, const double* grid, bool precompute_0p);
// Reference stage functions on host buffers (aft.cu; fourier.cpp:311-803).
void stage_aft_forward(sewald_gpu_ctx* ctx, const sewald_params_c& p, const double* field,
                       const sewald_fourier_geom_c& g, double* far, double* near, double* zero);
void stage_aft_inverse(sewald_gpu_ctx* ctx, const sewald_params_c& p, const sewald_fourier_geom_c& g,
                       const int32_t* near_rows, const double* far, const double* near, const double* zero,
                       double* field_out);
void stage_scale(sewald_gpu_ctx* ctx, const sewald_params_c& p, int kind, const sewald_modspec_c* spec,
                 const int32_t* table_n, const double* table, double xi, const sewald_fourier_geom_c& g,
                 const int32_t* near_rows, const double* far, const double* near, const double* zero,
                 double* far_out, double* near_out, double* zero_out);
void stage_precompute_0p(sewald_gpu_ctx* ctx, const sewald_params_c& p, int kind, double R, int32_t n_out[3],
                         double* table_out);
int build_table_0p(const sewald_params_c& p, int kind, double R, DevBuf& out, cudaStream_t st);
// Install (table != nullptr) or clear a caller-built D = 0 table on the session.
void session_set_table0p(sewald_gpu_session* s, const int32_t n[3], const double* table);
// Slab-distributed D = 0 solve stages (aft.cu / aft_d0.cu).
struct SlabBounds;
void aft_d0_geometry(sewald_gpu_session* s, bool use_table, int m[3], int n[3], int* h2, int* C);
void aft_d0_slab_forward(sewald_gpu_session* s, bool use_table, const double* grid_slab, int xa, int xb,
                         const SlabBounds& kzb, void* send);
void aft_d0_slab_middle(sewald_gpu_session* s, bool use_table, const void* recv, const SlabBounds& xbd, int ka,
                        int kb, void* send);
void aft_d0_slab_inverse(sewald_gpu_session* s, bool use_table, const void* recv, int xa, int xb,
                         const SlabBounds& kzb, double* flow_slab);

}  // namespace sewald_b200
