// Multi-GPU context of the C-ABI (sewald_gpu_multi_*): one process drives
// several GPUs of one node, so C / C++ callers of the drop-in
// (full_potential, realspace.h:46-47) scale without MPI or torch.
//
// One device context (stream, cached session: sorted sources, cell list,
// cuFFT plans) per GPU. A call:
//   1. every device uploads the inputs (the real-space sum needs every
//      source) and spreads its 1/W slice of the sources into its own grid;
//   2. the W grids are summed over NVLink peer memory: device d adds slab d
//      of every grid (reduce-scatter kernel reading the peers' buffers), then
//      copies the other W-1 reduced slabs from their owners (all-gather);
//   3. every device solves the (replicated, cheap at D = 3) k-space part and
//      evaluates its 1/W of the cell-ordered targets (real space + gather +
//      terms), exactly as Session.evaluate(part, nparts);
//   4. device 0 sums the W partial velocities (peer reads) and copies the
//      result to the caller.
// Cross-device ordering uses CUDA events; host threads (one per device)
// issue each device's work so the pageable uploads overlap.
//
// Several entries of dev_ids may name the same physical GPU (tests on a
// one-GPU box): those contexts share the device and their buffers are read
// directly.
#include "engine.h"

#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

using namespace sewald_b200;

struct sewald_gpu_multi {
    std::vector<int> dev;
    std::vector<sewald_gpu_ctx*> ctx;
    std::vector<cudaEvent_t> ev_spread, ev_rs, ev_ag, ev_eval;
    std::vector<std::unique_ptr<DevBuf>> u_part;     // per device: its partial velocity
    std::vector<std::unique_ptr<DevBuf>> ptr_table;  // per device: device copy of the peers' buffer pointers
    std::string err;
};

namespace sewald_b200 {
namespace {

constexpr int MR_THREADS = 256;

// dst[i] = sum_q src[q][i] for i in [i0, i1) (the reduce-scatter slab of
// this device); src[self] may alias dst.
__global__ void __launch_bounds__(MR_THREADS)
slab_sum_kernel(double* __restrict__ dst, const double* const* __restrict__ src, int nsrc, int64_t i0, int64_t i1) {
    for (int64_t i = i0 + blockIdx.x * (int64_t)MR_THREADS + threadIdx.x; i < i1;
         i += (int64_t)gridDim.x * MR_THREADS) {
        double acc = 0.0;
        for (int q = 0; q < nsrc; ++q) acc += src[q][i];
        dst[i] = acc;
    }
}

// dst[i] = src[i] for i in [i0, i1) (all-gather of one peer's slab).
__global__ void __launch_bounds__(MR_THREADS)
slab_copy_kernel(double* __restrict__ dst, const double* __restrict__ src, int64_t i0, int64_t i1) {
    for (int64_t i = i0 + blockIdx.x * (int64_t)MR_THREADS + threadIdx.x; i < i1;
         i += (int64_t)gridDim.x * MR_THREADS)
        dst[i] = src[i];
}

unsigned blocks_for(int64_t n) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + MR_THREADS - 1) / MR_THREADS, 148 * 8));
}

template <class F>
int multi_guard(sewald_gpu_multi* m, F&& fn) {
    try {
        fn();
        return SEWALD_OK;
    } catch (const EngineError& e) {
        m->err = e.what();
        return e.code;
    } catch (const std::invalid_argument& e) {
        m->err = e.what();
        return SEWALD_EINVAL;
    } catch (const std::domain_error& e) {
        m->err = e.what();
        return SEWALD_EDOMAIN;
    } catch (const std::exception& e) {
        m->err = e.what();
        return SEWALD_ERUNTIME;
    }
}

// Run fn(d) on one host thread per device; the first exception (lowest
// device index) is rethrown after all threads joined.
template <class F>
void per_device(sewald_gpu_multi* m, F&& fn) {
    const int W = (int)m->ctx.size();
    std::vector<std::exception_ptr> errs(W);
    std::vector<std::thread> th;
    for (int d = 0; d < W; ++d)
        th.emplace_back([&, d] {
            try {
                cuda_check(cudaSetDevice(m->dev[d]), "cudaSetDevice");
                fn(d);
            } catch (...) {
                errs[d] = std::current_exception();
            }
        });
    for (auto& t : th) t.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

void multi_pipeline(sewald_gpu_multi* m, const sewald_params_c* p, const double* x, const double* f,
                    const double* nu, int64_t N, const double* xt, int64_t Nt, int same, int use_table, int parts,
                    double* u_out) {
    if (!p) throw EngineError(SEWALD_EINVAL, "null parameters");
    if (N < 0 || Nt < 0) throw EngineError(SEWALD_EINVAL, "negative sizes");
    if (same && Nt != N && Nt != 0 && xt) throw EngineError(SEWALD_EINVAL, "starred evaluation needs one target per source");
    const int W = (int)m->ctx.size();
    std::vector<sewald_gpu_session*> S(W, nullptr);
    std::vector<double*> grid(W, nullptr), upart(W, nullptr);
    const int64_t nt = same ? N : Nt;
    // 1. upload + spread of this device's source slice
    per_device(m, [&](int d) {
        sewald_gpu_session* s = cached_session(m->ctx[d], *p);
        S[d] = s;
        session_set_targets(s, xt, Nt, same != 0);
        session_set_sources(s, x, f, nu, N);
        if (!same) session_set_targets(s, xt, Nt, false);
        upart[d] = static_cast<double*>(m->u_part[d]->ensure(sizeof(double) * 3 * std::max<int64_t>(nt, 1)));
        if (parts & 1) {
            const int64_t vol = (int64_t)s->g.n[0] * s->g.n[1] * s->g.n[2];
            grid[d] = static_cast<double*>(s->grid.ensure(sizeof(double) * s->C * vol));
            session_spread(s, N * d / W, N * (d + 1) / W, grid[d]);
        }
        cuda_check(cudaEventRecord(m->ev_spread[d], s->ctx->stream), "event");
    });
    // 2. grid all-reduce over peer memory (reduce-scatter, then all-gather)
    if ((parts & 1) && W > 1) {
        const int64_t len = (int64_t)S[0]->C * S[0]->g.n[0] * S[0]->g.n[1] * S[0]->g.n[2];
        per_device(m, [&](int d) {
            cudaStream_t st = S[d]->ctx->stream;
            for (int q = 0; q < W; ++q) cuda_check(cudaStreamWaitEvent(st, m->ev_spread[q], 0), "wait spread");
            // (a pageable H2D copy returns once the source is staged: h may go)
            const double** tab = static_cast<const double**>(m->ptr_table[d]->ensure(sizeof(double*) * W));
            std::vector<const double*> h(grid.begin(), grid.end());
            cuda_check(cudaMemcpyAsync(tab, h.data(), sizeof(double*) * W, cudaMemcpyHostToDevice, st), "ptr table");
            const int64_t i0 = len * d / W, i1 = len * (d + 1) / W;
            if (i1 > i0) slab_sum_kernel<<<blocks_for(i1 - i0), MR_THREADS, 0, st>>>(grid[d], tab, W, i0, i1);
            cuda_check(cudaGetLastError(), "slab sum");
            cuda_check(cudaEventRecord(m->ev_rs[d], st), "event");
        });
        per_device(m, [&](int d) {
            cudaStream_t st = S[d]->ctx->stream;
            for (int q = 0; q < W; ++q) {
                if (q == d) continue;
                cuda_check(cudaStreamWaitEvent(st, m->ev_rs[q], 0), "wait reduce");
                const int64_t i0 = len * q / W, i1 = len * (q + 1) / W;
                if (i1 > i0) slab_copy_kernel<<<blocks_for(i1 - i0), MR_THREADS, 0, st>>>(grid[d], grid[q], i0, i1);
            }
            cuda_check(cudaGetLastError(), "slab gather");
            cuda_check(cudaEventRecord(m->ev_ag[d], st), "event");
        });
    }
    // 3. solve + this device's part of the targets
    per_device(m, [&](int d) {
        sewald_gpu_session* s = S[d];
        // the transforms may reuse the grid buffer: every peer's reads of it are done first
        if ((parts & 1) && W > 1)
            for (int q = 0; q < W; ++q) cuda_check(cudaStreamWaitEvent(s->ctx->stream, m->ev_ag[q], 0), "wait gather");
        if (parts & 1) session_solve(s, grid[d], use_table != 0);
        if (nt > 0) {
            if (parts & 1) session_check_target_box(s);
            session_evaluate(s, d, W, parts, upart[d]);
        }
        session_read_singular(s);
        cuda_check(cudaEventRecord(m->ev_eval[d], s->ctx->stream), "event");
    });
    // 4. sum of the partial velocities on device 0, copy out
    per_device(m, [&](int d) {
        if (d != 0) {
            cuda_check(cudaStreamSynchronize(S[d]->ctx->stream), "evaluate sync");
            session_finish_singular(S[d]);
            return;
        }
        cudaStream_t st = S[0]->ctx->stream;
        for (int q = 0; q < W; ++q) cuda_check(cudaStreamWaitEvent(st, m->ev_eval[q], 0), "wait evaluate");
        if (nt > 0) {
            if (W > 1) {
                const double** tab = static_cast<const double**>(m->ptr_table[0]->ensure(sizeof(double*) * W));
                std::vector<const double*> h(upart.begin(), upart.end());
                cuda_check(cudaMemcpyAsync(tab, h.data(), sizeof(double*) * W, cudaMemcpyHostToDevice, st), "ptr table");
                slab_sum_kernel<<<blocks_for(3 * nt), MR_THREADS, 0, st>>>(upart[0], tab, W, 0, 3 * nt);
                cuda_check(cudaGetLastError(), "velocity sum");
            }
            cuda_check(cudaMemcpyAsync(u_out, upart[0], sizeof(double) * 3 * nt, cudaMemcpyDefault, st), "u copy");
        }
        cuda_check(cudaStreamSynchronize(st), "pipeline sync");
        session_finish_singular(S[0]);
    });
}

}  // namespace
}  // namespace sewald_b200

extern "C" {

int sewald_gpu_multi_create(int n_gpus, const int* dev_ids, sewald_gpu_multi** out) {
    if (!out || n_gpus < 1) return SEWALD_EINVAL;
    *out = nullptr;
    auto m = std::make_unique<sewald_gpu_multi>();
    for (int d = 0; d < n_gpus; ++d) m->dev.push_back(dev_ids ? dev_ids[d] : d);
    for (int d = 0; d < n_gpus; ++d) {
        sewald_gpu_ctx* c = nullptr;
        const int rc = sewald_gpu_create(m->dev[d], &c);
        if (rc != SEWALD_OK) {
            for (auto* x : m->ctx) sewald_gpu_destroy(x);
            return rc;
        }
        m->ctx.push_back(c);
    }
    // peer access between distinct physical devices (NVLink / NVSwitch)
    for (int a = 0; a < n_gpus; ++a)
        for (int b = 0; b < n_gpus; ++b) {
            if (m->dev[a] == m->dev[b]) continue;
            int ok = 0;
            cudaDeviceCanAccessPeer(&ok, m->dev[a], m->dev[b]);
            if (!ok) {
                for (auto* x : m->ctx) sewald_gpu_destroy(x);
                return SEWALD_ECUDA;
            }
            cudaSetDevice(m->dev[a]);
            const cudaError_t e = cudaDeviceEnablePeerAccess(m->dev[b], 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
                for (auto* x : m->ctx) sewald_gpu_destroy(x);
                return SEWALD_ECUDA;
            }
            cudaGetLastError();
        }
    m->ev_spread.resize(n_gpus);
    m->ev_rs.resize(n_gpus);
    m->ev_ag.resize(n_gpus);
    m->ev_eval.resize(n_gpus);
    for (int d = 0; d < n_gpus; ++d) {
        cudaSetDevice(m->dev[d]);
        cudaEventCreateWithFlags(&m->ev_spread[d], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&m->ev_rs[d], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&m->ev_ag[d], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&m->ev_eval[d], cudaEventDisableTiming);
    }
    for (int d = 0; d < n_gpus; ++d) {
        m->u_part.emplace_back(new DevBuf());
        m->ptr_table.emplace_back(new DevBuf());
    }
    *out = m.release();
    return SEWALD_OK;
}

void sewald_gpu_multi_destroy(sewald_gpu_multi* m) {
    if (!m) return;
    for (size_t d = 0; d < m->ctx.size(); ++d) {
        cudaSetDevice(m->dev[d]);
        cudaDeviceSynchronize();
        m->u_part[d].reset();  // freed with its device current
        m->ptr_table[d].reset();
        cudaEventDestroy(m->ev_spread[d]);
        cudaEventDestroy(m->ev_rs[d]);
        cudaEventDestroy(m->ev_ag[d]);
        cudaEventDestroy(m->ev_eval[d]);
    }
    for (auto* c : m->ctx) sewald_gpu_destroy(c);
    delete m;
}

const char* sewald_gpu_multi_last_error(const sewald_gpu_multi* m) { return m ? m->err.c_str() : "null context"; }

int sewald_gpu_multi_size(const sewald_gpu_multi* m) { return m ? (int)m->ctx.size() : 0; }

sewald_gpu_ctx* sewald_gpu_multi_context(sewald_gpu_multi* m, int d) {
    return (m && d >= 0 && d < (int)m->ctx.size()) ? m->ctx[d] : nullptr;
}

int sewald_gpu_multi_full_potential(sewald_gpu_multi* m, const sewald_params_c* p, const double* x,
                                    const double* f, const double* nu, int64_t N, const double* xt, int64_t Nt,
                                    int same_as_sources, int precompute_0p, double* u_out) {
    if (!m) return SEWALD_EINVAL;
    return multi_guard(m, [&] { multi_pipeline(m, p, x, f, nu, N, xt, Nt, same_as_sources, precompute_0p, 7, u_out); });
}

int sewald_gpu_multi_fourier_potential(sewald_gpu_multi* m, const sewald_params_c* p, const double* x,
                                       const double* f, const double* nu, int64_t N, const double* xt, int64_t Nt,
                                       int same_as_sources, int precompute_0p, double* u_out) {
    if (!m) return SEWALD_EINVAL;
    return multi_guard(m, [&] { multi_pipeline(m, p, x, f, nu, N, xt, Nt, same_as_sources, precompute_0p, 1, u_out); });
}

}  // extern "C"
