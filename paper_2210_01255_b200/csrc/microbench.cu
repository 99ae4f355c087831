// fp64 pipe peak microbenchmark (the roofline denominator for the fp64-bound
// kernels; MEASURED_PEAKS.json carries only HBM and bf16 numbers). Eight
// independent DFMA chains per thread, full-chip grid, CUDA-event timed.
#include "engine.h"

namespace {

__global__ void dfma_chain_kernel(double* out, int iters, double b, double c) {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-3, a2 = a0 + 2e-3, a3 = a0 + 3e-3;
    double a4 = a0 + 4e-3, a5 = a0 + 5e-3, a6 = a0 + 6e-3, a7 = a0 + 7e-3;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
    const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 123.456) out[0] = s;  // keep the chains live
}

}  // namespace

extern "C" int sewald_gpu_fp64_peak(sewald_gpu_ctx* ctx, double* tflops) {
    if (!ctx || !tflops) return SEWALD_EINVAL;
    try {
        using namespace sewald_b200;
        cuda_check(cudaSetDevice(ctx->device), "device");
        int sms = 0;
        cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device), "attr");
        double* out = nullptr;
        cuda_check(cudaMalloc(&out, 64), "malloc");
        const int blocks = sms * 8, threads = 256, iters = 2048;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        dfma_chain_kernel<<<blocks, threads, 0, ctx->stream>>>(out, 64, 0.999999, 1e-7);  // warm
        cudaEventRecord(e0, ctx->stream);
        dfma_chain_kernel<<<blocks, threads, 0, ctx->stream>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1, ctx->stream);
        cuda_check(cudaEventSynchronize(e1), "sync");
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFree(out);
        const double flops = 2.0 * 8.0 * 16.0 * (double)iters * blocks * threads;
        *tflops = flops / (ms * 1e-3) / 1e12;
        return SEWALD_OK;
    } catch (const sewald_b200::EngineError& e) {
        ctx->err = e.what();
        return e.code;
    }
}
