// FP64 mma.sync (m8n8k4) throughput probe vs DFMA on B200.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
    double c0 = 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0, c5 = 0, c6 = 0, c7 = 0;
    for (int i = 0; i < iters; ++i) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c2), "+d"(c3) : "d"(a), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c4), "+d"(c5) : "d"(a), "d"(b));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c6), "+d"(c7) : "d"(a), "d"(b));
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7;
}

int main() {
    double* o;
    cudaMalloc(&o, sizeof(double) * 148 * 8 * 1024);
    const int iters = 20000;
    for (int warps = 4; warps <= 16; warps *= 2) {
        dim3 grid(148 * 4), block(32 * warps / 4);
        dmma_loop<<<grid, block>>>(o, 100);
        cudaDeviceSynchronize();
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        dmma_loop<<<grid, block>>>(o, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double mmas = (double)grid.x * (block.x / 32) * iters * 4;
        printf("warps/SM %d: %.2f TFLOP/s fp64 mma.sync (%.1f ms)\n", warps, mmas * 512 / (ms * 1e-3) / 1e12, ms);
    }
    return 0;
}
