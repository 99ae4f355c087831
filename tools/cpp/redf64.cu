// Throughput of fp64 global reductions (RED.E.ADD.F64) to a 50 MB array
// (the c2 grid) with the access pattern of a tile-region scatter.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void red_rows(double* g, int n, int reps, int L) {
    // each warp adds a 19 x 19 x 19 region (rows of 19 contiguous z values) at a pseudo-random origin
    const int lane = threadIdx.x & 31;
    const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    for (int r = 0; r < reps; ++r) {
        unsigned h = (unsigned)(w * 2654435761u + r * 40503u);
        const int x0 = h % (n - L), y0 = (h >> 8) % (n - L), z0 = (h >> 16) % (n - L);
        for (int row = 0; row < L * L; ++row) {
            const int a = row / L, b = row % L;
            if (lane < L) atomicAdd(g + ((long long)(x0 + a) * n + (y0 + b)) * n + z0 + lane, 1.0);
        }
    }
}

int main() {
    const int n = 128, L = 19;
    double* g;
    cudaMalloc(&g, sizeof(double) * n * n * n);
    cudaMemset(g, 0, sizeof(double) * n * n * n);
    const int blocks = 148 * 8, threads = 256, reps = 4;
    red_rows<<<blocks, threads>>>(g, n, 1, L);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    red_rows<<<blocks, threads>>>(g, n, reps, L);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * (threads / 32) * reps * L * L * L;
    printf("RED.F64: %.3e ops in %.3f ms = %.1f Gops/s\n", ops, ms, ops / (ms * 1e-3) / 1e9);
    return 0;
}
