// fp64 reduction of tile regions into a grid: per-element RED.E.ADD.F64
// (the spread flush) against TMA bulk reductions (cp.reduce.async.bulk
// .add.f64 = UBLKRED: one instruction per contiguous z line of the region,
// the adds done by the memory system). Regions of L x L rows of 24 doubles
// (L = 23, the c2 spread tile) at pseudo-random 8-aligned origins.
// Usage: bulkred [n] (grid edge, default 128; 204 = the xi = 60 grid)
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int L = 23, LZ = 24;

__device__ __forceinline__ void origin(long long w, int r, int n, int& x0, int& y0, int& z0) {
    unsigned h = (unsigned)(w * 2654435761u + r * 40503u);
    const int nt = (n - LZ) / 8;
    x0 = 8 * (h % nt);
    y0 = 8 * ((h >> 8) % nt);
    z0 = 8 * ((h >> 16) % nt);
}

__global__ void red_rows(double* g, int n, int reps) {
    const int lane = threadIdx.x & 31;
    const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    for (int r = 0; r < reps; ++r) {
        int x0, y0, z0;
        origin(w, r, n, x0, y0, z0);
        for (int row = 0; row < L * L; ++row) {
            const int a = row / L, b = row % L;
            if (lane < L) atomicAdd(g + ((long long)(x0 + a) * n + (y0 + b)) * n + z0 + lane, 1.0);
        }
    }
}

// 8 rows per pass staged in shared memory (the warp's row block), one bulk
// reduction per row issued by lanes 0..7
__global__ void bulk_rows(double* g, int n, int reps) {
    __shared__ __align__(128) double stage[8][8][LZ];  // [warp][row][z]
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    double(*st)[LZ] = stage[wl];
    for (int r = 0; r < reps; ++r) {
        int x0, y0, z0;
        origin(w, r, n, x0, y0, z0);
        for (int rb = 0; rb < (L * L + 7) / 8; ++rb) {
            for (int e = lane; e < 8 * LZ; e += 32) st[e / LZ][e % LZ] = (e % LZ) < L ? 1.0 : 0.0;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            const int row = rb * 8 + lane;
            if (lane < 8 && row < L * L) {
                const int a = row / L, b = row % L;
                double* dst = g + ((long long)(x0 + a) * n + (y0 + b)) * n + z0;
                const uint32_t sa = (uint32_t)__cvta_generic_to_shared(st[lane]);
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;"
                             :: "l"(dst), "r"(sa), "r"(LZ * 8) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            __syncwarp();
        }
    }
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 128;
    double* g;
    const size_t cells = (size_t)n * n * n;
    cudaMalloc(&g, sizeof(double) * cells);
    cudaMemset(g, 0, sizeof(double) * cells);
    const int blocks = 148 * 4, threads = 256, reps = 4;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    const double vals = (double)blocks * (threads / 32) * reps * L * L * L;
    for (int v = 0; v < 2; ++v) {
        auto run = [&](int rp) {
            if (v == 0) red_rows<<<blocks, threads>>>(g, n, rp);
            else bulk_rows<<<blocks, threads>>>(g, n, rp);
        };
        run(1);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        run(reps);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("n=%d %s: %.3e values in %.3f ms = %.1f G values/s  (%s)\n", n, v ? "UBLKRED rows" : "RED.F64", vals,
               ms, vals / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    // check: both kernels add 1.0 per region element; total = 2 * (1 + reps) * vals / reps ... compare sums
    double* h = (double*)malloc(sizeof(double) * cells);
    cudaMemcpy(h, g, sizeof(double) * cells, cudaMemcpyDeviceToHost);
    double s = 0;
    for (size_t i = 0; i < cells; ++i) s += h[i];
    printf("sum %.6e expected %.6e\n", s, 2.0 * vals * (1 + reps) / reps);
    return 0;
}
