// Dependent-chain latency probe: DFMA, DMUL, DADD, MUFU rsqrt/rcp f64, LDS.64 (cycles per op).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chains(double* out, long long* cyc, double a, double b, int n) {
    __shared__ double sm[64];
    sm[threadIdx.x & 63] = (double)(threadIdx.x & 63);
    __syncthreads();
    double x = a, y = b;
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, y, 1e-300);
    t1 = clock64();
    cyc[0] = t1 - t0;
    // DMUL chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = x * y;
    t1 = clock64();
    cyc[1] = t1 - t0;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = x + y;
    t1 = clock64();
    cyc[2] = t1 - t0;
    // MUFU rsqrt f64 chain
    double r = a;
    t0 = clock64();
    for (int i = 0; i < n; ++i) asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(r));
    t1 = clock64();
    cyc[3] = t1 - t0;
    // MUFU rcp f64 chain
    double q = a;
    t0 = clock64();
    for (int i = 0; i < n; ++i) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(q));
    t1 = clock64();
    cyc[4] = t1 - t0;
    // LDS.64 chain (index from loaded value)
    int idx = threadIdx.x & 63;
    t0 = clock64();
    for (int i = 0; i < n; ++i) idx = ((int)sm[idx] + 1) & 63;
    t1 = clock64();
    cyc[5] = t1 - t0;
    out[threadIdx.x] = x + r + q + idx;
}

int main() {
    double* o;
    long long* c;
    cudaMalloc(&o, 1024 * 8);
    cudaMallocManaged(&c, 8 * 8);
    const int n = 4096;
    chains<<<1, 32>>>(o, c, 1.0000001, 0.9999999, n);
    cudaDeviceSynchronize();
    chains<<<1, 32>>>(o, c, 1.0000001, 0.9999999, n);
    cudaDeviceSynchronize();
    const char* nm[6] = {"DFMA", "DMUL", "DADD", "MUFU.RSQ64H", "MUFU.RCP64H", "LDS.64+F2I chain"};
    for (int k = 0; k < 6; ++k) printf("%-18s %.2f cycles/op\n", nm[k], (double)c[k] / n);
    return 0;
}
