// cuFFT plan variants for the strided x pass of the D = 0 solve (timing probe).
#include <cufft.h>
#include <cufftXt.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <algorithm>

static float time_exec(cufftHandle h, cufftDoubleComplex* in, cufftDoubleComplex* out, int dir) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cufftExecZ2Z(h, in, out, dir);
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) cufftExecZ2Z(h, in, out, dir);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

int main() {
    const int n0 = 960, h2 = 257, n1 = 512;
    const long long lines = (long long)h2 * n1;
    const size_t bytes = sizeof(cufftDoubleComplex) * (size_t)n0 * lines;
    cufftDoubleComplex *x, *y;
    cudaMalloc(&x, bytes);
    cudaMalloc(&y, bytes);
    { std::vector<double> hst(2 * (size_t)n0 * 1024); for (size_t i = 0; i < hst.size(); ++i) hst[i] = (double)((i * 2654435761u) % 1000) / 1000.0; for (size_t off = 0; off < bytes; off += hst.size() * 8) cudaMemcpy((char*)x + off, hst.data(), std::min(hst.size() * 8, bytes - off), cudaMemcpyHostToDevice); }
    int n[1] = {n0};
    {
        cufftHandle h;
        cufftPlanMany(&h, 1, n, n, (int)lines, 1, n, (int)lines, 1, CUFFT_Z2Z, (int)lines);
        printf("planMany auto, out-of-place: %.3f ms\n", time_exec(h, x, y, CUFFT_FORWARD));
        printf("planMany auto, in-place:     %.3f ms\n", time_exec(h, y, y, CUFFT_INVERSE));
        cufftDestroy(h);
    }
    {
        cufftHandle h;
        cufftCreate(&h);
        cufftSetAutoAllocation(h, 0);
        long long nn[1] = {n0}, e[1] = {n0};
        size_t ws = 0;
        cufftMakePlanMany64(h, 1, nn, e, lines, 1, e, lines, 1, CUFFT_Z2Z, lines, &ws);
        void* w;
        cudaMalloc(&w, ws + 16);
        cufftSetWorkArea(h, w);
        printf("makePlanMany64 manual ws=%zu MB, out-of-place: %.3f ms\n", ws >> 20, time_exec(h, x, y, CUFFT_FORWARD));
        printf("makePlanMany64 manual, in-place: %.3f ms\n", time_exec(h, y, y, CUFFT_INVERSE));
        cufftDestroy(h);
        cudaFree(w);
    }
    {
        cufftHandle h;
        cufftCreate(&h);
        long long nn[1] = {n0}, e[1] = {n0};
        size_t ws = 0;
        cufftXtMakePlanMany(h, 1, nn, e, lines, 1, CUDA_C_64F, e, lines, 1, CUDA_C_64F, lines, &ws, CUDA_C_64F);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cufftXtExec(h, x, y, CUFFT_FORWARD);
        cudaEventRecord(a);
        for (int i = 0; i < 5; ++i) cufftXtExec(h, x, y, CUFFT_FORWARD);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("XtMakePlanMany out-of-place: %.3f ms\n", ms / 5);
        cufftDestroy(h);
    }
    {
        // base offsets
        cufftDoubleComplex *big;
        cudaMalloc(&big, bytes * 2 + (64 << 20));
        cudaMemset(big, 0, bytes * 2 + (64 << 20));
        cufftHandle h;
        cufftPlanMany(&h, 1, n, n, (int)lines, 1, n, (int)lines, 1, CUFFT_Z2Z, (int)lines);
        const size_t offs[] = {0, 4096, 65536, 1 << 20, 2 << 20, 3 << 20, 17 << 20};
        for (size_t o : offs) {
            cufftDoubleComplex* in = (cufftDoubleComplex*)((char*)big + o);
            cufftDoubleComplex* out = (cufftDoubleComplex*)((char*)big + bytes + o + (32 << 20));
            printf("offset %zu KB: %.3f ms\n", o >> 10, time_exec(h, in, out, CUFFT_FORWARD));
        }
        cufftDestroy(h);
        cudaFree(big);
    }
    {
        cufftHandle h;
        cufftPlanMany(&h, 1, n, n, (int)lines, 1, n, 1, n0, CUFFT_Z2Z, (int)lines);
        printf("in strided -> out contiguous: %.3f ms\n", time_exec(h, x, y, CUFFT_FORWARD));
        cufftDestroy(h);
        cufftPlanMany(&h, 1, n, n, 1, n0, n, (int)lines, 1, CUFFT_Z2Z, (int)lines);
        printf("in contiguous -> out strided: %.3f ms\n", time_exec(h, y, x, CUFFT_INVERSE));
        cufftDestroy(h);
    }
    {
        // contiguous layout: [lines][n0]
        cufftHandle h;
        cufftPlanMany(&h, 1, n, n, 1, n0, n, 1, n0, CUFFT_Z2Z, (int)lines);
        printf("contiguous batched: %.3f ms\n", time_exec(h, x, y, CUFFT_FORWARD));
        cufftDestroy(h);
    }
    {
        // two half batches (kz ranges) to check batch-size effects
        cufftHandle h;
        cufftPlanMany(&h, 1, n, n, (int)lines, 1, n, (int)lines, 1, CUFFT_Z2Z, (int)(lines / 2));
        float t = time_exec(h, x, y, CUFFT_FORWARD);
        printf("planMany half batch: %.3f ms (x2 = %.3f)\n", t, 2 * t);
        cufftDestroy(h);
    }
    return 0;
}
