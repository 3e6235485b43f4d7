// Microbenchmark (profiling aid): cost of __syncthreads and of the clock reads themselves.
#include <cstdio>
#include <cuda_runtime.h>
template <int NB>
__global__ void k(long long* cyc, int mode) {
    __syncthreads();
    long long t0, t1;
    if (mode == 0) {
        t0 = clock64();
#pragma unroll
        for (int i = 0; i < NB; ++i) __syncthreads();
        t1 = clock64();
    } else {
        unsigned a, b;
        asm volatile("mov.u32 %0, %%clock;" : "=r"(a));
#pragma unroll
        for (int i = 0; i < NB; ++i) __syncthreads();
        asm volatile("mov.u32 %0, %%clock;" : "=r"(b));
        t0 = a; t1 = b;
    }
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    long long* c; long long h;
    cudaMalloc(&c, 8 * 148);
    for (int rep = 0; rep < 2; ++rep)
        for (int thr : {32, 256, 512})
            for (int mode : {0, 1}) {
                k<0><<<1, thr>>>(c, mode); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); long long h0 = h;
                k<1><<<1, thr>>>(c, mode); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); long long h1 = h;
                k<8><<<1, thr>>>(c, mode); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); long long h8 = h;
                if (rep) printf("threads %3d clock%s: 0 barriers %lld, 1: %lld, 8: %lld cycles\n", thr, mode ? "32" : "64", h0, h1, h8);
            }
    return 0;
}
