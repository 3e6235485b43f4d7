// Microbenchmark (profiling aid): fp64 FMA latency / throughput and shared-memory
// load latency on one SM, in SM cycles (clock64).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma_chain(double* out, long long* cyc, int n) {
    double a = threadIdx.x * 1e-3, b = 1.0000001, c = 1e-9;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { a = fma(a, b, c); }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_dfma_tput(double* out, long long* cyc, int n) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 1.0000001, c = 1e-9;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
        a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
    __syncthreads();
    long long t1 = clock64();
    out[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_ffma_tput(float* out, long long* cyc, int n) {
    float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const float b = 1.0000001f, c = 1e-9f;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
        a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
    }
    __syncthreads();
    long long t1 = clock64();
    out[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_lds_chain(double* out, long long* cyc, int n) {
    __shared__ int idx[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i + 33) & 1023;
    __syncthreads();
    int p = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) p = idx[p];
    long long t1 = clock64();
    out[threadIdx.x] = p;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double* d; float* f; long long* c; long long h;
    cudaMalloc(&d, 8192); cudaMalloc(&f, 8192); cudaMalloc(&c, 8);
    const int n = 4096;
    for (int rep = 0; rep < 2; ++rep) {
        k_dfma_chain<<<1, 32>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("DFMA dependent chain: %.2f cycles/FMA\n", double(h) / n);
        for (int thr : {32, 128, 256, 512, 1024}) {
            k_dfma_tput<<<1, thr>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            if (rep) printf("DFMA throughput, %4d threads: %.1f FMA/clk/SM\n", thr, double(thr) * 8 * n / h);
            k_ffma_tput<<<1, thr>>>(f, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            if (rep) printf("FFMA throughput, %4d threads: %.1f FMA/clk/SM\n", thr, double(thr) * 8 * n / h);
        }
        k_lds_chain<<<1, 32>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("LDS dependent chain: %.2f cycles/load\n", double(h) / n);
    }
    return 0;
}
