// Microbenchmark (profiling aid): cost of a cluster barrier (8 CTAs x 256 threads),
// alone and right after 64 KB of outstanding global stores.
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cl_arrive_relaxed() { asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
template <int MODE>
__global__ void __cluster_dims__(8, 1, 1) k(double* g, long long* cyc, int reps) {
    const int tid = threadIdx.x;
    cl_arrive(); cl_wait();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if (MODE == 1) {  // 64 KB of global stores per CTA before the barrier
            double* p = g + (size_t(blockIdx.x) * reps + r) * 8192;
            for (int e = tid; e < 8192; e += blockDim.x) p[e] = e;
        }
        if (MODE == 2) cl_arrive_relaxed(); else cl_arrive();
        cl_wait();
    }
    long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
}
int main() {
    double* g; long long* c; long long h[72];
    const int reps = 16;
    cudaMalloc(&g, size_t(72) * reps * 8192 * 8); cudaMalloc(&c, 72 * 8);
    for (int rep = 0; rep < 2; ++rep)
        for (int m = 0; m < 3; ++m) {
            if (m == 0) k<0><<<72, 256>>>(g, c, reps);
            if (m == 1) k<1><<<72, 256>>>(g, c, reps);
            if (m == 2) k<2><<<72, 256>>>(g, c, reps);
            cudaMemcpy(h, c, 72 * 8, cudaMemcpyDeviceToHost);
            long long s = 0; for (int i = 0; i < 72; ++i) s += h[i];
            if (rep) printf("mode %d (%s): %lld cycles per iteration\n", m,
                            m == 0 ? "release barrier" : m == 1 ? "64 KB stores + release barrier" : "relaxed barrier", s / 72);
        }
    return 0;
}
