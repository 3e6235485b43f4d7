// Microbenchmark (profiling aid): shared-memory load throughput per SM (cycles per
// warp-level load instruction) for 64-bit loads: consecutive, broadcast, 4-way conflict.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, long long* cyc, int n) {
    __shared__ double buf[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int idx;
    if (MODE == 0) idx = lane;                      // consecutive
    else if (MODE == 1) idx = 0;                    // broadcast
    else if (MODE == 2) idx = (lane & 7) + 32 * (lane >> 3);  // 4-way conflict
    else idx = 2 * lane;                            // 128-bit consecutive (below)
    idx += 64 * w;
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < n; ++it) {
        const int o = (it & 7) * 256;
        if (MODE == 3) {
            const double2 v0 = *reinterpret_cast<const double2*>(buf + idx + o);
            const double2 v1 = *reinterpret_cast<const double2*>(buf + idx + o + 512);
            a0 += v0.x; a1 += v0.y; a2 += v1.x; a3 += v1.y;
        } else {
            a0 += buf[idx + o]; a1 += buf[idx + o + 512]; a2 += buf[idx + o + 1024]; a3 += buf[idx + o + 1536];
        }
    }
    __syncthreads();
    long long t1 = clock64();
    out[threadIdx.x] = a0 + a1 + a2 + a3;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double* d; long long* c; long long h;
    cudaMalloc(&d, 8 * 1024); cudaMalloc(&c, 8);
    const int n = 2048;
    for (int rep = 0; rep < 2; ++rep)
        for (int thr : {256, 512}) {
            const char* names[4] = {"consecutive LDS.64", "broadcast LDS.64", "4-way conflict LDS.64", "consecutive LDS.128"};
            for (int m = 0; m < 4; ++m) {
                if (m == 0) k<0><<<1, thr>>>(d, c, n);
                if (m == 1) k<1><<<1, thr>>>(d, c, n);
                if (m == 2) k<2><<<1, thr>>>(d, c, n);
                if (m == 3) k<3><<<1, thr>>>(d, c, n);
                cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
                const double winst = double(thr / 32) * n * (m == 3 ? 2 : 4);
                if (rep) printf("%3d threads %-24s: %.2f cycles per warp load instruction (SM)\n", thr, names[m], h / winst);
            }
        }
    return 0;
}
