// Microbenchmark (profiling aid): moving N doubles from every CTA of an 8-CTA cluster
// into its right neighbour's shared memory, until the neighbour can use them:
//   0: cluster barrier + remote loads (ld.shared::cluster via mapped pointers)
//   1: st.async per element completing on the neighbour's mbarrier
//   2: cp.async.bulk shared::cta -> shared::cluster (one copy) on the neighbour's mbarrier
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ unsigned cl_map(const void* p, int rank) {
    unsigned r; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(su32(p)), "r"(rank)); return r;
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void wait_c(unsigned long long* m, unsigned ph) {
    asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(su32(m)), "r"(ph) : "memory");
}
template <int MODE>
__global__ void __cluster_dims__(8, 1, 1) k(long long* cyc, double* out, int n) {
    __shared__ __align__(16) double src[2048], dst[2048];
    __shared__ unsigned long long bar;
    cg::cluster_group cl = cg::this_cluster();
    const int q = cl.block_rank(), nb = (q + 1) & 7, tid = threadIdx.x;
    for (int e = tid; e < n; e += blockDim.x) src[e] = q * 10000 + e;
    if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
    cl_sync();
    long long t0 = clock64();
    if (MODE == 0) {
        cl_sync();
        const double* r = cl.map_shared_rank(src, (q + 7) & 7);
        for (int e = tid; e < n; e += blockDim.x) dst[e] = r[e];
        __syncthreads();
    } else if (MODE == 1) {
        const unsigned db = cl_map(dst, nb), bb = cl_map(&bar, nb);
        for (int e = tid; e < n; e += blockDim.x)
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(db + e * 8), "l"(__double_as_longlong(src[e])), "r"(bb) : "memory");
        if (tid == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&bar)), "r"(n * 8) : "memory");
        wait_c(&bar, 0);
    } else {
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                         ::"r"(cl_map(dst, nb)), "r"(su32(src)), "r"(n * 8), "r"(cl_map(&bar, nb)) : "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&bar)), "r"(n * 8) : "memory");
        }
        wait_c(&bar, 0);
    }
    long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
    double acc = 0; for (int e = tid; e < n; e += blockDim.x) acc += dst[e];
    out[blockIdx.x * 256 + tid] = acc;
    cl_sync();
}
int main() {
    long long* c; double* o; long long h[72];
    cudaMalloc(&c, 72 * 8); cudaMalloc(&o, 72 * 256 * 8);
    for (int rep = 0; rep < 2; ++rep)
        for (int n : {128, 1024, 2048})
            for (int m = 0; m < 3; ++m) {
                if (m == 0) k<0><<<72, 256>>>(c, o, n);
                if (m == 1) k<1><<<72, 256>>>(c, o, n);
                if (m == 2) k<2><<<72, 256>>>(c, o, n);
                cudaMemcpy(h, c, 72 * 8, cudaMemcpyDeviceToHost);
                long long s = 0, mx = 0; for (int i = 0; i < 72; ++i) { s += h[i]; mx = h[i] > mx ? h[i] : mx; }
                if (rep) printf("%5d doubles, mode %d (%s): mean %lld max %lld cycles\n", n, m,
                                m == 0 ? "barrier + remote loads" : m == 1 ? "st.async per element" : "bulk copy", s / 72, mx);
            }
    return 0;
}
