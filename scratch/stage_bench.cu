// Micro-benchmark: staging N bytes from L2 into shared memory, one CTA per SM.
// Variants: 0 = one TMA bulk copy by thread 0, 1 = nseg bulk copies by nseg threads,
// 2 = cp.async 16B by all threads, 3 = ld.global.v4 + st.shared by all threads.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__global__ void k(const char* src, int bytes, int variant, int nseg, long long* cyc, int reps) {
    extern __shared__ __align__(16) char sm[];
    __shared__ unsigned long long mbar;
    const char* s = src + static_cast<size_t>(blockIdx.x) * bytes;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned phase = 0;
    long long best = 1LL << 60;
    for (int r = 0; r < reps; ++r) {
        __syncthreads();
        long long t0 = clock64();
        if (variant <= 1) {
            const int segs = variant == 0 ? 1 : nseg;
            const int sb = bytes / segs;
            if (threadIdx.x < segs) {
                asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(su(&mbar)), "r"(sb) : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        su(sm + threadIdx.x * sb)),
                    "l"(s + threadIdx.x * sb), "r"(sb), "r"(su(&mbar))
                    : "memory");
            }
            __syncthreads();
            if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&mbar)) : "memory");
            asm volatile(
                "{\n.reg .pred P;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(
                    su(&mbar)),
                "r"(phase)
                : "memory");
            phase ^= 1;
        } else if (variant == 2) {
            for (int o = threadIdx.x * 16; o < bytes; o += blockDim.x * 16)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(sm + o)), "l"(s + o));
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
            __syncthreads();
        } else {
            for (int o = threadIdx.x * 16; o < bytes; o += blockDim.x * 16)
                *reinterpret_cast<int4*>(sm + o) = __ldcg(reinterpret_cast<const int4*>(s + o));
            __syncthreads();
        }
        long long t1 = clock64();
        if (r > 0 && t1 - t0 < best) best = t1 - t0;
    }
    if (threadIdx.x == 0) cyc[blockIdx.x] = best;
}

int main() {
    const int ctas = 72;
    char* src;
    long long* cyc;
    const int maxb = 160 * 1024;
    cudaMalloc(&src, static_cast<size_t>(ctas) * maxb);
    cudaMemset(src, 1, static_cast<size_t>(ctas) * maxb);
    cudaMallocManaged(&cyc, ctas * sizeof(long long));
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, maxb);
    const int sizes[] = {4096, 16384, 32768, 65536, 98304, 131072, 163840 - 16};
    const char* names[] = {"bulk x1", "bulk xN", "cp.async16", "ldg.v4"};
    for (int v = 0; v < 4; ++v)
        for (int nseg : {1, 10, 40}) {
            if (v != 1 && nseg != 1) continue;
            if (v == 1 && nseg == 1) continue;
            for (int b : sizes) {
                int bb = (b / (16 * nseg)) * 16 * nseg;
                k<<<ctas, 256, maxb>>>(src, bb, v, nseg, cyc, 6);
                cudaDeviceSynchronize();
                long long mx = 0, sum = 0;
                for (int i = 0; i < ctas; ++i) {
                    mx = cyc[i] > mx ? cyc[i] : mx;
                    sum += cyc[i];
                }
                printf("%-10s nseg=%2d bytes=%7d  mean %7lld cyc  max %7lld cyc  (%.1f B/cyc)\n", names[v], nseg, bb,
                       sum / ctas, mx, static_cast<double>(bb) / (sum / ctas));
            }
        }
    cudaError_t e = cudaGetLastError();
    printf("err %s\n", cudaGetErrorString(e));
    return 0;
}
