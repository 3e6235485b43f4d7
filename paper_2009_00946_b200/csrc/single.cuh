// Single-CTA whole-layer transforms (one CTA per (layer, instance), up to
// 1024 threads, the layer resident in one SM's shared memory).  Used by the
// DWT micro-benchmark to compare against the cluster-distributed transform.
#pragma once

#include "cluster.cuh"

namespace fewha_gpu {

template <typename T, int FLEN>
__global__ void __launch_bounds__(1024, 1) k_dwt_single(const GeoParams gp, const T* __restrict__ in,
                                                        T* __restrict__ out, int inverse) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* buf = reinterpret_cast<T*>(smem_raw);
    const int l = blockIdx.x, b = blockIdx.y;
    const int side = gp.side[l], P = side + 1, lsd = ilog2(side), ne = side * side;
    const size_t base = static_cast<size_t>(b) * gp.n + gp.coff[l];
    const int tid = threadIdx.x, nthr = blockDim.x;
    for (int e = tid; e < ne; e += nthr) buf[(e >> lsd) * P + (e & (side - 1))] = in[base + e];
    __syncthreads();
    if (inverse) {
        for (int s = 2; s <= side; s <<= 1) {
            synthesis_lines<T, FLEN, true>(buf, P, s, s, gp);
            synthesis_lines<T, FLEN, false>(buf, P, s, s, gp);
        }
    } else {
        for (int s = side; s >= 2; s >>= 1) {
            analysis_lines<T, FLEN, false>(buf, P, s, s, gp);
            analysis_lines<T, FLEN, true>(buf, P, s, s, gp);
        }
    }
    for (int e = tid; e < ne; e += nthr) out[base + e] = buf[(e >> lsd) * P + (e & (side - 1))];
}

}  // namespace fewha_gpu
