// One filter length of the cluster layer kernels (compiled with -DFEWHA_FLEN=N).
#include <cstdlib>

#include "cluster.cuh"
#include "frame.cuh"
#include "single.cuh"
#include "launch.hpp"

#ifndef FEWHA_FLEN
#error "compile with -DFEWHA_FLEN=<2|4|...|20>"
#endif

namespace fewha_gpu {

template <typename T, int FLEN>
cudaError_t launch_layer_cluster(bool inverse, const GeoParams& gp, const Bufs<T>& bf, int mode, int it, int count,
                                 cudaStream_t st, int gather, size_t smem) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(gp.ccl, gp.L, count);
    cfg.blockDim = dim3(256, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = gp.ccl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (griddepcontrol in the kernels)
    const char* pdl = std::getenv("FEWHA_PDL");
    attr[1].val.programmaticStreamSerializationAllowed = (pdl && pdl[0] == '1') ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    if (inverse) return cudaLaunchKernelEx(&cfg, k_inv_cluster<T, FLEN>, gp, bf, mode, it);
    return cudaLaunchKernelEx(&cfg, k_fwd_cluster<T, FLEN>, gp, bf, mode, it, gather);
}

// Opt in to the device maximum minus each kernel's static shared memory.
template <typename K>
static cudaError_t opt_in_max(K kernel, size_t maxopt) {
    cudaFuncAttributes fa{};
    cudaError_t e = cudaFuncGetAttributes(&fa, kernel);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(maxopt - fa.sharedSizeBytes));
}

template <typename T, int FLEN>
cudaError_t set_layer_cluster_attrs(size_t smem_inv, size_t smem_fwd) {
    cudaError_t e = opt_in_max(k_inv_cluster<T, FLEN>, smem_inv);
    if (e != cudaSuccess) return e;
    return opt_in_max(k_fwd_cluster<T, FLEN>, smem_fwd);
}

template <typename T, int FLEN>
static cudaLaunchConfig_t frame_cfg(const GeoParams& gp, size_t smem, cudaStream_t st, cudaLaunchAttribute* attr) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(gp.ccl, gp.L, 1);
    cfg.blockDim = dim3(256, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = gp.ccl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cfg;
}

// The opt-in persistent frame is instantiated for the presets' Daubechies-3
// filter only (FLEN 6); other orders report "does not fit" and use the graph.
template <typename T, int FLEN>
cudaError_t launch_frame_persistent(const GeoParams& gp, const Bufs<T>& bf, unsigned int* bar, cudaStream_t st,
                                    size_t smem) {
    if constexpr (FLEN != 6) return cudaErrorNotSupported;
    cudaError_t e = cudaMemsetAsync(bar, 0, sizeof(unsigned int), st);
    if (e != cudaSuccess) return e;
    cudaLaunchAttribute attr[2];
    cudaLaunchConfig_t cfg = frame_cfg<T, FLEN>(gp, smem, st, attr);
    if constexpr (FLEN == 6) return cudaLaunchKernelEx(&cfg, k_frame<T, FLEN>, gp, bf, bar);
    return cudaErrorNotSupported;
}

// The persistent frame needs every cluster co-resident (grid barrier): check
// the occupancy calculator before choosing it.
template <typename T, int FLEN>
cudaError_t frame_persistent_fits(const GeoParams& gp, size_t smem, int* ok) {
    *ok = 0;
    if constexpr (FLEN != 6) return cudaSuccess;
    else {
    int dev = 0, maxopt = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&maxopt, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    e = opt_in_max(k_frame<T, FLEN>, static_cast<size_t>(maxopt));
    if (e != cudaSuccess) return e;
    cudaLaunchAttribute attr[2];
    cudaLaunchConfig_t cfg = frame_cfg<T, FLEN>(gp, smem, nullptr, attr);
    cfg.numAttrs = 1;  // occupancy query: cluster dimension only
    int clusters = 0;
    e = cudaOccupancyMaxActiveClusters(&clusters, k_frame<T, FLEN>, &cfg);
    if (e != cudaSuccess) return e;
    *ok = clusters >= gp.L ? 1 : 0;
    return cudaSuccess;
    }
}

template <typename T, int FLEN>
cudaError_t launch_dwt_single(const GeoParams& gp, const T* in, T* out, int inverse, int count, int threads,
                              cudaStream_t st) {
    const size_t smem = static_cast<size_t>(gp.maxside) * (gp.maxside + 1) * sizeof(T);
    cudaError_t e = opt_in_max(k_dwt_single<T, FLEN>, 227 * 1024);
    if (e != cudaSuccess) return e;
    k_dwt_single<T, FLEN><<<dim3(gp.L, count), threads, smem, st>>>(gp, in, out, inverse);
    return cudaGetLastError();
}

#define FEWHA_INST(T)                                                                                          \
    template cudaError_t launch_layer_cluster<T, FEWHA_FLEN>(bool, const GeoParams&, const Bufs<T>&, int, int, int, \
                                                             cudaStream_t, int, size_t);                        \
    template cudaError_t set_layer_cluster_attrs<T, FEWHA_FLEN>(size_t, size_t);                                   \
    template cudaError_t launch_frame_persistent<T, FEWHA_FLEN>(const GeoParams&, const Bufs<T>&, unsigned int*,   \
                                                                cudaStream_t, size_t);                             \
    template cudaError_t frame_persistent_fits<T, FEWHA_FLEN>(const GeoParams&, size_t, int*);                     \
    template cudaError_t launch_dwt_single<T, FEWHA_FLEN>(const GeoParams&, const T*, T*, int, int, int, cudaStream_t);
FEWHA_INST(double)
FEWHA_INST(float)

}  // namespace fewha_gpu
