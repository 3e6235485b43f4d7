// One filter length of the cluster layer kernels (compiled with -DFEWHA_FLEN=N).
#include <cstdlib>

#include "cluster.cuh"
#include "launch.hpp"
#include "layer_whole.cuh"

#ifndef FEWHA_FLEN
#error "compile with -DFEWHA_FLEN=<2|4|...|20>"
#endif

namespace fewha_gpu {

template <typename T, int FLEN>
cudaError_t launch_layer_cluster(bool inverse, const GeoParams& gp, const Bufs<T>& bf, int mode, int it, int count,
                                 cudaStream_t st, int fit_term, size_t smem) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(gp.ccl, gp.L, count);
    cfg.blockDim = dim3(kClThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = gp.ccl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (griddepcontrol in the kernels)
    const char* pdl = std::getenv("FEWHA_PDL");  // on unless FEWHA_PDL=0 (as engine.cu pdl_enabled)
    attr[1].val.programmaticStreamSerializationAllowed = (pdl && pdl[0] == '0') ? 0 : 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    if (inverse) return cudaLaunchKernelEx(&cfg, k_inv_cluster<T, FLEN>, gp, bf, mode, it);
    return cudaLaunchKernelEx(&cfg, k_fwd_cluster<T, FLEN>, gp, bf, mode, it, fit_term);
}

// Whole-layer kernels of batched plans (layer_whole.cuh): grid (L, count), no cluster.
template <typename T, int FLEN>
cudaError_t launch_layer_whole(bool inverse, const GeoParams& gp, const Bufs<T>& bf, int mode, int it, int count,
                               cudaStream_t st, int fit_term) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(gp.L, count, 1);
    cfg.blockDim = dim3(Wl<T>::threads, 1, 1);
    cfg.dynamicSmemBytes = whole_layer_smem(gp.maxside, static_cast<int>(sizeof(T)));
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    const char* pdl = std::getenv("FEWHA_PDL");
    attr[0].val.programmaticStreamSerializationAllowed = (pdl && pdl[0] == '0') ? 0 : 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (inverse) return cudaLaunchKernelEx(&cfg, k_inv_layer<T, FLEN>, gp, bf, mode, it);
    return cudaLaunchKernelEx(&cfg, k_fwd_layer<T, FLEN>, gp, bf, mode, it, fit_term);
}

// Fused whole-layer forward + inverse (k_fwd_inv_layer): grid (L, count), ticketed CTAs.
template <typename T, int FLEN>
cudaError_t launch_layer_whole_fused(const GeoParams& gp, const Bufs<T>& bf, int fmode, int fit, int imode, int iit,
                                     int count, cudaStream_t st, int fit_term, unsigned long long* ctr) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(gp.L, count, 1);
    cfg.blockDim = dim3(Wl<T>::threads, 1, 1);
    cfg.dynamicSmemBytes = whole_layer_smem(gp.maxside, static_cast<int>(sizeof(T)));
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    const char* pdl = std::getenv("FEWHA_PDL");
    attr[0].val.programmaticStreamSerializationAllowed = (pdl && pdl[0] == '0') ? 0 : 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_fwd_inv_layer<T, FLEN>, gp, bf, fmode, fit, imode, iit, fit_term, ctr);
}
// CTAs of the fused whole-layer kernel resident per SM (0: it does not fit)
template <typename T, int FLEN>
cudaError_t whole_fused_capacity(const GeoParams& gp, int* per_sm) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, k_fwd_inv_layer<T, FLEN>, Wl<T>::threads,
                                                         whole_layer_smem(gp.maxside, static_cast<int>(sizeof(T))));
}

// Fused forward + inverse (k_fwd_inv_cluster): the cluster grid launched
// cooperatively so the instance barrier's CTAs are co-resident.
template <typename T, int FLEN>
cudaError_t launch_fused_cluster(const GeoParams& gp, const Bufs<T>& bf, int fmode, int fit, int imode, int iit,
                                 int count, cudaStream_t st, int fit_term, size_t smem, unsigned long long* bar,
                                 int pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(gp.ccl, gp.L, count);
    cfg.blockDim = dim3(kClThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[3];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = gp.ccl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    attr[2].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[2].val.programmaticStreamSerializationAllowed = pdl;
    cfg.attrs = attr;
    cfg.numAttrs = 3;
    return cudaLaunchKernelEx(&cfg, k_fwd_inv_cluster<T, FLEN>, gp, bf, fmode, fit, imode, iit, fit_term, bar);
}

// Clusters of the fused kernel that fit the device at once with `smem` bytes.
template <typename T, int FLEN>
cudaError_t fused_cluster_capacity(const GeoParams& gp, size_t smem, int* clusters) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(gp.ccl, gp.L, 1);
    cfg.blockDim = dim3(kClThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = gp.ccl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaOccupancyMaxActiveClusters(clusters, k_fwd_inv_cluster<T, FLEN>, &cfg);
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
    // 16-CTA clusters (FEWHA_CLUSTER_ROWS=8) are beyond the portable size 8
    for (const void* k : {(const void*)k_inv_cluster<T, FLEN>, (const void*)k_fwd_cluster<T, FLEN>,
                          (const void*)k_fwd_inv_cluster<T, FLEN>}) {
        const cudaError_t a = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (a != cudaSuccess) return a;
    }
    cudaError_t e = opt_in_max(k_inv_cluster<T, FLEN>, smem_inv);
    if (e != cudaSuccess) return e;
    e = opt_in_max(k_inv_layer<T, FLEN>, smem_inv);
    if (e != cudaSuccess) return e;
    e = opt_in_max(k_fwd_layer<T, FLEN>, smem_fwd);
    if (e != cudaSuccess) return e;
    e = opt_in_max(k_fwd_inv_cluster<T, FLEN>, smem_fwd);
    if (e != cudaSuccess) return e;
    e = opt_in_max(k_fwd_inv_layer<T, FLEN>, smem_fwd);
    if (e != cudaSuccess) return e;
    return opt_in_max(k_fwd_cluster<T, FLEN>, smem_fwd);
}

#define FEWHA_INST(T)                                                                                          \
    template cudaError_t launch_layer_cluster<T, FEWHA_FLEN>(bool, const GeoParams&, const Bufs<T>&, int, int, int, \
                                                             cudaStream_t, int, size_t);                        \
    template cudaError_t launch_fused_cluster<T, FEWHA_FLEN>(const GeoParams&, const Bufs<T>&, int, int, int, int, \
                                                             int, cudaStream_t, int, size_t, unsigned long long*, \
                                                             int);                                              \
    template cudaError_t fused_cluster_capacity<T, FEWHA_FLEN>(const GeoParams&, size_t, int*);                 \
    template cudaError_t launch_layer_whole<T, FEWHA_FLEN>(bool, const GeoParams&, const Bufs<T>&, int, int, int,   \
                                                           cudaStream_t, int);                                  \
    template cudaError_t launch_layer_whole_fused<T, FEWHA_FLEN>(const GeoParams&, const Bufs<T>&, int, int, int, int, \
                                                                 int, cudaStream_t, int, unsigned long long*); \
    template cudaError_t whole_fused_capacity<T, FEWHA_FLEN>(const GeoParams&, int*);                           \
    template cudaError_t set_layer_cluster_attrs<T, FEWHA_FLEN>(size_t, size_t);
FEWHA_INST(double)
FEWHA_INST(float)

}  // namespace fewha_gpu
