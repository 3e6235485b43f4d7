// Launchers of the filter-length-templated cluster kernels, instantiated one
// filter length per translation unit (layer_flen.cu, -DFEWHA_FLEN=N) so the
// build parallelises.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

#include "device.hpp"

namespace fewha_gpu {

template <typename T, int FLEN>
cudaError_t launch_layer_cluster(bool inverse, const GeoParams& gp, const Bufs<T>& bf, int mode, int it, int count,
                                 cudaStream_t st, int fit_term, size_t smem);

template <typename T, int FLEN>
cudaError_t launch_fused_cluster(const GeoParams& gp, const Bufs<T>& bf, int fmode, int fit, int imode, int iit,
                                 int count, cudaStream_t st, int fit_term, size_t smem, unsigned long long* bar,
                                 int pdl);

template <typename T, int FLEN>
cudaError_t fused_cluster_capacity(const GeoParams& gp, size_t smem, int* clusters);

template <typename T, int FLEN>
cudaError_t launch_layer_whole(bool inverse, const GeoParams& gp, const Bufs<T>& bf, int mode, int it, int count,
                               cudaStream_t st, int fit_term);

template <typename T, int FLEN>
cudaError_t launch_layer_whole_fused(const GeoParams& gp, const Bufs<T>& bf, int fmode, int fit, int imode, int iit,
                                     int count, cudaStream_t st, int fit_term, unsigned long long* ctr);

template <typename T, int FLEN>
cudaError_t whole_fused_capacity(const GeoParams& gp, int* per_sm);

template <typename T, int FLEN>
cudaError_t set_layer_cluster_attrs(size_t smem_inv, size_t smem_fwd);

}  // namespace fewha_gpu
