// Persistent cooperative frame kernel: one launch = one Reconstructor::step
// (reconstructor.hpp:310-355) for a single instance.
//
// Grid (C, L, 1) with clusters (C,1,1): cluster l owns layer l (bands as in
// cluster.cuh); the per-WFS tiles of Gamma^T C^-1 Gamma P are spread over all
// C*L CTAs.  Phases are separated by a hierarchical grid barrier: a cluster
// barrier, one gpu-scope release/acquire atomic per cluster, a cluster
// barrier.  The barrier count per frame is 2 + 3*iters - 1 (13 at 4 PCG
// iterations) instead of 16 kernel launch/drain gaps.
//
// Phase order (cf. engine.cu launch_frame, which runs the same phase
// functions as separate launches for batched instances):
//   RHS tiles | fwd(kRhs) + inv(kPcg, it=0) | { tiles | fwd(kPcg) | inv } x iters
//   with the last inv in kFit mode followed by the cluster-local fitting +
//   control law of DM l (L = M pairing, reconstructor.hpp:284-351).
#pragma once

#include "cluster.cuh"

namespace fewha_gpu {

// All clusters arrive; returns when every cluster has arrived `target` times
// in total.  Writes before the barrier are visible after it (cluster-scope
// release/acquire inside each cluster, gpu-scope release/acquire across).
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int target, cg::cluster_group& cl) {
    cl.sync();
    if (cl.block_rank() == 0 && threadIdx.x == 0) {
        __threadfence();
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        unsigned int v;
        while (true) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
            if (v >= target) break;
            __nanosleep(20);
        }
        __threadfence();
    }
    cl.sync();
}

__device__ __forceinline__ void fstamp(const GeoParams& gp, int& k) {
    if (gp.fstamps == nullptr || threadIdx.x != 0) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned blk = blockIdx.x + gridDim.x * blockIdx.y;
    if (k < 32) gp.fstamps[blk * 32 + k] = t;
    ++k;
}

template <typename T, int FLEN>
__global__ void __launch_bounds__(256, 1) k_frame(const GeoParams gp, const Bufs<T> bf, unsigned int* bar) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cg::cluster_group cl = cg::this_cluster();
    const int l = blockIdx.y, b = 0;
    const int C = static_cast<int>(gridDim.x);
    const int cta = blockIdx.y * C + blockIdx.x, ncta = C * static_cast<int>(gridDim.y);
    const unsigned int nclusters = gridDim.y;
    unsigned int nb = 0;
    int ks = 0;
    fstamp(gp, ks);

    // RHS: psi = Gamma^T C^-1 (s + Gamma P_dm a^(-1))  (reconstructor.hpp:316-319)
    for (int t = cta; t < gp.n_wtiles; t += ncta) {
        wfs_tile<T, true>(gp, bf, gp.closed, t, b, smem_raw);
        __syncthreads();
    }
    fstamp(gp, ks);
    grid_barrier(bar, ++nb * nclusters, cl);
    fstamp(gp, ks);
    // b1 = W sum P^T psi; r += b1 - b; b = b1; then iteration 0's z = r/J, rho, W^-1 z
    fwd_phase<T, FLEN>(gp, bf, kRhs, 0, 1, smem_raw, l, b, cl);
    fstamp(gp, ks);
    cl.sync();
    inv_phase<T, FLEN>(gp, bf, kPcg, 0, smem_raw, l, b, cl);
    fstamp(gp, ks);
    grid_barrier(bar, ++nb * nclusters, cl);
    fstamp(gp, ks);
    for (int it = 0; it < gp.iters; ++it) {
        for (int t = cta; t < gp.n_wtiles; t += ncta) {
            wfs_tile<T, false>(gp, bf, 0, t, b, smem_raw);
            __syncthreads();
        }
        fstamp(gp, ks);
        grid_barrier(bar, ++nb * nclusters, cl);
        fstamp(gp, ks);
        fwd_phase<T, FLEN>(gp, bf, kPcg, it, 1, smem_raw, l, b, cl);
        fstamp(gp, ks);
        grid_barrier(bar, ++nb * nclusters, cl);  // every mu partial of iteration `it`
        fstamp(gp, ks);
        if (it + 1 < gp.iters) {
            inv_phase<T, FLEN>(gp, bf, kPcg, it + 1, smem_raw, l, b, cl);
            fstamp(gp, ks);
            grid_barrier(bar, ++nb * nclusters, cl);
            fstamp(gp, ks);
        } else {
            inv_phase<T, FLEN>(gp, bf, kFit, 0, smem_raw, l, b, cl);
            fstamp(gp, ks);
        }
    }
    cl.sync();  // phi of layer l complete within the cluster
    if (l < gp.M) {
        const int a0 = gp.aoff[l], na = gp.nact[l] * gp.nact[l];
        const int rank = static_cast<int>(cl.block_rank());
        for (int k = rank * blockDim.x + threadIdx.x; k < na; k += C * blockDim.x) fit_actuator(gp, bf, 1, a0 + k, b);
    }
    if (cta == 0 && threadIdx.x == 0) frame_epilogue(gp, bf, b);
    fstamp(gp, ks);
}

}  // namespace fewha_gpu
