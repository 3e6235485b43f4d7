// sm_100a kernels of the FEWHA reconstructor: the per-WFS tile kernel, the
// fitting/control kernel, the operator-entry kernels and the shared device
// helpers (TMA bulk copies, programmatic dependent launch, the fused-PCG scalar
// step).  The cluster-distributed layer transforms and the adjoint gather are in
// cluster.cuh, the simulation harness in sim_kernels.cuh.
//
// Every operator of the reference's hot path (reconstructor.hpp:166-355) is a
// hand-written kernel.  No tensor cores: nothing on the path is a dense
// contraction; the kernels are HBM/L2-bandwidth and latency bound.
// Design points of this file:
//   * k_wfs: one CTA per 14 x 14 wavefront-node tile (+1-node halo = 256 nodes,
//     one per thread) of one WFS and instance.  The tile's stencil tables arrive
//     by one TMA bulk copy before the programmatic-launch wait; P (9 layers' 36
//     bilinear loads in flight per node), Gamma, C^-1 and Gamma^T then run in
//     shared memory, Gamma^T as a gather in the reference's scatter order
//     (operators.hpp:176-187);
//   * k_fit_control: one thread per actuator; the DM history and the fitting
//     stencils are loaded before the programmatic-launch wait; a^(1) is also
//     stored straight into a page-locked caller buffer (zero-copy output);
//   * PCG dots are per-CTA partials written to fixed slots and summed in fixed
//     order by every consumer (run-to-run bitwise deterministic); the scalar
//     recurrences (pcg.hpp:80-99) are evaluated redundantly by each consumer CTA
//     (pcg_scalar_from_sums), and the p/q/c/r updates are fused into the next
//     iteration's W^-1 kernel (cluster.cuh).
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <type_traits>

#include "device.hpp"

namespace fewha_gpu {

// Daubechies analysis (lo) / highpass (hi) taps of the configured order live in
// the kernel parameter block (GeoParams::flo/fhi): constant-bank operands, one
// copy per launch, no per-translation-unit __constant__ symbols.
template <typename T>
struct Filt;
template <>
struct Filt<double> {
    __device__ static double lo(const GeoParams& gp, int k) { return gp.flo[k]; }
    __device__ static double hi(const GeoParams& gp, int k) { return gp.fhi[k]; }
};
template <>
struct Filt<float> {
    __device__ static float lo(const GeoParams& gp, int k) { return gp.flo_f[k]; }
    __device__ static float hi(const GeoParams& gp, int k) { return gp.fhi_f[k]; }
};

// ---- TMA 1-D bulk copies (cp.async.bulk) completing on an mbarrier --------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* m, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* m, unsigned bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* m) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(m)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* m, unsigned parity) {
    asm volatile(
        "{\n.reg .pred P;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        "@!P bra WAIT_%=;\n}\n" ::"r"(smem_u32(m)),
        "r"(parity)
        : "memory");
}
// dst, src 16-byte aligned; bytes a multiple of 16 (callers round up inside padded buffers)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* m) {
    mbar_expect_tx(m, bytes);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(m))
                 : "memory");
}
__device__ __forceinline__ unsigned round16(unsigned v) { return (v + 15u) & ~15u; }

// A single-use-per-phase bulk loader: thread 0 issues, everyone waits.
struct Bulk {
    unsigned long long* mbar;
    unsigned phase;
    __device__ __forceinline__ void init() {
        if (threadIdx.x == 0) {
            mbar_init(mbar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
        phase = 0;
    }
    // thread 0 only
    __device__ __forceinline__ void begin() {
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    }
    __device__ __forceinline__ void copy(void* dst, const void* src, unsigned bytes) { bulk_g2s(dst, src, round16(bytes), mbar); }
    __device__ __forceinline__ void commit() { mbar_arrive(mbar); }
    // all threads
    __device__ __forceinline__ void wait() {
        mbar_wait(mbar, phase);
        phase ^= 1u;
    }
};

// ---- programmatic dependent launch -------------------------------------------
// Every frame kernel lets its successor launch at once (launch_dependents) and
// waits for its predecessor's results only where it first reads them
// (griddepcontrol.wait): launch latency and constant-table prefetches overlap
// the previous kernel's tail.  Both are no-ops for non-programmatic launches.
// Programmatic dependent launch protocol of the frame: every kernel triggers its
// dependents only AFTER its own griddepcontrol.wait.  A kernel's pre-wait prologue
// therefore runs while its predecessor (N-1) may still execute, but kernel N-2 and
// everything before it are complete and visible -- so the prologue may read the
// outputs of N-2 and older (constant tables, and the PCG vectors the previous
// inverse wrote), never those of N-1.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

template <typename T>
__device__ __forceinline__ const T* weights(const GeoParams& gp);
template <>
__device__ __forceinline__ const double* weights<double>(const GeoParams& gp) { return gp.td; }
template <>
__device__ __forceinline__ const float* weights<float>(const GeoParams& gp) { return gp.tf; }

__device__ __forceinline__ int bit_width(unsigned m) { return 32 - __clz(static_cast<int>(m)); }

// ---------------------------------------------------------------------------
// Deterministic block reduction (fixed shuffle tree, fixed warp order).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double block_sum(double v, double* scratch) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        for (int i = 0; i < nw; ++i) t += scratch[i];
    }
    __syncthreads();
    return t;  // valid in thread 0
}

template <typename T, bool COL>
__device__ __forceinline__ T& at(T* buf, int P, int line, int pos) {
    return COL ? buf[pos * P + line] : buf[line * P + pos];
}

// Per-thread output staging of the in-place DWT passes (4 fp64 / 8 fp32).
template <typename T>
struct SegOf {
    static constexpr int value = 4;  // (8 for fp32 doubled the registers: 118 vs 77 in the inverse, one CTA/SM less)
};

// ---------------------------------------------------------------------------
// Fused-PCG scalar step (pcg.hpp:72-99), evaluated for the iteration whose
// partial dots are complete.  Deterministic: fixed-order sum of the L slots.
// ---------------------------------------------------------------------------
struct ScalarStep {
    Carry out;
    int apply, log;
    double beta, alpha, logval;
};

__device__ inline ScalarStep pcg_scalar_from_sums(const GeoParams& gp, const Carry& in, double rho, double mu,
                                                   int first) {
    ScalarStep r;
    r.out = in;
    r.apply = 0;
    r.log = 0;
    r.beta = 0.0;
    r.alpha = 0.0;
    r.logval = 0.0;
    if (in.done || in.err) return r;
    if (first) r.out.rho_entry = rho;
    if (gp.tol > 0.0 && rho <= gp.tol * gp.tol * r.out.rho_entry) {  // offline exit, pcg.hpp:75-78
        r.log = 1;
        r.logval = rho;
        r.out.done = 1;
        return r;
    }
    if (rho == 0.0 && mu == 0.0) {  // exactly converged: no-op iteration, pcg.hpp:80-85
        r.log = 1;
        return r;
    }
    double beta, alpha;
    if (in.fresh) {
        beta = 0.0;
        alpha = rho / mu;
        r.out.fresh = 0;
    } else {
        beta = rho / in.rho_old;
        alpha = rho / (mu - rho * beta / in.alpha);
    }
    if (!isfinite(rho) || !isfinite(mu) || !isfinite(beta) || !isfinite(alpha)) {
        r.out.err = 1;
        return r;
    }
    r.out.rho_old = rho;
    r.out.alpha = alpha;
    r.apply = 1;
    r.log = 1;
    r.logval = rho;
    r.beta = beta;
    r.alpha = alpha;
    return r;
}



// ---------------------------------------------------------------------------
// Bilinear stencil pieces (operators.hpp:108-121): separable tables per
// (WFS, layer) built on the host in fp64 with the reference's expressions.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T bilinear(const T* g, int stride, int i0, int j0, T fy, T fx) {
    const T w00 = (T(1) - fy) * (T(1) - fx), w01 = (T(1) - fy) * fx;
    const T w10 = fy * (T(1) - fx), w11 = fy * fx;
    const T* r0 = g + i0 * stride + j0;
    return w00 * r0[0] + w01 * r0[1] + w10 * r0[stride] + w11 * r0[stride + 1];
}

// Sum over layers of the bilinear layer values at aperture node (i, j) of WFS w
// (propagate_point, operators.hpp:204-213).
template <typename T>
__device__ __forceinline__ T prop_layers(const GeoParams& gp, const T* layers, int w, int i, int j) {
    const T* tw = weights<T>(gp);
    T acc = T(0);
    for (int l = 0; l < gp.L; ++l) {
        const int* dir = gp.ti + gp.o_pl + (w * gp.L + l) * 4;
        const int ox = dir[0] + j, oy = dir[1] + i;
        acc += bilinear<T>(layers + gp.coff[l], gp.side[l], gp.ti[oy], gp.ti[ox], tw[oy], tw[ox]);
    }
    return acc;
}

// Same over DM screens (dm_screens, reconstructor.hpp:357-364).
template <typename T>
__device__ __forceinline__ T prop_dms(const GeoParams& gp, const T* dms, int w, int i, int j) {
    const T* tw = weights<T>(gp);
    T acc = T(0);
    for (int m = 0; m < gp.M; ++m) {
        const int* dir = gp.ti + gp.o_pd + (w * gp.M + m) * 2;
        const int ox = dir[0] + j, oy = dir[1] + i;
        acc += bilinear<T>(dms + gp.aoff[m], gp.nact[m], gp.ti[oy], gp.ti[ox], tw[oy], tw[ox]);
    }
    return acc;
}

// ---------------------------------------------------------------------------
// Phase B: per (WFS node tile, instance)
//   rhs=false: psi = fault * Gamma^T C^-1 Gamma P phi   (apply_M stage 2, :182-192)
//   rhs=true : psi = fault * Gamma^T C^-1 (s + [closed] Gamma P_dm a_prev2)
//              (add_dm_slopes :259-280 + build_rhs stage 1 :221-231)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void wstamp(const GeoParams& gp, int k) {
    if (gp.stamps == nullptr || threadIdx.x != 0) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned blk = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    gp.stamps[blk * 16 + k] = t;
}

// WFS tiles: 14 x 14 nodes, (14+2)^2 = 256 wavefront nodes = one per thread of a
// 256-thread CTA in the dominant phase (16 x 16 tiles on 512 threads left 37 % of
// the warps waiting at the barrier).  Resident CTAs per SM: 3 for single-instance
// plans; batches take four instances per CTA at 4 (fp64) / 6 (fp32) CTAs per SM
// (kWfsNi4Minb: more tiles in flight; k_wfs below).
#ifndef FEWHA_WFS_TILE
#define FEWHA_WFS_TILE 14
#endif
#ifndef FEWHA_WFS_THREADS
#define FEWHA_WFS_THREADS 256
#endif
#ifndef FEWHA_WFS_MINB_LAT
#define FEWHA_WFS_MINB_LAT 3
#endif
#ifndef FEWHA_WFS_MINB_BATCH
#define FEWHA_WFS_MINB_BATCH 4
#endif
#ifndef FEWHA_WFS_GLAT
// screens per load group of the latency plan: all 9 layers' 36 loads in flight at once
// (80 registers, 16 B of spills) beat groups of 7 (no spills): 0.1844 vs 0.1865 ms per frame
#define FEWHA_WFS_GLAT 9
#endif
// Batches: resident CTAs per SM with two / four instances per CTA, loads in groups of 2
// screens (no spills).  Batch 64 per step (profiles/r02_experiments.md, fourth session):
// fp64 two instances at 3/SM with groups of 3 (72 registers) 2.429 ms, 4/SM 2.359, 5/SM
// 2.294, 6/SM 2.292; four instances at 4/SM (64 registers) 2.229, 6/SM 2.294; fp32 four
// instances 2/SM 1.531, 4/SM 1.520, 6/SM (40 registers) 1.511.
constexpr int kWfsNi2Minb = 6;
template <typename T>
constexpr int kWfsNi4Minb = sizeof(T) == 8 ? 4 : 6;
constexpr int kWfsTile = FEWHA_WFS_TILE;  // WFS node tile side (compile-time: index math by constants)
constexpr int kWfsThreads = FEWHA_WFS_THREADS;  // threads per WFS tile CTA

// Shared memory of one WFS tile: stencil tables of the tile's halo rows and
// columns for every screen, then the wavefront, then the two slope grids.
template <typename T>
__host__ __device__ constexpr size_t wfs_tile_table_bytes(int screens) {
    constexpr int H = kWfsTile + 2;
    return ((static_cast<size_t>(screens) * 2 * H * sizeof(int) + 15) & ~size_t(15)) +
           ((static_cast<size_t>(screens) * 2 * H * sizeof(T) + 15) & ~size_t(15));
}
template <typename T>
__host__ __device__ constexpr size_t wfs_tile_smem(int screens, int ni = 1) {
    constexpr int H = kWfsTile + 2, Q = kWfsTile + 1;
    return wfs_tile_table_bytes<T>(screens) + static_cast<size_t>(ni) * (H * H + 2 * Q * Q) * sizeof(T);
}

// One WFS tile for NI consecutive instances b0 .. b0+NI-1 (batches: the tile's stencil
// tables, index math and bilinear weights are shared by the instances, and each thread
// keeps NI instances' loads in flight).
template <typename T, bool RHS, int G = 9, int NI = 1>
__device__ __forceinline__ void wfs_tile(const GeoParams& gp, const Bufs<T>& bf, int with_dm, int tile, int b0,
                                         int ninst, unsigned char* smem_raw) {
    constexpr int TS = kWfsTile, H = TS + 2, Q = TS + 1;
    int w, i0, j0;
    if (gp.n_wtiles <= kMaxWtCode) {
        const unsigned code = gp.wt_code[tile];
        w = static_cast<int>(code & 0xffu);
        i0 = static_cast<int>((code >> 8) & 0xfffu) * TS;
        j0 = static_cast<int>(code >> 20) * TS;
    } else {
        w = 0;
        while (w + 1 < gp.W && tile >= gp.wt_first[w + 1]) ++w;
        const int local = tile - gp.wt_first[w], trow = local / gp.wt_cols[w];
        i0 = trow * TS;
        j0 = (local - trow * gp.wt_cols[w]) * TS;
    }
    const int ns = gp.ns[w], np = ns + 1;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const bool screens_on = !RHS || with_dm;
    const int NS = RHS ? gp.M : gp.L;  // screens: DMs for the RHS, layers otherwise
    // stencil tables of the halo rows/columns: [screen][axis][H] (index), then weights
    const int ib = (NS * 2 * H * static_cast<int>(sizeof(int)) + 15) & ~15;
    int* tix = reinterpret_cast<int*>(smem_raw);
    T* tw = reinterpret_cast<T*>(smem_raw + ib);
    T* ph = tw + NS * 2 * H;  // [NI][H*H]
    T* sx = ph + NI * H * H;  // [NI][Q*Q]
    T* sy = sx + NI * Q * Q;
    __shared__ unsigned long long s_mbar;
    wstamp(gp, 0);
    if (screens_on) {
        // prebuilt per-tile tables (constant): fetched by one TMA bulk copy before
        // waiting on the predecessor kernel
        if (tid == 0) {
            mbar_init(&s_mbar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // smem reused by a persistent caller
            const int stride = RHS ? gp.tt_stride_d : gp.tt_stride_l;
            const unsigned char* src = gp.tblob + (RHS ? gp.tt_off_d : 0) + static_cast<size_t>(tile) * stride;
            bulk_g2s(smem_raw, src, static_cast<unsigned>(stride), &s_mbar);
            mbar_arrive(&s_mbar);
        }
        __syncthreads();
        pdl_wait();
        pdl_launch_dependents();
        mbar_wait(&s_mbar, 0);
    } else {
        pdl_wait();
        pdl_launch_dependents();
    }
    __syncthreads();
    wstamp(gp, 1);
    // 1. wavefront on the tile + 1-node halo (propagate_point, operators.hpp:204-213)
    const size_t inst_stride = RHS ? static_cast<size_t>(gp.A) : static_cast<size_t>(gp.n);
    const T* src = (RHS ? bf.a_prev2 : bf.phi) + static_cast<size_t>(b0) * inst_stride;
    for (int idx = tid; idx < H * H; idx += nthr) {
        const int a = idx / H, c = idx - a * H;
        const int i = i0 - 1 + a, j = j0 - 1 + c;
        T v[NI];
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) v[ni] = T(0);
        if (screens_on && i >= 0 && i < np && j >= 0 && j < np) {
            // screens in unrolled groups of G: a group's 4 G NI loads are in flight together
            // (padding screens of the last group read a valid node with weight 0)
            for (int s0 = 0; s0 < NS; s0 += G) {
                T q00[G][NI], q01[G][NI], q10[G][NI], q11[G][NI], fy[G], fx[G];
#pragma unroll
                for (int u = 0; u < G; ++u) {
                    const int sc = min(s0 + u, NS - 1);
                    const int* tx = tix + sc * 2 * H;
                    const T* wx = tw + sc * 2 * H;
                    const int stride = RHS ? gp.nact[sc] : gp.side[sc];
                    const T* r0 = src + (RHS ? gp.aoff[sc] : gp.coff[sc]) + tx[H + a] * stride + tx[c];
#pragma unroll
                    for (int ni = 0; ni < NI; ++ni) {
                        const T* rn = r0 + (ni < ninst ? ni : 0) * inst_stride;
                        q00[u][ni] = rn[0];
                        q01[u][ni] = rn[1];
                        q10[u][ni] = rn[stride];
                        q11[u][ni] = rn[stride + 1];
                    }
                    fy[u] = s0 + u < NS ? wx[H + a] : T(0);
                    fx[u] = wx[c];
                }
#pragma unroll
                for (int u = 0; u < G; ++u) {
                    if (s0 + u >= NS) break;
                    // bilinear(): w00 v00 + w01 v01 + w10 v10 + w11 v11 (operators.hpp:125-126)
                    const T w00 = (T(1) - fy[u]) * (T(1) - fx[u]), w01 = (T(1) - fy[u]) * fx[u];
                    const T w10 = fy[u] * (T(1) - fx[u]), w11 = fy[u] * fx[u];
#pragma unroll
                    for (int ni = 0; ni < NI; ++ni)
                        v[ni] += w00 * q00[u][ni] + w01 * q01[u][ni] + w10 * q10[u][ni] + w11 * q11[u][ni];
                }
            }
        }
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) ph[ni * H * H + idx] = v[ni];
    }
    __syncthreads();
    wstamp(gp, 2);
    // 2. weighted half-slopes on the (TS+1)^2 subapertures touching the tile
    const T iv = static_cast<T>(gp.inv_var[w]);
    const std::uint8_t* mask = gp.masks + gp.mkoff[w];
    for (int e = tid; e < NI * Q * Q; e += nthr) {
        const int ni = e / (Q * Q), idx = e - ni * Q * Q;
        const int a = idx / Q, c = idx - a * Q;
        const int i = i0 - 1 + a, j = j0 - 1 + c;
        const T* phn = ph + ni * H * H;
        T x = T(0), y = T(0);
        if (ni < ninst && i >= 0 && i < ns && j >= 0 && j < ns && mask[i * ns + j]) {
            const T p00 = phn[a * H + c], p01 = phn[a * H + c + 1];
            const T p10 = phn[(a + 1) * H + c], p11 = phn[(a + 1) * H + c + 1];
            T gx = T(0.5) * ((p01 - p00) + (p11 - p10));  // sh_apply, operators.hpp:160-161
            T gy = T(0.5) * ((p10 - p00) + (p11 - p01));
            if (RHS) {
                const double* meas = bf.meas + static_cast<size_t>(b0 + ni) * gp.S + gp.moff[w];
                const int k = i * ns + j;
                const T mx = static_cast<T>(meas[k]), my = static_cast<T>(meas[ns * ns + k]);
                gx = with_dm ? mx + gx : mx;
                gy = with_dm ? my + gy : my;
            }
            x = T(0.5) * (gx * iv);
            y = T(0.5) * (gy * iv);
        }
        sx[e] = x;
        sy[e] = y;
    }
    __syncthreads();
    wstamp(gp, 3);
    // 3. adjoint slopes: gather of the 4 neighbouring subapertures in the
    //    reference's scatter order (operators.hpp:176-187)
    for (int e = tid; e < NI * TS * TS; e += nthr) {
        const int ni = e / (TS * TS), idx = e - ni * TS * TS;
        const int a = idx / TS, c = idx - a * TS;
        const int i = i0 + a, j = j0 + c;
        if (ni >= ninst || i >= np || j >= np) continue;
        const T* sxn = sx + ni * Q * Q;
        const T* syn = sy + ni * Q * Q;
        T v = sxn[a * Q + c] + syn[a * Q + c];
        v += -sxn[a * Q + c + 1] + syn[a * Q + c + 1];
        v += sxn[(a + 1) * Q + c] - syn[(a + 1) * Q + c];
        v += -sxn[(a + 1) * Q + c + 1] - syn[(a + 1) * Q + c + 1];
        if (gp.fault != 1.0) v *= static_cast<T>(gp.fault);
        T* psi = bf.psi + static_cast<size_t>(b0 + ni) * gp.Nw + gp.woff[w];
        psi[i * np + j] = v;
    }
    wstamp(gp, 4);
}

// NI instances per CTA (grid.y = ceil(B / NI)).
template <typename T, bool RHS, int MINB, int NI = 1>
__global__ void __launch_bounds__(kWfsThreads, MINB) k_wfs(const GeoParams gp, const Bufs<T> bf, int with_dm, int count) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // screens per unrolled load group: FEWHA_WFS_GLAT (9) for the latency plan (3 CTAs/SM),
    // 5 for batches of one instance per CTA (4 CTAs/SM, 56 registers), 2 with two / four
    // instances per CTA (kWfsNi2Minb / kWfsNi4Minb CTAs/SM)
    constexpr int G = NI > 1 ? 2 : (MINB >= 4 && sizeof(T) == 8) ? 5 : FEWHA_WFS_GLAT;
    const int b0 = blockIdx.y * NI;
    wfs_tile<T, RHS, G, NI>(gp, bf, with_dm, gp.wt_base + blockIdx.x, b0, min(NI, count - b0), smem_raw);
}

// ---------------------------------------------------------------------------
// Fitting + control law (reconstructor.hpp:284-305, :335-351).
//   step=1: a~ from phi = W^-1 c; a1 = control(a~); rotate history; a_out = a1
//   step=0: out = a~ (fit_to_mirrors operator)
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void frame_epilogue(const GeoParams& gp, const Bufs<T>& bf, int b) {
    // publish status, seed the next frame's carry slot 0
    Carry c = bf.carry[b * (gp.iters + 1) + gp.iters];
    bf.status[b] = c.err;
    bf.nlog[b] = c.nlog;
    if (bf.frame_host) {  // the host's copy of this instance's rho log, status and count
        const int B = gridDim.y;
        double* hr = reinterpret_cast<double*>(bf.frame_host);
        for (int k = 0; k < gp.iters; ++k) hr[b * gp.iters + k] = bf.rho_log[b * gp.iters + k];
        int* hs = reinterpret_cast<int*>(hr + static_cast<size_t>(B) * gp.iters);
        hs[b] = c.err;
        hs[B + b] = c.nlog;
    }
    c.done = 0;
    c.err = 0;
    c.nlog = 0;
    c.rho_entry = 0.0;
    bf.carry[b * (gp.iters + 1)] = c;
}

// One actuator's fit + control.  Everything constant (the DM's layer group, the
// bilinear stencil of every layer) and the DM history (written by the previous
// frame, 21 launches back: kernels.cuh protocol) is loaded before the
// programmatic-launch wait; after it only the phi samples of the group (all in
// flight together) remain on the critical path.
template <typename T>
__device__ __forceinline__ void fit_actuator(const GeoParams& gp, const Bufs<T>& bf, int step, int k, int b,
                                             bool live) {
    int m = 0;
    while (m + 1 < gp.M && k >= gp.aoff[m + 1]) ++m;
    const int idx = k - gp.aoff[m], na = gp.nact[m];
    const int i = idx / na, j = idx % na;
    const size_t g = static_cast<size_t>(b) * gp.A + k;
    const int ofit = live ? gp.ti[gp.o_fit + m] : -1;
    // bilinear resampling of each layer of the DM's group (ascending layer order); the
    // stencils of the first kFitPre layers are resolved before the programmatic-launch
    // wait (register arrays; 16 of them held 128 registers and capped the kernel at 16
    // warps per SM), any further layers of the group (LTAO: all nine) after it
    constexpr int kFitPre = 4;
    int src[kFitPre], sd[kFitPre];
    T fy[kFitPre], fx[kFitPre];
    int cnt = 0;
    const T* tw = weights<T>(gp);
    if (live && ofit >= 0) {
        cnt = gp.ti[ofit];
#pragma unroll
        for (int q = 0; q < kFitPre; ++q) {
            src[q] = -1;
            sd[q] = 0;
            fy[q] = fx[q] = T(0);
            if (q < cnt) {
                const int l = gp.ti[ofit + 1 + 3 * q], ox = gp.ti[ofit + 2 + 3 * q], oy = gp.ti[ofit + 3 + 3 * q];
                const int ii = gp.ti[oy + i], jj = gp.ti[ox + j];
                if (ii >= 0 && jj >= 0) {  // a projected point off this layer's grid contributes zero
                    sd[q] = gp.side[l];
                    src[q] = gp.coff[l] + ii * sd[q] + jj;
                    fy[q] = tw[oy + i];
                    fx[q] = tw[ox + j];
                }
            }
        }
    }
    T a0 = T(0), a1 = T(0);
    if (live && step) {
        a0 = bf.a_prev[g];
        a1 = bf.a_prev2[g];
    }
    pdl_wait();
    pdl_launch_dependents();
    if (!live) return;
    // A non-finite PCG scalar makes the reference throw from pcg_solve before
    // fit_to_mirrors and the history rotation (reconstructor.hpp:325-351): no
    // command is produced and a^(-1), a^(0) stay as they were.  (The flag is read
    // alongside the phi samples below; only the stores wait for it.)
    const bool failed = step && bf.carry[b * (gp.iters + 1) + gp.iters].err != 0;
    const T* phi_b = bf.phi + static_cast<size_t>(b) * gp.n;
    T at;
    if (ofit < 0) {  // identity pairing, n_act = 2^J (reconstructor.hpp:304-307)
        at = phi_b[gp.coff[m] + i * gp.side[m] + j];
    } else {
        at = T(0);
#pragma unroll
        for (int q = 0; q < kFitPre; ++q) {
            if (q >= cnt) break;
            if (src[q] < 0) continue;
            at += bilinear<T>(phi_b + src[q], sd[q], 0, 0, fy[q], fx[q]);
        }
        for (int q = kFitPre; q < cnt; ++q) {
            const int l = gp.ti[ofit + 1 + 3 * q], ox = gp.ti[ofit + 2 + 3 * q], oy = gp.ti[ofit + 3 + 3 * q];
            const int ii = gp.ti[oy + i], jj = gp.ti[ox + j];
            if (ii < 0 || jj < 0) continue;
            at += bilinear<T>(phi_b + gp.coff[l] + ii * gp.side[l] + jj, gp.side[l], 0, 0, tw[oy + i], tw[ox + j]);
        }
    }
    if (!step) {
        bf.a_out[g] = at;
        return;
    }
    if (failed) return;
    const T gain = static_cast<T>(gp.gain);
    const T an = gp.closed ? a0 + gain * (at - a1) : (T(1) - gain) * a0 + gain * at;
    bf.a_prev2[g] = a0;
    bf.a_prev[g] = an;
    bf.a_out[g] = an;
    if (bf.a_host) bf.a_host[g] = static_cast<double>(an);  // posted PCIe write into the caller's buffer
}

template <typename T>
__global__ void __launch_bounds__(256) k_fit_control(const GeoParams gp, const Bufs<T> bf, int step) {
    const int b = blockIdx.y;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    fit_actuator(gp, bf, step, k < gp.A ? k : 0, b, k < gp.A);
    if (step && blockIdx.x == 0 && threadIdx.x == 0) frame_epilogue(gp, bf, b);
}

// ---------------------------------------------------------------------------
// Operator kernels used by the reference-facing per-operator entry points.
// ---------------------------------------------------------------------------

// P: nodal layers [B][n] -> wavefronts [B][Nw]  (operators.hpp:217-235)
template <typename T>
__global__ void k_propagate(const GeoParams gp, const T* layers, T* wf, int count) {
    const int b = blockIdx.y;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= gp.Nw || b >= count) return;
    int w = 0;
    while (w + 1 < gp.W && k >= gp.woff[w + 1]) ++w;
    const int np = gp.ns[w] + 1, idx = k - gp.woff[w];
    wf[static_cast<size_t>(b) * gp.Nw + k] = prop_layers<T>(gp, layers + static_cast<size_t>(b) * gp.n, w, idx / np, idx % np);
}

// Gamma of (P layers - P_dm dms) [+ meas_in] -> meas_out (sh_apply, add_dm_slopes,
// synthesize_measurements without noise).  Per subaperture.
//   src_wf: if non-null, wavefronts are read directly (plain Gamma)
template <typename T>
__global__ void k_slopes(const GeoParams gp, const T* src_wf, const T* layers, const T* dms, T dm_sign,
                         const double* meas_in, double* meas_out, int count) {
    const int b = blockIdx.y;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int total = gp.S / 2;  // subapertures over all WFS
    if (k >= total || b >= count) return;
    int w = 0;
    while (w + 1 < gp.W && k >= gp.moff[w + 1] / 2) ++w;
    const int ns = gp.ns[w], np = ns + 1, idx = k - gp.moff[w] / 2;
    const int i = idx / ns, j = idx % ns;
    const size_t ox = static_cast<size_t>(b) * gp.S + gp.moff[w] + idx, oy = ox + static_cast<size_t>(ns) * ns;
    double gx = 0.0, gy = 0.0;
    if (gp.masks[gp.mkoff[w] + idx]) {
        T p[4];
        for (int q = 0; q < 4; ++q) {
            const int ii = i + (q >> 1), jj = j + (q & 1);
            T v = T(0);
            if (src_wf) {
                v = src_wf[static_cast<size_t>(b) * gp.Nw + gp.woff[w] + ii * np + jj];
            } else {
                if (layers) v = prop_layers<T>(gp, layers + static_cast<size_t>(b) * gp.n, w, ii, jj);
                if (dms) v = v + dm_sign * prop_dms<T>(gp, dms + static_cast<size_t>(b) * gp.A, w, ii, jj);
            }
            p[q] = v;
        }
        gx = static_cast<double>(T(0.5) * ((p[1] - p[0]) + (p[3] - p[2])));
        gy = static_cast<double>(T(0.5) * ((p[2] - p[0]) + (p[3] - p[1])));
    }
    if (meas_in) {
        meas_out[ox] = meas_in[ox] + gx;
        meas_out[oy] = meas_in[oy] + gy;
    } else {
        meas_out[ox] = gx;
        meas_out[oy] = gy;
    }
}

// Gamma^T: meas [B][S] -> wavefronts [B][Nw]  (sh_transpose_apply, operators.hpp:168-188)
template <typename T>
__global__ void k_sh_transpose(const GeoParams gp, const double* meas, T* wf, int count) {
    const int b = blockIdx.y;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= gp.Nw || b >= count) return;
    int w = 0;
    while (w + 1 < gp.W && k >= gp.woff[w + 1]) ++w;
    const int ns = gp.ns[w], np = ns + 1, idx = k - gp.woff[w];
    const int i = idx / np, j = idx % np;
    const double* m = meas + static_cast<size_t>(b) * gp.S + gp.moff[w];
    const std::uint8_t* mask = gp.masks + gp.mkoff[w];
    auto half = [&](int a, int c, T& x, T& y) {
        x = T(0);
        y = T(0);
        if (a >= 0 && a < ns && c >= 0 && c < ns && mask[a * ns + c]) {
            x = T(0.5) * static_cast<T>(m[a * ns + c]);
            y = T(0.5) * static_cast<T>(m[ns * ns + a * ns + c]);
        }
    };
    T x, y, v;
    half(i - 1, j - 1, x, y);
    v = x + y;
    half(i - 1, j, x, y);
    v += -x + y;
    half(i, j - 1, x, y);
    v += x - y;
    half(i, j, x, y);
    v += -x - y;
    if (gp.fault != 1.0) v *= static_cast<T>(gp.fault);
    wf[static_cast<size_t>(b) * gp.Nw + k] = v;
}

template <typename Src, typename Dst>
__global__ void k_convert(const Src* in, Dst* out, size_t n) {
    const size_t k = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k < n) out[k] = static_cast<Dst>(in[k]);
}


}  // namespace fewha_gpu
