// sm_100a kernels of the FEWHA reconstructor.
//
// Every operator of the reference's hot path (reconstructor.hpp:166-355) is a
// hand-written kernel here.  No tensor cores: nothing on the path is a dense
// contraction; the kernels are HBM/L2-bandwidth and latency bound (SURVEY.md
// 8d).  Design points:
//   * a whole 2^J x 2^J layer lives in shared memory (odd pitch side+1, so
//     row-walks and column-walks are both bank-conflict free) while its
//     multilevel periodic Daubechies transform runs; each pass stages its
//     outputs in registers across one CTA barrier, so the transform is in
//     place with no second buffer (128 KiB fp64 at J=7);
//   * the per-WFS chain Gamma^T C^-1 Gamma P runs on 16x16 node tiles with a
//     one-node halo: P gather -> slopes -> adjoint slopes all in shared memory;
//   * the adjoint propagation P^T is an atomic-free separable gather: the
//     bilinear stencil factorises (x depends only on the column, y only on the
//     row, operators.hpp:208-210), so per layer tile a psi block is staged and
//     contracted along columns then rows, WFS in ascending order
//     (reconstructor.hpp:199-200) -- deterministic, no float atomics;
//   * PCG dots are per-layer CTA partials written to fixed slots and summed in
//     fixed order by every consumer (run-to-run bitwise deterministic); the
//     scalar recurrences (pcg.hpp:80-99) are evaluated redundantly by each
//     consumer CTA, and the p/q/c/r updates are fused into the next
//     iteration's W^-1 kernel.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

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
    static constexpr int value = sizeof(T) == 8 ? 4 : 8;
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
template <typename T, bool RHS>
__global__ void __launch_bounds__(256) k_wfs(const GeoParams gp, const Bufs<T> bf, int with_dm) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int TS = gp.wtile, H = TS + 2, Q = TS + 1;
    T* ph = reinterpret_cast<T*>(smem_raw);
    T* sx = ph + H * H;
    T* sy = sx + Q * Q;
    const int tile = blockIdx.x, b = blockIdx.y;
    const int w = gp.wtiles[3 * tile], i0 = gp.wtiles[3 * tile + 1], j0 = gp.wtiles[3 * tile + 2];
    const int ns = gp.ns[w], np = ns + 1;
    const int tid = threadIdx.x, nthr = blockDim.x;

    // 1. wavefront on the tile + 1-node halo
    for (int idx = tid; idx < H * H; idx += nthr) {
        const int i = i0 - 1 + idx / H, j = j0 - 1 + idx % H;
        T v = T(0);
        if (i >= 0 && i < np && j >= 0 && j < np) {
            if (!RHS) v = prop_layers<T>(gp, bf.phi + static_cast<size_t>(b) * gp.n, w, i, j);
            else if (with_dm) v = prop_dms<T>(gp, bf.a_prev2 + static_cast<size_t>(b) * gp.A, w, i, j);
        }
        ph[idx] = v;
    }
    __syncthreads();
    // 2. weighted half-slopes on the (TS+1)^2 subapertures touching the tile
    const T iv = static_cast<T>(gp.inv_var[w]);
    const std::uint8_t* mask = gp.masks + gp.mkoff[w];
    const double* meas = bf.meas + static_cast<size_t>(b) * gp.S + gp.moff[w];
    for (int idx = tid; idx < Q * Q; idx += nthr) {
        const int a = idx / Q, c = idx % Q;
        const int i = i0 - 1 + a, j = j0 - 1 + c;
        T x = T(0), y = T(0);
        if (i >= 0 && i < ns && j >= 0 && j < ns && mask[i * ns + j]) {
            const T p00 = ph[a * H + c], p01 = ph[a * H + c + 1];
            const T p10 = ph[(a + 1) * H + c], p11 = ph[(a + 1) * H + c + 1];
            T gx = T(0.5) * ((p01 - p00) + (p11 - p10));  // sh_apply, operators.hpp:160-161
            T gy = T(0.5) * ((p10 - p00) + (p11 - p01));
            if (RHS) {
                const int k = i * ns + j;
                const T mx = static_cast<T>(meas[k]), my = static_cast<T>(meas[ns * ns + k]);
                gx = with_dm ? mx + gx : mx;
                gy = with_dm ? my + gy : my;
            }
            x = T(0.5) * (gx * iv);
            y = T(0.5) * (gy * iv);
        }
        sx[idx] = x;
        sy[idx] = y;
    }
    __syncthreads();
    // 3. adjoint slopes: gather of the 4 neighbouring subapertures in the
    //    reference's scatter order (operators.hpp:176-187)
    T* psi = bf.psi + static_cast<size_t>(b) * gp.Nw + gp.woff[w];
    for (int idx = tid; idx < TS * TS; idx += nthr) {
        const int a = idx / TS, c = idx % TS;
        const int i = i0 + a, j = j0 + c;
        if (i >= np || j >= np) continue;
        T v = sx[a * Q + c] + sy[a * Q + c];
        v += -sx[a * Q + c + 1] + sy[a * Q + c + 1];
        v += sx[(a + 1) * Q + c] - sy[(a + 1) * Q + c];
        v += -sx[(a + 1) * Q + c + 1] - sy[(a + 1) * Q + c + 1];
        if (gp.fault != 1.0) v *= static_cast<T>(gp.fault);
        psi[i * np + j] = v;
    }
}

// ---------------------------------------------------------------------------
// Phase C1: y_l = sum_w P_{w,l}^T psi_w on one layer tile per CTA: separable
// gather (columns, then rows), WFS in ascending order.  No atomics.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) k_adjoint(const GeoParams gp, const T* __restrict__ psi_all, T* __restrict__ y_all) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int TP = gp.ltile;
    T* blk = reinterpret_cast<T*>(smem_raw);           // [rows_max][cols_max]
    T* hc = blk + gp.lt_rows_max * gp.lt_cols_max;     // [rows_max][TP]
    const int tile = blockIdx.x, b = blockIdx.y;
    const int l = gp.ltiles[3 * tile], I0 = gp.ltiles[3 * tile + 1], J0 = gp.ltiles[3 * tile + 2];
    const int side = gp.side[l];
    const int nI = min(TP, side - I0), nJ = min(TP, side - J0);
    const int tid = threadIdx.x, nthr = blockDim.x;
    const T* tw = weights<T>(gp);
    constexpr int kMaxPer = 16;
    T acc[kMaxPer];
#pragma unroll
    for (int q = 0; q < kMaxPer; ++q) acc[q] = T(0);

    for (int w = 0; w < gp.W; ++w) {
        const int* dir = gp.ti + gp.o_pl + (w * gp.L + l) * 4;
        const int ox = dir[0], oy = dir[1], orr = dir[2], occ = dir[3];
        const int* tr = gp.ti + gp.o_tr + (tile * gp.W + w) * 4;
        const int ilo = tr[0], ihi = tr[1], jlo = tr[2], jhi = tr[3];
        if (ilo >= ihi || jlo >= jhi) continue;  // footprint misses this tile
        const int nr = ihi - ilo, nc = jhi - jlo, np = gp.ns[w] + 1;
        const T* psi = psi_all + static_cast<size_t>(b) * gp.Nw + gp.woff[w];
        __syncthreads();
        for (int idx = tid; idx < nr * nc; idx += nthr) {
            const int r = idx / nc, c = idx % nc;
            blk[r * nc + c] = psi[(ilo + r) * np + jlo + c];
        }
        __syncthreads();
        for (int idx = tid; idx < nr * nJ; idx += nthr) {
            const int r = idx / nJ, tj = idx % nJ, J = J0 + tj;
            const int jl = gp.ti[occ + 2 * J], jh = gp.ti[occ + 2 * J + 1];
            T s = T(0);
            for (int j = jl; j < jh; ++j) {
                const T fx = tw[ox + j];
                const T wgt = gp.ti[ox + j] == J ? T(1) - fx : fx;
                s += wgt * blk[r * nc + (j - jlo)];
            }
            hc[r * TP + tj] = s;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kMaxPer; ++q) {
            const int idx = tid + q * nthr;
            if (idx >= TP * TP) break;
            const int ti_ = idx / TP, tj = idx % TP;
            if (ti_ >= nI || tj >= nJ) continue;
            const int I = I0 + ti_;
            const int il = gp.ti[orr + 2 * I], ih = gp.ti[orr + 2 * I + 1];
            T s = T(0);
            for (int i = il; i < ih; ++i) {
                const T fy = tw[oy + i];
                const T wgt = gp.ti[oy + i] == I ? T(1) - fy : fy;
                s += wgt * hc[(i - ilo) * TP + tj];
            }
            acc[q] += s;
        }
    }
    T* y = y_all + static_cast<size_t>(b) * gp.n + gp.coff[l];
#pragma unroll
    for (int q = 0; q < kMaxPer; ++q) {
        const int idx = tid + q * nthr;
        if (idx >= TP * TP) break;
        const int ti_ = idx / TP, tj = idx % TP;
        if (ti_ < nI && tj < nJ) y[(I0 + ti_) * side + J0 + tj] = acc[q];
    }
}

// ---------------------------------------------------------------------------
// Fitting + control law (reconstructor.hpp:284-305, :335-351).
//   step=1: a~ from phi = W^-1 c; a1 = control(a~); rotate history; a_out = a1
//   step=0: out = a~ (fit_to_mirrors operator)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) k_fit_control(const GeoParams gp, const Bufs<T> bf, int step) {
    const int b = blockIdx.y;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (step && blockIdx.x == 0 && threadIdx.x == 0) {
        // frame epilogue: publish status, seed the next frame's carry slot 0
        Carry c = bf.carry[b * (gp.iters + 1) + gp.iters];
        bf.status[b] = c.err;
        bf.nlog[b] = c.nlog;
        c.done = 0;
        c.err = 0;
        c.nlog = 0;
        c.rho_entry = 0.0;
        bf.carry[b * (gp.iters + 1)] = c;
    }
    if (k >= gp.A) return;
    int m = 0;
    while (m + 1 < gp.M && k >= gp.aoff[m + 1]) ++m;
    const int idx = k - gp.aoff[m], na = gp.nact[m];
    const int i = idx / na, j = idx % na;
    const int side = gp.side[m];
    const T* ph = bf.phi + static_cast<size_t>(b) * gp.n + gp.coff[m];
    const int ofit = gp.ti[gp.o_fit + m];
    T at;
    if (ofit < 0) {
        at = ph[i * side + j];
    } else {
        const T* tw = weights<T>(gp);
        at = bilinear<T>(ph, side, gp.ti[ofit + i], gp.ti[ofit + j], tw[ofit + i], tw[ofit + j]);
    }
    const size_t g = static_cast<size_t>(b) * gp.A + k;
    if (!step) {
        bf.a_out[g] = at;
        return;
    }
    const T a0 = bf.a_prev[g], a1 = bf.a_prev2[g], gain = static_cast<T>(gp.gain);
    const T an = gp.closed ? a0 + gain * (at - a1) : (T(1) - gain) * a0 + gain * at;
    bf.a_prev2[g] = a0;
    bf.a_prev[g] = an;
    bf.a_out[g] = an;
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
