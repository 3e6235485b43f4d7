// Device kernels of the closed-loop simulation harness: the
// callers of the hot path that feed it slopes and score its output, restated
// from the reference's simulation layer (proj/include/fewha/simulation.hpp) so
// a whole run_closed_loop stays on the device with no per-frame host transfer.
//
//   k_gauss          GaussianStream (simulation.hpp:40-58): std::mt19937_64 bits,
//                    Box-Muller pairs; one warp per stream, the 312-word twist
//                    split into its three data-parallel phases
//   k_atm_*          generate_atmosphere (simulation.hpp:76-127): spectrum shaping,
//                    inverse 2-D DFT (exact twiddles, e^{+i}), real part, mean
//                    removal, variance scaling
//   k_frozen_flow    truth_at_step (simulation.hpp:131-158)
//   k_noise_scatter  synthesize_measurements' noise (simulation.hpp:196-207): sigma_w
//                    times the stream on sx then sy of every active subaperture
//   k_quality_dir    evaluate_quality (simulation.hpp:228-269): per probe direction
//                    the propagated truth minus the DM correction on the annular-
//                    pupil nodes, piston removed, variance
//   k_layer_err      evaluate_quality's layer_rel_err (simulation.hpp:272-300)
// Reductions are fixed-order (block trees), so runs are bitwise reproducible; they
// differ from the reference's sequential sums by rounding only (~1e-16 relative).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "device.hpp"

namespace fewha_gpu {
namespace sim {

constexpr int kMtN = 312, kMtM = 156;

__device__ __forceinline__ unsigned long long mt_temper(unsigned long long y) {
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}
__device__ __forceinline__ unsigned long long mt_mix(unsigned long long cur, unsigned long long nxt,
                                                     unsigned long long far) {
    const unsigned long long x = (cur & 0xFFFFFFFF80000000ULL) | (nxt & 0x7FFFFFFFULL);
    const unsigned long long xa = x >> 1;
    return far ^ ((x & 1ULL) ? (xa ^ 0xB5026F5AA96619E9ULL) : xa);
}

// One warp per stream: stream s has seed seeds[s] and writes `count` normals to
// out + s * stride, in the reference's draw order (cos, sin of each pair).
// blockDim = 32.  (count is even for every caller; an odd count drops the
// final sin half, which GaussianStream would cache for the next call.)
__global__ void __launch_bounds__(32) k_gauss(const unsigned long long* __restrict__ seeds, int count,
                                              double* __restrict__ out, long long stride) {
    __shared__ unsigned long long mt[kMtN];
    __shared__ unsigned long long y[kMtN];
    const int lane = threadIdx.x;
    if (lane == 0) {  // std::mt19937_64 seeding ([rand.eng.mers]): sequential
        unsigned long long v = seeds[blockIdx.x];
        mt[0] = v;
        for (int i = 1; i < kMtN; ++i) {
            v = 6364136223846793005ULL * (v ^ (v >> 62)) + static_cast<unsigned long long>(i);
            mt[i] = v;
        }
    }
    __syncwarp();
    double* o = out + static_cast<long long>(blockIdx.x) * stride;
    for (int base = 0; base < count; base += kMtN) {
        // twist: [0, 156) read old words only; [156, 311) read the new words 156
        // back; 311 reads the new word 0 and the new word 155
        unsigned long long nw[5];
#pragma unroll
        for (int r = 0; r < 5; ++r) {
            const int i = lane + 32 * r;
            if (i < kMtM) nw[r] = mt_mix(mt[i], mt[i + 1], mt[i + kMtM]);
        }
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 5; ++r) {
            const int i = lane + 32 * r;
            if (i < kMtM) mt[i] = nw[r];
        }
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 5; ++r) {
            const int i = kMtM + lane + 32 * r;
            if (i < kMtN - 1) nw[r] = mt_mix(mt[i], mt[i + 1], mt[i - kMtM]);
        }
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 5; ++r) {
            const int i = kMtM + lane + 32 * r;
            if (i < kMtN - 1) mt[i] = nw[r];
        }
        __syncwarp();
        if (lane == 0) mt[kMtN - 1] = mt_mix(mt[kMtN - 1], mt[0], mt[kMtM - 1]);
        __syncwarp();
        for (int i = lane; i < kMtN; i += 32) y[i] = mt_temper(mt[i]);
        __syncwarp();
        // Box-Muller over the 156 pairs of this block of draws
        for (int p = lane; p < kMtN / 2; p += 32) {
            const int k = base + 2 * p;
            if (k >= count) continue;
            const double u1 = (static_cast<double>(y[2 * p] >> 11) + 1.0) * 0x1.0p-53;  // (0, 1]
            const double u2 = static_cast<double>(y[2 * p + 1] >> 11) * 0x1.0p-53;     // [0, 1)
            const double m = sqrt(-2.0 * log(u1));
            const double a = 2.0 * 3.141592653589793 * u2;
            double s, c;
            sincos(a, &s, &c);
            o[k] = m * c;
            if (k + 1 < count) o[k + 1] = m * s;
        }
        __syncwarp();
    }
}

// ---- generate_atmosphere ---------------------------------------------------------
// Layer table: side n, offset (nodal), period, target variance, normals offset.
struct AtmLayer {
    int n, off, zoff;
    double period, target;
};
struct AtmParams {
    AtmLayer lay[kMaxL];
    int L;
    double kappa0;
};

// spectrum (re, im) per node, shaped, DC zeroed; complex [n][n] interleaved at
// spec + 2*off.  grid (n, L), block n.
__global__ void k_atm_spectrum(const AtmParams ap, const double* __restrict__ z, double* __restrict__ spec) {
    const int l = blockIdx.y, ki = blockIdx.x, kj = threadIdx.x;
    const AtmLayer& la = ap.lay[l];
    const int n = la.n;
    if (ki >= n || kj >= n) return;
    const int wi = ki <= n / 2 ? ki : ki - n, wj = kj <= n / 2 ? kj : kj - n;
    const size_t idx = static_cast<size_t>(ki) * n + kj;
    const double re = z[la.zoff + 2 * idx], im = z[la.zoff + 2 * idx + 1];
    double* o = spec + 2 * (static_cast<size_t>(la.off) + idx);
    if (wi == 0 && wj == 0) {
        o[0] = 0.0;
        o[1] = 0.0;
        return;
    }
    const double kx = 2.0 * 3.141592653589793 * wj / la.period;
    const double ky = 2.0 * 3.141592653589793 * wi / la.period;
    const double amp = pow(kx * kx + ky * ky + ap.kappa0 * ap.kappa0, -11.0 / 12.0);
    o[0] = re * amp;  // std::complex(re, im) * amp
    o[1] = im * amp;
}

// inverse DFT along one axis (sum_k X(k) e^{+2 pi i k x / n}); cols = 0: along rows
// (x = column), 1: along columns.  grid (n, L), block n; dst may not alias src.
__global__ void k_atm_dft(const AtmParams ap, const double* __restrict__ src, double* __restrict__ dst, int cols) {
    const int l = blockIdx.y, line = blockIdx.x, x = threadIdx.x;
    const AtmLayer& la = ap.lay[l];
    const int n = la.n;
    if (line >= n || x >= n) return;
    const double* s = src + 2 * static_cast<size_t>(la.off);
    double re = 0.0, im = 0.0;
    for (int k = 0; k < n; ++k) {
        const size_t e = cols ? static_cast<size_t>(k) * n + line : static_cast<size_t>(line) * n + k;
        double sn, cs;
        sincospi(2.0 * static_cast<double>((k * x) % n) / n, &sn, &cs);  // exact argument reduction
        const double a = s[2 * e], b = s[2 * e + 1];
        re += a * cs - b * sn;
        im += a * sn + b * cs;
    }
    const size_t e = cols ? static_cast<size_t>(x) * n + line : static_cast<size_t>(line) * n + x;
    dst[2 * (static_cast<size_t>(la.off) + e)] = re;
    dst[2 * (static_cast<size_t>(la.off) + e) + 1] = im;
}

// Fixed-order block sum (blockDim a power of two <= 1024), valid in every thread.
__device__ __forceinline__ double block_sum_all(double v, double* red) {
    const int t = threadIdx.x;
    red[t] = v;
    __syncthreads();
    for (int s = blockDim.x >> 1; s > 0; s >>= 1) {
        if (t < s) red[t] += red[t + s];
        __syncthreads();
    }
    const double r = red[0];
    __syncthreads();
    return r;
}

// real part, mean removed, scaled to the target variance; one block (1024) per layer
__global__ void __launch_bounds__(1024) k_atm_finish(const AtmParams ap, const double* __restrict__ cplx,
                                                     double* __restrict__ out) {
    __shared__ double red[1024];
    const AtmLayer& la = ap.lay[blockIdx.x];
    const int nn = la.n * la.n;
    double s = 0.0;
    for (int e = threadIdx.x; e < nn; e += blockDim.x) s += cplx[2 * (static_cast<size_t>(la.off) + e)];
    const double mean = block_sum_all(s, red) / static_cast<double>(nn);
    double v = 0.0;
    for (int e = threadIdx.x; e < nn; e += blockDim.x) {
        const double d = cplx[2 * (static_cast<size_t>(la.off) + e)] - mean;
        v += d * d;
    }
    const double var = block_sum_all(v, red) / static_cast<double>(nn);
    const double scale = var > 0.0 ? sqrt(la.target / var) : 0.0;
    for (int e = threadIdx.x; e < nn; e += blockDim.x)
        out[la.off + e] = (cplx[2 * (static_cast<size_t>(la.off) + e)] - mean) * scale;
}

// ---- truth_at_step ----------------------------------------------------------------
struct FlowParams {
    int L;
    int n[kMaxL], off[kMaxL];
    double si[kMaxL], sj[kMaxL];  // row / column shifts in nodes (wind * step / spacing)
};
__global__ void k_frozen_flow(const FlowParams fp, const double* __restrict__ base, double* __restrict__ out) {
    const int l = blockIdx.y;
    const int n = fp.n[l];
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * n) return;
    const int i = e / n, j = e - i * n;
    const double dn = static_cast<double>(n);
    double ti = fmod(i + fp.si[l], dn), tj = fmod(j + fp.sj[l], dn);
    if (ti < 0) ti += n;
    if (tj < 0) tj += n;
    const int i0 = static_cast<int>(ti) % n, j0 = static_cast<int>(tj) % n;
    const int i1 = (i0 + 1) % n, j1 = (j0 + 1) % n;
    const double fi = ti - floor(ti), fj = tj - floor(tj);
    const double* b = base + fp.off[l];
    out[fp.off[l] + e] = (1 - fi) * ((1 - fj) * b[i0 * n + j0] + fj * b[i0 * n + j1]) +
                         fi * ((1 - fj) * b[i1 * n + j0] + fj * b[i1 * n + j1]);
}

// ---- synthesize_measurements' noise -----------------------------------------------
// pair t of the frame's stream: sx index, sy index, sigma (active subapertures in
// WFS then row-major order)
__global__ void k_noise_scatter(const int* __restrict__ ix, const int* __restrict__ iy,
                                const double* __restrict__ sigma, int pairs, const double* __restrict__ z,
                                double* __restrict__ noise) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= pairs) return;
    noise[ix[t]] = sigma[t] * z[2 * t];
    noise[iy[t]] = sigma[t] * z[2 * t + 1];
}

// ---- evaluate_quality ---------------------------------------------------------------
// Per (direction, screen) separable stencil tables over the finest WFS grid:
// idx/frac along x (by column j) and y (by row i), n entries each.
struct QualParams {
    int L, M, n, n_nodes, n_dir;
    int side[kMaxL], loff[kMaxL];
    int nact[kMaxM], aoff[kMaxM];
    const int* node;    // [n_nodes] i * n + j of the annular-pupil nodes, row-major
    const int* tidx;    // [(dir * (L+M) + s) * 2 + axis][n]
    const double* tw;   // same layout: bilinear fractions
};

__device__ __forceinline__ double bil(const double* g, int stride, int i0, int j0, double fy, double fx) {
    // bilinear_sample (operators.hpp:123-127): w00 v00 + w01 v01 + w10 v10 + w11 v11
    const double w00 = (1.0 - fy) * (1.0 - fx), w01 = (1.0 - fy) * fx, w10 = fy * (1.0 - fx), w11 = fy * fx;
    const double* r = g + i0 * stride + j0;
    return w00 * r[0] + w01 * r[1] + w10 * r[stride] + w11 * r[stride + 1];
}

// one block per direction: variance of the piston-removed residual -> var[dir]
__global__ void __launch_bounds__(512) k_quality_dir(const QualParams qp, const double* __restrict__ layers,
                                                    const double* __restrict__ dms, double* __restrict__ var) {
    extern __shared__ double res[];  // [n_nodes]
    __shared__ double red[512];
    const int dir = blockIdx.x, S = qp.L + qp.M, n = qp.n;
    double s = 0.0;
    for (int k = threadIdx.x; k < qp.n_nodes; k += blockDim.x) {
        const int node = qp.node[k], i = node / n, j = node - i * n;
        double t = 0.0, c = 0.0;
        for (int l = 0; l < qp.L; ++l) {  // propagate_point over the truth screens
            const size_t bx = (static_cast<size_t>(dir) * S + l) * 2 * n, by = bx + n;
            t += bil(layers + qp.loff[l], qp.side[l], qp.tidx[by + i], qp.tidx[bx + j], qp.tw[by + i], qp.tw[bx + j]);
        }
        for (int m = 0; m < qp.M; ++m) {
            const size_t bx = (static_cast<size_t>(dir) * S + qp.L + m) * 2 * n, by = bx + n;
            c += bil(dms + qp.aoff[m], qp.nact[m], qp.tidx[by + i], qp.tidx[bx + j], qp.tw[by + i], qp.tw[bx + j]);
        }
        res[k] = t - c;
        s += t - c;
    }
    const double mean = block_sum_all(s, red) / static_cast<double>(qp.n_nodes);
    double v = 0.0;
    for (int k = threadIdx.x; k < qp.n_nodes; k += blockDim.x) v += (res[k] - mean) * (res[k] - mean);
    const double vv = block_sum_all(v, red) / static_cast<double>(qp.n_nodes);
    if (threadIdx.x == 0) var[dir] = vv;
}

// layer_rel_err partial sums per layer (paired L = M only): DM l resampled on layer l's
// grid with the layer extent (bilinear_sample(dm, extent, ...)), both mean-removed.
// One block (1024) per layer -> part[l] = {num, den}.
struct LerrParams {
    int L;
    int side[kMaxL], loff[kMaxL], nact[kMaxL], aoff[kMaxL];
    const int* tidx;   // [l][side] dm-grid index of each layer node coordinate
    const double* tw;  // [l][side] fraction
    int toff[kMaxL];
};
__global__ void __launch_bounds__(1024) k_layer_err(const LerrParams lp, const double* __restrict__ layers,
                                                   const double* __restrict__ dms, double* __restrict__ part) {
    __shared__ double red[1024];
    const int l = blockIdx.x, nl = lp.side[l], na = lp.nact[l];
    const int nn = nl * nl;
    const double* lt = layers + lp.loff[l];
    const double* dm = dms + lp.aoff[l];
    const int* ti = lp.tidx + lp.toff[l];
    const double* tw = lp.tw + lp.toff[l];
    double st = 0.0, sr = 0.0;
    for (int e = threadIdx.x; e < nn; e += blockDim.x) {
        const int i = e / nl, j = e - i * nl;
        st += lt[e];
        sr += bil(dm, na, ti[i], ti[j], tw[i], tw[j]);
    }
    const double mean_t = block_sum_all(st, red) / nn;
    const double mean_r = block_sum_all(sr, red) / nn;
    double num = 0.0, den = 0.0;
    for (int e = threadIdx.x; e < nn; e += blockDim.x) {
        const int i = e / nl, j = e - i * nl;
        const double up = bil(dm, na, ti[i], ti[j], tw[i], tw[j]);
        const double diff = (up - mean_r) - (lt[e] - mean_t);
        num += diff * diff;
        den += (lt[e] - mean_t) * (lt[e] - mean_t);
    }
    const double a = block_sum_all(num, red), b = block_sum_all(den, red);
    if (threadIdx.x == 0) {
        part[2 * l] = a;
        part[2 * l + 1] = b;
    }
}

// field_rms and layer_rel_err of one frame from the per-direction variances and
// the per-layer partials (sequential, as the reference) -> rec[0..1]; rms_per_dir -> rec[2..]
__global__ void k_quality_finish(const double* __restrict__ var, int n_dir, const double* __restrict__ part, int L,
                                 int paired, double* __restrict__ rec) {
    if (threadIdx.x != 0) return;
    double sum_sq = 0.0;
    for (int d = 0; d < n_dir; ++d) {
        rec[2 + d] = sqrt(var[d]);
        sum_sq += var[d];
    }
    rec[0] = sqrt(sum_sq / n_dir);
    if (paired) {
        double num = 0.0, den = 0.0;
        for (int l = 0; l < L; ++l) {
            num += part[2 * l];
            den += part[2 * l + 1];
        }
        rec[1] = den > 0.0 ? sqrt(num / den) : 0.0;
    } else {
        rec[1] = __longlong_as_double(0x7ff8000000000000LL);  // NaN: no L = M pairing
    }
}

}  // namespace sim
}  // namespace fewha_gpu
