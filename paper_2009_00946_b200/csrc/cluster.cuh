// Cluster-distributed layer kernels.
//
// One thread-block cluster of C CTAs per (layer, instance) runs the multilevel
// periodic Daubechies transform (wavelet.hpp:115-201) with the ownership
// layout of clayout.hpp: at level s rank q owns the filter positions
// m in [q k, q k + k), k = s/(2C), so
//   * its input rows are the approximation rows it produced itself one level
//     finer (plus the row pass it already applied to them) -- column passes
//     read local shared memory; only the FLEN-2 halo rows after its band
//     (forward) or the FLEN/2-1 approximation rows before it (inverse) cross
//     distributed shared memory;
//   * one cluster barrier per level (ping-pong level buffers make the reads of
//     level s and the writes of level s/2 (forward) / 2s (inverse) disjoint);
//   * the coefficients it finalises (forward) / consumes (inverse) are a fixed
//     per-rank "compact" set, which is also the set of coefficient-domain
//     vector entries it updates in the fused PCG -- epilogues and updates are
//     rank-local, and their operands are prefetched by TMA bulk copies at
//     kernel start;
//   * the T x T tail (levels below 2C) is finished by rank 0 (forward) or
//     evaluated redundantly by every rank (inverse, so the first distributed
//     level needs no barrier).
// The adjoint propagation sum_w P^T psi_w is gathered straight into the
// level-S band (separable, atomic-free, WFS ascending).
// Determinism: every value has one producer and every reduction a fixed order.
#pragma once

#include <cooperative_groups.h>

#include "clayout.hpp"
#include "kernels.cuh"

namespace fewha_gpu {

namespace cg = cooperative_groups;

// Optional phase timestamps (%globaltimer, ns) for profiling: thread 0 of
// every CTA records stamp k into gp.stamps[block * 16 + k].
__device__ __forceinline__ void stamp(const GeoParams& gp, int k) {
    if (gp.stamps == nullptr || threadIdx.x != 0) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned blk = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    gp.stamps[blk * 16 + k] = t;
}

// ---- cluster barrier (split arrive / wait) and DSMEM addressing ------------
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cl_sync() {
    cl_arrive();
    cl_wait();
}
template <typename T>
__device__ __forceinline__ T* rmt(T* p, int rank) {
    return cg::this_cluster().map_shared_rank(p, static_cast<unsigned>(rank));
}

__device__ __forceinline__ int ilog2(int v) { return 31 - __clz(v); }

// --- local passes over the first `nlines` lines of the top-left s x s block
//     (in place, register staged, CTA barriers; all sizes powers of two) -----
template <typename T, int FLEN, bool COL>
__device__ __forceinline__ void analysis_lines(T* buf, int P, int s, int nlines, const GeoParams& gp) {
    constexpr int SEGM = SegOf<T>::value;
    constexpr int WIN = 2 * SEGM + FLEN - 2;
    const int h = s >> 1, mask = s - 1;
    const int seg = h < SEGM ? h : SEGM;
    const int segs = h >> ilog2(seg);
    const int nthr = blockDim.x, tid = threadIdx.x;
    int lines = nlines;
    while (lines * segs > nthr) lines >>= 1;
    const int lsh = ilog2(lines);
    for (int l0 = 0; l0 < nlines; l0 += lines) {
        const bool act = tid < lines * segs;
        const int line = l0 + (tid & (lines - 1)), m0 = (tid >> lsh) * seg;
        T a[SEGM], d[SEGM];
        if (act) {
            T win[WIN];  // sliding window: 2*seg+FLEN-2 reads for seg output pairs
#pragma unroll
            for (int q = 0; q < WIN; ++q) {
                if (q >= 2 * seg + FLEN - 2) break;
                win[q] = at<T, COL>(buf, P, line, (2 * m0 + q) & mask);
            }
#pragma unroll
            for (int e = 0; e < SEGM; ++e) {
                if (e >= seg) break;
                T sa = T(0), sd = T(0);
#pragma unroll
                for (int k = 0; k < FLEN; ++k) {
                    sa += Filt<T>::lo(gp, k) * win[2 * e + k];
                    sd += Filt<T>::hi(gp, k) * win[2 * e + k];
                }
                a[e] = sa;
                d[e] = sd;
            }
        }
        __syncthreads();
        if (act) {
#pragma unroll
            for (int e = 0; e < SEGM; ++e) {
                if (e >= seg) break;
                at<T, COL>(buf, P, line, m0 + e) = a[e];
                at<T, COL>(buf, P, line, h + m0 + e) = d[e];
            }
        }
        __syncthreads();
    }
}

template <typename T, int FLEN, bool COL>
__device__ __forceinline__ void synthesis_lines(T* buf, int P, int s, int nlines, const GeoParams& gp) {
    constexpr int SEGM = SegOf<T>::value;
    constexpr int HF = FLEN / 2;
    const int h = s >> 1, hmask = h - 1;
    const int seg = h < SEGM ? h : SEGM;
    const int segs = h >> ilog2(seg);
    const int nthr = blockDim.x, tid = threadIdx.x;
    int lines = nlines;
    while (lines * segs > nthr) lines >>= 1;
    const int lsh = ilog2(lines);
    for (int l0 = 0; l0 < nlines; l0 += lines) {
        const bool act = tid < lines * segs;
        const int line = l0 + (tid & (lines - 1)), m0 = (tid >> lsh) * seg;
        T wa[SEGM + HF - 1], wd[SEGM + HF - 1];
        if (act) {
#pragma unroll
            for (int i = 0; i < SEGM + HF - 1; ++i) {
                if (i >= seg + HF - 1) break;
                const int m = (m0 - (HF - 1) + i) & hmask;
                wa[i] = at<T, COL>(buf, P, line, m);
                wd[i] = at<T, COL>(buf, P, line, h + m);
            }
        }
        __syncthreads();
        if (act) {
#pragma unroll
            for (int u = 0; u < 2 * SEGM; ++u) {
                if (u >= 2 * seg) break;
                T acc = T(0);
#pragma unroll
                for (int kk = 0; kk < HF; ++kk) {
                    const int k = (u & 1) + 2 * kk;
                    const int wi = (u >> 1) - kk + HF - 1;
                    acc += wa[wi] * Filt<T>::lo(gp, k) + wd[wi] * Filt<T>::hi(gp, k);
                }
                at<T, COL>(buf, P, line, 2 * m0 + u) = acc;
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Per-CTA plan of one layer (clayout.hpp) and its compact sets.
// ---------------------------------------------------------------------------
constexpr int kMaxLev = 8;
struct LPlan {
    int S, C, lC, q, H, T, nlev, lsS;
    const int* off;   // [nlev+1] compact level offsets (no halo); [nlev] = tail block
    const int* offH;  // [nlev+1] the same with H halo rows
};
// Level offsets are computed once per CTA into shared memory (s_off: 2 x (kMaxLev+1));
// the caller runs __syncthreads before the plan's offsets are used.
__device__ __forceinline__ LPlan make_plan(int S, int C, int D, int q, int H, int* s_off) {
    LPlan p;
    p.S = S;
    p.C = C;
    p.lC = ilog2(C);
    p.q = q;
    p.H = H;
    p.T = clay::tail(S, C, D);
    p.nlev = clay::nlev(S, C, D);
    p.lsS = ilog2(S);
    const int t = threadIdx.x;
    if (t <= p.nlev) s_off[t] = clay::level_off(S, C, 0, t);
    if (t >= 32 && t - 32 <= p.nlev) s_off[kMaxLev + 1 + t - 32] = clay::level_off(S, C, H, t - 32);
    p.off = s_off;
    p.offH = s_off + kMaxLev + 1;
    return p;
}

// Visit every element rank q owns exactly once (thread-strided): f(o, zo, sc)
// with o = compact index (= offset inside the rank's HBM block), zo = index in
// the halo layout, sc = alpha-D scale index bit_width(max(row, col)).
template <typename F>
__device__ __forceinline__ void for_owned(const LPlan& p, F&& f) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    for (int lv = 0; lv < p.nlev; ++lv) {
        const int s = p.S >> lv, h = s >> 1, k = h >> p.lC;
        const int ls = ilog2(s), lh = ls - 1;
        const int o = p.off[lv], oh = p.offH[lv];
        const int nr = k + p.H;
        const int na = k << lh, n = na + (k << ls);
        for (int e = tid; e < n; e += nthr) {
            int zo;
            if (e < na) {
                zo = oh + (((e >> lh) + p.H) << lh) + (e & (h - 1));
            } else {
                const int e2 = e - na;
                zo = oh + (nr << lh) + (((e2 >> ls) + p.H) << ls) + (e2 & (s - 1));
            }
            f(o + e, zo, ls);
        }
    }
    if (p.q == 0) {
        const int o = p.off[p.nlev], oh = p.offH[p.nlev];
        const int T = p.T, lt = ilog2(T);
        for (int e = tid; e < T * T; e += nthr)
            f(o + e, oh + e, bit_width(static_cast<unsigned>(max(e >> lt, e & (T - 1)))));
    }
}

// Prefetch one contiguous block (count elements) into shared memory: a TMA bulk
// copy on mbar issued by thread `issuer` when source, destination and size are
// 16-byte aligned, a cooperative plain copy otherwise.  The caller runs
// __syncthreads, thread 0 arrives on mbar and everyone waits on it.
template <typename T>
__device__ __forceinline__ void prefetch_block(const T* src, T* dst, int count, unsigned long long* mbar, int issuer) {
    if (count <= 0) return;
    const unsigned bytes = static_cast<unsigned>(count) * sizeof(T);
    if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) | bytes) & 15u) == 0) {
        if (static_cast<int>(threadIdx.x) == issuer) bulk_g2s(dst, src, bytes, mbar);
    } else {
        for (int e = threadIdx.x; e < count; e += blockDim.x) dst[e] = src[e];
    }
}

// ---------------------------------------------------------------------------
// Tail levels (T x T, T <= 8 at C = 8) as fused 2-D passes: one output per
// thread, both filter directions at once, one CTA barrier per level.
// Forward level s: out(i,j) = sum_t1 F1[t1] sum_t2 F2[t2] x[2m1+t1][2m2+t2]
// (rows first, as wavelet.hpp:153-168), F = lo for the approximation half.
// ---------------------------------------------------------------------------
#ifndef FEWHA_FUSED_TAIL
#define FEWHA_FUSED_TAIL 16
#endif
constexpr int kFusedTail = FEWHA_FUSED_TAIL;  // tail levels s <= this as fused 2-D passes, larger ones separable
#ifndef FEWHA_CL_THREADS
#define FEWHA_CL_THREADS 256
#endif
constexpr int kClThreads = FEWHA_CL_THREADS;  // threads per CTA of the cluster layer kernels

template <typename T, int FLEN>
__device__ void tail_forward(const GeoParams& gp, const T* src, int ps, int Tt, T* b0, T* b1, T* f) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    const T* cur = src;
    int pc = ps;
    T* nxt = b0;
    int s0 = Tt;
    if (Tt > kFusedTail) {
        // levels s > 8: separable in-place row then column passes on b0 (pitch Tt+1);
        // the detail quadrants of each level are final
        const int lt = ilog2(Tt);
        for (int e = tid; e < Tt * Tt; e += nthr) b0[(e >> lt) * (Tt + 1) + (e & (Tt - 1))] = src[(e >> lt) * ps + (e & (Tt - 1))];
        __syncthreads();
        for (; s0 > kFusedTail; s0 >>= 1) {
            const int h = s0 >> 1, ls = ilog2(s0);
            analysis_lines<T, FLEN, false>(b0, Tt + 1, s0, s0, gp);
            analysis_lines<T, FLEN, true>(b0, Tt + 1, s0, s0, gp);
            for (int e = tid; e < s0 * s0; e += nthr) {  // the next level rewrites only the h x h block
                const int i = e >> ls, j = e & (s0 - 1);
                if (i >= h || j >= h) f[i * Tt + j] = b0[i * (Tt + 1) + j];
            }
        }
        cur = b0;
        pc = Tt + 1;
        nxt = b1;
    }
    stamp(gp, 6);
    for (int s = s0; s >= 2; s >>= 1) {
        const int h = s >> 1, ls = ilog2(s);
        for (int e = tid; e < s * s; e += nthr) {
            const int i = e >> ls, j = e & (s - 1);
            const int m1 = i & (h - 1), m2 = j & (h - 1);
            const bool a1 = i < h, a2 = j < h;
            T acc = T(0);
#pragma unroll
            for (int t1 = 0; t1 < FLEN; ++t1) {
                const T* row = cur + ((2 * m1 + t1) & (s - 1)) * pc;
                T r = T(0);
#pragma unroll
                for (int t2 = 0; t2 < FLEN; ++t2)
                    r += (a2 ? Filt<T>::lo(gp, t2) : Filt<T>::hi(gp, t2)) * row[(2 * m2 + t2) & (s - 1)];
                acc += (a1 ? Filt<T>::lo(gp, t1) : Filt<T>::hi(gp, t1)) * r;
            }
            if (a1 && a2 && s > 2) nxt[i * (Tt + 1) + j] = acc;
            else f[i * Tt + j] = acc;
        }
        __syncthreads();
        cur = nxt;
        pc = Tt + 1;
        nxt = nxt == b0 ? b1 : b0;
    }
    if (Tt == 1 && tid == 0) f[0] = src[0];
}

// Inverse level s (columns first, then rows: wavelet.hpp:170-196):
// out(2m1+u1, 2m2+u2) = sum_{kk2,b2} G_b2 sum_{kk1,b1} G_b1 X(b1 h + m1-kk1, b2 h + m2-kk2),
// X = previous level output in the LL quadrant, the tail coefficients elsewhere.
// Returns the buffer holding the T x T output (pitch T+1).
// The buffer tail_inverse(.., Tt, b0, b1) returns (fused levels alternate b0, b1,
// starting with b0; the separable levels stay in place).
template <typename T, int FLEN>
__device__ __forceinline__ T* tail_buffer(int Tt, T* b0, T* b1) {
    if (Tt == 1) return b0;
    const int sf = Tt < kFusedTail ? Tt : kFusedTail;
    return (ilog2(sf) & 1) ? b0 : b1;
}

template <typename T, int FLEN>
__device__ T* tail_inverse(const GeoParams& gp, const T* zt, int Tt, T* b0, T* b1) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    constexpr int HF = FLEN / 2;
    const T* cur = zt;  // LL source of level 2: the coarse coefficient itself
    int pc = Tt;
    T* nxt = b0;
    const int sf = Tt < kFusedTail ? Tt : kFusedTail;
    // the filter taps in registers (compile-time indices): an output's taps depend on its
    // row / column parity, selected per thread below -- a per-lane parity index into the
    // parameter bank would serialise the warp's constant loads
    T flo[FLEN], fhi[FLEN];
#pragma unroll
    for (int k = 0; k < FLEN; ++k) {
        flo[k] = Filt<T>::lo(gp, k);
        fhi[k] = Filt<T>::hi(gp, k);
    }
    for (int s = 2; s <= sf; s <<= 1) {
        const int h = s >> 1, ls = ilog2(s);
        for (int e = tid; e < s * s; e += nthr) {
            const int r = e >> ls, c = e & (s - 1);
            const int m1 = r >> 1, u1 = r & 1, m2 = c >> 1, u2 = c & 1;
            T l1[HF], h1[HF], l2[HF], h2[HF];
#pragma unroll
            for (int kk = 0; kk < HF; ++kk) {
                l1[kk] = u1 ? flo[2 * kk + 1] : flo[2 * kk];
                h1[kk] = u1 ? fhi[2 * kk + 1] : fhi[2 * kk];
                l2[kk] = u2 ? flo[2 * kk + 1] : flo[2 * kk];
                h2[kk] = u2 ? fhi[2 * kk + 1] : fhi[2 * kk];
            }
            T acc = T(0);
#pragma unroll
            for (int kk2 = 0; kk2 < HF; ++kk2) {
#pragma unroll
                for (int b2 = 0; b2 < 2; ++b2) {
                    const int cc = b2 * h + ((m2 - kk2) & (h - 1));
                    T y = T(0);
#pragma unroll
                    for (int kk1 = 0; kk1 < HF; ++kk1) {
                        const int ra = (m1 - kk1) & (h - 1);
                        const T xa = (cc < h) ? cur[ra * pc + cc] : zt[ra * Tt + cc];
                        const T xd = zt[(h + ra) * Tt + cc];
                        y += xa * l1[kk1] + xd * h1[kk1];
                    }
                    acc += y * (b2 == 0 ? l2[kk2] : h2[kk2]);
                }
            }
            nxt[r * (Tt + 1) + c] = acc;
        }
        __syncthreads();
        cur = nxt;
        pc = Tt + 1;
        nxt = nxt == b0 ? b1 : b0;
    }
    if (Tt == 1) {
        if (tid == 0) b0[0] = zt[0];
        __syncthreads();
        return b0;
    }
    T* buf = const_cast<T*>(cur);  // sf x sf output, pitch Tt+1
    stamp(gp, 6);
    for (int s = 2 * sf; s <= Tt; s <<= 1) {  // separable levels: columns, then rows (wavelet.hpp:170-196)
        const int h = s >> 1, ls = ilog2(s);
        for (int e = tid; e < s * s; e += nthr) {
            const int i = e >> ls, j = e & (s - 1);
            if (i >= h || j >= h) buf[i * (Tt + 1) + j] = zt[i * Tt + j];
        }
        __syncthreads();
        synthesis_lines<T, FLEN, true>(buf, Tt + 1, s, s, gp);
        if (s == Tt) stamp(gp, 7);
        synthesis_lines<T, FLEN, false>(buf, Tt + 1, s, s, gp);
    }
    stamp(gp, 8);
    return buf;
}

// ---------------------------------------------------------------------------
// Forward transform over the cluster.  x0 holds this rank's level-S input
// rows (band rows, pitch P, FLEN-2 spare rows for the halo); finals go to the
// compact set f; tb (C x (C+1)) is rank 0's tail block.
// ---------------------------------------------------------------------------
template <typename T, int FLEN>
__device__ void cdwt_forward(const GeoParams& gp, const LPlan& p, T* x0, T* x1, int P, T* f, T* tb, T* tb2) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int S = p.S, C = p.C, q = p.q;
    if (p.nlev == 0) {  // tail-only layer, whole on rank 0
        if (q == 0) tail_forward<T, FLEN>(gp, x0, P, S, tb, tb2, f);
        return;
    }
    analysis_lines<T, FLEN, false>(x0, P, S, S >> p.lC, gp);  // level-S row pass on the band rows
    constexpr int HR = FLEN - 2;
    constexpr int SEGM = SegOf<T>::value;
    constexpr int WIN = 2 * SEGM + FLEN - 2;
    T* cur = x0;
    T* nxt = x1;
    for (int lv = 0; lv < p.nlev; ++lv) {
        const int s = S >> lv, h = s >> 1, k = h >> p.lC, rows = 2 * k;
        const int ls = ilog2(s), lrows = ilog2(rows);
        const bool last = lv == p.nlev - 1;
        cl_sync();  // level-s input rows (row pass applied) of every rank are complete
        if (lv == 0) stamp(gp, 3);
        // the HR rows after mine (periodic) from their owners
        for (int e = tid; e < HR * s; e += nthr) {
            const int i = e >> ls, j = e & (s - 1);
            const int gm = ((q + 1) * rows + i) & (s - 1);
            const T* src = rmt(cur, gm >> lrows);
            cur[(rows + i) * P + j] = src[(gm & (rows - 1)) * P + j];
        }
        __syncthreads();
        if (lv == 0) stamp(gp, 4);
        // column analysis of my k positions, every column: thread = (column, seg positions)
        const int seg = k < SEGM ? k : SEGM;
        const int items = (k >> ilog2(seg)) * s;
        const int offA = p.off[lv], offD = offA + k * h;
        T* tbq = last ? rmt(tb, 0) : nullptr;
        for (int it = tid; it < items; it += nthr) {
            const int j = it & (s - 1), i0 = (it >> ls) * seg;
            T win[WIN];
#pragma unroll
            for (int t = 0; t < WIN; ++t) {
                if (t >= 2 * seg + FLEN - 2) break;
                win[t] = cur[(2 * i0 + t) * P + j];
            }
#pragma unroll
            for (int e = 0; e < SEGM; ++e) {
                if (e >= seg) break;
                T a = T(0), d = T(0);
#pragma unroll
                for (int t = 0; t < FLEN; ++t) {
                    a += Filt<T>::lo(gp, t) * win[2 * e + t];
                    d += Filt<T>::hi(gp, t) * win[2 * e + t];
                }
                const int i = i0 + e;
                if (j < h) {
                    if (last) tbq[(q * k + i) * (p.T + 1) + j] = a;  // tail rows [q k, q k + k)
                    else nxt[i * P + j] = a;
                } else {
                    f[offA + i * h + (j - h)] = a;
                }
                f[offD + i * s + j] = d;
            }
        }
        __syncthreads();
        if (lv == 0) stamp(gp, 5);
        if (!last) analysis_lines<T, FLEN, false>(nxt, P, h, k, gp);  // row pass of level h
        T* t_ = cur;
        cur = nxt;
        nxt = t_;
    }
    cl_sync();  // every rank's tail row is in rank 0's tb
    stamp(gp, 7);
    if (q == 0) tail_forward<T, FLEN>(gp, tb, p.T + 1, p.T, tb2, tb, f + p.off[p.nlev]);
}

// ---------------------------------------------------------------------------
// Inverse transform over the cluster.  z: the input in the halo layout with
// owned rows, halo rows and the tail block filled.  Returns the buffer holding
// this rank's band rows of the nodal output (pitch *outP).  For layers with
// distributed levels the caller must cl_wait() once before exiting (the
// matching arrive follows this rank's last remote read).
// ---------------------------------------------------------------------------
template <typename T, int FLEN>
__device__ T* cdwt_inverse(const GeoParams& gp, const LPlan& p, const T* z, T* x0, T* x1, T* aw, T* tl,
                           int P, int* outP) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int S = p.S, C = p.C, q = p.q, H = p.H;
    constexpr int HF = FLEN / 2;
    constexpr int SEGP = 4;  // output pairs per thread item
    const int Tt = p.T;
    // tl: rank 0's T x T tail output (pitch T+1), computed by rank 0 before the
    // cluster barrier that precedes this call; the first level reads it remotely
    stamp(gp, 4);
    const T* tl0 = q == 0 ? tl : rmt(tl, 0);
    T* prev = tl;
    T* cur = x0;
    T* other = x1;
    for (int lv = p.nlev - 1; lv >= 0; --lv) {
        const int s = S >> lv, h = s >> 1, k = h >> p.lC, m0 = q * k, nr = k + H;
        const int ls = ilog2(s), lk = ilog2(k);
        const bool first = lv == p.nlev - 1;
        if (!first) cl_sync();  // the previous level's outputs of every rank are complete
        const int oA = p.offH[lv], oD = oA + nr * h;
        // approximation rows m = m0 - H + i: columns [0,h) from the previous level's
        // output (own rows local, halo rows from their owners), [h,s) from z
        for (int e = tid; e < nr * s; e += nthr) {
            const int i = e >> ls, j = e & (s - 1);
            T v;
            if (j < h) {
                const int mm = (m0 - H + i) & (h - 1);
                if (first) {
                    v = tl0[mm * (Tt + 1) + j];
                } else {
                    const int own = mm >> lk;
                    const T* src = own == q ? prev : rmt(prev, own);
                    v = src[(mm & (k - 1)) * P + j];
                }
            } else {
                v = z[oA + i * h + (j - h)];
            }
            aw[i * s + j] = v;
        }
        if (lv == 0) cl_arrive();  // my last remote read is done (caller waits before exit)
        __syncthreads();
        // column synthesis: output rows t in [0, 2k) of level s, every column
        const int seg = k < SEGP ? k : SEGP;
        const int items = (k >> ilog2(seg)) * s;
        for (int it = tid; it < items; it += nthr) {
            const int j = it & (s - 1), i0 = (it >> ls) * seg;
            T wa[SEGP + HF - 1], wd[SEGP + HF - 1];
#pragma unroll
            for (int i = 0; i < SEGP + HF - 1; ++i) {
                if (i >= seg + HF - 1) break;
                wa[i] = aw[(i0 + i) * s + j];
                wd[i] = z[oD + (i0 + i) * s + j];
            }
#pragma unroll
            for (int u = 0; u < 2 * SEGP; ++u) {
                if (u >= 2 * seg) break;
                T acc = T(0);
#pragma unroll
                for (int kk = 0; kk < HF; ++kk) {
                    const int kf = (u & 1) + 2 * kk;
                    const int wi = (u >> 1) - kk + HF - 1;
                    acc += wa[wi] * Filt<T>::lo(gp, kf) + wd[wi] * Filt<T>::hi(gp, kf);
                }
                cur[(2 * i0 + u) * P + j] = acc;
            }
        }
        __syncthreads();
        synthesis_lines<T, FLEN, false>(cur, P, s, 2 * k, gp);  // row synthesis of my output rows
        prev = cur;
        cur = other;
        other = prev;
    }
    *outP = P;
    return prev;
}

// ---------------------------------------------------------------------------
// Adjoint propagation y_l = sum_w P_{w,l}^T psi_w (operators.hpp:241-260).
// The bilinear stencil is separable (operators.hpp:208-210), so per WFS
//   G(i, c)   = sum_q rw(i,q) psi(rs(i,q), c)      rows first, into shared G
//   y(i, J)  += sum_{c: idx_c in {J-1, J}} w(c, J) G(i, c)   then columns
// with w(c, J) = 1 - f_c (idx_c == J) or f_c (idx_c == J-1).  One CTA per
// gp.grows-row group of a layer (grid (side/grows, L, B): 288 CTAs at the ELT
// scale).  Staging per chunk of WFS: the tables by one TMA bulk copy and each
// WFS's psi rows [ilo, ihi) by one bulk copy each, issued by separate threads.
// All WFS of a chunk are row-contracted in one pass, then column-contracted in
// ascending WFS order into per-thread registers: one CTA barrier per chunk,
// deterministic, atomic-free.
// ---------------------------------------------------------------------------
// host-built staging descriptor of one (layer, row group, WFS) (engine.cu, o_gd)
struct GDesc {
    int ilo, ihi, jlo, jhi;  // psi source block of this row group
    int src;                 // psi source element offset (woff + ilo * np)
    int soff;                // psi stage byte offset inside its chunk
    int rtoff, rb;           // row-tap table of (layer, row group, WFS): byte offset in gblob, bytes
    int ctoff, cb;           // column stencil of (layer, WFS) -- shared by every row group: offset, bytes
    int pad0, pad1;
};
constexpr int kGDescInts = 12;

__device__ __forceinline__ int align16(int v) { return (v + 15) & ~15; }

// Stage WFS [w0, w1) (warp 0 only): the chunk's row-tap tables by lane 31 and its
// column stencils by lane 30 (one contiguous copy each: the row tables are stored per
// (layer, row group), the column stencils once per layer, WFS ascending), psi blocks
// by lanes 0..n-1.  The caller __syncwarp()s and lane 0 arrives.
// Stage layout: [row tables | column stencils | psi blocks].
__device__ __forceinline__ int gather_row_bytes(const GDesc* desc, int w0, int w1) {
    return desc[w1 - 1].rtoff + desc[w1 - 1].rb - desc[w0].rtoff;
}
template <typename T>
__device__ __forceinline__ void gather_issue(const GeoParams& gp, const T* psi_b, const GDesc* desc, int w0, int w1,
                                             unsigned char* stage, unsigned long long* mbar, bool tables, bool psi) {
    const int lane = threadIdx.x;
    if (tables && lane == 31) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        bulk_g2s(stage, gp.gblob + desc[w0].rtoff, static_cast<unsigned>(gather_row_bytes(desc, w0, w1)), mbar);
    }
    if (tables && lane == 30) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        const unsigned bytes = static_cast<unsigned>(desc[w1 - 1].ctoff + desc[w1 - 1].cb - desc[w0].ctoff);
        bulk_g2s(stage + gather_row_bytes(desc, w0, w1), gp.gblob + desc[w0].ctoff, bytes, mbar);
    }
    if (psi && lane < w1 - w0) {
        const int w = w0 + lane;
        const GDesc d = desc[w];
        const int nr = d.ihi - d.ilo, np = gp.ns[w] + 1;
        if (nr > 0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            const uintptr_t a = reinterpret_cast<uintptr_t>(psi_b + d.src);
            const unsigned shift = static_cast<unsigned>(a & 15u);
            bulk_g2s(stage + d.soff, reinterpret_cast<const void*>(a - shift),
                     round16(shift + nr * np * static_cast<unsigned>(sizeof(T))), mbar);
        }
    }
}

// Residency of the gather: 2 CTAs per SM with a 110 KB staging budget each for
// single-instance plans (fewer, larger WFS chunks: shortest chain), 3 per SM with
// 72 KB for batches (more row groups in flight: -10 % per launch at B = 64, but
// +3 % on the single frame).  The host splits the WFS into chunks that fit.
// Staging budget per CTA of each residency plan.
__host__ __device__ constexpr int gather_smem_kb(int minb) { return minb >= 4 ? 54 : minb == 3 ? 72 : 110; }

// Contract the staged row group, chunk by chunk (chunk 0 already issued by the caller).
template <typename T, int KM, int ROWS>
__device__ void gather_group(const GeoParams& gp, const T* __restrict__ psi_b, int l, T* __restrict__ y, T* gbuf,
                             unsigned char* stage, const GDesc* desc, unsigned long long* mbar) {
    const int side = gp.side[l];
    const int R = side < ROWS ? side : ROWS;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int lside = ilog2(side);
    const int groups = min(nthr >> lside, R);  // threads per layer column
    const int rows_pt = R / groups;            // group rows per thread
    const int J = tid & (side - 1), grp = tid >> lside;
    const int i0 = grp * rows_pt;
    const bool worker = grp < groups;
    const int gst = ROWS * gp.bd_cols_max;  // G stride per WFS
    const int km = KM > 0 ? KM : gp.gather_km;  // taps per row in the staged tables
    const int o_rw = align16(R * km * 2);      // row table: [src int16 R x km][weight R x km]
    const int o_idx = align16((side + 3) * 2);  // column stencil: [first int16 side+3][idx int16 nc][frac nc]
    T out[ROWS];
#pragma unroll
    for (int k = 0; k < ROWS; ++k) out[k] = T(0);
    for (int k = 0; k < gp.nchunk; ++k) {
        const int w0 = gp.gchunk[k], w1 = gp.gchunk[k + 1];
        if (k > 0 && tid < 32) {
            gather_issue<T>(gp, psi_b, desc, w0, w1, stage, mbar, true, true);
            __syncwarp();
            if (tid == 0) mbar_arrive(mbar);
        }
        mbar_wait(mbar, static_cast<unsigned>(k & 1));
        stamp(gp, 1);
        const int rt0 = desc[w0].rtoff, ct0 = desc[w0].ctoff;
        const unsigned char* cstage = stage + gather_row_bytes(desc, w0, w1);
        // ---- rows: G_w(i, c) for every WFS of the chunk, one pass.  Thread =
        // (WFS group, column): a column's R rows share the thread's index math and
        // the row taps are warp-uniform (broadcast) loads ----
        {
            constexpr int CL = 128;  // columns per thread group
            const int ng = nthr / CL > 0 ? nthr / CL : 1, gq = tid / CL, lane = tid % CL;
            for (int w = w0 + gq; w < w1; w += ng) {
                const GDesc d = desc[w];
                const int nr = d.ihi - d.ilo, np = gp.ns[w] + 1, nc = d.jhi - d.jlo;
                if (nr <= 0) continue;
                const unsigned char* tp = stage + (d.rtoff - rt0);
                const unsigned shift = static_cast<unsigned>(reinterpret_cast<uintptr_t>(psi_b + d.src) & 15u);
                const T* __restrict__ blk = reinterpret_cast<const T*>(stage + d.soff + shift) + d.jlo;  // blk[r*np + c]
                const short* __restrict__ rs = reinterpret_cast<const short*>(tp);
                const T* __restrict__ rw = reinterpret_cast<const T*>(tp + o_rw);
                T* __restrict__ G = gbuf + (w - w0) * gst;
                for (int c = lane; c < nc; c += CL) {
#pragma unroll
                    for (int i = 0; i < ROWS; ++i) {
                        if (i >= R) break;
                        T g = T(0);
                        if constexpr (KM > 0) {
#pragma unroll
                            for (int q = 0; q < KM; ++q) g += rw[i * KM + q] * blk[rs[i * KM + q] * np + c];
                        } else {  // dense aperture sampling of a coarse layer: runtime tap count
                            for (int q = 0; q < km; ++q) g += rw[i * km + q] * blk[rs[i * km + q] * np + c];
                        }
                        G[i * nc + c] = g;
                    }
                }
            }
        }
        __syncthreads();
        // ---- columns, WFS ascending ----
        if (worker) {
            for (int w = w0; w < w1; ++w) {
                const GDesc d = desc[w];
                const int nr = d.ihi - d.ilo, nc = d.jhi - d.jlo;
                if (nr <= 0) continue;
                const unsigned char* tp = cstage + (d.ctoff - ct0);
                const short* first = reinterpret_cast<const short*>(tp);
                const short* cidx = reinterpret_cast<const short*>(tp + o_idx);
                const T* cfr = reinterpret_cast<const T*>(tp + o_idx + align16(nc * 2));
                const T* G = gbuf + (w - w0) * gst;
                const int c0 = first[J], c1 = first[J + 2];
                if constexpr (KM == 0) {
                    for (int k2 = 0; k2 < ROWS; ++k2) {
                        if (k2 >= rows_pt) break;
                        const T* g = G + (i0 + k2) * nc;
                        T s = T(0);
                        for (int c = c0; c < c1; ++c) {
                            const T fr = cfr[c];
                            s += (cidx[c] == J ? T(1) - fr : fr) * g[c];
                        }
                        out[k2] += s;
                    }
                    continue;
                }
                constexpr int KQ = KM > 0 ? KM : 1;
                T wt[KQ];
                int cc[KQ];
#pragma unroll
                for (int q = 0; q < KQ; ++q) {
                    const int c = min(c0 + q, nc - 1);
                    const T fr = cfr[c];
                    wt[q] = c0 + q < c1 ? (cidx[c] == J ? T(1) - fr : fr) : T(0);
                    cc[q] = c;
                }
#pragma unroll
                for (int k2 = 0; k2 < ROWS; ++k2) {
                    if (k2 >= rows_pt) break;
                    const T* g = G + (i0 + k2) * nc;
                    T s = T(0);
#pragma unroll
                    for (int q = 0; q < KQ; ++q) s += wt[q] * g[cc[q]];
                    out[k2] += s;
                }
            }
        }
        __syncthreads();  // chunk consumed before the next one is staged
    }
    if (worker) {
#pragma unroll
        for (int k = 0; k < ROWS; ++k) {
            if (k >= rows_pt) break;
            y[(i0 + k) * side + J] = out[k];
        }
    }
}

// grid (side/grows, L, B): one CTA per gp.grows-row group of a layer; y nodal, row-major.
// Descriptors and chunk 0's tables are requested before the programmatic-launch
// wait (they are constant), the psi blocks after it.
template <typename T, int MINB>
__global__ void __launch_bounds__(256, MINB) k_gather(const GeoParams gp, const Bufs<T> bf) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ GDesc s_desc[kMaxW];
    __shared__ unsigned long long s_mbar;
    const int u = blockIdx.x, l = blockIdx.y, b = blockIdx.z;
    const int side = gp.side[l];
    const int R = side < gp.grows ? side : gp.grows;
    if (u * R >= side) return;
    const int tid = threadIdx.x;
    stamp(gp, 0);
    T* gbuf = reinterpret_cast<T*>(smem_raw);
    unsigned char* stage = smem_raw + align16(gp.gbuf_bytes);
    const T* psi = bf.psi + static_cast<size_t>(b) * gp.Nw;
    if (tid < 32) {
        if (tid < gp.W) {
            const int4* d = reinterpret_cast<const int4*>(gp.ti + gp.o_gd + ((l * kMaxGU + u) * kMaxW + tid) * kGDescInts);
            const int4 a = d[0], c = d[1], e = d[2];
            s_desc[tid] = GDesc{a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w, e.x, e.y, e.z, e.w};
        }
        if (tid == 0) {
            mbar_init(&s_mbar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncwarp();
        gather_issue<T>(gp, psi, s_desc, gp.gchunk[0], gp.gchunk[1], stage, &s_mbar, true, false);
    }
    pdl_wait();  // psi of the predecessor is complete
    pdl_launch_dependents();  // (after the wait: see the protocol in kernels.cuh)
    if (tid < 32) {
        gather_issue<T>(gp, psi, s_desc, gp.gchunk[0], gp.gchunk[1], stage, &s_mbar, false, true);
        __syncwarp();
        if (tid == 0) mbar_arrive(&s_mbar);
    }
    __syncthreads();  // descriptors visible
    stamp(gp, 12);
    T* y = bf.y + static_cast<size_t>(b) * gp.n + gp.coff[l] + static_cast<size_t>(u) * R * side;
#define FEWHA_GATHER_KM(ROWS)                                                                   \
    switch (gp.gather_km) {                                                                     \
        case 1: gather_group<T, 1, ROWS>(gp, psi, l, y, gbuf, stage, s_desc, &s_mbar); break;   \
        case 2: gather_group<T, 2, ROWS>(gp, psi, l, y, gbuf, stage, s_desc, &s_mbar); break;   \
        case 3: gather_group<T, 3, ROWS>(gp, psi, l, y, gbuf, stage, s_desc, &s_mbar); break;   \
        case 4: gather_group<T, 4, ROWS>(gp, psi, l, y, gbuf, stage, s_desc, &s_mbar); break;   \
        default: gather_group<T, 0, ROWS>(gp, psi, l, y, gbuf, stage, s_desc, &s_mbar); break;  \
    }
    if (gp.grows == 2) {
        FEWHA_GATHER_KM(2)
    } else if (gp.grows == 4) {
        FEWHA_GATHER_KM(4)
    } else {
        FEWHA_GATHER_KM(8)
    }
#undef FEWHA_GATHER_KM
    stamp(gp, 2);
}

// ---------------------------------------------------------------------------
// The direct gather (batched plans, gp.gather_direct): no row-contracted block in
// shared memory.  Per WFS a thread (layer column J, rows i0..i0+rows_pt-1) forms
//   h(r) = sum_b cw(J, b) psi(r, c0(J) + b)        for the psi rows r its rows touch,
//   y(i, J) += sum_a rw(i, a) h(r0(i) + a),
// the source runs [r0, r0 + KM) / [c0, c0 + KM) contiguous and zero-padded (host tables,
// engine.cu run_table).  r0 ascends with i, so the KM values h(r0(i) + .) live in a
// register ring that only moves forward: each psi value is read once per thread and
// instance, with no barrier between the two contractions and the staging budget all
// for psi blocks.  NI instances per CTA share the tables (instance ni's psi blocks at
// soff + ni * pad0, pad0 = the chunk's psi bytes per instance).
// ---------------------------------------------------------------------------
template <typename T, int NI>
__device__ __forceinline__ void gather_issue_direct(const GeoParams& gp, const T* psi_b, const GDesc* desc, int w0,
                                                    int w1, unsigned char* stage, unsigned long long* mbar,
                                                    bool tables, bool psi, int ninst) {
    const int lane = threadIdx.x;
    if (tables && lane == 31) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        bulk_g2s(stage, gp.gblob + desc[w0].rtoff, static_cast<unsigned>(gather_row_bytes(desc, w0, w1)), mbar);
    }
    if (tables && lane == 30) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        const unsigned bytes = static_cast<unsigned>(desc[w1 - 1].ctoff + desc[w1 - 1].cb - desc[w0].ctoff);
        bulk_g2s(stage + gather_row_bytes(desc, w0, w1), gp.gblob + desc[w0].ctoff, bytes, mbar);
    }
    const int nw = w1 - w0;
    if (!psi) return;
    for (int t = lane; t < nw * NI; t += 32) {
        const int ni = t / nw, w = w0 + (t - ni * nw);
        const GDesc d = desc[w];
        const int nr = d.ihi - d.ilo, np = gp.ns[w] + 1;
        if (nr > 0 && ni < ninst) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            const uintptr_t a = reinterpret_cast<uintptr_t>(psi_b + static_cast<size_t>(ni) * gp.Nw + d.src);
            const unsigned shift = static_cast<unsigned>(a & 15u);
            bulk_g2s(stage + d.soff + ni * d.pad0, reinterpret_cast<const void*>(a - shift),
                     round16(shift + nr * np * static_cast<unsigned>(sizeof(T))), mbar);
        }
    }
}

template <typename T, int KM, int ROWS, int NI>
__device__ void gather_direct_group(const GeoParams& gp, const T* __restrict__ psi_b, int l, T* __restrict__ y,
                                    unsigned char* stage, const GDesc* desc, unsigned long long* mbar, int ninst) {
    const int side = gp.side[l];
    const int R = side < ROWS ? side : ROWS;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int lside = ilog2(side);
    const int groups = min(nthr >> lside, R);
    const int rows_pt = R / groups;
    const int J = tid & (side - 1), grp = tid >> lside;
    const int i0 = grp * rows_pt;
    const bool worker = grp < groups;
    const int o_rw = align16(R * 2);     // row table: [r0 int16 R][rw R x KM]
    const int o_cw = align16(side * 2);  // column table: [c0 int16 side][cw side x KM]
    constexpr int RP = ROWS / 2;  // rows per thread: side <= 128 (host plan), 256 threads
    T out[NI][RP];
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
#pragma unroll
        for (int k = 0; k < RP; ++k) out[ni][k] = T(0);
    for (int k = 0; k < gp.nchunk; ++k) {
        const int w0 = gp.gchunk[k], w1 = gp.gchunk[k + 1];
        if (k > 0 && tid < 32) {
            gather_issue_direct<T, NI>(gp, psi_b, desc, w0, w1, stage, mbar, true, true, ninst);
            __syncwarp();
            if (tid == 0) mbar_arrive(mbar);
        }
        mbar_wait(mbar, static_cast<unsigned>(k & 1));
        const int rt0 = desc[w0].rtoff, ct0 = desc[w0].ctoff;
        const unsigned char* cstage = stage + gather_row_bytes(desc, w0, w1);
        if (worker) {
            for (int w = w0; w < w1; ++w) {
                const GDesc d = desc[w];
                const int nr = d.ihi - d.ilo, np = gp.ns[w] + 1, nc = d.jhi - d.jlo;
                if (nr <= 0) continue;
                const unsigned char* rt = stage + (d.rtoff - rt0);
                const unsigned char* ct = cstage + (d.ctoff - ct0);
                const int c0 = reinterpret_cast<const short*>(ct)[J];
                const T* __restrict__ cwp = reinterpret_cast<const T*>(ct + o_cw) + J * KM;
                T cw[KM];
                int cc[KM];
#pragma unroll
                for (int b = 0; b < KM; ++b) {
                    cw[b] = cwp[b];
                    cc[b] = min(c0 + b, nc - 1);
                }
                const T* blk[NI];
#pragma unroll
                for (int ni = 0; ni < NI; ++ni) {
                    const int nj = ni < ninst ? ni : 0;
                    const unsigned shift = static_cast<unsigned>(
                        reinterpret_cast<uintptr_t>(psi_b + static_cast<size_t>(nj) * gp.Nw + d.src) & 15u);
                    blk[ni] = reinterpret_cast<const T*>(stage + d.soff + nj * d.pad0 + shift) + d.jlo;
                }
                const short* __restrict__ r0t = reinterpret_cast<const short*>(rt);
                const T* __restrict__ rwt = reinterpret_cast<const T*>(rt + o_rw);
                auto hrow = [&](int r, T (&h)[NI]) {
                    const int ro = min(r, nr - 1) * np;
#pragma unroll
                    for (int ni = 0; ni < NI; ++ni) {
                        T s = T(0);
#pragma unroll
                        for (int b = 0; b < KM; ++b) s += cw[b] * blk[ni][ro + cc[b]];
                        h[ni] = s;
                    }
                };
                int cur = r0t[i0];
                T h[KM][NI];
#pragma unroll
                for (int a = 0; a < KM; ++a) hrow(cur + a, h[a]);
#pragma unroll
                for (int k2 = 0; k2 < RP; ++k2) {
                    if (k2 >= rows_pt) break;
                    const int r = r0t[i0 + k2];
                    while (cur < r) {  // advance the ring (first sources ascend with the row)
                        ++cur;
#pragma unroll
                        for (int a = 0; a + 1 < KM; ++a)
#pragma unroll
                            for (int ni = 0; ni < NI; ++ni) h[a][ni] = h[a + 1][ni];
                        hrow(cur + KM - 1, h[KM - 1]);
                    }
                    T wa[KM];
#pragma unroll
                    for (int a = 0; a < KM; ++a) wa[a] = rwt[(i0 + k2) * KM + a];
#pragma unroll
                    for (int ni = 0; ni < NI; ++ni) {
                        T s = T(0);
#pragma unroll
                        for (int a = 0; a < KM; ++a) s += wa[a] * h[a][ni];
                        out[ni][k2] += s;
                    }
                }
            }
        }
        __syncthreads();  // chunk consumed before the next one is staged
    }
    if (worker) {
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
            if (ni >= ninst) break;
#pragma unroll
            for (int k = 0; k < RP; ++k) {
                if (k >= rows_pt) break;
                y[static_cast<size_t>(ni) * gp.n + (i0 + k) * side + J] = out[ni][k];
            }
        }
    }
}

// grid (side/grows, L, ceil(B / NI)); plans with gp.gather_direct (compile-time taps, km <= 4)
template <typename T, int MINB, int NI>
__global__ void __launch_bounds__(256, MINB) k_gather_direct(const GeoParams gp, const Bufs<T> bf, int count, int late) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ GDesc s_desc[kMaxW];
    __shared__ unsigned long long s_mbar;
    const int u = blockIdx.x, l = blockIdx.y, b0 = blockIdx.z * NI;
    const int ninst = min(NI, count - b0);
    const int side = gp.side[l];
    const int R = side < gp.grows ? side : gp.grows;
    if (u * R >= side) return;
    const int tid = threadIdx.x;
    stamp(gp, 0);
    unsigned char* stage = smem_raw;
    const T* psi = bf.psi + static_cast<size_t>(b0) * gp.Nw;
    if (tid < 32) {
        if (tid < gp.W) {
            const int4* d = reinterpret_cast<const int4*>(gp.ti + gp.o_gd + ((l * kMaxGU + u) * kMaxW + tid) * kGDescInts);
            const int4 a = d[0], c = d[1], e = d[2];
            s_desc[tid] = GDesc{a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w, e.x, e.y, e.z, e.w};
        }
        if (tid == 0) {
            mbar_init(&s_mbar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncwarp();
        gather_issue_direct<T, NI>(gp, psi, s_desc, gp.gchunk[0], gp.gchunk[1], stage, &s_mbar, true, false, ninst);
    }
    pdl_wait();
    if (!late) pdl_launch_dependents();
    if (tid < 32) {
        gather_issue_direct<T, NI>(gp, psi, s_desc, gp.gchunk[0], gp.gchunk[1], stage, &s_mbar, false, true, ninst);
        __syncwarp();
        if (tid == 0) mbar_arrive(&s_mbar);
    }
    __syncthreads();
    stamp(gp, 12);
    T* y = bf.y + static_cast<size_t>(b0) * gp.n + gp.coff[l] + static_cast<size_t>(u) * R * side;
#define FEWHA_GATHER_D_KM(ROWS)                                                                                   \
    switch (gp.gather_km) {                                                                                       \
        case 1: gather_direct_group<T, 1, ROWS, NI>(gp, psi, l, y, stage, s_desc, &s_mbar, ninst); break;        \
        case 2: gather_direct_group<T, 2, ROWS, NI>(gp, psi, l, y, stage, s_desc, &s_mbar, ninst); break;        \
        case 3: gather_direct_group<T, 3, ROWS, NI>(gp, psi, l, y, stage, s_desc, &s_mbar, ninst); break;        \
        default: gather_direct_group<T, 4, ROWS, NI>(gp, psi, l, y, stage, s_desc, &s_mbar, ninst); break;       \
    }
    if (gp.grows == 2) {
        FEWHA_GATHER_D_KM(2)
    } else if (gp.grows == 4) {
        FEWHA_GATHER_D_KM(4)
    } else {
        FEWHA_GATHER_D_KM(8)
    }
#undef FEWHA_GATHER_D_KM
    if (late) pdl_launch_dependents();
    stamp(gp, 2);
}

// Deterministic sum of the dot partials of one iteration by warp 0: fixed
// per-lane strided order, fixed shuffle tree -- identical in every CTA.
__device__ __forceinline__ void warp_dot_sums(const double* rho_part, const double* mu_part, int n, double& rho,
                                              double& mu) {
    const int lane = threadIdx.x & 31;
    double a = 0.0, m = 0.0;
    for (int i = lane; i < n; i += 32) {
        a += rho_part[i];
        m += mu_part[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        m += __shfl_xor_sync(0xffffffffu, m, o);
    }
    rho = a;
    mu = m;
}

// ---------------------------------------------------------------------------
// Inverse kernel: grid (C, L, B), cluster (C,1,1).
//   kPlain: phi = W^-1 in;  kPcg: [update it-1] z = r/J, rho partial, phi = W^-1 z;
//   kFit: [final update] phi = W^-1 c
// Every rank prefetches its compact set of the operands, applies the fused
// update there (pcg.hpp:101-104) and forms z; the halo rows and the tail of z
// come from their owners after one cluster barrier.
// ---------------------------------------------------------------------------
template <typename T, int FLEN>
__device__ __forceinline__ void inv_phase(const GeoParams& gp, const Bufs<T>& bf, int mode, int it,
                                          unsigned char* smem_raw, int l, int b, int q, int C) {
    __shared__ double s_red[32];
    __shared__ double s_beta, s_alpha;
    __shared__ int s_apply;
    __shared__ unsigned long long s_mbar;
    const int S = gp.side[l];
    constexpr int H = FLEN / 2 - 1;
    __shared__ int s_off[2 * (kMaxLev + 1)];
    const LPlan p = make_plan(S, C, gp.ctail, q, H, s_off);
    const bool staged = gp.inv_staged != 0;
    const clay::InvSmem sm = clay::inv_smem(gp.maxside, C, gp.ctail, FLEN, static_cast<int>(sizeof(T)), gp.inv_staged);
    const int P = gp.maxside + 1;
    T* v[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) v[i] = reinterpret_cast<T*>(smem_raw + sm.v + i * sm.vstride);
    T *sr = v[0], *sj = v[1], *sp = v[2], *sq = v[3], *sc = v[4], *sm_ = v[5];  // staged operands
    T* z = reinterpret_cast<T*>(smem_raw + sm.z);
    T* x0 = reinterpret_cast<T*>(smem_raw + sm.x0);
    T* x1 = reinterpret_cast<T*>(smem_raw + sm.x1);
    T* aw = reinterpret_cast<T*>(smem_raw + sm.aw);
    T* tb = reinterpret_cast<T*>(smem_raw + sm.tb);
    T* tb2 = reinterpret_cast<T*>(smem_raw + sm.tb2);
    const size_t lbase = static_cast<size_t>(b) * gp.n + gp.coff[l];
    const int roff = clay::rank_off(S, C, gp.ctail, q), cnt = clay::owned_count(S, C, gp.ctail, q);
    const size_t vbase = lbase + roff;  // this rank's block of every coefficient-domain vector
    const int tid = threadIdx.x;
    const int slots = gp.L * C;  // dot partial slots per iteration
    const int upd = mode == kFit ? gp.iters : it;
    const bool may_update = mode != kPlain && upd > 0;
    stamp(gp, 0);
    if (tid == 0) {
        mbar_init(&s_mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (staged) prefetch_block(bf.jinv + gp.coff[l] + roff, sj, mode == kPlain ? 0 : cnt, &s_mbar, 0);  // constant
    // Before the wait (kernels.cuh protocol): r, c, p, q were last written by the
    // previous inverse (three launches back) or the previous frame -- except r at
    // it = 0, which the RHS forward kernel (the predecessor) updates.
    const bool r_early = mode == kFit || (mode == kPcg && it > 0);
    if (staged && mode != kPlain) {
        if (r_early) prefetch_block(bf.r + vbase, sr, cnt, &s_mbar, 0);
        prefetch_block(bf.c + vbase, sc, cnt, &s_mbar, 0);
        if (may_update) {
            prefetch_block(bf.p + vbase, sp, cnt, &s_mbar, 0);
            prefetch_block(bf.q + vbase, sq, cnt, &s_mbar, 0);
        }
    }
    Carry cin{};
    const int ci = b * (gp.iters + 1) + upd - 1;
    pdl_wait();  // the predecessor's outputs (Mz, mu partials; r at it = 0) are complete
    pdl_launch_dependents();
    if (may_update && tid == 0) cin = bf.carry[ci];
    // thread 0 issues every block and arrives at once (misaligned blocks: cooperative copies)
    if (!staged) {
        // operands read in place below
        sr = const_cast<T*>(mode == kPlain ? bf.in + vbase : bf.r + vbase);
        sj = const_cast<T*>(bf.jinv + gp.coff[l] + roff);
        sp = bf.p + vbase;
        sq = bf.q + vbase;
        sc = bf.c + vbase;
        sm_ = bf.mz + vbase;
    } else if (mode == kPlain) {
        prefetch_block(bf.in + vbase, sr, cnt, &s_mbar, 0);
    } else {
        if (!r_early) prefetch_block(bf.r + vbase, sr, cnt, &s_mbar, 0);
        if (may_update) prefetch_block(bf.mz + vbase, sm_, cnt, &s_mbar, 0);
    }
    if (tid == 0) mbar_arrive(&s_mbar);
    if (mode != kPlain && tid < 32) {
        // scalar recurrences of the iteration whose dots are complete (warp 0)
        ScalarStep st{};
        if (upd > 0) {
            double rho = 0.0, mu = 0.0;
            const size_t pi = (static_cast<size_t>(b) * gp.iters + (upd - 1)) * slots;
            warp_dot_sums(bf.rho_part + pi, bf.mu_part + pi, slots, rho, mu);
            if (tid == 0) {
                st = pcg_scalar_from_sums(gp, cin, rho, mu, upd - 1 == 0);
                if (l == 0 && q == 0) {
                    Carry o = st.out;
                    if (st.log) bf.rho_log[static_cast<size_t>(b) * gp.iters + o.nlog++] = st.logval;
                    bf.carry[ci + 1] = o;
                }
            }
        }
        if (tid == 0) {
            s_apply = st.apply;
            s_beta = st.beta;
            s_alpha = st.alpha;
        }
    }
    __syncthreads();  // scalars published, cooperative copies visible
    mbar_wait(&s_mbar, 0);
    stamp(gp, 1);
    double racc = 0.0;
    if (mode == kPlain) {
        for_owned(p, [&](int o, int zo, int) { z[zo] = sr[o]; });
    } else {
        const bool apply = s_apply != 0;
        const T beta = static_cast<T>(s_beta), alpha = static_cast<T>(s_alpha);
        T* pr = bf.r + vbase;  // (alias the operands when they are read in place)
        T* pp = bf.p + vbase;
        T* pq = bf.q + vbase;
        T* pc = bf.c + vbase;
        for_owned(p, [&](int o, int zo, int) {
            T rr = sr[o], cc = sc[o];
            const T ji = sj[o];
            if (apply) {  // pcg.hpp:101-104, z_old = r * (1/J)
                const T pn = rr * ji + beta * sp[o];
                const T qn = sm_[o] + beta * sq[o];
                cc = cc + alpha * pn;
                rr = rr - alpha * qn;
                pp[o] = pn;
                pq[o] = qn;
                pc[o] = cc;
                pr[o] = rr;
            }
            T vz;
            if (mode == kPcg) {
                vz = rr * ji;
                racc += static_cast<double>(rr) * static_cast<double>(vz);
            } else {
                vz = cc;
            }
            z[zo] = vz;
        });
    }
    if (mode == kPcg) {
        const double t = block_sum(racc, s_red);
        if (tid == 0) bf.rho_part[(static_cast<size_t>(b) * gp.iters + it) * slots + l * C + q] = t;
    }
    stamp(gp, 2);
    // rank 0 owns the whole T x T tail of z: it runs the tail levels before the
    // barrier (the other ranks read the tail output rows remotely at the first
    // distributed level); tail-only layers end here
    T* tl = tb;
    if (q == 0) {
        __syncthreads();  // z's tail complete
        tl = tail_inverse<T, FLEN>(gp, z + p.offH[p.nlev], p.T, tb, tb2);
    }
    if (p.nlev == 0) {
        if (q == 0) {
            T* __restrict__ phi = bf.phi + lbase;
            for (int e = tid; e < S * S; e += blockDim.x) phi[e] = tl[(e >> p.lsS) * (S + 1) + (e & (S - 1))];
        }
        return;
    }
    // every rank computes the same tail buffer choice (the tail level count is uniform)
    tl = tail_buffer<T, FLEN>(p.T, tb, tb2);
    {
        cl_sync();  // every rank's owned z is complete, rank 0's tail output too
        stamp(gp, 5);
        const int nthr = blockDim.x;
        for (int lv = 0; lv < p.nlev; ++lv) {
            const int s = S >> lv, h = s >> 1, k = h >> p.lC, m0 = q * k, nr = k + H;
            const int ls = ilog2(s), lh = ls - 1, lk = ilog2(k);
            const int oA = p.offH[lv], oD = oA + nr * h;
            const int na = H << lh, n = na + (H << ls);
            for (int e = tid; e < n; e += nthr) {
                const int i = e < na ? e >> lh : (e - na) >> ls;
                const int mm = (m0 - H + i) & (h - 1);
                const int own = mm >> lk, oi = (mm & (k - 1)) + H;
                const T* zr = rmt(z, own);
                if (e < na) {
                    const int c = e & (h - 1);
                    z[oA + i * h + c] = zr[oA + oi * h + c];
                } else {
                    const int c = (e - na) & (s - 1);
                    z[oD + i * s + c] = zr[oD + oi * s + c];
                }
            }
        }
        __syncthreads();
    }
    stamp(gp, 3);
    int outP = P;
    const T* out = cdwt_inverse<T, FLEN>(gp, p, z, x0, x1, aw, tl, P, &outP);
    stamp(gp, 9);
    const int R = clay::band_rows(S, C, gp.ctail, q), r0 = clay::band_row0(S, C, gp.ctail, q);
    T* __restrict__ phi = bf.phi + lbase + static_cast<size_t>(r0) * S;
    for (int e = tid; e < R * S; e += blockDim.x) phi[e] = out[(e >> p.lsS) * outP + (e & (S - 1))];
    cl_wait();  // no rank exits while its level outputs (or rank 0's tail) may still be read
}

template <typename T, int FLEN>
__global__ void __launch_bounds__(kClThreads) k_inv_cluster(const GeoParams gp, const Bufs<T> bf, int mode, int it) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cg::cluster_group cl = cg::this_cluster();
    inv_phase<T, FLEN>(gp, bf, mode, it, smem_raw, blockIdx.y, blockIdx.z, static_cast<int>(cl.block_rank()),
                       static_cast<int>(cl.num_blocks()));
    stamp(gp, 11);
}

// ---------------------------------------------------------------------------
// Forward kernel: grid (C, L, B), cluster (C,1,1).
//   band <- y (k_gather's sum_w P^T psi_w, or the bare wavelet op's input);
//   cluster W; epilogue per mode (kPlain / kApply / kPcg / kRhs) on the
//   rank's compact set.
//
// fit_term = 1: y is a fitting-term output sum_w P^T Gamma^T(...).  Its coarse
// (scale-0) coefficient is exactly zero in real arithmetic -- the bilinear
// weights of every aperture node sum to one and each subaperture's Gamma^T
// stencil (-x-y, x-y, -x+y, x+y; operators.hpp:182-185) sums to zero, so
// sum(y) = 0 and the periodic Daubechies coarse coefficient is sum(y)/2^J.
// The reference evaluates it as cancellation noise (~1e-16 relative in fp64,
// measured 8e-11 of ||c|| after the 1/(alpha d_0) amplification); an fp32
// evaluation inflates that noise to ~1e-2 of ||c||, so fp32 engines
// (gp.piston_exact) use the exact value.
// ---------------------------------------------------------------------------
template <typename T, int FLEN>
__device__ __forceinline__ void fwd_phase(const GeoParams& gp, const Bufs<T>& bf, int mode, int it, int fit_term,
                                          unsigned char* smem_raw, int l, int b, int q, int C) {
    __shared__ double s_red[32];
    __shared__ unsigned long long s_mbar[2];
    __shared__ double s_ad[16];  // alpha d_{l,scale} (operators.hpp:307-332)
    __shared__ int s_off[2 * (kMaxLev + 1)];
    const int S = gp.side[l];
    const LPlan p = make_plan(S, C, gp.ctail, q, 0, s_off);
    const int nthr = blockDim.x, tid = threadIdx.x;
    const clay::FwdSmem sm = clay::fwd_smem(gp.maxside, C, gp.ctail, FLEN, static_cast<int>(sizeof(T)), gp.tonly);
    const int P = gp.maxside + 1;
    T* x0 = reinterpret_cast<T*>(smem_raw + sm.x0);
    T* e0 = reinterpret_cast<T*>(smem_raw + sm.e0);
    T* e1 = reinterpret_cast<T*>(smem_raw + sm.e1);
    T* x1 = reinterpret_cast<T*>(smem_raw + sm.x1);
    T* f = reinterpret_cast<T*>(smem_raw + sm.f);
    T* tb = reinterpret_cast<T*>(smem_raw + sm.tb);
    T* tb2 = reinterpret_cast<T*>(smem_raw + sm.tb2);
    const int R = clay::band_rows(S, C, gp.ctail, q), r0 = clay::band_row0(S, C, gp.ctail, q);
    const size_t lbase = static_cast<size_t>(b) * gp.n + gp.coff[l];
    const int roff = clay::rank_off(S, C, gp.ctail, q), cnt = clay::owned_count(S, C, gp.ctail, q);
    const size_t vbase = lbase + roff;
    stamp(gp, 0);
    double my_ad = 0.0;
    if (tid >= 64 && tid < 64 + 16 && tid - 64 <= gp.lorder[l]) my_ad = gp.td[gp.ti[gp.o_reg + l] + tid - 64];
    if (tid == 0) {
        mbar_init(&s_mbar[0], 1);
        mbar_init(&s_mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (mode == kPcg) prefetch_block(bf.jinv + gp.coff[l] + roff, e1, cnt, &s_mbar[0], 0);  // constant
    // epilogue operands (this rank's blocks), requested before the wait (kernels.cuh
    // protocol: r / b / the operator input were written three or more launches back or
    // before the frame), consumed after the transform
    if (mode == kApply) {
        prefetch_block(bf.in + vbase, e0, cnt, &s_mbar[0], 0);
    } else if (mode == kPcg) {
        prefetch_block(bf.r + vbase, e0, cnt, &s_mbar[0], 0);
    } else if (mode == kRhs) {
        prefetch_block(bf.r + vbase, e0, cnt, &s_mbar[0], 0);
        prefetch_block(bf.b + vbase, e1, cnt, &s_mbar[0], 0);
    }
    if (tid == 0) mbar_arrive(&s_mbar[0]);
    pdl_wait();  // y of the predecessor (the gather) is complete
    pdl_launch_dependents();
    // the band of y (one bulk copy into x1's space, then into the odd-pitch x0); thread 0
    // issues every block and arrives at once (misaligned blocks: cooperative copies).
    // Shard groups: the band is the rank-order sum of the members' partials, read
    // directly from their buffers (the former k_exchange, fused here).
    if (bf.nsum > 0) {
        const size_t off = lbase + static_cast<size_t>(r0) * S;
        for (int e = tid; e < R * S; e += nthr) {
            T v = bf.ysum[0][off + e];
            for (int r = 1; r < bf.nsum; ++r) v += bf.ysum[r][off + e];
            x1[e] = v;
        }
    } else {
        prefetch_block(bf.y + lbase + static_cast<size_t>(r0) * S, x1, R * S, &s_mbar[1], 0);
    }
    if (tid == 0) mbar_arrive(&s_mbar[1]);
    if (tid >= 64 && tid < 64 + 16) s_ad[tid - 64] = my_ad;
    __syncthreads();  // s_ad, cooperative copies
    mbar_wait(&s_mbar[1], 0);
    stamp(gp, 1);
    for (int e = tid; e < R * S; e += nthr) x0[(e >> p.lsS) * P + (e & (S - 1))] = x1[e];
    __syncthreads();
    stamp(gp, 2);
    cdwt_forward<T, FLEN>(gp, p, x0, x1, P, f, tb, tb2);
    __syncthreads();
    stamp(gp, 9);
    mbar_wait(&s_mbar[0], 0);
    const double* ad = s_ad;
    const bool zero_piston = fit_term && gp.piston_exact;
    double macc = 0.0;
    T* __restrict__ out = bf.out + vbase;
    T* __restrict__ mz = bf.mz + vbase;
    T* __restrict__ pr = bf.r + vbase;
    T* __restrict__ pb = bf.b + vbase;
    const int o00 = (zero_piston && q == 0) ? p.off[p.nlev] : -1;  // tail (0,0)
    for_owned(p, [&](int o, int, int sc) {
        const T wy = o == o00 ? T(0) : f[o];
        if (mode == kPlain) {
            out[o] = wy;
        } else if (mode == kApply) {
            out[o] = wy + static_cast<T>(ad[sc]) * e0[o];
        } else if (mode == kPcg) {
            const T zz = e0[o] * e1[o];
            const T s = wy + static_cast<T>(ad[sc]) * zz;
            mz[o] = s;
            macc += static_cast<double>(s) * static_cast<double>(zz);
        } else {  // kRhs: r += b1 - b ; b = b1
            pr[o] = e0[o] + (wy - e1[o]);
            pb[o] = wy;
        }
    });
    if (mode == kPcg) {
        const double t = block_sum(macc, s_red);
        if (tid == 0) bf.mu_part[(static_cast<size_t>(b) * gp.iters + it) * (gp.L * C) + l * C + q] = t;
    }
    stamp(gp, 10);
}

template <typename T, int FLEN>
__global__ void __launch_bounds__(kClThreads) k_fwd_cluster(const GeoParams gp, const Bufs<T> bf, int mode, int it,
                                                      int fit_term) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cg::cluster_group cl = cg::this_cluster();
    fwd_phase<T, FLEN>(gp, bf, mode, it, fit_term, smem_raw, blockIdx.y, blockIdx.z, static_cast<int>(cl.block_rank()),
                       static_cast<int>(cl.num_blocks()));
    stamp(gp, 11);
}

// ---------------------------------------------------------------------------
// Barrier over the L x C CTAs of one instance (the fused kernel below; the
// cooperative launch makes them co-resident).  ctr: the instance's monotonic
// arrival counter, never reset -- arrival k of the e-th barrier on it reads
// old in [e n, (e+1) n), so the target needs no per-launch state.  Release /
// acquire at GPU scope order every CTA's global writes (Mz, r, b, mu partials)
// before the other CTAs' reads; the proxy fences let the inverse phase's TMA
// bulk copies read them and overwrite shared memory the forward phase used.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void instance_barrier(unsigned long long* ctr, unsigned long long n) {
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned long long old, v;
        asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;\n" : "=l"(old) : "l"(ctr) : "memory");
        const unsigned long long target = (old / n + 1) * n;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(ctr) : "memory");
        } while (v < target);
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    }
    __syncthreads();
}

// Fused forward(k) + inverse(k+1): the W of one apply_M (or of the RHS) and the
// next W^-1 with the PCG update between them in one launch.  The scalar
// recurrence needs the global mu = (s, z) of the forward epilogue, so the two
// phases meet at one barrier over the instance's L x C CTAs instead of a
// kernel boundary (grid (C, L, B), cluster (C,1,1), cooperative).  Shared
// memory is the union of the two phases' maps; the forward phase ends after
// its last cluster barrier, so no rank reads a peer's forward buffers once
// the instance barrier is passed.
template <typename T, int FLEN>
__global__ void __launch_bounds__(kClThreads) k_fwd_inv_cluster(const GeoParams gp, const Bufs<T> bf, int fmode, int fit,
                                                          int imode, int iit, int fit_term,
                                                          unsigned long long* bar) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cg::cluster_group cl = cg::this_cluster();
    const int q = static_cast<int>(cl.block_rank()), C = static_cast<int>(cl.num_blocks());
    fwd_phase<T, FLEN>(gp, bf, fmode, fit, fit_term, smem_raw, blockIdx.y, blockIdx.z, q, C);
    instance_barrier(bar + blockIdx.z, static_cast<unsigned long long>(gp.L) * C);
    inv_phase<T, FLEN>(gp, bf, imode, iit, smem_raw, blockIdx.y, blockIdx.z, q, C);
    stamp(gp, 11);
}

}  // namespace fewha_gpu
