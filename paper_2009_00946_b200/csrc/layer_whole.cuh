// Whole-layer transform kernels for batched plans (throughput).
//
// The cluster kernels (cluster.cuh) spread one layer's transform over C CTAs for the
// shortest single-frame chain; their cost is barriers and shared-memory latency
// chains, not arithmetic (profiles/r02_experiments.md: ~77 SM-us per 128^2 layer in a
// 64-instance step).  With many instances in flight the GPU is full anyway, so here one
// CTA owns a whole (layer, instance): the S x S layer sits in shared memory (pitch S+1)
// and every Mallat level is an in-place separable pass (wavelet.hpp:115-196) separated
// by CTA barriers only -- no cluster barriers, no DSMEM.  The fused PCG update (inverse)
// and the epilogues (forward) stream the coefficient-domain vectors straight from and to
// global memory in their rank-blocked cluster layout (clayout.hpp), so state is shared
// with the cluster kernels and the host converts it as before.
// Same operations and operation order as the cluster kernels per element; the dot
// partials of a layer go to slot l*C (the other C-1 slots of the layer are zero).
#pragma once

#include "cluster.cuh"

namespace fewha_gpu {

// Threads per CTA and resident CTAs per SM: the fp64 layer (132 KB at 128^2) allows one
// CTA per SM, so 512 threads; the fp32 layer (66 KB) three, at 256 threads each.
template <typename T>
struct Wl {
    static constexpr int threads = sizeof(T) == 8 ? 512 : 256;
    static constexpr int minb = sizeof(T) == 8 ? 1 : 3;
};

// Visit every coefficient of layer side S in rank-blocked HBM order (coeff_perm,
// engine.cu): f(o, row, col) with o the index inside the layer block and (row, col) its
// Mallat position.  Thread-strided inside each contiguous block (coalesced).
template <typename F>
__device__ __forceinline__ void for_layer(int S, int C, int D, F&& f) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int nl = clay::nlev(S, C, D), Tt = clay::tail(S, C, D), lC = ilog2(C);
    const int nq = clay::dist(S, C, D) ? C : 1;
    for (int q = 0; q < nq; ++q) {
        int o = clay::rank_off(S, C, D, q);
        for (int lv = 0; lv < nl; ++lv) {
            const int s = S >> lv, h = s >> 1, k = h >> lC, m0 = q * k;
            const int lh = ilog2(h), ls = ilog2(s);
            for (int e = tid; e < k * h; e += nthr) f(o + e, m0 + (e >> lh), h + (e & (h - 1)));
            o += k * h;
            for (int e = tid; e < k * s; e += nthr) f(o + e, h + m0 + (e >> ls), e & (s - 1));
            o += k * s;
        }
        if (q == 0) {
            const int lt = ilog2(Tt);
            for (int e = tid; e < Tt * Tt; e += nthr) f(o + e, e >> lt, e & (Tt - 1));
        }
    }
}

// Position of coefficient o (index in the layer's rank-blocked block, multiple of 4) for
// the flat walks below: the layer block is contiguous, so every thread takes groups of
// 4 at a fixed stride with independent loads (no per-block loop, whose global-memory
// latency would add up over the ~2C+1 blocks of a layer).
struct LayerMap {
    int S, C, nl, T, rank0, per;  // rank 0's block size (levels + tail), the other ranks' (levels)
    int lC;
    const int* off;  // [nl + 1] level offsets inside a rank block (no halo), in shared memory
};
// s_off: kMaxLev + 1 ints of shared memory; the caller syncs before layer_pos
__device__ __forceinline__ LayerMap layer_map(int S, int C, int D, int* s_off) {
    LayerMap m;
    m.S = S;
    m.C = C;
    m.nl = clay::nlev(S, C, D);
    m.T = clay::tail(S, C, D);
    m.lC = ilog2(C);
    if (static_cast<int>(threadIdx.x) <= m.nl) s_off[threadIdx.x] = clay::level_off(S, C, 0, threadIdx.x);
    m.off = s_off;
    m.per = clay::level_off(S, C, 0, m.nl);
    m.rank0 = m.per + m.T * m.T;
    return m;
}
__device__ __forceinline__ void layer_pos(const LayerMap& m, int o, int& row, int& col) {
    int q = 0, ol = o;
    if (o >= m.rank0) {
        q = 1 + (o - m.rank0) / m.per;
        ol = (o - m.rank0) - (q - 1) * m.per;
    }
    if (q == 0 && ol >= m.per) {  // rank 0's tail block
        const int e = ol - m.per;
        row = e / m.T;
        col = e - row * m.T;
        return;
    }
    int lv = 0;
    while (lv + 1 < m.nl && ol >= m.off[lv + 1]) ++lv;
    const int s = m.S >> lv, h = s >> 1, k = h >> m.lC, m0 = q * k;
    const int e = ol - m.off[lv];
    if (e < k * h) {
        row = m0 + e / h;
        col = h + (e & (h - 1));
    } else {
        const int e2 = e - k * h;
        row = h + m0 + e2 / s;
        col = e2 & (s - 1);
    }
}

// 4-vectors of the coefficient type (16-byte aligned groups: every block offset is a
// multiple of 4 elements)
template <typename T>
struct Vec4 {
    T v[4];
};
template <typename T>
__device__ __forceinline__ Vec4<T> ld4(const T* p) {
    Vec4<T> r;
    if constexpr (sizeof(T) == 8) {
        const double2 a = reinterpret_cast<const double2*>(p)[0], b = reinterpret_cast<const double2*>(p)[1];
        r.v[0] = a.x; r.v[1] = a.y; r.v[2] = b.x; r.v[3] = b.y;
    } else {
        const float4 a = *reinterpret_cast<const float4*>(p);
        r.v[0] = a.x; r.v[1] = a.y; r.v[2] = a.z; r.v[3] = a.w;
    }
    return r;
}
template <typename T>
__device__ __forceinline__ void st4(T* p, const Vec4<T>& r) {
    if constexpr (sizeof(T) == 8) {
        reinterpret_cast<double2*>(p)[0] = make_double2(r.v[0], r.v[1]);
        reinterpret_cast<double2*>(p)[1] = make_double2(r.v[2], r.v[3]);
    } else {
        *reinterpret_cast<float4*>(p) = make_float4(r.v[0], r.v[1], r.v[2], r.v[3]);
    }
}

// L2 prefetch of a contiguous range (cp.async.bulk.prefetch.L2): issued by the warps of
// a CTA in 16 KB pieces, no completion to wait for.  The forward kernels stream the
// epilogue's r toward L2 while the transform (shared memory and barriers, no HBM traffic)
// runs (batch 64: -0.4 % per step; prefetching the fused inverse's c, p, q as well: +1 %).
__device__ __forceinline__ void l2_prefetch(const void* p, size_t bytes) {
    const char* c = static_cast<const char*>(p);
    constexpr size_t kPiece = 16384;
    const size_t pieces = (bytes + kPiece - 1) / kPiece;
    for (size_t i = threadIdx.x; i < pieces; i += blockDim.x) {
        const size_t off = i * kPiece;
        const unsigned sz = static_cast<unsigned>(min(kPiece, bytes - off));
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(c + off), "r"(sz) : "memory");
    }
}

// The coarse corner (levels <= kWlCorner) runs as fused 2-D passes (tail_forward /
// tail_inverse, one CTA barrier per level instead of four) on a small scratch.
constexpr int kWlCorner = 16;
__host__ __device__ constexpr int wl_scratch_elems() { return 3 * kWlCorner * (kWlCorner + 1) + kWlCorner * kWlCorner; }
__host__ __device__ constexpr size_t whole_layer_smem(int maxside, int elem) {
    return (static_cast<size_t>(maxside) * (maxside + 1) + wl_scratch_elems()) * elem;
}

// Inverse: grid (L, B).  kPlain: phi = W^-1 in; kPcg: [update it-1] z = r/J, rho
// partial, phi = W^-1 z; kFit: [final update] phi = W^-1 c.
// MZS (fused forward + inverse, k_fwd_inv_layer): Mz of the fast path is read from the
// layer buffer, where the forward phase left it at each element's (row, col) -- the same
// thread owns the same element in both phases' flat walks.
template <typename T, int FLEN, bool MZS>
__device__ __forceinline__ void inv_layer_body(const GeoParams& gp, const Bufs<T>& bf, int mode, int it,
                                               unsigned char* smem_raw, const int l, const int b) {
    __shared__ double s_red[32];
    __shared__ double s_beta, s_alpha;
    __shared__ int s_apply;
    const int tid = threadIdx.x;
    const int S = gp.side[l], C = gp.ccl, D = gp.ctail, P = S + 1;
    T* buf = reinterpret_cast<T*>(smem_raw);
    const size_t lbase = static_cast<size_t>(b) * gp.n + gp.coff[l];
    const int slots = gp.L * C;
    const int upd = mode == kFit ? gp.iters : it;
    const int ci = b * (gp.iters + 1) + upd - 1;
    stamp(gp, 0);
    __shared__ int s_off[kMaxLev + 1];
    const LayerMap lm = layer_map(S, C, D, s_off);  // (published by the barrier below)
    pdl_wait();  // the predecessor's outputs (Mz, mu partials; r at it = 0) are complete
    pdl_launch_dependents();
    if (mode != kPlain && tid < 32) {  // scalar recurrences of the iteration whose dots are complete
        ScalarStep st{};
        if (upd > 0) {
            Carry cin{};
            if (tid == 0) cin = bf.carry[ci];
            double rho = 0.0, mu = 0.0;
            const size_t pi = (static_cast<size_t>(b) * gp.iters + (upd - 1)) * slots;
            warp_dot_sums(bf.rho_part + pi, bf.mu_part + pi, slots, rho, mu);
            if (tid == 0) {
                st = pcg_scalar_from_sums(gp, cin, rho, mu, upd - 1 == 0);
                if (l == 0) {
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
    __syncthreads();
    stamp(gp, 1);
    double racc = 0.0;
    if (mode == kPlain) {
        const T* in = bf.in + lbase;
        for_layer(S, C, D, [&](int o, int row, int col) { buf[row * P + col] = in[o]; });
    } else {
        const bool apply = s_apply != 0;
        const T beta = static_cast<T>(s_beta), alpha = static_cast<T>(s_alpha);
        T* pr = bf.r + lbase;
        T* pp = bf.p + lbase;
        T* pq = bf.q + lbase;
        T* pc = bf.c + lbase;
        const T* pm = bf.mz + lbase;
        const T* pj = bf.jinv + gp.coff[l];
        // one element (pcg.hpp:101-104, z_old = r * (1/J)); returns z
        auto upd1 = [&](T& rr, T& cc, T ji, T pv, T qv, T mv, T& pn, T& qn) {
            if (apply) {
                pn = rr * ji + beta * pv;
                qn = mv + beta * qv;
                cc = cc + alpha * pn;
                rr = rr - alpha * qn;
            }
            T vz;
            if (mode == kPcg) {
                vz = rr * ji;
                racc += static_cast<double>(rr) * static_cast<double>(vz);
            } else {
                vz = cc;
            }
            return vz;
        };
        const int nel = S * S;
        struct Ops {
            Vec4<T> rr, cc, ji, pv, qv, mv;
        };
        auto load = [&](int o) {
            Ops x{};
            x.rr = ld4(pr + o);
            x.cc = ld4(pc + o);
            x.ji = ld4(pj + o);
            if (apply) {
                x.pv = ld4(pp + o);
                x.qv = ld4(pq + o);
                if constexpr (!MZS) x.mv = ld4(pm + o);
            }
            return x;
        };
        auto finish = [&](int o, Ops& x) {
            int row, col;
            layer_pos(lm, o, row, col);
            Vec4<T> pn{}, qn{};
            if constexpr (MZS) {
                if (apply) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) x.mv.v[u] = buf[row * P + col + u];
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                buf[row * P + col + u] =
                    upd1(x.rr.v[u], x.cc.v[u], x.ji.v[u], x.pv.v[u], x.qv.v[u], x.mv.v[u], pn.v[u], qn.v[u]);
            if (apply) {
                st4(pp + o, pn);
                st4(pq + o, qn);
                st4(pc + o, x.cc);
                st4(pr + o, x.rr);
            }
        };
        if (S >= 4 && lm.T >= 4) {  // two groups per pass: both loads in flight before either is used
            const int step = 4 * blockDim.x;
            for (int o = 4 * tid; o < nel; o += 2 * step) {
                Ops a = load(o);
                const bool two = o + step < nel;
                Ops b2{};
                if (two) b2 = load(o + step);
                finish(o, a);
                if (two) finish(o + step, b2);
            }
        } else {
            for_layer(S, C, D, [&](int o, int row, int col) {
                T rr = pr[o], cc = pc[o], pn = T(0), qn = T(0);
                const T pv = apply ? pp[o] : T(0), qv = apply ? pq[o] : T(0), mv = apply ? pm[o] : T(0);
                buf[row * P + col] = upd1(rr, cc, pj[o], pv, qv, mv, pn, qn);
                if (apply) {
                    pp[o] = pn;
                    pq[o] = qn;
                    pc[o] = cc;
                    pr[o] = rr;
                }
            });
        }
    }
    if (mode == kPcg) {
        const double t = block_sum(racc, s_red);
        double* rp = bf.rho_part + (static_cast<size_t>(b) * gp.iters + it) * slots + l * C;
        if (tid < C) rp[tid] = tid == 0 ? t : 0.0;
    } else {
        __syncthreads();
    }
    stamp(gp, 2);
    int s0 = 2;
    if (S >= kWlCorner) {  // levels 2..kWlCorner: fused 2-D passes on the corner copy
        constexpr int K = kWlCorner;
        T* zt = buf + S * P;  // K x K coefficients (pitch K), then two (K+1)-pitch buffers
        T* b0 = zt + K * K;
        T* b1 = b0 + K * (K + 1);
        for (int e = tid; e < K * K; e += blockDim.x) zt[e] = buf[(e / K) * P + (e % K)];
        __syncthreads();
        const T* co = tail_inverse<T, FLEN>(gp, zt, K, b0, b1);
        for (int e = tid; e < K * K; e += blockDim.x) buf[(e / K) * P + (e % K)] = co[(e / K) * (K + 1) + (e % K)];
        __syncthreads();
        s0 = 2 * K;
    }
    for (int s = s0; s <= S; s <<= 1) {  // columns, then rows (wavelet.hpp:170-196)
        synthesis_lines<T, FLEN, true>(buf, P, s, s, gp);
        synthesis_lines<T, FLEN, false>(buf, P, s, s, gp);
        if (s == S / 2) stamp(gp, 3);
    }
    stamp(gp, 4);
    T* __restrict__ phi = bf.phi + lbase;
    const int ls = ilog2(S);
    for (int e = tid; e < S * S; e += blockDim.x) phi[e] = buf[(e >> ls) * P + (e & (S - 1))];
    stamp(gp, 5);
}

template <typename T, int FLEN>
__global__ void __launch_bounds__(Wl<T>::threads, Wl<T>::minb) k_inv_layer(const GeoParams gp, const Bufs<T> bf, int mode, int it) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    inv_layer_body<T, FLEN, false>(gp, bf, mode, it, smem_raw, blockIdx.x, blockIdx.y);
}

// Forward: grid (L, B).  buf <- y; W y in place; epilogue per mode (as fwd_phase).
// KEEP (fused forward + inverse): the kPcg fast path leaves Mz in the layer buffer at each
// element's (row, col) instead of storing it (the inverse phase reads it there).
template <typename T, int FLEN, bool KEEP>
__device__ __forceinline__ void fwd_layer_body(const GeoParams& gp, const Bufs<T>& bf, int mode, int it, int fit_term,
                                               unsigned char* smem_raw, const int l, const int b) {
    __shared__ double s_red[32];
    __shared__ double s_ad[16];  // alpha d_{l,scale} (operators.hpp:307-332)
    const int tid = threadIdx.x;
    const int S = gp.side[l], C = gp.ccl, D = gp.ctail, P = S + 1, ls = ilog2(S);
    T* buf = reinterpret_cast<T*>(smem_raw);
    const size_t lbase = static_cast<size_t>(b) * gp.n + gp.coff[l];
    stamp(gp, 0);
    if (tid < 16 && tid <= gp.lorder[l]) s_ad[tid] = gp.td[gp.ti[gp.o_reg + l] + tid];
    __shared__ int s_off[kMaxLev + 1];
    const LayerMap lm = layer_map(S, C, D, s_off);  // (published by the barrier after the y load)
    pdl_wait();  // y of the predecessor (the gather) is complete
    pdl_launch_dependents();
    const T* __restrict__ y = bf.y + lbase;
    stamp(gp, 1);
    constexpr int U = 4;
    if (S * S % (4 * U * Wl<T>::threads) == 0) {  // 4 vector loads in flight per thread per pass
        for (int e0 = 4 * tid; e0 < S * S; e0 += 4 * U * blockDim.x) {
            Vec4<T> v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = ld4(y + e0 + 4 * u * blockDim.x);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int e = e0 + 4 * u * blockDim.x;
                T* dst = buf + (e >> ls) * P + (e & (S - 1));
#pragma unroll
                for (int k = 0; k < 4; ++k) dst[k] = v[u].v[k];
            }
        }
    } else {
        for (int e = tid; e < S * S; e += blockDim.x) buf[(e >> ls) * P + (e & (S - 1))] = y[e];
    }
    __syncthreads();
    if (mode == kPcg || mode == kRhs) {  // the epilogue's r toward L2 during the transform
        const size_t lb = static_cast<size_t>(S) * S * sizeof(T);
        l2_prefetch(bf.r + lbase, lb);
    }
    stamp(gp, 2);
    const int slo = S >= kWlCorner ? 2 * kWlCorner : 2;
    for (int s = S; s >= slo; s >>= 1) {  // rows, then columns (wavelet.hpp:153-168)
        analysis_lines<T, FLEN, false>(buf, P, s, s, gp);
        analysis_lines<T, FLEN, true>(buf, P, s, s, gp);
        if (s == S) stamp(gp, 3);
    }
    if (S >= kWlCorner) {  // levels kWlCorner..2: fused 2-D passes, finals back into the corner
        constexpr int K = kWlCorner;
        T* fk = buf + S * P;  // K x K finals (pitch K), then two (K+1)-pitch buffers
        T* b0 = fk + K * K;
        T* b1 = b0 + K * (K + 1);
        tail_forward<T, FLEN>(gp, buf, P, K, b0, b1, fk);
        __syncthreads();
        for (int e = tid; e < K * K; e += blockDim.x) buf[(e / K) * P + (e % K)] = fk[e];
        __syncthreads();
    }
    stamp(gp, 4);
    const bool zero_piston = fit_term && gp.piston_exact;
    double macc = 0.0;
    T* __restrict__ out = bf.out + lbase;
    T* __restrict__ mz = bf.mz + lbase;
    T* __restrict__ pr = bf.r + lbase;
    T* __restrict__ pb = bf.b + lbase;
    const T* __restrict__ in = bf.in + lbase;
    const T* __restrict__ pj = bf.jinv + gp.coff[l];
    // one element: operand values x0 (in / r), x1 (jinv / b); results into y0 (out / mz / r), y1 (b)
    auto epi1 = [&](int row, int col, T x0, T x1, T& y0, T& y1) {
        const T wy = (zero_piston && (row | col) == 0) ? T(0) : buf[row * P + col];
        const int sc = bit_width(static_cast<unsigned>(max(row, col)));
        if (mode == kPlain) {
            y0 = wy;
        } else if (mode == kApply) {
            y0 = wy + static_cast<T>(s_ad[sc]) * x0;
        } else if (mode == kPcg) {
            const T zz = x0 * x1;
            const T s = wy + static_cast<T>(s_ad[sc]) * zz;
            y0 = s;
            macc += static_cast<double>(s) * static_cast<double>(zz);
        } else {  // kRhs: r += b1 - b ; b = b1
            y0 = x0 + (wy - x1);
            y1 = wy;
        }
    };
    const T* src0 = mode == kApply ? in : pr;                                  // (unused by kPlain)
    const T* src1 = mode == kPcg ? pj : pb;                                    // (kPcg, kRhs)
    T* dst0 = mode == kPcg ? mz : mode == kRhs ? pr : out;
    if (S >= 4 && lm.T >= 4) {
        const int step = 4 * blockDim.x;
        auto fin = [&](int o, const Vec4<T>& x0, const Vec4<T>& x1) {
            int row, col;
            layer_pos(lm, o, row, col);
            Vec4<T> y0{}, y1{};
#pragma unroll
            for (int u = 0; u < 4; ++u) epi1(row, col + u, x0.v[u], x1.v[u], y0.v[u], y1.v[u]);
            if (KEEP && mode == kPcg) {
#pragma unroll
                for (int u = 0; u < 4; ++u) buf[row * P + col + u] = y0.v[u];
            } else {
                st4(dst0 + o, y0);
            }
            if (mode == kRhs) st4(pb + o, y1);
        };
        for (int o = 4 * tid; o < S * S; o += 2 * step) {  // two groups per pass (loads in flight together)
            const bool two = o + step < S * S;
            Vec4<T> a0{}, a1{}, b0{}, b1{};
            if (mode != kPlain) {
                a0 = ld4(src0 + o);
                if (two) b0 = ld4(src0 + o + step);
            }
            if (mode == kPcg || mode == kRhs) {
                a1 = ld4(src1 + o);
                if (two) b1 = ld4(src1 + o + step);
            }
            fin(o, a0, a1);
            if (two) fin(o + step, b0, b1);
        }
    } else {
        for_layer(S, C, D, [&](int o, int row, int col) {
            T y0 = T(0), y1 = T(0);
            epi1(row, col, mode != kPlain ? src0[o] : T(0), (mode == kPcg || mode == kRhs) ? src1[o] : T(0), y0, y1);
            dst0[o] = y0;
            if (mode == kRhs) pb[o] = y1;
        });
    }
    if (mode == kPcg) {
        const double t = block_sum(macc, s_red);
        double* mp = bf.mu_part + (static_cast<size_t>(b) * gp.iters + it) * (gp.L * C) + l * C;
        if (tid < C) mp[tid] = tid == 0 ? t : 0.0;
    }
    stamp(gp, 5);
}

template <typename T, int FLEN>
__global__ void __launch_bounds__(Wl<T>::threads, Wl<T>::minb) k_fwd_layer(const GeoParams gp, const Bufs<T> bf, int mode, int it,
                                                             int fit_term) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    fwd_layer_body<T, FLEN, false>(gp, bf, mode, it, fit_term, smem_raw, blockIdx.x, blockIdx.y);
}

// Fused forward(k) + inverse(k+1) for batched plans: grid (L, B) of ordinary CTAs; the
// inverse phase's scalar recurrence needs every layer's mu partial, so the L layer CTAs
// of one instance meet at one barrier between the phases.  Co-residency without a
// cluster or a cooperative launch: each CTA takes a ticket in the order CTAs start and
// works on (layer, instance) = (t mod L, t / L) of it, so every ticket below the
// highest one belongs to a CTA that is running or done -- only the newest instance can
// be incomplete, and its missing CTAs start as soon as any other CTA exits (the device
// holds more than L CTAs at once).  ctr[B] is the ticket counter, ctr[0..B) the
// per-instance barrier counters; all monotonic (launches never overlap: the next fused
// launch waits on kernels that waited on this one).  Mz of the fast path never leaves
// shared memory (-2n per instance and iteration) and the kernel boundary between the
// phases is gone.  Same operations in the same order as k_fwd_layer + k_inv_layer:
// results are bitwise equal.
template <typename T, int FLEN>
__global__ void __launch_bounds__(Wl<T>::threads, Wl<T>::minb) k_fwd_inv_layer(const GeoParams gp, const Bufs<T> bf, int fmode,
                                                                 int fit, int imode, int iit, int fit_term,
                                                                 unsigned long long* ctr) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int s_t;
    const int B = gridDim.y, nb = gp.L * B;
    if (threadIdx.x == 0) s_t = static_cast<int>(atomicAdd(ctr + B, 1ull) % static_cast<unsigned long long>(nb));
    __syncthreads();
    const int t = s_t, l = t % gp.L, b = t / gp.L;
    fwd_layer_body<T, FLEN, true>(gp, bf, fmode, fit, fit_term, smem_raw, l, b);
    // the RHS pass (fmode kRhs) feeds only iteration 0's inverse, which reads its own
    // elements (same thread) and no scalars: no barrier
    if (fmode == kPcg) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned long long n = static_cast<unsigned long long>(gp.L);
            unsigned long long old, v;
            asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;\n" : "=l"(old) : "l"(ctr + b) : "memory");
            const unsigned long long target = (old / n + 1) * n;
            do {
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(ctr + b) : "memory");
            } while (v < target);
        }
    }
    __syncthreads();
    inv_layer_body<T, FLEN, true>(gp, bf, imode, iit, smem_raw, l, b);
}

}  // namespace fewha_gpu
