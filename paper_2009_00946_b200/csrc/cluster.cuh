// Cluster-distributed layer kernels.
//
// One thread-block cluster per (layer, instance): rank r of the cluster owns
// rows [r*R, r*R + R) of the 2^J x 2^J layer in its shared memory (pitch
// side+1, odd, so row walks and column walks are bank-conflict free).  The
// multilevel periodic Daubechies transform (wavelet.hpp:115-201) runs across
// the cluster:
//   * row passes touch only local rows;
//   * column passes read remote rows through distributed shared memory
//     (cooperative_groups map_shared_rank), stage results in registers across
//     one cluster barrier and write local rows -- 2 cluster barriers per
//     distributed level;
//   * levels with s <= R live entirely in rank 0 and finish there.
// Latency discipline: every global operand a kernel needs (PCG vectors of the
// band, gather tables, psi blocks) is requested up front with cp.async into
// shared memory, so each kernel pays one memory round trip per phase instead
// of one per loop iteration.  The adjoint propagation sum_w P^T psi_w is
// gathered straight into the band (separable, atomic-free, WFS ascending), so
// the forward transform never round-trips its input through HBM.
#pragma once

#include <cooperative_groups.h>

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

// ---- cp.async (LDGSTS) helpers ---------------------------------------------
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src));
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
template <typename T>
__device__ __forceinline__ void cp_async_elem(T* dst, const T* src) {
    if constexpr (sizeof(T) == 8) cp_async8(dst, src);
    else cp_async4(dst, src);
}
// contiguous bytes, cooperative over the CTA (sizes and addresses multiples of 4)
__device__ __forceinline__ void cp_async_bytes(void* dst, const void* src, int nbytes) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    auto* d = static_cast<unsigned char*>(dst);
    const auto* s = static_cast<const unsigned char*>(src);
    if (((reinterpret_cast<uintptr_t>(d) | reinterpret_cast<uintptr_t>(s) | static_cast<uintptr_t>(nbytes)) & 15) == 0) {
        for (int o = tid * 16; o < nbytes; o += nthr * 16) cp_async16(d + o, s + o);
    } else {
        for (int o = tid * 4; o < nbytes; o += nthr * 4) cp_async4(d + o, s + o);
    }
}

template <typename T>
struct Band {
    T* loc;            // this rank's band: R rows x P
    T* rem[kMaxC];     // every rank's band (generic DSMEM addresses)
    int R, P, rank, rsh;
    __device__ __forceinline__ T* row(int i) const { return rem[i >> rsh] + (i & (R - 1)) * P; }
};

__device__ __forceinline__ int ilog2(int v) { return 31 - __clz(v); }

// --- local passes over the first `nlines` lines of the top-left s x s block
//     (in place, register staged, CTA barriers; all sizes powers of two) -----
template <typename T, int FLEN, bool COL>
__device__ __forceinline__ void analysis_lines(T* buf, int P, int s, int nlines, const GeoParams& gp) {
    constexpr int SEGM = SegOf<T>::value;
    constexpr int WIN = 2 * SEGM + FLEN - 2;
    const int h = s >> 1, mask = s - 1;
    const int seg = h < SEGM ? h : SEGM;
    const int segs = h / seg;
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
    const int segs = h / seg;
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

// --- distributed column passes (s >= 2R: s/R ranks active) -----------------
// Forward: output row o of my band is approximation m = o (o < s/2) or detail
// m = o - s/2; rows x[(2m+k) & (s-1)] come from any rank.  A thread walks SEG
// consecutive output rows of one column with a sliding window of 2*SEG+FLEN-2
// remote reads.
template <typename T, int FLEN>
__device__ __forceinline__ void fwd_columns_cluster(const Band<T>& bd, int s, const GeoParams& gp,
                                                    cg::cluster_group& cl) {
    constexpr int SEG = 8;
    constexpr int WIN = 2 * SEG + FLEN - 2;
    const int h = s >> 1, mask = s - 1;
    const bool active = bd.rank < (s >> bd.rsh);
    const int seg = bd.R < SEG ? bd.R : SEG;
    const int segs = bd.R / seg;
    const int items = segs * s;
    const int ssh = ilog2(s);
    const int tid = threadIdx.x, nthr = blockDim.x;
    T out[2][SEG];
    int jj[2], oo[2];
    cl.sync();  // row pass results of every rank visible
    if (s == gp.maxside) stamp(gp, 4);
#pragma unroll
    for (int rep = 0; rep < 2; ++rep) {
        const int it = tid + rep * nthr;
        jj[rep] = it & (s - 1);
        oo[rep] = bd.rank * bd.R + (it >> ssh) * seg;
        if (!active || it >= items) continue;
        const int o0 = oo[rep];
        const bool detail = o0 >= h;
        const int m0 = detail ? o0 - h : o0;
        const int j = jj[rep];
        T win[WIN];
#pragma unroll
        for (int q = 0; q < WIN; ++q) {
            if (q >= 2 * seg + FLEN - 2) break;
            win[q] = bd.row((2 * m0 + q) & mask)[j];
        }
#pragma unroll
        for (int e = 0; e < SEG; ++e) {
            if (e >= seg) break;
            T acc = T(0);
#pragma unroll
            for (int k = 0; k < FLEN; ++k)
                acc += (detail ? Filt<T>::hi(gp, k) : Filt<T>::lo(gp, k)) * win[2 * e + k];
            out[rep][e] = acc;
        }
    }
    if (s == gp.maxside) stamp(gp, 5);
    cl.sync();  // every rank done reading before anyone overwrites
    if (s == gp.maxside) stamp(gp, 8);
#pragma unroll
    for (int rep = 0; rep < 2; ++rep) {
        const int it = tid + rep * nthr;
        if (!active || it >= items) continue;
        const int lr = oo[rep] - bd.rank * bd.R;
#pragma unroll
        for (int e = 0; e < SEG; ++e) {
            if (e >= seg) break;
            bd.loc[(lr + e) * bd.P + jj[rep]] = out[rep][e];
        }
    }
    __syncthreads();
}

// Inverse: output row t of my band from a-rows m and d-rows h+m, m = (t>>1)-kk.
template <typename T, int FLEN>
__device__ __forceinline__ void inv_columns_cluster(const Band<T>& bd, int s, const GeoParams& gp,
                                                    cg::cluster_group& cl) {
    constexpr int SEG = 4;  // output pairs per thread item
    constexpr int HF = FLEN / 2;
    const int h = s >> 1, hmask = h - 1;
    const bool active = bd.rank < (s >> bd.rsh);
    const int npairs = bd.R >> 1;
    const int seg = npairs < SEG ? npairs : SEG;
    const int segs = npairs / seg;
    const int items = segs * s;
    const int ssh = ilog2(s);
    const int tid = threadIdx.x, nthr = blockDim.x;
    T wa[2][SEG + HF - 1], wd[2][SEG + HF - 1];
    int jj[2], tt[2];
    cl.sync();  // previous level complete on every rank
#pragma unroll
    for (int rep = 0; rep < 2; ++rep) {
        const int it = tid + rep * nthr;
        jj[rep] = it & (s - 1);
        tt[rep] = bd.rank * bd.R + 2 * (it >> ssh) * seg;
        if (!active || it >= items) continue;
        const int m0 = tt[rep] >> 1;
#pragma unroll
        for (int i = 0; i < SEG + HF - 1; ++i) {
            if (i >= seg + HF - 1) break;
            const int m = (m0 - (HF - 1) + i) & hmask;
            wa[rep][i] = bd.row(m)[jj[rep]];
            wd[rep][i] = bd.row(h + m)[jj[rep]];
        }
    }
    cl.sync();  // reads done before local rows are overwritten
#pragma unroll
    for (int rep = 0; rep < 2; ++rep) {
        const int it = tid + rep * nthr;
        if (!active || it >= items) continue;
        const int lr = tt[rep] - bd.rank * bd.R;
#pragma unroll
        for (int u = 0; u < 2 * SEG; ++u) {
            if (u >= 2 * seg) break;
            T acc = T(0);
#pragma unroll
            for (int kk = 0; kk < HF; ++kk) {
                const int k = (u & 1) + 2 * kk;
                const int wi = (u >> 1) - kk + HF - 1;
                acc += wa[rep][wi] * Filt<T>::lo(gp, k) + wd[rep][wi] * Filt<T>::hi(gp, k);
            }
            bd.loc[(lr + u) * bd.P + jj[rep]] = acc;
        }
    }
    __syncthreads();
}

// Full transforms over the cluster.  `side` = layer side (power of two).
template <typename T, int FLEN>
__device__ void cluster_dwt_forward(const Band<T>& bd, int side, const GeoParams& gp, cg::cluster_group& cl) {
    int s = side;
    for (; s >= 2 * bd.R; s >>= 1) {
        if (bd.rank < (s >> bd.rsh)) analysis_lines<T, FLEN, false>(bd.loc, bd.P, s, bd.R, gp);
        if (s == side) stamp(gp, 3);
        fwd_columns_cluster<T, FLEN>(bd, s, gp, cl);
        if (s == side) stamp(gp, 6);
    }
    stamp(gp, 7);
    if (bd.rank == 0) {
        for (; s >= 2; s >>= 1) {
            analysis_lines<T, FLEN, false>(bd.loc, bd.P, s, s, gp);
            analysis_lines<T, FLEN, true>(bd.loc, bd.P, s, s, gp);
        }
    }
}

template <typename T, int FLEN>
__device__ void cluster_dwt_inverse(const Band<T>& bd, int side, const GeoParams& gp, cg::cluster_group& cl) {
    const int local_top = side < bd.R ? side : bd.R;
    if (bd.rank == 0) {
        for (int s = 2; s <= local_top; s <<= 1) {
            synthesis_lines<T, FLEN, true>(bd.loc, bd.P, s, s, gp);
            synthesis_lines<T, FLEN, false>(bd.loc, bd.P, s, s, gp);
        }
    }
    stamp(gp, 4);
    for (int s = 2 * bd.R; s <= side; s <<= 1) {
        inv_columns_cluster<T, FLEN>(bd, s, gp, cl);
        if (bd.rank < (s >> bd.rsh)) synthesis_lines<T, FLEN, false>(bd.loc, bd.P, s, bd.R, gp);
    }
}

template <typename T>
__device__ __forceinline__ Band<T> make_band(T* loc, int side, cg::cluster_group& cl) {
    Band<T> bd;
    bd.loc = loc;
    bd.R = side < 16 ? side : 16;
    bd.rsh = ilog2(bd.R);
    bd.P = side + 1;
    bd.rank = static_cast<int>(cl.block_rank());
    const int C = static_cast<int>(cl.num_blocks());
    for (int r = 0; r < kMaxC; ++r) bd.rem[r] = r < C ? cl.map_shared_rank(loc, r) : loc;
    return bd;
}

// ---------------------------------------------------------------------------
// Band gather of sum_w P_{w,l}^T psi_w (operators.hpp:241-260, WFS ascending).
// Per WFS, a host-built blob (GeoParams::gblob at o_gb) holds the padded
// separable gather tables: column taps (int16 source column relative to the
// WFS's first contributing column, weight) for every layer column and row taps
// (int16 absolute aperture row, weight) for every layer row.  WFS are staged
// in chunks that fit gp.chunk_bytes: descriptors first, then every psi block
// and table with cp.async, one wait, one barrier.  Then per thread (layer
// column J, a group of band rows): column contraction into a thread-private
// smem column, row contraction into registers.
// ---------------------------------------------------------------------------
constexpr int kRowsPerThreadMax = 16;

struct WDesc {
    int ilo, ihi, jlo, jhi;  // psi source block of this band
    int blob;                // byte offset of the (w,l) gather blob
    int pad[3];
};

template <typename T, int KM>
__device__ __forceinline__ void gather_contract(const T* blk, int nr, int nc, const short* cs, const T* cw,
                                                const short* rs, const T* rw, int ilo, int J, int i0, int rows_pt,
                                                T* hc, int nthr, int tid, T (&out)[kRowsPerThreadMax]) {
    int c[KM];
    T wx[KM];
#pragma unroll
    for (int q = 0; q < KM; ++q) {
        c[q] = cs[J * KM + q];
        wx[q] = cw[J * KM + q];
    }
    int ra = rs[i0 * KM] - ilo, rb = ra;
#pragma unroll
    for (int q = 0; q < KM; ++q) rb = max(rb, rs[(i0 + rows_pt - 1) * KM + q] - ilo);
    ra = min(max(ra, 0), nr - 1);
    rb = min(max(rb, ra), nr - 1);
    for (int r = ra; r <= rb; ++r) {
        const T* row = blk + r * nc;
        T h = T(0);
#pragma unroll
        for (int q = 0; q < KM; ++q) h += wx[q] * row[c[q]];
        hc[(r - ra) * nthr + tid] = h;
    }
#pragma unroll
    for (int k = 0; k < kRowsPerThreadMax; ++k) {
        if (k >= rows_pt) break;
        const short* rr = rs + (i0 + k) * KM;
        const T* ww = rw + (i0 + k) * KM;
        T s = T(0);
#pragma unroll
        for (int q = 0; q < KM; ++q) s += ww[q] * hc[min(max(rr[q] - ilo - ra, 0), rb - ra) * nthr + tid];
        out[k] += s;
    }
}

// shared-memory layout of one staged WFS: [block nr*nc T][col src side*KM short]
// [row src R*KM short][col w side*KM T][row w R*KM T], each 16-byte aligned
__device__ __forceinline__ int align16(int v) { return (v + 15) & ~15; }

// psi block staged as the contiguous full rows [ilo, ihi) of the WFS grid
// (np columns), fetched from the 16-byte aligned address at or below its start.
template <typename T>
__device__ __forceinline__ int staged_bytes(const WDesc& d, int side, int R, int KM, int np) {
    return align16((d.ihi - d.ilo) * np * static_cast<int>(sizeof(T)) + 16) + align16(side * KM * 2) +
           align16(R * KM * 2) + align16(side * KM * static_cast<int>(sizeof(T))) +
           align16(R * KM * static_cast<int>(sizeof(T)));
}

template <typename T>
__device__ void gather_band(const GeoParams& gp, const T* __restrict__ psi_b, int l, const Band<T>& bd, bool owner,
                            T* hc, unsigned char* stage, WDesc* desc, Bulk& bulk) {
    const int side = gp.side[l];
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int KM = gp.gather_km;
    const int groups = min(nthr / side, bd.R);  // threads per layer column
    const int rows_pt = bd.R / groups;          // band rows per thread
    const int J = tid & (side - 1), grp = tid >> ilog2(side);
    const int i0 = grp * rows_pt;
    const bool worker = owner && grp < groups;
    T out[kRowsPerThreadMax];
#pragma unroll
    for (int q = 0; q < kRowsPerThreadMax; ++q) out[q] = T(0);
    // descriptors of every WFS for this (layer, rank), one parallel load
    for (int w = tid; w < gp.W; w += nthr) {
        const int* bs = gp.ti + gp.o_bs + ((w * gp.L + l) * kMaxC + bd.rank) * 4;
        WDesc d;
        d.ilo = bs[0];
        d.ihi = bs[1];
        d.jlo = bs[2];
        d.jhi = bs[3];
        d.blob = gp.ti[gp.o_gb + w * gp.L + l];
        desc[w] = d;
    }
    __syncthreads();
    stamp(gp, 12);
    const unsigned char* blob = gp.gblob;
    int w0 = 0;
    while (w0 < gp.W) {
        int w1 = w0, used = 0;
        while (w1 < gp.W) {
            const int need = staged_bytes<T>(desc[w1], side, bd.R, KM, gp.ns[w1] + 1);
            if (w1 > w0 && used + need > gp.chunk_bytes) break;
            used += need;
            ++w1;
        }
        // ---- stage the chunk: thread 0 issues TMA bulk copies, everyone waits ----
        if (tid == 0) {
            bulk.begin();
            int off = 0;
            for (int w = w0; w < w1; ++w) {
                const WDesc d = desc[w];
                const int nr = d.ihi - d.ilo, np = gp.ns[w] + 1;
                unsigned char* p = stage + off;
                off += staged_bytes<T>(d, side, bd.R, KM, np);
                if (nr <= 0) continue;
                const T* src = psi_b + gp.woff[w] + d.ilo * np;
                const uintptr_t a = reinterpret_cast<uintptr_t>(src);
                const unsigned shift = static_cast<unsigned>(a & 15u);
                bulk.copy(p, reinterpret_cast<const void*>(a - shift), shift + nr * np * static_cast<unsigned>(sizeof(T)));
                p += align16(nr * np * static_cast<int>(sizeof(T)) + 16);
                const unsigned char* g = blob + d.blob;  // [col src][row src][col w][row w]
                const int cs_b = side * KM * 2, cw_b = side * KM * static_cast<int>(sizeof(T));
                const int g_rs = align16(cs_b), g_cw = g_rs + align16(cs_b), g_rw = g_cw + align16(cw_b);
                const int r0 = bd.rank * bd.R;
                bulk.copy(p, g, cs_b);
                p += align16(cs_b);
                bulk.copy(p, g + g_rs + r0 * KM * 2, bd.R * KM * 2);
                p += align16(bd.R * KM * 2);
                bulk.copy(p, g + g_cw, cw_b);
                p += align16(cw_b);
                bulk.copy(p, g + g_rw + r0 * KM * static_cast<int>(sizeof(T)), bd.R * KM * static_cast<int>(sizeof(T)));
            }
            bulk.commit();
        }
        stamp(gp, 13);
        bulk.wait();
        stamp(gp, 1);
        // ---- contract ----
        if (worker) {
            int off = 0;
            for (int w = w0; w < w1; ++w) {
                const WDesc d = desc[w];
                const int nr = d.ihi - d.ilo, np = gp.ns[w] + 1;
                const unsigned char* p = stage + off;
                off += staged_bytes<T>(d, side, bd.R, KM, np);
                if (nr <= 0) continue;
                const unsigned shift =
                    static_cast<unsigned>(reinterpret_cast<uintptr_t>(psi_b + gp.woff[w] + d.ilo * np) & 15u);
                const T* blk = reinterpret_cast<const T*>(p + shift) + d.jlo;  // (r, c) at blk[r*np + c]
                p += align16(nr * np * static_cast<int>(sizeof(T)) + 16);
                const short* cs = reinterpret_cast<const short*>(p);
                p += align16(side * KM * 2);
                const short* rs = reinterpret_cast<const short*>(p);
                p += align16(bd.R * KM * 2);
                const T* cw = reinterpret_cast<const T*>(p);
                p += align16(side * KM * static_cast<int>(sizeof(T)));
                const T* rw = reinterpret_cast<const T*>(p);
                if (KM == 2) gather_contract<T, 2>(blk, nr, np, cs, cw, rs, rw, d.ilo, J, i0, rows_pt, hc, nthr, tid, out);
                else if (KM == 3) gather_contract<T, 3>(blk, nr, np, cs, cw, rs, rw, d.ilo, J, i0, rows_pt, hc, nthr, tid, out);
                else gather_contract<T, 4>(blk, nr, np, cs, cw, rs, rw, d.ilo, J, i0, rows_pt, hc, nthr, tid, out);
            }
        }
        __syncthreads();  // chunk consumed before the next one is staged
        w0 = w1;
    }
    if (worker) {
#pragma unroll
        for (int k = 0; k < kRowsPerThreadMax; ++k) {
            if (k >= rows_pt) break;
            bd.loc[(i0 + k) * bd.P + J] = out[k];
        }
    }
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
// Phase A: grid (C, L, B), cluster (C,1,1); rank r owns band rows.
//   kPlain: phi = W^-1 in;  kPcg: [update it-1] z = r/J, rho partial, phi = W^-1 z;
//   kFit: [final update] phi = W^-1 c
// Shared memory: band | prefetched band slices of r, 1/J, p, q, c, Mz.
// ---------------------------------------------------------------------------
template <typename T, int FLEN>
__device__ __forceinline__ void inv_phase(const GeoParams& gp, const Bufs<T>& bf, int mode, int it, unsigned char* smem_raw, int l,
                          int b, cg::cluster_group& cl) {
    __shared__ double s_red[32];
    __shared__ double s_beta, s_alpha;
    __shared__ int s_apply;
    const int side = gp.side[l];
    const int lsd = ilog2(side);
    Band<T> bd = make_band<T>(reinterpret_cast<T*>(smem_raw), side, cl);
    const int C = static_cast<int>(cl.num_blocks());
    const bool owner = (bd.rank << bd.rsh) < side;  // holds rows of this layer
    const int r0 = bd.rank * bd.R;
    const int ne = owner ? bd.R * side : 0;
    const size_t base = static_cast<size_t>(b) * gp.n + gp.coff[l] + static_cast<size_t>(r0) * side;
    const size_t jbase = gp.coff[l] + static_cast<size_t>(r0) * side;
    const int nthr = blockDim.x, tid = threadIdx.x;
    const int slots = gp.L * C;  // dot partial slots per iteration
    stamp(gp, 0);
    // prefetch region after the band (16-byte aligned)
    T* pre = reinterpret_cast<T*>(smem_raw + align16(bd.R * bd.P * static_cast<int>(sizeof(T))));
    const int nb = ne * static_cast<int>(sizeof(T));
    T *sr = pre, *sj = pre + ne, *sp = pre + 2 * ne, *sq = pre + 3 * ne, *sc = pre + 4 * ne, *sm = pre + 5 * ne;
    const int upd = mode == kFit ? gp.iters : it;
    const bool may_update = mode != kPlain && upd > 0;
    __shared__ unsigned long long s_mbar;
    Bulk bulk{&s_mbar, 0};
    bulk.init();
    if (tid == 0) {  // band slices by TMA bulk copy (16 KiB each at J=7 fp64)
        bulk.begin();
        if (nb > 0 && mode != kPlain) bulk.copy(sj, bf.jinv + jbase, nb);  // constant: before the wait
    }
    pdl_wait();  // the predecessor's outputs (r, c, p, q, Mz, dot partials) are complete
    if (tid == 0) {
        if (nb > 0) {
            if (mode == kPlain) {
                bulk.copy(sr, bf.in + base, nb);
            } else {
                bulk.copy(sr, bf.r + base, nb);
                bulk.copy(sc, bf.c + base, nb);
                if (may_update) {
                    bulk.copy(sp, bf.p + base, nb);
                    bulk.copy(sq, bf.q + base, nb);
                    bulk.copy(sm, bf.mz + base, nb);
                }
            }
        }
        bulk.commit();
    }
    if (mode != kPlain && tid < 32) {
        // scalar recurrences of the iteration whose dots are complete (warp 0)
        ScalarStep st{};
        if (upd > 0) {
            double rho = 0.0, mu = 0.0;
            const int ci = b * (gp.iters + 1) + upd - 1;
            const size_t pi = (static_cast<size_t>(b) * gp.iters + (upd - 1)) * slots;
            warp_dot_sums(bf.rho_part + pi, bf.mu_part + pi, slots, rho, mu);
            if (tid == 0) {
                st = pcg_scalar_from_sums(gp, bf.carry[ci], rho, mu, upd - 1 == 0);
                if (l == 0 && bd.rank == 0) {
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
    bulk.wait();
    __syncthreads();
    stamp(gp, 1);
    if (mode == kPlain) {
        for (int e = tid; e < ne; e += nthr) bd.loc[(e >> lsd) * bd.P + (e & (side - 1))] = sr[e];
    } else {
        const bool apply = s_apply != 0;
        const T beta = static_cast<T>(s_beta), alpha = static_cast<T>(s_alpha);
        double racc = 0.0;
        T* __restrict__ pr = bf.r + base;
        T* __restrict__ pp = bf.p + base;
        T* __restrict__ pq = bf.q + base;
        T* __restrict__ pc = bf.c + base;
        for (int e = tid; e < ne; e += nthr) {
            T rr = sr[e], cc = sc[e];
            const T ji = sj[e];
            if (apply) {  // pcg.hpp:101-104, z_old = r * (1/J)
                const T pn = rr * ji + beta * sp[e];
                const T qn = sm[e] + beta * sq[e];
                cc = cc + alpha * pn;
                rr = rr - alpha * qn;
                pp[e] = pn;
                pq[e] = qn;
                pc[e] = cc;
                pr[e] = rr;
            }
            T v;
            if (mode == kPcg) {
                v = rr * ji;
                racc += static_cast<double>(rr) * static_cast<double>(v);
            } else {
                v = cc;
            }
            bd.loc[(e >> lsd) * bd.P + (e & (side - 1))] = v;
        }
        if (mode == kPcg) {
            const double t = block_sum(racc, s_red);
            if (tid == 0)
                bf.rho_part[(static_cast<size_t>(b) * gp.iters + it) * slots + l * C + bd.rank] = t;
        }
    }
    __syncthreads();
    stamp(gp, 2);
    cluster_dwt_inverse<T, FLEN>(bd, side, gp, cl);
    __syncthreads();
    stamp(gp, 9);
    for (int e = tid; e < ne; e += nthr) bf.phi[base + e] = bd.loc[(e >> lsd) * bd.P + (e & (side - 1))];
}

template <typename T, int FLEN>
__global__ void __launch_bounds__(256) k_inv_cluster(const GeoParams gp, const Bufs<T> bf, int mode, int it) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cg::cluster_group cl = cg::this_cluster();
    pdl_launch_dependents();
    inv_phase<T, FLEN>(gp, bf, mode, it, smem_raw, blockIdx.y, blockIdx.z, cl);
    cl.sync();  // no rank exits while its shared memory may still be read
    stamp(gp, 11);
}

// ---------------------------------------------------------------------------
// Phase C: grid (C, L, B), cluster (C,1,1).
//   band <- sum_w P^T psi_w (gather=1) or y (gather=0, bare wavelet op);
//   cluster W; epilogue per mode (kPlain / kApply / kPcg / kRhs).
// Shared memory: band | epilogue prefetch (2 slices) | hc | staged chunk.
//
// gather = 1: y is a fitting-term output sum_w P^T Gamma^T(...).  Its coarse
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
__device__ __forceinline__ void fwd_phase(const GeoParams& gp, const Bufs<T>& bf, int mode, int it, int gather,
                          unsigned char* smem_raw, int l, int b, cg::cluster_group& cl) {
    __shared__ double s_red[32];
    __shared__ WDesc s_desc[kMaxW];
    const int side = gp.side[l];
    const int lsd = ilog2(side);
    T* band = reinterpret_cast<T*>(smem_raw);
    Band<T> bd = make_band<T>(band, side, cl);
    const int C = static_cast<int>(cl.num_blocks());
    const bool owner = (bd.rank << bd.rsh) < side;
    const int r0 = bd.rank * bd.R;
    const int ne = owner ? bd.R * side : 0;
    const size_t base = static_cast<size_t>(b) * gp.n + gp.coff[l] + static_cast<size_t>(r0) * side;
    const size_t jbase = gp.coff[l] + static_cast<size_t>(r0) * side;
    const int nthr = blockDim.x, tid = threadIdx.x;
    stamp(gp, 0);
    const int band_b = align16(bd.R * bd.P * static_cast<int>(sizeof(T)));
    const int slice_b = align16(bd.R * gp.maxside * static_cast<int>(sizeof(T)));
    T* e0 = reinterpret_cast<T*>(smem_raw + band_b);
    T* e1 = reinterpret_cast<T*>(smem_raw + band_b + slice_b);
    T* hc = reinterpret_cast<T*>(smem_raw + band_b + 2 * slice_b);
    unsigned char* stage = smem_raw + band_b + 2 * slice_b + align16(gp.hc_rows * nthr * static_cast<int>(sizeof(T)));
    const int nb = ne * static_cast<int>(sizeof(T));
    __shared__ unsigned long long s_mbar[2];
    Bulk epi{&s_mbar[0], 0}, stg{&s_mbar[1], 0};
    epi.init();
    stg.init();
    pdl_wait();  // psi / y / r / b of the predecessor kernels are complete
    // epilogue operands by TMA bulk copy, requested now, consumed after the transform
    if (tid == 0) {
        epi.begin();
        if (nb > 0) {
            if (mode == kApply) {
                epi.copy(e0, bf.in + base, nb);
            } else if (mode == kPcg) {
                epi.copy(e0, bf.r + base, nb);
                epi.copy(e1, bf.jinv + jbase, nb);
            } else if (mode == kRhs) {
                epi.copy(e0, bf.r + base, nb);
                epi.copy(e1, bf.b + base, nb);
            }
        }
        epi.commit();
    }
    if (!gather) {
        if (tid == 0) {
            stg.begin();
            if (nb > 0) stg.copy(hc, bf.y + base, nb);
            stg.commit();
        }
        stg.wait();
        for (int e = tid; e < ne; e += nthr) bd.loc[(e >> lsd) * bd.P + (e & (side - 1))] = hc[e];
    } else {
        gather_band<T>(gp, bf.psi + static_cast<size_t>(b) * gp.Nw, l, bd, owner, hc, stage, s_desc, stg);
    }
    __syncthreads();
    stamp(gp, 2);
    cluster_dwt_forward<T, FLEN>(bd, side, gp, cl);
    __syncthreads();
    stamp(gp, 9);
    epi.wait();
    const double* ad = gp.td + gp.ti[gp.o_reg + l];
    double macc = 0.0;
    for (int e = tid; e < ne; e += nthr) {
        const int i = r0 + (e >> lsd), j = e & (side - 1);
        const size_t g = base + e;
        const T wy = (gather && gp.piston_exact && i == 0 && j == 0) ? T(0) : bd.loc[(e >> lsd) * bd.P + j];
        if (mode == kPlain) {
            bf.out[g] = wy;
        } else if (mode == kApply) {
            const T adv = static_cast<T>(ad[bit_width(static_cast<unsigned>(max(i, j)))]);
            bf.out[g] = wy + adv * e0[e];
        } else if (mode == kPcg) {
            const T adv = static_cast<T>(ad[bit_width(static_cast<unsigned>(max(i, j)))]);
            const T z = e0[e] * e1[e];
            const T s = wy + adv * z;
            bf.mz[g] = s;
            macc += static_cast<double>(s) * static_cast<double>(z);
        } else {  // kRhs: r += b1 - b ; b = b1
            bf.r[g] = e0[e] + (wy - e1[e]);
            bf.b[g] = wy;
        }
    }
    if (mode == kPcg) {
        const double t = block_sum(macc, s_red);
        if (tid == 0)
            bf.mu_part[(static_cast<size_t>(b) * gp.iters + it) * (gp.L * C) + l * C + bd.rank] = t;
    }
    stamp(gp, 10);
}

template <typename T, int FLEN>
__global__ void __launch_bounds__(256) k_fwd_cluster(const GeoParams gp, const Bufs<T> bf, int mode, int it,
                                                      int gather) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cg::cluster_group cl = cg::this_cluster();
    pdl_launch_dependents();
    fwd_phase<T, FLEN>(gp, bf, mode, it, gather, smem_raw, blockIdx.y, blockIdx.z, cl);
    cl.sync();
    stamp(gp, 11);
}

}  // namespace fewha_gpu
