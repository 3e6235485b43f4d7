// Ownership layout of the cluster-distributed layer transforms (host + device).
//
// A layer of side S (power of two) is transformed by one cluster of C CTAs
// (ranks).  Distributed Mallat levels are s = S, S/2, ..., 2C (when S >= 2C);
// at level s every rank q owns the k = s/(2C) filter positions
// m in [q k, q k + k) and therefore
//   * needs the 2k input rows [2 q k, 2 q k + 2k) of the level -- exactly the
//     rows it produced as approximation rows one level finer, so only the
//     FLEN-2 halo rows after them cross distributed shared memory;
//   * finalises the coefficients
//       A: rows [m0, m0+k), columns [h, s)   (row details of approximation rows)
//       D: rows [h+m0, h+m0+k), columns [0, s)
//     which is the set it also owns in the inverse transform and in the PCG
//     vector updates (its "compact" set, stored level by level: A block then
//     D block, each row-major).
// The levels below 2C (the T x T top-left block, T = C) are the tail, finished
// by rank 0.  Layers with S < 2C are tail-only (T = S) on rank 0.
// A halo variant of the compact layout reserves H extra rows in front of every
// level block (the inverse transform's filter support, H = FLEN/2 - 1).
//
// The coefficient-domain vectors (c, b, r, p, q, Mz, J, operator in/out) are
// stored RANK-BLOCKED in HBM: per layer, rank 0's compact set, then rank 1's,
// ... (no padding), so every rank reads and writes one contiguous block.  The
// host converts to and from the reference's Mallat order at the API boundary.
#pragma once

#ifdef __CUDACC__
#define FEWHA_HD __host__ __device__ __forceinline__
#else
#define FEWHA_HD inline
#endif

namespace fewha_gpu {
namespace clay {

// log2 of a power of two (C, S and all level sizes are powers of two)
FEWHA_HD int lg2(int v) {
#ifdef __CUDA_ARCH__
    return 31 - __clz(v);
#else
    int r = 0;
    while ((1 << (r + 1)) <= v) ++r;
    return r;
#endif
}
// Tail size D (a power of two, C <= D): levels s >= 2D are distributed over
// the cluster, the D x D tail (levels below) runs on rank 0 inside one CTA --
// the coarse levels cost a cluster barrier each but almost no arithmetic, so
// finishing them locally is cheaper.  Layers with S < 2D are tail-only (whole
// layer on rank 0).  The host picks D = 4C (measured best), else 2C, else C, whose kernels
// fit in shared memory (GeoParams::ctail).
FEWHA_HD bool dist(int S, int C, int D) { return S >= 2 * D; }
FEWHA_HD int tail(int S, int C, int D) { return dist(S, C, D) ? D : S; }
FEWHA_HD int nlev(int S, int C, int D) {
    int n = 0;
    for (int s = S; dist(s, C, D); s >>= 1) ++n;
    return n;
}
// band rows of rank q at level S (input of the forward gather, output of the inverse)
FEWHA_HD int band_rows(int S, int C, int D, int q) { return dist(S, C, D) ? S >> lg2(C) : (q == 0 ? S : 0); }
FEWHA_HD int band_row0(int S, int C, int D, int q) { return dist(S, C, D) ? q * (S >> lg2(C)) : 0; }
// offset (elements) of level lv's block in the compact layout with H halo rows;
// lv == nlev gives the tail block's offset
FEWHA_HD int level_off(int S, int C, int H, int lv) {  // (independent of D)
    int off = 0;
    const int lc = lg2(C);
    for (int i = 0; i < lv; ++i) {
        const int s = S >> i, h = s >> 1, k = h >> lc;
        off += (k + H) * (h + s);
    }
    return off;
}
// total compact size (elements), tail block always reserved
FEWHA_HD int compact_size(int S, int C, int D, int H) {
    const int T = tail(S, C, D);
    return level_off(S, C, H, nlev(S, C, D)) + T * T;
}
// elements rank q owns, and the offset of its block inside the layer (rank-blocked order)
FEWHA_HD int owned_count(int S, int C, int D, int q) {
    const int T = tail(S, C, D);
    if (!dist(S, C, D)) return q == 0 ? T * T : 0;
    return level_off(S, C, 0, nlev(S, C, D)) + (q == 0 ? T * T : 0);
}
FEWHA_HD int rank_off(int S, int C, int D, int q) {
    if (q == 0) return 0;
    const int T = tail(S, C, D);
    if (!dist(S, C, D)) return T * T;
    return q * level_off(S, C, 0, nlev(S, C, D)) + T * T;
}

FEWHA_HD int a16(int v) { return (v + 15) & ~15; }

// Shared-memory map of the forward kernel (bytes from the dynamic base).
//   x0: level-S input band (+ FLEN-2 halo rows), e0/e1: epilogue operands
//   (compact), x1: ping-pong level buffer (first the bulk-copied y band),
//   f: finals (compact), tb/tb2: tail ping-pong.
struct FwdSmem {
    int x0, e0, e1, x1, f, tb, tb2, total;
};
// largest tail block of any layer (distributed tail D, or a tail-only layer of side < 2D)
FEWHA_HD int tail_max(int maxside, int C, int D) {
    const int Tm = tail(maxside, C, D), tonly = maxside < D ? maxside : D;
    return Tm > tonly ? Tm : tonly;
}
// tonly: the largest tail-only layer side of the geometry (0: none)
FEWHA_HD FwdSmem fwd_smem(int maxside, int C, int D, int flen, int elem, int tonly) {
    FwdSmem m{};
    const int P = maxside + 1, R = band_rows(maxside, C, D, 0);
    const int xrows = (R + flen - 2) > tonly ? (R + flen - 2) : tonly;  // tail-only layers use the band too
    const int xb = a16(xrows * P * elem), cb = a16(compact_size(maxside, C, D, 0) * elem);
    m.x0 = 0;
    m.e0 = xb;
    m.e1 = m.e0 + cb;
    m.x1 = m.e1 + cb;
    m.f = m.x1 + xb;
    m.tb = m.f + cb;
    const int Tb = tail_max(maxside, C, D);
    m.tb2 = m.tb + a16(Tb * (Tb + 1) * elem);
    m.total = m.tb2 + a16(Tb * (Tb + 1) * elem);
    return m;
}

// Shared-memory map of the inverse kernel (bytes).
//   v: 6 prefetched compact vectors (r, 1/J, p, q, c, Mz or the operator input),
//   z: the transform input in the halo layout, x0/x1: ping-pong level outputs,
//   aw: assembled approximation rows of one level, tb/tb2: tail ping-pong.
struct InvSmem {
    int v, vstride, z, x0, x1, aw, tb, tb2, total;
};
// staged = 0: the six vectors are read straight from global memory (batch mode:
// the smaller footprint doubles the resident clusters per SM)
FEWHA_HD InvSmem inv_smem(int maxside, int C, int D, int flen, int elem, int staged = 1) {
    InvSmem m{};
    const int P = maxside + 1, R = band_rows(maxside, C, D, 0), H = flen / 2 - 1;
    m.vstride = staged ? a16(compact_size(maxside, C, D, 0) * elem) : 0;
    m.v = 0;
    m.z = 6 * m.vstride;
    m.x0 = m.z + a16(compact_size(maxside, C, D, H) * elem);
    m.x1 = m.x0 + a16(R * P * elem);
    m.aw = m.x1 + a16(R * P * elem);
    const int kmax = dist(maxside, C, D) ? maxside >> (lg2(C) + 1) : 0;
    m.tb = m.aw + a16((kmax + H) * maxside * elem);
    // tb2 aliases x1: the tail is finished (and, if its output sits in tb2, consumed
    // by the first distributed level, which writes x0) before x1 is first written
    const int Tb = tail_max(maxside, C, D);
    const int tbb = a16(Tb * (Tb + 1) * elem);
    if (tbb <= a16(R * P * elem)) {
        m.tb2 = m.x1;
        m.total = m.tb + tbb;
    } else {  // tail larger than a band: no aliasing
        m.tb2 = m.tb + tbb;
        m.total = m.tb2 + tbb;
    }
    return m;
}

}  // namespace clay
}  // namespace fewha_gpu
