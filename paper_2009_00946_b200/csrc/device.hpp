// Shared host/device definitions for the FEWHA sm_100a kernels.
//
// HBM layout (per instance b of a batch; all vectors batch-major, contiguous):
//   coefficient-domain vectors c, b, r, p, q, Mz, J, and the nodal layer
//   grids phi (W^-1 z) and y (sum_w P_w^T psi_w): [b][n], per layer a
//   2^J x 2^J row-major block at coff[l]            (operators.hpp:67-91)
//   psi (Gamma^T C^-1 Gamma P phi per WFS): [b][N_w], (n_s+1)^2 at woff[w]
//   slopes: [b][S] fp64, [sx | sy] per WFS at moff[w]   (operators.hpp:35-65)
//   DM commands a_prev2, a_prev, a_out: [b][A], n_act^2 at aoff[m]
// Geometry tables are shared by all instances (ti/td/tf, see plan.cpp).
#pragma once

#include <cstdint>

namespace fewha_gpu {

constexpr int kMaxL = 16;
constexpr int kMaxW = 16;
constexpr int kMaxM = 16;
constexpr int kMaxC = 16;  // CTAs per layer cluster (8: portable; 16: non-portable opt-in)
constexpr int kMaxGU = 64;      // row groups per layer (max side 128 / the smallest row group, 2)
constexpr int kMaxWtCode = 1024;  // WFS tiles with a constant-bank position code

// Fused-PCG carry (pcg.hpp:32-38 PcgScalars plus per-frame bookkeeping).
struct Carry {
    double rho_old, alpha, rho_entry;
    int fresh, done, err, nlog;
};

struct GeoParams {
    int L, W, M;
    int n, S, Nw, A;
    int iters, closed, maxside;
    int side[kMaxL], lorder[kMaxL], coff[kMaxL];
    int ns[kMaxW], moff[kMaxW], woff[kMaxW], mkoff[kMaxW];
    int nact[kMaxM], aoff[kMaxM];
    double inv_var[kMaxW];
    double alpha, gain, tol, fault;
    int piston_exact;  // fp32 engines: the fitting term's coarse coefficient is exactly 0 (see k_layer_forward)
    int gather_ni;  // instances per k_gather CTA (batched plans 2, else 1; host plan, cluster.cuh k_gather_ni)
    double flo[20], fhi[20];  // Daubechies taps of the configured order (wavelet.hpp:100-107)
    float flo_f[20], fhi_f[20];
    // tables
    const int* ti;
    const double* td;
    const float* tf;
    const std::uint8_t* masks;
    // table directory offsets (into ti)
    int o_pl;   // [(w*L+l)*4 + {0 x-table, 1 y-table, 2 row ranges, 3 col ranges}]
    int o_pd;   // [(w*M+m)*2 + {0 x-table, 1 y-table}] for DM screens
    int o_fit;  // [m] fit table (n_act entries) or -1 for identity
    int o_reg;  // [l] offset into td of d_{l,0..J}
    // tiles
    const int* wtiles;  // [n_wtiles][3] (w, i0, j0) for the per-WFS kernels (host bookkeeping)
    int n_wtiles, wtile;
    int wt_first[kMaxW + 1];  // first tile of each WFS (prefix), tiles row-major per WFS
    int wt_cols[kMaxW];       // tiles per row of WFS w
    int wa, wb;               // WFS owned by this plan's per-WFS kernels (all unless sharded)
    // tile -> (w | i0/16 << 8 | j0/16 << 20), so a WFS tile CTA decodes its position from
    // the constant bank (n_wtiles <= kMaxWtCode; larger geometries search wt_first)
    unsigned wt_code[kMaxWtCode];
    int wt_base, wt_count;    // their tiles: [wt_base, wt_base + wt_count)
    const unsigned char* tblob;  // per-tile stencil tables [tile][screen][axis][H] idx, then weights
    int tt_stride_l, tt_stride_d, tt_off_d;  // byte stride per tile (layer / DM screens), DM base
    // v2 cluster path
    int ccl;          // CTAs per layer cluster
    int ctail;        // tail size D of distributed layers (clayout.hpp)
    int tonly;        // largest tail-only layer side (S < 2D; 0: none) -- sizes the forward band buffer
    int grows;        // layer rows per CTA of the adjoint gather (4: latency, 8: batches)
    int inv_staged;   // inverse kernel: operands staged in shared memory by TMA (1) or read from global (0)
    int gather_km;    // max gather taps per layer row/column
    int o_bs;         // [((w*L+l)*kMaxGU + u)*4] psi source block {ilo, ihi, jlo, jhi} of each gather row group
    int gather_direct;  // 1: k_gather_direct and its tables (batched plans), 0: k_gather / k_gather_ni
    int bd_cols_max;
    unsigned long long* stamps;  // optional phase timestamps [block][16] (nullptr: off)
    const unsigned char* gblob;  // per-(w,l) gather blobs of the engine's precision (see cluster.cuh)
    int chunk_bytes;  // shared-memory bytes of the largest staged WFS chunk of the gather
    int nchunk;                 // WFS chunks of the gather: [gchunk[k], gchunk[k+1])
    int gchunk[kMaxW + 1];
    int o_gd;                   // [((l*kMaxGU + u)*kMaxW + w)*8] gather staging descriptors (int4-aligned)
    int gbuf_bytes;   // the gather's double-buffered row-contracted block (see cluster.cuh)
    int gather_minb;  // k_gather residency plan: resident CTAs per SM (2, 3 or 4; cluster.cuh)
};

enum LayerMode : int {
    kPlain = 0,   // inverse: phi = W^-1 in        forward: out = W y
    kApply = 1,   // forward: out = W y + alpha D in  (apply_M)
    kPcg = 2,     // inverse: [update] z = r/J, rho, phi = W^-1 z ; forward: s = W y + aDz, mu
    kFit = 3,     // inverse: [final update] phi = W^-1 c
    kRhs = 4,     // forward: b1 = W y ; r += b1 - b ; b = b1
};

// kernel kinds reported by fewha_gpu_profile_step
enum KernelKind : int {
    kKindWfsRhs = 0,   // k_wfs<RHS>: Gamma^T C^-1 (s + Gamma P_dm a)
    kKindAdjoint = 1,  // (unused id: the adjoint is k_gather, kKindGather)
    kKindFwdRhs = 2,   // k_layer_forward kRhs: b1 = W y, r += b1 - b
    kKindInvPcg0 = 3,  // k_layer_inverse kPcg it=0: z = r/J, W^-1 z
    kKindInvPcg = 4,   // k_layer_inverse kPcg it>0: fused p,q,c,r update + z + W^-1 z
    kKindWfs = 5,      // k_wfs: Gamma^T C^-1 Gamma P phi
    kKindFwdPcg = 6,   // k_layer_forward kPcg: s = W y + alpha D z, mu
    kKindInvFit = 7,   // k_layer_inverse kFit: last update + W^-1 c
    kKindFit = 8,      // k_fit_control
    kKindGather = 9,   // k_gather: y = sum_w P^T psi_w
    // k_fwd_inv_cluster (fused forward + inverse, single-instance latency plans)
    kKindFwdRhsInv0 = 10,  // kRhs forward + kPcg it=0 inverse
    kKindFwdInvPcg = 11,   // kPcg forward (it k) + kPcg inverse (it k+1)
    kKindFwdInvFit = 12,   // kPcg forward (last it) + kFit inverse
};

template <typename T>
struct Bufs {
    // coefficient domain [B][n]
    T *c, *b, *r, *p, *q, *mz;
    const T* jac;   // [n] shared Jacobi diagonal
    const T* jinv;  // [n] shared 1/J (z = r * (1/J): one rounding vs r/J, well inside tolerance)
    T *phi, *y;    // nodal [B][n]
    T* psi;        // [B][Nw]
    const double* meas;  // [B][S]
    T *a_prev2, *a_prev, *a_out;  // [B][A]
    const T* in;   // operator input [B][n] (plain / apply modes)
    T* out;        // operator output [B][n]
    Carry* carry;  // [B][iters+1]
    double* rho_part;  // [B][iters][L]
    double* mu_part;   // [B][iters][L]
    double* rho_log;   // [B][iters]
    int* status;       // [B]
    int* nlog;         // [B]
    // per-WFS shard groups: the forward kernel stages y = sum_r ysum[r] (the
    // members' partial adjoint layer sums, rank order; peer loads across devices) instead
    // of y -- the exchange fused into the band staging (nsum = 0: off)
    const T* ysum[kMaxW];
    int nsum;
    // zero-copy frame outputs (page-locked host memory, written by k_fit_control; null: off)
    double* a_host;         // a1 [B][A] straight into the caller's buffer
    unsigned char* frame_host;  // mirror of the rho_log | status | nlog block
};

}  // namespace fewha_gpu
