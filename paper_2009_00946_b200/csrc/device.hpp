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
    int filt_off;  // offset of the wavelet order in the constant filter table
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
    const int* wtiles;  // [n_wtiles][3] (w, i0, j0) for the per-WFS kernels
    int n_wtiles, wtile;
    const int* ltiles;  // [n_ltiles][3] (l, I0, J0) for the adjoint-propagation kernel
    int n_ltiles, ltile, lt_rows_max, lt_cols_max;
    int o_tr;  // [(tile*W + w)*4] psi source block {ilo, ihi, jlo, jhi} of each layer tile (into ti)
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
    kKindAdjoint = 1,  // k_adjoint: sum_w P^T psi
    kKindFwdRhs = 2,   // k_layer_forward kRhs: b1 = W y, r += b1 - b
    kKindInvPcg0 = 3,  // k_layer_inverse kPcg it=0: z = r/J, W^-1 z
    kKindInvPcg = 4,   // k_layer_inverse kPcg it>0: fused p,q,c,r update + z + W^-1 z
    kKindWfs = 5,      // k_wfs: Gamma^T C^-1 Gamma P phi
    kKindFwdPcg = 6,   // k_layer_forward kPcg: s = W y + alpha D z, mu
    kKindInvFit = 7,   // k_layer_inverse kFit: last update + W^-1 c
    kKindFit = 8,      // k_fit_control
};

template <typename T>
struct Bufs {
    // coefficient domain [B][n]
    T *c, *b, *r, *p, *q, *mz;
    const T* jac;  // [n] shared
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
};

}  // namespace fewha_gpu
