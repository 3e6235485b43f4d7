// Host engine of the B200-native FEWHA reconstructor (see engine.hpp).
#include "engine.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <climits>
#include <cstdint>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numbers>
#include <stdexcept>
#include <type_traits>

#include "daubechies_table.h"
#include "device.hpp"
#include "cluster.cuh"
#include "layer_whole.cuh"
#include "clayout.hpp"
#include "launch.hpp"
#include "nccl_dl.hpp"
#include "sim_kernels.cuh"

namespace fewha_gpu {

#define CK(x)                                                                                        \
    do {                                                                                             \
        cudaError_t e_ = (x);                                                                        \
        if (e_ != cudaSuccess)                                                                       \
            throw std::runtime_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " + \
                                     __FILE__ + ":" + std::to_string(__LINE__));                     \
    } while (0)

namespace {

// ---------------------------------------------------------------------------
// Geometry tables (host, fp64, reference expressions)
// ---------------------------------------------------------------------------

struct Stencil1 {
    int idx;
    double f;
};

// 1-D half of bilinear_stencil (operators.hpp:108-121): u = (p + e/2)/spacing,
// j0 = min(floor(u), n-2), f = u - j0 (before clamping at 0), idx = max(j0, 0).
Stencil1 stencil1(int n, double extent, double p) {
    const double spacing = extent / (n - 1);
    const double u = (p + extent / 2.0) / spacing;
    constexpr double eps = 1e-9;
    if (u < -eps || u > n - 1 + eps) throw std::runtime_error("propagation: evaluation point outside layer grid");
    const int j0 = std::min(static_cast<int>(std::floor(u)), n - 2);
    return {std::max(j0, 0), u - j0};
}

struct Plan {
    GeoParams gp{};
    std::vector<int> ti;
    std::vector<double> td;
    std::vector<std::uint8_t> masks;
    std::vector<int> wtiles;
    std::vector<unsigned char> gblob, tblob;
    std::vector<int> perm;  // Mallat coefficient index -> rank-blocked HBM index (clayout.hpp)
    int maxside = 0;
};

// Rank-blocked order of the coefficient-domain vectors: per layer, rank q's
// owned set (level blocks A then D rows, then the tail on rank 0) at
// rank_off(q), in the order the kernels' for_owned() visits it.
std::vector<int> coeff_perm(const GeoParams& gp) {
    std::vector<int> perm(static_cast<size_t>(gp.n), -1);
    const int C = gp.ccl, D = gp.ctail;
    for (int l = 0; l < gp.L; ++l) {
        const int S = gp.side[l], base = gp.coff[l];
        for (int q = 0; q < C; ++q) {
            int o = base + clay::rank_off(S, C, D, q);
            for (int lv = 0; lv < clay::nlev(S, C, D); ++lv) {
                const int s = S >> lv, h = s / 2, k = h / C, m0 = q * k;
                for (int i = 0; i < k; ++i)
                    for (int c = 0; c < h; ++c) perm[static_cast<size_t>(base + (m0 + i) * S + h + c)] = o++;
                for (int i = 0; i < k; ++i)
                    for (int c = 0; c < s; ++c) perm[static_cast<size_t>(base + (h + m0 + i) * S + c)] = o++;
            }
            if (q == 0) {
                const int T = clay::tail(S, C, D);
                for (int i = 0; i < T; ++i)
                    for (int j = 0; j < T; ++j) perm[static_cast<size_t>(base + i * S + j)] = o++;
            }
            if (o != base + clay::rank_off(S, C, D, q) + clay::owned_count(S, C, D, q))
                throw std::logic_error("coefficient layout: rank block size mismatch");
        }
    }
    for (int v : perm)
        if (v < 0) throw std::logic_error("coefficient layout: unassigned coefficient");
    return perm;
}

int push_table(Plan& pl, const std::vector<Stencil1>& t) {
    const int off = static_cast<int>(pl.ti.size());
    for (const auto& s : t) {
        pl.ti.push_back(s.idx);
        pl.td.push_back(s.f);
    }
    return off;
}

// ranges[I] = [first, last+1) of source nodes whose stencil touches target node I
int push_ranges(Plan& pl, const std::vector<Stencil1>& t, int n_target) {
    const int off = static_cast<int>(pl.ti.size());
    for (int I = 0; I < n_target; ++I) {
        int lo = static_cast<int>(t.size()), hi = 0;
        for (int j = 0; j < static_cast<int>(t.size()); ++j) {
            if (t[j].idx == I || t[j].idx + 1 == I) {
                lo = std::min(lo, j);
                hi = std::max(hi, j + 1);
            }
        }
        if (hi <= lo) lo = hi = 0;
        pl.ti.push_back(lo);
        pl.ti.push_back(hi);
        pl.td.push_back(0.0);
        pl.td.push_back(0.0);
    }
    return off;
}

// wa..wb: the WFS this plan's per-WFS kernels own (all of them unless sharded,
// SURVEY 8e): the WFS kernels run only those tiles and the adjoint gather sums
// only those WFS.
Plan build_plan(const Geometry& g, int elem_bytes, int batch, int wa = 0, int wb = -1) {
    Plan pl;
    GeoParams& gp = pl.gp;
    const int L = static_cast<int>(g.layers.size()), W = static_cast<int>(g.wfs.size()),
              M = static_cast<int>(g.dms.size());
    if (L > kMaxL || W > kMaxW || M > kMaxM)
        throw ConfigError("invalid geometry: at most 16 layers, 16 wfs and 16 dms are supported on the device");
    if (wb < 0) wb = W;
    if (wa < 0 || wa >= wb || wb > W) throw ArgError("shard: empty or out-of-range WFS range");
    gp.wa = wa;
    gp.wb = wb;
    gp.L = L;
    gp.W = W;
    gp.M = M;
    gp.n = static_cast<int>(g.coeff_dim());
    gp.S = static_cast<int>(g.measurement_dim());
    gp.Nw = static_cast<int>(g.wavefront_dim());
    gp.A = static_cast<int>(g.act_dim());
    gp.iters = g.pcg_iters;
    gp.closed = g.closed_loop ? 1 : 0;
    gp.alpha = g.alpha;
    gp.gain = g.gain;
    gp.tol = g.pcg_tol;
    gp.fault = g.fault == "sh_adjoint" ? 1.0 + 1e-6 : 1.0;  // reconstructor.hpp:120

    int off = 0;
    for (int l = 0; l < L; ++l) {
        if (g.layers[l].order > 7)
            throw ConfigError("invalid geometry: layer grid_order > 7 exceeds the on-chip transform (see DESIGN.md)");
        gp.side[l] = g.layers[l].side();
        gp.lorder[l] = g.layers[l].order;
        gp.coff[l] = off;
        off += gp.side[l] * gp.side[l];
        pl.maxside = std::max(pl.maxside, gp.side[l]);
    }
    gp.maxside = pl.maxside;
    int mo = 0, wo = 0, mk = 0;
    for (int w = 0; w < W; ++w) {
        const int ns = g.wfs[w].n_subap;
        gp.ns[w] = ns;
        gp.moff[w] = mo;
        gp.woff[w] = wo;
        gp.mkoff[w] = mk;
        gp.inv_var[w] = 1.0 / g.wfs[w].noise_variance;  // operators.hpp:280
        mo += 2 * ns * ns;
        wo += (ns + 1) * (ns + 1);
        mk += ns * ns;
        pl.masks.insert(pl.masks.end(), g.wfs[w].mask.begin(), g.wfs[w].mask.end());
    }
    int ao = 0;
    for (int m = 0; m < M; ++m) {
        gp.nact[m] = g.dms[m].n_act;
        gp.aoff[m] = ao;
        ao += g.dms[m].n_act * g.dms[m].n_act;
    }

    // directory slots first, filled below
    gp.o_pl = 0;
    pl.ti.assign(static_cast<size_t>(W * L * 4 + W * M * 2 + M + L), 0);
    pl.td.assign(pl.ti.size(), 0.0);
    gp.o_pd = W * L * 4;
    gp.o_fit = gp.o_pd + W * M * 2;
    gp.o_reg = gp.o_fit + M;

    auto aperture_axis = [&](int w, const Star& s, double h, int n, double extent, bool x_axis) {
        const int np = g.wfs[w].n_subap + 1;
        const double d = g.diameter / (np - 1);
        const double c = s.footprint(h);
        std::vector<Stencil1> t(static_cast<size_t>(np));
        for (int j = 0; j < np; ++j) {
            const double x = -g.diameter / 2.0 + j * d;  // operators.hpp:227-231
            const double p = c * x + (x_axis ? s.theta_x : s.theta_y) * h;
            t[j] = stencil1(n, extent, p);
        }
        return t;
    };

    for (int w = 0; w < W; ++w) {
        for (int l = 0; l < L; ++l) {
            const auto& lay = g.layers[l];
            const auto tx = aperture_axis(w, g.stars[w], lay.height, lay.side(), lay.extent, true);
            const auto ty = aperture_axis(w, g.stars[w], lay.height, lay.side(), lay.extent, false);
            int* dir = &pl.ti[static_cast<size_t>((w * L + l) * 4)];
            const int ox = push_table(pl, tx), oy = push_table(pl, ty);
            const int orr = push_ranges(pl, ty, lay.side()), occ = push_ranges(pl, tx, lay.side());
            dir = &pl.ti[static_cast<size_t>((w * L + l) * 4)];
            dir[0] = ox;
            dir[1] = oy;
            dir[2] = orr;
            dir[3] = occ;
        }
        for (int m = 0; m < M; ++m) {
            const auto& dm = g.dms[m];
            const auto tx = aperture_axis(w, g.stars[w], dm.height, dm.n_act, dm.extent, true);
            const auto ty = aperture_axis(w, g.stars[w], dm.height, dm.n_act, dm.extent, false);
            const int ox = push_table(pl, tx), oy = push_table(pl, ty);
            pl.ti[static_cast<size_t>(gp.o_pd + (w * M + m) * 2)] = ox;
            pl.ti[static_cast<size_t>(gp.o_pd + (w * M + m) * 2 + 1)] = oy;
        }
    }
    // fitting tables.  Reference L = M pairing (reconstructor.hpp:294-302): DM m
    // samples layer m on its own extent -- identity copy when n_act = 2^J (-1).
    // Projection fitting (L != M extension): DM m sums its layer group at the
    // actuator positions shifted by theta_m * h_l.  Block: [cnt, (l, ox, oy) x cnt].
    for (int m = 0; m < M; ++m) {
        const auto& dm = g.dms[m];
        std::vector<int> group = g.projection ? dm.layers : std::vector<int>{m};
        if (!g.projection && dm.n_act == g.layers[m].side()) {
            pl.ti[static_cast<size_t>(gp.o_fit + m)] = -1;
            continue;
        }
        const double da = dm.extent / (dm.n_act - 1);
        std::vector<std::array<int, 3>> entries;
        for (int l : group) {
            const auto& lay = g.layers[static_cast<size_t>(l)];
            const int side = lay.side();
            // reference path: bilinear_sample(grid, dm.extent, ...) -- the DM extent is the layer's
            const double e_grid = g.projection ? lay.extent : dm.extent;
            std::vector<Stencil1> tx(static_cast<size_t>(dm.n_act)), ty(static_cast<size_t>(dm.n_act));
            // projection: points off the layer grid contribute zero (index -1)
            auto st = [&](double p) {
                if (g.projection) {
                    const double u = (p + e_grid / 2.0) / (e_grid / (side - 1));
                    if (u < -1e-9 || u > side - 1 + 1e-9) return Stencil1{-1, 0.0};
                }
                return stencil1(side, e_grid, p);
            };
            for (int j = 0; j < dm.n_act; ++j) {
                const double p = -dm.extent / 2.0 + j * da;
                tx[j] = st(g.projection ? p + dm.theta_x * lay.height : p);
                ty[j] = st(g.projection ? p + dm.theta_y * lay.height : p);
            }
            const int ox = push_table(pl, tx);
            const int oy = g.projection ? push_table(pl, ty) : ox;
            entries.push_back({l, ox, oy});
        }
        const int off = static_cast<int>(pl.ti.size());
        pl.ti.push_back(static_cast<int>(entries.size()));
        for (const auto& en : entries) pl.ti.insert(pl.ti.end(), en.begin(), en.end());
        pl.td.resize(pl.ti.size(), 0.0);
        pl.ti[static_cast<size_t>(gp.o_fit + m)] = off;
    }
    // alpha * regularizer per (layer, scale) (operators.hpp:307-321)
    const double kappa0 = 2.0 * std::numbers::pi / g.outer_scale;
    for (int l = 0; l < L; ++l) {
        const auto& lay = g.layers[l];
        pl.ti[static_cast<size_t>(gp.o_reg + l)] = static_cast<int>(pl.td.size());
        for (int j = 0; j <= lay.order; ++j) {
            const double kappa = std::ldexp(2.0 * std::numbers::pi / lay.extent, j);
            const double d = std::pow(kappa * kappa + kappa0 * kappa0, g.spectral_exponent) / lay.strength;
            pl.td.push_back(g.alpha * d);
            pl.ti.push_back(0);
        }
    }

    // WFS tiles: 16 x 16 nodes
    gp.wtile = kWfsTile;
    for (int w = 0; w < W; ++w) {
        const int np = g.wfs[w].n_subap + 1;
        gp.wt_first[w] = static_cast<int>(pl.wtiles.size() / 3);
        gp.wt_cols[w] = (np + gp.wtile - 1) / gp.wtile;
        for (int i0 = 0; i0 < np; i0 += gp.wtile)
            for (int j0 = 0; j0 < np; j0 += gp.wtile) pl.wtiles.insert(pl.wtiles.end(), {w, i0, j0});
    }
    gp.n_wtiles = static_cast<int>(pl.wtiles.size() / 3);
    gp.wt_first[W] = gp.n_wtiles;
    for (int t = 0; t < gp.n_wtiles && t < kMaxWtCode; ++t)
        gp.wt_code[t] = static_cast<unsigned>(pl.wtiles[3 * t]) |
                        (static_cast<unsigned>(pl.wtiles[3 * t + 1] / gp.wtile) << 8) |
                        (static_cast<unsigned>(pl.wtiles[3 * t + 2] / gp.wtile) << 20);
    gp.wt_base = gp.wt_first[wa];
    gp.wt_count = gp.wt_first[wb] - gp.wt_first[wa];
    // per-tile stencil tables of the tile's halo rows/columns for every screen, in the
    // shared-memory layout of wfs_tile (kernels.cuh): [screen][axis][H] idx | [screen][axis][H] weight
    {
        constexpr int H = kWfsTile + 2;
        auto a16 = [](size_t v) { return (v + 15) & ~size_t(15); };
        auto build = [&](int NS, bool dms) {
            const size_t ib = a16(static_cast<size_t>(NS) * 2 * H * sizeof(int));
            const size_t stride = ib + a16(static_cast<size_t>(NS) * 2 * H * elem_bytes);
            const size_t base = pl.tblob.size();
            pl.tblob.resize(base + stride * gp.n_wtiles, 0);
            for (int t = 0; t < gp.n_wtiles; ++t) {
                const int w = pl.wtiles[3 * t], i0 = pl.wtiles[3 * t + 1], j0 = pl.wtiles[3 * t + 2];
                const int np = g.wfs[w].n_subap + 1;
                unsigned char* p = pl.tblob.data() + base + stride * t;
                for (int sc = 0; sc < NS; ++sc)
                    for (int axis = 0; axis < 2; ++axis) {
                        const int off = dms ? pl.ti[static_cast<size_t>(gp.o_pd + (w * M + sc) * 2 + axis)]
                                            : pl.ti[static_cast<size_t>(gp.o_pl + (w * L + sc) * 4 + axis)];
                        for (int kk = 0; kk < H; ++kk) {
                            const int node = std::min(std::max((axis ? i0 : j0) - 1 + kk, 0), np - 1);
                            const int q = (sc * 2 + axis) * H + kk;
                            std::memcpy(p + q * sizeof(int), &pl.ti[static_cast<size_t>(off + node)], sizeof(int));
                            const double wv = pl.td[static_cast<size_t>(off + node)];
                            if (elem_bytes == 8) std::memcpy(p + ib + q * 8, &wv, 8);
                            else {
                                const float f = static_cast<float>(wv);
                                std::memcpy(p + ib + q * 4, &f, 4);
                            }
                        }
                    }
            }
            return std::pair<size_t, size_t>{base, stride};
        };
        const auto tl = build(L, false);
        const auto td_ = build(M, true);
        gp.tt_stride_l = static_cast<int>(tl.second);
        gp.tt_stride_d = static_cast<int>(td_.second);
        gp.tt_off_d = static_cast<int>(td_.first);
    }

    // ---- cluster path: C = maxside / min(R, maxside) CTAs per layer, R = 16 band rows per rank
    // (FEWHA_CLUSTER_ROWS = 8: 16-CTA clusters, non-portable); band rows per rank: clayout.hpp
    {
        int band = 16;
        if (const char* v = std::getenv("FEWHA_CLUSTER_ROWS")) {
            const int r = std::atoi(v);
            if (r == 8 || r == 16) band = r;
        }
        const int R = std::min(band, pl.maxside);
        gp.ccl = pl.maxside / R;
        if (gp.ccl > kMaxC) throw ConfigError("invalid geometry: layer side exceeds the cluster transform");
        auto tonly_of = [&](int D) {  // largest tail-only layer side for tail size D
            int t = 0;
            for (int l = 0; l < L; ++l)
                if (!clay::dist(gp.side[l], gp.ccl, D)) t = std::max(t, gp.side[l]);
            return t;
        };
        // tail size: D = 4C (measured best at the ELT scale), else 2C, else C -- the first whose layer kernels fit the sm_100 opt-in
        // shared memory (227 KB less static) in fp64 -- fp32 engines use the same layout, so
        // their fp64 preconditioner probes share the coefficient permutation
        {
            // Batches (> 2 instances) instead keep the forward and the streamed-operand
            // inverse at two CTAs per SM (<= 113 KB each), which the 32^2 tail buffers break.
            constexpr int kSmemBudget = 227 * 1024 - 2048, kTwoPerSm = 113 * 1024 - 2048;
            const int flen = 2 * g.wavelet_order, C = gp.ccl;
            gp.ctail = C;
            // candidates: a 32^2 tail (4C at C = 8, 2C at C = 16; measured best at the ELT
            // scale), then 2C
            const int D0 = C <= 8 ? 4 * C : 2 * C;
            for (int D : {D0, 2 * C}) {
                if (D > pl.maxside / 2) continue;
                const int t = tonly_of(D);
                const bool fits = clay::inv_smem(pl.maxside, C, D, flen, 8).total <= kSmemBudget &&
                                  clay::fwd_smem(pl.maxside, C, D, flen, 8, t).total <= kSmemBudget;
                const bool two = clay::inv_smem(pl.maxside, C, D, flen, 8, 0).total <= kTwoPerSm &&
                                 clay::fwd_smem(pl.maxside, C, D, flen, 8, t).total <= kTwoPerSm;
                if (fits && (batch <= 2 || two)) {
                    gp.ctail = D;
                    break;
                }
            }
            if (const char* v = std::getenv("FEWHA_TAIL")) {  // profiling override (power of two in [C, maxside/2])
                const int D = std::atoi(v);
                if (D >= C && D <= std::max(C, pl.maxside / 2) && (D & (D - 1)) == 0) gp.ctail = D;
            }
            gp.tonly = tonly_of(gp.ctail);
        }
        // gather tables: per (w,l) and axis, for every layer node the (source, weight) list,
        // ascending source (operators.hpp:129-135 weights as bilinear_stencil assigns them)
        struct Entry { int src; double w; };
        std::vector<std::vector<std::vector<Entry>>> rows(W * L), cols(W * L);
        std::vector<std::vector<Stencil1>> colst(W * L);  // per psi column: layer column idx, fraction
        int km = 1;
        for (int w = 0; w < W; ++w)
            for (int l = 0; l < L; ++l) {
                const auto& lay = g.layers[l];
                const int side = lay.side();
                const auto tx = aperture_axis(w, g.stars[w], lay.height, side, lay.extent, true);
                const auto ty = aperture_axis(w, g.stars[w], lay.height, side, lay.extent, false);
                auto build = [&](const std::vector<Stencil1>& t) {
                    std::vector<std::vector<Entry>> out(static_cast<size_t>(side));
                    for (int s = 0; s < static_cast<int>(t.size()); ++s) {
                        out[t[s].idx].push_back({s, 1.0 - t[s].f});
                        out[t[s].idx + 1].push_back({s, t[s].f});
                    }
                    for (auto& v : out) km = std::max(km, static_cast<int>(v.size()));
                    return out;
                };
                rows[w * L + l] = build(ty);
                cols[w * L + l] = build(tx);
                colst[w * L + l] = tx;
            }
        // (km > 4: coarse layers under dense aperture sampling take the runtime-tap path)
        gp.gather_km = km;
        // the direct gather (cluster.cuh k_gather_direct) wherever the tap counts are
        // compile-time (km <= 4), else k_gather (runtime taps); FEWHA_GATHER_DIRECT = 0 forces
        // k_gather.  Measured (ELT MCAO-84, fp64): single frame 0.1864 -> 0.180 ms, batch-64
        // gather launch 145 -> 113 us
        int direct = km <= 4;
        if (const char* v = std::getenv("FEWHA_GATHER_DIRECT")) direct = std::atoi(v) == 1 && km <= 4;
        gp.gather_direct = direct;
        // psi source blocks per (w, l, gather row group u)
        // rows per gather CTA: 4 for a single instance (288 CTAs at the ELT scale, two per
        // SM; 8: 0.1945 ms), 8 for batches (batch 64, 4 instances per CTA: 2.48 vs 2.63 ms per
        // step); FEWHA_GATHER_ROWS overrides
        gp.grows = batch <= 2 || km > 4 ? 4 : 8;
        if (const char* v = std::getenv("FEWHA_GATHER_ROWS")) {
            const int r = std::atoi(v);
            if (r == 2 || r == 4 || r == 8) gp.grows = r;
        }
        // (k_gather_direct: layer sides <= 128 -- at most half the group rows per thread)
        if (pl.maxside > 128) direct = gp.gather_direct = 0;
        auto grp_rows = [&](int side) { return std::min(gp.grows, side); };
        gp.o_bs = static_cast<int>(pl.ti.size());
        pl.ti.resize(pl.ti.size() + static_cast<size_t>(W * L * kMaxGU * 4), 0);
        pl.td.resize(pl.ti.size(), 0.0);
        int rmax = 1, cmax = 1;
        for (int w = 0; w < W; ++w)
            for (int l = 0; l < L; ++l) {
                const auto& rt = rows[w * L + l];
                const auto& ct = cols[w * L + l];
                const int side = static_cast<int>(rt.size());
                int jlo = INT32_MAX, jhi = 0;
                for (const auto& v : ct)
                    for (const auto& en : v) {
                        jlo = std::min(jlo, en.src);
                        jhi = std::max(jhi, en.src + 1);
                    }
                const int Rl = grp_rows(side);
                for (int u = 0; u < side / Rl; ++u) {
                    const int I0 = u * Rl;
                    int ilo = INT32_MAX, ihi = 0;
                    for (int I = I0; I < I0 + Rl; ++I)
                        for (const auto& en : rt[I]) {
                            ilo = std::min(ilo, en.src);
                            ihi = std::max(ihi, en.src + 1);
                        }
                    int* bs = &pl.ti[static_cast<size_t>(gp.o_bs + ((w * L + l) * kMaxGU + u) * 4)];
                    if (ilo < ihi && jlo < jhi) {
                        bs[0] = ilo; bs[1] = ihi; bs[2] = jlo; bs[3] = jhi;
                        rmax = std::max(rmax, ihi - ilo);
                        cmax = std::max(cmax, jhi - jlo);
                    } else {  // no source rows: empty block, but the WFS-wide column origin stays
                        bs[0] = bs[1] = 0;  // (the gather blob's column sources are relative to it)
                        bs[2] = jlo < jhi ? jlo : 0;
                        bs[3] = jlo < jhi ? jhi : 0;
                    }
                }
            }
        (void)rmax;
        gp.bd_cols_max = cmax;
        // staged bytes per WFS (mirrors gather_tab_bytes()/psi_bytes() in cluster.cuh)
        auto a16 = [](size_t v) { return (v + 15) & ~size_t(15); };
        // row-tap table of one (layer, row group, WFS) and column stencil of one (layer, WFS)
        // (direct gather: [first source int16 per node][km weights per node], for the R group
        // rows and for the side layer columns)
        auto row_bytes = [&](int R) {
            if (direct) return a16(static_cast<size_t>(R) * 2) + a16(static_cast<size_t>(R) * km * elem_bytes);
            return a16(static_cast<size_t>(R) * km * 2) + a16(static_cast<size_t>(R) * km * elem_bytes);
        };
        auto col_bytes = [&](int side, int nc) {
            if (direct) return a16(static_cast<size_t>(side) * 2) + a16(static_cast<size_t>(side) * km * elem_bytes);
            return a16(static_cast<size_t>(side + 3) * 2) + a16(static_cast<size_t>(nc) * 2) +
                   a16(static_cast<size_t>(nc) * elem_bytes);
        };
        auto tab_bytes = [&](int R, int side, int nc) { return row_bytes(R) + col_bytes(side, nc); };
        // WFS chunks (same for every row group): greedy over w by the worst row group's bytes,
        // within a budget that keeps two gather CTAs per SM
        auto need_of = [&](int w, int l, int u) {
            const int side = gp.side[l], Rl = grp_rows(side);
            const int* bs = &pl.ti[static_cast<size_t>(gp.o_bs + ((w * L + l) * kMaxGU + u) * 4)];
            return std::pair<size_t, size_t>(
                tab_bytes(Rl, side, bs[3] - bs[2]),
                a16(static_cast<size_t>(bs[1] - bs[0]) * (g.wfs[w].n_subap + 1) * elem_bytes + 16));
        };
        // instances per CTA of the direct gather (batched plans: 4, sharing the staged tables;
        // batch 64 fp64: 2.48 ms per step vs 2.54 with 2; FEWHA_GATHER_NI = 1, 2 or 4 overrides)
        gp.gather_ni = batch > 2 ? 4 : 1;
        if (const char* v = std::getenv("FEWHA_GATHER_NI")) {
            const int ni = std::atoi(v);
            if (ni == 1 || ni == 2 || ni == 4) gp.gather_ni = ni;
        }
        if (!direct) gp.gather_ni = 1;
        const size_t NIg = static_cast<size_t>(gp.gather_ni);
        std::vector<size_t> need_max(static_cast<size_t>(W), 0);
        for (int w = 0; w < W; ++w)
            for (int l = 0; l < L; ++l)
                for (int u = 0; u < gp.side[l] / grp_rows(gp.side[l]); ++u) {
                    const auto nb = need_of(w, l, u);
                    need_max[static_cast<size_t>(w)] = std::max(need_max[static_cast<size_t>(w)], nb.first + NIg * nb.second);
                }
        // k_gather's row-contracted blocks G of every WFS of a chunk (group rows x widest psi
        // block); the direct gather has none
        gp.gbuf_bytes = direct ? 0 : static_cast<int>(a16(static_cast<size_t>(W) * gp.grows * cmax * elem_bytes));
        const size_t fixed = a16(static_cast<size_t>(gp.gbuf_bytes)) + 1024;  // + static shared memory
        // residency plan of the gather (cluster.cuh gather_smem_kb): 2 CTAs/SM for a single
        // instance (direct: 0.180 ms vs 0.184 at 3); batches of the direct gather, 4 instances
        // per CTA: fp64 2 (2.48 ms per step vs 2.64 at 3, which spills), fp32 4 (1.58 vs 1.62
        // at 2); k_gather batches 3.  FEWHA_GATHER_MINB overrides: 2, 3 or 4
        gp.gather_minb = batch <= 2 ? 2 : !direct ? 3 : elem_bytes == 4 ? 4 : 2;
        if (const char* v = std::getenv("FEWHA_GATHER_MINB")) {
            const int m = std::atoi(v);
            if (m >= 2 && m <= 4) gp.gather_minb = m;
        }
        const size_t limit = static_cast<size_t>(gather_smem_kb(gp.gather_minb)) * 1024;
        const size_t budget = limit > fixed ? limit - fixed : 0;
        gp.nchunk = 0;
        gp.gchunk[0] = wa;
        size_t used = 0, chunk_max = 0;
        for (int w = wa; w < wb; ++w) {
            if (need_max[static_cast<size_t>(w)] > budget)
                throw ConfigError("invalid geometry: adjoint gather does not fit in shared memory");
            if (w > gp.gchunk[gp.nchunk] && used + need_max[static_cast<size_t>(w)] > budget) {
                gp.gchunk[++gp.nchunk] = w;
                used = 0;
            }
            used += need_max[static_cast<size_t>(w)];
            chunk_max = std::max(chunk_max, used);
        }
        gp.gchunk[++gp.nchunk] = wb;
        gp.chunk_bytes = static_cast<int>(chunk_max);
        // gather tables (mirrors k_gather() in cluster.cuh), in gblob:
        //   column stencils, once per (layer, WFS), WFS ascending within a layer:
        //     [first int16 side+3][col idx int16 nc][col frac nc]
        //   row-tap tables per (layer, row group), WFS ascending:
        //     [row src int16 R x KM][row w R x KM]   padded row taps of the group
        // every part 16-byte aligned.  Row sources are relative to the group's psi block row
        // ilo (zero-weight padding clamped into the block); column entries are the psi block
        // columns jlo.. with their layer column idx and bilinear fraction f (layer column J
        // receives 1-f from idx == J and f from idx == J-1, operators.hpp:129-135);
        // first[k] = first block column with idx >= k-1.  The column stencil depends on the
        // WFS and the layer only, so every row group of the layer stages the same copy.
        pl.gblob.clear();
        auto padded = [&](const std::vector<std::vector<Entry>>& tab, std::vector<int>& src, std::vector<double>& wt) {
            const int side = static_cast<int>(tab.size());
            src.assign(static_cast<size_t>(side) * km, 0);
            wt.assign(static_cast<size_t>(side) * km, 0.0);
            int carry = 0;
            for (const auto& v : tab)
                if (!v.empty()) { carry = v.front().src; break; }
            for (int I = 0; I < side; ++I)
                for (int q = 0; q < km; ++q) {
                    const bool valid = q < static_cast<int>(tab[I].size());
                    if (valid) carry = tab[I][q].src;
                    src[static_cast<size_t>(I) * km + q] = carry;
                    wt[static_cast<size_t>(I) * km + q] = valid ? tab[I][q].w : 0.0;
                }
        };
        auto put_i16 = [&](const std::vector<int>& src, int i0, int n, int rel, int lim) {
            const size_t start = pl.gblob.size();
            for (int I = i0; I < i0 + n; ++I)
                for (int q = 0; q < km; ++q) {
                    int v = src[static_cast<size_t>(I) * km + q] - rel;
                    v = std::min(std::max(v, 0), std::max(lim - 1, 0));
                    if (v > 32767) throw ConfigError("invalid geometry: gather index overflow");
                    const short s16 = static_cast<short>(v);
                    const auto* p = reinterpret_cast<const unsigned char*>(&s16);
                    pl.gblob.insert(pl.gblob.end(), p, p + 2);
                }
            pl.gblob.resize(start + a16(pl.gblob.size() - start), 0);
        };
        auto put_wt = [&](const std::vector<double>& wt, int i0, int n) {
            const size_t start = pl.gblob.size();
            for (int I = i0; I < i0 + n; ++I)
                for (int q = 0; q < km; ++q) {
                    const double v = wt[static_cast<size_t>(I) * km + q];
                    if (elem_bytes == 8) {
                        const auto* p = reinterpret_cast<const unsigned char*>(&v);
                        pl.gblob.insert(pl.gblob.end(), p, p + 8);
                    } else {
                        const float f = static_cast<float>(v);
                        const auto* p = reinterpret_cast<const unsigned char*>(&f);
                        pl.gblob.insert(pl.gblob.end(), p, p + 4);
                    }
                }
            pl.gblob.resize(start + a16(pl.gblob.size() - start), 0);
        };
        auto put_raw = [&](const void* p, size_t n) {
            const auto* b = static_cast<const unsigned char*>(p);
            pl.gblob.insert(pl.gblob.end(), b, b + n);
        };
        auto pad16 = [&](size_t start) { pl.gblob.resize(start + a16(pl.gblob.size() - start), 0); };
        // direct-gather tables: per layer node (row or column) the first source of its
        // contiguous source run and km weights (zero-padded); first sources ascend with the
        // node (empty nodes carry their neighbour's), which the kernel's row ring relies on
        auto run_table = [&](const std::vector<std::vector<Entry>>& tab, std::vector<int>& first,
                             std::vector<double>& wt) {
            const int side = static_cast<int>(tab.size());
            first.assign(static_cast<size_t>(side), 0);
            wt.assign(static_cast<size_t>(side) * km, 0.0);
            int carry = 0;
            for (const auto& v : tab)
                if (!v.empty()) { carry = v.front().src; break; }
            for (int I = 0; I < side; ++I) {
                if (!tab[I].empty()) carry = tab[I].front().src;
                first[static_cast<size_t>(I)] = carry;
                for (const auto& en : tab[I]) {
                    const int a = en.src - carry;
                    if (a < 0 || a >= km) throw std::logic_error("gather tables: non-contiguous taps");
                    wt[static_cast<size_t>(I) * km + a] = en.w;
                }
                if (I > 0 && first[static_cast<size_t>(I)] < first[static_cast<size_t>(I - 1)])
                    throw std::logic_error("gather tables: descending taps");
            }
        };
        auto put_first = [&](const std::vector<int>& first, int i0, int n, int rel, int lim) {
            const size_t start = pl.gblob.size();
            for (int I = i0; I < i0 + n; ++I) {
                const int v = std::min(std::max(first[static_cast<size_t>(I)] - rel, 0), std::max(lim - 1, 0));
                if (v > 32767) throw ConfigError("invalid geometry: gather index overflow");
                const short s16 = static_cast<short>(v);
                const auto* p = reinterpret_cast<const unsigned char*>(&s16);
                pl.gblob.insert(pl.gblob.end(), p, p + 2);
            }
            pl.gblob.resize(start + a16(pl.gblob.size() - start), 0);
        };
        // column stencils: jlo/jhi of a (w, l) are the same in every row group (bs[2], bs[3])
        std::vector<size_t> coff_wl(static_cast<size_t>(W * L), 0);
        std::vector<int> dfirst;
        std::vector<double> dwt;
        for (int l = 0; l < L; ++l)
            for (int w = 0; w < W && direct; ++w) {
                const int side = gp.side[l];
                const int* bs = &pl.ti[static_cast<size_t>(gp.o_bs + ((w * L + l) * kMaxGU + 0) * 4)];
                const size_t start = pl.gblob.size();
                coff_wl[static_cast<size_t>(w * L + l)] = start;
                run_table(cols[w * L + l], dfirst, dwt);
                put_first(dfirst, 0, side, bs[2], bs[3] - bs[2]);
                put_wt(dwt, 0, side);
                if (pl.gblob.size() - start != col_bytes(side, bs[3] - bs[2])) throw std::logic_error("gather tables: size mismatch");
            }
        for (int l = 0; l < L; ++l)
            for (int w = 0; w < W && !direct; ++w) {
                const int side = gp.side[l];
                const int* bs = &pl.ti[static_cast<size_t>(gp.o_bs + ((w * L + l) * kMaxGU + 0) * 4)];
                const int jlo = bs[2], nc = bs[3] - bs[2];
                const auto& tx = colst[w * L + l];
                const size_t start = pl.gblob.size();
                coff_wl[static_cast<size_t>(w * L + l)] = start;
                size_t p0 = pl.gblob.size();
                for (int k = 0; k < side + 3; ++k) {
                    int f0 = nc;
                    for (int c = 0; c < nc; ++c)
                        if (tx[static_cast<size_t>(jlo + c)].idx >= k - 1) { f0 = c; break; }
                    const short v = static_cast<short>(f0);
                    put_raw(&v, 2);
                }
                pad16(p0);
                p0 = pl.gblob.size();
                for (int c = 0; c < nc; ++c) {
                    const short v = static_cast<short>(tx[static_cast<size_t>(jlo + c)].idx);
                    put_raw(&v, 2);
                }
                pad16(p0);
                p0 = pl.gblob.size();
                for (int c = 0; c < nc; ++c) {
                    const double fr = tx[static_cast<size_t>(jlo + c)].f;
                    if (elem_bytes == 8) put_raw(&fr, 8);
                    else {
                        const float ff = static_cast<float>(fr);
                        put_raw(&ff, 4);
                    }
                }
                pad16(p0);
                if (pl.gblob.size() - start != col_bytes(side, nc)) throw std::logic_error("gather tables: size mismatch");
            }
        // row-tap tables
        std::vector<size_t> roff_lu(static_cast<size_t>(L * kMaxGU), 0);
        std::vector<int> rsrc;
        std::vector<double> rwt;
        for (int l = 0; l < L; ++l)
            for (int u = 0; u < gp.side[l] / grp_rows(gp.side[l]); ++u) {
                roff_lu[static_cast<size_t>(l * kMaxGU + u)] = pl.gblob.size();
                const int side = gp.side[l];
                const int Rl = grp_rows(side), I0 = u * Rl;
                for (int w = 0; w < W; ++w) {
                    const int* bs = &pl.ti[static_cast<size_t>(gp.o_bs + ((w * L + l) * kMaxGU + u) * 4)];
                    const size_t start = pl.gblob.size();
                    if (direct) {
                        run_table(rows[w * L + l], rsrc, rwt);
                        put_first(rsrc, I0, Rl, bs[0], bs[1] - bs[0]);
                    } else {
                        padded(rows[w * L + l], rsrc, rwt);
                        put_i16(rsrc, I0, Rl, bs[0], bs[1] - bs[0]);
                    }
                    put_wt(rwt, I0, Rl);
                    if (pl.gblob.size() - start != row_bytes(Rl)) throw std::logic_error("gather tables: size mismatch");
                }
            }
        // staging descriptors per (layer, row group, WFS), kGDescInts ints (mirrors GDesc in cluster.cuh):
        //   ilo ihi jlo jhi | psi source element offset | psi stage byte offset in its chunk |
        //   row table offset, bytes | column stencil offset, bytes | pad pad
        // A chunk stages [its WFS's row tables | their column stencils | psi blocks].
        pl.ti.resize((pl.ti.size() + 3) & ~size_t(3), 0);  // int4-aligned
        gp.o_gd = static_cast<int>(pl.ti.size());
        pl.ti.resize(pl.ti.size() + static_cast<size_t>(L * kMaxGU * kMaxW * kGDescInts), 0);
        pl.td.resize(pl.ti.size(), 0.0);
        for (int l = 0; l < L; ++l)
            for (int u = 0; u < gp.side[l] / grp_rows(gp.side[l]); ++u) {
                const int Rl = grp_rows(gp.side[l]);
                for (int k = 0; k < gp.nchunk; ++k) {
                    size_t tsum = 0, psum = 0;
                    for (int w = gp.gchunk[k]; w < gp.gchunk[k + 1]; ++w) {
                        tsum += need_of(w, l, u).first;
                        psum += need_of(w, l, u).second;
                    }
                    size_t poff = tsum;
                    for (int w = gp.gchunk[k]; w < gp.gchunk[k + 1]; ++w) {
                        const int* bs = &pl.ti[static_cast<size_t>(gp.o_bs + ((w * L + l) * kMaxGU + u) * 4)];
                        const auto nb = need_of(w, l, u);
                        int* d = &pl.ti[static_cast<size_t>(gp.o_gd + ((l * kMaxGU + u) * kMaxW + w) * kGDescInts)];
                        d[0] = bs[0]; d[1] = bs[1]; d[2] = bs[2]; d[3] = bs[3];
                        d[4] = gp.woff[w] + bs[0] * (g.wfs[w].n_subap + 1);
                        d[5] = static_cast<int>(poff);
                        d[6] = static_cast<int>(roff_lu[static_cast<size_t>(l * kMaxGU + u)] + static_cast<size_t>(w) * row_bytes(Rl));
                        d[7] = static_cast<int>(row_bytes(Rl));
                        d[8] = static_cast<int>(coff_wl[static_cast<size_t>(w * L + l)]);
                        d[9] = static_cast<int>(col_bytes(gp.side[l], bs[3] - bs[2]));
                        d[10] = static_cast<int>(psum);  // psi bytes of the chunk per instance (k_gather_direct)
                        poff += nb.second;
                    }
                }
            }
    }
    pl.perm = coeff_perm(gp);
    return pl;
}

template <typename T>
T* dalloc(size_t n) {
    void* p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    CK(cudaMemset(p, 0, std::max<size_t>(n, 1) * sizeof(T)));
    return static_cast<T*>(p);
}

struct DevFree {
    std::vector<void*> ptrs;
    void add(void* p) { ptrs.push_back(p); }
    ~DevFree() {
        for (void* p : ptrs) cudaFree(p);
    }
};

// Per-batch device workspace of one element type.
template <typename T>
struct Work {
    int count = 0;
    Bufs<T> bf{};
    T *in = nullptr, *out = nullptr, *a = nullptr;
    double* meas = nullptr;
    double* meas2 = nullptr;
    size_t frame_out_bytes = 0;  // rho_log | status | nlog block (state workspaces)
    void alloc(const GeoParams& gp, int cnt, DevFree& fr, bool state) {
        count = cnt;
        const size_t n = static_cast<size_t>(gp.n) * cnt;
        auto A = [&](auto* tag, size_t k) {
            using U = std::remove_pointer_t<decltype(tag)>;
            U* p = dalloc<U>(k);
            fr.add(p);
            return p;
        };
        bf.phi = A((T*)nullptr, n);
        bf.y = A((T*)nullptr, n);
        bf.psi = A((T*)nullptr, static_cast<size_t>(gp.Nw) * cnt + 16);  // bulk copies may read 16 B past rows
        meas = A((double*)nullptr, static_cast<size_t>(gp.S) * cnt);
        meas2 = A((double*)nullptr, static_cast<size_t>(gp.S) * cnt);
        bf.meas = meas;
        in = A((T*)nullptr, n);
        out = A((T*)nullptr, n);
        a = A((T*)nullptr, static_cast<size_t>(gp.A) * cnt);
        bf.in = in;
        bf.out = out;
        bf.a_out = a;
        bf.a_prev2 = a;
        if (state) {
            bf.c = A((T*)nullptr, n);
            bf.b = A((T*)nullptr, n);
            bf.r = A((T*)nullptr, n);
            bf.p = A((T*)nullptr, n);
            bf.q = A((T*)nullptr, n);
            bf.mz = A((T*)nullptr, n);
            const size_t aa = static_cast<size_t>(gp.A) * cnt;
            bf.a_prev2 = A((T*)nullptr, aa);
            bf.a_prev = A((T*)nullptr, aa);
            bf.a_out = A((T*)nullptr, aa);
            bf.carry = A((Carry*)nullptr, static_cast<size_t>(gp.iters + 1) * cnt);
            const size_t np = static_cast<size_t>(gp.iters) * gp.L * kMaxC * cnt;
            bf.rho_part = A((double*)nullptr, np);
            bf.mu_part = A((double*)nullptr, np);
            // per-frame host outputs in one block (one D2H copy): rho_log [cnt][iters] doubles,
            // then status [cnt] and nlog [cnt] ints
            const size_t nr = static_cast<size_t>(gp.iters) * cnt;
            frame_out_bytes = nr * sizeof(double) + 2 * static_cast<size_t>(cnt) * sizeof(int);
            auto* blk = A((unsigned char*)nullptr, frame_out_bytes);
            bf.rho_log = reinterpret_cast<double*>(blk);
            bf.status = reinterpret_cast<int*>(blk + nr * sizeof(double));
            bf.nlog = bf.status + cnt;
        }
        CK(cudaDeviceSynchronize());  // the zero fills (legacy stream) land before stream work uses the buffers
    }
};

}  // namespace

// ---------------------------------------------------------------------------
// Typed launchers
// ---------------------------------------------------------------------------
// Programmatic dependent launch between the frame's kernels: opt-in
// (FEWHA_PDL=1) -- measured neutral-to-negative on the ELT frame.
inline bool pdl_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("FEWHA_PDL");  // on by default (measured 0.210 -> 0.202 ms); FEWHA_PDL=0 disables
        return !(v && v[0] == '0');
    }();
    return on;
}

template <typename T>
struct Launch {
    static size_t wfs_smem(const GeoParams& gp, int ni = 1) { return wfs_tile_smem<T>(std::max(gp.L, gp.M), ni); }
    // instances per WFS-tile CTA for a batch of `count` (FEWHA_WFS_NI overrides)
    static int wfs_ni(int count) {
        static const int env = [] {
            const char* v = std::getenv("FEWHA_WFS_NI");
            return v ? std::atoi(v) : 0;
        }();
        if (count <= 2) return 1;
        // batches: 4 instances per CTA (B = 64 fp64 per step: 2.284 ms with 2 at 6 CTAs/SM,
        // 2.237 with 4 at 4/SM; fp32 -17 % against 1 instance)
        return env == 1 || env == 2 || env == 4 ? env : 4;
    }
    static size_t gather_smem(const GeoParams& gp) {
        return ((static_cast<size_t>(gp.gbuf_bytes) * gp.gather_ni + 15) & ~size_t(15)) + static_cast<size_t>(gp.chunk_bytes);
    }
    static size_t a16(size_t v) { return (v + 15) & ~size_t(15); }
    // shared-memory maps: clayout.hpp (the kernels derive the same offsets)
    static size_t inv_cl_smem(const GeoParams& gp, int flen, int staged = 1) {
        return static_cast<size_t>(
            clay::inv_smem(gp.maxside, gp.ccl, gp.ctail, flen, static_cast<int>(sizeof(T)), staged).total);
    }
    // TMA staging of the inverse kernel's operands pays for a single instance (latency);
    // batches stream them from global memory at twice the residency
    // 16-CTA clusters stream too: a staged inverse (one CTA per SM) would not let
    // nine 16-CTA clusters be resident at once
    static int inv_staged_for(const GeoParams& gp, int count) {
        const char* v = std::getenv("FEWHA_INV_STAGE");  // read per plan (tests switch it between engines)
        const int mode = v ? std::atoi(v) : -1;
        return mode >= 0 ? (mode ? 1 : 0) : (count <= 2 && gp.ccl <= 8 ? 1 : 0);
    }
    static size_t fwd_cl_smem(const GeoParams& gp, int flen) {
        return static_cast<size_t>(
            clay::fwd_smem(gp.maxside, gp.ccl, gp.ctail, flen, static_cast<int>(sizeof(T)), gp.tonly).total);
    }

#define FEWHA_FLEN_SWITCH(flen, CALL)          \
    switch (flen) {                            \
        case 2: CALL(2); break;                \
        case 4: CALL(4); break;                \
        case 6: CALL(6); break;                \
        case 8: CALL(8); break;                \
        case 10: CALL(10); break;              \
        case 12: CALL(12); break;              \
        case 14: CALL(14); break;              \
        case 16: CALL(16); break;              \
        case 18: CALL(18); break;              \
        default: CALL(20); break;              \
    }

    // The dynamic shared-memory opt-in is a per-function, process-global attribute:
    // set it to the device maximum once so engines of different geometries coexist.
    static void set_attrs(const GeoParams& gp, int flen) {
        int dev = 0, maxopt = 0;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&maxopt, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        if (inv_cl_smem(gp, flen) > static_cast<size_t>(maxopt) || fwd_cl_smem(gp, flen) > static_cast<size_t>(maxopt) ||
            wfs_smem(gp) > static_cast<size_t>(maxopt) || gather_smem(gp) > static_cast<size_t>(maxopt))
            throw ConfigError("invalid geometry: layer kernels exceed the device's shared memory");
        const size_t m = static_cast<size_t>(maxopt);
#define FEWHA_SET(N) CK((set_layer_cluster_attrs<T, N>(m, m)))
        FEWHA_FLEN_SWITCH(flen, FEWHA_SET)
#undef FEWHA_SET
        auto opt_in = [&](auto kernel, size_t need) {
            cudaFuncAttributes fa{};
            CK(cudaFuncGetAttributes(&fa, kernel));
            if (need + fa.sharedSizeBytes > m)
                throw ConfigError("invalid geometry: layer kernels exceed the device's shared memory");
            CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(m - fa.sharedSizeBytes)));
        };
        opt_in(k_wfs<T, false, FEWHA_WFS_MINB_LAT>, wfs_smem(gp));
        opt_in(k_wfs<T, true, FEWHA_WFS_MINB_LAT>, wfs_smem(gp));
        opt_in(k_wfs<T, false, FEWHA_WFS_MINB_BATCH>, wfs_smem(gp));
        opt_in(k_wfs<T, true, FEWHA_WFS_MINB_BATCH>, wfs_smem(gp));
        opt_in(k_wfs<T, false, kWfsNi2Minb, 2>, wfs_smem(gp, 2));
        opt_in(k_wfs<T, true, kWfsNi2Minb, 2>, wfs_smem(gp, 2));
        opt_in(k_wfs<T, false, kWfsNi4Minb<T>, 4>, wfs_smem(gp, 4));
        opt_in(k_wfs<T, true, kWfsNi4Minb<T>, 4>, wfs_smem(gp, 4));
        opt_in(k_gather<T, 2>, gather_smem(gp));
        opt_in(k_gather<T, 3>, gather_smem(gp));
        opt_in(k_gather<T, 4>, gather_smem(gp));
#define FEWHA_GD_OPT(M, N) opt_in(k_gather_direct<T, M, N>, gather_smem(gp));
        FEWHA_GD_OPT(2, 1) FEWHA_GD_OPT(3, 1) FEWHA_GD_OPT(4, 1)
        FEWHA_GD_OPT(2, 2) FEWHA_GD_OPT(3, 2) FEWHA_GD_OPT(4, 2)
        FEWHA_GD_OPT(2, 4) FEWHA_GD_OPT(3, 4) FEWHA_GD_OPT(4, 4)
#undef FEWHA_GD_OPT
    }
    // layer kernels: grid (C, L, count), cluster (C,1,1)
    static void cl(int flen, bool inverse, const GeoParams& gp, const Bufs<T>& bf, int mode, int it, int count,
                   cudaStream_t st, int fit_term = 1) {
        GeoParams g2 = gp;
        g2.inv_staged = inv_staged_for(gp, count);
        const size_t smem = inverse ? inv_cl_smem(g2, flen, g2.inv_staged) : fwd_cl_smem(g2, flen);
#define FEWHA_LAUNCH(N) CK((launch_layer_cluster<T, N>(inverse, g2, bf, mode, it, count, st, fit_term, smem)))
        FEWHA_FLEN_SWITCH(flen, FEWHA_LAUNCH)
#undef FEWHA_LAUNCH
    }
    // whole-layer kernels (batched plans): grid (L, count)
    static void whole(int flen, bool inverse, const GeoParams& gp, const Bufs<T>& bf, int mode, int it, int count,
                      cudaStream_t st, int fit_term = 1) {
#define FEWHA_LAUNCH(N) CK((launch_layer_whole<T, N>(inverse, gp, bf, mode, it, count, st, fit_term)))
        FEWHA_FLEN_SWITCH(flen, FEWHA_LAUNCH)
#undef FEWHA_LAUNCH
    }
    // whole-layer fused forward (fmode, fit) + inverse (imode, iit): one launch, the L layer
    // CTAs of an instance meet at a ticketed barrier (k_fwd_inv_layer; ctr: count + 1 counters)
    static void whole_fused(int flen, const GeoParams& gp, const Bufs<T>& bf, int fmode, int fit, int imode, int iit,
                            int count, cudaStream_t st, unsigned long long* ctr) {
#define FEWHA_LAUNCH(N) CK((launch_layer_whole_fused<T, N>(gp, bf, fmode, fit, imode, iit, count, st, 1, ctr)))
        FEWHA_FLEN_SWITCH(flen, FEWHA_LAUNCH)
#undef FEWHA_LAUNCH
    }
    static int whole_fused_per_sm(const GeoParams& gp, int flen) {
        int per_sm = 0;
#define FEWHA_CAP(N) CK((whole_fused_capacity<T, N>(gp, &per_sm)))
        FEWHA_FLEN_SWITCH(flen, FEWHA_CAP)
#undef FEWHA_CAP
        return per_sm;
    }
    // fused forward (fmode, fit) + inverse (imode, iit): one cooperative cluster launch
    static void fused(int flen, const GeoParams& gp, const Bufs<T>& bf, int fmode, int fit, int imode, int iit,
                      int count, cudaStream_t st, unsigned long long* bar) {
        GeoParams g2 = gp;
        g2.inv_staged = inv_staged_for(gp, count);
        const size_t smem = fused_cl_smem(g2, flen, g2.inv_staged);
#define FEWHA_LAUNCH(N) \
    CK((launch_fused_cluster<T, N>(g2, bf, fmode, fit, imode, iit, count, st, 1, smem, bar, pdl_enabled() ? 1 : 0)))
        FEWHA_FLEN_SWITCH(flen, FEWHA_LAUNCH)
#undef FEWHA_LAUNCH
    }
    static size_t fused_cl_smem(const GeoParams& gp, int flen, int staged) {
        return std::max(inv_cl_smem(gp, flen, staged), fwd_cl_smem(gp, flen));
    }
    // clusters of the fused kernel resident at once (0: it does not fit)
    static int fused_capacity(const GeoParams& gp, int flen, int count) {
        GeoParams g2 = gp;
        g2.inv_staged = inv_staged_for(gp, count);
        int clusters = 0;
#define FEWHA_CAP(N) CK((fused_cluster_capacity<T, N>(g2, fused_cl_smem(g2, flen, g2.inv_staged), &clusters)))
        FEWHA_FLEN_SWITCH(flen, FEWHA_CAP)
#undef FEWHA_CAP
        return clusters;
    }
    // programmatic dependent launch config (the kernels call griddepcontrol)
    static cudaLaunchConfig_t pdl_cfg(dim3 grid, size_t smem, cudaStream_t st, cudaLaunchAttribute* attr,
                                      int threads = 256) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(threads, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cfg;
    }
    static void wfs(bool rhs, const GeoParams& gp, const Bufs<T>& bf, int with_dm, int count, cudaStream_t st) {
        cudaLaunchAttribute attr[1];
        const int ni = wfs_ni(count);
        cudaLaunchConfig_t cfg =
            pdl_cfg(dim3(gp.wt_count, (count + ni - 1) / ni), wfs_smem(gp, ni), st, attr, kWfsThreads);
        constexpr int LAT = FEWHA_WFS_MINB_LAT, BAT = FEWHA_WFS_MINB_BATCH;
        static const bool bat_lat = [] {  // profiling: batches on the latency instantiation
            const char* v = std::getenv("FEWHA_WFS_BATCH_MINB");
            return v && std::atoi(v) == LAT;
        }();
        if (ni == 2) {
            if (rhs) CK(cudaLaunchKernelEx(&cfg, k_wfs<T, true, kWfsNi2Minb, 2>, gp, bf, with_dm, count));
            else CK(cudaLaunchKernelEx(&cfg, k_wfs<T, false, kWfsNi2Minb, 2>, gp, bf, with_dm, count));
        } else if (ni == 4) {
            if (rhs) CK(cudaLaunchKernelEx(&cfg, k_wfs<T, true, kWfsNi4Minb<T>, 4>, gp, bf, with_dm, count));
            else CK(cudaLaunchKernelEx(&cfg, k_wfs<T, false, kWfsNi4Minb<T>, 4>, gp, bf, with_dm, count));
        } else if (count <= 2 || bat_lat) {
            if (rhs) CK(cudaLaunchKernelEx(&cfg, k_wfs<T, true, LAT>, gp, bf, with_dm, count));
            else CK(cudaLaunchKernelEx(&cfg, k_wfs<T, false, LAT>, gp, bf, with_dm, count));
        } else {
            if (rhs) CK(cudaLaunchKernelEx(&cfg, k_wfs<T, true, BAT>, gp, bf, with_dm, count));
            else CK(cudaLaunchKernelEx(&cfg, k_wfs<T, false, BAT>, gp, bf, with_dm, count));
        }
    }
    // y = sum_w P^T psi_w: one CTA per gp.grows rows of every layer
    static void gather(const GeoParams& gp, const Bufs<T>& bf, int count, cudaStream_t st) {
        cudaLaunchAttribute attr[1];
        const int groups = gp.maxside / std::min(gp.grows, gp.maxside);
        if (gp.gather_direct) {
            const int ni = gp.gather_ni;
            // dependents launched after the contraction for batches (batch 64 fp64: 2.48 vs
            // 2.63 ms per step with the early trigger, whose waiting forward CTAs slow the
            // gather's last waves), at the start for single frames; FEWHA_GATHER_LATE overrides
            static const int late_env = [] {
                const char* v = std::getenv("FEWHA_GATHER_LATE");
                return v ? std::atoi(v) : -1;
            }();
            const int late = late_env >= 0 ? late_env : count > 2;
            cudaLaunchConfig_t cfg = pdl_cfg(dim3(groups, gp.L, (count + ni - 1) / ni), gather_smem(gp), st, attr);
#define FEWHA_GD_LAUNCH(N)                                                                            \
    if (gp.gather_minb == 4) CK(cudaLaunchKernelEx(&cfg, k_gather_direct<T, 4, N>, gp, bf, count, late));      \
    else if (gp.gather_minb == 3) CK(cudaLaunchKernelEx(&cfg, k_gather_direct<T, 3, N>, gp, bf, count, late)); \
    else CK(cudaLaunchKernelEx(&cfg, k_gather_direct<T, 2, N>, gp, bf, count, late));
            if (ni == 4) {
                FEWHA_GD_LAUNCH(4)
            } else if (ni == 2) {
                FEWHA_GD_LAUNCH(2)
            } else {
                FEWHA_GD_LAUNCH(1)
            }
#undef FEWHA_GD_LAUNCH
            return;
        }
        cudaLaunchConfig_t cfg = pdl_cfg(dim3(groups, gp.L, count), gather_smem(gp), st, attr);
        if (gp.gather_minb == 4) CK(cudaLaunchKernelEx(&cfg, k_gather<T, 4>, gp, bf));
        else if (gp.gather_minb == 3) CK(cudaLaunchKernelEx(&cfg, k_gather<T, 3>, gp, bf));
        else CK(cudaLaunchKernelEx(&cfg, k_gather<T, 2>, gp, bf));
    }
    static void fit(const GeoParams& gp, const Bufs<T>& bf, int step, int count, cudaStream_t st) {
        cudaLaunchAttribute attr[1];
        cudaLaunchConfig_t cfg = pdl_cfg(dim3((gp.A + 255) / 256, count), 0, st, attr);
        CK(cudaLaunchKernelEx(&cfg, k_fit_control<T>, gp, bf, step));
    }
};

// ---------------------------------------------------------------------------
// Engine implementation
// ---------------------------------------------------------------------------
struct EngineImpl {
    Geometry g;
    int precision, batch, device, flen;
    Plan plan;
    DevFree fr;
    GeoParams gp{};      // with device table pointers (engine precision)
    GeoParams gp64{};    // fp64 plan for the preconditioner probes (== gp in fp64 engines)
    GeoParams gpf{};     // plan of the frame's per-WFS kernels (== gp unless sharded)
    // StepTelemetry (reconstructor.hpp:94-102): opt-in event-record nodes in the frame graph
    bool telemetry_on = false, telem_pending = false;
    long long step_counter = 0;
    std::vector<cudaEvent_t> tev;
    std::vector<int> tkind;
    // per-WFS sharding: this engine owns WFS [gpf.wa, gpf.wb)
    void* host_out = nullptr;  // pinned staging of the per-frame rho/status/nlog block
    bool sharded = false;
    int shard_rank = 0, shard_world = 1;
    std::vector<void*> ypart;  // [iters+1] partial adjoint layer sums [B][n], one per exchange
    ncclComm_t comm = nullptr;  // multi-process exchange (NCCL); null for in-process groups
    cudaStream_t stream = nullptr, user_stream = nullptr;
    bool own_stream = false;
    cudaGraphExec_t graph = nullptr;
    bool has_precond = false;
    // fused forward + inverse launches (k_fwd_inv_cluster): opt-in (FEWHA_FUSE=1) when
    // every instance's L clusters fit the device at once; per-instance
    // monotonic barrier counters
    bool fuse_ok = false;
    unsigned long long* fbar = nullptr;
    // batched plans: layer transforms one CTA per (layer, instance) (layer_whole.cuh)
    bool whole_layer = false;
    bool use_whole() const { return whole_layer && !sharded && peer_sum.empty(); }
    // whole-layer plans: forward(k) + inverse(k+1) in one launch (k_fwd_inv_layer), opt-in
    // (FEWHA_FUSE_WHOLE=1; measured no faster than the split launches)
    bool whole_fuse = false;
    unsigned long long* wbar = nullptr;  // [batch] instance barrier counters + the ticket counter
    bool use_whole_fused() const { return whole_fuse && use_whole(); }
    bool fused_frame() const { return fuse_ok && !whole_layer && !telemetry_on && !(sharded && !comm); }
    // optional per-phase timestamps of the cluster kernels (profiling only)
    unsigned long long* stamp_buf = nullptr;
    int stamp_slot = -1;  // < 0: stamping off
    static constexpr int kStampSlots = 32, kStampBlocks = 16384;
    GeoParams gps() {
        GeoParams g2 = gpf;
        if (stamp_slot >= 0 && stamp_slot < kStampSlots) {
            g2.stamps = stamp_buf + static_cast<size_t>(stamp_slot++) * kStampBlocks * 16;
        }
        return g2;
    }
    std::vector<double> precond;
    std::unique_ptr<struct SimState> sim;  // closed-loop simulation harness, built on first use
    void* jac = nullptr;
    void* jinv = nullptr;  // 1/J
    // state (precision T) -- one of the two is used
    Work<double> sd, od, pd;  // state / ops / probes (fp64)
    Work<float> sf, of;        // state / ops (fp32)

    cudaStream_t s() const { return user_stream ? user_stream : stream; }

    template <typename T>
    Work<T>& state();
    template <typename T>
    Work<T>& ops();

    GeoParams upload_plan(const Plan& plan) {
        int* ti = dalloc<int>(plan.ti.size());
        double* td = dalloc<double>(plan.td.size());
        float* tf = dalloc<float>(plan.td.size());
        std::uint8_t* mk = dalloc<std::uint8_t>(plan.masks.size());
        int* wt = dalloc<int>(plan.wtiles.size());
        unsigned char* gb = dalloc<unsigned char>(plan.gblob.size());
        fr.add(gb);
        unsigned char* tb = dalloc<unsigned char>(plan.tblob.size());
        fr.add(tb);
        if (!plan.tblob.empty())
            CK(cudaMemcpy(tb, plan.tblob.data(), plan.tblob.size(), cudaMemcpyHostToDevice));
        if (!plan.gblob.empty())
            CK(cudaMemcpy(gb, plan.gblob.data(), plan.gblob.size(), cudaMemcpyHostToDevice));
        for (void* p : {(void*)ti, (void*)td, (void*)tf, (void*)mk, (void*)wt}) fr.add(p);
        std::vector<float> tdf(plan.td.begin(), plan.td.end());
        CK(cudaMemcpy(ti, plan.ti.data(), plan.ti.size() * sizeof(int), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(td, plan.td.data(), plan.td.size() * sizeof(double), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(tf, tdf.data(), tdf.size() * sizeof(float), cudaMemcpyHostToDevice));
        if (!plan.masks.empty())
            CK(cudaMemcpy(mk, plan.masks.data(), plan.masks.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(wt, plan.wtiles.data(), plan.wtiles.size() * sizeof(int), cudaMemcpyHostToDevice));
        GeoParams g = plan.gp;
        g.ti = ti;
        g.td = td;
        g.tf = tf;
        g.masks = mk;
        g.wtiles = wt;
        g.gblob = gb;
        g.tblob = tb;
        return g;
    }

    void invalidate_graph() {
        if (graph) cudaGraphExecDestroy(graph);
        graph = nullptr;
        if (graph_tmpl) cudaGraphDestroy(graph_tmpl);
        graph_tmpl = nullptr;
        fit_node = nullptr;
        fit_a_host = nullptr;
    }

    // Zero-copy DM output: when the caller's DM buffer is page-locked, the frame's
    // fit/control kernel also stores a1 straight into it (posted PCIe writes inside
    // the kernel instead of a D2H copy after the graph); its `a_host` argument is
    // repointed per call.
    cudaGraph_t graph_tmpl = nullptr;   // the captured frame (node handles for updates)
    cudaGraphNode_t fit_node = nullptr;  // k_fit_control of the frame
    double* fit_a_host = nullptr;        // what the node currently writes to
    template <typename T>
    void find_fit_node() {
        size_t nn = 0;
        CK(cudaGraphGetNodes(graph_tmpl, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        CK(cudaGraphGetNodes(graph_tmpl, nodes.data(), &nn));
        for (auto nd : nodes) {
            cudaGraphNodeType ty;
            CK(cudaGraphNodeGetType(nd, &ty));
            if (ty != cudaGraphNodeTypeKernel) continue;
            cudaKernelNodeParams kp{};
            CK(cudaGraphKernelNodeGetParams(nd, &kp));
            if (kp.func == reinterpret_cast<void*>(k_fit_control<T>)) fit_node = nd;
        }
    }
    template <typename T>
    void set_fit_a_host(double* a) {
        if (!fit_node || a == fit_a_host) return;
        cudaKernelNodeParams kp{};
        CK(cudaGraphKernelNodeGetParams(fit_node, &kp));
        Bufs<T> bf = *static_cast<const Bufs<T>*>(kp.kernelParams[1]);
        bf.a_host = a;
        void* args[3] = {kp.kernelParams[0], &bf, kp.kernelParams[2]};
        kp.kernelParams = args;
        CK(cudaGraphExecKernelNodeSetParams(graph, fit_node, &kp));
        fit_a_host = a;
    }

    // ---- one frame of Reconstructor::step on the state workspace ----------
    // The frame is iters+2 segments; segments 0..iters end with an adjoint gather
    // whose layer sums are exchanged between shards when sharded:
    //   seg 0          RHS: Gamma^T C^-1 (s + Gamma P_dm a) -> sum P^T psi
    //   seg 1          W (RHS, r update) | W^-1 z_0 | Gamma..P | sum P^T psi
    //   seg k (2..it)  W (PCG k-2)       | update + W^-1 z_{k-1} | ... | sum P^T psi
    //   seg it+1       W (PCG it-1)      | last update + W^-1 c | fit + control
    // `mark(kind)` runs after every launch (profiling hook; a no-op for capture).
    template <typename T>
    Bufs<T> frame_bufs() {
        Bufs<T> bf = state<T>().bf;
        bf.jac = static_cast<const T*>(jac);
        bf.jinv = static_cast<const T*>(jinv);
        bf.frame_host = static_cast<unsigned char*>(host_out);  // page-locked mirror (null: copied)
        return bf;
    }
    int n_segments() const { return gp.iters + 2; }

    // in-process shard group: the members' partial buffers of the previous segment, read
    // by this member's next forward kernel (set by group_step_device)
    std::vector<const void*> peer_sum;

    template <typename T, typename Mark>
    void launch_segment(int seg, cudaStream_t st, Mark&& mark) {
        Bufs<T> bf = frame_bufs<T>();
        const int B = batch, it = gp.iters;
        if (seg >= 1 && !peer_sum.empty()) {
            bf.nsum = static_cast<int>(peer_sum.size());
            for (size_t r = 0; r < peer_sum.size(); ++r) bf.ysum[r] = static_cast<const T*>(peer_sum[r]);
        }
        const bool wl = use_whole();
        if (seg >= 1 && use_whole_fused()) {  // W of the previous gather and the next W^-1 in one launch
            const int fmode = seg == 1 ? kRhs : kPcg, fit = seg == 1 ? 0 : seg - 2;
            if (seg <= it) {
                Launch<T>::whole_fused(flen, gps(), bf, fmode, fit, kPcg, seg - 1, B, st, wbar);
                mark(seg == 1 ? kKindFwdRhsInv0 : kKindFwdInvPcg);
                Launch<T>::wfs(false, gps(), bf, 0, B, st);
                mark(kKindWfs);
                Launch<T>::gather(gps(), bf, B, st);
                mark(kKindGather);
                return;
            }
            Launch<T>::whole_fused(flen, gps(), bf, fmode, fit, kFit, 0, B, st, wbar);
            mark(kKindFwdInvFit);
            Launch<T>::fit(gpf, bf, 1, B, st);
            mark(kKindFit);
            return;
        }
        auto layer = [&](bool inverse, int mode, int k) {
            if (wl) Launch<T>::whole(flen, inverse, gps(), bf, mode, k, B, st);
            else Launch<T>::cl(flen, inverse, gps(), bf, mode, k, B, st);
        };
        auto gather = [&] {
            Bufs<T> gb = bf;
            if (sharded) gb.y = static_cast<T*>(ypart[static_cast<size_t>(seg)]);  // partial sums
            Launch<T>::gather(gps(), gb, B, st);
            mark(kKindGather);
        };
        if (seg == 0) {  // RHS with the pseudo open-loop term (reconstructor.hpp:316-323)
            Launch<T>::wfs(true, gps(), bf, gp.closed, B, st);
            mark(kKindWfsRhs);
            gather();
            return;
        }
        if (fused_frame()) {  // W of the previous gather and the next W^-1 in one launch
            const int fmode = seg == 1 ? kRhs : kPcg, fit = seg == 1 ? 0 : seg - 2;
            if (seg <= it) {
                Launch<T>::fused(flen, gps(), bf, fmode, fit, kPcg, seg - 1, B, st, fbar);
                mark(seg == 1 ? kKindFwdRhsInv0 : kKindFwdInvPcg);
                Launch<T>::wfs(false, gps(), bf, 0, B, st);
                mark(kKindWfs);
                gather();
                return;
            }
            Launch<T>::fused(flen, gps(), bf, fmode, fit, kFit, 0, B, st, fbar);
            mark(kKindFwdInvFit);
            Launch<T>::fit(gpf, bf, 1, B, st);
            mark(kKindFit);
            return;
        }
        // W of the previous gather: the RHS (r += b1 - b) or PCG iteration seg-2
        if (seg == 1) {
            layer(false, kRhs, 0);
            mark(kKindFwdRhs);
        } else {
            layer(false, kPcg, seg - 2);
            mark(kKindFwdPcg);
        }
        if (seg <= it) {  // fused PCG (pcg.hpp:68-106): update of k-1 fused into k's W^-1
            const int k = seg - 1;
            layer(true, kPcg, k);
            mark(k == 0 ? kKindInvPcg0 : kKindInvPcg);
            Launch<T>::wfs(false, gps(), bf, 0, B, st);
            mark(kKindWfs);
            gather();
            return;
        }
        // last update + fitting W^-1 c, then fit + control + rotation
        layer(true, kFit, 0);
        mark(kKindInvFit);
        Launch<T>::fit(gpf, bf, 1, B, st);
        mark(kKindFit);
    }

    // NCCL exchange of segment `seg`'s partial layer sums (multi-process shards)
    template <typename T>
    void exchange_nccl(int seg, cudaStream_t st) {
        const auto& api = NcclApi::get();
        api.check(api.AllReduce(ypart[static_cast<size_t>(seg)], state<T>().bf.y,
                                static_cast<size_t>(gp.n) * batch, sizeof(T) == 8 ? ncclFloat64 : ncclFloat32,
                                ncclSum, comm, st),
                  "ncclAllReduce");
    }

    template <typename T, typename Mark>
    void launch_frame(cudaStream_t st, Mark&& mark) {
        if (sharded && !comm) throw ArgError("shard group members step through fewha_gpu_group_step_device");
        for (int seg = 0; seg < n_segments(); ++seg) {
            launch_segment<T>(seg, st, mark);
            if (sharded && seg <= gp.iters) exchange_nccl<T>(seg, st);
        }
        CK(cudaGetLastError());
    }

    template <typename T>
    void launch_frame(cudaStream_t st) {
        launch_frame<T>(st, [](int) {});
    }

    // Eager frame with an event after every launch: per-launch device times.
    template <typename T>
    int profile_frame(float* ms, int* kinds, int max) {
        const cudaStream_t st = s();
        std::vector<cudaEvent_t> ev;
        std::vector<int> kk;
        cudaEvent_t e0;
        CK(cudaEventCreate(&e0));
        CK(cudaEventRecord(e0, st));
        launch_frame<T>(st, [&](int kind) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            CK(cudaEventRecord(e, st));
            ev.push_back(e);
            kk.push_back(kind);
        });
        CK(cudaEventSynchronize(ev.back()));
        int n = 0;
        cudaEvent_t prev = e0;
        for (size_t i = 0; i < ev.size(); ++i) {
            float t = 0.f;
            CK(cudaEventElapsedTime(&t, prev, ev[i]));
            if (n < max) {
                ms[n] = t;
                kinds[n] = kk[i];
                ++n;
            }
            prev = ev[i];
        }
        for (auto e : ev) cudaEventDestroy(e);
        cudaEventDestroy(e0);
        return n;
    }

    template <typename T>
    void ensure_graph() {
        if (graph) return;
        if (sharded && !comm) throw ArgError("shard group members step through fewha_gpu_group_step_device");
        cudaGraph_t gr;
        // profiling (FEWHA_GRAPH_STAMPS=1 after fewha_gpu_phase_stamps enabled the buffer): the
        // captured launches record their phase stamps, so the overlapped (PDL) timeline of a
        // real graph frame can be read back
        struct Stamps {
            int& slot;
            bool on;
            ~Stamps() {
                if (on) slot = -1;
            }
        } graph_stamps{stamp_slot, stamp_buf != nullptr && std::getenv("FEWHA_GRAPH_STAMPS") != nullptr};
        if (graph_stamps.on) stamp_slot = 0;
        CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
        if (telemetry_on) {  // event-record nodes around every launch (StepTelemetry)
            tkind.clear();
            size_t k = 0;
            auto rec = [&] {
                if (k == tev.size()) {
                    cudaEvent_t e;
                    CK(cudaEventCreate(&e));
                    tev.push_back(e);
                }
                CK(cudaEventRecordWithFlags(tev[k++], stream, cudaEventRecordExternal));  // a graph node
            };
            rec();
            launch_frame<T>(stream, [&](int kind) {
                tkind.push_back(kind);
                rec();
            });
        } else {
            launch_frame<T>(stream);
        }
        CK(cudaStreamEndCapture(stream, &gr));
        CK(cudaGraphInstantiate(&graph, gr, 0));
        graph_tmpl = gr;
        find_fit_node<T>();
    }

    // ---- apply_M on a double workspace (also the preconditioner probes) ----
    template <typename T>
    void apply_M_dev(Work<T>& w, int count, cudaStream_t st, const GeoParams& g) {
        Bufs<T> bf = w.bf;
        Launch<T>::cl(flen, true, g, bf, kPlain, 0, count, st);
        Launch<T>::wfs(false, g, bf, 0, count, st);
        Launch<T>::gather(g, bf, count, st);
        Launch<T>::cl(flen, false, g, bf, kApply, 0, count, st);
    }

    void build_precond() {
        CK(cudaSetDevice(device));
        const size_t n = static_cast<size_t>(gp.n);
        std::vector<double> diag(n, 0.0);
        // probe list (operators.hpp:381-417)
        struct Probe {
            size_t rep;
            int l, scale, oi, oj, block;
        };
        std::vector<Probe> probes;
        if (g.precond == Precond::exact) {
            if (static_cast<long long>(n) > g.dense_cap)
                throw ConfigError("preconditioner: exact mode needs coefficient dimension <= " +
                                  std::to_string(g.dense_cap) + ", got " + std::to_string(n));
            for (size_t k = 0; k < n; ++k) probes.push_back({k, -1, 0, 0, 0, 0});
        } else {
            for (int l = 0; l < gp.L; ++l) {
                const int side = gp.side[l], order = gp.lorder[l];
                for (int scale = 0; scale <= order; ++scale) {
                    const int block = scale == 0 ? 1 : 1 << (scale - 1);
                    for (int orient = scale == 0 ? 0 : 1; orient <= (scale == 0 ? 0 : 3); ++orient) {
                        const int oi = orient >= 2 ? block : 0;
                        const int oj = (orient == 1 || orient == 3) ? block : 0;
                        const size_t rep = gp.coff[l] + static_cast<size_t>(oi + block / 2) * side + (oj + block / 2);
                        probes.push_back({rep, l, scale, oi, oj, block});
                    }
                }
            }
        }
        const int chunk = static_cast<int>(std::min<size_t>(probes.size(), n <= 20000 ? 256 : 64));
        if (pd.count < chunk) pd.alloc(gp, chunk, fr, false);
        std::vector<double> probed(probes.size());
        std::vector<double> one(1, 1.0), got(1);
        for (size_t p0 = 0; p0 < probes.size(); p0 += chunk) {
            const int cnt = static_cast<int>(std::min<size_t>(chunk, probes.size() - p0));
            CK(cudaMemsetAsync(pd.in, 0, sizeof(double) * n * cnt, stream));
            for (int k = 0; k < cnt; ++k)
                CK(cudaMemcpyAsync(pd.in + k * n + plan.perm[probes[p0 + k].rep], one.data(), sizeof(double),
                                   cudaMemcpyHostToDevice, stream));
            apply_M_dev<double>(pd, cnt, stream, gp64);
            for (int k = 0; k < cnt; ++k)
                CK(cudaMemcpyAsync(&probed[p0 + k], pd.out + k * n + plan.perm[probes[p0 + k].rep], sizeof(double),
                                   cudaMemcpyDeviceToHost, stream));
            CK(cudaStreamSynchronize(stream));
        }
        for (size_t k = 0; k < probes.size(); ++k) {
            const Probe& pr = probes[k];
            if (pr.l < 0) {
                diag[pr.rep] = probed[k];
                continue;
            }
            const double alpha_d = plan.td[plan.ti[gp.o_reg + pr.l] + pr.scale];
            double value;
            if (g.precond == Precond::balanced) {
                const double ex = g.balance_exponent;
                value = std::pow(probed[k], ex) * std::pow(alpha_d, 1.0 - ex);
            } else {
                const double t_hat = probed[k] - alpha_d;
                const double wgt = pr.scale == 0 ? g.coarse_weight : 1.0;
                value = alpha_d + wgt * t_hat;
            }
            const int side = gp.side[pr.l];
            for (int i = pr.oi; i < pr.oi + pr.block; ++i)
                for (int j = pr.oj; j < pr.oj + pr.block; ++j) diag[gp.coff[pr.l] + static_cast<size_t>(i) * side + j] = value;
        }
        for (double v : diag)
            if (!(v > 0.0))
                throw std::runtime_error("preconditioner: non-positive diagonal entry (operator symmetry broken?)");
        precond = diag;
        std::vector<double> inv(n), dperm(n);
        for (size_t k = 0; k < n; ++k) {  // device copies in the rank-blocked order
            dperm[static_cast<size_t>(plan.perm[k])] = diag[k];
            inv[static_cast<size_t>(plan.perm[k])] = 1.0 / diag[k];
        }
        diag.swap(dperm);
        // uploads ordered on the frame stream (non-blocking: it does not wait for the
        // legacy stream), complete before the first frame can read them
        const cudaStream_t fs = s();
        CK(cudaStreamSynchronize(fs));
        if (precision == 64) {
            CK(cudaMemcpyAsync(jac, diag.data(), n * sizeof(double), cudaMemcpyHostToDevice, fs));
            CK(cudaMemcpyAsync(jinv, inv.data(), n * sizeof(double), cudaMemcpyHostToDevice, fs));
            CK(cudaStreamSynchronize(fs));
        } else {
            std::vector<float> f(diag.begin(), diag.end()), fi(inv.begin(), inv.end());
            CK(cudaMemcpyAsync(jac, f.data(), n * sizeof(float), cudaMemcpyHostToDevice, fs));
            CK(cudaMemcpyAsync(jinv, fi.data(), n * sizeof(float), cudaMemcpyHostToDevice, fs));
            CK(cudaStreamSynchronize(fs));
        }
        has_precond = true;
    }
};

template <>
Work<double>& EngineImpl::state<double>() { return sd; }
template <>
Work<float>& EngineImpl::state<float>() { return sf; }
template <>
Work<double>& EngineImpl::ops<double>() { return od; }
template <>
Work<float>& EngineImpl::ops<float>() { return of; }

// ---------------------------------------------------------------------------

namespace {
template <typename T>
void h2d_conv(T* dst, const double* src, size_t n, cudaStream_t st) {
    if constexpr (std::is_same_v<T, double>) {
        CK(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
    } else {
        std::vector<float> tmp(src, src + n);
        CK(cudaMemcpyAsync(dst, tmp.data(), n * sizeof(float), cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
    }
}
template <typename T>
void d2h_conv(double* dst, const T* src, size_t n, cudaStream_t st) {
    if constexpr (std::is_same_v<T, double>) {
        CK(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    } else {
        std::vector<float> tmp(n);
        CK(cudaMemcpyAsync(tmp.data(), src, n * sizeof(float), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        std::copy(tmp.begin(), tmp.end(), dst);
    }
}
// Coefficient-domain vectors: the API's Mallat order <-> the device's
// rank-blocked order (clayout.hpp), `count` instances of n.
template <typename T>
void h2d_coeff(T* dst, const double* src, const std::vector<int>& perm, size_t count, cudaStream_t st) {
    const size_t n = perm.size();
    std::vector<double> tmp(n * count);
    for (size_t b = 0; b < count; ++b)
        for (size_t i = 0; i < n; ++i) tmp[b * n + static_cast<size_t>(perm[i])] = src[b * n + i];
    h2d_conv<T>(dst, tmp.data(), n * count, st);
}
template <typename T>
void d2h_coeff(double* dst, const T* src, const std::vector<int>& perm, size_t count, cudaStream_t st) {
    const size_t n = perm.size();
    std::vector<double> tmp(n * count);
    d2h_conv<T>(tmp.data(), src, n * count, st);
    for (size_t b = 0; b < count; ++b)
        for (size_t i = 0; i < n; ++i) dst[b * n + i] = tmp[b * n + static_cast<size_t>(perm[i])];
}
}  // namespace

Engine::Engine(Geometry g, int precision, int batch, int device) : p_(std::make_unique<EngineImpl>()) {
    if (precision != 64 && precision != 32) throw ArgError("precision must be 64 or 32");
    if (batch < 1) throw ArgError("batch must be >= 1");
    auto& P = *p_;
    P.g = std::move(g);
    P.precision = precision;
    P.batch = batch;
    P.device = device;
    P.flen = 2 * P.g.wavelet_order;
    auto set_filters = [&](GeoParams& gpx) {
        // Daubechies taps of the configured order, hi_k = (-1)^k lo_{len-1-k} (wavelet.hpp:104-106)
        const auto lo = daubechies(P.g.wavelet_order);
        const int len = static_cast<int>(lo.size());
        for (int k = 0; k < len; ++k) {
            const double hi = (k % 2 == 0 ? 1.0 : -1.0) * lo[len - 1 - k];
            gpx.flo[k] = lo[k];
            gpx.fhi[k] = hi;
            gpx.flo_f[k] = static_cast<float>(lo[k]);
            gpx.fhi_f[k] = static_cast<float>(hi);
        }
    };
    P.plan = build_plan(P.g, precision / 8, batch);
    P.plan.gp.piston_exact = precision == 32 ? 1 : 0;
    set_filters(P.plan.gp);
    Plan plan64;
    if (precision == 32) {  // the preconditioner probes run in fp64 with their own tables
        plan64 = build_plan(P.g, 8, batch);
        plan64.gp.piston_exact = 0;
        set_filters(plan64.gp);
    }
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw ArgError("device ordinal out of range");
    CK(cudaSetDevice(device));
    P.gp = P.upload_plan(P.plan);
    P.gp64 = precision == 64 ? P.gp : P.upload_plan(plan64);
    P.gpf = P.gp;
    CK(cudaStreamCreateWithFlags(&P.stream, cudaStreamNonBlocking));
    P.own_stream = true;
    if (precision == 64) {
        Launch<double>::set_attrs(P.gp, P.flen);
        P.sd.alloc(P.gp, batch, P.fr, true);
        P.jac = dalloc<double>(P.gp.n);
        P.jinv = dalloc<double>(P.gp.n);
    } else {
        Launch<float>::set_attrs(P.gp, P.flen);
        P.sf.alloc(P.gp, batch, P.fr, true);
        P.jac = dalloc<float>(P.gp.n);
        P.jinv = dalloc<float>(P.gp.n);
    }
    Launch<double>::set_attrs(P.gp64, P.flen);  // probes always fp64
    P.fr.add(P.jac);
    P.fr.add(P.jinv);
    {
        // opt-in (FEWHA_FUSE=1): measured slower than the split launches
        const char* fz = std::getenv("FEWHA_FUSE");
        if (fz && fz[0] == '1') {
            const int cap = precision == 64 ? Launch<double>::fused_capacity(P.gp, P.flen, batch)
                                            : Launch<float>::fused_capacity(P.gp, P.flen, batch);
            P.fuse_ok = cap >= P.gp.L * batch;
        }
        // whole-layer transforms for batches (> 2 instances) when a layer fits one CTA's
        // shared memory; FEWHA_WHOLE_LAYER=0/1 overrides (tests, A/B)
        {
            int maxopt = 0;
            CK(cudaDeviceGetAttribute(&maxopt, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
            const bool fits = whole_layer_smem(P.gp.maxside, precision / 8) + 1024 <= static_cast<size_t>(maxopt);
            const char* wv = std::getenv("FEWHA_WHOLE_LAYER");
            P.whole_layer = fits && (wv ? wv[0] == '1' : batch > 2);
            const char* fw = std::getenv("FEWHA_FUSE_WHOLE");
            if (P.whole_layer && fw && fw[0] == '1') {
                int sms = 0;
                CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
                const int per_sm = precision == 64 ? Launch<double>::whole_fused_per_sm(P.gp, P.flen)
                                                   : Launch<float>::whole_fused_per_sm(P.gp, P.flen);
                // the ticketed barrier needs more than L CTAs resident at once; opt-in
                // (FEWHA_FUSE_WHOLE=1): batch 64 fp64 -0.8 %, fp32 +4 % per step
                P.whole_fuse = fw && fw[0] == '1' && per_sm * sms > P.gp.L;
            }
        }
        P.fbar = dalloc<unsigned long long>(static_cast<size_t>(batch));
        P.fr.add(P.fbar);
        CK(cudaMemset(P.fbar, 0, sizeof(unsigned long long) * static_cast<size_t>(batch)));
        P.wbar = dalloc<unsigned long long>(static_cast<size_t>(batch) + 1);
        P.fr.add(P.wbar);
        CK(cudaMemset(P.wbar, 0, sizeof(unsigned long long) * (static_cast<size_t>(batch) + 1)));
    }
    // the table uploads and zero fills above ran on the legacy stream: let them land
    // before anything is issued on the (non-blocking) frame stream
    CK(cudaDeviceSynchronize());
    reset();
}

Engine::~Engine() {
    if (!p_) return;
    cudaSetDevice(p_->device);
    p_->invalidate_graph();
    for (auto ev : p_->tev) cudaEventDestroy(ev);
    if (p_->host_out) cudaFreeHost(p_->host_out);
    if (p_->comm) NcclApi::get().CommDestroy(p_->comm);
    if (p_->own_stream && p_->stream) cudaStreamDestroy(p_->stream);
}

const Geometry& Engine::geometry() const { return p_->g; }
int Engine::precision() const { return p_->precision; }
int Engine::batch() const { return p_->batch; }
bool Engine::has_preconditioner() const { return p_->has_precond; }
std::vector<double> Engine::preconditioner() const { return p_->precond; }

void Engine::override_loop(int loop_mode, double gain) {
    auto& P = *p_;
    if (loop_mode == 0 || loop_mode == 1) {
        P.g.closed_loop = loop_mode == 0;
        P.gp.closed = loop_mode == 0 ? 1 : 0;
    }
    if (gain >= 0.0) {
        if (gain > 1.0) throw ConfigError("invalid geometry: gain out of [0,1]");
        P.g.gain = gain;
        P.gp.gain = gain;
    }
    P.gpf.closed = P.gp.closed;
    P.gpf.gain = P.gp.gain;
    P.invalidate_graph();
}

// ---------------------------------------------------------------------------
// Per-WFS sharding
// ---------------------------------------------------------------------------
std::pair<int, int> shard_range(const Geometry& g, int rank, int world) {
    const int W = static_cast<int>(g.wfs.size());
    if (world < 1 || world > W) throw ArgError("shard: world must be in [1, number of WFS]");
    if (rank < 0 || rank >= world) throw ArgError("shard: rank out of range");
    // contiguous WFS ranges minimising the largest per-rank cost (linear
    // partition, exact DP); cost = (n_s+1)^2 wavefront nodes of the WFS
    std::vector<double> pre(static_cast<size_t>(W) + 1, 0.0);
    for (int w = 0; w < W; ++w) {
        const double np = g.wfs[w].n_subap + 1.0;
        pre[static_cast<size_t>(w) + 1] = pre[static_cast<size_t>(w)] + np * np;
    }
    const double inf = 1e300;
    // best[k][j]: min over partitions of WFS [0, j) into k ranges of the max range cost
    std::vector<std::vector<double>> best(static_cast<size_t>(world) + 1, std::vector<double>(static_cast<size_t>(W) + 1, inf));
    std::vector<std::vector<int>> cut(best.size(), std::vector<int>(static_cast<size_t>(W) + 1, 0));
    best[0][0] = 0.0;
    for (int k = 1; k <= world; ++k)
        for (int j = k; j <= W; ++j)
            for (int i = k - 1; i < j; ++i) {  // last range [i, j); ties keep the earliest cut
                const double v = std::max(best[k - 1][i], pre[j] - pre[i]);
                if (v < best[k][j]) {
                    best[k][j] = v;
                    cut[k][j] = i;
                }
            }
    std::vector<int> bounds(static_cast<size_t>(world) + 1);
    bounds[static_cast<size_t>(world)] = W;
    for (int k = world, j = W; k > 0; --k) {
        j = cut[k][j];
        bounds[static_cast<size_t>(k) - 1] = j;
    }
    return {bounds[static_cast<size_t>(rank)], bounds[static_cast<size_t>(rank) + 1]};
}

void Engine::shard(int rank, int world, const void* nccl_id) {
    auto& P = *p_;
    CK(cudaSetDevice(P.device));
    const auto [wa, wb] = shard_range(P.g, rank, world);
    if (P.comm) {
        NcclApi::get().CommDestroy(P.comm);
        P.comm = nullptr;
    }
    P.shard_rank = rank;
    P.shard_world = world;
    P.sharded = world > 1 || nccl_id != nullptr;
    Plan sp = build_plan(P.g, P.precision / 8, P.batch, wa, wb);
    sp.gp.piston_exact = P.gp.piston_exact;
    std::copy(std::begin(P.gp.flo), std::end(P.gp.flo), sp.gp.flo);
    std::copy(std::begin(P.gp.fhi), std::end(P.gp.fhi), sp.gp.fhi);
    std::copy(std::begin(P.gp.flo_f), std::end(P.gp.flo_f), sp.gp.flo_f);
    std::copy(std::begin(P.gp.fhi_f), std::end(P.gp.fhi_f), sp.gp.fhi_f);
    sp.gp.closed = P.gp.closed;
    sp.gp.gain = P.gp.gain;
    P.gpf = world > 1 ? P.upload_plan(sp) : P.gp;
    if (P.sharded && P.ypart.empty()) {
        const size_t es = P.precision / 8, bytes = es * static_cast<size_t>(P.gp.n) * P.batch;
        for (int e = 0; e <= P.gp.iters; ++e) {
            void* p = nullptr;
            CK(cudaMalloc(&p, bytes));
            CK(cudaMemset(p, 0, bytes));
            P.fr.add(p);
            P.ypart.push_back(p);
        }
    }
    if (nccl_id) {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        const auto& api = NcclApi::get();
        api.check(api.CommInitRank(&P.comm, world, id, rank), "ncclCommInitRank");
    }
    CK(cudaDeviceSynchronize());  // shard table uploads (legacy stream) land before the frame stream reads them
    P.invalidate_graph();
}

std::pair<int, int> Engine::shard_wfs() const { return {p_->gpf.wa, p_->gpf.wb}; }

void* Engine::shard_partial(int seg) const {
    const auto& P = *p_;
    if (!P.sharded || seg < 0 || seg >= static_cast<int>(P.ypart.size())) return nullptr;
    return P.ypart[static_cast<size_t>(seg)];
}

// In-process shard group (one process driving the members, on one device or on
// several with peer access): segments in lockstep on every member's stream; the
// exchange after segment k is fused into every member's next forward kernel, which
// stages its y band as the rank-order sum of all members' partial buffers of segment
// k (cluster.cuh fwd_phase; NVLink peer loads across devices) after waiting for every
// member's segment k (cross-stream events).  A member's partial buffer of segment k is
// rewritten only in the next frame, after every member's last segment, which waited for
// all segments >= k+1, so no buffer is read and rewritten concurrently.
void group_step_device(const std::vector<Engine*>& members) {
    const int world = static_cast<int>(members.size());
    if (world < 1 || world > kMaxW) throw ArgError("shard group: 1..16 members");
    std::vector<EngineImpl*> m(static_cast<size_t>(world));
    for (int r = 0; r < world; ++r) {
        m[static_cast<size_t>(r)] = members[static_cast<size_t>(r)]->p_.get();
        const auto& P = *m[static_cast<size_t>(r)];
        if (!P.sharded || P.comm || P.shard_rank != r || P.shard_world != world)
            throw ArgError("shard group: member " + std::to_string(r) + " is not rank " + std::to_string(r) + " of " +
                           std::to_string(world) + " without NCCL");
        if (P.precision != m[0]->precision || P.batch != m[0]->batch || P.gp.n != m[0]->gp.n)
            throw ArgError("shard group: members differ in precision, batch or geometry");
    }
    for (auto* P : m) {
        CK(cudaSetDevice(P->device));
        if (!P->has_precond) P->build_precond();
        for (auto* Q : m)
            if (Q->device != P->device) {
                const cudaError_t pe = cudaDeviceEnablePeerAccess(Q->device, 0);
                if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) CK(pe);
                if (pe == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError();
            }
    }
    // two event sets (segment parity): member r's segment s waits for every member's
    // segment s-1, whose gathers wrote the partial sums its forward kernel reads
    std::vector<cudaEvent_t> ev(2 * static_cast<size_t>(world));
    for (int r = 0; r < world; ++r) {
        CK(cudaSetDevice(m[static_cast<size_t>(r)]->device));
        for (int e = 0; e < 2; ++e)
            CK(cudaEventCreateWithFlags(&ev[static_cast<size_t>(e * world + r)], cudaEventDisableTiming));
    }
    auto run = [&](auto tag) {
        using T = decltype(tag);
        const int nseg = m[0]->n_segments();
        for (int seg = 0; seg < nseg; ++seg) {
            const int cur = seg & 1, prv = cur ^ 1;
            for (int r = 0; r < world; ++r) {
                auto* P = m[static_cast<size_t>(r)];
                CK(cudaSetDevice(P->device));
                P->peer_sum.clear();
                if (seg >= 1) {  // y of this segment's forward = sum of segment seg-1's partials
                    for (int q = 0; q < world; ++q) {
                        if (q != r) CK(cudaStreamWaitEvent(P->s(), ev[static_cast<size_t>(prv * world + q)], 0));
                        P->peer_sum.push_back(m[static_cast<size_t>(q)]->ypart[static_cast<size_t>(seg - 1)]);
                    }
                }
                P->launch_segment<T>(seg, P->s(), [](int) {});
                P->peer_sum.clear();
                CK(cudaEventRecord(ev[static_cast<size_t>(cur * world + r)], P->s()));
            }
        }
    };
    if (m[0]->precision == 64) run(double{});
    else run(float{});
    for (int r = 0; r < world; ++r) {
        CK(cudaSetDevice(m[static_cast<size_t>(r)]->device));
        for (int e = 0; e < 2; ++e) CK(cudaEventDestroy(ev[static_cast<size_t>(e * world + r)]));
    }
}

void Engine::build_preconditioner() { p_->build_precond(); }

// Page-locked host memory the device can store to (FEWHA_ZERO_COPY=0: never).
static bool page_locked(const void* p) {
    static const bool on = [] {
        const char* v = std::getenv("FEWHA_ZERO_COPY");
        return !(v && v[0] == '0');
    }();
    if (!on) return false;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost && at.devicePointer == p;
}

void Engine::step(const double* slopes, double* coeffs, double* dm, double* rho, int* n_rho) {
    auto& P = *p_;
    CK(cudaSetDevice(P.device));
    if (!P.has_precond) P.build_precond();
    const size_t B = P.batch, S = P.gp.S, n = P.gp.n, A = P.gp.A, it = P.gp.iters;
    const cudaStream_t st = P.s();
    double* meas = P.precision == 64 ? P.sd.meas : P.sf.meas;
    const size_t fob = P.precision == 64 ? P.sd.frame_out_bytes : P.sf.frame_out_bytes;
    if (!P.host_out) {  // page-locked mirror of the rho/status/nlog block, written by the frame itself
        CK(cudaMallocHost(&P.host_out, fob));
        P.invalidate_graph();
    }
    if (P.precision == 64) P.ensure_graph<double>();
    else P.ensure_graph<float>();
    double* dm_direct = (dm && P.fit_node && page_locked(dm)) ? dm : nullptr;
    if (P.precision == 64) P.set_fit_a_host<double>(dm_direct);
    else P.set_fit_a_host<float>(dm_direct);
    CK(cudaMemcpyAsync(meas, slopes, B * S * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaGraphLaunch(P.graph, st));
    ++P.step_counter;
    P.telem_pending = P.telemetry_on;
    if (P.precision == 64) {
        if (dm && !dm_direct) CK(cudaMemcpyAsync(dm, P.sd.bf.a_out, B * A * sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (coeffs) d2h_coeff<double>(coeffs, P.sd.bf.c, P.plan.perm, B, st);
    } else {
        CK(cudaStreamSynchronize(st));
        if (coeffs) d2h_coeff<float>(coeffs, P.sf.bf.c, P.plan.perm, B, st);
        if (dm && !dm_direct) d2h_conv<float>(dm, P.sf.bf.a_out, B * A, st);
    }
    const auto* hrho = static_cast<const double*>(P.host_out);
    const int* status = reinterpret_cast<const int*>(hrho + B * it);
    const int* nl = status + B;
    if (rho) std::copy(hrho, hrho + B * it, rho);
    if (n_rho) std::copy(nl, nl + B, n_rho);
    for (size_t b = 0; b < B; ++b)
        if (status[b]) throw std::runtime_error("pcg_solve: non-finite scalar (indefinite operator?)");
}

void Engine::reset() {
    auto& P = *p_;
    CK(cudaSetDevice(P.device));
    const size_t B = P.batch, n = P.gp.n, A = P.gp.A;
    // Frames run on a non-blocking stream (the engine's or the caller's), which does
    // not order against the legacy default stream: finish any frame in flight, zero
    // the state on the frame stream and return only when it has landed.
    const cudaStream_t st = P.s();
    CK(cudaStreamSynchronize(st));
    auto zero_state = [&](auto& w, size_t es) {
        for (void* ptr : {(void*)w.bf.c, (void*)w.bf.b, (void*)w.bf.r, (void*)w.bf.p, (void*)w.bf.q, (void*)w.bf.mz})
            CK(cudaMemsetAsync(ptr, 0, B * n * es, st));
        for (void* ptr : {(void*)w.bf.a_prev2, (void*)w.bf.a_prev, (void*)w.bf.a_out})
            CK(cudaMemsetAsync(ptr, 0, B * A * es, st));
        std::vector<Carry> c(B * (P.gp.iters + 1));
        for (auto& x : c) x = Carry{0.0, 0.0, 0.0, 1, 0, 0, 0};  // PcgScalars{} : fresh
        CK(cudaMemcpyAsync(w.bf.carry, c.data(), c.size() * sizeof(Carry), cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
    };
    if (P.precision == 64) zero_state(P.sd, sizeof(double));
    else zero_state(P.sf, sizeof(float));
}

void Engine::get_state(int inst, double* c, double* b, double* r, double* p, double* q, double* sc, double* a_prev2,
                       double* a_prev) {
    auto& P = *p_;
    if (inst < 0 || inst >= P.batch) throw ArgError("instance out of range");
    CK(cudaSetDevice(P.device));
    const size_t n = P.gp.n, A = P.gp.A;
    auto get = [&](auto& w) {
        using T = std::remove_pointer_t<decltype(w.bf.c)>;
        const cudaStream_t st = P.s();
        CK(cudaStreamSynchronize(st));
        // any output may be null (skipped): e.g. the scalars alone after every step
        if (c) d2h_coeff<T>(c, w.bf.c + inst * n, P.plan.perm, 1, st);
        if (b) d2h_coeff<T>(b, w.bf.b + inst * n, P.plan.perm, 1, st);
        if (r) d2h_coeff<T>(r, w.bf.r + inst * n, P.plan.perm, 1, st);
        if (p) d2h_coeff<T>(p, w.bf.p + inst * n, P.plan.perm, 1, st);
        if (q) d2h_coeff<T>(q, w.bf.q + inst * n, P.plan.perm, 1, st);
        if (a_prev2) d2h_conv<T>(a_prev2, w.bf.a_prev2 + inst * A, A, st);
        if (a_prev) d2h_conv<T>(a_prev, w.bf.a_prev + inst * A, A, st);
        Carry cr;
        CK(cudaMemcpyAsync(&cr, w.bf.carry + inst * (P.gp.iters + 1), sizeof(Carry), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        sc[0] = cr.rho_old;
        sc[1] = cr.alpha;
        sc[2] = cr.fresh ? 1.0 : 0.0;
    };
    if (P.precision == 64) get(P.sd);
    else get(P.sf);
}

void Engine::set_state(int inst, const double* c, const double* b, const double* r, const double* p, const double* q,
                       const double* sc, const double* a_prev2, const double* a_prev) {
    auto& P = *p_;
    if (inst < 0 || inst >= P.batch) throw ArgError("instance out of range");
    CK(cudaSetDevice(P.device));
    const size_t n = P.gp.n, A = P.gp.A;
    auto set = [&](auto& w) {
        using T = std::remove_pointer_t<decltype(w.bf.c)>;
        const cudaStream_t st = P.s();
        CK(cudaStreamSynchronize(st));
        h2d_coeff<T>(w.bf.c + inst * n, c, P.plan.perm, 1, st);
        h2d_coeff<T>(w.bf.b + inst * n, b, P.plan.perm, 1, st);
        h2d_coeff<T>(w.bf.r + inst * n, r, P.plan.perm, 1, st);
        h2d_coeff<T>(w.bf.p + inst * n, p, P.plan.perm, 1, st);
        h2d_coeff<T>(w.bf.q + inst * n, q, P.plan.perm, 1, st);
        h2d_conv<T>(w.bf.a_prev2 + inst * A, a_prev2, A, st);
        h2d_conv<T>(w.bf.a_prev + inst * A, a_prev, A, st);
        Carry cr{sc[0], sc[1], 0.0, sc[2] != 0.0 ? 1 : 0, 0, 0, 0};
        CK(cudaMemcpyAsync(w.bf.carry + inst * (P.gp.iters + 1), &cr, sizeof(Carry), cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
    };
    if (P.precision == 64) set(P.sd);
    else set(P.sf);
}

void Engine::set_stream(void* stream) {
    p_->user_stream = static_cast<cudaStream_t>(stream);
}

void Engine::step_device(const void* d_slopes) {
    auto& P = *p_;
    CK(cudaSetDevice(P.device));
    if (!P.has_precond) P.build_precond();
    const cudaStream_t st = P.s();
    double* meas = P.precision == 64 ? P.sd.meas : P.sf.meas;
    if (d_slopes && d_slopes != meas)
        CK(cudaMemcpyAsync(meas, d_slopes, sizeof(double) * P.gp.S * P.batch, cudaMemcpyDeviceToDevice, st));
    // device-resident frames never store into a caller's host buffer from an earlier step()
    if (P.precision == 64) {
        P.ensure_graph<double>();
        P.set_fit_a_host<double>(nullptr);
    } else {
        P.ensure_graph<float>();
        P.set_fit_a_host<float>(nullptr);
    }
    CK(cudaGraphLaunch(P.graph, st));
    ++P.step_counter;
    P.telem_pending = P.telemetry_on;
}

void Engine::enable_telemetry(bool on) {
    auto& P = *p_;
    if (P.telemetry_on == on) return;
    P.telemetry_on = on;
    P.telem_pending = false;
    P.invalidate_graph();
}

// StepTelemetry of the last graph frame (reconstructor.hpp:94-102) from the event
// nodes: stage1 = W^-1 kernels, stage2 = per-WFS kernels (incl. RHS), stage3 =
// P^T / W / alpha D kernels (incl. RHS), pcg = the fused PCG iterations (first
// W^-1 through the last W; the last update is fused into the fitting W^-1), fit =
// fitting W^-1 + fit + control.  Times are in microseconds.
StepTelemetry Engine::last_telemetry() {
    auto& P = *p_;
    StepTelemetry t;
    t.step = P.step_counter;
    if (!P.telem_pending) return t;
    CK(cudaSetDevice(P.device));
    CK(cudaEventSynchronize(P.tev[P.tkind.size()]));
    bool in_pcg = false;
    for (size_t i = 0; i < P.tkind.size(); ++i) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, P.tev[i], P.tev[i + 1]));
        const double us = 1000.0 * ms;
        const int k = P.tkind[i];
        if (k == kKindInvPcg0) in_pcg = true;
        if (k == kKindInvFit) in_pcg = false;
        if (k == kKindInvPcg0 || k == kKindInvPcg || k == kKindInvFit) t.stage1_us += us;
        else if (k == kKindWfsRhs || k == kKindWfs) t.stage2_us += us;
        else if (k == kKindGather || k == kKindFwdRhs || k == kKindFwdPcg) t.stage3_us += us;
        if (in_pcg) t.pcg_us += us;
        if (k == kKindInvFit || k == kKindFit) t.fit_us += us;
        t.total_us += us;
    }
    t.valid = true;
    return t;
}

// Per-launch device times of the last graph frame from its telemetry event nodes
// (kinds as profile_step); 0 when telemetry is off or no frame ran since.
int Engine::last_launch_times(float* ms, int* kinds, int max) {
    auto& P = *p_;
    if (!P.telem_pending) return 0;
    CK(cudaSetDevice(P.device));
    CK(cudaEventSynchronize(P.tev[P.tkind.size()]));
    int n = 0;
    for (size_t i = 0; i < P.tkind.size() && n < max; ++i, ++n) {
        CK(cudaEventElapsedTime(&ms[n], P.tev[i], P.tev[i + 1]));
        kinds[n] = P.tkind[i];
    }
    return n;
}

void Engine::load_slopes(const void* src, bool on_device) {
    auto& P = *p_;
    CK(cudaSetDevice(P.device));
    double* meas = P.precision == 64 ? P.sd.meas : P.sf.meas;
    CK(cudaMemcpyAsync(meas, src, sizeof(double) * P.gp.S * P.batch,
                       on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, P.s()));
}

// Outputs of the last device frame (any may be null): st.c, a^(1), the rho log
// and its length; raises on a non-finite PCG scalar like step().
void Engine::read_outputs(double* coeffs, double* dm, double* rho, int* n_rho) {
    auto& P = *p_;
    CK(cudaSetDevice(P.device));
    const cudaStream_t st = P.s();
    const size_t B = P.batch, A = P.gp.A, it = P.gp.iters;
    CK(cudaStreamSynchronize(st));
    auto rd = [&](auto& w) {
        using T = std::remove_pointer_t<decltype(w.bf.c)>;
        if (coeffs) d2h_coeff<T>(coeffs, w.bf.c, P.plan.perm, B, st);
        if (dm) d2h_conv<T>(dm, w.bf.a_out, B * A, st);
        std::vector<unsigned char> blk(w.frame_out_bytes);
        CK(cudaMemcpyAsync(blk.data(), w.bf.rho_log, blk.size(), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const auto* hr = reinterpret_cast<const double*>(blk.data());
        const int* status = reinterpret_cast<const int*>(hr + B * it);
        if (rho) std::copy(hr, hr + B * it, rho);
        if (n_rho) std::copy(status + B, status + 2 * B, n_rho);
        for (size_t b = 0; b < B; ++b)
            if (status[b]) throw std::runtime_error("pcg_solve: non-finite scalar (indefinite operator?)");
    };
    if (P.precision == 64) rd(P.sd);
    else rd(P.sf);
}

void Engine::sync_check() {
    auto& P = *p_;
    CK(cudaSetDevice(P.device));
    const cudaStream_t st = P.s();
    std::vector<int> status(P.batch);
    const int* dstat = P.precision == 64 ? P.sd.bf.status : P.sf.bf.status;
    CK(cudaMemcpyAsync(status.data(), dstat, status.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int s : status)
        if (s) throw std::runtime_error("pcg_solve: non-finite scalar (indefinite operator?)");
}

PlanInfo Engine::plan_info() const {
    const auto& P = *p_;
    PlanInfo pi;
    pi.cluster_ctas = P.gp.ccl;
    pi.tail = P.gp.ctail;
    pi.gather_rows = P.gp.grows;
    pi.gather_ctas_per_sm = P.gp.gather_minb;
    pi.inverse_staged = P.precision == 64 ? Launch<double>::inv_staged_for(P.gp, P.batch) : Launch<float>::inv_staged_for(P.gp, P.batch);
    pi.wfs_ctas_per_sm = P.batch <= 2 ? FEWHA_WFS_MINB_LAT : FEWHA_WFS_MINB_BATCH;
    pi.wfs_tiles = P.gp.wt_count;
    pi.launches_per_step = launches_per_step();
    pi.whole_layer = P.use_whole_fused() ? 2 : P.use_whole() ? 1 : 0;
    pi.gather_instances = P.gp.gather_ni;
    pi.gather_direct = P.gp.gather_direct;
    pi.wfs_instances = P.precision == 64 ? Launch<double>::wfs_ni(P.batch) : Launch<float>::wfs_ni(P.batch);
    if (pi.wfs_instances == 2) pi.wfs_ctas_per_sm = kWfsNi2Minb;
    else if (pi.wfs_instances == 4) pi.wfs_ctas_per_sm = P.precision == 64 ? kWfsNi4Minb<double> : kWfsNi4Minb<float>;
    return pi;
}

int Engine::launches_per_step() const {
    const int it = p_->gp.iters;
    return (p_->fused_frame() || p_->use_whole_fused()) ? 4 + 3 * it : 5 + 4 * it;
}

int Engine::profile_step(float* ms, int* kinds, int max) {
    auto& P = *p_;
    CK(cudaSetDevice(P.device));
    if (!P.has_precond) P.build_precond();
    if (P.stamp_buf) {
        CK(cudaMemset(P.stamp_buf, 0, sizeof(unsigned long long) * EngineImpl::kStampSlots * EngineImpl::kStampBlocks * 16));
        P.stamp_slot = 0;
    }
    struct Off {
        int& s;
        ~Off() { s = -1; }
    } off{P.stamp_slot};
    return P.precision == 64 ? P.profile_frame<double>(ms, kinds, max) : P.profile_frame<float>(ms, kinds, max);
}

// Micro-benchmark of the cluster layer transform kernel (variant, threads: unused).  Returns mean ms per launch over `reps`.
float Engine::bench_dwt(int variant, int inverse, int reps, int threads) {
    auto& P = *p_;
    CK(cudaSetDevice(P.device));
    float ms = 0.f;
    auto run = [&](auto& w) {
        using T = std::remove_pointer_t<decltype(w.in)>;
        if (w.count < 1) w.alloc(P.gp, 1, P.fr, false);
        Bufs<T> bf = w.bf;
        auto once = [&] {
            Launch<T>::cl(P.flen, inverse != 0, P.gp, bf, kPlain, 0, 1, P.stream, 0);
        };
        for (int i = 0; i < 3; ++i) once();
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        CK(cudaEventRecord(a, P.stream));
        for (int i = 0; i < reps; ++i) once();
        CK(cudaEventRecord(b, P.stream));
        CK(cudaEventSynchronize(b));
        CK(cudaEventElapsedTime(&ms, a, b));
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    };
    if (P.precision == 64) run(P.od);
    else run(P.of);
    return ms / reps;
}

void Engine::enable_stamps(bool on) {
    auto& P = *p_;
    CK(cudaSetDevice(P.device));
    if (on && !P.stamp_buf) {
        void* p = nullptr;
        CK(cudaMalloc(&p, sizeof(unsigned long long) * EngineImpl::kStampSlots * EngineImpl::kStampBlocks * 16));
        P.stamp_buf = static_cast<unsigned long long*>(p);
        P.fr.add(p);
    }
}

int Engine::read_stamps(unsigned long long* out, size_t n) {
    auto& P = *p_;
    if (!P.stamp_buf) return 0;
    const size_t total = static_cast<size_t>(EngineImpl::kStampSlots) * EngineImpl::kStampBlocks * 16;
    CK(cudaMemcpy(out, P.stamp_buf, sizeof(unsigned long long) * std::min(n, total), cudaMemcpyDeviceToHost));
    return static_cast<int>(std::min(n, total));
}

void Engine::device_buffers(void** slopes, void** coeffs, void** dm, double** rho, int** status, int** n_rho) {
    auto& P = *p_;
    auto fill = [&](auto& w) {
        *slopes = w.meas;
        *coeffs = w.bf.c;
        *dm = w.bf.a_out;
        *rho = w.bf.rho_log;
        *status = w.bf.status;
        *n_rho = w.bf.nlog;
    };
    if (P.precision == 64) fill(P.sd);
    else fill(P.sf);
}

// ---- operator entry points --------------------------------------------------
namespace {
template <typename T, typename F>
void with_ops(EngineImpl& P, int count, F&& f) {
    if (count < 1) throw ArgError("count must be >= 1");
    CK(cudaSetDevice(P.device));
    Work<T>& w = P.ops<T>();
    if (w.count < count) w.alloc(P.gp, std::max(count, w.count), P.fr, false);
    f(w);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(P.stream));
}
}  // namespace

#define FEWHA_DISPATCH(body)                        \
    if (p_->precision == 64) {                      \
        using T = double;                           \
        body                                        \
    } else {                                        \
        using T = float;                            \
        body                                        \
    }

void Engine::apply_M(const double* in, double* out, int count) {
    auto& P = *p_;
    FEWHA_DISPATCH({
        with_ops<T>(P, count, [&](Work<T>& w) {
            h2d_coeff<T>(w.in, in, P.plan.perm, count, P.stream);
            P.apply_M_dev<T>(w, count, P.stream, P.gp);
            d2h_coeff<T>(out, w.out, P.plan.perm, count, P.stream);
        });
    })
}

void Engine::build_rhs(const double* meas, double* out, int count) {
    auto& P = *p_;
    FEWHA_DISPATCH({
        with_ops<T>(P, count, [&](Work<T>& w) {
            CK(cudaMemcpyAsync(w.meas, meas, sizeof(double) * P.gp.S * count, cudaMemcpyHostToDevice, P.stream));
            Bufs<T> bf = w.bf;
            Launch<T>::wfs(true, P.gp, bf, 0, count, P.stream);
            Launch<T>::gather(P.gp, bf, count, P.stream);
            Launch<T>::cl(P.flen, false, P.gp, bf, kPlain, 0, count, P.stream);
            d2h_coeff<T>(out, w.out, P.plan.perm, count, P.stream);
        });
    })
}

void Engine::add_dm_slopes(const double* a, double* meas, int count) {
    auto& P = *p_;
    FEWHA_DISPATCH({
        with_ops<T>(P, count, [&](Work<T>& w) {
            h2d_conv<T>(w.a, a, static_cast<size_t>(P.gp.A) * count, P.stream);
            CK(cudaMemcpyAsync(w.meas, meas, sizeof(double) * P.gp.S * count, cudaMemcpyHostToDevice, P.stream));
            const int sub = P.gp.S / 2;
            k_slopes<T><<<dim3((sub + 255) / 256, count), 256, 0, P.stream>>>(P.gp, nullptr, nullptr, w.a, T(1),
                                                                               w.meas, w.meas2, count);
            CK(cudaMemcpyAsync(meas, w.meas2, sizeof(double) * P.gp.S * count, cudaMemcpyDeviceToHost, P.stream));
        });
    })
}

void Engine::forward_slopes(const double* layers, const double* a, double* meas, int count) {
    auto& P = *p_;
    FEWHA_DISPATCH({
        with_ops<T>(P, count, [&](Work<T>& w) {
            h2d_conv<T>(w.in, layers, static_cast<size_t>(P.gp.n) * count, P.stream);
            if (a) h2d_conv<T>(w.a, a, static_cast<size_t>(P.gp.A) * count, P.stream);
            const int sub = P.gp.S / 2;
            k_slopes<T><<<dim3((sub + 255) / 256, count), 256, 0, P.stream>>>(P.gp, nullptr, w.in, a ? w.a : nullptr,
                                                                               T(-1), nullptr, w.meas2, count);
            CK(cudaMemcpyAsync(meas, w.meas2, sizeof(double) * P.gp.S * count, cudaMemcpyDeviceToHost, P.stream));
        });
    })
}

void Engine::fit(const double* c, double* a, int count) {
    auto& P = *p_;
    FEWHA_DISPATCH({
        with_ops<T>(P, count, [&](Work<T>& w) {
            h2d_coeff<T>(w.in, c, P.plan.perm, count, P.stream);
            Bufs<T> bf = w.bf;
            Launch<T>::cl(P.flen, true, P.gp, bf, kPlain, 0, count, P.stream);
            Launch<T>::fit(P.gp, bf, 0, count, P.stream);
            d2h_conv<T>(a, w.a, static_cast<size_t>(P.gp.A) * count, P.stream);
        });
    })
}

void Engine::wavelet(int inverse, double* data, int count) {
    auto& P = *p_;
    FEWHA_DISPATCH({
        with_ops<T>(P, count, [&](Work<T>& w) {
            const size_t n = static_cast<size_t>(P.gp.n) * count;
            Bufs<T> bf = w.bf;
            if (inverse) {
                h2d_coeff<T>(w.in, data, P.plan.perm, count, P.stream);
                Launch<T>::cl(P.flen, true, P.gp, bf, kPlain, 0, count, P.stream);
                d2h_conv<T>(data, bf.phi, n, P.stream);
            } else {
                h2d_conv<T>(bf.y, data, n, P.stream);
                Launch<T>::cl(P.flen, false, P.gp, bf, kPlain, 0, count, P.stream, /*fit_term=*/0);
                d2h_coeff<T>(data, w.out, P.plan.perm, count, P.stream);
            }
        });
    })
}

// The frame's fused per-WFS kernel (k_wfs, kernels.cuh wfs_tile) as an operator:
//   rhs = 0: psi = Gamma^T C^-1 Gamma P phi          (apply_M stage 2, reconstructor.hpp:182-192)
//   rhs = 1: psi = Gamma^T C^-1 (s + Gamma P_dm a)   (add_dm_slopes :259-280 + build_rhs :221-231;
//            a == null: psi = Gamma^T C^-1 s)
void Engine::wfs_operator(int rhs, const double* in, const double* meas, double* psi, int count) {
    auto& P = *p_;
    FEWHA_DISPATCH({
        with_ops<T>(P, count, [&](Work<T>& w) {
            Bufs<T> bf = w.bf;
            int with_dm = 0;
            if (rhs) {
                if (in) {
                    h2d_conv<T>(w.a, in, static_cast<size_t>(P.gp.A) * count, P.stream);
                    with_dm = 1;
                }
                CK(cudaMemcpyAsync(w.meas, meas, sizeof(double) * P.gp.S * count, cudaMemcpyHostToDevice, P.stream));
            } else {
                h2d_conv<T>(bf.phi, in, static_cast<size_t>(P.gp.n) * count, P.stream);
            }
            Launch<T>::wfs(rhs != 0, P.gp, bf, with_dm, count, P.stream);
            d2h_conv<T>(psi, bf.psi, static_cast<size_t>(P.gp.Nw) * count, P.stream);
        });
    })
}

void Engine::propagate(const double* layers, double* wf, int count) {
    auto& P = *p_;
    FEWHA_DISPATCH({
        with_ops<T>(P, count, [&](Work<T>& w) {
            h2d_conv<T>(w.in, layers, static_cast<size_t>(P.gp.n) * count, P.stream);
            k_propagate<T><<<dim3((P.gp.Nw + 255) / 256, count), 256, 0, P.stream>>>(P.gp, w.in, w.bf.psi, count);
            d2h_conv<T>(wf, w.bf.psi, static_cast<size_t>(P.gp.Nw) * count, P.stream);
        });
    })
}

void Engine::propagate_transpose(const double* wf, double* layers, int count) {
    auto& P = *p_;
    FEWHA_DISPATCH({
        with_ops<T>(P, count, [&](Work<T>& w) {
            h2d_conv<T>(w.bf.psi, wf, static_cast<size_t>(P.gp.Nw) * count, P.stream);
            Launch<T>::gather(P.gp, w.bf, count, P.stream);
            d2h_conv<T>(layers, w.bf.y, static_cast<size_t>(P.gp.n) * count, P.stream);
        });
    })
}

void Engine::sh(const double* wf, double* meas, int count) {
    auto& P = *p_;
    FEWHA_DISPATCH({
        with_ops<T>(P, count, [&](Work<T>& w) {
            h2d_conv<T>(w.bf.psi, wf, static_cast<size_t>(P.gp.Nw) * count, P.stream);
            const int sub = P.gp.S / 2;
            k_slopes<T><<<dim3((sub + 255) / 256, count), 256, 0, P.stream>>>(P.gp, w.bf.psi, nullptr, nullptr, T(1),
                                                                               nullptr, w.meas2, count);
            CK(cudaMemcpyAsync(meas, w.meas2, sizeof(double) * P.gp.S * count, cudaMemcpyDeviceToHost, P.stream));
        });
    })
}

void Engine::sh_transpose(const double* meas, double* wf, int count) {
    auto& P = *p_;
    FEWHA_DISPATCH({
        with_ops<T>(P, count, [&](Work<T>& w) {
            CK(cudaMemcpyAsync(w.meas, meas, sizeof(double) * P.gp.S * count, cudaMemcpyHostToDevice, P.stream));
            k_sh_transpose<T><<<dim3((P.gp.Nw + 255) / 256, count), 256, 0, P.stream>>>(P.gp, w.meas, w.bf.psi, count);
            d2h_conv<T>(wf, w.bf.psi, static_cast<size_t>(P.gp.Nw) * count, P.stream);
        });
    })
}


// ---------------------------------------------------------------------------
// Closed-loop simulation harness on the device (reference
// simulation.hpp:40-345).  Host code only builds tables and issues launches:
// a run_closed_loop moves no data between host and device per frame.
// ---------------------------------------------------------------------------
namespace {
std::uint64_t splitmix64(std::uint64_t x) {  // simulation.hpp:31-36
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
constexpr double kPi = 3.14159265358979323846;
}  // namespace

struct SimState {
    DevFree fr;
    int n = 0, S = 0, A = 0, L = 0, M = 0, pairs = 0, n_dir = 0, nodes = 0;
    bool paired = false, wind = false;
    sim::AtmParams ap{};
    sim::QualParams qp{};
    sim::LerrParams lp{};
    std::vector<std::pair<double, double>> wind_sp;  // per layer (row, column) node shift per step
    double *truth = nullptr, *layers = nullptr, *cplx = nullptr, *cplx2 = nullptr, *z_atm = nullptr;
    double *noise = nullptr, *dm = nullptr, *zero_dm = nullptr, *var = nullptr, *part = nullptr;
    int *nx = nullptr, *ny = nullptr;
    double* sig = nullptr;
    unsigned long long* seeds = nullptr;  // device seed slots
    int seed_cap = 0;
    double* z = nullptr;                   // noise normals [chunk][2 pairs]
    int z_cap = 0;
    template <typename T>
    T* alloc(size_t k) {
        T* p = dalloc<T>(k);
        fr.add(p);
        return p;
    }
};

namespace {
SimState& sim_state(EngineImpl& P) {
    if (P.sim) return *P.sim;
    CK(cudaSetDevice(P.device));
    auto st = std::make_unique<SimState>();
    SimState& S = *st;
    const Geometry& g = P.g;
    S.n = P.gp.n;
    S.S = P.gp.S;
    S.A = P.gp.A;
    S.L = P.gp.L;
    S.M = P.gp.M;
    S.paired = !g.projection && g.layers.size() == g.dms.size();
    // atmosphere: per layer side, nodal offset, normals offset, period, target variance
    S.ap.L = S.L;
    S.ap.kappa0 = 2.0 * kPi / g.outer_scale;
    for (int l = 0; l < S.L; ++l) {
        const int nl = g.layers[l].side();
        S.ap.lay[l] = {nl, P.gp.coff[l], 2 * P.gp.coff[l], g.layers[l].extent / (nl - 1) * nl,
                       g.layers[l].strength * g.truth_strength};
    }
    S.wind = !g.wind.empty();
    for (int l = 0; S.wind && l < S.L; ++l) {
        const double sp = g.layers[l].extent / (g.layers[l].side() - 1);
        S.wind_sp.push_back({g.wind[l].second / sp, g.wind[l].first / sp});
    }
    S.truth = S.alloc<double>(S.n);
    S.layers = S.alloc<double>(S.n);
    S.cplx = S.alloc<double>(2 * static_cast<size_t>(S.n));
    S.cplx2 = S.alloc<double>(2 * static_cast<size_t>(S.n));
    S.z_atm = S.alloc<double>(2 * static_cast<size_t>(S.n));
    S.noise = S.alloc<double>(S.S);
    S.dm = S.alloc<double>(std::max(S.A, 1));
    S.zero_dm = S.alloc<double>(std::max(S.A, 1));
    // noise scatter table: active subapertures, WFS then row-major (simulation.hpp:196-207)
    std::vector<int> ix, iy;
    std::vector<double> sg;
    for (size_t w = 0; w < g.wfs.size(); ++w) {
        const int ns = g.wfs[w].n_subap;
        const double sigma = std::sqrt(g.wfs[w].noise_variance);
        for (int k = 0; k < ns * ns; ++k)
            if (g.wfs[w].mask[static_cast<size_t>(k)]) {
                ix.push_back(P.gp.moff[w] + k);
                iy.push_back(P.gp.moff[w] + ns * ns + k);
                sg.push_back(sigma);
            }
    }
    S.pairs = static_cast<int>(ix.size());
    S.nx = S.alloc<int>(ix.size());
    S.ny = S.alloc<int>(iy.size());
    S.sig = S.alloc<double>(sg.size());
    CK(cudaMemcpy(S.nx, ix.data(), ix.size() * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(S.ny, iy.data(), iy.size() * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(S.sig, sg.data(), sg.size() * sizeof(double), cudaMemcpyHostToDevice));
    // quality: annular-pupil nodes of the finest WFS grid and per (direction, screen)
    // stencil tables (evaluate_quality, simulation.hpp:228-269)
    int n_sub = 0;
    for (const auto& w : g.wfs) n_sub = std::max(n_sub, w.n_subap);
    const int nq = n_sub + 1;
    const double d = g.diameter / (nq - 1), r_out = g.r_out(), r_in = g.r_in();
    std::vector<int> nodes;
    for (int i = 0; i < nq; ++i)
        for (int j = 0; j < nq; ++j) {
            const double x = -r_out + j * d, y = -r_out + i * d, r2 = x * x + y * y;
            if (r2 <= r_out * r_out * (1.0 + 1e-12) && r2 >= r_in * r_in * (1.0 - 1e-12)) nodes.push_back(i * nq + j);
        }
    std::vector<std::pair<double, double>> dirs;  // EvaluationConfig::directions (geometry.hpp:122-133)
    const int nps = g.eval_n_per_side;
    for (int i = 0; i < nps; ++i)
        for (int j = 0; j < nps; ++j) {
            const double fy = nps == 1 ? 0.0 : -1.0 + 2.0 * i / (nps - 1);
            const double fx = nps == 1 ? 0.0 : -1.0 + 2.0 * j / (nps - 1);
            dirs.push_back({fx * g.eval_half_width, fy * g.eval_half_width});
        }
    S.n_dir = static_cast<int>(dirs.size());
    S.nodes = static_cast<int>(nodes.size());
    const int NS = S.L + S.M;
    std::vector<int> tix(static_cast<size_t>(S.n_dir) * NS * 2 * nq);
    std::vector<double> tw(tix.size());
    for (int dd = 0; dd < S.n_dir; ++dd)
        for (int sc = 0; sc < NS; ++sc) {
            const bool lay = sc < S.L;
            const int side = lay ? g.layers[sc].side() : g.dms[sc - S.L].n_act;
            const double ext = lay ? g.layers[sc].extent : g.dms[sc - S.L].extent;
            const double h = lay ? g.layers[sc].height : g.dms[sc - S.L].height;
            for (int axis = 0; axis < 2; ++axis)
                for (int k = 0; k < nq; ++k) {
                    const double p = -r_out + k * d + (axis ? dirs[dd].second : dirs[dd].first) * h;
                    const Stencil1 st1 = stencil1(side, ext, p);
                    const size_t o = ((static_cast<size_t>(dd) * NS + sc) * 2 + axis) * nq + k;
                    tix[o] = st1.idx;
                    tw[o] = st1.f;
                }
        }
    int* dnode = S.alloc<int>(nodes.size());
    int* dtix = S.alloc<int>(tix.size());
    double* dtw = S.alloc<double>(tw.size());
    CK(cudaMemcpy(dnode, nodes.data(), nodes.size() * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dtix, tix.data(), tix.size() * sizeof(int), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dtw, tw.data(), tw.size() * sizeof(double), cudaMemcpyHostToDevice));
    S.qp.L = S.L;
    S.qp.M = S.M;
    S.qp.n = nq;
    S.qp.n_nodes = S.nodes;
    S.qp.n_dir = S.n_dir;
    for (int l = 0; l < S.L; ++l) {
        S.qp.side[l] = P.gp.side[l];
        S.qp.loff[l] = P.gp.coff[l];
    }
    for (int m = 0; m < S.M; ++m) {
        S.qp.nact[m] = P.gp.nact[m];
        S.qp.aoff[m] = P.gp.aoff[m];
    }
    S.qp.node = dnode;
    S.qp.tidx = dtix;
    S.qp.tw = dtw;
    S.var = S.alloc<double>(std::max(S.n_dir, 1));
    S.part = S.alloc<double>(2 * static_cast<size_t>(std::max(S.L, 1)));
    if (S.paired) {  // layer_rel_err tables: DM l on layer l's nodes with the layer extent
        std::vector<int> li;
        std::vector<double> lw;
        S.lp.L = S.L;
        for (int l = 0; l < S.L; ++l) {
            const int nl = g.layers[l].side(), na = g.dms[l].n_act;
            const double ext = g.layers[l].extent, dl = ext / (nl - 1);
            S.lp.side[l] = nl;
            S.lp.loff[l] = P.gp.coff[l];
            S.lp.nact[l] = na;
            S.lp.aoff[l] = P.gp.aoff[l];
            S.lp.toff[l] = static_cast<int>(li.size());
            for (int k = 0; k < nl; ++k) {
                const Stencil1 st1 = stencil1(na, ext, -ext / 2.0 + k * dl);
                li.push_back(st1.idx);
                lw.push_back(st1.f);
            }
        }
        int* dli = S.alloc<int>(li.size());
        double* dlw = S.alloc<double>(lw.size());
        CK(cudaMemcpy(dli, li.data(), li.size() * sizeof(int), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dlw, lw.data(), lw.size() * sizeof(double), cudaMemcpyHostToDevice));
        S.lp.tidx = dli;
        S.lp.tw = dlw;
    }
    CK(cudaFuncSetAttribute(sim::k_quality_dir, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(std::max<size_t>(S.nodes * sizeof(double), 1))));
    CK(cudaDeviceSynchronize());
    P.sim = std::move(st);
    return *P.sim;
}

// normals of `streams` GaussianStreams (seeds on the host) -> S.z [stream][count]
void sim_normals(EngineImpl& P, SimState& S, const std::vector<unsigned long long>& seeds, int count, double* out,
                 cudaStream_t st) {
    if (static_cast<int>(seeds.size()) > S.seed_cap) {
        S.seed_cap = static_cast<int>(seeds.size());
        S.seeds = S.alloc<unsigned long long>(seeds.size());
    }
    CK(cudaMemcpyAsync(S.seeds, seeds.data(), seeds.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice, st));
    sim::k_gauss<<<static_cast<unsigned>(seeds.size()), 32, 0, st>>>(S.seeds, count, out, count);
    CK(cudaGetLastError());
    (void)P;
}

// generate_atmosphere(g, seed) -> S.truth
void sim_atmosphere(EngineImpl& P, SimState& S, std::uint64_t seed, cudaStream_t st) {
    int maxn = 0;
    for (int l = 0; l < S.L; ++l) maxn = std::max(maxn, S.ap.lay[l].n);
    // one stream per layer, 2 n^2 normals each, laid out at 2 * coff[l]
    for (int l = 0; l < S.L; ++l) {
        const std::vector<unsigned long long> sd{splitmix64(seed ^ (0x51a9e4c7ULL + static_cast<std::uint64_t>(l)))};
        sim_normals(P, S, sd, 2 * S.ap.lay[l].n * S.ap.lay[l].n, S.z_atm + 2 * static_cast<size_t>(P.gp.coff[l]), st);
        CK(cudaStreamSynchronize(st));  // the seed slot is reused by the next layer
    }
    sim::k_atm_spectrum<<<dim3(maxn, S.L), maxn, 0, st>>>(S.ap, S.z_atm, S.cplx);
    sim::k_atm_dft<<<dim3(maxn, S.L), maxn, 0, st>>>(S.ap, S.cplx, S.cplx2, 0);
    sim::k_atm_dft<<<dim3(maxn, S.L), maxn, 0, st>>>(S.ap, S.cplx2, S.cplx, 1);
    sim::k_atm_finish<<<S.L, 1024, 0, st>>>(S.ap, S.cplx, S.truth);
    CK(cudaGetLastError());
}

// truth_at_step(truth, g, step) -> out (the truth itself when there is no wind or step 0)
const double* sim_truth_at_step(SimState& S, const double* base, int step, double* out, cudaStream_t st) {
    if (!S.wind || step == 0) return base;
    sim::FlowParams fp{};
    fp.L = S.L;
    int maxnn = 0;
    for (int l = 0; l < S.L; ++l) {
        fp.n[l] = S.ap.lay[l].n;
        fp.off[l] = S.ap.lay[l].off;
        fp.si[l] = S.wind_sp[static_cast<size_t>(l)].first * step;
        fp.sj[l] = S.wind_sp[static_cast<size_t>(l)].second * step;
        maxnn = std::max(maxnn, fp.n[l] * fp.n[l]);
    }
    sim::k_frozen_flow<<<dim3((maxnn + 255) / 256, S.L), 256, 0, st>>>(fp, base, out);
    CK(cudaGetLastError());
    return out;
}

// synthesize_measurements(layers, a, g, noise_seed): forward model + the frame's noise
// (normals z of its stream, or none) -> meas (device)
void sim_slopes(EngineImpl& P, SimState& S, const double* layers, const double* a, const double* z, double* meas,
                cudaStream_t st) {
    const double* noise = nullptr;
    if (z) {
        sim::k_noise_scatter<<<(S.pairs + 255) / 256, 256, 0, st>>>(S.nx, S.ny, S.sig, S.pairs, z, S.noise);
        noise = S.noise;
    }
    const int sub = S.S / 2;
    k_slopes<double><<<dim3((sub + 255) / 256, 1), 256, 0, st>>>(P.gp64, nullptr, layers, a, -1.0, noise, meas, 1);
    CK(cudaGetLastError());
}

// evaluate_quality(layers, a, g) -> rec[0] field_rms, rec[1] layer_rel_err, rec[2..] rms_per_dir
void sim_quality(SimState& S, const double* layers, const double* a, double* rec, cudaStream_t st) {
    sim::k_quality_dir<<<S.n_dir, 512, S.nodes * sizeof(double), st>>>(S.qp, layers, a, S.var);
    if (S.paired) sim::k_layer_err<<<S.L, 1024, 0, st>>>(S.lp, layers, a, S.part);
    sim::k_quality_finish<<<1, 32, 0, st>>>(S.var, S.n_dir, S.part, S.L, S.paired ? 1 : 0, rec);
    CK(cudaGetLastError());
}

// the engine's a^(-1) (state a_prev2, instance 0) as doubles
const double* sim_dm(EngineImpl& P, SimState& S, cudaStream_t st) {
    if (P.precision == 64) return P.sd.bf.a_prev2;
    k_convert<float, double><<<(S.A + 255) / 256, 256, 0, st>>>(P.sf.bf.a_prev2, S.dm, static_cast<size_t>(S.A));
    CK(cudaGetLastError());
    return S.dm;
}
}  // namespace

// A bare GaussianStream on the device (for known-answer tests of k_gauss).
void sim_gauss_stream(int device, unsigned long long seed, int count, double* out) {
    CK(cudaSetDevice(device));
    unsigned long long* ds = dalloc<unsigned long long>(1);
    double* dz = dalloc<double>(static_cast<size_t>(count));
    CK(cudaMemcpy(ds, &seed, sizeof(seed), cudaMemcpyHostToDevice));
    sim::k_gauss<<<1, 32>>>(ds, count, dz, count);
    const cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) CK(cudaMemcpy(out, dz, sizeof(double) * count, cudaMemcpyDeviceToHost));
    cudaFree(ds);
    cudaFree(dz);
    CK(e);
}

int Engine::sim_quality_size() {
    return 2 + sim_state(*p_).n_dir;
}

void Engine::sim_atmosphere(unsigned long long seed, int step, double* layers_out) {
    auto& P = *p_;
    CK(cudaSetDevice(P.device));
    SimState& S = sim_state(P);
    const cudaStream_t st = P.stream;
    fewha_gpu::sim_atmosphere(P, S, seed, st);
    const double* l = sim_truth_at_step(S, S.truth, step, S.layers, st);
    CK(cudaMemcpyAsync(layers_out, l, sizeof(double) * S.n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
}

void Engine::sim_synthesize(const double* layers, const double* a, unsigned long long noise_seed, double* meas) {
    auto& P = *p_;
    CK(cudaSetDevice(P.device));
    SimState& S = sim_state(P);
    const cudaStream_t st = P.stream;
    CK(cudaMemcpyAsync(S.layers, layers, sizeof(double) * S.n, cudaMemcpyHostToDevice, st));
    if (a) CK(cudaMemcpyAsync(S.dm, a, sizeof(double) * S.A, cudaMemcpyHostToDevice, st));
    double* z = nullptr;
    if (P.g.sim_noise) {
        if (S.z_cap < 1) {
            S.z = S.alloc<double>(2 * static_cast<size_t>(S.pairs));
            S.z_cap = 1;
        }
        sim_normals(P, S, {splitmix64(noise_seed ^ 0x6e0f7a3dULL)}, 2 * S.pairs, S.z, st);
        z = S.z;
    }
    Work<double>& w = P.pd.count ? P.pd : P.od;
    if (w.count < 1) w.alloc(P.gp64, 1, P.fr, false);
    sim_slopes(P, S, S.layers, a ? S.dm : nullptr, z, w.meas2, st);
    CK(cudaMemcpyAsync(meas, w.meas2, sizeof(double) * S.S, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
}

void Engine::sim_quality(const double* layers, const double* a, double* rec) {
    auto& P = *p_;
    CK(cudaSetDevice(P.device));
    SimState& S = sim_state(P);
    const cudaStream_t st = P.stream;
    CK(cudaMemcpyAsync(S.layers, layers, sizeof(double) * S.n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(S.dm, a, sizeof(double) * S.A, cudaMemcpyHostToDevice, st));
    double* d = S.alloc<double>(2 + S.n_dir);
    fewha_gpu::sim_quality(S, S.layers, S.dm, d, st);
    CK(cudaMemcpyAsync(rec, d, sizeof(double) * (2 + S.n_dir), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
}

// run_closed_loop (simulation.hpp:321-345) with every frame on the device: the
// handle's state is reset (a fresh Reconstructor in the reference), the truth
// generated once, the noise streams of a chunk of frames generated together, and
// per frame only kernel launches: frozen flow, slopes into the frame's input
// slot, quality of a^(-1), the frame graph, its rho log kept on the device.
// rec: [n_steps][2 + n_dir] (field_rms, layer_rel_err, rms_per_dir); rho
// [n_steps][iters]; unc_final {uncorrected field RMS, final field RMS}.
void Engine::run_closed_loop(int n_steps, unsigned long long atm_seed, unsigned long long noise_seed, double* rec,
                             double* rho, double* unc_final) {
    auto& P = *p_;
    if (n_steps < 1) throw ArgError("run_closed_loop: n_steps must be >= 1");
    if (P.batch != 1 || P.sharded) throw ArgError("run_closed_loop: single-instance, unsharded handles only");
    CK(cudaSetDevice(P.device));
    SimState& S = sim_state(P);
    if (!P.has_precond) P.build_precond();
    reset();
    const cudaStream_t st = P.s();
    fewha_gpu::sim_atmosphere(P, S, atm_seed, st);
    const int RW = 2 + S.n_dir, it = P.gp.iters;
    double* drec = S.alloc<double>(static_cast<size_t>(n_steps) * RW);
    double* drho = S.alloc<double>(static_cast<size_t>(n_steps) * it);
    double* dunc = S.alloc<double>(static_cast<size_t>(RW));
    constexpr int kChunk = 128;
    const int zc = 2 * S.pairs;
    if (P.g.sim_noise && S.z_cap < kChunk) {
        S.z = S.alloc<double>(static_cast<size_t>(kChunk) * std::max(zc, 1));
        S.z_cap = kChunk;
    }
    double* meas = P.precision == 64 ? P.sd.meas : P.sf.meas;
    const double* rho_log = P.precision == 64 ? P.sd.bf.rho_log : P.sf.bf.rho_log;
    if (P.precision == 64) {
        P.ensure_graph<double>();
        P.set_fit_a_host<double>(nullptr);
    } else {
        P.ensure_graph<float>();
        P.set_fit_a_host<float>(nullptr);
    }
    const double* lay = S.truth;
    for (int k0 = 0; k0 < n_steps; k0 += kChunk) {
        const int nk = std::min(kChunk, n_steps - k0);
        if (P.g.sim_noise) {  // the chunk's noise streams, one warp each
            std::vector<unsigned long long> seeds(static_cast<size_t>(nk));
            for (int k = 0; k < nk; ++k)
                seeds[static_cast<size_t>(k)] =
                    splitmix64(splitmix64(noise_seed + static_cast<std::uint64_t>(k0 + k)) ^ 0x6e0f7a3dULL);
            sim_normals(P, S, seeds, zc, S.z, st);
        }
        for (int k = 0; k < nk; ++k) {
            const int step = k0 + k;
            lay = sim_truth_at_step(S, S.truth, step, S.layers, st);
            const double* a2 = sim_dm(P, S, st);
            sim_slopes(P, S, lay, a2, P.g.sim_noise ? S.z + static_cast<size_t>(k) * zc : nullptr,
                       meas, st);
            fewha_gpu::sim_quality(S, lay, a2, drec + static_cast<size_t>(step) * RW, st);
            CK(cudaGraphLaunch(P.graph, st));
            CK(cudaMemcpyAsync(drho + static_cast<size_t>(step) * it, rho_log, sizeof(double) * it,
                               cudaMemcpyDeviceToDevice, st));
            ++P.step_counter;
        }
        CK(cudaStreamSynchronize(st));  // the chunk's normals are consumed before the next chunk
    }
    fewha_gpu::sim_quality(S, lay, S.zero_dm, dunc, st);
    CK(cudaMemcpyAsync(rec, drec, sizeof(double) * static_cast<size_t>(n_steps) * RW, cudaMemcpyDeviceToHost, st));
    if (rho) CK(cudaMemcpyAsync(rho, drho, sizeof(double) * static_cast<size_t>(n_steps) * it, cudaMemcpyDeviceToHost, st));
    double unc[2];
    CK(cudaMemcpyAsync(unc, dunc, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    unc[1] = rec[static_cast<size_t>(n_steps - 1) * RW];
    if (unc_final) {
        unc_final[0] = unc[0];
        unc_final[1] = unc[1];
    }
    sync_check();
}

}  // namespace fewha_gpu
