// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (never linked by the product).
//
// A C-ABI shim over the UNMODIFIED reference implementation.  It is compiled
// in place against /root/reference/proj/include (nothing is copied into this
// repo) by oracle/Makefile into oracle/_ref/libfewha_ref.so.  It is used to
//   * pin the C restatement in oracle/fewha_oracle.c (tests/test_oracle_*.py),
//   * generate the golden fixtures under tests/golden/ (make_golden.py),
//   * time the reference CPU solver for bench.py's cpu_baseline / --impl reference.
//
// Entry points mirror the reference C++ API used by callers of the hot path:
//   load_config            proj/include/fewha/config_io.hpp:181
//   Reconstructor ctor     proj/include/fewha/reconstructor.hpp:112
//   build_preconditioner   reconstructor.hpp:250
//   step                   reconstructor.hpp:310
//   apply_M / build_rhs    reconstructor.hpp:166 / :215
//   add_dm_slopes / fit    reconstructor.hpp:259 / :284
//   synthesize_measurements, generate_atmosphere  simulation.hpp:164 / :76
//   GaussianStream, truth_at_step, evaluate_quality, run_closed_loop
//                          simulation.hpp:40 / :131 / :228 / :321
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "fewha/config_io.hpp"
#include "fewha/reconstructor.hpp"
#include "fewha/simulation.hpp"

using namespace fewha;

namespace {

struct RefHandle {
    SystemGeometry g;
    std::unique_ptr<Reconstructor> rec;
    ReconstructorState st;
    std::unique_ptr<AtmosphereTruth> truth;
    std::uint64_t truth_seed = ~0ULL;
    std::string err;
};

thread_local std::string g_last_error;

std::size_t total_act(const SystemGeometry& g) {
    std::size_t a = 0;
    for (const auto& d : g.dms) a += static_cast<std::size_t>(d.n_act) * d.n_act;
    return a;
}
std::size_t total_wf(const SystemGeometry& g) {
    std::size_t a = 0;
    for (const auto& w : g.wfs) a += static_cast<std::size_t>(w.n_subap + 1) * (w.n_subap + 1);
    return a;
}

void mirrors_to_flat(const MirrorShapes& a, double* out) {
    for (const auto& m : a.dm) {
        std::memcpy(out, m.data(), m.size() * sizeof(double));
        out += m.size();
    }
}
void flat_to_mirrors(const double* in, MirrorShapes& a) {
    for (auto& m : a.dm) {
        std::memcpy(m.data(), in, m.size() * sizeof(double));
        in += m.size();
    }
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const config_error& e) {
        g_last_error = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return 1;
    }
}

const AtmosphereTruth& truth_for(RefHandle* h, std::uint64_t seed) {
    if (!h->truth || h->truth_seed != seed) {
        h->truth = std::make_unique<AtmosphereTruth>(generate_atmosphere(h->g, seed));
        h->truth_seed = seed;
    }
    return *h->truth;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

// Load a preset exactly as the reference CLI does (load_config ->
// finalize_geometry) and build a Reconstructor + zero state.
// loop_mode: -1 keep, 0 closed, 1 open.  gain < 0: keep.
int ref_create(const char* path, int threads, int loop_mode, double gain, void** out) {
    return guarded([&] {
        auto h = std::make_unique<RefHandle>();
        h->g = load_config(path);
        if (loop_mode == 0) h->g.loop_mode = LoopMode::closed;
        if (loop_mode == 1) h->g.loop_mode = LoopMode::open;
        if (gain >= 0.0) h->g.gain = gain;
        h->rec = std::make_unique<Reconstructor>(h->g, threads);
        h->st = ReconstructorState::zero(h->g);
        *out = h.release();
    });
}

void ref_destroy(void* hp) { delete static_cast<RefHandle*>(hp); }

// dims: [n_coeff, n_meas, n_act_total, L, W, M, iters, n_wavefront_total, threads]
void ref_dims(void* hp, long long* d) {
    auto* h = static_cast<RefHandle*>(hp);
    d[0] = static_cast<long long>(h->g.coeff_dim());
    d[1] = static_cast<long long>(h->g.measurement_dim());
    d[2] = static_cast<long long>(total_act(h->g));
    d[3] = static_cast<long long>(h->g.layers.size());
    d[4] = static_cast<long long>(h->g.wfs.size());
    d[5] = static_cast<long long>(h->g.dms.size());
    d[6] = h->g.solver.pcg_max_iter;
    d[7] = static_cast<long long>(total_wf(h->g));
    d[8] = h->rec->threads();
}

// Derived geometry (finalize_geometry, geometry.hpp:366-377): layer extents,
// DM extents, concatenated active masks (n_s^2 per WFS, row-major).
void ref_geometry(void* hp, double* layer_extent, double* dm_extent, unsigned char* masks) {
    auto* h = static_cast<RefHandle*>(hp);
    for (std::size_t l = 0; l < h->g.layers.size(); ++l) layer_extent[l] = h->g.layers[l].extent;
    for (std::size_t m = 0; m < h->g.dms.size(); ++m) dm_extent[m] = h->g.dms[m].extent;
    for (const auto& w : h->g.wfs) {
        std::memcpy(masks, w.active_mask.on.data(), w.active_mask.on.size());
        masks += w.active_mask.on.size();
    }
}

int ref_build_preconditioner(void* hp) {
    return guarded([&] { static_cast<RefHandle*>(hp)->rec->build_preconditioner(); });
}

void ref_preconditioner(void* hp, double* out) {
    const auto& p = static_cast<RefHandle*>(hp)->rec->preconditioner();
    std::memcpy(out, p.data(), p.size() * sizeof(double));
}

// One reconstruction frame on the handle's own state.  Any output may be NULL.
// rho_out receives up to `iters` values; *n_rho the log length.
int ref_step(void* hp, const double* meas, double* c_out, double* dm_out, double* rho_out, int* n_rho,
             double* step_us) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        std::span<const double> m(meas, h->g.measurement_dim());
        const auto t0 = std::chrono::steady_clock::now();
        MirrorShapes a = h->rec->step(h->st, m);
        const auto t1 = std::chrono::steady_clock::now();
        if (step_us) *step_us = std::chrono::duration<double, std::micro>(t1 - t0).count();
        if (c_out) std::memcpy(c_out, h->st.c.data(), h->st.c.size() * sizeof(double));
        if (dm_out) mirrors_to_flat(a, dm_out);
        const auto& rho = h->rec->last_telemetry().rho;
        if (rho_out) std::memcpy(rho_out, rho.data(), rho.size() * sizeof(double));
        if (n_rho) *n_rho = static_cast<int>(rho.size());
    });
}

void ref_reset(void* hp) { static_cast<RefHandle*>(hp)->st.reset(); }

// State transfer: c, b, r, p, q (n each), scalars {rho_old, alpha, fresh},
// a_prev2 (A), a_prev (A).  Matches ReconstructorState (reconstructor.hpp:61-92).
void ref_get_state(void* hp, double* c, double* b, double* r, double* p, double* q, double* sc,
                   double* a_prev2, double* a_prev) {
    auto* h = static_cast<RefHandle*>(hp);
    const std::size_t n = h->st.c.size() * sizeof(double);
    std::memcpy(c, h->st.c.data(), n);
    std::memcpy(b, h->st.b.data(), n);
    std::memcpy(r, h->st.r.data(), n);
    std::memcpy(p, h->st.p.data(), n);
    std::memcpy(q, h->st.q.data(), n);
    sc[0] = h->st.pcg.rho_old;
    sc[1] = h->st.pcg.alpha;
    sc[2] = h->st.pcg.fresh ? 1.0 : 0.0;
    mirrors_to_flat(h->st.a_prev2, a_prev2);
    mirrors_to_flat(h->st.a_prev, a_prev);
}

void ref_set_state(void* hp, const double* c, const double* b, const double* r, const double* p,
                   const double* q, const double* sc, const double* a_prev2, const double* a_prev) {
    auto* h = static_cast<RefHandle*>(hp);
    const std::size_t n = h->st.c.size();
    h->st.c.assign(c, c + n);
    h->st.b.assign(b, b + n);
    h->st.r.assign(r, r + n);
    h->st.p.assign(p, p + n);
    h->st.q.assign(q, q + n);
    h->st.pcg.rho_old = sc[0];
    h->st.pcg.alpha = sc[1];
    h->st.pcg.fresh = sc[2] != 0.0;
    flat_to_mirrors(a_prev2, h->st.a_prev2);
    flat_to_mirrors(a_prev, h->st.a_prev);
}

int ref_apply_M(void* hp, const double* in, double* out) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        const std::size_t n = h->g.coeff_dim();
        h->rec->apply_M(std::span<const double>(in, n), std::span<double>(out, n));
    });
}

int ref_build_rhs(void* hp, const double* meas, double* b_out) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        h->rec->build_rhs(std::span<const double>(meas, h->g.measurement_dim()),
                          std::span<double>(b_out, h->g.coeff_dim()));
    });
}

// meas += Gamma P_dm a  (closed-loop pseudo open-loop term)
int ref_add_dm_slopes(void* hp, const double* a_flat, double* meas) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        MirrorShapes a = MirrorShapes::zero(h->g);
        flat_to_mirrors(a_flat, a);
        h->rec->add_dm_slopes(a, std::span<double>(meas, h->g.measurement_dim()));
    });
}

int ref_fit(void* hp, const double* coeffs, double* dm_out) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        auto a = h->rec->fit_to_mirrors(std::span<const double>(coeffs, h->g.coeff_dim()));
        mirrors_to_flat(a, dm_out);
    });
}

// Per-layer W^-1 (dir=1) or W (dir=0) on the concatenated coefficient vector.
int ref_wavelet(void* hp, int dir, double* data) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        const auto& lay = h->rec->coeff_layout();
        for (std::size_t l = 0; l < lay.side.size(); ++l) {
            const int s = lay.side[l];
            Grid2D grid(s, s);
            std::memcpy(grid.data(), data + lay.offset[l], grid.size() * sizeof(double));
            if (dir) h->rec->wavelet().inverse(grid);
            else h->rec->wavelet().forward(grid);
            std::memcpy(data + lay.offset[l], grid.data(), grid.size() * sizeof(double));
        }
    });
}

// P: nodal layers (n) -> concatenated wavefronts ((n_s+1)^2 per WFS).
int ref_propagate(void* hp, const double* layers, double* wf_out) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        const auto& lay = h->rec->coeff_layout();
        std::vector<Grid2D> grids;
        for (std::size_t l = 0; l < lay.side.size(); ++l) {
            grids.emplace_back(lay.side[l], lay.side[l]);
            std::memcpy(grids.back().data(), layers + lay.offset[l], grids.back().size() * sizeof(double));
        }
        for (std::size_t w = 0; w < h->g.wfs.size(); ++w) {
            const int n = h->g.wfs[w].n_subap + 1;
            Grid2D wf(n, n);
            propagate(grids, h->g, static_cast<int>(w), wf);
            std::memcpy(wf_out, wf.data(), wf.size() * sizeof(double));
            wf_out += wf.size();
        }
    });
}

// P^T: concatenated wavefronts -> nodal layers, sum over WFS in ascending order.
int ref_propagate_transpose(void* hp, const double* wf_in, double* layers_out) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        const auto& lay = h->rec->coeff_layout();
        std::vector<Grid2D> wfs;
        const double* p = wf_in;
        for (const auto& w : h->g.wfs) {
            wfs.emplace_back(w.n_subap + 1, w.n_subap + 1);
            std::memcpy(wfs.back().data(), p, wfs.back().size() * sizeof(double));
            p += wfs.back().size();
        }
        for (std::size_t l = 0; l < lay.side.size(); ++l) {
            Grid2D acc(lay.side[l], lay.side[l]);
            for (std::size_t w = 0; w < wfs.size(); ++w)
                propagate_transpose_layer(wfs[w], h->g, static_cast<int>(w), static_cast<int>(l), acc);
            std::memcpy(layers_out + lay.offset[l], acc.data(), acc.size() * sizeof(double));
        }
    });
}

// Gamma: concatenated wavefronts -> measurement vector.
int ref_sh(void* hp, const double* wf_in, double* meas_out) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        const auto& ml = h->rec->measurement_layout();
        const double* p = wf_in;
        std::span<double> m(meas_out, ml.total);
        for (std::size_t w = 0; w < h->g.wfs.size(); ++w) {
            const int n = h->g.wfs[w].n_subap + 1;
            Grid2D wf(n, n);
            std::memcpy(wf.data(), p, wf.size() * sizeof(double));
            p += wf.size();
            h->rec->sh(static_cast<int>(w), wf, ml.sx(m, h->g, static_cast<int>(w)),
                       ml.sy(m, h->g, static_cast<int>(w)));
        }
    });
}

// Gamma^T: measurement vector -> concatenated wavefronts.
int ref_sh_transpose(void* hp, const double* meas, double* wf_out) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        const auto& ml = h->rec->measurement_layout();
        std::span<const double> m(meas, ml.total);
        for (std::size_t w = 0; w < h->g.wfs.size(); ++w) {
            const int n = h->g.wfs[w].n_subap + 1;
            Grid2D wf(n, n);
            h->rec->sh_transpose(static_cast<int>(w), ml.sx(m, h->g, static_cast<int>(w)),
                                 ml.sy(m, h->g, static_cast<int>(w)), wf);
            std::memcpy(wf_out, wf.data(), wf.size() * sizeof(double));
            wf_out += wf.size();
        }
    });
}

// Truth layers of generate_atmosphere(g, seed) (simulation.hpp:76), nodal, n values.
int ref_atmosphere(void* hp, unsigned long long seed, double* layers_out) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        const auto& t = truth_for(h, seed);
        for (const auto& l : t.layers) {
            std::memcpy(layers_out, l.data(), l.size() * sizeof(double));
            layers_out += l.size();
        }
    });
}

// synthesize_measurements(truth_at_step(truth(seed), k), a_prev2 or none, splitmix64(seed + k))
// -- exactly the slope stream run_bench feeds to step (bench.hpp:144-154).
int ref_synthesize(void* hp, unsigned long long seed, int k, const double* a_prev2, double* meas_out) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        const auto& t = truth_for(h, seed);
        const auto layers = truth_at_step(t, h->g, k);
        std::unique_ptr<MirrorShapes> corr;
        if (a_prev2) {
            corr = std::make_unique<MirrorShapes>(MirrorShapes::zero(h->g));
            flat_to_mirrors(a_prev2, *corr);
        }
        const auto meas = synthesize_measurements(layers, corr.get(), h->g,
                                                  splitmix64(seed + static_cast<std::uint64_t>(k)));
        std::memcpy(meas_out, meas.data(), meas.size() * sizeof(double));
    });
}

// Record a closed-loop run from the current state: per frame k the slopes
// fed to step (synthesised with the state's own a_prev2), then step.
// Outputs per frame (any may be NULL): meas [S], c [n], dm [A], rho [iters],
// step wall time [us].
int ref_record(void* hp, unsigned long long seed, int k0, int frames, double* meas_out, double* c_out,
               double* dm_out, double* rho_out, double* us_out) {
    auto* h = static_cast<RefHandle*>(hp);
    const std::size_t S = h->g.measurement_dim(), n = h->g.coeff_dim(), A = total_act(h->g);
    const int it = h->g.solver.pcg_max_iter;
    return guarded([&] {
        const auto& t = truth_for(h, seed);
        for (int f = 0; f < frames; ++f) {
            const int k = k0 + f;
            const auto layers = truth_at_step(t, h->g, k);
            const auto meas = synthesize_measurements(layers, &h->st.a_prev2, h->g,
                                                      splitmix64(seed + static_cast<std::uint64_t>(k)));
            const auto t0 = std::chrono::steady_clock::now();
            MirrorShapes a = h->rec->step(h->st, meas);
            const auto t1 = std::chrono::steady_clock::now();
            if (us_out) us_out[f] = std::chrono::duration<double, std::micro>(t1 - t0).count();
            if (meas_out) std::memcpy(meas_out + f * S, meas.data(), S * sizeof(double));
            if (c_out) std::memcpy(c_out + f * n, h->st.c.data(), n * sizeof(double));
            if (dm_out) mirrors_to_flat(a, dm_out + f * A);
            if (rho_out) {
                const auto& rho = h->rec->last_telemetry().rho;
                for (int i = 0; i < it; ++i)
                    rho_out[f * it + i] = i < static_cast<int>(rho.size()) ? rho[i] : 0.0;
            }
        }
    });
}

// Time `frames` steps over a caller-provided slope stream (stream_len frames,
// cycled), steady_clock around step only (bench.hpp:128-131 methodology).
int ref_time_steps(void* hp, const double* meas_stream, int stream_len, int frames, double* us_out) {
    auto* h = static_cast<RefHandle*>(hp);
    const std::size_t S = h->g.measurement_dim();
    return guarded([&] {
        for (int f = 0; f < frames; ++f) {
            std::span<const double> m(meas_stream + (f % stream_len) * S, S);
            const auto t0 = std::chrono::steady_clock::now();
            h->rec->step(h->st, m);
            const auto t1 = std::chrono::steady_clock::now();
            us_out[f] = std::chrono::duration<double, std::micro>(t1 - t0).count();
        }
    });
}

// Gaussian stream of the simulation (simulation.hpp:40-58): the first `count`
// draws of GaussianStream(seed).
int ref_gauss(unsigned long long seed, int count, double* out) {
    return guarded([&] {
        GaussianStream g(seed);
        for (int i = 0; i < count; ++i) out[i] = g();
    });
}

// truth_at_step(generate_atmosphere(seed), k) (simulation.hpp:131-158), nodal [n].
int ref_truth_at_step(void* hp, unsigned long long seed, int k, double* layers_out) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        for (const auto& l : truth_at_step(truth_for(h, seed), h->g, k)) {
            std::memcpy(layers_out, l.data(), l.size() * sizeof(double));
            layers_out += l.size();
        }
    });
}

// evaluate_quality(layers, correction, g) (simulation.hpp:228-305): out =
// [field_rms, layer_rel_err, rms_per_dir...].
int ref_quality(void* hp, const double* layers, const double* dm_flat, double* out) {
    auto* h = static_cast<RefHandle*>(hp);
    return guarded([&] {
        std::vector<Grid2D> lay;
        for (const auto& lc : h->g.layers) {
            Grid2D gl(lc.n_nodes(), lc.n_nodes());
            std::memcpy(gl.data(), layers, gl.size() * sizeof(double));
            layers += gl.size();
            lay.push_back(std::move(gl));
        }
        MirrorShapes corr = MirrorShapes::zero(h->g);
        flat_to_mirrors(dm_flat, corr);
        const QualityRecord q = evaluate_quality(lay, corr, h->g);
        out[0] = q.field_rms;
        out[1] = q.layer_rel_err;
        for (std::size_t d = 0; d < q.rms_per_dir.size(); ++d) out[2 + d] = q.rms_per_dir[d];
    });
}

// run_closed_loop(g, n_steps, {atm, noise}, threads) (simulation.hpp:321-345):
// per step field_rms, layer_rel_err, rho [iters] (0-padded); scalars out2 =
// [uncorrected_field_rms, final_field_rms].
int ref_run_closed_loop(void* hp, int n_steps, unsigned long long atm, unsigned long long noise, int threads,
                        double* field_rms, double* layer_err, double* rho, double* out2) {
    auto* h = static_cast<RefHandle*>(hp);
    const int it = h->g.solver.pcg_max_iter;
    return guarded([&] {
        const LoopResult r = run_closed_loop(h->g, n_steps, LoopSeeds{atm, noise}, threads);
        for (int k = 0; k < n_steps; ++k) {
            const auto& q = r.records[static_cast<std::size_t>(k)];
            field_rms[k] = q.field_rms;
            layer_err[k] = q.layer_rel_err;
            for (int i = 0; i < it; ++i) rho[k * it + i] = i < static_cast<int>(q.rho.size()) ? q.rho[i] : 0.0;
        }
        out2[0] = r.uncorrected_field_rms;
        out2[1] = r.final_field_rms;
    });
}

// Wavelet transform on a single square grid (for filter-order coverage).
int ref_wavelet_grid(int order, int n, int dir, double* data) {
    return guarded([&] {
        Wavelet2D wv(order);
        Grid2D g(n, n);
        std::memcpy(g.data(), data, g.size() * sizeof(double));
        if (dir) wv.inverse(g);
        else wv.forward(g);
        std::memcpy(data, g.data(), g.size() * sizeof(double));
    });
}

}  // extern "C"
