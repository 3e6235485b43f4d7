// extern "C" boundary (include/fewha_gpu.h): maps C++ exceptions onto the
// reference's error taxonomy -- config_error -> FEWHA_CONFIG (CLI exit 2),
// runtime_error -> FEWHA_RUNTIME (exit 1), invalid_argument -> FEWHA_ARG
// (tools/fewha_cli.cpp:31-33, :157-163).
#include "fewha_gpu.h"

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "engine.hpp"
#include "nccl_dl.hpp"

using fewha_gpu::ArgError;
using fewha_gpu::ConfigError;
using fewha_gpu::Engine;

struct fewha_gpu_handle {
    std::unique_ptr<Engine> eng;  // the engine (member 0 of a multi-device handle)
    // fewha_gpu_create_multi with n_devices > 1: shard members 1..n-1 (member 0 is eng)
    // of an in-process per-WFS group stepped together by fewha_gpu_step
    std::vector<std::unique_ptr<Engine>> more;
    std::string err;
    bool group() const { return !more.empty(); }
    std::vector<Engine*> members() const {
        std::vector<Engine*> m{eng.get()};
        for (const auto& e : more) m.push_back(e.get());
        return m;
    }
};

namespace {
thread_local std::string g_create_error;

template <typename F>
int guard(std::string& err, F&& f) {
    try {
        f();
        err.clear();
        return FEWHA_OK;
    } catch (const ConfigError& e) {
        err = e.what();
        return FEWHA_CONFIG;
    } catch (const ArgError& e) {
        err = e.what();
        return FEWHA_ARG;
    } catch (const std::invalid_argument& e) {
        err = e.what();
        return FEWHA_ARG;
    } catch (const std::exception& e) {
        err = e.what();
        return FEWHA_RUNTIME;
    }
}

int create(fewha_gpu::Geometry (*parse)(const std::string&), const char* src, int precision, int batch, int device,
           fewha_gpu_t* out) {
    if (!out || !src) {
        g_create_error = "null argument";
        return FEWHA_ARG;
    }
    *out = nullptr;
    return guard(g_create_error, [&] {
        auto h = std::make_unique<fewha_gpu_handle>();
        h->eng = std::make_unique<Engine>(parse(src), precision, batch, device);
        *out = h.release();
    });
}

#define H_GUARD(body)                    \
    if (!h) return FEWHA_ARG;            \
    return guard(h->err, [&] { body; });
}  // namespace

extern "C" {

int fewha_gpu_create(const char* path, int precision, int batch, int device, fewha_gpu_t* out) {
    return create(&fewha_gpu::parse_preset_file, path, precision, batch, device, out);
}

int fewha_gpu_create_from_json(const char* text, int precision, int batch, int device, fewha_gpu_t* out) {
    return create(&fewha_gpu::parse_preset_text, text, precision, batch, device, out);
}

int fewha_gpu_create_multi(const char* path, int precision, int batch, const int* devices, int n_devices,
                           fewha_gpu_t* out) {
    if (!out || !path || !devices || n_devices < 1) {
        g_create_error = "null argument or no device";
        return FEWHA_ARG;
    }
    *out = nullptr;
    return guard(g_create_error, [&] {
        const auto g = fewha_gpu::parse_preset_file(path);
        auto h = std::make_unique<fewha_gpu_handle>();
        h->eng = std::make_unique<Engine>(g, precision, batch, devices[0]);
        for (int r = 1; r < n_devices; ++r) h->more.push_back(std::make_unique<Engine>(g, precision, batch, devices[r]));
        if (n_devices > 1) {  // per-WFS shards of one frame, exchanged by peer loads
            auto m = h->members();
            for (int r = 0; r < n_devices; ++r) m[static_cast<size_t>(r)]->shard(r, n_devices, nullptr);
        }
        *out = h.release();
    });
}

int fewha_gpu_override_loop(fewha_gpu_t h, int loop_mode, double gain) { H_GUARD(h->eng->override_loop(loop_mode, gain)) }

const char* fewha_gpu_create_error(void) { return g_create_error.c_str(); }
const char* fewha_gpu_last_error(fewha_gpu_t h) { return h ? h->err.c_str() : "null handle"; }
void fewha_gpu_destroy(fewha_gpu_t h) { delete h; }

int fewha_gpu_dims(fewha_gpu_t h, fewha_gpu_dims_t* d) {
    H_GUARD({
        const auto& g = h->eng->geometry();
        d->n_coeff = static_cast<long long>(g.coeff_dim());
        d->n_slopes = static_cast<long long>(g.measurement_dim());
        d->n_act = static_cast<long long>(g.act_dim());
        d->n_wavefront = static_cast<long long>(g.wavefront_dim());
        d->n_layers = static_cast<int>(g.layers.size());
        d->n_wfs = static_cast<int>(g.wfs.size());
        d->n_dms = static_cast<int>(g.dms.size());
        d->pcg_iters = g.pcg_iters;
        d->batch = h->eng->batch();
        d->precision = h->eng->precision();
    })
}

int fewha_gpu_preset_info(const char* path, fewha_gpu_dims_t* d, double* layer_extent, double* dm_extent,
                          unsigned char* masks) {
    if (!path) return FEWHA_ARG;
    return guard(g_create_error, [&] {
        const auto g = fewha_gpu::parse_preset_file(path);
        if (d) {
            d->n_coeff = static_cast<long long>(g.coeff_dim());
            d->n_slopes = static_cast<long long>(g.measurement_dim());
            d->n_act = static_cast<long long>(g.act_dim());
            d->n_wavefront = static_cast<long long>(g.wavefront_dim());
            d->n_layers = static_cast<int>(g.layers.size());
            d->n_wfs = static_cast<int>(g.wfs.size());
            d->n_dms = static_cast<int>(g.dms.size());
            d->pcg_iters = g.pcg_iters;
            d->batch = 0;
            d->precision = 0;
        }
        if (layer_extent)
            for (size_t l = 0; l < g.layers.size(); ++l) layer_extent[l] = g.layers[l].extent;
        if (dm_extent)
            for (size_t m = 0; m < g.dms.size(); ++m) dm_extent[m] = g.dms[m].extent;
        if (masks)
            for (const auto& w : g.wfs) {
                std::memcpy(masks, w.mask.data(), w.mask.size());
                masks += w.mask.size();
            }
    });
}

int fewha_gpu_geometry(fewha_gpu_t h, double* layer_extent, double* dm_extent, unsigned char* masks) {
    H_GUARD({
        const auto& g = h->eng->geometry();
        for (size_t l = 0; l < g.layers.size(); ++l) layer_extent[l] = g.layers[l].extent;
        for (size_t m = 0; m < g.dms.size(); ++m) dm_extent[m] = g.dms[m].extent;
        for (const auto& w : g.wfs) {
            std::memcpy(masks, w.mask.data(), w.mask.size());
            masks += w.mask.size();
        }
    })
}

int fewha_gpu_build_preconditioner(fewha_gpu_t h) {
    H_GUARD(for (auto* m : h->members()) m->build_preconditioner())
}

int fewha_gpu_preconditioner(fewha_gpu_t h, double* out) {
    H_GUARD({
        if (!h->eng->has_preconditioner()) h->eng->build_preconditioner();
        const auto v = h->eng->preconditioner();
        std::memcpy(out, v.data(), v.size() * sizeof(double));
    })
}

int fewha_gpu_step(fewha_gpu_t h, const double* slopes, double* coeffs, double* dm, double* rho, int* n_rho) {
    H_GUARD({
        if (!slopes) throw ArgError("step: null slopes");
        if (!h->group()) {
            h->eng->step(slopes, coeffs, dm, rho, n_rho);
        } else {  // every shard reconstructs the same frame; the replicated outputs are read from member 0
            const auto m = h->members();
            for (auto* e : m) e->load_slopes(slopes, false);
            fewha_gpu::group_step_device(m);
            for (size_t r = 1; r < m.size(); ++r) m[r]->sync_check();
            h->eng->read_outputs(coeffs, dm, rho, n_rho);
        }
    })
}

int fewha_gpu_reset(fewha_gpu_t h) { H_GUARD(for (auto* m : h->members()) m->reset()) }

int fewha_gpu_get_state(fewha_gpu_t h, int instance, fewha_gpu_state_t* st) {
    H_GUARD(h->eng->get_state(instance, st->c, st->b, st->r, st->p, st->q, st->scalars, st->a_prev2, st->a_prev))
}

int fewha_gpu_set_state(fewha_gpu_t h, int instance, const fewha_gpu_state_t* st) {
    H_GUARD(for (auto* m : h->members())
                m->set_state(instance, st->c, st->b, st->r, st->p, st->q, st->scalars, st->a_prev2, st->a_prev))
}

int fewha_gpu_set_stream(fewha_gpu_t h, void* stream) { H_GUARD(h->eng->set_stream(stream)) }

int fewha_gpu_device_buffers(fewha_gpu_t h, fewha_gpu_device_t* o) {
    H_GUARD(h->eng->device_buffers(&o->slopes, &o->coeffs, &o->dm, &o->rho, &o->status, &o->n_rho))
}

int fewha_gpu_load_slopes(fewha_gpu_t h, const void* src, int on_device) {
    H_GUARD({
        if (!src) throw ArgError("load_slopes: null source");
        for (auto* m : h->members()) m->load_slopes(src, on_device != 0);
    })
}
int fewha_gpu_step_device(fewha_gpu_t h, const void* d_slopes) {
    H_GUARD({
        if (!h->group()) {
            h->eng->step_device(d_slopes);
        } else {
            const auto m = h->members();
            if (d_slopes)
                for (auto* e : m) e->load_slopes(d_slopes, true);
            fewha_gpu::group_step_device(m);
        }
    })
}
int fewha_gpu_sync(fewha_gpu_t h) { H_GUARD(for (auto* m : h->members()) m->sync_check()) }
int fewha_gpu_launches_per_step(fewha_gpu_t h) { return h ? h->eng->launches_per_step() : -1; }
int fewha_gpu_plan_info(fewha_gpu_t h, fewha_gpu_plan_t* out) {
    if (!out) return FEWHA_ARG;
    H_GUARD({
        const auto pi = h->eng->plan_info();
        out->cluster_ctas = pi.cluster_ctas;
        out->tail = pi.tail;
        out->gather_rows = pi.gather_rows;
        out->gather_ctas_per_sm = pi.gather_ctas_per_sm;
        out->inverse_staged = pi.inverse_staged;
        out->wfs_ctas_per_sm = pi.wfs_ctas_per_sm;
        out->wfs_tiles = pi.wfs_tiles;
        out->launches_per_step = pi.launches_per_step;
        out->whole_layer = pi.whole_layer;
        out->gather_instances = pi.gather_instances;
        out->wfs_instances = pi.wfs_instances;
        out->gather_direct = pi.gather_direct;
    })
}
float fewha_gpu_debug_bench_dwt(fewha_gpu_t h, int variant, int inverse, int reps, int threads) {
    float ms = -1.f;
    if (!h) return ms;
    guard(h->err, [&] { ms = h->eng->bench_dwt(variant, inverse, reps, threads); });
    return ms;
}
int fewha_gpu_phase_stamps(fewha_gpu_t h, unsigned long long* out, long long n) {
    if (!h) return -1;
    int got = 0;
    const int rc = guard(h->err, [&] {
        h->eng->enable_stamps(true);
        got = out ? h->eng->read_stamps(out, static_cast<size_t>(n)) : 0;
    });
    return rc ? -rc : got;
}
int fewha_gpu_profile_step(fewha_gpu_t h, float* ms, int* kinds, int max) {
    if (!h) return -1;
    int n = -1;
    const int rc = guard(h->err, [&] { n = h->eng->profile_step(ms, kinds, max); });
    return rc ? -rc : n;
}

int fewha_gpu_apply_M(fewha_gpu_t h, const double* in, double* out, int count) { H_GUARD(h->eng->apply_M(in, out, count)) }
int fewha_gpu_build_rhs(fewha_gpu_t h, const double* meas, double* out, int count) {
    H_GUARD(h->eng->build_rhs(meas, out, count))
}
int fewha_gpu_add_dm_slopes(fewha_gpu_t h, const double* a, double* meas, int count) {
    H_GUARD(h->eng->add_dm_slopes(a, meas, count))
}
int fewha_gpu_fit_to_mirrors(fewha_gpu_t h, const double* c, double* a, int count) { H_GUARD(h->eng->fit(c, a, count)) }
int fewha_gpu_wavelet(fewha_gpu_t h, int inverse, double* data, int count) {
    H_GUARD(h->eng->wavelet(inverse, data, count))
}
int fewha_gpu_propagate(fewha_gpu_t h, const double* layers, double* wf, int count) {
    H_GUARD(h->eng->propagate(layers, wf, count))
}
int fewha_gpu_propagate_transpose(fewha_gpu_t h, const double* wf, double* layers, int count) {
    H_GUARD(h->eng->propagate_transpose(wf, layers, count))
}
int fewha_gpu_sh(fewha_gpu_t h, const double* wf, double* meas, int count) { H_GUARD(h->eng->sh(wf, meas, count)) }
int fewha_gpu_sh_transpose(fewha_gpu_t h, const double* meas, double* wf, int count) {
    H_GUARD(h->eng->sh_transpose(meas, wf, count))
}
int fewha_gpu_forward_slopes(fewha_gpu_t h, const double* layers, const double* a, double* meas, int count) {
    H_GUARD(h->eng->forward_slopes(layers, a, meas, count))
}

int fewha_gpu_wfs_operator(fewha_gpu_t h, int rhs, const double* in, const double* meas, double* psi, int count) {
    H_GUARD({
        if (rhs ? !meas : !in) throw ArgError("wfs_operator: null input");
        h->eng->wfs_operator(rhs, in, meas, psi, count);
    })
}

int fewha_gpu_enable_telemetry(fewha_gpu_t h, int on) { H_GUARD(h->eng->enable_telemetry(on != 0)) }

int fewha_gpu_last_telemetry(fewha_gpu_t h, fewha_gpu_telemetry_t* out) {
    if (!out) return FEWHA_ARG;
    H_GUARD({
        const auto t = h->eng->last_telemetry();
        out->step = t.step;
        out->valid = t.valid ? 1 : 0;
        out->stage1_us = t.stage1_us;
        out->stage2_us = t.stage2_us;
        out->stage3_us = t.stage3_us;
        out->pcg_us = t.pcg_us;
        out->fit_us = t.fit_us;
        out->total_us = t.total_us;
    })
}

int fewha_gpu_last_launch_times(fewha_gpu_t h, float* ms, int* kinds, int max) {
    if (!h || !ms || !kinds) return -FEWHA_ARG;
    int n = 0;
    const int rc = guard(h->err, [&] { n = h->eng->last_launch_times(ms, kinds, max); });
    return rc ? -rc : n;
}

// ---- closed-loop simulation harness on the device ----
int fewha_gpu_sim_gauss(int device, unsigned long long seed, int count, double* out) {
    if (!out || count < 0) return FEWHA_ARG;
    return guard(g_create_error, [&] { fewha_gpu::sim_gauss_stream(device, seed, count, out); });
}
int fewha_gpu_sim_quality_size(fewha_gpu_t h) {
    if (!h) return -FEWHA_ARG;
    int n = 0;
    const int rc = guard(h->err, [&] { n = h->eng->sim_quality_size(); });
    return rc ? -rc : n;
}
int fewha_gpu_sim_atmosphere(fewha_gpu_t h, unsigned long long seed, int step, double* layers) {
    H_GUARD({
        if (!layers || step < 0) throw ArgError("sim_atmosphere: null output or negative step");
        h->eng->sim_atmosphere(seed, step, layers);
    })
}
int fewha_gpu_sim_synthesize(fewha_gpu_t h, const double* layers, const double* a, unsigned long long noise_seed,
                             double* meas) {
    H_GUARD({
        if (!layers || !meas) throw ArgError("sim_synthesize: null argument");
        h->eng->sim_synthesize(layers, a, noise_seed, meas);
    })
}
int fewha_gpu_sim_quality(fewha_gpu_t h, const double* layers, const double* a, double* rec) {
    H_GUARD({
        if (!layers || !a || !rec) throw ArgError("sim_quality: null argument");
        h->eng->sim_quality(layers, a, rec);
    })
}
int fewha_gpu_run_closed_loop(fewha_gpu_t h, int n_steps, unsigned long long atmosphere_seed,
                              unsigned long long noise_seed, double* rec, double* rho, double* unc_final) {
    H_GUARD({
        if (!rec) throw ArgError("run_closed_loop: null record buffer");
        h->eng->run_closed_loop(n_steps, atmosphere_seed, noise_seed, rec, rho, unc_final);
    })
}

// ---- per-WFS sharding ----
int fewha_gpu_shard_range(const char* path, int rank, int world, int* wfs_begin, int* wfs_end) {
    if (!path) return FEWHA_ARG;
    return guard(g_create_error, [&] {
        const auto r = fewha_gpu::shard_range(fewha_gpu::parse_preset_file(path), rank, world);
        if (wfs_begin) *wfs_begin = r.first;
        if (wfs_end) *wfs_end = r.second;
    });
}

int fewha_gpu_nccl_unique_id(unsigned char* id) {
    if (!id) return FEWHA_ARG;
    return guard(g_create_error, [&] {
        const auto& api = fewha_gpu::NcclApi::get();
        ncclUniqueId u;
        api.check(api.GetUniqueId(&u), "ncclGetUniqueId");
        static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
        std::memcpy(id, &u, sizeof(u));
    });
}

int fewha_gpu_shard(fewha_gpu_t h, int rank, int world, const unsigned char* nccl_id) {
    H_GUARD(h->eng->shard(rank, world, nccl_id))
}

int fewha_gpu_shard_wfs(fewha_gpu_t h, int* wfs_begin, int* wfs_end) {
    H_GUARD({
        const auto r = h->eng->shard_wfs();
        if (wfs_begin) *wfs_begin = r.first;
        if (wfs_end) *wfs_end = r.second;
    })
}

int fewha_gpu_group_step_device(fewha_gpu_t* members, int world) {
    if (!members || world < 1) return FEWHA_ARG;
    for (int r = 0; r < world; ++r)
        if (!members[r]) return FEWHA_ARG;
    return guard(members[0]->err, [&] {
        std::vector<Engine*> m;
        for (int r = 0; r < world; ++r) m.push_back(members[r]->eng.get());
        fewha_gpu::group_step_device(m);
    });
}

}  // extern "C"
