// Reference-side drop-in test: the reference's own callers' loops run through
// fewha_gpu::Reconstructor (include/fewha_gpu_reconstructor.hpp, over the C-ABI)
// and through the unmodified fewha::Reconstructor, side by side.
//
// Compiled by tests/cpp/Makefile against the reference headers
// (/root/reference/proj/include, unmodified) and the in-tree libfewha_gpu.so;
// run on a GPU by tests/test_gpu_dropin.py.  Exit status 0 = every check passed.
//
//   run_bench loop      bench.hpp:144-154 (closed loop: synthesize_measurements
//                       with st.a_prev2 feedback, splitmix64 noise seeds)
//   run_closed_loop     simulation.hpp:321-345 (+ evaluate_quality per frame)
//   StateMirror::full   every ReconstructorState field vs the reference's
//   reset               ReconstructorState::reset (reconstructor.hpp:81-91)
//   errors              config_error / invalid_argument as the reference throws
#include <fewha/config_io.hpp>
#include <fewha/reconstructor.hpp>
#include <fewha/simulation.hpp>

#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "fewha_gpu_reconstructor.hpp"

namespace {
int failures = 0;

void expect(bool ok, const std::string& what, double v = 0.0) {
    std::printf("%s %-58s %.3e\n", ok ? "ok  " : "FAIL", what.c_str(), v);
    if (!ok) ++failures;
}

std::vector<double> flat(const fewha::MirrorShapes& a) {
    std::vector<double> out;
    for (const auto& m : a.dm) out.insert(out.end(), m.data(), m.data() + m.size());
    return out;
}

double rel(const std::vector<double>& a, const std::vector<double>& b) { return fewha::rel_err(a, b); }

// bench.hpp:144-154, both reconstructors fed their own closed-loop measurements
void run_bench_loop(const std::string& name, const fewha::SystemGeometry& g, int frames, std::uint64_t seed,
                    fewha_gpu::StateMirror mirror) {
    const fewha::AtmosphereTruth truth = fewha::generate_atmosphere(g, seed);
    fewha::Reconstructor ref(g);
    ref.build_preconditioner();
    fewha_gpu::Options opt;
    opt.mirror = mirror;
    fewha_gpu::Reconstructor gpu(g, opt);
    gpu.build_preconditioner();
    expect(fewha::rel_err(gpu.preconditioner(), ref.preconditioner()) <= 1e-12, name + ": preconditioner",
           fewha::rel_err(gpu.preconditioner(), ref.preconditioner()));
    fewha::ReconstructorState st_ref = fewha::ReconstructorState::zero(g);
    fewha::ReconstructorState st_gpu = fewha::ReconstructorState::zero(g);
    double worst_c = 0, worst_a = 0, worst_rho = 0, worst_state = 0;
    for (int k = 0; k < frames; ++k) {
        const auto layers = fewha::truth_at_step(truth, g, k);
        const auto m_ref = fewha::synthesize_measurements(layers, &st_ref.a_prev2, g,
                                                          fewha::splitmix64(seed + static_cast<std::uint64_t>(k)));
        const auto m_gpu = fewha::synthesize_measurements(layers, &st_gpu.a_prev2, g,
                                                          fewha::splitmix64(seed + static_cast<std::uint64_t>(k)));
        const auto a_ref = ref.step(st_ref, m_ref);
        const auto a_gpu = gpu.step(st_gpu, m_gpu);
        worst_c = std::max(worst_c, rel(st_gpu.c, st_ref.c));
        worst_a = std::max(worst_a, rel(flat(a_gpu), flat(a_ref)));
        worst_a = std::max(worst_a, rel(flat(st_gpu.a_prev2), flat(st_ref.a_prev2)));
        worst_rho = std::max(worst_rho, rel(gpu.last_telemetry().rho, ref.last_telemetry().rho));
        if (gpu.last_telemetry().step != ref.last_telemetry().step) expect(false, name + ": telemetry step counter");
        if (mirror == fewha_gpu::StateMirror::full) {
            for (auto [u, v] : {std::pair{&st_gpu.b, &st_ref.b}, {&st_gpu.r, &st_ref.r}, {&st_gpu.p, &st_ref.p},
                                {&st_gpu.q, &st_ref.q}})
                worst_state = std::max(worst_state, rel(*u, *v));
            worst_state = std::max(worst_state, std::abs(st_gpu.pcg.rho_old - st_ref.pcg.rho_old) /
                                                    std::abs(st_ref.pcg.rho_old));
            if (st_gpu.pcg.fresh != st_ref.pcg.fresh) worst_state = 1.0;
        }
    }
    const std::string tag = name + (mirror == fewha_gpu::StateMirror::full ? " [full]" : " [outputs]");
    expect(worst_c <= 1e-9, tag + ": run_bench loop st.c", worst_c);
    expect(worst_a <= 1e-9, tag + ": run_bench loop a^(1), a^(-1)", worst_a);
    expect(worst_rho <= 1e-9, tag + ": run_bench loop rho", worst_rho);
    if (mirror == fewha_gpu::StateMirror::full)
        expect(worst_state <= 1e-9, tag + ": full state b, r, p, q, scalars", worst_state);
    // an outputs-mode caller can still read the whole state on demand
    gpu.pull_state(st_gpu);
    expect(rel(st_gpu.r, st_ref.r) <= 1e-9, tag + ": pull_state r", rel(st_gpu.r, st_ref.r));
}

// simulation.hpp:321-345 with the reconstructor swapped
void run_closed_loop(const std::string& name, const fewha::SystemGeometry& g, int n_steps) {
    const fewha::LoopResult want = fewha::run_closed_loop(g, n_steps, {}, 0);
    const fewha::AtmosphereTruth truth = fewha::generate_atmosphere(g, fewha::LoopSeeds{}.atmosphere);
    fewha_gpu::Reconstructor rec(g);
    rec.build_preconditioner();
    fewha::ReconstructorState st = fewha::ReconstructorState::zero(g);
    double worst = 0, worst_rho = 0;
    for (int k = 0; k < n_steps; ++k) {
        const auto layers_k = fewha::truth_at_step(truth, g, k);
        const auto meas = fewha::synthesize_measurements(
            layers_k, &st.a_prev2, g, fewha::splitmix64(fewha::LoopSeeds{}.noise + static_cast<std::uint64_t>(k)));
        const fewha::QualityRecord q = fewha::evaluate_quality(layers_k, st.a_prev2, g);
        rec.step(st, meas);
        const auto& w = want.records[static_cast<std::size_t>(k)];
        worst = std::max(worst, std::abs(q.field_rms - w.field_rms) / std::max(w.field_rms, 1e-300));
        worst_rho = std::max(worst_rho, rel(rec.last_telemetry().rho, w.rho));
    }
    expect(worst <= 1e-9, name + ": run_closed_loop field_rms per frame", worst);
    expect(worst_rho <= 1e-9, name + ": run_closed_loop rho per frame", worst_rho);
}

void reset_and_errors(const std::string& name, const fewha::SystemGeometry& g) {
    fewha::Reconstructor ref(g);
    fewha_gpu::Reconstructor gpu(g);
    fewha::ReconstructorState st_ref = fewha::ReconstructorState::zero(g), st = fewha::ReconstructorState::zero(g);
    const auto m1 = fewha::synthesize_measurements(fewha::generate_atmosphere(g, 5).layers, nullptr, g, 19);
    const auto m2 = fewha::synthesize_measurements(fewha::generate_atmosphere(g, 6).layers, nullptr, g, 23);
    gpu.step(st, m1);
    gpu.step(st, m2);
    st.reset();  // the caller's own reset: the wrapper sees it and uploads the cold state
    const auto a = gpu.step(st, m1);
    const auto a_ref = ref.step(st_ref, m1);
    expect(rel(flat(a), flat(a_ref)) <= 1e-9, name + ": reset == cold start", rel(flat(a), flat(a_ref)));
    std::vector<double> x(gpu.coeff_layout().total), y(x.size()), y_ref(x.size());
    for (std::size_t i = 0; i < x.size(); ++i) x[i] = std::sin(0.37 * static_cast<double>(i));
    gpu.apply_M(x, y);
    ref.apply_M(x, y_ref);
    expect(rel(y, y_ref) <= 1e-12, name + ": apply_M", rel(y, y_ref));
    bool threw = false;
    try {
        std::vector<double> short_meas(3);
        gpu.step(st, short_meas);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    expect(threw, name + ": size mismatch -> std::invalid_argument");
    threw = false;
    fewha::SystemGeometry bad = g;
    bad.gain = 1.5;
    try {
        fewha_gpu::Reconstructor r(bad);
    } catch (const fewha::config_error&) {
        threw = true;
    }
    expect(threw, name + ": invalid geometry -> fewha::config_error");
}
}  // namespace

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : "presets";
    for (const char* name : {"small_mcao", "maory"}) {
        const fewha::SystemGeometry g = fewha::load_config(dir + "/" + name + ".json");
        const int frames = std::string(name) == "maory" ? 6 : 12;
        run_bench_loop(name, g, frames, 1, fewha_gpu::StateMirror::outputs);
        run_bench_loop(name, g, frames, 2, fewha_gpu::StateMirror::full);
        run_closed_loop(name, g, frames);
        reset_and_errors(name, g);
    }
    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "PASSED", failures);
    return failures ? 1 : 0;
}
