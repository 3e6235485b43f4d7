// include/fewha_gpu_reconstructor.hpp -- header-only C++ drop-in for the
// reference's fewha::Reconstructor (proj/include/fewha/reconstructor.hpp:104-386)
// over the C-ABI of include/fewha_gpu.h.
//
// A reference-side caller swaps one type:
//
//     #include <fewha/config_io.hpp>
//     #include "fewha_gpu_reconstructor.hpp"
//     fewha::SystemGeometry g = fewha::load_config(path);        // config_io.hpp:181
//     fewha_gpu::Reconstructor rec(g);                            // was fewha::Reconstructor rec(g)
//     rec.build_preconditioner();                                 // reconstructor.hpp:250
//     fewha::ReconstructorState st = fewha::ReconstructorState::zero(g);
//     fewha::MirrorShapes a = rec.step(st, meas);                 // reconstructor.hpp:310
//     rec.last_telemetry().rho;                                   // reconstructor.hpp:147
//
// Geometry: the wrapper serialises the caller's SystemGeometry with the
// reference's own geometry_to_json (config_io.hpp:197) and the library parses it
// with the same schema, defaults and validation (fewha_gpu_create_from_json), so
// both sides see the same derived extents and masks.
//
// State: the reference keeps ReconstructorState in the caller's hands and updates
// it in place; here the state lives in HBM and the wrapper mirrors it.
//   StateMirror::full     every step uploads the caller's state (c, b, r, p, q, PCG
//                         scalars, a^(-1), a^(0)) and mirrors all of it back --
//                         exactly the reference's semantics for any caller, at the
//                         cost of ~10 n doubles of PCIe traffic per frame.
//   StateMirror::outputs  (default) the device state is authoritative while the
//                         caller keeps stepping the same ReconstructorState object:
//                         after each step st.c, st.pcg, st.a_prev2 and st.a_prev
//                         are mirrored (what callers read: run_closed_loop and
//                         run_bench use st.a_prev2, st.c); b, r, p, q are fetched by
//                         pull_state(st).  A different state object, or one whose
//                         PCG scalars no longer match the mirrored ones (e.g. after
//                         st.reset(), reconstructor.hpp:81-91), is uploaded in full
//                         before the step.  Callers that edit b, r, p, q or c by
//                         hand use StateMirror::full or push_state(st).
//
// Errors map back to the reference's exception types: FEWHA_CONFIG ->
// fewha::config_error, FEWHA_ARG -> std::invalid_argument, FEWHA_RUNTIME ->
// std::runtime_error (non-finite PCG scalar, CUDA failure).
#pragma once

#include <fewha/config_io.hpp>
#include <fewha/reconstructor.hpp>

#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "fewha_gpu.h"

namespace fewha_gpu {

enum class StateMirror { outputs, full };

struct Options {
    int precision = 64;  // 64 (parity mode) or 32
    int device = 0;      // CUDA ordinal
    StateMirror mirror = StateMirror::outputs;
};

namespace detail {
[[noreturn]] inline void raise(int code, const char* msg) {
    const std::string m = msg ? msg : "fewha_gpu: unknown error";
    if (code == FEWHA_CONFIG) throw fewha::config_error(m);
    if (code == FEWHA_ARG) throw std::invalid_argument(m);
    throw std::runtime_error(m);
}
}  // namespace detail

class Reconstructor {
public:
    explicit Reconstructor(fewha::SystemGeometry geom, int threads = 0) : Reconstructor(std::move(geom), Options{}) {
        (void)threads;  // the device path has no host thread pool
    }
    Reconstructor(fewha::SystemGeometry geom, Options opt)
        : geom_(std::move(geom)),
          opt_(opt),
          mlay_(fewha::MeasurementLayout::of(geom_)),
          clay_(fewha::CoeffLayout::of(geom_)) {
        const std::string text = fewha::geometry_to_json(geom_).dump();
        const int rc = fewha_gpu_create_from_json(text.c_str(), opt_.precision, 1, opt_.device, &h_);
        if (rc != FEWHA_OK) detail::raise(rc, fewha_gpu_create_error());
        fewha_gpu_dims_t d{};
        check(fewha_gpu_dims(h_, &d));
        n_ = static_cast<std::size_t>(d.n_coeff);
        S_ = static_cast<std::size_t>(d.n_slopes);
        A_ = static_cast<std::size_t>(d.n_act);
        iters_ = d.pcg_iters;
        if (n_ != clay_.total || S_ != mlay_.total)
            throw std::logic_error("fewha_gpu::Reconstructor: device layout differs from the reference's");
        a_buf_.assign(A_, 0.0);
        rho_buf_.assign(static_cast<std::size_t>(iters_), 0.0);
    }
    ~Reconstructor() {
        if (h_) fewha_gpu_destroy(h_);
    }
    Reconstructor(const Reconstructor&) = delete;
    Reconstructor& operator=(const Reconstructor&) = delete;

    static int default_threads(const fewha::SystemGeometry& g) { return fewha::Reconstructor::default_threads(g); }

    const fewha::SystemGeometry& geometry() const { return geom_; }
    const fewha::MeasurementLayout& measurement_layout() const { return mlay_; }
    const fewha::CoeffLayout& coeff_layout() const { return clay_; }
    const fewha::StepTelemetry& last_telemetry() const { return telemetry_; }
    int threads() const { return 1; }
    fewha_gpu_t handle() const { return h_; }

    void build_preconditioner() {
        check(fewha_gpu_build_preconditioner(h_));
        precond_.assign(n_, 0.0);
        check(fewha_gpu_preconditioner(h_, precond_.data()));
    }
    const std::vector<double>& preconditioner() const { return precond_; }

    // -- operator entry points (reconstructor.hpp:166-305) ---------------------------
    void apply_M(std::span<const double> c_in, std::span<double> c_out) {
        if (c_in.size() != n_ || c_out.size() != n_) throw std::invalid_argument("apply_M: coefficient length mismatch");
        check(fewha_gpu_apply_M(h_, c_in.data(), c_out.data(), 1));
    }
    void build_rhs(std::span<const double> meas, std::span<double> b_out) {
        if (meas.size() != S_ || b_out.size() != n_) throw std::invalid_argument("build_rhs: length mismatch");
        check(fewha_gpu_build_rhs(h_, meas.data(), b_out.data(), 1));
    }
    void add_dm_slopes(const fewha::MirrorShapes& a, std::span<double> meas) {
        if (meas.size() != S_) throw std::invalid_argument("add_dm_slopes: length mismatch");
        const auto flat = flatten(a);
        check(fewha_gpu_add_dm_slopes(h_, flat.data(), meas.data(), 1));
    }
    fewha::MirrorShapes fit_to_mirrors(std::span<const double> coeffs) {
        if (coeffs.size() != n_) throw std::invalid_argument("fit_to_mirrors: coefficient length mismatch");
        check(fewha_gpu_fit_to_mirrors(h_, coeffs.data(), a_buf_.data(), 1));
        return unflatten(a_buf_.data());
    }

    // -- the hot path: one loop step (reconstructor.hpp:310-355) -----------------------
    fewha::MirrorShapes step(fewha::ReconstructorState& st, std::span<const double> meas) {
        if (meas.size() != S_) throw std::invalid_argument("step: measurement length mismatch");
        if (st.c.size() != n_ || st.r.size() != n_ || st.b.size() != n_ || st.p.size() != n_ || st.q.size() != n_)
            throw std::invalid_argument("step: state does not match the geometry");
        if (precond_.empty()) build_preconditioner();
        if (opt_.mirror == StateMirror::full || bound_ != &st || !same_scalars(st.pcg)) push_state(st);
        telemetry_ = fewha::StepTelemetry{};
        telemetry_.step = ++step_counter_;
        int nr = 0;
        check(fewha_gpu_step(h_, meas.data(), st.c.data(), a_buf_.data(), rho_buf_.data(), &nr));
        telemetry_.rho.assign(rho_buf_.begin(), rho_buf_.begin() + nr);
        fewha_gpu_telemetry_t t{};
        if (fewha_gpu_last_telemetry(h_, &t) == FEWHA_OK && t.valid) {
            telemetry_.stage1_us = t.stage1_us;
            telemetry_.stage2_us = t.stage2_us;
            telemetry_.stage3_us = t.stage3_us;
            telemetry_.pcg_us = t.pcg_us;
            telemetry_.total_us = t.total_us;
        }
        fewha::MirrorShapes a_next = unflatten(a_buf_.data());
        if (opt_.mirror == StateMirror::full) {
            pull_state(st);
        } else {  // the history rotation (reconstructor.hpp:350-351) and the carried scalars
            st.a_prev2 = std::move(st.a_prev);
            st.a_prev = a_next;
            pull_scalars(st);
        }
        return a_next;
    }

    // -- explicit state transfer --------------------------------------------------------
    void push_state(const fewha::ReconstructorState& st) {
        auto a2 = flatten(st.a_prev2), a1 = flatten(st.a_prev);
        fewha_gpu_state_t s{};
        s.c = const_cast<double*>(st.c.data());
        s.b = const_cast<double*>(st.b.data());
        s.r = const_cast<double*>(st.r.data());
        s.p = const_cast<double*>(st.p.data());
        s.q = const_cast<double*>(st.q.data());
        s.scalars[0] = st.pcg.rho_old;
        s.scalars[1] = st.pcg.alpha;
        s.scalars[2] = st.pcg.fresh ? 1.0 : 0.0;
        s.a_prev2 = a2.data();
        s.a_prev = a1.data();
        check(fewha_gpu_set_state(h_, 0, &s));
        bound_ = &st;
        scalars_ = st.pcg;
    }
    void pull_state(fewha::ReconstructorState& st) {
        std::vector<double> a2(A_), a1(A_);
        fewha_gpu_state_t s{};
        s.c = st.c.data();
        s.b = st.b.data();
        s.r = st.r.data();
        s.p = st.p.data();
        s.q = st.q.data();
        s.a_prev2 = a2.data();
        s.a_prev = a1.data();
        check(fewha_gpu_get_state(h_, 0, &s));
        st.pcg.rho_old = s.scalars[0];
        st.pcg.alpha = s.scalars[1];
        st.pcg.fresh = s.scalars[2] != 0.0;
        st.a_prev2 = unflatten(a2.data());
        st.a_prev = unflatten(a1.data());
        bound_ = &st;
        scalars_ = st.pcg;
    }

private:
    void check(int rc) const {
        if (rc != FEWHA_OK) detail::raise(rc, fewha_gpu_last_error(h_));
    }
    bool same_scalars(const fewha::PcgScalars& s) const {
        return s.fresh == scalars_.fresh && std::memcmp(&s.rho_old, &scalars_.rho_old, sizeof(double)) == 0 &&
               std::memcmp(&s.alpha, &scalars_.alpha, sizeof(double)) == 0;
    }
    void pull_scalars(fewha::ReconstructorState& st) {
        fewha_gpu_state_t s{};  // null vectors: the PCG scalars alone
        check(fewha_gpu_get_state(h_, 0, &s));
        st.pcg.rho_old = s.scalars[0];
        st.pcg.alpha = s.scalars[1];
        st.pcg.fresh = s.scalars[2] != 0.0;
        bound_ = &st;
        scalars_ = st.pcg;
    }
    std::vector<double> flatten(const fewha::MirrorShapes& a) const {
        std::vector<double> out;
        out.reserve(A_);
        for (const auto& m : a.dm) out.insert(out.end(), m.data(), m.data() + m.size());
        if (out.size() != A_) throw std::invalid_argument("mirror shapes do not match the geometry");
        return out;
    }
    fewha::MirrorShapes unflatten(const double* v) const {
        fewha::MirrorShapes a = fewha::MirrorShapes::zero(geom_);
        for (auto& m : a.dm) {
            std::memcpy(m.data(), v, m.size() * sizeof(double));
            v += m.size();
        }
        return a;
    }

    fewha::SystemGeometry geom_;
    Options opt_;
    fewha::MeasurementLayout mlay_;
    fewha::CoeffLayout clay_;
    fewha_gpu_t h_ = nullptr;
    std::size_t n_ = 0, S_ = 0, A_ = 0;
    int iters_ = 0;
    std::vector<double> a_buf_, rho_buf_, precond_;
    fewha::StepTelemetry telemetry_;
    int step_counter_ = -1;
    const fewha::ReconstructorState* bound_ = nullptr;
    fewha::PcgScalars scalars_{};
};

}  // namespace fewha_gpu
