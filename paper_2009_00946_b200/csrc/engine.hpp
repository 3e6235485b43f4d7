// Host-side engine: owns the geometry tables, the device-resident state of
// `batch` reconstructor instances, and the captured per-frame CUDA graph.
#pragma once

#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "geometry.hpp"

namespace fewha_gpu {

struct EngineImpl;

// StepTelemetry (reconstructor.hpp:94-102), device-timed
struct StepTelemetry {
    long long step = 0;
    bool valid = false;
    double stage1_us = 0, stage2_us = 0, stage3_us = 0, pcg_us = 0, fit_us = 0, total_us = 0;
};

// Execution plan an engine chose for its batch size (engine.cu build_plan / Launch)
struct PlanInfo {
    int cluster_ctas = 0, tail = 0, gather_rows = 0, gather_ctas_per_sm = 0, inverse_staged = 0, wfs_ctas_per_sm = 0,
        wfs_tiles = 0, launches_per_step = 0, whole_layer = 0, gather_instances = 1, wfs_instances = 1,
        gather_direct = 0;
};

class Engine;
// contiguous WFS range [first, second) of shard `rank` of `world` (balanced by wavefront nodes)
std::pair<int, int> shard_range(const Geometry& g, int rank, int world);
// GaussianStream(seed) (simulation.hpp:40-58) drawn on the device: count normals
void sim_gauss_stream(int device, unsigned long long seed, int count, double* out);
// one frame of an in-process shard group, members in rank order
void group_step_device(const std::vector<Engine*>& members);

class Engine {
public:
    Engine(Geometry g, int precision, int batch, int device);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    const Geometry& geometry() const;
    int precision() const;
    int batch() const;

    void override_loop(int loop_mode, double gain);
    void build_preconditioner();
    bool has_preconditioner() const;
    std::vector<double> preconditioner() const;

    // Reconstructor::step for all instances; host fp64 buffers (outputs may be null).
    void step(const double* slopes, double* coeffs, double* dm, double* rho, int* n_rho);
    void reset();
    void get_state(int instance, double* c, double* b, double* r, double* p, double* q, double* sc,
                   double* a_prev2, double* a_prev);
    void set_state(int instance, const double* c, const double* b, const double* r, const double* p,
                   const double* q, const double* sc, const double* a_prev2, const double* a_prev);

    // device-resident path
    void set_stream(void* stream);
    void step_device(const void* d_slopes);
    void load_slopes(const void* src, bool on_device);
    void sync_check();
    void read_outputs(double* coeffs, double* dm, double* rho, int* n_rho);
    void enable_telemetry(bool on);
    StepTelemetry last_telemetry();
    int last_launch_times(float* ms, int* kinds, int max);
    int launches_per_step() const;
    PlanInfo plan_info() const;
    int profile_step(float* ms, int* kinds, int max);
    void enable_stamps(bool on);
    float bench_dwt(int variant, int inverse, int reps, int threads);
    int read_stamps(unsigned long long* out, size_t n);
    void device_buffers(void** slopes, void** coeffs, void** dm, double** rho, int** status, int** n_rho);

    // per-WFS sharding: own WFS shard_range(g, rank, world); nccl_id
    // (128-byte ncclUniqueId) joins a multi-process NCCL exchange, null forms an
    // in-process group member (group_step_device)
    void shard(int rank, int world, const void* nccl_id);
    std::pair<int, int> shard_wfs() const;
    void* shard_partial(int seg) const;
    friend void group_step_device(const std::vector<Engine*>& members);

    // operator entry points (count stacked host inputs)
    void apply_M(const double* in, double* out, int count);
    void build_rhs(const double* meas, double* out, int count);
    void add_dm_slopes(const double* a, double* meas, int count);
    void fit(const double* c, double* a, int count);
    void wavelet(int inverse, double* data, int count);
    void propagate(const double* layers, double* wf, int count);
    void propagate_transpose(const double* wf, double* layers, int count);
    void sh(const double* wf, double* meas, int count);
    void sh_transpose(const double* meas, double* wf, int count);
    void forward_slopes(const double* layers, const double* a, double* meas, int count);
    void wfs_operator(int rhs, const double* in, const double* meas, double* psi, int count);

    // closed-loop simulation harness on the device (simulation.hpp)
    int sim_quality_size();  // 2 + probe directions
    void sim_atmosphere(unsigned long long seed, int step, double* layers_out);
    void sim_synthesize(const double* layers, const double* a, unsigned long long noise_seed, double* meas);
    void sim_quality(const double* layers, const double* a, double* rec);
    void run_closed_loop(int n_steps, unsigned long long atm_seed, unsigned long long noise_seed, double* rec,
                         double* rho, double* unc_final);

private:
    std::unique_ptr<EngineImpl> p_;
};

}  // namespace fewha_gpu
