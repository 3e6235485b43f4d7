/* include/fewha_gpu.h -- C-ABI of the B200-native FEWHA reconstructor.
 *
 * Drop-in boundary for the reference's hot path, reference
 * /root/reference/proj/include/fewha/ (file:line of the API each entry
 * replaces is given per function).  Plain pointers and sizes only; every
 * entry returns a status:
 *   FEWHA_OK (0)      success
 *   FEWHA_RUNTIME (1) runtime failure: non-finite PCG scalar, out-of-grid
 *                     interpolation, non-positive preconditioner, CUDA error
 *                     (reference: std::runtime_error; CLI exit code 1,
 *                     tools/fewha_cli.cpp:31-33, :157-163)
 *   FEWHA_CONFIG (2)  configuration error (reference: fewha::config_error;
 *                     CLI exit code 2)
 *   FEWHA_ARG (3)     bad argument / size mismatch (reference:
 *                     std::invalid_argument)
 * The message of the last failure is returned by fewha_gpu_last_error(h)
 * (or fewha_gpu_create_error() when no handle exists yet).
 *
 * Threading: one handle is externally single-threaded, like
 * Reconstructor::step.  Host buffers are caller-owned and
 * complete on return; device state is library-owned and resident in HBM.
 * Host vectors are always fp64; precision 32 computes in fp32 on the device.
 *
 * Layouts follow the reference exactly:
 *   slopes       per WFS [sx (n_s^2 row-major) | sy (n_s^2)]      operators.hpp:35-65
 *   coefficients per layer 2^J x 2^J Mallat layout, row-major   operators.hpp:67-91
 *   wavefronts   per WFS (n_s+1)^2 row-major                     operators.hpp:141-145
 *   DM commands  per DM n_act^2 row-major                        reconstructor.hpp:34-41
 * A `batch` handle holds `batch` independent instances (same geometry);
 * per-frame arrays are then batch-major ([instance][...]).
 */
#ifndef FEWHA_GPU_H
#define FEWHA_GPU_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FEWHA_OK 0
#define FEWHA_RUNTIME 1
#define FEWHA_CONFIG 2
#define FEWHA_ARG 3

typedef struct fewha_gpu_handle* fewha_gpu_t;

typedef struct {
    long long n_coeff;     /* n   = sum_l 4^J_l            (SystemGeometry::coeff_dim, geometry.hpp:171) */
    long long n_slopes;    /* S   = sum_w 2 n_s^2          (measurement_dim, geometry.hpp:176)          */
    long long n_act;       /* A   = sum_m n_act^2          (MirrorShapes, reconstructor.hpp:34-41)      */
    long long n_wavefront; /* N_w = sum_w (n_s+1)^2                                                    */
    int n_layers, n_wfs, n_dms, pcg_iters, batch, precision;
} fewha_gpu_dims_t;

/* Caller-owned host buffers for ReconstructorState (reconstructor.hpp:61-92). */
typedef struct {
    double *c, *b, *r, *p, *q; /* n each */
    double scalars[3];         /* PcgScalars {rho_old, alpha, fresh}, pcg.hpp:32-38 */
    double *a_prev2, *a_prev;  /* A each */
} fewha_gpu_state_t;

/* Device pointers (for CUDA-resident callers; valid until destroy). */
typedef struct {
    void* slopes;   /* [batch][S]  fp64 input slot read by fewha_gpu_step_device  */
    void* coeffs;   /* [batch][n]  st.c, element type = precision                  */
    void* dm;       /* [batch][A]  a^(1) of the last frame, element type = precision */
    double* rho;    /* [batch][iters] rho log of the last frame                   */
    int* status;    /* [batch] 0 ok, 1 non-finite PCG scalar                      */
    int* n_rho;     /* [batch] rho log length (< iters only with pcg_tolerance)    */
} fewha_gpu_device_t;

/* --- lifecycle ------------------------------------------------------------ */

/* load_config (config_io.hpp:181) + Reconstructor(geometry) (reconstructor.hpp:112).
 * precision: 64 or 32.  batch >= 1 independent instances.  device: CUDA ordinal.
 * Parses the JSON preset, validates it (geometry.hpp:281-362, same messages)
 * and derives extents and active masks (finalize_geometry, geometry.hpp:366-377).
 * L != M presets are accepted only with "fitting": see DESIGN.md (L=M otherwise,
 * as the reference).  */
int fewha_gpu_create(const char* preset_json_path, int precision, int batch, int device, fewha_gpu_t* out);
int fewha_gpu_create_from_json(const char* json_text, int precision, int batch, int device, fewha_gpu_t* out);
/* The SURVEY 8(b) multi-device form: devices[0..n_devices) (repeats allowed).  One
 * device: the same handle as fewha_gpu_create.  Several: an in-process per-WFS shard
 * group (fewha_gpu_shard semantics, one shard per listed device, peer access between
 * them): fewha_gpu_step / _step_device / _load_slopes / _reset / _set_state /
 * _build_preconditioner / _sync act on every shard and step them together (the
 * partial adjoint layer sums are summed in rank order from the shards' buffers);
 * outputs, state reads and the operator entry points come from shard 0 (the
 * replicated state is bitwise identical on every shard). */
int fewha_gpu_create_multi(const char* preset_json_path, int precision, int batch, const int* devices, int n_devices,
                           fewha_gpu_t* out);
/* loop_mode: -1 keep, 0 closed, 1 open; gain < 0 keeps (test hooks, like editing SystemGeometry) */
int fewha_gpu_override_loop(fewha_gpu_t h, int loop_mode, double gain);
const char* fewha_gpu_create_error(void);
const char* fewha_gpu_last_error(fewha_gpu_t h);
void fewha_gpu_destroy(fewha_gpu_t h);

int fewha_gpu_dims(fewha_gpu_t h, fewha_gpu_dims_t* out);
/* Host-only preset derivation (no device touched): load_config + finalize_geometry
 * (config_io.hpp:181, geometry.hpp:366-377).  Any output may be NULL. */
int fewha_gpu_preset_info(const char* preset_json_path, fewha_gpu_dims_t* dims, double* layer_extent,
                          double* dm_extent, unsigned char* masks);
/* derived geometry: layer extents [L], DM extents [M], masks [sum n_s^2] (uint8) */
int fewha_gpu_geometry(fewha_gpu_t h, double* layer_extent, double* dm_extent, unsigned char* masks);

/* --- preconditioner (Reconstructor::build_preconditioner, reconstructor.hpp:250;
 *     preconditioner_build, operators.hpp:367-425).  Built on the device from
 *     batched apply_M probes; lazily by the first step if never called. */
int fewha_gpu_build_preconditioner(fewha_gpu_t h);
int fewha_gpu_preconditioner(fewha_gpu_t h, double* out /* n */);

/* --- the hot path: Reconstructor::step (reconstructor.hpp:310-355) ---------
 * slopes [batch][S] (host, fp64).  Outputs may be NULL:
 *   coeffs_out [batch][n] = st.c after the step; dm_out [batch][A] = a^(1);
 *   rho_out [batch][iters] = last_telemetry().rho; n_rho [batch].
 * A page-locked dm_out is written directly by the frame's last kernel (no D2H copy). */
int fewha_gpu_step(fewha_gpu_t h, const double* slopes, double* coeffs_out, double* dm_out, double* rho_out,
                   int* n_rho);
/* ReconstructorState::reset (reconstructor.hpp:81-91) on every instance */
int fewha_gpu_reset(fewha_gpu_t h);
/* get_state: any vector pointer of *st may be NULL (not copied); scalars always are */
int fewha_gpu_get_state(fewha_gpu_t h, int instance, fewha_gpu_state_t* st);
int fewha_gpu_set_state(fewha_gpu_t h, int instance, const fewha_gpu_state_t* st);

/* --- CUDA-resident path (benchmarks, pipelines) ------------------------- */
int fewha_gpu_set_stream(fewha_gpu_t h, void* cuda_stream);
int fewha_gpu_device_buffers(fewha_gpu_t h, fewha_gpu_device_t* out);
/* Stage slopes [batch][S] fp64 into the resident slot, asynchronously on the
 * handle's stream (src on the device when on_device != 0, else host). */
int fewha_gpu_load_slopes(fewha_gpu_t h, const void* src, int on_device);
/* One frame from device slopes [batch][S] fp64 (NULL: use the library's slopes
 * slot).  Asynchronous on the handle's stream; no status check. */
int fewha_gpu_step_device(fewha_gpu_t h, const void* d_slopes);
/* Synchronise the stream and report the per-instance PCG status. */
int fewha_gpu_sync(fewha_gpu_t h);
/* Kernel launches of one step_device frame (for launch accounting). */
int fewha_gpu_launches_per_step(fewha_gpu_t h);
/* The execution plan the handle chose for its batch size (DESIGN.md "Batch-mode
 * choices"): CTAs per layer cluster, tail block side D of the cluster transforms,
 * adjoint-gather rows per CTA and its resident CTAs per SM, whether the inverse
 * kernel stages its operands by TMA (1) or streams them (0), resident WFS-tile
 * CTAs per SM, WFS tiles, kernel launches per frame. */
typedef struct {
    int cluster_ctas, tail, gather_rows, gather_ctas_per_sm, inverse_staged, wfs_ctas_per_sm, wfs_tiles,
        launches_per_step;
    int whole_layer; /* 1: layer transforms one CTA per (layer, instance) (batched plans), 2: the same with
                        forward(k) + inverse(k+1) fused in one launch (k_fwd_inv_layer), 0: clusters */
    int gather_instances, wfs_instances; /* instances per CTA of the adjoint gather / WFS-tile kernels */
    int gather_direct; /* 1: the direct gather (compile-time taps), 0: the row-contracted k_gather */
} fewha_gpu_plan_t;
int fewha_gpu_plan_info(fewha_gpu_t h, fewha_gpu_plan_t* out);
/* Runs ONE frame eagerly (not from the graph) with a CUDA event after every
 * launch on the handle's stream; writes per-launch device ms and kernel kind
 * (0 wfs_rhs, 1 adjoint, 2 fwd_rhs, 3 inv_pcg0, 4 inv_pcg, 5 wfs, 6 fwd_pcg,
 * 7 inv_fit, 8 fit_control).  Advances the state like a step.  Returns the
 * number of launches (< 0 on error). */
int fewha_gpu_profile_step(fewha_gpu_t h, float* ms, int* kinds, int max);
/* Profiling: the first call (out == NULL) enables per-phase %globaltimer stamps
 * of the cluster layer kernels for later fewha_gpu_profile_step frames; a call
 * with a buffer copies [32 launches][4096 blocks][16 stamps] (ns) out. */
int fewha_gpu_phase_stamps(fewha_gpu_t h, unsigned long long* out, long long n);

/* --- operator entry points (reconstructor.hpp:141-305, operators.hpp) ------
 * Each applies the operator to `count` stacked inputs (host, fp64). */
int fewha_gpu_apply_M(fewha_gpu_t h, const double* in, double* out, int count);              /* :166-212 */
int fewha_gpu_build_rhs(fewha_gpu_t h, const double* meas, double* b_out, int count);        /* :215-247 */
int fewha_gpu_add_dm_slopes(fewha_gpu_t h, const double* a, double* meas_inout, int count);  /* :259-280 */
int fewha_gpu_fit_to_mirrors(fewha_gpu_t h, const double* c, double* a_out, int count);      /* :284-305 */
int fewha_gpu_wavelet(fewha_gpu_t h, int inverse, double* data, int count); /* wavelet.hpp:115-143 per layer */
int fewha_gpu_propagate(fewha_gpu_t h, const double* layers, double* wf, int count);         /* operators.hpp:217 */
int fewha_gpu_propagate_transpose(fewha_gpu_t h, const double* wf, double* layers, int count); /* :241-268 */
int fewha_gpu_sh(fewha_gpu_t h, const double* wf, double* meas, int count);                  /* :145-164 */
int fewha_gpu_sh_transpose(fewha_gpu_t h, const double* meas, double* wf, int count);        /* :168-188 */
/* Noise-free forward model s = Gamma (P phi - P_dm a) (simulation.hpp:164-199);
 * a may be NULL (no correction).  layers: nodal [count][n]. */
int fewha_gpu_forward_slopes(fewha_gpu_t h, const double* layers, const double* a, double* meas, int count);

/* The frame's fused per-WFS kernel (k_wfs) applied on its own, so the hot-path
 * tile kernel is parity-tested in isolation (wavefronts [count][N_w] out):
 *   rhs = 0: psi = Gamma^T C^-1 Gamma P in, in = nodal layers [count][n]
 *            (apply_M stage 2, reconstructor.hpp:182-192)
 *   rhs = 1: psi = Gamma^T C^-1 (meas + Gamma P_dm in), in = DM commands
 *            [count][A] or NULL, meas [count][S] (add_dm_slopes :259-280 +
 *            build_rhs stage 1 :221-231).  The sh_adjoint fault factor applies. */
int fewha_gpu_wfs_operator(fewha_gpu_t h, int rhs, const double* in, const double* meas, double* psi, int count);

/* --- StepTelemetry (reconstructor.hpp:94-102; bench.hpp:214-228 CSV schema) ---
 * Opt-in: enabling re-captures the frame graph with an event-record node around
 * every launch (which also serialises programmatic launch overlap, so frames
 * run a few microseconds slower while it is on).  After a frame,
 * fewha_gpu_last_telemetry waits for it and fills the device-timed stages:
 *   stage1_us  W^-1 kernels (reference: per-layer W^-1 kernels)
 *   stage2_us  per-WFS Gamma/P/C^-1/Gamma^T kernels incl. the RHS
 *   stage3_us  P^T / W / alpha D kernels incl. the RHS
 *   pcg_us     the PCG iterations (first W^-1 .. last W)
 *   fit_us     fitting W^-1 (with the fused last update) + fit + control
 *   total_us   the whole frame
 * rho is returned by fewha_gpu_step (rho_out). */
typedef struct {
    long long step; /* frames run by this handle (StepTelemetry::step) */
    int valid;      /* 0: telemetry off, or no frame since it was enabled */
    double stage1_us, stage2_us, stage3_us, pcg_us, fit_us, total_us;
} fewha_gpu_telemetry_t;
int fewha_gpu_enable_telemetry(fewha_gpu_t h, int on);
int fewha_gpu_last_telemetry(fewha_gpu_t h, fewha_gpu_telemetry_t* out);
/* Per-launch device times (ms) and kernel kinds (as fewha_gpu_profile_step) of
 * the last graph frame, from the same event nodes.  Returns the launch count
 * (0: telemetry off or no frame since), < 0 on error. */
int fewha_gpu_last_launch_times(fewha_gpu_t h, float* ms, int* kinds, int max);

/* --- closed-loop simulation harness on the device -----------
 * The reference's simulation layer (simulation.hpp) restated in CUDA, so long
 * closed loops run with no per-frame host transfer: GaussianStream (mt19937_64 +
 * Box-Muller, :40-58, one warp per stream), generate_atmosphere (:76-127, inverse
 * 2-D DFT on the device), truth_at_step (:131-158), synthesize_measurements
 * (:164-212: the device forward model + the noise stream), evaluate_quality
 * (:228-305).  Quality records: [0] field_rms, [1] layer_rel_err (NaN without an
 * L = M pairing), [2..] rms_per_dir; their length is fewha_gpu_sim_quality_size. */
int fewha_gpu_sim_quality_size(fewha_gpu_t h);
/* GaussianStream(seed): `count` (even) standard normals drawn on `device` (no handle;
 * errors via fewha_gpu_create_error) */
int fewha_gpu_sim_gauss(int device, unsigned long long seed, int count, double* out);
/* truth_at_step(generate_atmosphere(g, seed), g, step) -> layers [n] (nodal) */
int fewha_gpu_sim_atmosphere(fewha_gpu_t h, unsigned long long seed, int step, double* layers);
/* synthesize_measurements(layers, a or none, g, noise_seed) -> meas [S] */
int fewha_gpu_sim_synthesize(fewha_gpu_t h, const double* layers, const double* a, unsigned long long noise_seed,
                             double* meas);
/* evaluate_quality(layers, a, g) -> rec [fewha_gpu_sim_quality_size] */
int fewha_gpu_sim_quality(fewha_gpu_t h, const double* layers, const double* a, double* rec);
/* run_closed_loop(g, n_steps, {atmosphere_seed, noise_seed}) (simulation.hpp:321-345) on
 * this handle (batch 1; its state is reset first, as a fresh Reconstructor): rec
 * [n_steps][quality size], rho [n_steps][iters] (may be NULL), unc_final {uncorrected
 * field RMS of the last step's truth, final field RMS} (may be NULL). */
int fewha_gpu_run_closed_loop(fewha_gpu_t h, int n_steps, unsigned long long atmosphere_seed,
                              unsigned long long noise_seed, double* rec, double* rho, double* unc_final);

/* --- per-WFS sharding (the north star's multi-GPU split) -------
 * Shard `rank` of `world` owns a contiguous WFS range, balanced by wavefront
 * nodes: its WFS kernels (Gamma, C^-1, P) run only those WFS and its adjoint
 * gather sums only their P^T psi.  The partial layer sums are all-reduced after
 * the RHS and after every apply_M (iters+1 exchanges per frame); everything else
 * (W, W^-1, alpha D, Jacobi, dots, updates, fit) is replicated and stays bitwise
 * identical on every shard.  Not in the reference (its solver is single-node,
 * SPEC.md:381); it replaces the per-WFS loop inside apply_M (reconstructor.hpp:
 * 180-195) and build_rhs (:222-240) across processes. */
/* host only: the WFS range [begin, end) of shard rank/world of a preset */
int fewha_gpu_shard_range(const char* preset_json_path, int rank, int world, int* wfs_begin, int* wfs_end);
/* a fresh 128-byte ncclUniqueId (rank 0 creates it and broadcasts it) */
int fewha_gpu_nccl_unique_id(unsigned char* id);
/* Make h shard rank/world.  nccl_id (128 bytes): join a multi-process NCCL
 * exchange (one process per GPU; the frame graph captures ncclAllReduce).
 * nccl_id NULL and world > 1: member of an in-process group, stepped only by
 * fewha_gpu_group_step_device.  world 1 with an id runs the NCCL path alone. */
int fewha_gpu_shard(fewha_gpu_t h, int rank, int world, const unsigned char* nccl_id);
int fewha_gpu_shard_wfs(fewha_gpu_t h, int* wfs_begin, int* wfs_end);
/* One frame of an in-process group (members[r] = shard r, each with its own
 * slopes slot and stream): segments in lockstep, each exchange a fixed
 * rank-order sum of the members' partial layer sums read directly from their
 * buffers (peer loads across devices).  Asynchronous; fewha_gpu_sync each. */
int fewha_gpu_group_step_device(fewha_gpu_t* members, int world);

#ifdef __cplusplus
}
#endif
#endif
