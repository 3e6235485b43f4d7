/* oracle/fewha_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C CPU restatement of the FEWHA reference hot path
 * (Reconstructor::step, proj/include/fewha/reconstructor.hpp:310-355) used as
 * the parity oracle for the CUDA path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it.  Scalar, single-threaded, fp64,
 * same operand order as the reference wherever the reference fixes one.
 *
 * Pinned against the reference itself: tests/test_oracle.py compares every
 * entry point with oracle/_ref/libfewha_ref.so (the unmodified reference built
 * by oracle/Makefile) and with the committed fixtures in tests/golden/.
 */
#ifndef FEWHA_ORACLE_H
#define FEWHA_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirror of SystemGeometry (geometry.hpp:145-183) as flat arrays.  The
 * Python side (oracle/oracle.py) fills it from the same JSON preset. */
typedef struct {
    double diameter, obstruction_fraction, illumination_threshold;
    int obstruction_is_area; /* 1 = "area", 0 = "diameter" */
    int n_wfs;
    const int* n_subap;
    const double* noise_variance;
    const int* star_is_lgs;
    const double* theta_x;
    const double* theta_y;
    const double* star_height; /* LGS height, ignored for NGS */
    int n_layers;
    const double* layer_height;
    const int* layer_order;
    const double* layer_extent; /* <= 0: derive (geometry.hpp:269-275) */
    const double* layer_strength;
    int n_dms;
    const int* n_act;
    const double* dm_height;
    int pcg_max_iter;
    double pcg_tolerance, alpha;
    int wavelet_order;
    double outer_scale, spectral_exponent;
    int precond_mode; /* 0 exact, 1 approximate, 2 balanced */
    double precond_coarse_weight, precond_balance_exponent;
    long long dense_size_cap;
    int fault_sh_adjoint;
    int loop_closed;
    double gain;
    /* L != M extension (not in the reference; "fitting": "projection"): per DM a
     * science direction, a layer-group bitmask (0 = default nearest-height
     * grouping) and an extent (<= 0 = derived).  The DM shape is
     * sum_{l in group} bilinear(phi_l; x + theta*h_l), x on the actuator grid,
     * built from the reference's bilinear_sample (operators.hpp:123-127). */
    int projection;
    const double* dm_theta_x;
    const double* dm_theta_y;
    const int* dm_layer_mask;
    const double* dm_extent_in;
} orc_config;

typedef struct orc orc_t;

/* returns NULL on error; err receives the message; *code = 2 config, 1 runtime */
orc_t* orc_create(const orc_config* cfg, char* err, int errlen, int* code);
void orc_destroy(orc_t* h);
const char* orc_last_error(const orc_t* h);

/* dims: n_coeff, n_meas, n_act_total, L, W, M, iters, n_wavefront_total */
void orc_dims(const orc_t* h, long long* d);
void orc_geometry(const orc_t* h, double* layer_extent, double* dm_extent, unsigned char* masks);

int orc_wavelet_grid(int order, int n, int dir, double* data); /* dir 0 forward, 1 inverse */
int orc_wavelet(orc_t* h, int dir, double* data);
int orc_propagate(orc_t* h, const double* layers, double* wf);
int orc_propagate_transpose(orc_t* h, const double* wf, double* layers);
int orc_sh(orc_t* h, const double* wf, double* meas);
int orc_sh_transpose(orc_t* h, const double* meas, double* wf);
int orc_apply_M(orc_t* h, const double* in, double* out);
int orc_build_rhs(orc_t* h, const double* meas, double* b);
int orc_add_dm_slopes(orc_t* h, const double* a, double* meas);
int orc_fit(orc_t* h, const double* c, double* a);

int orc_build_preconditioner(orc_t* h);
void orc_preconditioner(const orc_t* h, double* out);

int orc_step(orc_t* h, const double* meas, double* c_out, double* dm_out, double* rho_out, int* n_rho);
void orc_reset(orc_t* h);
void orc_get_state(const orc_t* h, double* c, double* b, double* r, double* p, double* q, double* sc,
                   double* a_prev2, double* a_prev);
void orc_set_state(orc_t* h, const double* c, const double* b, const double* r, const double* p,
                   const double* q, const double* sc, const double* a_prev2, const double* a_prev);

/* Stand-alone fused PCG on a caller operator (pcg.hpp:51-108), for stub tests. */
typedef void (*orc_apply_fn)(void* ctx, const double* in, double* out);
int orc_pcg(orc_apply_fn fn, void* ctx, size_t n, const double* jacobi, double* c, double* r, double* p,
            double* q, double* scalars /* rho_old, alpha, fresh */, int max_iter, double rel_tol,
            double* rho_log, int* n_log, char* err, int errlen);

#ifdef __cplusplus
}
#endif
#endif
