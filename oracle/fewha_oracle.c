/* oracle/fewha_oracle.c -- TEST INFRASTRUCTURE ONLY (see fewha_oracle.h).
 *
 * Scalar fp64 restatement of the reference reconstructor.  Every function
 * cites the reference line range it restates (paths relative to
 * /root/reference/proj/include/fewha/).  It never calls the product library
 * and the product never calls it.
 */
#include "fewha_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "daubechies_table.h"

#define PI 3.14159265358979323846

struct orc {
    orc_config cfg; /* pointers below are owned copies */
    int *n_subap, *star_is_lgs, *layer_order, *n_act;
    double *noise_variance, *theta_x, *theta_y, *star_height, *layer_height, *layer_extent, *layer_strength,
        *dm_height, *dm_extent;
    unsigned char* masks; /* concatenated n_s^2 per WFS */
    int* dm_group;        /* projection fitting: layer bitmask per DM */
    double *dm_tx, *dm_ty;
    size_t *mask_off, *meas_off, *wf_off, *coeff_off, *act_off;
    int* side;
    size_t n, S, Nw, A;
    double lo[20], hi[20];
    int flen;
    double* reg; /* [L][J+1] regularizer d_{l,j} */
    int reg_stride;
    double* precond;
    double sh_fault;
    /* state (reconstructor.hpp:61-92) */
    double *c, *b, *r, *p, *q, *a_prev2, *a_prev;
    double rho_old, alpha_c;
    int fresh;
    /* scratch */
    double *layer_work, *wf_work, *meas_work, *b1, *z, *s, *tmp;
    char err[512];
};

static void set_err(orc_t* h, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(h->err, sizeof h->err, fmt, ap);
    va_end(ap);
}

const char* orc_last_error(const orc_t* h) { return h->err; }

/* ---- grid.hpp:61-71 Kahan dot ------------------------------------------ */
static double kdot(const double* a, const double* b, size_t n) {
    double sum = 0.0, comp = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double term = a[i] * b[i] - comp;
        const double next = sum + term;
        comp = (next - sum) - term;
        sum = next;
    }
    return sum;
}

/* ---- wavelet.hpp:100-201 periodic Mallat DWT ---------------------------- */
static void set_filters(double* lo, double* hi, int* flen, int order) {
    const int off = kDaubechiesOffset[order - 1], len = kDaubechiesOffset[order] - off;
    for (int k = 0; k < len; ++k) lo[k] = kDaubechies[off + k];
    for (int k = 0; k < len; ++k) hi[k] = (k % 2 == 0 ? 1.0 : -1.0) * lo[len - 1 - k]; /* :104-106 */
    *flen = len;
}

/* analysis over a strided line x[0], x[st], ... (m entries); :153-168 */
static void analysis(double* x, int st, int m, const double* lo, const double* hi, int flen, double* tmp) {
    const int half = m / 2, mask = m - 1;
    for (int i = 0; i < half; ++i) {
        double a = 0.0, d = 0.0;
        for (int k = 0; k < flen; ++k) {
            const double v = x[(size_t)((2 * i + k) & mask) * st];
            a += lo[k] * v;
            d += hi[k] * v;
        }
        tmp[i] = a;
        tmp[half + i] = d;
    }
    for (int i = 0; i < m; ++i) x[(size_t)i * st] = tmp[i];
}

/* synthesis; :170-181 */
static void synthesis(double* x, int st, int m, const double* lo, const double* hi, int flen, double* tmp) {
    const int half = m / 2, mask = m - 1;
    for (int i = 0; i < m; ++i) tmp[i] = 0.0;
    for (int i = 0; i < half; ++i) {
        const double a = x[(size_t)i * st], d = x[(size_t)(half + i) * st];
        for (int k = 0; k < flen; ++k) tmp[(2 * i + k) & mask] += a * lo[k] + d * hi[k];
    }
    for (int i = 0; i < m; ++i) x[(size_t)i * st] = tmp[i];
}

/* forward: per level rows then columns (:115-125); the reference's
 * transpose + row pass reads the same operands in the same order as a
 * strided column pass, so results are identical. */
static void dwt_forward(double* g, int n, const double* lo, const double* hi, int flen, double* tmp) {
    for (int s = n; s >= 2; s /= 2) {
        for (int i = 0; i < s; ++i) analysis(g + (size_t)i * n, 1, s, lo, hi, flen, tmp);
        for (int j = 0; j < s; ++j) analysis(g + j, n, s, lo, hi, flen, tmp);
    }
}

/* inverse: per level columns then rows (:128-138) */
static void dwt_inverse(double* g, int n, const double* lo, const double* hi, int flen, double* tmp) {
    for (int s = 2; s <= n; s *= 2) {
        for (int j = 0; j < s; ++j) synthesis(g + j, n, s, lo, hi, flen, tmp);
        for (int i = 0; i < s; ++i) synthesis(g + (size_t)i * n, 1, s, lo, hi, flen, tmp);
    }
}

int orc_wavelet_grid(int order, int n, int dir, double* data) {
    if (order < 1 || order > 10 || n < 1 || (n & (n - 1))) return 2;
    double lo[20], hi[20], *tmp = malloc(sizeof(double) * (size_t)n);
    int flen;
    set_filters(lo, hi, &flen, order);
    if (dir) dwt_inverse(data, n, lo, hi, flen, tmp);
    else dwt_forward(data, n, lo, hi, flen, tmp);
    free(tmp);
    return 0;
}

static int bit_width(unsigned m) {
    int b = 0;
    while (m) {
        ++b;
        m >>= 1;
    }
    return b;
}

/* ---- geometry.hpp:189-251 masks via adaptive Simpson --------------------- */
typedef struct {
    double y0, y1, r_out, r_in;
} chord_ctx;

static double overlap(const chord_ctx* c, double half) {
    if (half <= 0.0) return 0.0;
    const double hi = c->y1 < half ? c->y1 : half;
    const double lo = c->y0 > -half ? c->y0 : -half;
    const double v = hi - lo;
    return v > 0.0 ? v : 0.0;
}

static double clipped_chord(const chord_ctx* c, double x) {
    const double c_out = c->r_out * c->r_out > x * x ? sqrt(c->r_out * c->r_out - x * x) : 0.0;
    const double c_in = c->r_in * c->r_in > x * x ? sqrt(c->r_in * c->r_in - x * x) : 0.0;
    return overlap(c, c_out) - overlap(c, c_in);
}

static double asimpson(const chord_ctx* c, double a, double b, double fa, double fm, double fb, double whole,
                       double tol, int depth) {
    const double m = 0.5 * (a + b);
    const double lm = 0.5 * (a + m), rm = 0.5 * (m + b);
    const double flm = clipped_chord(c, lm), frm = clipped_chord(c, rm);
    const double left = (m - a) / 6.0 * (fa + 4.0 * flm + fm);
    const double right = (b - m) / 6.0 * (fm + 4.0 * frm + fb);
    if (depth <= 0 || fabs(left + right - whole) <= 15.0 * tol) return left + right + (left + right - whole) / 15.0;
    return asimpson(c, a, m, fa, flm, fm, left, 0.5 * tol, depth - 1) +
           asimpson(c, m, b, fm, frm, fb, right, 0.5 * tol, depth - 1);
}

static double fill_fraction(const orc_t* h, int w, int i, int j) {
    const double D = h->cfg.diameter;
    const double d = D / h->n_subap[w];
    const double x0 = -D / 2.0 + j * d;
    const double y0 = -D / 2.0 + i * d;
    chord_ctx c;
    c.y0 = y0;
    c.y1 = y0 + d;
    c.r_out = D / 2.0;
    const double f = h->cfg.obstruction_is_area ? sqrt(h->cfg.obstruction_fraction) : h->cfg.obstruction_fraction;
    c.r_in = f * D / 2.0;
    const double a = x0, b = x0 + d, tol = 1e-12 * d * d;
    const double fa = clipped_chord(&c, a), fb = clipped_chord(&c, b), fm = clipped_chord(&c, 0.5 * (a + b));
    const double whole = (b - a) / 6.0 * (fa + 4.0 * fm + fb);
    const double area = asimpson(&c, a, b, fa, fm, fb, whole, tol, 40);
    return area / (d * d);
}

/* geometry.hpp:74-76 */
static double footprint(const orc_t* h, int w, double layer_h) {
    return h->star_is_lgs[w] ? 1.0 - layer_h / h->star_height[w] : 1.0;
}

/* geometry.hpp:256-275 */
static double layer_extent_derived(const orc_t* h, int l) {
    double side = 0.0;
    for (int w = 0; w < h->cfg.n_wfs; ++w) {
        const double s = footprint(h, w, h->layer_height[l]) * h->cfg.diameter +
                         2.0 * hypot(h->theta_x[w], h->theta_y[w]) * h->layer_height[l];
        if (s > side) side = s;
    }
    const int nn = 1 << h->layer_order[l];
    return side + 2.0 * side / (nn - 1);
}

/* ---- operators.hpp:108-135 bilinear stencil / sample / scatter ---------- */
static int stencil(orc_t* h, int n, double extent, double px, double py, int* i0o, int* j0o, double* w) {
    const double spacing = extent / (n - 1);
    const double u = (px + extent / 2.0) / spacing;
    const double t = (py + extent / 2.0) / spacing;
    const double eps = 1e-9;
    if (u < -eps || u > n - 1 + eps || t < -eps || t > n - 1 + eps) {
        set_err(h, "propagation: evaluation point outside layer grid");
        return 1;
    }
    int j0 = (int)floor(u), i0 = (int)floor(t);
    if (j0 > n - 2) j0 = n - 2;
    if (i0 > n - 2) i0 = n - 2;
    const double fx = u - j0, fy = t - i0;
    *i0o = i0 > 0 ? i0 : 0;
    *j0o = j0 > 0 ? j0 : 0;
    w[0] = (1 - fy) * (1 - fx);
    w[1] = (1 - fy) * fx;
    w[2] = fy * (1 - fx);
    w[3] = fy * fx;
    return 0;
}

static int sample(orc_t* h, const double* v, int n, double extent, double px, double py, double* out) {
    int i0, j0;
    double w[4];
    if (stencil(h, n, extent, px, py, &i0, &j0, w)) return 1;
    const double* r0 = v + (size_t)i0 * n;
    const double* r1 = r0 + n;
    *out = w[0] * r0[j0] + w[1] * r0[j0 + 1] + w[2] * r1[j0] + w[3] * r1[j0 + 1];
    return 0;
}

static int scatter(orc_t* h, double* v, int n, double extent, double px, double py, double val) {
    int i0, j0;
    double w[4];
    if (stencil(h, n, extent, px, py, &i0, &j0, w)) return 1;
    double* r0 = v + (size_t)i0 * n;
    double* r1 = r0 + n;
    r0[j0] += val * w[0];
    r0[j0 + 1] += val * w[1];
    r1[j0] += val * w[2];
    r1[j0 + 1] += val * w[3];
    return 0;
}

/* ---- operators.hpp:145-188 Shack-Hartmann ------------------------------- */
static void sh_apply(const orc_t* h, int w, const double* phi, double* sx, double* sy) {
    const int n = h->n_subap[w], np = n + 1;
    const unsigned char* mask = h->masks + h->mask_off[w];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const size_t k = (size_t)i * n + j;
            if (!mask[k]) {
                sx[k] = 0.0;
                sy[k] = 0.0;
                continue;
            }
            const double p00 = phi[(size_t)i * np + j], p01 = phi[(size_t)i * np + j + 1];
            const double p10 = phi[(size_t)(i + 1) * np + j], p11 = phi[(size_t)(i + 1) * np + j + 1];
            sx[k] = 0.5 * ((p01 - p00) + (p11 - p10));
            sy[k] = 0.5 * ((p10 - p00) + (p11 - p01));
        }
}

static void sh_transpose_apply(const orc_t* h, int w, const double* sx, const double* sy, double* phi) {
    const int n = h->n_subap[w], np = n + 1;
    const unsigned char* mask = h->masks + h->mask_off[w];
    memset(phi, 0, sizeof(double) * (size_t)np * np);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const size_t k = (size_t)i * n + j;
            if (!mask[k]) continue;
            const double x = 0.5 * sx[k], y = 0.5 * sy[k];
            phi[(size_t)i * np + j] += -x - y;
            phi[(size_t)i * np + j + 1] += x - y;
            phi[(size_t)(i + 1) * np + j] += -x + y;
            phi[(size_t)(i + 1) * np + j + 1] += x + y;
        }
    if (h->sh_fault != 1.0) /* reconstructor.hpp:159-160 fault fixture */
        for (size_t k = 0; k < (size_t)np * np; ++k) phi[k] *= h->sh_fault;
}

/* ---- operators.hpp:204-260 propagation ------------------------------------ */
/* screens: L layers (ext, height, side) or M DMs */
static int propagate_wfs(orc_t* h, int w, const double* const* screens, const int* sides, const double* extents,
                         const double* heights, int n_screens, double* phi) {
    const int np = h->n_subap[w] + 1;
    const double D = h->cfg.diameter, d = D / (np - 1);
    for (int i = 0; i < np; ++i) {
        const double y = -D / 2.0 + i * d;
        for (int j = 0; j < np; ++j) {
            const double x = -D / 2.0 + j * d;
            double acc = 0.0;
            for (int s = 0; s < n_screens; ++s) {
                const double c = footprint(h, w, heights[s]);
                double v;
                if (sample(h, screens[s], sides[s], extents[s], c * x + h->theta_x[w] * heights[s],
                           c * y + h->theta_y[w] * heights[s], &v))
                    return 1;
                acc += v;
            }
            phi[(size_t)i * np + j] = acc;
        }
    }
    return 0;
}

static int propagate_transpose_layer(orc_t* h, const double* phi, int w, int l, double* acc) {
    const int np = h->n_subap[w] + 1, n = h->side[l];
    const double D = h->cfg.diameter, d = D / (np - 1);
    const double hl = h->layer_height[l], c = footprint(h, w, hl);
    for (int i = 0; i < np; ++i) {
        const double y = -D / 2.0 + i * d;
        for (int j = 0; j < np; ++j) {
            const double x = -D / 2.0 + j * d;
            if (scatter(h, acc, n, h->layer_extent[l], c * x + h->theta_x[w] * hl, c * y + h->theta_y[w] * hl,
                        phi[(size_t)i * np + j]))
                return 1;
        }
    }
    return 0;
}

static int layer_screens(orc_t* h, const double* layers, const double** scr) {
    for (int l = 0; l < h->cfg.n_layers; ++l) scr[l] = layers + h->coeff_off[l];
    return 0;
}

int orc_propagate(orc_t* h, const double* layers, double* wf) {
    const double* scr[64];
    layer_screens(h, layers, scr);
    for (int w = 0; w < h->cfg.n_wfs; ++w)
        if (propagate_wfs(h, w, scr, h->side, h->layer_extent, h->layer_height, h->cfg.n_layers, wf + h->wf_off[w]))
            return 1;
    return 0;
}

int orc_propagate_transpose(orc_t* h, const double* wf, double* layers) {
    for (int l = 0; l < h->cfg.n_layers; ++l) {
        double* acc = layers + h->coeff_off[l];
        memset(acc, 0, sizeof(double) * (size_t)h->side[l] * h->side[l]);
        for (int w = 0; w < h->cfg.n_wfs; ++w)
            if (propagate_transpose_layer(h, wf + h->wf_off[w], w, l, acc)) return 1;
    }
    return 0;
}

int orc_sh(orc_t* h, const double* wf, double* meas) {
    for (int w = 0; w < h->cfg.n_wfs; ++w) {
        const size_t n2 = (size_t)h->n_subap[w] * h->n_subap[w];
        sh_apply(h, w, wf + h->wf_off[w], meas + h->meas_off[w], meas + h->meas_off[w] + n2);
    }
    return 0;
}

int orc_sh_transpose(orc_t* h, const double* meas, double* wf) {
    for (int w = 0; w < h->cfg.n_wfs; ++w) {
        const size_t n2 = (size_t)h->n_subap[w] * h->n_subap[w];
        sh_transpose_apply(h, w, meas + h->meas_off[w], meas + h->meas_off[w] + n2, wf + h->wf_off[w]);
    }
    return 0;
}

int orc_wavelet(orc_t* h, int dir, double* data) {
    for (int l = 0; l < h->cfg.n_layers; ++l) {
        if (dir) dwt_inverse(data + h->coeff_off[l], h->side[l], h->lo, h->hi, h->flen, h->tmp);
        else dwt_forward(data + h->coeff_off[l], h->side[l], h->lo, h->hi, h->flen, h->tmp);
    }
    return 0;
}

/* ---- reconstructor.hpp:166-212 apply_M ------------------------------------ */
int orc_apply_M(orc_t* h, const double* in, double* out) {
    const int L = h->cfg.n_layers, W = h->cfg.n_wfs;
    /* stage 1 */
    memcpy(h->layer_work, in, sizeof(double) * h->n);
    orc_wavelet(h, 1, h->layer_work);
    /* stage 2 */
    const double* scr[64];
    layer_screens(h, h->layer_work, scr);
    for (int w = 0; w < W; ++w) {
        const size_t n2 = (size_t)h->n_subap[w] * h->n_subap[w];
        double* wf = h->wf_work + h->wf_off[w];
        double* sl = h->meas_work + h->meas_off[w];
        if (propagate_wfs(h, w, scr, h->side, h->layer_extent, h->layer_height, L, wf)) return 1;
        sh_apply(h, w, wf, sl, sl + n2);
        const double iv = 1.0 / h->noise_variance[w]; /* operators.hpp:280 */
        for (size_t k = 0; k < 2 * n2; ++k) sl[k] *= iv;
        sh_transpose_apply(h, w, sl, sl + n2, wf);
    }
    /* stage 3 */
    for (int l = 0; l < L; ++l) {
        double* acc = h->layer_work + h->coeff_off[l];
        const int side = h->side[l];
        memset(acc, 0, sizeof(double) * (size_t)side * side);
        for (int w = 0; w < W; ++w)
            if (propagate_transpose_layer(h, h->wf_work + h->wf_off[w], w, l, acc)) return 1;
        dwt_forward(acc, side, h->lo, h->hi, h->flen, h->tmp);
        double* o = out + h->coeff_off[l];
        const double* ci = in + h->coeff_off[l];
        memcpy(o, acc, sizeof(double) * (size_t)side * side);
        /* operators.hpp:324-332 */
        for (int i = 0; i < side; ++i)
            for (int j = 0; j < side; ++j) {
                const size_t k = (size_t)i * side + j;
                o[k] += h->cfg.alpha * h->reg[l * h->reg_stride + bit_width((unsigned)(i > j ? i : j))] * ci[k];
            }
    }
    return 0;
}

/* ---- reconstructor.hpp:215-247 build_rhs ---------------------------------- */
int orc_build_rhs(orc_t* h, const double* meas, double* bout) {
    const int L = h->cfg.n_layers, W = h->cfg.n_wfs;
    for (int w = 0; w < W; ++w) {
        const size_t n2 = (size_t)h->n_subap[w] * h->n_subap[w];
        double* sl = h->meas_work + h->meas_off[w];
        const double iv = 1.0 / h->noise_variance[w];
        for (size_t k = 0; k < 2 * n2; ++k) sl[k] = meas[h->meas_off[w] + k] * iv;
        sh_transpose_apply(h, w, sl, sl + n2, h->wf_work + h->wf_off[w]);
    }
    for (int l = 0; l < L; ++l) {
        double* acc = bout + h->coeff_off[l];
        memset(acc, 0, sizeof(double) * (size_t)h->side[l] * h->side[l]);
        for (int w = 0; w < W; ++w)
            if (propagate_transpose_layer(h, h->wf_work + h->wf_off[w], w, l, acc)) return 1;
        dwt_forward(acc, h->side[l], h->lo, h->hi, h->flen, h->tmp);
    }
    return 0;
}

/* ---- reconstructor.hpp:259-280 add_dm_slopes (+ dm_screens :357-364) ------ */
int orc_add_dm_slopes(orc_t* h, const double* a, double* meas) {
    const int M = h->cfg.n_dms;
    const double* scr[64];
    for (int m = 0; m < M; ++m) scr[m] = a + h->act_off[m];
    double* wf = h->wf_work;
    for (int w = 0; w < h->cfg.n_wfs; ++w) {
        const size_t n2 = (size_t)h->n_subap[w] * h->n_subap[w];
        double* sl = h->meas_work + h->meas_off[w];
        if (propagate_wfs(h, w, scr, h->n_act, h->dm_extent, h->dm_height, M, wf + h->wf_off[w])) return 1;
        sh_apply(h, w, wf + h->wf_off[w], sl, sl + n2);
        for (size_t k = 0; k < 2 * n2; ++k) meas[h->meas_off[w] + k] += sl[k];
    }
    return 0;
}

/* ---- reconstructor.hpp:284-305 fit_to_mirrors ----------------------------- */
int orc_fit(orc_t* h, const double* c, double* a) {
    if (h->cfg.projection) { /* L != M extension */
        memcpy(h->layer_work, c, sizeof(double) * h->n);
        orc_wavelet(h, 1, h->layer_work);
        for (int m = 0; m < h->cfg.n_dms; ++m) {
            const int na = h->n_act[m];
            const double e = h->dm_extent[m], da = e / (na - 1);
            double* out = a + h->act_off[m];
            for (int i = 0; i < na; ++i)
                for (int j = 0; j < na; ++j) {
                    const double px = -e / 2.0 + j * da, py = -e / 2.0 + i * da;
                    double acc = 0.0;
                    for (int l = 0; l < h->cfg.n_layers; ++l) {
                        if (!(h->dm_group[m] >> l & 1)) continue;
                        { /* projected point off this layer's grid: zero contribution */
                            const double ex = h->layer_extent[l], sp = ex / (h->side[l] - 1);
                            const double u = (px + h->dm_tx[m] * h->layer_height[l] + ex / 2.0) / sp;
                            const double t = (py + h->dm_ty[m] * h->layer_height[l] + ex / 2.0) / sp;
                            if (u < -1e-9 || u > h->side[l] - 1 + 1e-9 || t < -1e-9 || t > h->side[l] - 1 + 1e-9) continue;
                        }
                        double v;
                        if (sample(h, h->layer_work + h->coeff_off[l], h->side[l], h->layer_extent[l],
                                   px + h->dm_tx[m] * h->layer_height[l], py + h->dm_ty[m] * h->layer_height[l], &v))
                            return 1;
                        acc += v;
                    }
                    out[(size_t)i * na + j] = acc;
                }
        }
        return 0;
    }
    for (int l = 0; l < h->cfg.n_layers; ++l) {
        const int side = h->side[l];
        double* grid = h->layer_work + h->coeff_off[l];
        memcpy(grid, c + h->coeff_off[l], sizeof(double) * (size_t)side * side);
        dwt_inverse(grid, side, h->lo, h->hi, h->flen, h->tmp);
        const int na = h->n_act[l];
        double* out = a + h->act_off[l];
        if (na == side) {
            memcpy(out, grid, sizeof(double) * (size_t)side * side);
            continue;
        }
        const double e = h->dm_extent[l], da = e / (na - 1);
        for (int i = 0; i < na; ++i)
            for (int j = 0; j < na; ++j)
                if (sample(h, grid, side, e, -e / 2.0 + j * da, -e / 2.0 + i * da, &out[(size_t)i * na + j]))
                    return 1;
    }
    return 0;
}

/* ---- pcg.hpp:51-108 fused PCG --------------------------------------------- */
typedef struct {
    orc_t* h;
} mctx;
static void apply_m_cb(void* ctx, const double* in, double* out) { orc_apply_M(((mctx*)ctx)->h, in, out); }

int orc_pcg(orc_apply_fn fn, void* ctx, size_t n, const double* jac, double* c, double* r, double* p, double* q,
            double* sc, int max_iter, double rel_tol, double* rho_log, int* n_log, char* err, int errlen) {
    *n_log = 0;
    if (max_iter < 1) {
        snprintf(err, (size_t)errlen, "pcg_solve: max_iter must be >= 1");
        return 3;
    }
    for (size_t i = 0; i < n; ++i)
        if (!(jac[i] > 0.0)) {
            snprintf(err, (size_t)errlen, "pcg_solve: preconditioner entries must be > 0");
            return 3;
        }
    double* z = malloc(sizeof(double) * n);
    double* s = malloc(sizeof(double) * n);
    double rho_entry = -1.0;
    int rc = 0;
    for (int it = 0; it < max_iter; ++it) {
        for (size_t i = 0; i < n; ++i) z[i] = r[i] / jac[i];
        fn(ctx, z, s);
        const double rho = kdot(r, z, n), mu = kdot(s, z, n);
        if (rho_entry < 0.0) rho_entry = rho;
        if (rel_tol > 0.0 && rho <= rel_tol * rel_tol * rho_entry) {
            rho_log[(*n_log)++] = rho;
            break;
        }
        if (rho == 0.0 && mu == 0.0) {
            rho_log[(*n_log)++] = 0.0;
            continue;
        }
        double beta, alpha;
        if (sc[2] != 0.0) {
            beta = 0.0;
            alpha = rho / mu;
            sc[2] = 0.0;
        } else {
            beta = rho / sc[0];
            alpha = rho / (mu - rho * beta / sc[1]);
        }
        if (!isfinite(rho) || !isfinite(mu) || !isfinite(beta) || !isfinite(alpha)) {
            snprintf(err, (size_t)errlen, "pcg_solve: non-finite scalar (indefinite operator?)");
            rc = 1;
            break;
        }
        sc[0] = rho;
        sc[1] = alpha;
        for (size_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
        for (size_t i = 0; i < n; ++i) q[i] = s[i] + beta * q[i];
        for (size_t i = 0; i < n; ++i) c[i] += alpha * p[i];
        for (size_t i = 0; i < n; ++i) r[i] -= alpha * q[i];
        rho_log[(*n_log)++] = rho;
    }
    free(z);
    free(s);
    return rc;
}

/* ---- operators.hpp:367-425 preconditioner --------------------------------- */
int orc_build_preconditioner(orc_t* h) {
    const size_t n = h->n;
    double* e = calloc(n, sizeof(double));
    double* me = malloc(sizeof(double) * n);
    double* diag = calloc(n, sizeof(double));
    int rc = 0;
    if (h->cfg.precond_mode == 0) {
        if ((long long)n > h->cfg.dense_size_cap) {
            set_err(h, "preconditioner: exact mode needs coefficient dimension <= %lld, got %zu",
                    h->cfg.dense_size_cap, n);
            rc = 2;
            goto done;
        }
        for (size_t k = 0; k < n; ++k) {
            e[k] = 1.0;
            if (orc_apply_M(h, e, me)) {
                rc = 1;
                goto done;
            }
            e[k] = 0.0;
            diag[k] = me[k];
        }
    } else {
        for (int l = 0; l < h->cfg.n_layers; ++l) {
            const int side = h->side[l], order = h->layer_order[l];
            for (int scale = 0; scale <= order; ++scale) {
                const int block = scale == 0 ? 1 : 1 << (scale - 1);
                for (int orient = scale == 0 ? 0 : 1; orient <= (scale == 0 ? 0 : 3); ++orient) {
                    const int oi = orient >= 2 ? block : 0;
                    const int oj = (orient == 1 || orient == 3) ? block : 0;
                    const size_t rep = h->coeff_off[l] + (size_t)(oi + block / 2) * side + (oj + block / 2);
                    const double alpha_d = h->cfg.alpha * h->reg[l * h->reg_stride + scale];
                    e[rep] = 1.0;
                    if (orc_apply_M(h, e, me)) {
                        rc = 1;
                        goto done;
                    }
                    e[rep] = 0.0;
                    const double probed = me[rep];
                    double value;
                    if (h->cfg.precond_mode == 2) {
                        const double ex = h->cfg.precond_balance_exponent;
                        value = pow(probed, ex) * pow(alpha_d, 1.0 - ex);
                    } else {
                        const double t_hat = probed - alpha_d;
                        const double wgt = scale == 0 ? h->cfg.precond_coarse_weight : 1.0;
                        value = alpha_d + wgt * t_hat;
                    }
                    for (int i = oi; i < oi + block; ++i)
                        for (int j = oj; j < oj + block; ++j) diag[h->coeff_off[l] + (size_t)i * side + j] = value;
                }
            }
        }
    }
    for (size_t k = 0; k < n; ++k)
        if (!(diag[k] > 0.0)) {
            set_err(h, "preconditioner: non-positive diagonal entry (operator symmetry broken?)");
            rc = 1;
            goto done;
        }
    free(h->precond);
    h->precond = diag;
    diag = NULL;
done:
    free(e);
    free(me);
    free(diag);
    return rc;
}

void orc_preconditioner(const orc_t* h, double* out) {
    if (h->precond) memcpy(out, h->precond, sizeof(double) * h->n);
}

/* ---- reconstructor.hpp:310-355 step --------------------------------------- */
int orc_step(orc_t* h, const double* meas, double* c_out, double* dm_out, double* rho_out, int* n_rho) {
    if (!h->precond) {
        int rc = orc_build_preconditioner(h);
        if (rc) return rc;
    }
    const size_t n = h->n, A = h->A;
    double* mw = malloc(sizeof(double) * h->S);
    memcpy(mw, meas, sizeof(double) * h->S);
    if (h->cfg.loop_closed && orc_add_dm_slopes(h, h->a_prev2, mw)) {
        free(mw);
        return 1;
    }
    if (orc_build_rhs(h, mw, h->b1)) {
        free(mw);
        return 1;
    }
    free(mw);
    for (size_t k = 0; k < n; ++k) h->r[k] += h->b1[k] - h->b[k];
    double* t = h->b;
    h->b = h->b1;
    h->b1 = t;

    double sc[3] = {h->rho_old, h->alpha_c, h->fresh ? 1.0 : 0.0};
    double rho_log[1024];
    int n_log = 0;
    mctx ctx = {h};
    int iters = h->cfg.pcg_max_iter > 1024 ? 1024 : h->cfg.pcg_max_iter;
    char err[256];
    int rc = orc_pcg(apply_m_cb, &ctx, n, h->precond, h->c, h->r, h->p, h->q, sc, iters, h->cfg.pcg_tolerance,
                     rho_log, &n_log, err, sizeof err);
    if (rc) {
        set_err(h, "%s", err);
        return rc;
    }
    h->rho_old = sc[0];
    h->alpha_c = sc[1];
    h->fresh = sc[2] != 0.0;

    double* a_tilde = malloc(sizeof(double) * A);
    if (orc_fit(h, h->c, a_tilde)) {
        free(a_tilde);
        return 1;
    }
    const double g = h->cfg.gain;
    double* a_next = malloc(sizeof(double) * A);
    for (size_t k = 0; k < A; ++k)
        a_next[k] = h->cfg.loop_closed ? h->a_prev[k] + g * (a_tilde[k] - h->a_prev2[k])
                                       : (1.0 - g) * h->a_prev[k] + g * a_tilde[k];
    memcpy(h->a_prev2, h->a_prev, sizeof(double) * A);
    memcpy(h->a_prev, a_next, sizeof(double) * A);
    if (c_out) memcpy(c_out, h->c, sizeof(double) * n);
    if (dm_out) memcpy(dm_out, a_next, sizeof(double) * A);
    if (rho_out) memcpy(rho_out, rho_log, sizeof(double) * (size_t)n_log);
    if (n_rho) *n_rho = n_log;
    free(a_tilde);
    free(a_next);
    return 0;
}

void orc_reset(orc_t* h) {
    memset(h->c, 0, sizeof(double) * h->n);
    memset(h->b, 0, sizeof(double) * h->n);
    memset(h->r, 0, sizeof(double) * h->n);
    memset(h->p, 0, sizeof(double) * h->n);
    memset(h->q, 0, sizeof(double) * h->n);
    memset(h->a_prev2, 0, sizeof(double) * h->A);
    memset(h->a_prev, 0, sizeof(double) * h->A);
    h->rho_old = 0.0;
    h->alpha_c = 0.0;
    h->fresh = 1;
}

void orc_get_state(const orc_t* h, double* c, double* b, double* r, double* p, double* q, double* sc,
                   double* a_prev2, double* a_prev) {
    const size_t nb = sizeof(double) * h->n, ab = sizeof(double) * h->A;
    memcpy(c, h->c, nb);
    memcpy(b, h->b, nb);
    memcpy(r, h->r, nb);
    memcpy(p, h->p, nb);
    memcpy(q, h->q, nb);
    sc[0] = h->rho_old;
    sc[1] = h->alpha_c;
    sc[2] = h->fresh ? 1.0 : 0.0;
    memcpy(a_prev2, h->a_prev2, ab);
    memcpy(a_prev, h->a_prev, ab);
}

void orc_set_state(orc_t* h, const double* c, const double* b, const double* r, const double* p, const double* q,
                   const double* sc, const double* a_prev2, const double* a_prev) {
    const size_t nb = sizeof(double) * h->n, ab = sizeof(double) * h->A;
    memcpy(h->c, c, nb);
    memcpy(h->b, b, nb);
    memcpy(h->r, r, nb);
    memcpy(h->p, p, nb);
    memcpy(h->q, q, nb);
    h->rho_old = sc[0];
    h->alpha_c = sc[1];
    h->fresh = sc[2] != 0.0;
    memcpy(h->a_prev2, a_prev2, ab);
    memcpy(h->a_prev, a_prev, ab);
}

/* ---- construction: finalize_geometry (geometry.hpp:366-377), validation subset,
 *      regularizer_build (operators.hpp:307-321) ------------------------------ */
#define DUPI(dst, src, cnt)                                                     \
    do {                                                                        \
        (dst) = malloc(sizeof(int) * (size_t)((cnt) > 0 ? (cnt) : 1));          \
        if ((cnt) > 0) memcpy((dst), (src), sizeof(int) * (size_t)(cnt));       \
    } while (0)
#define DUPD(dst, src, cnt)                                                     \
    do {                                                                        \
        (dst) = malloc(sizeof(double) * (size_t)((cnt) > 0 ? (cnt) : 1));       \
        if ((cnt) > 0) memcpy((dst), (src), sizeof(double) * (size_t)(cnt));    \
    } while (0)

orc_t* orc_create(const orc_config* cfg, char* err, int errlen, int* code) {
    *code = 0;
    if (cfg->n_wfs < 1 || cfg->n_layers < 1 || cfg->n_layers > 64 || cfg->n_dms > 64) {
        snprintf(err, (size_t)errlen, "invalid geometry: empty or oversized wfs/layer/dm list");
        *code = 2;
        return NULL;
    }
    if (!cfg->projection && cfg->n_dms != cfg->n_layers) { /* geometry.hpp:294-296 */
        snprintf(err, (size_t)errlen,
                 "invalid geometry: dm count %d != layer count %d (only the L = M identity-fitting mode is supported)",
                 cfg->n_dms, cfg->n_layers);
        *code = 2;
        return NULL;
    }
    if (cfg->wavelet_order < 1 || cfg->wavelet_order > 10) {
        snprintf(err, (size_t)errlen, "invalid geometry: wavelet order out of 1..10");
        *code = 2;
        return NULL;
    }
    orc_t* h = calloc(1, sizeof(orc_t));
    h->cfg = *cfg;
    const int W = cfg->n_wfs, L = cfg->n_layers, M = cfg->n_dms;
    DUPI(h->n_subap, cfg->n_subap, W);
    DUPI(h->star_is_lgs, cfg->star_is_lgs, W);
    DUPI(h->layer_order, cfg->layer_order, L);
    DUPI(h->n_act, cfg->n_act, M);
    DUPD(h->noise_variance, cfg->noise_variance, W);
    DUPD(h->theta_x, cfg->theta_x, W);
    DUPD(h->theta_y, cfg->theta_y, W);
    DUPD(h->star_height, cfg->star_height, W);
    DUPD(h->layer_height, cfg->layer_height, L);
    DUPD(h->layer_extent, cfg->layer_extent, L);
    DUPD(h->layer_strength, cfg->layer_strength, L);
    DUPD(h->dm_height, cfg->dm_height, M);
    h->dm_extent = malloc(sizeof(double) * (size_t)M);

    for (int l = 0; l < L; ++l)
        if (h->layer_extent[l] <= 0.0) h->layer_extent[l] = layer_extent_derived(h, l);
    h->dm_group = calloc((size_t)(M > 0 ? M : 1), sizeof(int));
    h->dm_tx = calloc((size_t)(M > 0 ? M : 1), sizeof(double));
    h->dm_ty = calloc((size_t)(M > 0 ? M : 1), sizeof(double));
    if (!cfg->projection) {
        for (int m = 0; m < M; ++m) h->dm_extent[m] = h->layer_extent[m]; /* geometry.hpp:374 */
    } else {
        int any = 0;
        for (int m = 0; m < M; ++m) {
            h->dm_group[m] = cfg->dm_layer_mask ? cfg->dm_layer_mask[m] : 0;
            h->dm_tx[m] = cfg->dm_theta_x ? cfg->dm_theta_x[m] : 0.0;
            h->dm_ty[m] = cfg->dm_theta_y ? cfg->dm_theta_y[m] : 0.0;
            any |= h->dm_group[m];
        }
        if (!any) /* each layer to the DM of nearest conjugation height (ties: lower index) */
            for (int l = 0; l < L; ++l) {
                int best = 0;
                for (int m = 1; m < M; ++m)
                    if (fabs(h->dm_height[m] - h->layer_height[l]) < fabs(h->dm_height[best] - h->layer_height[l])) best = m;
                h->dm_group[best] |= 1 << l;
            }
        for (int m = 0; m < M; ++m) {
            if (cfg->dm_extent_in && cfg->dm_extent_in[m] > 0.0) {
                h->dm_extent[m] = cfg->dm_extent_in[m];
                continue;
            }
            /* the layer_extent rule (geometry.hpp:256-275) at the DM height, n_act nodes */
            double side = 0.0;
            for (int w = 0; w < cfg->n_wfs; ++w) {
                const double s = footprint(h, w, h->dm_height[m]) * cfg->diameter +
                                 2.0 * hypot(h->theta_x[w], h->theta_y[w]) * h->dm_height[m];
                if (s > side) side = s;
            }
            h->dm_extent[m] = side + 2.0 * side / (h->n_act[m] - 1);
        }
    }

    h->mask_off = malloc(sizeof(size_t) * (size_t)(W + 1));
    h->meas_off = malloc(sizeof(size_t) * (size_t)(W + 1));
    h->wf_off = malloc(sizeof(size_t) * (size_t)(W + 1));
    h->mask_off[0] = h->meas_off[0] = h->wf_off[0] = 0;
    for (int w = 0; w < W; ++w) {
        const size_t ns = (size_t)h->n_subap[w];
        h->mask_off[w + 1] = h->mask_off[w] + ns * ns;
        h->meas_off[w + 1] = h->meas_off[w] + 2 * ns * ns;
        h->wf_off[w + 1] = h->wf_off[w] + (ns + 1) * (ns + 1);
    }
    h->S = h->meas_off[W];
    h->Nw = h->wf_off[W];
    h->masks = malloc(h->mask_off[W] ? h->mask_off[W] : 1);
    for (int w = 0; w < W; ++w) {
        const int ns = h->n_subap[w];
        for (int i = 0; i < ns; ++i)
            for (int j = 0; j < ns; ++j)
                h->masks[h->mask_off[w] + (size_t)i * ns + j] =
                    fill_fraction(h, w, i, j) >= cfg->illumination_threshold ? 1 : 0;
    }
    h->coeff_off = malloc(sizeof(size_t) * (size_t)(L + 1));
    h->side = malloc(sizeof(int) * (size_t)L);
    h->coeff_off[0] = 0;
    int maxJ = 0;
    for (int l = 0; l < L; ++l) {
        h->side[l] = 1 << h->layer_order[l];
        h->coeff_off[l + 1] = h->coeff_off[l] + (size_t)h->side[l] * h->side[l];
        if (h->layer_order[l] > maxJ) maxJ = h->layer_order[l];
    }
    h->n = h->coeff_off[L];
    h->act_off = malloc(sizeof(size_t) * (size_t)(M + 1));
    h->act_off[0] = 0;
    for (int m = 0; m < M; ++m) h->act_off[m + 1] = h->act_off[m] + (size_t)h->n_act[m] * h->n_act[m];
    h->A = h->act_off[M];

    set_filters(h->lo, h->hi, &h->flen, cfg->wavelet_order);
    h->reg_stride = maxJ + 1;
    h->reg = malloc(sizeof(double) * (size_t)(L * h->reg_stride));
    const double kappa0 = 2.0 * PI / cfg->outer_scale;
    for (int l = 0; l < L; ++l)
        for (int j = 0; j <= h->layer_order[l]; ++j) {
            const double kappa = ldexp(2.0 * PI / h->layer_extent[l], j);
            h->reg[l * h->reg_stride + j] =
                pow(kappa * kappa + kappa0 * kappa0, cfg->spectral_exponent) / h->layer_strength[l];
        }
    h->sh_fault = cfg->fault_sh_adjoint ? 1.0 + 1e-6 : 1.0;

    const size_t n = h->n;
    h->c = calloc(n, sizeof(double));
    h->b = calloc(n, sizeof(double));
    h->r = calloc(n, sizeof(double));
    h->p = calloc(n, sizeof(double));
    h->q = calloc(n, sizeof(double));
    h->b1 = calloc(n, sizeof(double));
    h->a_prev2 = calloc(h->A ? h->A : 1, sizeof(double));
    h->a_prev = calloc(h->A ? h->A : 1, sizeof(double));
    h->layer_work = calloc(n, sizeof(double));
    h->wf_work = calloc(h->Nw, sizeof(double));
    h->meas_work = calloc(h->S, sizeof(double));
    h->tmp = calloc((size_t)1 << maxJ, sizeof(double));
    h->fresh = 1;
    return h;
}

void orc_destroy(orc_t* h) {
    if (!h) return;
    void* ptrs[] = {h->n_subap, h->star_is_lgs, h->layer_order, h->n_act, h->noise_variance, h->theta_x,
                    h->theta_y, h->star_height, h->layer_height, h->layer_extent, h->layer_strength, h->dm_height,
                    h->dm_extent, h->masks, h->mask_off, h->meas_off, h->wf_off, h->coeff_off, h->act_off,
                    h->side, h->reg, h->precond, h->dm_group, h->dm_tx, h->dm_ty, h->c, h->b, h->r, h->p, h->q, h->a_prev2, h->a_prev,
                    h->layer_work, h->wf_work, h->meas_work, h->b1, h->z, h->s, h->tmp};
    for (size_t i = 0; i < sizeof ptrs / sizeof ptrs[0]; ++i) free(ptrs[i]);
    free(h);
}

void orc_dims(const orc_t* h, long long* d) {
    d[0] = (long long)h->n;
    d[1] = (long long)h->S;
    d[2] = (long long)h->A;
    d[3] = h->cfg.n_layers;
    d[4] = h->cfg.n_wfs;
    d[5] = h->cfg.n_dms;
    d[6] = h->cfg.pcg_max_iter;
    d[7] = (long long)h->Nw;
}

void orc_geometry(const orc_t* h, double* layer_extent, double* dm_extent, unsigned char* masks) {
    memcpy(layer_extent, h->layer_extent, sizeof(double) * (size_t)h->cfg.n_layers);
    memcpy(dm_extent, h->dm_extent, sizeof(double) * (size_t)h->cfg.n_dms);
    memcpy(masks, h->masks, h->mask_off[h->cfg.n_wfs]);
}
