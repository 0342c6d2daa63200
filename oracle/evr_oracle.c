/*
 * evr_oracle.c -- CPU restatement of the evrecon hot path (TEST ORACLE).
 *
 * Not product code: see the header comment in evr_oracle.h.  Each function
 * cites the reference function it restates; the arithmetic follows the
 * reference expression order term by term and the
 * file must be compiled with -ffp-contract=off so no a*b+c is fused.
 *
 * Pointwise passes are OpenMP-parallel over rows (results do not depend on
 * the partition); every reduction runs serially in index order.
 */
#include "evr_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define IDX(i, j) ((int64_t)(i) * W + (j))

int evo_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

static inline double dmin(double a, double b) { return b < a ? b : a; }
static inline double dmax(double a, double b) { return b > a ? b : a; }
/* np.clip(x, lo, hi) == minimum(maximum(x, lo), hi) */
static inline double dclip(double x, double lo, double hi) {
    return dmin(dmax(x, lo), hi);
}

/* pipeline.py:114-121 apply_event: Python's max(value, u_min) keeps value
 * unless u_min > value; min(.., u_max) keeps it unless u_max < it. */
void evo_ingest(double *f, int64_t *raw, int H, int W, const evo_event *ev,
                int64_t n, double c_pos, double c_neg, double u_min,
                double u_max) {
    (void)H;
    for (int64_t k = 0; k < n; ++k) {
        const int64_t at = IDX(ev[k].y, ev[k].x);
        const double c = ev[k].polarity > 0 ? c_pos : c_neg;
        double v = f[at] * c;
        if (u_min > v) v = u_min;
        if (u_max < v) v = u_max;
        f[at] = v;
        raw[at] = ev[k].t; /* surface.py:124-127, last event wins */
    }
}

/* surface.py:141-142: age = clip(now - raw, 0, win); t = t_scale*(1 - age/win) */
void evo_normalize(const double *raw, int64_t N, double now, double t_scale,
                   double window, double *t) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < N; ++k) {
        const double age = dclip(now - raw[k], 0.0, window);
        t[k] = t_scale * (1.0 - age / window);
    }
}

/* surface.py:93-104: forward differences, zero on the last column / row */
void evo_grad(const double *u, int H, int W, double *gx, double *gy) {
#pragma omp parallel for schedule(static)
    for (int i = 0; i < H; ++i)
        for (int j = 0; j < W; ++j) {
            gx[IDX(i, j)] = j < W - 1 ? u[IDX(i, j + 1)] - u[IDX(i, j)] : 0.0;
            gy[IDX(i, j)] = i < H - 1 ? u[IDX(i + 1, j)] - u[IDX(i, j)] : 0.0;
        }
}

/* surface.py:107-121: x part first, then the y part added into it.  The
 * last column of qx and last row of qy are never read. */
static inline double div_at(const double *qx, const double *qy, int H, int W,
                            int i, int j) {
    double d;
    if (j == 0)
        d = qx[IDX(i, 0)];
    else if (j == W - 1)
        d = -qx[IDX(i, W - 2)];
    else
        d = qx[IDX(i, j)] - qx[IDX(i, j - 1)];
    if (i == 0)
        d = d + qy[IDX(0, j)];
    else if (i == H - 1)
        d = d - qy[IDX(H - 2, j)];
    else
        d = d + (qy[IDX(i, j)] - qy[IDX(i - 1, j)]);
    return d;
}

void evo_div(const double *qx, const double *qy, int H, int W, double *out) {
#pragma omp parallel for schedule(static)
    for (int i = 0; i < H; ++i)
        for (int j = 0; j < W; ++j) out[IDX(i, j)] = div_at(qx, qy, H, W, i, j);
}

/* surface.py:146-196 denoise_timestamps */
void evo_denoise(const double *t_in, int H, int W, double weight, int iters,
                 double t_scale, double *t_out) {
    const int64_t N = (int64_t)H * W;
    const double tau = 1.0 / sqrt(8.0), sigma = tau;
    const double shrink = tau * weight;
    double *u = t_out;
    double *ub = malloc(sizeof(double) * N);
    double *px = calloc(N, sizeof(double));
    double *py = calloc(N, sizeof(double));
    memcpy(u, t_in, sizeof(double) * N);
    memcpy(ub, t_in, sizeof(double) * N);
    for (int it = 0; it < iters; ++it) {
        /* dual ascent + unit-ball projection (surface.py:168-183) */
#pragma omp parallel for schedule(static)
        for (int i = 0; i < H; ++i)
            for (int j = 0; j < W; ++j) {
                const int64_t k = IDX(i, j);
                double gx = j < W - 1 ? ub[k + 1] - ub[k] : 0.0;
                double gy = i < H - 1 ? ub[k + W] - ub[k] : 0.0;
                gx = gx * sigma;
                double a = px[k] + gx;
                gy = gy * sigma;
                double b = py[k] + gy;
                double n = sqrt(a * a + b * b);
                n = dmax(n, 1.0);
                px[k] = a / n;
                py[k] = b / n;
            }
        /* primal step with the L1 soft shrink (surface.py:185-193) */
#pragma omp parallel for schedule(static)
        for (int i = 0; i < H; ++i)
            for (int j = 0; j < W; ++j) {
                const int64_t k = IDX(i, j);
                const double t1 = div_at(px, py, H, W, i, j) * tau + u[k];
                const double g = dclip(t1 - t_in[k], -shrink, shrink);
                const double un = t1 - g;
                ub[k] = un * 2.0 - u[k];
                u[k] = un;
            }
    }
    for (int64_t k = 0; k < N; ++k) u[k] = dclip(u[k], 0.0, t_scale);
    free(ub);
    free(px);
    free(py);
}

/* surface.py:199-205 compute_metric: G = 1 + tx*tx + ty*ty left to right */
void evo_metric(const double *t, int H, int W, double *tx, double *ty,
                double *G, double *sqrtG) {
    evo_grad(t, H, W, tx, ty);
    const int64_t N = (int64_t)H * W;
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < N; ++k) {
        G[k] = 1.0 + tx[k] * tx[k] + ty[k] * ty[k];
        sqrtG[k] = sqrt(G[k]);
    }
}

/* surface.py:81-90 MetricField.coeffs */
void evo_coeffs(const double *tx, const double *ty, const double *G, int64_t N,
                double *a11, double *a12, double *a22, double *a31,
                double *a32) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < N; ++k) {
        a11[k] = (1.0 + ty[k] * ty[k]) / G[k];
        a12[k] = -(tx[k] * ty[k]) / G[k];
        a22[k] = (1.0 + tx[k] * tx[k]) / G[k];
        a31[k] = tx[k] / G[k];
        a32[k] = ty[k] / G[k];
    }
}

typedef struct {
    double *a11, *a12, *a22, *a31, *a32;
} coeffs_t;

static coeffs_t coeffs_alloc(const double *tx, const double *ty,
                             const double *G, int64_t N) {
    coeffs_t c;
    c.a11 = malloc(sizeof(double) * N);
    c.a12 = malloc(sizeof(double) * N);
    c.a22 = malloc(sizeof(double) * N);
    c.a31 = malloc(sizeof(double) * N);
    c.a32 = malloc(sizeof(double) * N);
    evo_coeffs(tx, ty, G, N, c.a11, c.a12, c.a22, c.a31, c.a32);
    return c;
}

static void coeffs_free(coeffs_t *c) {
    free(c->a11);
    free(c->a12);
    free(c->a22);
    free(c->a31);
    free(c->a32);
}

/* surface.py:214-236 */
void evo_surface_gradient(const double *u, const double *tx, const double *ty,
                          const double *G, int H, int W, double *out) {
    const int64_t N = (int64_t)H * W;
    coeffs_t c = coeffs_alloc(tx, ty, G, N);
    double *ux = malloc(sizeof(double) * N), *uy = malloc(sizeof(double) * N);
    evo_grad(u, H, W, ux, uy);
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < N; ++k) {
        out[3 * k + 0] = c.a11[k] * ux[k] + c.a12[k] * uy[k];
        out[3 * k + 1] = c.a12[k] * ux[k] + c.a22[k] * uy[k];
        out[3 * k + 2] = c.a31[k] * ux[k] + c.a32[k] * uy[k];
    }
    free(ux);
    free(uy);
    coeffs_free(&c);
}

/* surface.py:239-252: -div(A^T p) */
void evo_surface_gradient_adjoint(const double *p, const double *tx,
                                  const double *ty, const double *G, int H,
                                  int W, double *out) {
    const int64_t N = (int64_t)H * W;
    coeffs_t c = coeffs_alloc(tx, ty, G, N);
    double *qx = malloc(sizeof(double) * N), *qy = malloc(sizeof(double) * N);
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < N; ++k) {
        const double p1 = p[3 * k], p2 = p[3 * k + 1], p3 = p[3 * k + 2];
        qx[k] = c.a11[k] * p1 + c.a12[k] * p2 + c.a31[k] * p3;
        qy[k] = c.a12[k] * p1 + c.a22[k] * p2 + c.a32[k] * p3;
    }
    evo_div(qx, qy, H, W, out);
    for (int64_t k = 0; k < N; ++k) out[k] = -out[k];
    free(qx);
    free(qy);
    coeffs_free(&c);
}

/* solve.py:88-100: beta = tau*lam*sqrtG, root of the KL prox quadratic */
void evo_prox_data(const double *u_bar, const double *f, const double *sqrtG,
                   int64_t N, double tau, double lam, double u_min,
                   double u_max, double *out) {
    const double tl = tau * lam;
    for (int64_t k = 0; k < N; ++k) {
        const double beta = tl * sqrtG[k];
        const double s = u_bar[k] - beta;
        const double root = 0.5 * (s + sqrt(s * s + 4.0 * beta * f[k]));
        out[k] = dclip(root, u_min, u_max);
    }
}

/* solve.py:103-108: p / max(1, |p| / sqrtG) */
void evo_prox_dual(const double *p, const double *sqrtG, int64_t N,
                   double *out) {
    for (int64_t k = 0; k < N; ++k) {
        const double a = p[3 * k], b = p[3 * k + 1], c = p[3 * k + 2];
        const double nrm = sqrt(a * a + b * b + c * c);
        const double s = dmax(1.0, nrm / sqrtG[k]);
        out[3 * k] = a / s;
        out[3 * k + 1] = b / s;
        out[3 * k + 2] = c / s;
    }
}

/* solve.py:111-118 (tolerance-only: summation order differs from numpy) */
double evo_energy(const double *u, const double *f, const double *tx,
                  const double *ty, const double *G, const double *sqrtG,
                  int H, int W, double lam) {
    const int64_t N = (int64_t)H * W;
    double *su = malloc(sizeof(double) * 3 * N);
    evo_surface_gradient(u, tx, ty, G, H, W, su);
    double tv = 0.0, data = 0.0;
    for (int64_t k = 0; k < N; ++k) {
        const double s = su[3 * k] * su[3 * k] + su[3 * k + 1] * su[3 * k + 1] +
                         su[3 * k + 2] * su[3 * k + 2];
        tv += sqrt(G[k] * s);
        data += (u[k] - f[k] * log(u[k])) * sqrtG[k];
    }
    free(su);
    return tv + lam * data;
}

/* One primal-dual iteration state in SoA planes (solve.py:128-143 _Loop). */
typedef struct {
    int H, W;
    coeffs_t c;
    double *sa[5];
    double *u, *p1, *p2, *p3, *qx, *qy, *v, *un;
} pd_loop;

static void pd_loop_init(pd_loop *L, const double *tx, const double *ty,
                         const double *G, int H, int W, const double *u0,
                         const double *p0, double sigma) {
    const int64_t N = (int64_t)H * W;
    L->H = H;
    L->W = W;
    L->c = coeffs_alloc(tx, ty, G, N);
    double *a[5] = {L->c.a11, L->c.a12, L->c.a22, L->c.a31, L->c.a32};
    for (int m = 0; m < 5; ++m) {
        L->sa[m] = malloc(sizeof(double) * N);
        for (int64_t k = 0; k < N; ++k) L->sa[m][k] = sigma * a[m][k];
    }
    L->u = malloc(sizeof(double) * N);
    L->un = malloc(sizeof(double) * N);
    L->v = malloc(sizeof(double) * N);
    L->qx = malloc(sizeof(double) * N);
    L->qy = malloc(sizeof(double) * N);
    L->p1 = malloc(sizeof(double) * N);
    L->p2 = malloc(sizeof(double) * N);
    L->p3 = malloc(sizeof(double) * N);
    memcpy(L->u, u0, sizeof(double) * N);
    for (int64_t k = 0; k < N; ++k) {
        L->p1[k] = p0 ? p0[3 * k] : 0.0;
        L->p2[k] = p0 ? p0[3 * k + 1] : 0.0;
        L->p3[k] = p0 ? p0[3 * k + 2] : 0.0;
    }
}

static void pd_loop_free(pd_loop *L) {
    coeffs_free(&L->c);
    for (int m = 0; m < 5; ++m) free(L->sa[m]);
    free(L->u);
    free(L->un);
    free(L->v);
    free(L->qx);
    free(L->qy);
    free(L->p1);
    free(L->p2);
    free(L->p3);
}

/* solve.py:144-168 descent_point: q = A^T p, then div(q)*tau + u -> out */
static void pd_descent_point(pd_loop *L, double tau, double *out) {
    const int H = L->H, W = L->W;
    const int64_t N = (int64_t)H * W;
    const coeffs_t c = L->c;
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < N; ++k) {
        L->qx[k] = c.a11[k] * L->p1[k] + c.a12[k] * L->p2[k] + c.a31[k] * L->p3[k];
        L->qy[k] = c.a12[k] * L->p1[k] + c.a22[k] * L->p2[k] + c.a32[k] * L->p3[k];
    }
#pragma omp parallel for schedule(static)
    for (int i = 0; i < H; ++i)
        for (int j = 0; j < W; ++j)
            out[IDX(i, j)] = div_at(L->qx, L->qy, H, W, i, j) * tau + L->u[IDX(i, j)];
}

/* solve.py:170-201 dual_ascent on the over-relaxed point v */
static void pd_dual_ascent(pd_loop *L, const double *v, const double *sqrtG) {
    const int H = L->H, W = L->W;
    double *const *sa = L->sa;
#pragma omp parallel for schedule(static)
    for (int i = 0; i < H; ++i)
        for (int j = 0; j < W; ++j) {
            const int64_t k = IDX(i, j);
            const double gx = j < W - 1 ? v[k + 1] - v[k] : 0.0;
            const double gy = i < H - 1 ? v[k + W] - v[k] : 0.0;
            double p1 = L->p1[k] + sa[0][k] * gx + sa[1][k] * gy;
            double p2 = L->p2[k] + sa[1][k] * gx + sa[2][k] * gy;
            double p3 = L->p3[k] + sa[3][k] * gx + sa[4][k] * gy;
            double n = sqrt(p1 * p1 + p2 * p2 + p3 * p3);
            n = n / sqrtG[k];
            n = dmax(n, 1.0);
            L->p1[k] = p1 / n;
            L->p2[k] = p2 / n;
            L->p3[k] = p3 / n;
        }
}

static double rel_norm_change(const double *u, const double *u_old, int64_t N) {
    double d = 0.0, o = 0.0;
    for (int64_t k = 0; k < N; ++k) {
        const double e = u[k] - u_old[k];
        d += e * e;
        o += u_old[k] * u_old[k];
    }
    return sqrt(d) / dmax(sqrt(o), 1e-30);
}

/* solve.py:207-261 primal_dual_solve */
int evo_pd_solve(const double *f, const double *tx, const double *ty,
                 const double *G, const double *sqrtG, int H, int W,
                 const evo_config *cfg, double *u, double *p,
                 double *rel_change_out, double *energy_trace,
                 double *rel_trace) {
    const int64_t N = (int64_t)H * W;
    pd_loop L;
    pd_loop_init(&L, tx, ty, G, H, W, u, p, cfg->sigma);
    const double tau = cfg->tau;
    const double tl = tau * cfg->lam;
    double *beta = malloc(sizeof(double) * N);
    double *fb = malloc(sizeof(double) * N);
    for (int64_t k = 0; k < N; ++k) {
        beta[k] = tl * sqrtG[k];
        fb[k] = 4.0 * beta[k] * f[k];
    }
    const int track_all = cfg->convergence_tol > 0 || energy_trace || rel_trace;
    double rel = INFINITY;
    int iterations = 0;
    for (int it = 0; it < cfg->max_iterations; ++it) {
        pd_descent_point(&L, tau, L.un);
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < N; ++k) {
            const double s = L.un[k] - beta[k];
            const double r = (s + sqrt(s * s + fb[k])) * 0.5;
            L.un[k] = dclip(r, cfg->u_min, cfg->u_max);
        }
        iterations = it + 1;
        if (track_all || it == cfg->max_iterations - 1)
            rel = rel_norm_change(L.un, L.u, N);
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < N; ++k) L.v[k] = L.un[k] * 2.0 - L.u[k];
        pd_dual_ascent(&L, L.v, sqrtG);
        double *tmp = L.u; /* loop.u = u (fresh array) */
        L.u = L.un;
        L.un = tmp;
        if (energy_trace) energy_trace[it] = evo_energy(L.u, f, tx, ty, G, sqrtG, H, W, cfg->lam);
        if (rel_trace) rel_trace[it] = rel;
        if (cfg->convergence_tol > 0 && rel < cfg->convergence_tol) break;
    }
    memcpy(u, L.u, sizeof(double) * N);
    for (int64_t k = 0; k < N; ++k) {
        p[3 * k] = L.p1[k];
        p[3 * k + 1] = L.p2[k];
        p[3 * k + 2] = L.p3[k];
    }
    if (rel_change_out) *rel_change_out = rel;
    free(beta);
    free(fb);
    pd_loop_free(&L);
    return iterations;
}

/* solve.py:264-293 rof_manifold_solve (tau = sigma = 1/sqrt(8+4*sqrt2)) */
void evo_rof_solve(const double *f, const double *tx, const double *ty,
                   const double *G, const double *sqrtG, int H, int W,
                   double lam, int iters, double *u_out) {
    const int64_t N = (int64_t)H * W;
    const double step = 1.0 / sqrt(8.0 + 4.0 * sqrt(2.0));
    const double tl = step * lam;
    double *wf = malloc(sizeof(double) * N), *inv = malloc(sizeof(double) * N);
    for (int64_t k = 0; k < N; ++k) {
        const double w = tl * sqrtG[k];
        wf[k] = w * f[k];
        inv[k] = 1.0 / (1.0 + w);
    }
    pd_loop L;
    pd_loop_init(&L, tx, ty, G, H, W, f, NULL, step);
    for (int it = 0; it < iters; ++it) {
        pd_descent_point(&L, step, L.un);
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < N; ++k) {
            L.un[k] = (L.un[k] + wf[k]) * inv[k];
            L.v[k] = L.un[k] * 2.0 - L.u[k];
        }
        pd_dual_ascent(&L, L.v, sqrtG);
        double *tmp = L.u;
        L.u = L.un;
        L.un = tmp;
    }
    memcpy(u_out, L.u, sizeof(double) * N);
    free(wf);
    free(inv);
    pd_loop_free(&L);
}

/* ---- data-term / regulariser variants the reference does not ship ------
 * (BASELINE configs[1]: "TV and TGV regularisers, KL vs ROF/L1 data terms").
 * Parity is UNPINNED against the reference (it has no such code); these
 * restate the published algorithms (Chambolle-Pock 2011 primal-dual; TGV of
 * Bredies-Kunisch-Pock 2010) on the reference's manifold operators, in the
 * operation order the CUDA kernels use, so the GPU is checked bit for bit. */

/* data-term prox at one pixel: t1 = div*tau + u (the descent point),
 * beta = (tau*lam)*sqrtG.  kind 0 = KL (solve.py:235-242, box), 1 = ROF
 * (solve.py:283-287), 2 = L1 (|u - f| sqrtG: soft shrink toward f, the
 * surface denoiser's rule surface.py:188-191 with a per-pixel threshold). */
static inline double data_prox(int kind, double t1, double f, double beta,
                               double u_min, double u_max) {
    if (kind == 0) {
        const double s = t1 - beta;
        return dclip((s + sqrt(s * s + (4.0 * beta) * f)) * 0.5, u_min, u_max);
    }
    if (kind == 1) return (t1 + beta * f) * (1.0 / (1.0 + beta));
    const double g = dclip(t1 - f, -beta, beta);
    return t1 - g;
}

/* Manifold TV with the L1 data term: rof_manifold_solve's loop (cold start
 * u = f, p = 0, tau = sigma = 1/sqrt(8+4*sqrt2)) with the L1 prox. */
void evo_l1_solve(const double *f, const double *tx, const double *ty,
                  const double *G, const double *sqrtG, int H, int W,
                  double lam, int iters, double *u_out) {
    const int64_t N = (int64_t)H * W;
    const double step = 1.0 / sqrt(8.0 + 4.0 * sqrt(2.0));
    const double tl = step * lam;
    pd_loop L;
    pd_loop_init(&L, tx, ty, G, H, W, f, NULL, step);
    for (int it = 0; it < iters; ++it) {
        pd_descent_point(&L, step, L.un);
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < N; ++k) {
            L.un[k] = data_prox(2, L.un[k], f[k], tl * sqrtG[k], 0.0, 0.0);
            L.v[k] = L.un[k] * 2.0 - L.u[k];
        }
        pd_dual_ascent(&L, L.v, sqrtG);
        double *tmp = L.u;
        L.u = L.un;
        L.un = tmp;
    }
    memcpy(u_out, L.u, sizeof(double) * N);
    pd_loop_free(&L);
}

/* Second-order manifold TGV:
 *   min_{u,w} alpha1 |A (grad u - w)|_g + alpha0 |E w| + D(u, f)
 * E w = (fx w1, fy w2, (fy w1 + fx w2) / 2) (forward differences, 0 on the
 * last column / row, like grad_x / grad_y), |q|^2 = q11^2 + q22^2 + 2 q12^2;
 * E* q = -(div(q11, q12), div(q12, q22)) with div_xy.  Chambolle-Pock with
 * tau = sigma = 1/sqrt(17 + 4*sqrt2) (|A grad|^2 <= 8 + 4*sqrt2, |A| <= 1,
 * |E|^2 <= 8).  Cold start u = f, w = p = q = 0.  Per iteration:
 *   q = A^T p; u+ = prox_D(div(q)*tau + u);
 *   w+ = w + (q + div_sym)*tau, div_sym = (div(q11, q12), div(q12, q22));
 *   u_bar = u+*2 - u, w_bar = w+*2 - w;
 *   p = proj_{alpha1 sqrtG}(p + sigma A (grad u_bar - w_bar));
 *   Q = proj_{alpha0}(Q + sigma E w_bar).
 * w_out (may be NULL) receives w as (H, W, 2). */
void evo_tgv_solve(const double *f, const double *tx, const double *ty,
                   const double *G, const double *sqrtG, int H, int W,
                   double lam, double alpha0, double alpha1, int kind,
                   double u_min, double u_max, int iters, double *u_out,
                   double *w_out) {
    const int64_t N = (int64_t)H * W;
    const double step = 1.0 / sqrt(17.0 + 4.0 * sqrt(2.0));
    const double tl = step * lam;
    pd_loop L;
    pd_loop_init(&L, tx, ty, G, H, W, f, NULL, step);
    double *w1 = calloc(N, sizeof(double)), *w2 = calloc(N, sizeof(double));
    double *w1n = malloc(sizeof(double) * N), *w2n = malloc(sizeof(double) * N);
    double *b1 = malloc(sizeof(double) * N), *b2 = malloc(sizeof(double) * N);
    double *q11 = calloc(N, sizeof(double)), *q22 = calloc(N, sizeof(double));
    double *q12 = calloc(N, sizeof(double));
    const coeffs_t c = L.c;
    double *const *sa = L.sa;
    for (int it = 0; it < iters; ++it) {
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < N; ++k) {
            L.qx[k] = c.a11[k] * L.p1[k] + c.a12[k] * L.p2[k] + c.a31[k] * L.p3[k];
            L.qy[k] = c.a12[k] * L.p1[k] + c.a22[k] * L.p2[k] + c.a32[k] * L.p3[k];
        }
#pragma omp parallel for schedule(static)
        for (int i = 0; i < H; ++i)
            for (int j = 0; j < W; ++j) {
                const int64_t k = IDX(i, j);
                const double t1 = div_at(L.qx, L.qy, H, W, i, j) * step + L.u[k];
                L.un[k] = data_prox(kind, t1, f[k], tl * sqrtG[k], u_min, u_max);
                L.v[k] = L.un[k] * 2.0 - L.u[k];
                const double e1 = div_at(q11, q12, H, W, i, j);
                const double e2 = div_at(q12, q22, H, W, i, j);
                w1n[k] = w1[k] + (L.qx[k] + e1) * step;
                w2n[k] = w2[k] + (L.qy[k] + e2) * step;
                b1[k] = w1n[k] * 2.0 - w1[k];
                b2[k] = w2n[k] * 2.0 - w2[k];
            }
#pragma omp parallel for schedule(static)
        for (int i = 0; i < H; ++i)
            for (int j = 0; j < W; ++j) {
                const int64_t k = IDX(i, j);
                const double *v = L.v;
                const double gx = (j < W - 1 ? v[k + 1] - v[k] : 0.0) - b1[k];
                const double gy = (i < H - 1 ? v[k + W] - v[k] : 0.0) - b2[k];
                double p1 = L.p1[k] + sa[0][k] * gx + sa[1][k] * gy;
                double p2 = L.p2[k] + sa[1][k] * gx + sa[2][k] * gy;
                double p3 = L.p3[k] + sa[3][k] * gx + sa[4][k] * gy;
                double n = sqrt(p1 * p1 + p2 * p2 + p3 * p3);
                n = n / (alpha1 * sqrtG[k]);
                n = dmax(n, 1.0);
                L.p1[k] = p1 / n;
                L.p2[k] = p2 / n;
                L.p3[k] = p3 / n;
                const double e11 = j < W - 1 ? b1[k + 1] - b1[k] : 0.0;
                const double e22 = i < H - 1 ? b2[k + W] - b2[k] : 0.0;
                const double e12 = ((i < H - 1 ? b1[k + W] - b1[k] : 0.0) +
                                    (j < W - 1 ? b2[k + 1] - b2[k] : 0.0)) * 0.5;
                const double a = q11[k] + step * e11;
                const double b = q22[k] + step * e22;
                const double d = q12[k] + step * e12;
                double m = sqrt(a * a + b * b + (d * d) * 2.0);
                m = dmax(m / alpha0, 1.0);
                q11[k] = a / m;
                q22[k] = b / m;
                q12[k] = d / m;
            }
        double *tmp = L.u;
        L.u = L.un;
        L.un = tmp;
        tmp = w1;
        w1 = w1n;
        w1n = tmp;
        tmp = w2;
        w2 = w2n;
        w2n = tmp;
    }
    memcpy(u_out, L.u, sizeof(double) * N);
    if (w_out)
        for (int64_t k = 0; k < N; ++k) {
            w_out[2 * k] = w1[k];
            w_out[2 * k + 1] = w2[k];
        }
    free(w1);
    free(w2);
    free(w1n);
    free(w2n);
    free(b1);
    free(b2);
    free(q11);
    free(q22);
    free(q12);
    pd_loop_free(&L);
}

/* pipeline.py:142-171 process_packet (non-empty packet) with the window of
 * pipeline.py:128-132 supplied by the caller. */
int evo_process_packet(double *u, double *f, int64_t *raw, double *p, int H,
                       int W, const evo_event *ev, int64_t n, double window,
                       const evo_config *cfg, double *rel_change_out,
                       double *t_out, double *G_out) {
    const int64_t N = (int64_t)H * W;
    evo_ingest(f, raw, H, W, ev, n, cfg->c_pos, cfg->c_neg, cfg->u_min, cfg->u_max);
    const int64_t now = ev[n - 1].t;
    double *t = calloc(N, sizeof(double));
    double *tx = malloc(sizeof(double) * N), *ty = malloc(sizeof(double) * N);
    double *G = malloc(sizeof(double) * N), *sg = malloc(sizeof(double) * N);
    if (cfg->manifold_enabled) {
        double *rawf = malloc(sizeof(double) * N);
        double *tn = malloc(sizeof(double) * N);
        for (int64_t k = 0; k < N; ++k) rawf[k] = (double)raw[k];
        evo_normalize(rawf, N, (double)now, cfg->t_scale, window, tn);
        evo_denoise(tn, H, W, cfg->denoise_weight, cfg->denoise_iterations,
                    cfg->t_scale, t);
        free(rawf);
        free(tn);
    }
    /* flat_metric (surface.py:208-211) equals compute_metric of t = 0 */
    evo_metric(t, H, W, tx, ty, G, sg);
    if (t_out) memcpy(t_out, t, sizeof(double) * N);
    if (G_out) memcpy(G_out, G, sizeof(double) * N);
    const int iters = evo_pd_solve(f, tx, ty, G, sg, H, W, cfg, u, p,
                                   rel_change_out, NULL, NULL);
    memcpy(f, u, sizeof(double) * N); /* re-anchor f <- u (pipeline.py:169) */
    free(t);
    free(tx);
    free(ty);
    free(G);
    free(sg);
    return iters;
}
