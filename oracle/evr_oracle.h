/*
 * evr_oracle.h -- CPU restatement of the evrecon per-packet hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA path
 * (paper_1607_06283_b200/csrc) and the CPU baseline leg of bench.py.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it.  The product path never links or calls it.
 *
 * Every function restates one reference function in plain C99, in the
 * reference's exact floating-point operation order (compiled with
 * -ffp-contract=off, no fast-math), so that on IEEE-754 binary64 it is
 * bit-identical to numpy.  Pinned against golden vectors produced by the
 * reference itself (tests/golden/make_golden.py) in tests/test_oracle.py.
 *
 * Layout: fields are row-major (H, W) float64 indexed [y*W + x]; dual
 * fields p are (H, W, 3) interleaved, exactly like the reference state.
 */
#ifndef EVR_ORACLE_H
#define EVR_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Packed event, identical layout to evr_event in include/evr.h. */
typedef struct {
    int64_t t;
    int32_t x;
    int16_t y;
    int16_t polarity;
} evo_event;

typedef struct {
    double lam, u_min, u_max, tau, sigma, convergence_tol;
    int32_t max_iterations;
    int32_t manifold_enabled;
    double t_scale;
    double denoise_weight;
    int32_t denoise_iterations;
    int32_t _pad;
    double c_pos, c_neg;
} evo_config;

/* pipeline.py:114-121 apply_event (+ surface.py:124-127), n events in order */
void evo_ingest(double *f, int64_t *raw, int H, int W, const evo_event *ev,
                int64_t n, double c_pos, double c_neg, double u_min, double u_max);

/* surface.py:130-143 normalize_timestamps; raw given as float64 */
void evo_normalize(const double *raw, int64_t N, double now, double t_scale,
                   double window, double *t);

/* surface.py:93-104 grad_x / grad_y */
void evo_grad(const double *u, int H, int W, double *gx, double *gy);

/* surface.py:107-121 div_xy */
void evo_div(const double *qx, const double *qy, int H, int W, double *out);

/* surface.py:146-196 denoise_timestamps (flat TV-L1 primal-dual) */
void evo_denoise(const double *t_in, int H, int W, double weight, int iters,
                 double t_scale, double *t_out);

/* surface.py:199-205 compute_metric */
void evo_metric(const double *t, int H, int W, double *tx, double *ty,
                double *G, double *sqrtG);

/* surface.py:81-90 MetricField.coeffs */
void evo_coeffs(const double *tx, const double *ty, const double *G, int64_t N,
                double *a11, double *a12, double *a22, double *a31, double *a32);

/* surface.py:214-236 surface_gradient -> out (H,W,3) */
void evo_surface_gradient(const double *u, const double *tx, const double *ty,
                          const double *G, int H, int W, double *out);

/* surface.py:239-252 surface_gradient_adjoint -> out (H,W) */
void evo_surface_gradient_adjoint(const double *p, const double *tx,
                                  const double *ty, const double *G, int H,
                                  int W, double *out);

/* solve.py:88-100 prox_data (elementwise over N) */
void evo_prox_data(const double *u_bar, const double *f, const double *sqrtG,
                   int64_t N, double tau, double lam, double u_min,
                   double u_max, double *out);

/* solve.py:103-108 prox_dual (p interleaved (N,3)) */
void evo_prox_dual(const double *p, const double *sqrtG, int64_t N, double *out);

/* solve.py:111-118 energy (sequential summation order) */
double evo_energy(const double *u, const double *f, const double *tx,
                  const double *ty, const double *G, const double *sqrtG,
                  int H, int W, double lam);

/* solve.py:207-261 primal_dual_solve.  u (H,W) and p (H,W,3) are the warm
 * start on entry and the result on exit.  energy_trace / rel_trace (length
 * max_iterations, may be NULL) receive the per-iteration trace rows. */
int evo_pd_solve(const double *f, const double *tx, const double *ty,
                 const double *G, const double *sqrtG, int H, int W,
                 const evo_config *cfg, double *u, double *p,
                 double *rel_change_out, double *energy_trace,
                 double *rel_trace);

/* solve.py:264-293 rof_manifold_solve; u_out (H,W) */
void evo_rof_solve(const double *f, const double *tx, const double *ty,
                   const double *G, const double *sqrtG, int H, int W,
                   double lam, int iters, double *u_out);

/* Not in the reference (parity unpinned, see evr_oracle.c): manifold TV
 * with the L1 data term, and second-order manifold TGV with data term kind
 * 0 = KL (box [u_min, u_max]), 1 = ROF, 2 = L1.  w_out (H,W,2) may be NULL. */
void evo_l1_solve(const double *f, const double *tx, const double *ty,
                  const double *G, const double *sqrtG, int H, int W,
                  double lam, int iters, double *u_out);
void evo_tgv_solve(const double *f, const double *tx, const double *ty,
                   const double *G, const double *sqrtG, int H, int W,
                   double lam, double alpha0, double alpha1, int kind,
                   double u_min, double u_max, int iters, double *u_out,
                   double *w_out);

/* pipeline.py:142-171 process_packet for a non-empty packet, given the
 * window the caller derived from packet_starts (pipeline.py:124-132).
 * State arrays are updated in place; t_out/tx_out/... (may be NULL) receive
 * the packet's surface and metric (the debug_sink view).  Returns the
 * iteration count. */
int evo_process_packet(double *u, double *f, int64_t *raw, double *p, int H,
                       int W, const evo_event *ev, int64_t n, double window,
                       const evo_config *cfg, double *rel_change_out,
                       double *t_out, double *G_out);

int evo_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
