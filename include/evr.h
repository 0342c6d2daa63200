/*
 * evr.h -- C ABI of the B200-native per-packet event reconstruction
 *          (arXiv 1607.06283), the drop-in for the evrecon hot path.
 *
 * The reference (/root/reference/pkg/src/evrecon) is a pure-Python/numpy
 * package with no FFI; its "operator API" is the Python module surface.
 * Each entry point below names the reference function it replaces
 * (file:line).  The Python host package paper_1607_06283_b200 binds this
 * header with ctypes and re-exports the reference names; INTEGRATION.md
 * shows the binding a maintainer of the reference would add.
 *
 * Conventions
 *  - Plain C: pointers + sizes, no C++ or torch types.  Every call returns
 *    EVR_OK (0) or a negative evr_status; evr_last_error(ctx) describes the
 *    last failure on that context.  Nothing throws across the ABI.
 *  - Host arrays are row-major (H, W) float64 / int64, dual fields p are
 *    (H, W, 3) float64 interleaved -- exactly the reference's numpy layouts.
 *    Host pointers are borrowed for the duration of the call only.
 *  - One evr_ctx per (event stream, device).  Calls on a context are
 *    serialised on its own CUDA stream; use one host thread per context.
 *  - EVR_PREC_F64 reproduces the reference bit for bit (every stage, every
 *    packet).  EVR_PREC_F32 runs the surface and the solver in binary32
 *    (ingest stays binary64/int64 and bit-exact); it is held to 1e-4
 *    max-abs on log u against the reference.
 */
#ifndef EVR_H
#define EVR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EVR_ABI_VERSION 1

typedef enum {
    EVR_OK = 0,
    EVR_ERR_INVALID = -1,     /* bad argument (maps to ValueError) */
    EVR_ERR_CUDA = -2,        /* CUDA runtime failure */
    EVR_ERR_OOM = -3,         /* device allocation failed */
    EVR_ERR_RANGE = -4,       /* event coordinate outside the sensor */
    EVR_ERR_UNSUPPORTED = -5  /* shape/mode not supported by this call */
} evr_status;

typedef enum { EVR_PREC_F64 = 0, EVR_PREC_F32 = 1 } evr_precision;

/* Solver-engine selection for the per-packet path. */
typedef enum {
    EVR_ENGINE_AUTO = 0,      /* shared-memory resident for small sensors (<= 2 rows
                                 per SM), else streaming */
    EVR_ENGINE_STREAMING = 1, /* fused list: temporally blocked tiles in HBM/L2 */
    EVR_ENGINE_RESIDENT = 2   /* persistent kernel, row bands on chip (registers +
                                 shared memory) */
} evr_engine;

/* One camera event: events.py:35-43 Event(x, y, polarity, timestamp).
 * 16 bytes, little endian; numpy dtype
 * [('t','<i8'),('x','<i4'),('y','<i2'),('polarity','<i2')]. */
typedef struct {
    int64_t t;
    int32_t x;
    int16_t y;
    int16_t polarity;
} evr_event;

/* SolverConfig (solve.py:41-78), ManifoldConfig (pipeline.py:71-84) and
 * Thresholds (pipeline.py:51-68; c_pos/c_neg are host math.exp values). */
typedef struct {
    double lam, u_min, u_max, tau, sigma, convergence_tol;
    int32_t max_iterations;
    int32_t manifold_enabled;
    double t_scale;
    double denoise_weight;
    int32_t denoise_iterations;
    int32_t engine; /* evr_engine */
    double c_pos, c_neg;
} evr_config;

/* SolveResult.iterations / .rel_change (solve.py:81-85).  packet_ms: the
 * packet's device time from the start of its event upload to the end of its
 * frame download, filled by evr_frame_wait (the frame pipeline's analogue of
 * run_stream's per-packet solve_ms, pipeline.py:239-249); 0 elsewhere. */
typedef struct {
    int32_t iterations;
    float packet_ms;
    double rel_change;
} evr_solve_info;

typedef struct evr_ctx evr_ctx;

/* ---- lifetime ---------------------------------------------------------- */
const char *evr_version(void);
int evr_device_count(int *count);
/* A context for an H x W sensor on `device` (H, W >= 1; the stencil entry
 * points need H, W >= 2 like the reference's div_xy, surface.py:107-121). */
int evr_create(evr_ctx **out, int device, int height, int width, int precision);
void evr_destroy(evr_ctx *ctx);
const char *evr_last_error(const evr_ctx *ctx);
int evr_set_config(evr_ctx *ctx, const evr_config *cfg);
/* engine actually used by the per-packet path (after AUTO resolution) */
int evr_active_engine(evr_ctx *ctx, int *engine);
/* human-readable kernel shape of the per-packet path, e.g.
 * "k_resident_col<f64,NT=384,RB=2> x130 CTAs" (NUL-terminated, truncated) */
int evr_engine_detail(evr_ctx *ctx, char *buf, int len);

/* ---- stream state: ReconstructionState (pipeline.py:87-111) ------------- */
/* init_state (pipeline.py:102-111): u = f = (u_min+u_max)/2, raw = 0, p = 0 */
int evr_init_state(evr_ctx *ctx);
/* NULL pointers leave that field untouched. */
int evr_set_state(evr_ctx *ctx, const double *u, const double *f,
                  const int64_t *raw, const double *p);
int evr_get_state(evr_ctx *ctx, double *u, double *f, int64_t *raw, double *p);

/* ---- hot path ------------------------------------------------------------ */
/* apply_event (pipeline.py:114-121) for n events in stream order, with
 * update_timestamp_map (surface.py:124-127).  Bit-exact, duplicates
 * included.  Host events. */
int evr_ingest(evr_ctx *ctx, const evr_event *events, int64_t n);
/* process_packet (pipeline.py:142-171) for a non-empty packet: ingest,
 * normalize/denoise/metric (_packet_metric, pipeline.py:124-139), the
 * warm-started primal_dual_solve and the f <- u re-anchor.  `window` is the
 * surface window the host derived from packet_starts (pipeline.py:128-132;
 * ignored when the manifold is disabled).  Synchronous; host events. */
int evr_process_packet(evr_ctx *ctx, const evr_event *events, int64_t n,
                       double window, evr_solve_info *info);
/* Same, asynchronous: enqueue on the context stream and return.  Host
 * events are staged through pinned memory before the call returns. */
int evr_process_packet_async(evr_ctx *ctx, const evr_event *events, int64_t n,
                             double window);
/* Same, events already resident in device memory (`dev_events`). */
int evr_process_packet_device(evr_ctx *ctx, const evr_event *dev_events,
                              int64_t n, double window);
/* process_packet in two halves, for callers that look at the surface
 * between them (debug_sink, pipeline.py:162-163) or need the host-driven
 * solve (convergence_tol > 0 early stop, per-iteration energy trace rows
 * of solve.py:255-256).  begin = ingest + surface; solve = primal-dual +
 * re-anchor.  energy_trace / rel_trace have max_iterations slots (NULL ok);
 * info->iterations says how many were filled. */
int evr_packet_begin(evr_ctx *ctx, const evr_event *events, int64_t n,
                     double window);
int evr_packet_solve(evr_ctx *ctx, evr_solve_info *info, double *energy_trace,
                     double *rel_trace);
/* Wait for queued packets; info (may be NULL) gets the last packet's result. */
int evr_synchronize(evr_ctx *ctx, evr_solve_info *info);
/* Current frame u (the value process_packet returns), float64 (H, W). */
int evr_get_frame(evr_ctx *ctx, double *u_out);
/* evr_get_frame enqueued on the context stream without waiting (complete
 * after evr_synchronize); asynchronous when u_out is pinned host memory */
int evr_get_frame_async(evr_ctx *ctx, double *u_out);
/* Streaming engine, whole-sensor contexts: primal-dual / TV-L1 iterations
 * fused per launch by the temporally blocked tile kernels (1 = one march
 * launch per iteration, 2..4 = tiles, 0 = the EVR_TILE_K default).
 * Results are bit-identical for every k; this is a performance knob. */
int evr_set_tile_k(evr_ctx *ctx, int k);
/* Measurement hook (bench.py's roofline): times `reps` back-to-back launches
 * of the streaming list's iteration kernel -- which = 0 the primal-dual tile
 * (solve.py:233-258), 1 the TV-L1 tile (surface.py:167-193) -- on the
 * context stream with CUDA events, on the packed state the last packet left
 * (scratch: the next packet re-packs from the state planes).  Whole-sensor
 * streaming contexts only. */
int evr_time_iteration_kernel(evr_ctx *ctx, int which, int reps, float *us_per_launch,
                              int *iterations_per_launch);
/* Pipelined read-back for streams (run_stream, pipeline.py:206-276, with
 * packet k+1 computing while frame k travels to the host).  Submit, right
 * after evr_process_packet_async, snapshots this packet's frame u (float64
 * (H, W) into u_out, pinned host memory, or NULL for the record only) and
 * its SolveResult record; the copy runs on a second stream, so the caller
 * may enqueue the next packet at once.  Wait blocks until ticket's frame and
 * record are on the host.  At most 4 tickets in flight; waits in any order.
 * An event outside the sensor is reported by the wait of that packet. */
int evr_frame_submit(evr_ctx *ctx, double *u_out, int64_t *ticket);
int evr_frame_wait(evr_ctx *ctx, int64_t ticket, evr_solve_info *info);
/* page-locked host buffers for frames / events (cudaHostAlloc) */
int evr_host_alloc(size_t bytes, void **out);
int evr_host_free(void *p);
/* Last packet's denoised surface t and metric determinant G (the
 * debug_sink view, pipeline.py:162-163).  Either pointer may be NULL. */
int evr_get_surface(evr_ctx *ctx, double *t_out, double *G_out);
/* Last packet's metric field (compute_metric / flat_metric outputs). */
int evr_get_metric(evr_ctx *ctx, double *tx, double *ty, double *G, double *sqrtG);
/* Frame quantised to 8-bit gray on device (pgm.py:14-22 to_gray,
 * floor(255*(u-lo)/(hi-lo)+0.5) clipped to [0,255]). */
int evr_get_frame_u8(evr_ctx *ctx, double lo, double hi, uint8_t *out);
/* Device pointer of the event staging buffer with room for `n` events
 * (grows on demand); for zero-copy producers. */
int evr_event_buffer(evr_ctx *ctx, int64_t n, evr_event **dev_ptr);
/* CUDA stream handle (cudaStream_t) the context runs on. */
void *evr_stream(evr_ctx *ctx);
/* Count of kernel launches this context issued (graph nodes included). */
int64_t evr_launch_count(const evr_ctx *ctx);

/* Diagnostics: enable (1) / disable (0) / keep (-1) the resident engine's
 * phase timeline (globaltimer ns per phase mark, 256 slots per CTA) and
 * copy up to n words of it to out (may be NULL). */
int evr_debug_timeline(evr_ctx *ctx, int enable, uint64_t *out, int64_t n);

/* ---- row-band groups: one sensor over several contexts / GPUs ------------ */
/* The megapixel configuration (BASELINE configs[4]): the
 * sensor's rows are split into n_bands contiguous bands, band b on
 * devices[b] (NULL: all on device 0); every packet runs the streaming step
 * list on all bands in lock step with one halo row exchanged per half-step
 * over peer copies (NVLink between GPUs).  Bit-identical to evr_ctx. */
typedef struct evr_group evr_group;
int evr_group_create(evr_group **out, int n_bands, const int *devices,
                     int height, int width, int precision);
void evr_group_destroy(evr_group *grp);
const char *evr_group_last_error(const evr_group *grp);
int evr_group_band(evr_group *grp, int b, int *y0, int *y1, int *device);
int evr_group_set_config(evr_group *grp, const evr_config *cfg);
int evr_group_init_state(evr_group *grp);
/* full-sensor host arrays, as evr_set_state / evr_get_state */
int evr_group_set_state(evr_group *grp, const double *u, const double *f,
                        const int64_t *raw, const double *p);
int evr_group_get_state(evr_group *grp, double *u, double *f, int64_t *raw,
                        double *p);
/* process_packet (pipeline.py:142-171) over all bands; synchronous */
int evr_group_process_packet(evr_group *grp, const evr_event *events,
                             int64_t n, double window, evr_solve_info *info);
int evr_group_get_frame(evr_group *grp, double *u_out);
int64_t evr_group_launch_count(const evr_group *grp);

/* ---- event text front-end (host only, no device) ------------------------ */
/* Text event parser: the grammar and validation of parse_event_line /
 * read_stream (events.py:65-130) straight into packed events.  `st` carries
 * the 1-based line number, the event index and the running maximum
 * timestamp across calls (zero-initialise it for a new stream).  Parsing
 * stops at the end of `text`, after `cap` events, or at the first invalid
 * line: then EVR_ERR_INVALID, *err_kind = EVR_PARSE_BAD_LINE (malformed,
 * negative or out-of-sensor: the reference's EventParseError) or
 * EVR_PARSE_ORDER (timestamp below running_max - slack: StreamOrderError),
 * *err_offset = byte offset of that line, `st` as before that line.
 * *consumed = bytes of whole lines consumed. */
enum { EVR_PARSE_OK = 0, EVR_PARSE_BAD_LINE = 1, EVR_PARSE_ORDER = 2 };
typedef struct {
    int64_t line_no;
    int64_t index;
    int64_t running_max;
    int32_t have_max;
    int32_t _pad;
} evr_parse_state;
int evr_parse_events(const char *text, int64_t len, int width, int height,
                     int64_t slack, evr_parse_state *st, evr_event *out,
                     int64_t cap, int64_t *n_out, int64_t *consumed,
                     int64_t *err_offset, int32_t *err_kind);

/* ---- operator-level API on host arrays of the context's shape ----------- */
/* grad_x / grad_y (surface.py:93-104) */
int evr_op_grad(evr_ctx *ctx, const double *u, double *gx, double *gy);
/* div_xy (surface.py:107-121) */
int evr_op_div(evr_ctx *ctx, const double *qx, const double *qy, double *out);
/* normalize_timestamps (surface.py:130-143); raw as float64 like the
 * reference's np.asarray(raw_map, dtype=np.float64) */
int evr_op_normalize(evr_ctx *ctx, const double *raw, double now,
                     double t_scale, double window, double *t_out);
/* denoise_timestamps (surface.py:146-196) */
int evr_op_denoise(evr_ctx *ctx, const double *t_in, double weight,
                   int iterations, double t_scale, double *t_out);
/* compute_metric (surface.py:199-205) */
int evr_op_metric(evr_ctx *ctx, const double *t, double *tx, double *ty,
                  double *G, double *sqrtG);
/* MetricField.coeffs (surface.py:81-90): out = 5 planes a11,a12,a22,a31,a32 */
int evr_op_coeffs(evr_ctx *ctx, const double *tx, const double *ty,
                  const double *G, double *out5);
/* surface_gradient (surface.py:214-236): out (H, W, 3) */
int evr_op_surface_gradient(evr_ctx *ctx, const double *u, const double *tx,
                            const double *ty, const double *G, double *out);
/* surface_gradient_adjoint (surface.py:239-252): p (H, W, 3) -> out (H, W) */
int evr_op_surface_gradient_adjoint(evr_ctx *ctx, const double *p,
                                    const double *tx, const double *ty,
                                    const double *G, double *out);
/* prox_data (solve.py:88-100), elementwise */
int evr_op_prox_data(evr_ctx *ctx, const double *u_bar, const double *f,
                     const double *sqrtG, double tau, double lam, double u_min,
                     double u_max, double *out);
/* prox_dual (solve.py:103-108): p (H, W, 3) */
int evr_op_prox_dual(evr_ctx *ctx, const double *p, const double *sqrtG,
                     double *out);
/* energy (solve.py:111-118) */
int evr_op_energy(evr_ctx *ctx, const double *u, const double *f,
                  const double *tx, const double *ty, const double *G,
                  const double *sqrtG, double lam, double *out);
/* primal_dual_solve (solve.py:207-261) on a given metric.  u_init / p_init
 * may be NULL (defaults u = f, p = 0).  energy_trace / rel_trace (length
 * cfg->max_iterations, may be NULL) receive the trace rows. */
int evr_op_pd_solve(evr_ctx *ctx, const evr_config *cfg, const double *f,
                    const double *tx, const double *ty, const double *G,
                    const double *sqrtG, const double *u_init,
                    const double *p_init, double *u_out, double *p_out,
                    evr_solve_info *info, double *energy_trace,
                    double *rel_trace);
/* to_gray (pgm.py:14-22): floor(255*(image-lo)/(hi-lo) + 0.5) clipped to
 * [0, 255], uint8 (H, W) */
int evr_op_to_gray(evr_ctx *ctx, const double *image, double lo, double hi,
                   uint8_t *out);
/* rof_manifold_solve (solve.py:264-293) */
int evr_op_rof_solve(evr_ctx *ctx, const double *f, const double *tx,
                     const double *ty, const double *G, const double *sqrtG,
                     double lam, int iterations, double *u_out);
/* Not in the reference (BASELINE configs[1] names them; parity unpinned,
 * restated in oracle/evr_oracle.c): manifold TV with the L1 data term
 * lam * sum |u - f| sqrtG (rof_manifold_solve's loop, cold start), and
 * second-order manifold TGV
 *   min_{u,w} alpha1 |A (grad u - w)|_g + alpha0 |E w| + D(u, f)
 * with D = KL (data_term 0, box [u_min, u_max]), ROF (1) or L1 (2); w_out
 * (H, W, 2) may be NULL. */
int evr_op_l1_solve(evr_ctx *ctx, const double *f, const double *tx,
                    const double *ty, const double *G, const double *sqrtG,
                    double lam, int iterations, double *u_out);
int evr_op_tgv_solve(evr_ctx *ctx, const double *f, const double *tx,
                     const double *ty, const double *G, const double *sqrtG,
                     double lam, double alpha0, double alpha1, int data_term,
                     double u_min, double u_max, int iterations,
                     double *u_out, double *w_out);

/* ---- event simulator: simulate.py:51-103 generate_events - */
/* Events of a (n, H, W) stack of LOG intensities (the caller takes np.log,
 * simulate.py:60) with strictly increasing integer frame timestamps, under
 * thresholds dp, dn > 0; sorted by (t, y, x, polarity) like the reference's
 * lexsort.  Limits of the packed sort key: H <= 32767, W <= 65535, frame time
 * span < 2^30 ticks. */
typedef struct evr_sim evr_sim;
int evr_sim_create(evr_sim **out, int device);
void evr_sim_destroy(evr_sim *sim);
const char *evr_sim_last_error(const evr_sim *sim);
int evr_sim_generate(evr_sim *sim, const double *log_frames,
                     const int64_t *frame_timestamps, int n, int H, int W,
                     double dp, double dn, int64_t *n_events);
/* copy the generated events out (cap >= n_events) */
int evr_sim_events(evr_sim *sim, evr_event *out, int64_t cap);
/* device pointer of the generated events (valid until the next generate or
 * destroy), for evr_process_packet_device */
int evr_sim_device_events(evr_sim *sim, const evr_event **dev_events,
                          int64_t *n);

#ifdef __cplusplus
}
#endif
#endif /* EVR_H */
