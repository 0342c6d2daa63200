// evr_capi.cu -- the C ABI (include/evr.h): per-stream device context,
// captured CUDA graphs of the per-packet sequence, and the operator API.
//
// Engines
//   streaming: one launch per half-step over HBM/L2-resident SoA planes
//              (evr_kernels.cuh); the whole packet is one CUDA graph.
//   resident : one persistent kernel per packet, state on chip in row bands
//              (evr_resident.cuh); used when the sensor fits (AUTO).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/evr.h"
#include "evr_kernels.cuh"
#include "evr_tile.cuh"
#include "evr_resident.cuh"
#include "evr_resident_col.cuh"

using namespace evr;

namespace {

constexpr int kNT = 256;          // 1-D block size
constexpr int kIngestNT = 256;    // ingest CTA size (events per chunk)
constexpr int kRedBlocks = 296;   // reduction partial blocks (2 x 148 SMs)

enum Field {
  F_U, F_UN, F_V, F_P1, F_P2, F_P3,
  F_T, F_TU, F_TUB, F_TPX, F_TPY,
  F_TX, F_TY, F_G, F_SG, F_A11, F_A12, F_A22, F_A31, F_A32, F_BETA, F_FB,
  F_COUNT
};

}  // namespace

constexpr int kFrameSlots = 4;
struct FrameRec {
  evr_solve_info info;
  int err;
  int pad;
};

struct evr_ctx {
  int device = 0;
  int H = 0, W = 0;
  int64_t N = 0;
  int prec = EVR_PREC_F64;
  evr_config cfg{};
  bool cfg_set = false;
  cudaStream_t stream = nullptr;
  // device memory
  char* slab = nullptr;
  size_t field_stride = 0;  // bytes between planes
  double* f = nullptr;
  int64_t* raw = nullptr;
  double* aos_a = nullptr;  // (H, W, 3) staging
  double* aos_b = nullptr;
  double* part = nullptr;   // reduction partials
  unsigned* rticket = nullptr;  // k_relchange's last-CTA ticket
  int* d_stop = nullptr;         // fused list, convergence_tol > 0: the stop flag
  double* d_hist = nullptr;      // traced host-driven solve: per-iteration rel_change | energy
  int hist_cap = 0;
  double* d_scalar = nullptr;
  int* d_err = nullptr;
  evr_solve_info* d_info = nullptr;
  // packet staging: [PacketHdr | events...] on device and 2 pinned host slots
  char* d_stage = nullptr;
  char* h_stage[2] = {nullptr, nullptr};
  cudaEvent_t stage_done[2] = {nullptr, nullptr};
  int stage_slot = 0;
  int64_t ev_cap = 0;
  evr_solve_info* h_info = nullptr;
  int64_t seq = 0;
  // graphs: 0 = surface, 1 = solve, 2 = whole packet
  cudaGraphExec_t graph[3] = {nullptr, nullptr, nullptr};
  int64_t graph_launches[3] = {0, 0, 0};
  int64_t launches = 0;
  int engine = EVR_ENGINE_STREAMING;  // resolved
  int tile_k = 0;                     // fused iterations per tile launch (0 = EVR_TILE_K default)
  // resident engine plan + buffers
  int r_nb = 0, r_R = 0, r_nt = 0, r_ms = 0;
  size_t r_smem = 0, r_frame = 0;
  void* d_pack = nullptr;                 // packed state of the fused streaming list
  unsigned long long* d_flags = nullptr;  // per-CTA progress words
  void* d_xchg = nullptr;                 // boundary-row ping-pong buffer
  unsigned* d_ticket = nullptr;
  unsigned long long* d_rx = nullptr;     // k_resident_col: per-iteration rel_change partials
  int* d_perm = nullptr;                  // k_resident_col: band of each CTA (SM order)
  unsigned long long* d_trace = nullptr;  // optional resident phase timeline
  // band geometry: local plane rows [0, H) are global rows row0 + [0, H);
  // own rows [own_lo, own_hi]; a whole-sensor context owns all its rows
  int row0 = 0, Htot = 0, own_lo = 0, own_hi = -1;
  bool banded = false;
  // bands: the contexts of the bands above / below (their packed state is
  // read in place by the fused iteration kernels; peer memory across GPUs)
  const evr_ctx* nb_up = nullptr;
  const evr_ctx* nb_dn = nullptr;
  // pipelined frame read-back (evr_frame_submit / evr_frame_wait): per slot a
  // device snapshot of u (float64) + the packet record, copied to the host on
  // a second stream while the next packet runs
  cudaStream_t cstream = nullptr;
  double* d_fr[kFrameSlots] = {};
  FrameRec* d_rec = nullptr;
  FrameRec* h_rec = nullptr;
  double* fr_host[kFrameSlots] = {};
  cudaEvent_t fr_ready[kFrameSlots] = {};
  cudaEvent_t fr_done[kFrameSlots] = {};
  cudaEvent_t pk_t0[kFrameSlots] = {};    // packet start (before its H2D), timing the frame pipeline
  int64_t pk_seq[kFrameSlots] = {-1, -1, -1, -1};  // the ticket whose start pk_t0 holds
  int64_t fr_ticket[kFrameSlots] = {-1, -1, -1, -1};
  int64_t fr_next = 0;
  int* h_err = nullptr;  // pinned error-flag read-back of evr_synchronize
  double* tgv = nullptr;  // operator API TGV planes (9 x N), allocated on first use
  std::string err;

  template <class T> T* fld(int k) const { return reinterpret_cast<T*>(slab + field_stride * k); }
  PacketHdr* hdr() const { return reinterpret_cast<PacketHdr*>(d_stage); }
  Geo geo(int ilo, int ihi) const { return Geo{W, row0, Htot, ilo, ihi}; }
  Geo geo_own() const { return geo(own_lo, own_hi); }
  // the metric also covers the halo row above (its q feeds the first row)
  Geo geo_metric() const { return geo(banded && row0 + own_lo > 0 ? own_lo - 1 : own_lo, own_hi); }
  int64_t own_off() const { return (int64_t)own_lo * W; }
  int64_t own_n() const { return (int64_t)(own_hi - own_lo + 1) * W; }
};

namespace {

int fail(evr_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return code;
}

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? EVR_ERR_OOM : EVR_ERR_CUDA,  \
                  "%s failed: %s", #call, cudaGetErrorString(e_));                    \
  } while (0)

#define CHECK_CTX()                                                   \
  do {                                                                \
    if (!ctx) return EVR_ERR_INVALID;                                 \
    cudaError_t e_ = cudaSetDevice(ctx->device);                      \
    if (e_ != cudaSuccess)                                            \
      return fail(ctx, EVR_ERR_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e_)); \
  } while (0)

inline dim3 grid2d(const evr_ctx* c) { return dim3((c->W + 31) / 32, (c->H + 7) / 8); }
inline dim3 grid_geo(const Geo& g) { return dim3((g.W + 31) / 32, (g.ihi - g.ilo + 1 + 7) / 8); }
inline dim3 block2d() { return dim3(32, 8); }
inline unsigned grid1d(int64_t n) { return (unsigned)((n + kNT - 1) / kNT); }
inline int red_blocks(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(kRedBlocks, (n + kNT - 1) / kNT));
}

int launch_err(evr_ctx* ctx, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ctx, EVR_ERR_CUDA, "%s launch: %s", what, cudaGetErrorString(e));
  return EVR_OK;
}

template <class T> CoefPlanes<T> coefs(const evr_ctx* c) {
  return CoefPlanes<T>{c->fld<T>(F_A11), c->fld<T>(F_A12), c->fld<T>(F_A22), c->fld<T>(F_A31),
                       c->fld<T>(F_A32)};
}

// ---- per-packet sequence (streaming engine) -------------------------------

// banded ordered ingest: ~2 CTAs per SM, each owning a block of own rows
void launch_ingest(evr_ctx* ctx) {
  const int nrows = ctx->own_hi - ctx->own_lo + 1;
  const int rows_per = std::max(1, (nrows + 295) / 296);
  const int nb = (nrows + rows_per - 1) / rows_per;
  const evr_config& g = ctx->cfg;
  k_ingest<kIngestNT><<<nb, kIngestNT, 0, ctx->stream>>>(
      ctx->hdr(), ctx->f + ctx->own_off(), ctx->raw + ctx->own_off(), ctx->Htot, ctx->W,
      ctx->row0 + ctx->own_lo, nrows, rows_per, g.c_pos, g.c_neg, g.u_min, g.u_max, ctx->d_err);
}

// The per-packet sequence of the streaming engine as a list of steps, one
// launch each (evr_group runs the split list on every band in lock step and
// exchanges halo rows between steps).
enum StepKind {
  ST_INGEST, ST_NORM, ST_TVD, ST_TVP, ST_TVFIN, ST_METRIC, ST_PDP, ST_REL, ST_PDD, ST_EPI,
  // fused list (whole-sensor contexts): packed state, one launch per iteration
  ST_NORMF, ST_TVF, ST_TVFINF, ST_PACK, ST_PDF, ST_RELF, ST_UNPACK,
  // whole-sensor fused list: TV-L1 end + metric + pack in one launch, the
  // final tile leaving u_{M-1}, epilogue + rel_change in one launch
  ST_MPACK, ST_PDFIN, ST_UNREL
};
struct Step {
  int kind, it;
  int buf = 0;  // fused list: packed set read (TVF, PDF, RELF) / holding the result (TVFINF, UNPACK)
  int k = 1;    // fused list: iterations per launch (1 = march kernel, > 1 = tile kernel)
};

// which: 0 = surface (ingest .. metric), 1 = solve (primal-dual + epilogue), 2 = both.
// fused: one launch per TV-L1 / primal-dual iteration (k_tv_march,
// k_pd_march) on the packed, ping-ponged state, or -- tk > 1, whole-sensor
// contexts -- tk iterations per launch (k_tv_tile, k_pd_tile; a remainder
// of 2..tk-1 iterations as one shorter tile, C3 float32 3 + 2 march launches
// -> 2 tiles); the last primal-dual iteration always runs alone, so
// rel_change sees the u of the two last iterations.  Split list (bands with EVR_GROUP_SPLIT): one launch
// per half-step with halo rows exchanged between half-steps.
std::vector<Step> packet_steps(const evr_config& g, int which, bool fused, int tk = 1,
                               bool whole = false) {
  std::vector<Step> v;
  const int D = g.denoise_iterations, M = g.max_iterations;
  tk = std::max(tk, 1);
  static const int fuse = [] {  // A/B switch of the whole-sensor fusions (bit 0 MPACK, bit 1 PDFIN/UNREL)
    const char* e = getenv("EVR_FUSE");
    return e ? atoi(e) : 3;
  }();
  if (whole && fused && which == 2 && tk > 1 && M >= 2 && g.convergence_tol <= 0 && fuse) {
    // whole-sensor packet: up to 4 launches fewer than the general list below
    v.push_back({ST_INGEST, 0});
    int b = 0;
    if (g.manifold_enabled) {
      v.push_back({ST_NORMF, 0});
      for (int k = 0; k < D;) {
        const int kk = std::min(tk, D - k);
        v.push_back({ST_TVF, k, b, kk});
        b ^= 1;
        k += kk;
      }
    }
    if (fuse & 1) {
      v.push_back({ST_MPACK, 0, b});  // b: the TV set holding the last iteration
    } else {
      if (g.manifold_enabled) v.push_back({ST_TVFINF, D, b});
      v.push_back({ST_METRIC, 0});
      v.push_back({ST_PACK, 0});
    }
    b = 0;
    if (fuse & 2) {
      for (int k = 0, rem = M; rem > 0;) {  // every launch 2..4 iterations (the built tiles)
        int kk = std::min(tk, rem);
        if (rem - kk == 1) kk = kk < 4 ? kk + 1 : kk - 1;
        v.push_back({rem == kk ? ST_PDFIN : ST_PDF, k, b, kk});
        b ^= 1;
        k += kk;
        rem -= kk;
      }
      v.push_back({ST_UNREL, M, b});
    } else {
      for (int k = 0; k < M;) {
        const int kk = std::max(1, std::min(tk, M - 1 - k));
        v.push_back({ST_PDF, k, b, kk});
        if (k == M - 1) v.push_back({ST_RELF, k, b});
        b ^= 1;
        k += kk;
      }
      v.push_back({ST_UNPACK, M, b});
    }
    return v;
  }
  if (which != 1) {
    v.push_back({ST_INGEST, 0});
    if (g.manifold_enabled) {
      v.push_back({fused ? ST_NORMF : ST_NORM, 0});
      int b = 0;
      for (int k = 0; k < D;) {
        if (fused) {
          const int kk = std::min(tk, D - k);  // the remainder as one shorter tile
          v.push_back({ST_TVF, k, b, kk});
          b ^= 1;
          k += kk;
        } else {
          v.push_back({ST_TVD, k});
          v.push_back({ST_TVP, k});
          ++k;
        }
      }
      v.push_back({fused ? ST_TVFINF : ST_TVFIN, D, b});
    }
    v.push_back({ST_METRIC, 0});
  }
  if (which != 0) {
    if (fused) v.push_back({ST_PACK, 0});
    int b = 0;
    // convergence_tol > 0 (fused list): one march launch per iteration, each
    // followed by its rel_change, all no-ops after the stop (device flag)
    const bool early = fused && g.convergence_tol > 0;
    for (int k = 0; k < M;) {
      if (fused) {
        const int kk = early ? 1 : std::max(1, std::min(tk, M - 1 - k));
        v.push_back({ST_PDF, k, b, kk});
        if (k == M - 1 || early) v.push_back({ST_RELF, k, b});
        b ^= 1;
        k += kk;
      } else {
        v.push_back({ST_PDP, k});
        if (k == M - 1) v.push_back({ST_REL, k});
        v.push_back({ST_PDD, k});
        ++k;
      }
    }
    v.push_back({fused ? ST_UNPACK : ST_EPI, M, b});
  }
  return v;
}

// temporal blocking of the whole-sensor fused list: iterations per tile
// launch (EVR_TILE_K overrides; 1 = one march launch per iteration).
// Measured on B200 (tools/tilerun.sh, tools/f64run.sh), K = 4: float32 C3
// 0.94 -> 0.72 ms, C4 0.38 -> 0.23, C5 3.2 -> 1.9; float64 C3 2.84 -> 2.27,
// C4 0.66 -> 0.57.
int env_tile_k() {
  static const int env = [] {
    const char* e = getenv("EVR_TILE_K");
    if (!e) return 0;
    const int v = atoi(e);
    return v >= 1 && v <= 4 ? v : 1;
  }();
  return env;
}
bool env_tile_k_set() { return env_tile_k() > 0; }
int tile_k(int prec) {
  (void)prec;
  return env_tile_k() ? env_tile_k() : 4;
}

// fused iterations: rows per warp strip (RY), rows of loads in flight ahead
// of the arithmetic (D, the register budget), threads per CTA; measured on
// B200 at 640x480 .. 2048x2048 (tools/sweep_march.sh)
#ifndef EVR_MARCH_RY
#define EVR_MARCH_RY 4
#endif
#ifndef EVR_MARCH_D32
#define EVR_MARCH_D32 4
#endif
#ifndef EVR_MARCH_D64
#define EVR_MARCH_D64 1
#endif
constexpr int kMarchRY = EVR_MARCH_RY, kMarchNT = 128;
template <class T> struct MarchDepth { static constexpr int tv = EVR_MARCH_D32, pd = EVR_MARCH_D32; };
template <> struct MarchDepth<double> { static constexpr int tv = EVR_MARCH_D64, pd = EVR_MARCH_D64; };
inline unsigned march_grid(const evr_ctx* c) {
  const int rows = c->own_hi - c->own_lo + 1;
  const int64_t warps = (int64_t)((c->W + kStrip - 1) / kStrip) * ((rows + kMarchRY - 1) / kMarchRY);
  return (unsigned)((warps + kMarchNT / 32 - 1) / (kMarchNT / 32));
}

// packed state of the fused list: TV {u, u_bar, px, py} x 2, solver
// {p1, p2, p3, u} x 2, then the solver constants (1 quad per pixel for
// float, 2 for double)
template <class T> struct Packed {
  Q4<T>* tv[2];
  Q4<T>* pd[2];
  Q4<T>* cst;
};
template <class T> Packed<T> packed(const evr_ctx* c) {
  Q4<T>* b = reinterpret_cast<Q4<T>*>(c->d_pack);
  const int64_t N = c->N;
  return Packed<T>{{b, b + N}, {b + 2 * N, b + 3 * N}, b + 4 * N};
}
inline size_t packed_bytes(int64_t N, int prec) {
  return prec == EVR_PREC_F64 ? (size_t)N * 6 * 32 : (size_t)N * 5 * 16;
}

// row sources of a fused iteration: `buf` maps a context to the packed
// buffer read (the same one in the neighbours), E quads per pixel
template <class Q, class Buf>
MarchRows<Q> march_rows(const evr_ctx* c, Buf buf, int E) {
  MarchRows<Q> r;
  r.own = buf(c);
  r.y0 = c->row0 + c->own_lo;
  r.y1 = c->row0 + c->own_hi + 1;
  r.olo = c->own_lo;
  r.E = E;
  r.up = c->nb_up ? buf(c->nb_up) + (int64_t)c->nb_up->own_hi * c->W * E : nullptr;
  r.dn = c->nb_dn ? buf(c->nb_dn) + (int64_t)c->nb_dn->own_lo * c->W * E : nullptr;
  return r;
}

template <class T> CoefPlanes<T> coefs(const evr_ctx* c);

// iteration kernels go out with programmatic stream serialization (PDL,
// see pdl_wait_and_release); EVR_PDL=0 turns it off for A/B timing
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("EVR_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
template <class... KArgs, class... Args>
void launch_pdl(void (*k)(KArgs...), unsigned grid, unsigned block, cudaStream_t s,
                Args&&... args) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(block);
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&lc, k, std::forward<Args>(args)...);
}

template <class T>
void relchange(evr_ctx* ctx, const T* un, const T* u, int iterations, int stride = 1,
               bool early_stop = false, double* hist = nullptr) {
  const int nb = red_blocks(ctx->own_n());
  launch_pdl(k_relchange<T, kNT>, nb, kNT, ctx->stream, un + ctx->own_off() * stride,
             u + ctx->own_off() * stride, ctx->own_n(), ctx->part, stride, ctx->rticket,
             ctx->d_info, iterations, ctx->d_scalar + 2, early_stop ? ctx->cfg.convergence_tol : 0.0,
             early_stop ? ctx->d_stop : nullptr, hist);
}

// temporally blocked tiles (evr_tile.cuh): a CTA of G warps covers 32 x
// G*RPT region pixels and keeps the (32 - 2K) x (G*RPT - 2K) interior
#ifndef EVR_TILE32_RPT
#define EVR_TILE32_RPT 8
#endif
#ifndef EVR_TILE32_G
#define EVR_TILE32_G 8
#endif
#ifndef EVR_TILE32_MINB
#define EVR_TILE32_MINB 2
#endif
#ifndef EVR_TILE64_RPT
#define EVR_TILE64_RPT 3  // 3 rows per thread: no spills at 126 registers (C3 f64 k_pd_tile 45.5 -> 43.4 us)
#endif
#ifndef EVR_TILE64_G
#define EVR_TILE64_G 8
#endif
#ifndef EVR_TILE64_MINB
#define EVR_TILE64_MINB 2  // 2 CTAs per SM (<= 128 registers): C3 f64 2.84 -> 2.27 ms
#endif
template <class T> struct TileShape;
template <> struct TileShape<float> {
  static constexpr int RPT = EVR_TILE32_RPT, G = EVR_TILE32_G, MINB = EVR_TILE32_MINB;
};
template <> struct TileShape<double> {
  static constexpr int RPT = EVR_TILE64_RPT, G = EVR_TILE64_G, MINB = EVR_TILE64_MINB;
};
// Rows per thread of a context's tiles: the float kernels come in RPT = 8,
// 7, 6 (regions of 64, 56, 48 rows); the one whose whole waves (MINB CTAs
// per SM) cover the sensor with the fewest region rows per SM wins -- e.g.
// 1280x720, K = 4: RPT 8 -> 702 tiles = 2.4 waves rounded to 3, RPT 7 ->
// 810 tiles = 2.7 waves, 12 % fewer rows computed per SM.
int sm_count(int device) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return sms;
}
// whole waves x region rows of one launch shape (the model both choices use)
template <class T> int64_t tile_cost(const evr_ctx* c, int K, int rpt) {
  constexpr int G = TileShape<T>::G;
  const int64_t slots = (int64_t)sm_count(c->device) * TileShape<T>::MINB;
  const int tiw = 32 - 2 * K, tih = G * rpt - 2 * K;
  const int64_t ctas = (int64_t)((c->W + tiw - 1) / tiw) * ((c->own_hi - c->own_lo + tih) / tih);
  return (ctas + slots - 1) / slots * (G * rpt);
}
template <class T> int tile_rpt(const evr_ctx* c, int K) {
  if (!std::is_same<T, float>::value || TileShape<T>::RPT != 8) return TileShape<T>::RPT;
  int best = 8;
  int64_t best_cost = -1;
  for (int rpt = 8; rpt >= 6; --rpt) {
    const int64_t cost = tile_cost<T>(c, K, rpt);
    if (best_cost < 0 || cost < best_cost) best = rpt, best_cost = cost;
  }
  return best;
}
// Iterations per tile launch when neither EVR_TILE_K nor evr_set_tile_k
// fixes it: a launch of K iterations costs K x its waves, so the time per
// iteration goes with the waves of the K's best shape; ties go to the larger
// K (fewer HBM round trips).  Measured float64: 1280x720 K=3 1.82 ms vs K=4
// 1.86 (4.7 vs 5.5 waves), 2048^2 4.71 vs 4.92, 640x480 K=4 0.455 vs 0.481.
template <class T> int auto_tile_k(const evr_ctx* c) {
  int best = 4;
  int64_t best_cost = -1;
  for (int K = 4; K >= 3; --K) {
    const int64_t cost = tile_cost<T>(c, K, tile_rpt<T>(c, K));
    if (best_cost < 0 || cost < best_cost) best = K, best_cost = cost;
  }
  return best;
}
int ctx_tile_k(const evr_ctx* c) {
  if (c->tile_k > 0) return c->tile_k;
  if (env_tile_k_set()) return env_tile_k();
  // float32 tiles are cheap enough per iteration that the 1/K share of
  // memory traffic decides: K = 4 measured best on C3-C5 (2048^2: 1.59 ms vs
  // 1.64 at K = 3 although K = 3 needs fewer waves)
  return c->prec == EVR_PREC_F64 ? auto_tile_k<double>(c) : 4;
}
template <class T, int K, int RPT> dim3 tile_grid(const evr_ctx* c) {
  constexpr int TIW = 32 - 2 * K, TIH = TileShape<T>::G * RPT - 2 * K;
  const int rows = c->own_hi - c->own_lo + 1;
  return dim3((c->W + TIW - 1) / TIW, (rows + TIH - 1) / TIH);
}
template <class... KArgs, class... Args>
void launch_pdl2(void (*k)(KArgs...), dim3 grid, unsigned block, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = grid;
  lc.blockDim = dim3(block);
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&lc, k, std::forward<Args>(args)...);
}
template <class T, int RPT, bool B>
void tv_tile_rpt(evr_ctx* ctx, int K, const MarchRows<Q4<T>>& in, const MarchRows<T>& f0,
                 Q4<T>* out, T sigma, T tau, T shrink, int early) {
  constexpr int G = TileShape<T>::G, MB = TileShape<T>::MINB;
  const int H = ctx->Htot, W = ctx->W;
  cudaStream_t s = ctx->stream;
  if (K == 2)
    launch_pdl2(k_tv_tile<T, 2, RPT, G, MB, B>, tile_grid<T, 2, RPT>(ctx), 32 * G, s, in, f0, out,
                H, W, sigma, tau, shrink, early);
  else if (K == 3)
    launch_pdl2(k_tv_tile<T, 3, RPT, G, MB, B>, tile_grid<T, 3, RPT>(ctx), 32 * G, s, in, f0, out,
                H, W, sigma, tau, shrink, early);
  else
    launch_pdl2(k_tv_tile<T, 4, RPT, G, MB, B>, tile_grid<T, 4, RPT>(ctx), 32 * G, s, in, f0, out,
                H, W, sigma, tau, shrink, early);
}
template <class T, bool B>
void tv_tile_shape(evr_ctx* ctx, int K, const MarchRows<Q4<T>>& in, const MarchRows<T>& f0,
                   Q4<T>* out, T sigma, T tau, T shrink, int early) {
  constexpr int R0 = TileShape<T>::RPT;
  const int rpt = tile_rpt<T>(ctx, K);
  if constexpr (std::is_same<T, float>::value && R0 == 8) {
    if (rpt == 7) return tv_tile_rpt<T, 7, B>(ctx, K, in, f0, out, sigma, tau, shrink, early);
    if (rpt == 6) return tv_tile_rpt<T, 6, B>(ctx, K, in, f0, out, sigma, tau, shrink, early);
  }
  tv_tile_rpt<T, R0, B>(ctx, K, in, f0, out, sigma, tau, shrink, early);
}
template <class T>
int launch_tv_tile(evr_ctx* ctx, int K, const MarchRows<Q4<T>>& in, const MarchRows<T>& f0,
                   Q4<T>* out, T sigma, T tau, T shrink, int early) {
  if (ctx->banded)
    tv_tile_shape<T, true>(ctx, K, in, f0, out, sigma, tau, shrink, 0);
  else
    tv_tile_shape<T, false>(ctx, K, in, f0, out, sigma, tau, shrink, early);
  return 1;
}
// Clustered primal-dual tiles (k_pd_tile<..., CX, CY>): EVR_TILE_CLUSTER
// = "CXxCY" (2x2, 4x2, 2x4; unset or 1x1 = the one-CTA regions).
int env_tile_cluster() {
  static const int env = [] {
    const char* e = getenv("EVR_TILE_CLUSTER");
    if (!e) return 0;
    if (!strcmp(e, "2x2")) return 22;
    if (!strcmp(e, "4x2")) return 42;
    if (!strcmp(e, "2x4")) return 24;
    return 0;
  }();
  return env;
}
template <class... KArgs, class... Args>
void launch_cluster(void (*k)(KArgs...), dim3 grid, unsigned block, int cx, int cy,
                    cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = grid;
  lc.blockDim = dim3(block);
  lc.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cx;
  at[0].val.clusterDim.y = cy;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = pdl_enabled() ? 2 : 1;
  cudaLaunchKernelEx(&lc, k, std::forward<Args>(args)...);
}
// TMA region loads (k_pd_tile with MetricPackF64Tma): EVR_TILE_TMA=1
bool env_tile_tma() {
  static const bool env = [] {
    const char* e = getenv("EVR_TILE_TMA");
    return e && atoi(e) != 0;
  }();
  return env;
}
// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
using TmaEncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
TmaEncodeFn tma_encode_fn() {
  static TmaEncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess || q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<TmaEncodeFn>(p);
  }();
  return fn;
}
// a whole-sensor plane of `per_px` doubles per pixel as a 2-D tensor, boxes
// of RH rows x 32 pixels
bool tma_plane(CUtensorMap* tm, const void* base, int W, int H, int per_px, int RH) {
  const TmaEncodeFn fn = tma_encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)per_px * W, (cuuint64_t)H};
  const cuuint64_t strides[1] = {(cuuint64_t)per_px * W * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)(32 * per_px), (cuuint32_t)RH};
  const cuuint32_t estr[2] = {1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
template <class... KArgs, class... Args>
void launch_pdl_smem(void (*k)(KArgs...), dim3 grid, unsigned block, size_t smem, cudaStream_t s,
                     Args&&... args) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = grid;
  lc.blockDim = dim3(block);
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&lc, k, std::forward<Args>(args)...);
}
template <int K, int RPT>
bool pd_tile_tma(evr_ctx* ctx, const MarchRows<Q4<double>>& in, const MetricPackF64& m,
                 Q4<double>* out, double tau, double sigma, double lo, double hi, int early,
                 double* prev) {
  constexpr int G = TileShape<double>::G, MB = TileShape<double>::MINB, RH = G * RPT;
  if (ctx->banded) return false;
  MetricPackF64Tma mt;
  static_cast<MetricPackF64&>(mt) = m;
  if (!tma_plane(&mt.tc, m.c, ctx->W, ctx->Htot, 8, RH) ||
      !tma_plane(&mt.ts, in.own, ctx->W, ctx->Htot, 4, RH))
    return false;
  constexpr size_t smem = (size_t)RH * 32 * 3 * sizeof(Q4<double>);
  auto k = prev ? k_pd_tile<double, K, RPT, G, MB, MetricPackF64Tma, false, DT_KL, true>
                : k_pd_tile<double, K, RPT, G, MB, MetricPackF64Tma, false, DT_KL, false>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);  // two CTAs' boxes per SM
  launch_pdl_smem(k, tile_grid<double, K, RPT>(ctx), 32 * G, smem, ctx->stream, in, mt, out,
                  ctx->Htot, ctx->W, tau, sigma, lo, hi, early, prev);
  return true;
}
template <class T, int K, int RPT, int CX, int CY, class M>
void pd_tile_cl(evr_ctx* ctx, const MarchRows<Q4<T>>& in, const M& m, Q4<T>* out, T tau,
                T sigma, T lo, T hi, int early, T* prev) {
  constexpr int G = TileShape<T>::G, MB = TileShape<T>::MINB;
  constexpr int TIW = 32 * CX - 2 * K, TIH = G * RPT * CY - 2 * K;
  const int rows = ctx->own_hi - ctx->own_lo + 1;
  const dim3 grid(CX * ((ctx->W + TIW - 1) / TIW), CY * ((rows + TIH - 1) / TIH));
  launch_cluster(prev ? k_pd_tile<T, K, RPT, G, MB, M, false, DT_KL, true, CX, CY>
                      : k_pd_tile<T, K, RPT, G, MB, M, false, DT_KL, false, CX, CY>,
                 grid, 32 * G, CX, CY, ctx->stream, in, m, out, ctx->Htot, ctx->W, tau, sigma, lo,
                 hi, early, prev);
}
template <class T, int K, int RPT, class M>
bool pd_tile_cluster(evr_ctx* ctx, int shape, const MarchRows<Q4<T>>& in, const M& m,
                     Q4<T>* out, T tau, T sigma, T lo, T hi, int early, T* prev) {
  if (shape == 22) pd_tile_cl<T, K, RPT, 2, 2>(ctx, in, m, out, tau, sigma, lo, hi, early, prev);
  else if (shape == 42) pd_tile_cl<T, K, RPT, 4, 2>(ctx, in, m, out, tau, sigma, lo, hi, early, prev);
  else if (shape == 24) pd_tile_cl<T, K, RPT, 2, 4>(ctx, in, m, out, tau, sigma, lo, hi, early, prev);
  else return false;
  return true;
}
// step: tau = sigma for operator solves (no context config); < 0 = the config's
template <class T, int RPT, bool B, class M, int DT = DT_KL>
void pd_tile_rpt(evr_ctx* ctx, int K, const MarchRows<Q4<T>>& in, const M& m, Q4<T>* out,
                 double step = -1.0, int early = 0, T* prev = nullptr) {
  constexpr int G = TileShape<T>::G, MB = TileShape<T>::MINB;
  const evr_config& g = ctx->cfg;
  const int H = ctx->Htot, W = ctx->W;
  cudaStream_t s = ctx->stream;
  const T tau = (T)(step < 0 ? g.tau : step), sigma = (T)(step < 0 ? g.sigma : step);
  const T lo = (T)g.u_min, hi = (T)g.u_max;
  if constexpr (!B && DT == DT_KL && std::is_same<M, MetricPackF64>::value) {
    if (env_tile_tma() && !env_tile_cluster()) {
      if (K == 3 && pd_tile_tma<3, RPT>(ctx, in, m, out, tau, sigma, lo, hi, early, prev)) return;
      if (K == 4 && pd_tile_tma<4, RPT>(ctx, in, m, out, tau, sigma, lo, hi, early, prev)) return;
    }
  }
  if constexpr (!B && DT == DT_KL && std::is_same<T, double>::value) {
    const int cl = env_tile_cluster();
    if (cl && K == 3 && pd_tile_cluster<T, 3, RPT>(ctx, cl, in, m, out, tau, sigma, lo, hi, early, prev))
      return;
    if (cl && K == 4 && pd_tile_cluster<T, 4, RPT>(ctx, cl, in, m, out, tau, sigma, lo, hi, early, prev))
      return;
  }
  if (K == 2)
    launch_pdl2(prev ? k_pd_tile<T, 2, RPT, G, MB, M, B, DT, !B> : k_pd_tile<T, 2, RPT, G, MB, M, B, DT>,
                tile_grid<T, 2, RPT>(ctx), 32 * G, s, in, m, out, H, W, tau, sigma, lo, hi, early,
                prev);
  else if (K == 3)
    launch_pdl2(prev ? k_pd_tile<T, 3, RPT, G, MB, M, B, DT, !B> : k_pd_tile<T, 3, RPT, G, MB, M, B, DT>,
                tile_grid<T, 3, RPT>(ctx), 32 * G, s, in, m, out, H, W, tau, sigma, lo, hi, early,
                prev);
  else
    launch_pdl2(prev ? k_pd_tile<T, 4, RPT, G, MB, M, B, DT, !B> : k_pd_tile<T, 4, RPT, G, MB, M, B, DT>,
                tile_grid<T, 4, RPT>(ctx), 32 * G, s, in, m, out, H, W, tau, sigma, lo, hi, early,
                prev);
}
template <class T, bool B, class M>
void pd_tile_shape(evr_ctx* ctx, int K, const MarchRows<Q4<T>>& in, const M& m, Q4<T>* out,
                   int early, T* prev = nullptr) {
  constexpr int R0 = TileShape<T>::RPT;
  const int rpt = tile_rpt<T>(ctx, K);
  if constexpr (std::is_same<T, float>::value && R0 == 8) {
    if (rpt == 7) return pd_tile_rpt<T, 7, B>(ctx, K, in, m, out, -1.0, early, prev);
    if (rpt == 6) return pd_tile_rpt<T, 6, B>(ctx, K, in, m, out, -1.0, early, prev);
  }
  pd_tile_rpt<T, R0, B>(ctx, K, in, m, out, -1.0, early, prev);
}
template <class T, class M>
int launch_pd_tile(evr_ctx* ctx, int K, const MarchRows<Q4<T>>& in, const M& m, Q4<T>* out,
                   int early, T* prev = nullptr) {
  if (ctx->banded)
    pd_tile_shape<T, true>(ctx, K, in, m, out, 0);
  else
    pd_tile_shape<T, false>(ctx, K, in, m, out, early, prev);
  return 1;
}

// launches of one step (returns the kernel count)
template <class T> int launch_step(evr_ctx* ctx, const Step& st) {
  const evr_config& g = ctx->cfg;
  cudaStream_t s = ctx->stream;
  const Geo own = ctx->geo_own();
  const int64_t off = ctx->own_off(), n = ctx->own_n();
  const double step = 1.0 / std::sqrt(8.0);  // surface.py:158
  T *t = ctx->fld<T>(F_T), *tu = ctx->fld<T>(F_TU), *tub = ctx->fld<T>(F_TUB);
  T *px = ctx->fld<T>(F_TPX), *py = ctx->fld<T>(F_TPY);
  T* bufs[2] = {ctx->fld<T>(F_U), ctx->fld<T>(F_UN)};
  switch (st.kind) {
    case ST_INGEST:
      launch_ingest(ctx);
      return 1;
    case ST_NORM:
      k_normalize_tvinit<T><<<grid1d(n), kNT, 0, s>>>(ctx->raw + off, ctx->hdr(), g.t_scale,
                                                      t + off, tu + off, tub + off, px + off,
                                                      py + off, n);
      return 1;
    case ST_TVD:
      k_tv_dual<T><<<grid_geo(own), block2d(), 0, s>>>(tub, px, py, own, (T)step);
      return 1;
    case ST_TVP:
      k_tv_primal<T><<<grid_geo(own), block2d(), 0, s>>>(px, py, tu, tub, t, own, (T)step,
                                                         (T)(step * g.denoise_weight));
      return 1;
    case ST_TVFIN:
      k_tv_finish<T><<<grid1d(n), kNT, 0, s>>>(tu + off, t + off, (T)g.t_scale, n);
      return 1;
    case ST_METRIC: {
      const Geo mg = ctx->geo_metric();
      k_metric_setup<T><<<grid_geo(mg), block2d(), 0, s>>>(
          t, ctx->f, ctx->fld<T>(F_TX), ctx->fld<T>(F_TY), ctx->fld<T>(F_G), ctx->fld<T>(F_SG),
          coefs<T>(ctx), ctx->fld<T>(F_BETA), ctx->fld<T>(F_FB), mg, (T)(g.tau * g.lam),
          g.manifold_enabled ? 0 : 1);
      return 1;
    }
    case ST_PDP:
      k_pd_primal<T><<<grid_geo(own), block2d(), 0, s>>>(
          ctx->fld<T>(F_P1), ctx->fld<T>(F_P2), ctx->fld<T>(F_P3), coefs<T>(ctx),
          bufs[st.it & 1], ctx->fld<T>(F_BETA), ctx->fld<T>(F_FB), bufs[(st.it + 1) & 1],
          ctx->fld<T>(F_V), own, (T)g.tau, (T)g.u_min, (T)g.u_max);
      return 1;
    case ST_REL:
      relchange<T>(ctx, bufs[(st.it + 1) & 1], bufs[st.it & 1], st.it + 1);
      return 1;
    case ST_PDD:
      k_pd_dual<T><<<grid_geo(own), block2d(), 0, s>>>(
          ctx->fld<T>(F_V), ctx->fld<T>(F_P1), ctx->fld<T>(F_P2), ctx->fld<T>(F_P3),
          coefs<T>(ctx), ctx->fld<T>(F_SG), own, (T)g.sigma);
      return 1;
    case ST_EPI: {
      T* last = bufs[g.max_iterations & 1];
      k_epilogue<T><<<grid1d(n), kNT, 0, s>>>(last + off, ctx->fld<T>(F_U) + off, ctx->f + off, n);
      return 1;
    }
    // ---- fused list (whole-sensor context: off = 0, n = N)
    case ST_NORMF:  // own rows; a band's halo rows come from its neighbours
      k_normalize_pack<T><<<grid1d(n), kNT, 0, s>>>(ctx->raw + off, ctx->hdr(), g.t_scale, t + off,
                                                    packed<T>(ctx).tv[0] + off, n);
      return 1;
    case ST_TVF: {  // reads set st.buf, writes the other
      const int a = st.buf;
      const auto in = march_rows<Q4<T>>(ctx, [a](const evr_ctx* c) { return packed<T>(c).tv[a]; }, 1);
      Q4<T>* out = packed<T>(ctx).tv[a ^ 1];
      const T sh = (T)(step * g.denoise_weight);
      if (st.k > 1) {
        const auto f0 = march_rows<T>(ctx, [](const evr_ctx* c) { return c->fld<T>(F_T); }, 1);
        return launch_tv_tile<T>(ctx, st.k, in, f0, out, (T)step, (T)step, sh, st.it > 0 ? 1 : 0);
      }
      if (ctx->banded)
        launch_pdl(k_tv_march<T, kMarchRY, MarchDepth<T>::tv, true>, march_grid(ctx), kMarchNT, s,
                   in.own, in, (const T*)t, out, ctx->Htot, ctx->W, (T)step, (T)step, sh);
      else
        launch_pdl(k_tv_march<T, kMarchRY, MarchDepth<T>::tv, false>, march_grid(ctx), kMarchNT, s,
                   in.own, in, (const T*)t, out, ctx->Htot, ctx->W, (T)step, (T)step, sh);
      return 1;
    }
    case ST_TVFINF:  // st.buf = the set holding the last iteration
      k_tv_finish_packed<T><<<grid1d(n), kNT, 0, s>>>(packed<T>(ctx).tv[st.buf] + off, t + off,
                                                      (T)g.t_scale, n);
      return 1;
    case ST_PACK: {
      const Packed<T> P = packed<T>(ctx);
      if (g.convergence_tol > 0) CK(cudaMemsetAsync(ctx->d_stop, 0, sizeof(int), s));
      constexpr int E = sizeof(T) == 8 ? 2 : 1;
      k_pack_solver<T><<<grid1d(n), kNT, 0, s>>>(
          ctx->fld<T>(F_P1) + off, ctx->fld<T>(F_P2) + off, ctx->fld<T>(F_P3) + off,
          ctx->fld<T>(F_U) + off, ctx->fld<T>(F_TX) + off, ctx->fld<T>(F_TY) + off,
          CoefPlanes<T>{ctx->fld<T>(F_A11) + off, ctx->fld<T>(F_A12) + off,
                        ctx->fld<T>(F_A22) + off, ctx->fld<T>(F_A31) + off,
                        ctx->fld<T>(F_A32) + off},
          ctx->fld<T>(F_SG) + off, ctx->fld<T>(F_BETA) + off, ctx->fld<T>(F_FB) + off,
          P.pd[0] + off, P.cst + off * E, n);
      return 1;
    }
    case ST_PDF:
    case ST_PDFIN: {
      const int a = st.buf;
      constexpr int E = sizeof(T) == 8 ? 2 : 1;
      using M = typename MetricPack<T>::type;
      const auto in = march_rows<Q4<T>>(ctx, [a](const evr_ctx* c) { return packed<T>(c).pd[a]; }, 1);
      const auto cr = march_rows<Q4<T>>(ctx, [](const evr_ctx* c) { return packed<T>(c).cst; }, E);
      M m;
      if constexpr (std::is_same<T, float>::value)
        m = M{cr.own, cr, (float)(g.tau * g.lam)};
      else
        m = M{cr.own, cr};
      Q4<T>* out = packed<T>(ctx).pd[a ^ 1];
      // not the first iteration launch after the pack: constants loaded early
      if (st.k > 1)
        return launch_pd_tile<T>(ctx, st.k, in, m, out, st.it > 0 ? 1 : 0,
                                 st.kind == ST_PDFIN ? ctx->fld<T>(F_UN) : (T*)nullptr);
      if (ctx->banded)
        launch_pdl(k_pd_march<T, kMarchRY, MarchDepth<T>::pd, M, true>, march_grid(ctx), kMarchNT,
                   s, in.own, in, m, out, ctx->Htot, ctx->W, (T)g.tau, (T)g.sigma, (T)g.u_min,
                   (T)g.u_max, (const int*)nullptr);
      else
        launch_pdl(k_pd_march<T, kMarchRY, MarchDepth<T>::pd, M, false>, march_grid(ctx), kMarchNT,
                   s, in.own, in, m, out, ctx->Htot, ctx->W, (T)g.tau, (T)g.sigma, (T)g.u_min,
                   (T)g.u_max, (const int*)(g.convergence_tol > 0 ? ctx->d_stop : nullptr));
      return 1;
    }
    case ST_MPACK: {  // st.buf: the TV set holding the last iteration
      const Packed<T> P = packed<T>(ctx);
      k_metric_pack<T><<<grid2d(ctx), block2d(), 0, s>>>(
          P.tv[st.buf], ctx->f, ctx->fld<T>(F_P1), ctx->fld<T>(F_P2), ctx->fld<T>(F_P3),
          ctx->fld<T>(F_U), t, ctx->fld<T>(F_TX), ctx->fld<T>(F_TY), ctx->fld<T>(F_G),
          ctx->fld<T>(F_SG), P.pd[0], P.cst, ctx->H, ctx->W, (T)g.t_scale, (T)(g.tau * g.lam),
          g.manifold_enabled ? 0 : 1);
      return 1;
    }
    case ST_UNREL: {  // st.buf: the set holding the last iteration, F_UN: u_{M-1}
      const Packed<T> P = packed<T>(ctx);
      launch_pdl(k_unpack_rel<T, kNT>, red_blocks(n), kNT, s, (const Q4<T>*)P.pd[st.buf],
                 (const T*)ctx->fld<T>(F_UN), ctx->fld<T>(F_P1), ctx->fld<T>(F_P2),
                 ctx->fld<T>(F_P3), ctx->fld<T>(F_U), ctx->f, n, ctx->part, ctx->rticket,
                 ctx->d_info, st.it);
      return 1;
    }
    case ST_RELF: {  // u of the last two iterations, the w of the packed quads
      const Packed<T> P = packed<T>(ctx);
      relchange<T>(ctx, &P.pd[st.buf ^ 1]->w, &P.pd[st.buf]->w, st.it + 1, 4,
                   g.convergence_tol > 0 && !ctx->banded);
      return 1;
    }
    case ST_UNPACK:  // st.buf = the set holding the last iteration
      if (g.convergence_tol > 0)  // the set of the last executed iteration (device count)
        k_unpack_solver<T><<<grid1d(n), kNT, 0, s>>>(
            packed<T>(ctx).pd[0] + off, ctx->fld<T>(F_P1) + off, ctx->fld<T>(F_P2) + off,
            ctx->fld<T>(F_P3) + off, ctx->fld<T>(F_U) + off, ctx->f + off, n,
            packed<T>(ctx).pd[1] + off, ctx->d_info);
      else
        k_unpack_solver<T><<<grid1d(n), kNT, 0, s>>>(packed<T>(ctx).pd[st.buf] + off,
                                                     ctx->fld<T>(F_P1) + off, ctx->fld<T>(F_P2) + off,
                                                     ctx->fld<T>(F_P3) + off, ctx->fld<T>(F_U) + off,
                                                     ctx->f + off, n);
      return 1;
  }
  return 0;
}

template <class T> int enqueue_packet(evr_ctx* ctx, int which) {
  int n = 0;
  const int tk = ctx->banded ? 1 : ctx_tile_k(ctx);
  for (const Step& st : packet_steps(ctx->cfg, which, !ctx->banded, tk, !ctx->banded))
    n += launch_step<T>(ctx, st);
  int rc = launch_err(ctx, "packet");
  return rc ? rc : n;
}

// ---- resident engine glue ---------------------------------------------------

// Instantiated shapes of k_resident: threads per CTA (a thread per sensor
// column when W <= NT), CH = 2 rows per register chunk, and where the CTA's
// frame of planes lives (shared memory, else a global-memory slice).
constexpr int kResidentCH = 2;
constexpr int kAutoResidentRows = 2;  // AUTO: resident while rows per CTA <= this
template <class T> struct ResidentKernel {
  int nt, ms;
  void (*fn)(ResArgs<T>);
};
template <class T> const ResidentKernel<T>* resident_pick(int W, int ms) {
  static const ResidentKernel<T> table[] = {
      {128, PLANES_SMEM, k_resident<T, 128, kResidentCH, PLANES_SMEM>},
      {384, PLANES_SMEM, k_resident<T, 384, kResidentCH, PLANES_SMEM>},
      {512, PLANES_SMEM, k_resident<T, 512, kResidentCH, PLANES_SMEM>},
  };
  const int nt = W <= 128 ? 128 : W <= 384 ? 384 : 512;
  for (const auto& k : table)
    if (k.nt == nt && k.ms == ms) return &k;
  return nullptr;
}

// column-per-thread variant (evr_resident_col.cuh): W <= NT, bands of RB rows
template <class T> struct ResidentColKernel {
  int nt, rb;
  void (*fn)(ResArgs<T>);
};
template <class T> const ResidentColKernel<T>* resident_col_pick(int W, int R) {
  static const ResidentColKernel<T> table[] = {
      {128, 1, k_resident_col<T, 128, 1>}, {128, 2, k_resident_col<T, 128, 2>},
      {256, 1, k_resident_col<T, 256, 1>}, {256, 2, k_resident_col<T, 256, 2>},
      {352, 1, k_resident_col<T, 352, 1>}, {352, 2, k_resident_col<T, 352, 2>},  // 346 wide
      {384, 1, k_resident_col<T, 384, 1>}, {384, 2, k_resident_col<T, 384, 2>},
      {512, 1, k_resident_col<T, 512, 1>}, {512, 2, k_resident_col<T, 512, 2>},
  };
  static const bool off = [] {
    const char* e = getenv("EVR_RESIDENT_COL");
    return e && e[0] == '0';
  }();
  if (off) return nullptr;
  for (const auto& k : table)
    if (W <= k.nt && R == k.rb) return &k;
  return nullptr;
}

// Band decomposition: one CTA per SM at most, equal band heights R: the
// column-per-thread kernel when W <= 512, else the plane-frame kernel with
// its frame in shared memory (nothing else: an engine that does not fit
// hands the sensor to the streaming list).
template <class T> bool resident_plan(evr_ctx* ctx) {
  int sms = 0, optin = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device) != cudaSuccess ||
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device) !=
          cudaSuccess)
    return false;
  const int H = ctx->H, W = ctx->W;
  const int R = (H + std::min(H, sms) - 1) / std::min(H, sms);
  const int nb = (H + R - 1) / R;
  const size_t frame = resident_frame_bytes<T>(R, W);
  const int nt = W <= 128 ? 128 : W <= 384 ? 384 : 512;
  const size_t static_smem = sizeof(IngestShared<512>) + 64 * sizeof(double) + 64;
  const bool smem_fits = frame + static_smem + 1024 <= (size_t)optin;
  const ResidentColKernel<T>* ck = resident_col_pick<T>(W, R);
  const size_t csmem = resident_col_smem<T>(R, W);
  int ms, nt_used = nt;
  size_t smem;
  if (ck && csmem + sizeof(IngestShared<512>) + 64 * sizeof(double) + 1024 <= (size_t)optin) {
    ms = PLANES_COL;
    smem = csmem;
    nt_used = ck->nt;
  } else if (smem_fits) {
    ms = PLANES_SMEM;
    smem = frame;
  } else {
    return false;
  }
  ctx->r_nb = nb;
  ctx->r_R = R;
  ctx->r_nt = nt_used;
  ctx->r_ms = ms;
  ctx->r_smem = smem;
  ctx->r_frame = frame;
  return true;
}

// Band order by SM: the block scheduler spreads a one-CTA-per-SM grid over
// the GPCs (blockIdx 0, 1, 2, ... -> SM 144, 145, 146, 147, 142, 143, 0, 1,
// 16, 17, ...), so consecutive bands -- the pairs that exchange halo rows
// every iteration -- would sit on distant SMs.  A probe grid of the same
// shape (one CTA per SM) records where each blockIdx lands; band b then goes
// to the CTA on the b-th lowest SM id.  Any permutation is correct (every
// index in the kernel is the band's); this one only shortens the halo paths
// when the placement repeats.  Measured (same box): C2 f64 0.2276 ->
// 0.2359 ms, C1 0.152 -> 0.160 -- neighbouring SMs (same TPC) hand off
// slower than the scheduler's spread -- so it is off unless EVR_SM_ORDER=1.
__global__ void k_smid_probe(int* out) {
  extern __shared__ unsigned char probe_smem[];
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    out[blockIdx.x] = (int)smid;
    probe_smem[0] = 0;
  }
}
bool sm_order_enabled() {
  static const bool on = [] {
    const char* e = getenv("EVR_SM_ORDER");
    return e && e[0] == '1';
  }();
  return on;
}
int resident_sm_order(evr_ctx* ctx) {
  const int nb = ctx->r_nb;
  int optin = 0;
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  const int smem = std::max((int)ctx->r_smem, optin / 2 + 1024);  // one probe CTA per SM
  CK(cudaFuncSetAttribute(k_smid_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaMalloc(&ctx->d_perm, sizeof(int) * nb));
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(nb);
  lc.blockDim = dim3(ctx->r_nt);
  lc.dynamicSmemBytes = smem;
  lc.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  CK(cudaLaunchKernelEx(&lc, k_smid_probe, ctx->d_perm));
  std::vector<int> sm(nb), order(nb), perm(nb);
  CK(cudaMemcpyAsync(sm.data(), ctx->d_perm, sizeof(int) * nb, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < nb; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return sm[x] < sm[y]; });
  for (int band = 0; band < nb; ++band) perm[order[band]] = band;
  CK(cudaMemcpy(ctx->d_perm, perm.data(), sizeof(int) * nb, cudaMemcpyHostToDevice));
  return EVR_OK;
}

template <class T> int resident_alloc(evr_ctx* ctx) {
  cudaFree(ctx->d_flags);
  cudaFree(ctx->d_xchg);
  cudaFree(ctx->d_ticket);
  cudaFree(ctx->d_rx);
  ctx->d_rx = nullptr;
  ctx->d_flags = nullptr;
  ctx->d_xchg = nullptr;
  ctx->d_ticket = nullptr;
  CK(cudaMalloc(&ctx->d_flags, sizeof(unsigned long long) * ctx->r_nb));
  CK(cudaMemset(ctx->d_flags, 0, sizeof(unsigned long long) * ctx->r_nb));
  // 4 slots per column: the plane-frame kernel uses 3, k_resident_col 4
  const size_t xbytes = sizeof(unsigned long long) * LLWords<T>::N * 2 * ctx->r_nb * 2 * 4 * (size_t)ctx->W;
  CK(cudaMalloc(&ctx->d_xchg, xbytes));
  CK(cudaMemset(ctx->d_xchg, 0, xbytes));  // no stale tag can match a live one
  CK(cudaMalloc(&ctx->d_ticket, sizeof(unsigned)));
  CK(cudaMemset(ctx->d_ticket, 0, sizeof(unsigned)));
  CK(cudaMalloc(&ctx->d_rx, sizeof(unsigned long long) * 8 * ctx->r_nb));
  CK(cudaMemset(ctx->d_rx, 0, sizeof(unsigned long long) * 8 * ctx->r_nb));
  const void* fn = nullptr;
  if (ctx->r_ms == PLANES_COL) {
    const ResidentColKernel<T>* ck = resident_col_pick<T>(ctx->W, ctx->r_R);
    fn = ck ? (const void*)ck->fn : nullptr;
  } else {
    const ResidentKernel<T>* k = resident_pick<T>(ctx->W, ctx->r_ms);
    fn = k ? (const void*)k->fn : nullptr;
  }
  if (!fn) return fail(ctx, EVR_ERR_UNSUPPORTED, "no resident kernel shape");
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->r_smem));
  cudaFree(ctx->d_perm);
  ctx->d_perm = nullptr;
  if (ctx->r_ms == PLANES_COL && sm_order_enabled()) return resident_sm_order(ctx);
  return EVR_OK;
}

template <class T> int resident_enqueue(evr_ctx* ctx, int which) {
  if (which != 2)
    return fail(ctx, EVR_ERR_UNSUPPORTED, "resident engine runs whole packets only");
  const evr_config& g = ctx->cfg;
  ResArgs<T> a;
  a.hdr = ctx->hdr();
  a.f = ctx->f;
  a.raw = ctx->raw;
  a.u = ctx->fld<T>(F_U);
  a.p1 = ctx->fld<T>(F_P1);
  a.p2 = ctx->fld<T>(F_P2);
  a.p3 = ctx->fld<T>(F_P3);
  a.t = ctx->fld<T>(F_T);
  a.tx = ctx->fld<T>(F_TX);
  a.ty = ctx->fld<T>(F_TY);
  a.G = ctx->fld<T>(F_G);
  a.sg = ctx->fld<T>(F_SG);
  a.xchg = reinterpret_cast<T*>(ctx->d_xchg);
  a.frames = nullptr;
  a.flags = ctx->d_flags;
  a.part = ctx->part;
  a.ticket = ctx->d_ticket;
  a.rx = ctx->d_rx;
  a.tol = g.convergence_tol;
  a.info = ctx->d_info;
  a.err = ctx->d_err;
  a.trace = ctx->d_trace;
  a.perm = ctx->d_perm;
  a.H = ctx->H;
  a.W = ctx->W;
  a.nb = ctx->r_nb;
  a.R = ctx->r_R;
  a.tv_iters = g.denoise_iterations;
  a.pd_iters = g.max_iterations;
  a.manifold = g.manifold_enabled;
  a.t_scale = g.t_scale;
  a.c_pos = g.c_pos;
  a.c_neg = g.c_neg;
  a.u_min = g.u_min;
  a.u_max = g.u_max;
  const double step = 1.0 / std::sqrt(8.0);  // surface.py:158
  a.tau = (T)g.tau;
  a.sigma = (T)g.sigma;
  a.tl = (T)(g.tau * g.lam);
  a.tv_step = (T)step;
  a.shrink = (T)(step * g.denoise_weight);
  a.t_scaleT = (T)g.t_scale;
  a.uminT = (T)g.u_min;
  a.umaxT = (T)g.u_max;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(ctx->r_nb);
  lc.blockDim = dim3(ctx->r_nt);
  lc.dynamicSmemBytes = ctx->r_smem;
  lc.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident
  attr[0].val.cooperative = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  cudaError_t e;
  if (ctx->r_ms == PLANES_COL) {
    e = cudaLaunchKernelEx(&lc, resident_col_pick<T>(ctx->W, ctx->r_R)->fn, a);
  } else {
    e = cudaLaunchKernelEx(&lc, resident_pick<T>(ctx->W, ctx->r_ms)->fn, a);
  }
  if (e != cudaSuccess) return fail(ctx, EVR_ERR_CUDA, "resident launch: %s", cudaGetErrorString(e));
  return 1;
}

int enqueue_packet_any(evr_ctx* ctx, int which) {
  if (ctx->engine >= EVR_ENGINE_RESIDENT) {
    return ctx->prec == EVR_PREC_F64 ? resident_enqueue<double>(ctx, which)
                                     : resident_enqueue<float>(ctx, which);
  }
  return ctx->prec == EVR_PREC_F64 ? enqueue_packet<double>(ctx, which)
                                   : enqueue_packet<float>(ctx, which);
}

void drop_graphs(evr_ctx* ctx) {
  for (auto& g : ctx->graph)
    if (g) {
      cudaGraphExecDestroy(g);
      g = nullptr;
    }
}

// Launch packet stage `which` (0 surface, 1 solve, 2 both) through a CUDA
// graph captured on first use.
int launch_stage(evr_ctx* ctx, int which) {
  if (!ctx->graph[which]) {
    cudaGraph_t graph;
    CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    int n = enqueue_packet_any(ctx, which);
    cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
    if (n < 0) {
      if (e == cudaSuccess) cudaGraphDestroy(graph);
      return n;
    }
    CK(e);
    e = cudaGraphInstantiate(&ctx->graph[which], graph, 0);
    cudaGraphDestroy(graph);
    CK(e);
    ctx->graph_launches[which] = n;
  }
  CK(cudaGraphLaunch(ctx->graph[which], ctx->stream));
  ctx->launches += ctx->graph_launches[which];
  return EVR_OK;
}

int ensure_stage(evr_ctx* ctx, int64_t n) {
  if (n <= ctx->ev_cap) return EVR_OK;
  int64_t cap = std::max<int64_t>(n, std::max<int64_t>(4096, ctx->ev_cap * 2));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < 2; ++i)
    if (ctx->h_stage[i]) cudaFreeHost(ctx->h_stage[i]);
  if (ctx->d_stage) cudaFree(ctx->d_stage);
  ctx->h_stage[0] = ctx->h_stage[1] = nullptr;
  ctx->d_stage = nullptr;
  const size_t bytes = sizeof(PacketHdr) + (size_t)cap * sizeof(evr_event);
  CK(cudaMalloc(&ctx->d_stage, bytes));
  CK(cudaMallocHost(&ctx->h_stage[0], bytes));
  CK(cudaMallocHost(&ctx->h_stage[1], bytes));
  ctx->ev_cap = cap;
  drop_graphs(ctx);  // graphs bake the staging address
  return EVR_OK;
}

int validate_events(evr_ctx* ctx, const evr_event* ev, int64_t n) {
  for (int64_t k = 0; k < n; ++k)
    if (ev[k].x < 0 || ev[k].x >= ctx->W || ev[k].y < 0 || ev[k].y >= ctx->Htot)
      return fail(ctx, EVR_ERR_RANGE, "event %lld at (%d, %d) outside the %dx%d sensor",
                  (long long)k, (int)ev[k].x, (int)ev[k].y, ctx->W, ctx->Htot);
  return EVR_OK;
}

// Stage host events + header into pinned memory and copy them to the device.
int stage_host_packet(evr_ctx* ctx, const evr_event* ev, int64_t n, double window) {
  int rc;
  if ((rc = validate_events(ctx, ev, n))) return rc;
  if ((rc = ensure_stage(ctx, n))) return rc;
  const int slot = ctx->stage_slot;
  ctx->stage_slot ^= 1;
  CK(cudaEventSynchronize(ctx->stage_done[slot]));  // previous copy from this slot
  char* h = ctx->h_stage[slot];
  PacketHdr hdr{n, ev[n - 1].t, window, ++ctx->seq};
  std::memcpy(h, &hdr, sizeof hdr);
  std::memcpy(h + sizeof hdr, ev, (size_t)n * sizeof(evr_event));
  CK(cudaMemcpyAsync(ctx->d_stage, h, sizeof hdr + (size_t)n * sizeof(evr_event),
                     cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaEventRecord(ctx->stage_done[slot], ctx->stream));
  return EVR_OK;
}

// Device-resident events: copy into the staging slot (unless the producer
// wrote there directly through evr_event_buffer) and fill the header.
__global__ void k_stage_device(PacketHdr* hdr, evr_event* dst, const evr_event* __restrict__ src,
                               int64_t n, double window, int64_t seq) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n && dst != src) dst[k] = src[k];
  if (k == 0) {
    hdr->n = n;
    hdr->now = src[n - 1].t;
    hdr->window = window;
    hdr->seq = seq;
  }
}

int stage_device_packet(evr_ctx* ctx, const evr_event* dev, int64_t n, double window) {
  int rc;
  if ((rc = ensure_stage(ctx, n))) return rc;
  evr_event* dst = reinterpret_cast<evr_event*>(ctx->d_stage + sizeof(PacketHdr));
  k_stage_device<<<grid1d(n), kNT, 0, ctx->stream>>>(ctx->hdr(), dst, dev, n, window, ++ctx->seq);
  ctx->launches += 1;
  return launch_err(ctx, "stage");
}

// convergence_tol > 0: both engines stop on the device (the column resident
// kernel folds rel_change every iteration; the fused streaming list runs one
// march launch + rel_change per iteration behind a device stop flag); only
// band contexts still drive the iterations from the host
bool solve_needs_host_loop(const evr_ctx* ctx) {
  return ctx->cfg.convergence_tol > 0 && ctx->banded;
}

// Host-driven solve for convergence_tol > 0 and/or traces (solve.py:233-258):
// rel_change every iteration, early stop, optional energy rows.
template <class T>
int solve_host_loop(evr_ctx* ctx, const evr_config& g, evr_solve_info* info, double* etrace,
                    double* rtrace, bool write_state) {
  const bool track = g.convergence_tol > 0 || etrace || rtrace;
  // without a tolerance the iteration count is fixed: the traces go to a
  // device history read back once, no host round trip per iteration
  const bool sync_each = g.convergence_tol > 0;
  double* hist = nullptr;
  if (!sync_each && (etrace || rtrace)) {
    if (ctx->hist_cap < g.max_iterations) {
      cudaFree(ctx->d_hist);
      ctx->d_hist = nullptr;
      CK(cudaMalloc(&ctx->d_hist, sizeof(double) * 2 * g.max_iterations));
      ctx->hist_cap = g.max_iterations;
    }
    hist = ctx->d_hist;  // [rel_change x hist_cap | energy x hist_cap]
  }
  T* bufs[2] = {ctx->fld<T>(F_U), ctx->fld<T>(F_UN)};
  int iterations = 0, cur_i = 0;
  double rel = INFINITY;
  for (int it = 0; it < g.max_iterations; ++it) {
    T* cur = bufs[cur_i];
    T* nxt = bufs[cur_i ^ 1];
    T* v = ctx->fld<T>(F_V);
    const Geo own = ctx->geo_own();
    k_pd_primal<T><<<grid_geo(own), block2d(), 0, ctx->stream>>>(
        ctx->fld<T>(F_P1), ctx->fld<T>(F_P2), ctx->fld<T>(F_P3), coefs<T>(ctx), cur,
        ctx->fld<T>(F_BETA), ctx->fld<T>(F_FB), nxt, v, own, (T)g.tau, (T)g.u_min, (T)g.u_max);
    iterations = it + 1;
    ctx->launches += 1;
    if (track || it == g.max_iterations - 1) {
      relchange<T>(ctx, nxt, cur, iterations, 1, false, hist);
      ctx->launches += 1;
    }
    k_pd_dual<T><<<grid_geo(own), block2d(), 0, ctx->stream>>>(
        v, ctx->fld<T>(F_P1), ctx->fld<T>(F_P2), ctx->fld<T>(F_P3), coefs<T>(ctx),
        ctx->fld<T>(F_SG), own, (T)g.sigma);
    ctx->launches += 1;
    cur_i ^= 1;
    if (etrace) {
      const int nb = red_blocks(ctx->N);
      k_energy_partial<T, kNT><<<nb, kNT, 0, ctx->stream>>>(nxt, ctx->f, coefs<T>(ctx),
                                                           ctx->fld<T>(F_G), ctx->fld<T>(F_SG),
                                                           ctx->H, ctx->W, ctx->part);
      k_energy_final<kNT><<<1, kNT, 0, ctx->stream>>>(
          ctx->part, nb, g.lam, hist ? hist + ctx->hist_cap + it : ctx->d_scalar);
      ctx->launches += 2;
      if (!hist)
        CK(cudaMemcpyAsync(&etrace[it], ctx->d_scalar, sizeof(double), cudaMemcpyDeviceToHost,
                           ctx->stream));
    }
    if (sync_each) {
      CK(cudaMemcpyAsync(ctx->h_info, ctx->d_info, sizeof(evr_solve_info),
                         cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      rel = ctx->h_info->rel_change;
      if (rtrace) rtrace[it] = rel;
      if (g.convergence_tol > 0 && rel < g.convergence_tol) break;
    }
  }
  T* last = bufs[cur_i];
  if (write_state) {
    k_epilogue<T><<<grid1d(ctx->N), kNT, 0, ctx->stream>>>(last, ctx->fld<T>(F_U), ctx->f,
                                                          ctx->N);
    ctx->launches += 1;
  } else if (last != bufs[0]) {
    CK(cudaMemcpyAsync(bufs[0], last, sizeof(T) * ctx->N, cudaMemcpyDeviceToDevice,
                       ctx->stream));
  }
  int rc = launch_err(ctx, "solve loop");
  if (rc) return rc;
  if (hist) {
    if (rtrace)
      CK(cudaMemcpyAsync(rtrace, hist, sizeof(double) * iterations, cudaMemcpyDeviceToHost,
                         ctx->stream));
    if (etrace)
      CK(cudaMemcpyAsync(etrace, hist + ctx->hist_cap, sizeof(double) * iterations,
                         cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaMemcpyAsync(ctx->h_info, ctx->d_info, sizeof(evr_solve_info), cudaMemcpyDeviceToHost,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (info) {
    info->iterations = iterations;
    info->rel_change = sync_each ? rel : ctx->h_info->rel_change;
  }
  return EVR_OK;
}

int check_err_flag(evr_ctx* ctx) {
  int h = 0;
  CK(cudaMemcpy(&h, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost));
  if (h) {
    CK(cudaMemset(ctx->d_err, 0, sizeof(int)));
    return fail(ctx, EVR_ERR_RANGE, "a device-side event lay outside the %dx%d sensor", ctx->W,
                ctx->H);
  }
  return EVR_OK;
}

int require_config(evr_ctx* ctx) {
  if (!ctx->cfg_set) return fail(ctx, EVR_ERR_INVALID, "evr_set_config has not been called");
  return EVR_OK;
}

int require_f64(evr_ctx* ctx) {
  if (ctx->prec != EVR_PREC_F64)
    return fail(ctx, EVR_ERR_UNSUPPORTED, "operator API needs an EVR_PREC_F64 context");
  return EVR_OK;
}

int require_stencil(evr_ctx* ctx) {
  if (ctx->H < 2 || ctx->W < 2)
    return fail(ctx, EVR_ERR_UNSUPPORTED, "stencil operators need H, W >= 2 (got %dx%d)",
                ctx->H, ctx->W);
  return EVR_OK;
}

// State I/O covers the context's own rows (all rows of a whole-sensor
// context; a band's rows without its halos).
template <class T> int set_state_t(evr_ctx* ctx, const double* u, const double* f,
                                   const int64_t* raw, const double* p) {
  const int64_t N = ctx->own_n(), o = ctx->own_off();
  cudaStream_t s = ctx->stream;
  if (u) {
    CK(cudaMemcpyAsync(ctx->aos_a, u, sizeof(double) * N, cudaMemcpyHostToDevice, s));
    k_convert<double, T><<<grid1d(N), kNT, 0, s>>>(ctx->aos_a, ctx->fld<T>(F_U) + o, N);
  }
  if (f) CK(cudaMemcpyAsync(ctx->f + o, f, sizeof(double) * N, cudaMemcpyHostToDevice, s));
  if (raw) CK(cudaMemcpyAsync(ctx->raw + o, raw, sizeof(int64_t) * N, cudaMemcpyHostToDevice, s));
  if (p) {
    CK(cudaMemcpyAsync(ctx->aos_b, p, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, s));
    k_aos_to_planes<T><<<grid1d(N), kNT, 0, s>>>(ctx->aos_b, ctx->fld<T>(F_P1) + o,
                                                 ctx->fld<T>(F_P2) + o, ctx->fld<T>(F_P3) + o, N);
  }
  int rc = launch_err(ctx, "set_state");
  if (rc) return rc;
  CK(cudaStreamSynchronize(s));
  return EVR_OK;
}

template <class T> int get_state_t(evr_ctx* ctx, double* u, double* f, int64_t* raw, double* p) {
  const int64_t N = ctx->own_n(), o = ctx->own_off();
  cudaStream_t s = ctx->stream;
  if (u) {
    k_convert<T, double><<<grid1d(N), kNT, 0, s>>>(ctx->fld<T>(F_U) + o, ctx->aos_a, N);
    CK(cudaMemcpyAsync(u, ctx->aos_a, sizeof(double) * N, cudaMemcpyDeviceToHost, s));
  }
  if (f) CK(cudaMemcpyAsync(f, ctx->f + o, sizeof(double) * N, cudaMemcpyDeviceToHost, s));
  if (raw) CK(cudaMemcpyAsync(raw, ctx->raw + o, sizeof(int64_t) * N, cudaMemcpyDeviceToHost, s));
  if (p) {
    k_planes_to_aos<T><<<grid1d(N), kNT, 0, s>>>(ctx->fld<T>(F_P1) + o, ctx->fld<T>(F_P2) + o,
                                                 ctx->fld<T>(F_P3) + o, ctx->aos_b, N);
    CK(cudaMemcpyAsync(p, ctx->aos_b, sizeof(double) * 3 * N, cudaMemcpyDeviceToHost, s));
  }
  int rc = launch_err(ctx, "get_state");
  if (rc) return rc;
  CK(cudaStreamSynchronize(s));
  return EVR_OK;
}

template <class T> int get_plane_t(evr_ctx* ctx, int field, double* out) {
  const int64_t N = ctx->own_n(), o = ctx->own_off();
  k_convert<T, double><<<grid1d(N), kNT, 0, ctx->stream>>>(ctx->fld<T>(field) + o, ctx->aos_a, N);
  CK(cudaMemcpyAsync(out, ctx->aos_a, sizeof(double) * N, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return launch_err(ctx, "get_plane");
}

int h2d(evr_ctx* ctx, void* dst, const void* src, size_t bytes) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return EVR_OK;
}

int d2h_sync(evr_ctx* ctx, void* dst, const void* src, size_t bytes) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return EVR_OK;
}

}  // namespace

// =========================================================================
namespace {

// Snapshot of one packet's result on the context stream: the frame u (as
// float64) into a per-slot device buffer, plus the solve record and the
// device error flag (then cleared), so the next packet may run while the
// copy stream reads the slot back.
template <class T>
__global__ void k_frame_snapshot(const T* __restrict__ u, double* __restrict__ out, int64_t n,
                                 const evr_solve_info* info, int* err, FrameRec* rec) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride)
    out[k] = (double)u[k];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    rec->info = *info;
    rec->err = *err;
    *err = 0;
  }
}

int ensure_frame_slots(evr_ctx* ctx) {
  if (ctx->cstream) return EVR_OK;
  CK(cudaStreamCreateWithFlags(&ctx->cstream, cudaStreamNonBlocking));
  for (int i = 0; i < kFrameSlots; ++i) {
    CK(cudaMalloc(&ctx->d_fr[i], sizeof(double) * std::max<int64_t>(ctx->own_n(), 1)));
    CK(cudaEventCreateWithFlags(&ctx->fr_ready[i], cudaEventDisableTiming));
    CK(cudaEventCreate(&ctx->fr_done[i]));
    CK(cudaEventCreate(&ctx->pk_t0[i]));
  }
  CK(cudaMalloc(&ctx->d_rec, sizeof(FrameRec) * kFrameSlots));
  CK(cudaMallocHost(&ctx->h_rec, sizeof(FrameRec) * kFrameSlots));
  return EVR_OK;
}

// start of the packet whose frame the next evr_frame_submit takes (the
// frame pipeline's per-packet time: H2D .. solve .. frame D2H)
int mark_packet_start(evr_ctx* ctx) {
  int rc;
  if ((rc = ensure_frame_slots(ctx))) return rc;
  const int s = (int)(ctx->fr_next % kFrameSlots);
  if (ctx->fr_ticket[s] >= 0) return EVR_OK;  // slot still in flight: no timing for this one
  CK(cudaEventRecord(ctx->pk_t0[s], ctx->stream));
  ctx->pk_seq[s] = ctx->fr_next;
  return EVR_OK;
}

// float64 operator solves with the ROF / L1 data terms on the temporally
// blocked tiles (k_pd_tile<.., DT>, bit-identical to the split
// k_rof_primal / k_l1_primal + k_pd_dual loop): the planes set up by
// k_solver_setup are packed once, the iterations run K per launch (a
// remainder of one merges into the last tile, 3 + 1 -> 4 or 4 + 1 -> 3 + 2),
// and u comes back from the packed set.  iterations >= 2.  Returns the
// plane holding u.
template <int DT>
double* op_tile_solve(evr_ctx* ctx, int iterations, const double* fslot, double step) {
  cudaStream_t s = ctx->stream;
  const int64_t N = ctx->N;
  const Packed<double> P = packed<double>(ctx);
  k_pack_solver<double><<<grid1d(N), kNT, 0, s>>>(
      ctx->fld<double>(F_P1), ctx->fld<double>(F_P2), ctx->fld<double>(F_P3),
      ctx->fld<double>(F_U), ctx->fld<double>(F_TX), ctx->fld<double>(F_TY), coefs<double>(ctx),
      ctx->fld<double>(F_SG), ctx->fld<double>(F_BETA), ctx->fld<double>(F_FB), P.pd[0], P.cst, N,
      fslot);
  const int tk = std::max(2, ctx_tile_k(ctx));
  std::vector<int> ks;  // iterations per launch, each in [2, 4] (the built tiles)
  for (int rem = iterations; rem > 0;) {
    int kk = std::min(tk, rem);
    if (rem - kk == 1) kk = kk < 4 ? kk + 1 : kk - 1;
    ks.push_back(kk);
    rem -= kk;
  }
  int b = 0;
  const auto cr = march_rows<Q4<double>>(ctx, [](const evr_ctx* c) { return packed<double>(c).cst; }, 2);
  const MetricPackF64 m{cr.own, cr};
  bool first = true;
  for (int kk : ks) {
    const auto in = march_rows<Q4<double>>(ctx, [b](const evr_ctx* c) { return packed<double>(c).pd[b]; }, 1);
    pd_tile_rpt<double, TileShape<double>::RPT, false, MetricPackF64, DT>(
        ctx, kk, in, m, packed<double>(ctx).pd[b ^ 1], step, first ? 0 : 1);
    first = false;
    b ^= 1;
  }
  k_unpack_solver<double><<<grid1d(N), kNT, 0, s>>>(P.pd[b], ctx->fld<double>(F_P1),
                                                    ctx->fld<double>(F_P2), ctx->fld<double>(F_P3),
                                                    ctx->fld<double>(F_U), ctx->f, N);
  ctx->launches += 2 + (int64_t)ks.size();
  return ctx->fld<double>(F_U);
}

}  // namespace

extern "C" {

const char* evr_version(void) { return "evr-b200 0.1.0 (sm_100a)"; }

int evr_device_count(int* count) {
  if (!count) return EVR_ERR_INVALID;
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    *count = 0;
    return EVR_ERR_CUDA;
  }
  return EVR_OK;
}

const char* evr_last_error(const evr_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int evr_create(evr_ctx** out, int device, int height, int width, int precision) {
  if (!out) return EVR_ERR_INVALID;
  *out = nullptr;
  if (height < 1 || width < 1) return EVR_ERR_INVALID;
  if (precision != EVR_PREC_F64 && precision != EVR_PREC_F32) return EVR_ERR_INVALID;
  evr_ctx* ctx = new evr_ctx();
  ctx->device = device;
  ctx->H = height;
  ctx->W = width;
  ctx->N = (int64_t)height * width;
  ctx->prec = precision;
  ctx->row0 = 0;
  ctx->Htot = height;
  ctx->own_lo = 0;
  ctx->own_hi = height - 1;
  auto bail = [&](int rc) {
    std::string msg = ctx->err;
    evr_destroy(ctx);
    (void)msg;
    return rc;
  };
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return bail(EVR_ERR_CUDA);
  const size_t esz = precision == EVR_PREC_F64 ? 8 : 4;
  ctx->field_stride = ((size_t)ctx->N * esz + 255) / 256 * 256;
  const int64_t N = ctx->N;
  int rc = [&]() -> int {
    CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    CK(cudaMalloc(&ctx->slab, ctx->field_stride * F_COUNT));
    CK(cudaMemsetAsync(ctx->slab, 0, ctx->field_stride * F_COUNT, ctx->stream));
    CK(cudaMalloc(&ctx->f, sizeof(double) * N));
    CK(cudaMalloc(&ctx->d_pack, packed_bytes(N, precision)));
    CK(cudaMalloc(&ctx->raw, sizeof(int64_t) * N));
    CK(cudaMalloc(&ctx->aos_a, sizeof(double) * 3 * N));
    CK(cudaMalloc(&ctx->aos_b, sizeof(double) * 3 * N));
    CK(cudaMalloc(&ctx->part, sizeof(double) * 2 * kRedBlocks));
    CK(cudaMalloc(&ctx->rticket, sizeof(unsigned)));
    CK(cudaMalloc(&ctx->d_stop, sizeof(int)));
    CK(cudaMemsetAsync(ctx->d_stop, 0, sizeof(int), ctx->stream));
    CK(cudaMemsetAsync(ctx->rticket, 0, sizeof(unsigned), ctx->stream));
    CK(cudaMalloc(&ctx->d_scalar, sizeof(double) * 4));
    CK(cudaMalloc(&ctx->d_err, sizeof(int)));
    CK(cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream));
    CK(cudaMalloc(&ctx->d_info, sizeof(evr_solve_info)));
    CK(cudaMemsetAsync(ctx->d_info, 0, sizeof(evr_solve_info), ctx->stream));
    CK(cudaMallocHost(&ctx->h_info, sizeof(evr_solve_info)));
    CK(cudaMallocHost(&ctx->h_err, sizeof(int)));
    *ctx->h_err = 0;
    for (int i = 0; i < 2; ++i) {
      CK(cudaEventCreateWithFlags(&ctx->stage_done[i], cudaEventDisableTiming));
      CK(cudaEventRecord(ctx->stage_done[i], ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return EVR_OK;
  }();
  if (rc) return bail(rc);
  *out = ctx;
  return EVR_OK;
}

void evr_destroy(evr_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  drop_graphs(ctx);
  cudaFree(ctx->slab);
  cudaFree(ctx->d_stop);
  cudaFree(ctx->d_hist);
  cudaFree(ctx->d_pack);
  cudaFree(ctx->f);
  cudaFree(ctx->raw);
  cudaFree(ctx->aos_a);
  cudaFree(ctx->aos_b);
  cudaFree(ctx->part);
  cudaFree(ctx->rticket);
  cudaFree(ctx->d_scalar);
  cudaFree(ctx->d_err);
  cudaFree(ctx->d_info);
  cudaFree(ctx->d_stage);
  cudaFree(ctx->d_flags);
  cudaFree(ctx->d_xchg);
  cudaFree(ctx->d_ticket);
  cudaFree(ctx->d_perm);
  cudaFree(ctx->d_trace);
  for (int i = 0; i < 2; ++i) {
    if (ctx->h_stage[i]) cudaFreeHost(ctx->h_stage[i]);
    if (ctx->stage_done[i]) cudaEventDestroy(ctx->stage_done[i]);
  }
  if (ctx->h_info) cudaFreeHost(ctx->h_info);
  if (ctx->h_err) cudaFreeHost(ctx->h_err);
  if (ctx->cstream) cudaStreamSynchronize(ctx->cstream);
  for (int i = 0; i < kFrameSlots; ++i) {
    cudaFree(ctx->d_fr[i]);
    if (ctx->fr_ready[i]) cudaEventDestroy(ctx->fr_ready[i]);
    if (ctx->fr_done[i]) cudaEventDestroy(ctx->fr_done[i]);
    if (ctx->pk_t0[i]) cudaEventDestroy(ctx->pk_t0[i]);
  }
  cudaFree(ctx->d_rec);
  cudaFree(ctx->tgv);
  if (ctx->h_rec) cudaFreeHost(ctx->h_rec);
  if (ctx->cstream) cudaStreamDestroy(ctx->cstream);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int evr_set_config(evr_ctx* ctx, const evr_config* cfg) {
  CHECK_CTX();
  if (!cfg) return fail(ctx, EVR_ERR_INVALID, "null config");
  if (cfg->max_iterations < 1) return fail(ctx, EVR_ERR_INVALID, "max_iterations must be >= 1");
  if (cfg->manifold_enabled && cfg->denoise_iterations < 1)
    return fail(ctx, EVR_ERR_INVALID, "denoise iterations must be >= 1");
  if (!(0 < cfg->u_min && cfg->u_min < cfg->u_max))
    return fail(ctx, EVR_ERR_INVALID, "need 0 < u_min < u_max");
  ctx->cfg = *cfg;
  ctx->cfg_set = true;
  drop_graphs(ctx);
  ctx->engine = EVR_ENGINE_STREAMING;
  // tags of the resident exchange are (packet << 16) + step: a packet's
  // steps must stay below 2^16
  const bool tags_fit = (int64_t)cfg->denoise_iterations + cfg->max_iterations + 4 < 65536;
  if (cfg->engine == EVR_ENGINE_RESIDENT && !tags_fit)
    return fail(ctx, EVR_ERR_UNSUPPORTED, "resident engine: more than 65531 iterations per packet");
  if (cfg->engine != EVR_ENGINE_STREAMING && tags_fit && ctx->H >= 2 && ctx->W >= 2) {
    // AUTO: the resident kernel while each CTA owns at most
    // kAutoResidentRows rows, else the fused streaming list (measured on
    // B200, profiles/r01_summary.md: at 640x480 and beyond the streaming
    // tiles beat every resident variant).  RESIDENT: whenever it fits.
    bool ok = cfg->engine == EVR_ENGINE_AUTO || cfg->engine == EVR_ENGINE_RESIDENT;
    if (ok)
      ok = ctx->prec == EVR_PREC_F64 ? resident_plan<double>(ctx) : resident_plan<float>(ctx);
    if (ok && cfg->engine == EVR_ENGINE_AUTO && ctx->r_R > kAutoResidentRows) ok = false;
    // the device-side early stop lives in the column kernel only
    if (ok && cfg->convergence_tol > 0 && ctx->r_ms != PLANES_COL) ok = false;
    if (ok) {
      ctx->engine = EVR_ENGINE_RESIDENT;
      int rc = ctx->prec == EVR_PREC_F64 ? resident_alloc<double>(ctx) : resident_alloc<float>(ctx);
      if (rc) return rc;
    } else if (cfg->engine != EVR_ENGINE_AUTO) {
      return fail(ctx, EVR_ERR_UNSUPPORTED, "engine %d does not fit a %dx%d sensor", cfg->engine,
                  ctx->W, ctx->H);
    }
  }
  return EVR_OK;
}

int evr_engine_detail(evr_ctx* ctx, char* buf, int len) {
  if (!ctx || !buf || len < 1) return EVR_ERR_INVALID;
  const char* ty = ctx->prec == EVR_PREC_F64 ? "f64" : "f32";
  if (ctx->engine == EVR_ENGINE_STREAMING) {
    if (ctx->banded)
      snprintf(buf, len, "streaming split half-steps (band rows %d..%d of %d)", ctx->row0,
               ctx->row0 + ctx->H - 1, ctx->Htot);
    else {
      const int tk = ctx_tile_k(ctx);
      if (tk > 1) {
        const bool d = ctx->prec == EVR_PREC_F64;
        const int rpt = d ? tile_rpt<double>(ctx, tk) : tile_rpt<float>(ctx, tk);
        const int G = d ? TileShape<double>::G : TileShape<float>::G;
        const int tiw = 32 - 2 * tk, tih = G * rpt - 2 * tk;
        const bool whole = ctx->cfg.convergence_tol <= 0 && ctx->cfg.max_iterations >= 2;
        snprintf(buf, len,
                 "streaming k_tv_tile/k_pd_tile<%s,K=%d> %d iterations per launch, %dx%d tiles, "
                 "%d CTAs x %d%s",
                 ty, tk, tk, tiw, tih, ((ctx->W + tiw - 1) / tiw) * ((ctx->H + tih - 1) / tih),
                 32 * G,
                 whole ? ", fused metric+pack and epilogue+rel_change"
                       : " (+ k_pd_march per iteration with a convergence_tol)");
      } else {
        snprintf(buf, len, "streaming k_tv_march/k_pd_march<%s,RY=%d> %u CTAs x %d", ty,
                 kMarchRY, march_grid(ctx), kMarchNT);
      }
    }
  } else {
    const char* k = ctx->r_ms == PLANES_COL ? "k_resident_col" : "k_resident(smem frames)";
    snprintf(buf, len, "%s<%s,NT=%d,RB=%d> x%d CTAs, %zu B smem", k, ty, ctx->r_nt, ctx->r_R,
             ctx->r_nb, ctx->r_smem);
  }
  return EVR_OK;
}

int evr_active_engine(evr_ctx* ctx, int* engine) {
  if (!ctx || !engine) return EVR_ERR_INVALID;
  *engine = ctx->engine;
  return EVR_OK;
}

int evr_init_state(evr_ctx* ctx) {
  CHECK_CTX();
  int rc;
  if ((rc = require_config(ctx))) return rc;
  const double mid = 0.5 * (ctx->cfg.u_min + ctx->cfg.u_max);  // pipeline.py:105
  const int64_t N = ctx->N;
  cudaStream_t s = ctx->stream;
  k_fill<double><<<grid1d(N), kNT, 0, s>>>(ctx->f, mid, N);
  if (ctx->prec == EVR_PREC_F64) {
    k_fill<double><<<grid1d(N), kNT, 0, s>>>(ctx->fld<double>(F_U), mid, N);
  } else {
    k_fill<float><<<grid1d(N), kNT, 0, s>>>(ctx->fld<float>(F_U), (float)mid, N);
  }
  CK(cudaMemsetAsync(ctx->raw, 0, sizeof(int64_t) * N, s));
  for (int k : {F_P1, F_P2, F_P3}) CK(cudaMemsetAsync(ctx->slab + ctx->field_stride * k, 0, ctx->field_stride, s));
  if ((rc = launch_err(ctx, "init_state"))) return rc;
  CK(cudaStreamSynchronize(s));
  return EVR_OK;
}

int evr_set_state(evr_ctx* ctx, const double* u, const double* f, const int64_t* raw,
                  const double* p) {
  CHECK_CTX();
  return ctx->prec == EVR_PREC_F64 ? set_state_t<double>(ctx, u, f, raw, p)
                                   : set_state_t<float>(ctx, u, f, raw, p);
}

int evr_get_state(evr_ctx* ctx, double* u, double* f, int64_t* raw, double* p) {
  CHECK_CTX();
  return ctx->prec == EVR_PREC_F64 ? get_state_t<double>(ctx, u, f, raw, p)
                                   : get_state_t<float>(ctx, u, f, raw, p);
}

int evr_ingest(evr_ctx* ctx, const evr_event* events, int64_t n) {
  CHECK_CTX();
  int rc;
  if ((rc = require_config(ctx))) return rc;
  if (n <= 0) return EVR_OK;
  if (!events) return fail(ctx, EVR_ERR_INVALID, "null events");
  if ((rc = stage_host_packet(ctx, events, n, 1.0))) return rc;
  launch_ingest(ctx);
  ctx->launches += 1;
  if ((rc = launch_err(ctx, "ingest"))) return rc;
  CK(cudaStreamSynchronize(ctx->stream));
  return check_err_flag(ctx);
}

// Split packet API used when the host needs the surface between the two
// halves (debug_sink) or a host-driven solve (convergence_tol, trace).
int evr_packet_begin(evr_ctx* ctx, const evr_event* events, int64_t n, double window) {
  CHECK_CTX();
  int rc;
  if ((rc = require_config(ctx))) return rc;
  if (n <= 0 || !events) return fail(ctx, EVR_ERR_INVALID, "empty packet");
  if ((rc = stage_host_packet(ctx, events, n, window))) return rc;
  if (ctx->engine >= EVR_ENGINE_RESIDENT) {
    // the resident kernel fuses the whole packet; run the streaming
    // surface stage here so the host can look at it between the halves
    int r = ctx->prec == EVR_PREC_F64 ? enqueue_packet<double>(ctx, 0) : enqueue_packet<float>(ctx, 0);
    if (r < 0) return r;
    ctx->launches += r;
    return EVR_OK;
  }
  return launch_stage(ctx, 0);
}

int evr_packet_solve(evr_ctx* ctx, evr_solve_info* info, double* energy_trace,
                     double* rel_trace) {
  CHECK_CTX();
  int rc;
  if ((rc = require_config(ctx))) return rc;
  if (solve_needs_host_loop(ctx) || energy_trace || rel_trace || ctx->engine >= EVR_ENGINE_RESIDENT) {
    rc = ctx->prec == EVR_PREC_F64
             ? solve_host_loop<double>(ctx, ctx->cfg, info, energy_trace, rel_trace, true)
             : solve_host_loop<float>(ctx, ctx->cfg, info, energy_trace, rel_trace, true);
    if (rc) return rc;
    return check_err_flag(ctx);
  }
  if ((rc = launch_stage(ctx, 1))) return rc;
  return evr_synchronize(ctx, info);
}

int evr_process_packet(evr_ctx* ctx, const evr_event* events, int64_t n, double window,
                       evr_solve_info* info) {
  CHECK_CTX();
  int rc;
  if ((rc = require_config(ctx))) return rc;
  if (solve_needs_host_loop(ctx)) {
    if ((rc = evr_packet_begin(ctx, events, n, window))) return rc;
    return evr_packet_solve(ctx, info, nullptr, nullptr);
  }
  if ((rc = evr_process_packet_async(ctx, events, n, window))) return rc;
  return evr_synchronize(ctx, info);
}

int evr_process_packet_async(evr_ctx* ctx, const evr_event* events, int64_t n, double window) {
  CHECK_CTX();
  int rc;
  if ((rc = require_config(ctx))) return rc;
  if (n <= 0 || !events) return fail(ctx, EVR_ERR_INVALID, "empty packet");
  if (solve_needs_host_loop(ctx))
    return fail(ctx, EVR_ERR_UNSUPPORTED, "convergence_tol > 0 needs evr_process_packet");
  if ((rc = mark_packet_start(ctx))) return rc;
  if ((rc = stage_host_packet(ctx, events, n, window))) return rc;
  return launch_stage(ctx, 2);
}

int evr_process_packet_device(evr_ctx* ctx, const evr_event* dev_events, int64_t n,
                              double window) {
  CHECK_CTX();
  int rc;
  if ((rc = require_config(ctx))) return rc;
  if (n <= 0 || !dev_events) return fail(ctx, EVR_ERR_INVALID, "empty packet");
  if (solve_needs_host_loop(ctx))
    return fail(ctx, EVR_ERR_UNSUPPORTED, "convergence_tol > 0 needs evr_process_packet");
  if ((rc = mark_packet_start(ctx))) return rc;
  if ((rc = stage_device_packet(ctx, dev_events, n, window))) return rc;
  return launch_stage(ctx, 2);
}

int evr_synchronize(evr_ctx* ctx, evr_solve_info* info) {
  CHECK_CTX();
  if (info) {
    CK(cudaMemcpyAsync(ctx->h_info, ctx->d_info, sizeof(evr_solve_info), cudaMemcpyDeviceToHost,
                       ctx->stream));
  }
  // the device error flag rides the same stream (no extra blocking copy)
  CK(cudaMemcpyAsync(ctx->h_err, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (info) *info = *ctx->h_info;
  if (*ctx->h_err) {
    *ctx->h_err = 0;
    CK(cudaMemset(ctx->d_err, 0, sizeof(int)));
    return fail(ctx, EVR_ERR_RANGE, "a device-side event lay outside the %dx%d sensor", ctx->W,
                ctx->H);
  }
  return EVR_OK;
}


int evr_set_tile_k(evr_ctx* ctx, int k) {
  CHECK_CTX();
  if (k < 0 || k > 4) return fail(ctx, EVR_ERR_INVALID, "tile iterations must be in [0, 4]");
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->tile_k = k;
  drop_graphs(ctx);
  return EVR_OK;
}

int evr_time_iteration_kernel(evr_ctx* ctx, int which, int reps, float* us_per_launch,
                              int* iterations_per_launch) {
  CHECK_CTX();
  if (!us_per_launch || reps < 1 || (which != 0 && which != 1))
    return fail(ctx, EVR_ERR_INVALID, "bad arguments");
  int rc;
  if ((rc = require_config(ctx))) return rc;
  if (ctx->engine != EVR_ENGINE_STREAMING || ctx->banded || !ctx->d_pack)
    return fail(ctx, EVR_ERR_UNSUPPORTED, "only the whole-sensor streaming list has iteration kernels");
  const int tk = ctx_tile_k(ctx);
  // the packed sets hold the last packet's state: re-running iterations on
  // them changes nothing the next packet reads (it packs from the planes)
  Step st{which == 0 ? ST_PDF : ST_TVF, 1, 0, tk};  // it = 1: a steady-state launch
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto one = [&](int i) {
    st.buf = i & 1;
    return ctx->prec == EVR_PREC_F64 ? launch_step<double>(ctx, st) : launch_step<float>(ctx, st);
  };
  one(0);
  CK(cudaEventRecord(e0, ctx->stream));
  for (int i = 0; i < reps; ++i) one(i + 1);
  CK(cudaEventRecord(e1, ctx->stream));
  CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if ((rc = launch_err(ctx, "time_iteration_kernel"))) return rc;
  *us_per_launch = 1000.f * ms / reps;
  if (iterations_per_launch) *iterations_per_launch = tk;
  return EVR_OK;
}

int evr_frame_submit(evr_ctx* ctx, double* u_out, int64_t* ticket) {
  CHECK_CTX();
  if (!ticket) return fail(ctx, EVR_ERR_INVALID, "null ticket");
  int rc;
  if ((rc = ensure_frame_slots(ctx))) return rc;
  const int64_t t = ctx->fr_next;
  const int s = (int)(t % kFrameSlots);
  if (ctx->fr_ticket[s] >= 0)
    return fail(ctx, EVR_ERR_INVALID, "all %d frame slots are in flight: wait ticket %lld first",
                kFrameSlots, (long long)ctx->fr_ticket[s]);
  const int64_t N = ctx->own_n(), o = ctx->own_off();
  const int grid = (int)std::min<int64_t>((N + kNT - 1) / kNT, 4 * 148);
  if (ctx->prec == EVR_PREC_F64)
    k_frame_snapshot<double><<<std::max(grid, 1), kNT, 0, ctx->stream>>>(
        ctx->fld<double>(F_U) + o, ctx->d_fr[s], N, ctx->d_info, ctx->d_err, ctx->d_rec + s);
  else
    k_frame_snapshot<float><<<std::max(grid, 1), kNT, 0, ctx->stream>>>(
        ctx->fld<float>(F_U) + o, ctx->d_fr[s], N, ctx->d_info, ctx->d_err, ctx->d_rec + s);
  ctx->launches += 1;
  if ((rc = launch_err(ctx, "frame_snapshot"))) return rc;
  CK(cudaEventRecord(ctx->fr_ready[s], ctx->stream));
  CK(cudaStreamWaitEvent(ctx->cstream, ctx->fr_ready[s], 0));
  if (u_out)
    CK(cudaMemcpyAsync(u_out, ctx->d_fr[s], sizeof(double) * N, cudaMemcpyDeviceToHost,
                       ctx->cstream));
  CK(cudaMemcpyAsync(ctx->h_rec + s, ctx->d_rec + s, sizeof(FrameRec), cudaMemcpyDeviceToHost,
                     ctx->cstream));
  CK(cudaEventRecord(ctx->fr_done[s], ctx->cstream));
  ctx->fr_ticket[s] = t;
  ctx->fr_host[s] = u_out;
  ctx->fr_next = t + 1;
  *ticket = t;
  return EVR_OK;
}

int evr_frame_wait(evr_ctx* ctx, int64_t ticket, evr_solve_info* info) {
  CHECK_CTX();
  const int s = (int)(((ticket % kFrameSlots) + kFrameSlots) % kFrameSlots);
  if (ticket < 0 || !ctx->cstream || ctx->fr_ticket[s] != ticket)
    return fail(ctx, EVR_ERR_INVALID, "unknown frame ticket %lld", (long long)ticket);
  CK(cudaEventSynchronize(ctx->fr_done[s]));
  ctx->fr_ticket[s] = -1;
  ctx->fr_host[s] = nullptr;
  const FrameRec r = ctx->h_rec[s];
  if (info) {
    *info = r.info;
    info->packet_ms = 0.0f;
    if (ctx->pk_seq[s] == ticket) cudaEventElapsedTime(&info->packet_ms, ctx->pk_t0[s], ctx->fr_done[s]);
  }
  ctx->pk_seq[s] = -1;
  if (r.err)
    return fail(ctx, EVR_ERR_RANGE, "a device-side event lay outside the %dx%d sensor", ctx->W,
                ctx->H);
  return EVR_OK;
}

int evr_get_frame(evr_ctx* ctx, double* u_out) {
  CHECK_CTX();
  if (!u_out) return fail(ctx, EVR_ERR_INVALID, "null output");
  return ctx->prec == EVR_PREC_F64 ? get_plane_t<double>(ctx, F_U, u_out)
                                   : get_plane_t<float>(ctx, F_U, u_out);
}

int evr_get_frame_async(evr_ctx* ctx, double* u_out) {
  CHECK_CTX();
  if (!u_out) return fail(ctx, EVR_ERR_INVALID, "null output");
  const int64_t N = ctx->own_n(), o = ctx->own_off();
  const double* src;
  if (ctx->prec == EVR_PREC_F64) {
    src = ctx->fld<double>(F_U) + o;
  } else {
    k_convert<float, double><<<grid1d(N), kNT, 0, ctx->stream>>>(ctx->fld<float>(F_U) + o,
                                                                 ctx->aos_a, N);
    int rc = launch_err(ctx, "get_frame_async");
    if (rc) return rc;
    src = ctx->aos_a;
  }
  CK(cudaMemcpyAsync(u_out, src, sizeof(double) * N, cudaMemcpyDeviceToHost, ctx->stream));
  return EVR_OK;
}

int evr_host_alloc(size_t bytes, void** out) {
  if (!out) return EVR_ERR_INVALID;
  *out = nullptr;
  const cudaError_t e = cudaHostAlloc(out, bytes > 0 ? bytes : 1, cudaHostAllocPortable);
  return e == cudaSuccess ? EVR_OK : e == cudaErrorMemoryAllocation ? EVR_ERR_OOM : EVR_ERR_CUDA;
}

int evr_host_free(void* p) {
  if (p && cudaFreeHost(p) != cudaSuccess) return EVR_ERR_CUDA;
  return EVR_OK;
}

int evr_get_surface(evr_ctx* ctx, double* t_out, double* G_out) {
  CHECK_CTX();
  int rc = EVR_OK;
  if (t_out)
    rc = ctx->prec == EVR_PREC_F64 ? get_plane_t<double>(ctx, F_T, t_out)
                                   : get_plane_t<float>(ctx, F_T, t_out);
  if (!rc && G_out)
    rc = ctx->prec == EVR_PREC_F64 ? get_plane_t<double>(ctx, F_G, G_out)
                                   : get_plane_t<float>(ctx, F_G, G_out);
  return rc;
}

int evr_get_metric(evr_ctx* ctx, double* tx, double* ty, double* G, double* sqrtG) {
  CHECK_CTX();
  double* outs[4] = {tx, ty, G, sqrtG};
  const int fl[4] = {F_TX, F_TY, F_G, F_SG};
  for (int m = 0; m < 4; ++m) {
    if (!outs[m]) continue;
    int rc = ctx->prec == EVR_PREC_F64 ? get_plane_t<double>(ctx, fl[m], outs[m])
                                       : get_plane_t<float>(ctx, fl[m], outs[m]);
    if (rc) return rc;
  }
  return EVR_OK;
}

int evr_get_frame_u8(evr_ctx* ctx, double lo, double hi, uint8_t* out) {
  CHECK_CTX();
  if (!out || !(hi > lo)) return fail(ctx, EVR_ERR_INVALID, "bad gray range");
  uint8_t* d = reinterpret_cast<uint8_t*>(ctx->aos_a);
  if (ctx->prec == EVR_PREC_F64)
    k_to_gray<double><<<grid1d(ctx->N), kNT, 0, ctx->stream>>>(ctx->fld<double>(F_U), lo, hi, d, ctx->N);
  else
    k_to_gray<float><<<grid1d(ctx->N), kNT, 0, ctx->stream>>>(ctx->fld<float>(F_U), lo, hi, d, ctx->N);
  ctx->launches += 1;
  int rc = launch_err(ctx, "to_gray");
  if (rc) return rc;
  return d2h_sync(ctx, out, d, (size_t)ctx->N);
}

int evr_event_buffer(evr_ctx* ctx, int64_t n, evr_event** dev_ptr) {
  CHECK_CTX();
  if (!dev_ptr || n < 1) return fail(ctx, EVR_ERR_INVALID, "bad event buffer request");
  int rc = ensure_stage(ctx, n);
  if (rc) return rc;
  *dev_ptr = reinterpret_cast<evr_event*>(ctx->d_stage + sizeof(PacketHdr));
  return EVR_OK;
}

int evr_debug_timeline(evr_ctx* ctx, int enable, uint64_t* out, int64_t n) {
  CHECK_CTX();
  if (enable >= 0) {
    if (enable && !ctx->d_trace) {
      CK(cudaMalloc(&ctx->d_trace, sizeof(unsigned long long) * 256 * std::max(ctx->r_nb, 1)));
      CK(cudaMemset(ctx->d_trace, 0, sizeof(unsigned long long) * 256 * std::max(ctx->r_nb, 1)));
    } else if (!enable && ctx->d_trace) {
      CK(cudaStreamSynchronize(ctx->stream));
      cudaFree(ctx->d_trace);
      ctx->d_trace = nullptr;
    }
    drop_graphs(ctx);
  }
  if (out && ctx->d_trace) {
    const int64_t m = std::min<int64_t>(n, 256 * (int64_t)std::max(ctx->r_nb, 1));
    return d2h_sync(ctx, out, ctx->d_trace, sizeof(uint64_t) * m);
  }
  return EVR_OK;
}

void* evr_stream(evr_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int64_t evr_launch_count(const evr_ctx* ctx) { return ctx ? ctx->launches : 0; }

// ---- operator API (float64 contexts) ---------------------------------------
#define OP_PROLOGUE(stencil)                     \
  CHECK_CTX();                                   \
  {                                              \
    int rc_ = require_f64(ctx);                  \
    if (!rc_ && (stencil)) rc_ = require_stencil(ctx); \
    if (rc_) return rc_;                         \
  }                                              \
  const int64_t N = ctx->N;                      \
  const size_t B = sizeof(double) * N;           \
  cudaStream_t s = ctx->stream;                  \
  (void)B; (void)s;

int evr_op_grad(evr_ctx* ctx, const double* u, double* gx, double* gy) {
  OP_PROLOGUE(false);
  double *du = ctx->fld<double>(F_T), *dx = ctx->fld<double>(F_TX), *dy = ctx->fld<double>(F_TY);
  int rc;
  if ((rc = h2d(ctx, du, u, B))) return rc;
  k_op_grad<<<grid2d(ctx), block2d(), 0, s>>>(du, dx, dy, ctx->H, ctx->W);
  ctx->launches += 1;
  if ((rc = launch_err(ctx, "grad"))) return rc;
  CK(cudaMemcpyAsync(gx, dx, B, cudaMemcpyDeviceToHost, s));
  return d2h_sync(ctx, gy, dy, B);
}

int evr_op_div(evr_ctx* ctx, const double* qx, const double* qy, double* out) {
  OP_PROLOGUE(true);
  double *a = ctx->fld<double>(F_TX), *b = ctx->fld<double>(F_TY), *o = ctx->fld<double>(F_T);
  int rc;
  if ((rc = h2d(ctx, a, qx, B)) || (rc = h2d(ctx, b, qy, B))) return rc;
  k_op_div<<<grid2d(ctx), block2d(), 0, s>>>(a, b, o, ctx->H, ctx->W, 0);
  ctx->launches += 1;
  if ((rc = launch_err(ctx, "div"))) return rc;
  return d2h_sync(ctx, out, o, B);
}

int evr_op_normalize(evr_ctx* ctx, const double* raw, double now, double t_scale, double window,
                     double* t_out) {
  OP_PROLOGUE(false);
  if (!(window > 0)) return fail(ctx, EVR_ERR_INVALID, "t_window must be positive, got %g", window);
  double *r = ctx->fld<double>(F_TX), *t = ctx->fld<double>(F_T);
  int rc;
  if ((rc = h2d(ctx, r, raw, B))) return rc;
  k_op_normalize<<<grid1d(N), kNT, 0, s>>>(r, now, t_scale, window, t, N);
  ctx->launches += 1;
  if ((rc = launch_err(ctx, "normalize"))) return rc;
  return d2h_sync(ctx, t_out, t, B);
}

int evr_op_denoise(evr_ctx* ctx, const double* t_in, double weight, int iterations, double t_scale,
                   double* t_out) {
  OP_PROLOGUE(true);
  if (!(weight > 0)) return fail(ctx, EVR_ERR_INVALID, "denoise weight must be positive, got %g", weight);
  if (iterations < 1) return fail(ctx, EVR_ERR_INVALID, "iterations must be >= 1, got %d", iterations);
  double *t = ctx->fld<double>(F_T), *tu = ctx->fld<double>(F_TU), *tub = ctx->fld<double>(F_TUB);
  double *px = ctx->fld<double>(F_TPX), *py = ctx->fld<double>(F_TPY);
  int rc;
  if ((rc = h2d(ctx, t, t_in, B))) return rc;
  CK(cudaMemcpyAsync(tu, t, B, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpyAsync(tub, t, B, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemsetAsync(px, 0, B, s));
  CK(cudaMemsetAsync(py, 0, B, s));
  const double step = 1.0 / std::sqrt(8.0);
  for (int it = 0; it < iterations; ++it) {
    k_tv_dual<double><<<grid2d(ctx), block2d(), 0, s>>>(tub, px, py, ctx->geo_own(), step);
    k_tv_primal<double><<<grid2d(ctx), block2d(), 0, s>>>(px, py, tu, tub, t, ctx->geo_own(), step,
                                                          step * weight);
  }
  k_tv_finish<double><<<grid1d(N), kNT, 0, s>>>(tu, tub, t_scale, N);
  ctx->launches += 2 * iterations + 1;
  if ((rc = launch_err(ctx, "denoise"))) return rc;
  return d2h_sync(ctx, t_out, tub, B);
}

int evr_op_metric(evr_ctx* ctx, const double* t, double* tx, double* ty, double* G, double* sqrtG) {
  OP_PROLOGUE(false);
  double* dt = ctx->fld<double>(F_T);
  int rc;
  if ((rc = h2d(ctx, dt, t, B))) return rc;
  k_op_metric<<<grid2d(ctx), block2d(), 0, s>>>(dt, ctx->fld<double>(F_TX), ctx->fld<double>(F_TY),
                                                ctx->fld<double>(F_G), ctx->fld<double>(F_SG),
                                                ctx->H, ctx->W);
  ctx->launches += 1;
  if ((rc = launch_err(ctx, "metric"))) return rc;
  CK(cudaMemcpyAsync(tx, ctx->fld<double>(F_TX), B, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(ty, ctx->fld<double>(F_TY), B, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(G, ctx->fld<double>(F_G), B, cudaMemcpyDeviceToHost, s));
  return d2h_sync(ctx, sqrtG, ctx->fld<double>(F_SG), B);
}

// upload a caller MetricField and build the coefficient planes
static int upload_metric(evr_ctx* ctx, const double* tx, const double* ty, const double* G,
                         const double* sqrtG) {
  const size_t B = sizeof(double) * ctx->N;
  int rc;
  if ((rc = h2d(ctx, ctx->fld<double>(F_TX), tx, B)) || (rc = h2d(ctx, ctx->fld<double>(F_TY), ty, B)) ||
      (rc = h2d(ctx, ctx->fld<double>(F_G), G, B)))
    return rc;
  if (sqrtG && (rc = h2d(ctx, ctx->fld<double>(F_SG), sqrtG, B))) return rc;
  k_op_coeffs<<<grid1d(ctx->N), kNT, 0, ctx->stream>>>(ctx->fld<double>(F_TX), ctx->fld<double>(F_TY),
                                                       ctx->fld<double>(F_G), coefs<double>(ctx), ctx->N);
  ctx->launches += 1;
  return launch_err(ctx, "coeffs");
}

int evr_op_coeffs(evr_ctx* ctx, const double* tx, const double* ty, const double* G, double* out5) {
  OP_PROLOGUE(false);
  int rc;
  if ((rc = upload_metric(ctx, tx, ty, G, nullptr))) return rc;
  const int fl[5] = {F_A11, F_A12, F_A22, F_A31, F_A32};
  for (int m = 0; m < 5; ++m)
    CK(cudaMemcpyAsync(out5 + m * N, ctx->fld<double>(fl[m]), B, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return EVR_OK;
}

int evr_op_surface_gradient(evr_ctx* ctx, const double* u, const double* tx, const double* ty,
                            const double* G, double* out) {
  OP_PROLOGUE(false);
  int rc;
  if ((rc = upload_metric(ctx, tx, ty, G, nullptr))) return rc;
  double* du = ctx->fld<double>(F_T);
  if ((rc = h2d(ctx, du, u, B))) return rc;
  k_op_surface_gradient<<<grid2d(ctx), block2d(), 0, s>>>(du, coefs<double>(ctx), ctx->aos_a, ctx->H,
                                                          ctx->W);
  ctx->launches += 1;
  if ((rc = launch_err(ctx, "surface_gradient"))) return rc;
  return d2h_sync(ctx, out, ctx->aos_a, 3 * B);
}

int evr_op_surface_gradient_adjoint(evr_ctx* ctx, const double* p, const double* tx, const double* ty,
                                    const double* G, double* out) {
  OP_PROLOGUE(true);
  int rc;
  if ((rc = upload_metric(ctx, tx, ty, G, nullptr))) return rc;
  if ((rc = h2d(ctx, ctx->aos_a, p, 3 * B))) return rc;
  double *qx = ctx->fld<double>(F_TU), *qy = ctx->fld<double>(F_TUB), *o = ctx->fld<double>(F_T);
  k_op_q<<<grid1d(N), kNT, 0, s>>>(ctx->aos_a, coefs<double>(ctx), qx, qy, N);
  k_op_div<<<grid2d(ctx), block2d(), 0, s>>>(qx, qy, o, ctx->H, ctx->W, 1);
  ctx->launches += 2;
  if ((rc = launch_err(ctx, "surface_gradient_adjoint"))) return rc;
  return d2h_sync(ctx, out, o, B);
}

int evr_op_prox_data(evr_ctx* ctx, const double* u_bar, const double* f, const double* sqrtG,
                     double tau, double lam, double u_min, double u_max, double* out) {
  OP_PROLOGUE(false);
  double *a = ctx->fld<double>(F_T), *b = ctx->fld<double>(F_TU), *c = ctx->fld<double>(F_SG),
         *o = ctx->fld<double>(F_TUB);
  int rc;
  if ((rc = h2d(ctx, a, u_bar, B)) || (rc = h2d(ctx, b, f, B)) || (rc = h2d(ctx, c, sqrtG, B)))
    return rc;
  k_op_prox_data<<<grid1d(N), kNT, 0, s>>>(a, b, c, tau * lam, u_min, u_max, o, N);
  ctx->launches += 1;
  if ((rc = launch_err(ctx, "prox_data"))) return rc;
  return d2h_sync(ctx, out, o, B);
}

int evr_op_prox_dual(evr_ctx* ctx, const double* p, const double* sqrtG, double* out) {
  OP_PROLOGUE(false);
  int rc;
  if ((rc = h2d(ctx, ctx->aos_a, p, 3 * B)) || (rc = h2d(ctx, ctx->fld<double>(F_SG), sqrtG, B)))
    return rc;
  k_op_prox_dual<<<grid1d(N), kNT, 0, s>>>(ctx->aos_a, ctx->fld<double>(F_SG), ctx->aos_b, N);
  ctx->launches += 1;
  if ((rc = launch_err(ctx, "prox_dual"))) return rc;
  return d2h_sync(ctx, out, ctx->aos_b, 3 * B);
}

int evr_op_energy(evr_ctx* ctx, const double* u, const double* f, const double* tx, const double* ty,
                  const double* G, const double* sqrtG, double lam, double* out) {
  OP_PROLOGUE(false);
  int rc;
  if ((rc = upload_metric(ctx, tx, ty, G, sqrtG))) return rc;
  if ((rc = h2d(ctx, ctx->fld<double>(F_T), u, B)) || (rc = h2d(ctx, ctx->aos_a, f, B))) return rc;
  const int nb = red_blocks(N);
  k_energy_partial<double, kNT><<<nb, kNT, 0, s>>>(ctx->fld<double>(F_T), ctx->aos_a, coefs<double>(ctx),
                                                   ctx->fld<double>(F_G), ctx->fld<double>(F_SG),
                                                   ctx->H, ctx->W, ctx->part);
  k_energy_final<kNT><<<1, kNT, 0, s>>>(ctx->part, nb, lam, ctx->d_scalar);
  ctx->launches += 2;
  if ((rc = launch_err(ctx, "energy"))) return rc;
  return d2h_sync(ctx, out, ctx->d_scalar, sizeof(double));
}

int evr_op_pd_solve(evr_ctx* ctx, const evr_config* cfg, const double* f, const double* tx,
                    const double* ty, const double* G, const double* sqrtG, const double* u_init,
                    const double* p_init, double* u_out, double* p_out, evr_solve_info* info,
                    double* energy_trace, double* rel_trace) {
  OP_PROLOGUE(true);
  if (!cfg || cfg->max_iterations < 1) return fail(ctx, EVR_ERR_INVALID, "bad solver config");
  int rc;
  if ((rc = upload_metric(ctx, tx, ty, G, sqrtG))) return rc;
  // the op API works on scratch copies: stash the stream state's f aside
  double* fdev = ctx->aos_b;  // first N doubles of the (H,W,3) scratch
  if ((rc = h2d(ctx, fdev, f, B))) return rc;
  if ((rc = h2d(ctx, ctx->fld<double>(F_U), u_init ? u_init : f, B))) return rc;
  if (p_init) {
    if ((rc = h2d(ctx, ctx->aos_a, p_init, 3 * B))) return rc;
    k_aos_to_planes<double><<<grid1d(N), kNT, 0, s>>>(ctx->aos_a, ctx->fld<double>(F_P1),
                                                      ctx->fld<double>(F_P2), ctx->fld<double>(F_P3), N);
  } else {
    for (int k : {F_P1, F_P2, F_P3}) CK(cudaMemsetAsync(ctx->fld<double>(k), 0, B, s));
  }
  k_solver_setup<double><<<grid1d(N), kNT, 0, s>>>(
      ctx->fld<double>(F_TX), ctx->fld<double>(F_TY), ctx->fld<double>(F_G), ctx->fld<double>(F_SG),
      fdev, coefs<double>(ctx), ctx->fld<double>(F_BETA), ctx->fld<double>(F_FB), N,
      cfg->tau * cfg->lam, 0);
  ctx->launches += 2;
  if ((rc = launch_err(ctx, "pd setup"))) return rc;
  double* saved_f = ctx->f;
  ctx->f = fdev;  // energy trace reads f; the fused list's epilogue writes f = u there
  if (!energy_trace && !rel_trace && !ctx->banded) {
    // no per-iteration trace: the streaming engine's solve list on this
    // context's planes -- temporally blocked tiles (rel_change of the last
    // iteration folded on the device) or, with a tolerance, one march launch
    // + rel_change per iteration behind the device stop flag; no host round
    // trip per iteration either way
    const evr_config saved_cfg = ctx->cfg;
    ctx->cfg = *cfg;
    int n = 0;
    for (const Step& st : packet_steps(ctx->cfg, 1, true, ctx_tile_k(ctx), false))
      n += launch_step<double>(ctx, st);
    ctx->cfg = saved_cfg;
    ctx->launches += n;
    rc = launch_err(ctx, "pd solve");
    if (!rc && info) {
      CK(cudaMemcpyAsync(ctx->h_info, ctx->d_info, sizeof(evr_solve_info), cudaMemcpyDeviceToHost,
                         s));
      CK(cudaStreamSynchronize(s));
      *info = *ctx->h_info;
    }
  } else {
    rc = solve_host_loop<double>(ctx, *cfg, info, energy_trace, rel_trace, false);
  }
  ctx->f = saved_f;
  if (rc) return rc;
  k_planes_to_aos<double><<<grid1d(N), kNT, 0, s>>>(ctx->fld<double>(F_P1), ctx->fld<double>(F_P2),
                                                    ctx->fld<double>(F_P3), ctx->aos_a, N);
  ctx->launches += 1;
  CK(cudaMemcpyAsync(u_out, ctx->fld<double>(F_U), B, cudaMemcpyDeviceToHost, s));
  return d2h_sync(ctx, p_out, ctx->aos_a, 3 * B);
}

int evr_op_to_gray(evr_ctx* ctx, const double* image, double lo, double hi, uint8_t* out) {
  OP_PROLOGUE(false);
  if (!(hi > lo)) return fail(ctx, EVR_ERR_INVALID, "bounds must satisfy u_min < u_max");
  int rc;
  if ((rc = h2d(ctx, ctx->fld<double>(F_T), image, B))) return rc;
  uint8_t* d = reinterpret_cast<uint8_t*>(ctx->aos_a);
  k_to_gray<double><<<grid1d(N), kNT, 0, s>>>(ctx->fld<double>(F_T), lo, hi, d, N);
  ctx->launches += 1;
  if ((rc = launch_err(ctx, "to_gray"))) return rc;
  return d2h_sync(ctx, out, d, (size_t)N);
}

int evr_op_rof_solve(evr_ctx* ctx, const double* f, const double* tx, const double* ty, const double* G,
                     const double* sqrtG, double lam, int iterations, double* u_out) {
  OP_PROLOGUE(true);
  if (!(lam > 0)) return fail(ctx, EVR_ERR_INVALID, "lam must be positive, got %g", lam);
  int rc;
  if ((rc = upload_metric(ctx, tx, ty, G, sqrtG))) return rc;
  double* fdev = ctx->aos_b;
  if ((rc = h2d(ctx, fdev, f, B))) return rc;
  CK(cudaMemcpyAsync(ctx->fld<double>(F_U), fdev, B, cudaMemcpyDeviceToDevice, s));
  for (int k : {F_P1, F_P2, F_P3}) CK(cudaMemsetAsync(ctx->fld<double>(k), 0, B, s));
  const double step = 1.0 / std::sqrt(8.0 + 4.0 * std::sqrt(2.0));  // solve.py:38, :277
  k_solver_setup<double><<<grid1d(N), kNT, 0, s>>>(
      ctx->fld<double>(F_TX), ctx->fld<double>(F_TY), ctx->fld<double>(F_G), ctx->fld<double>(F_SG),
      fdev, coefs<double>(ctx), ctx->fld<double>(F_BETA), ctx->fld<double>(F_FB), N, step * lam, 1);
  if (iterations >= 2 && !ctx->banded) {  // the tiles (K iterations per launch)
    double* uo = op_tile_solve<DT_ROF>(ctx, iterations, nullptr, step);
    ctx->launches += 1;
    if ((rc = launch_err(ctx, "rof"))) return rc;
    return d2h_sync(ctx, u_out, uo, B);
  }
  double* bufs[2] = {ctx->fld<double>(F_U), ctx->fld<double>(F_UN)};
  for (int it = 0; it < iterations; ++it) {
    double* cur = bufs[it & 1];
    double* nxt = bufs[(it + 1) & 1];
    double* v = ctx->fld<double>(F_V);
    k_rof_primal<double><<<grid2d(ctx), block2d(), 0, s>>>(
        ctx->fld<double>(F_P1), ctx->fld<double>(F_P2), ctx->fld<double>(F_P3), coefs<double>(ctx),
        cur, ctx->fld<double>(F_BETA), ctx->fld<double>(F_FB), nxt, v, ctx->geo_own(), step);
    k_pd_dual<double><<<grid2d(ctx), block2d(), 0, s>>>(v, ctx->fld<double>(F_P1), ctx->fld<double>(F_P2),
                                                        ctx->fld<double>(F_P3), coefs<double>(ctx),
                                                        ctx->fld<double>(F_SG), ctx->geo_own(), step);
  }
  ctx->launches += 1 + 2 * (int64_t)iterations;
  if ((rc = launch_err(ctx, "rof"))) return rc;
  return d2h_sync(ctx, u_out, bufs[iterations & 1], B);
}

// Manifold TV + L1 data term (not in the reference; parity unpinned, CPU
// restatement oracle/evr_oracle.c evo_l1_solve): rof_manifold_solve's loop
// (solve.py:264-293) with the L1 prox.
int evr_op_l1_solve(evr_ctx* ctx, const double* f, const double* tx, const double* ty,
                    const double* G, const double* sqrtG, double lam, int iterations,
                    double* u_out) {
  OP_PROLOGUE(true);
  if (!(lam > 0)) return fail(ctx, EVR_ERR_INVALID, "lam must be positive, got %g", lam);
  int rc;
  if ((rc = upload_metric(ctx, tx, ty, G, sqrtG))) return rc;
  double* fdev = ctx->aos_b;
  if ((rc = h2d(ctx, fdev, f, B))) return rc;
  CK(cudaMemcpyAsync(ctx->fld<double>(F_U), fdev, B, cudaMemcpyDeviceToDevice, s));
  for (int k : {F_P1, F_P2, F_P3}) CK(cudaMemsetAsync(ctx->fld<double>(k), 0, B, s));
  const double step = 1.0 / std::sqrt(8.0 + 4.0 * std::sqrt(2.0));
  k_solver_setup<double><<<grid1d(N), kNT, 0, s>>>(
      ctx->fld<double>(F_TX), ctx->fld<double>(F_TY), ctx->fld<double>(F_G), ctx->fld<double>(F_SG),
      fdev, coefs<double>(ctx), ctx->fld<double>(F_BETA), ctx->fld<double>(F_FB), N, step * lam, 0);
  if (iterations >= 2 && !ctx->banded) {  // the tiles: beta = (tau lam) sqrtG, f in the last slot
    double* uo = op_tile_solve<DT_L1>(ctx, iterations, fdev, step);
    ctx->launches += 1;
    if ((rc = launch_err(ctx, "l1"))) return rc;
    return d2h_sync(ctx, u_out, uo, B);
  }
  double* bufs[2] = {ctx->fld<double>(F_U), ctx->fld<double>(F_UN)};
  for (int it = 0; it < iterations; ++it) {
    double* v = ctx->fld<double>(F_V);
    k_l1_primal<double><<<grid2d(ctx), block2d(), 0, s>>>(
        ctx->fld<double>(F_P1), ctx->fld<double>(F_P2), ctx->fld<double>(F_P3), coefs<double>(ctx),
        bufs[it & 1], ctx->fld<double>(F_SG), fdev, bufs[(it + 1) & 1], v, ctx->geo_own(), step,
        step * lam);
    k_pd_dual<double><<<grid2d(ctx), block2d(), 0, s>>>(v, ctx->fld<double>(F_P1), ctx->fld<double>(F_P2),
                                                        ctx->fld<double>(F_P3), coefs<double>(ctx),
                                                        ctx->fld<double>(F_SG), ctx->geo_own(), step);
  }
  ctx->launches += 1 + 2 * (int64_t)iterations;
  if ((rc = launch_err(ctx, "l1"))) return rc;
  return d2h_sync(ctx, u_out, bufs[iterations & 1], B);
}

// Second-order manifold TGV with a KL / ROF / L1 data term (not in the
// reference; parity unpinned, CPU restatement oracle/evr_oracle.c
// evo_tgv_solve).  Cold start u = f, w = p = Q = 0; tau = sigma =
// 1/sqrt(17 + 4*sqrt2).  w_out (H, W, 2) may be NULL.
int evr_op_tgv_solve(evr_ctx* ctx, const double* f, const double* tx, const double* ty,
                     const double* G, const double* sqrtG, double lam, double alpha0,
                     double alpha1, int data_term, double u_min, double u_max, int iterations,
                     double* u_out, double* w_out) {
  OP_PROLOGUE(true);
  if (!(lam > 0)) return fail(ctx, EVR_ERR_INVALID, "lam must be positive, got %g", lam);
  if (!(alpha0 > 0) || !(alpha1 > 0))
    return fail(ctx, EVR_ERR_INVALID, "TGV weights must be positive, got alpha0=%g alpha1=%g",
                alpha0, alpha1);
  if (data_term < 0 || data_term > 2)
    return fail(ctx, EVR_ERR_INVALID, "unknown data term %d", data_term);
  if (data_term == 0 && !(u_min < u_max))
    return fail(ctx, EVR_ERR_INVALID, "box must satisfy u_min < u_max");
  int rc;
  // the ping-pong sets of k_tgv_iter: w1, w2 and q11, q22, q12 twice, plus
  // the second dual set (the first is F_P1..F_P3)
  if (!ctx->tgv) CK(cudaMalloc(&ctx->tgv, 13 * B));
  if ((rc = upload_metric(ctx, tx, ty, G, sqrtG))) return rc;
  double* fdev = ctx->aos_b;
  if ((rc = h2d(ctx, fdev, f, B))) return rc;
  CK(cudaMemcpyAsync(ctx->fld<double>(F_U), fdev, B, cudaMemcpyDeviceToDevice, s));
  for (int k : {F_P1, F_P2, F_P3}) CK(cudaMemsetAsync(ctx->fld<double>(k), 0, B, s));
  double* t = ctx->tgv;
  CK(cudaMemsetAsync(t, 0, 13 * B, s));
  const double step = 1.0 / std::sqrt(17.0 + 4.0 * std::sqrt(2.0));
  k_solver_setup<double><<<grid1d(N), kNT, 0, s>>>(
      ctx->fld<double>(F_TX), ctx->fld<double>(F_TY), ctx->fld<double>(F_G), ctx->fld<double>(F_SG),
      fdev, coefs<double>(ctx), ctx->fld<double>(F_BETA), ctx->fld<double>(F_FB), N, step * lam, 0);
  const TgvSet<double> sets[2] = {
      {ctx->fld<double>(F_U), t, t + N, ctx->fld<double>(F_P1), ctx->fld<double>(F_P2),
       ctx->fld<double>(F_P3), t + 4 * N, t + 5 * N, t + 6 * N},
      {ctx->fld<double>(F_UN), t + 2 * N, t + 3 * N, t + 10 * N, t + 11 * N, t + 12 * N,
       t + 7 * N, t + 8 * N, t + 9 * N}};
  for (int it = 0; it < iterations; ++it) {
    const int a = it & 1;
    k_tgv_iter<double><<<grid2d(ctx), block2d(), 0, s>>>(
        sets[a], sets[a ^ 1], coefs<double>(ctx), ctx->fld<double>(F_SG), fdev, ctx->geo_own(),
        step, step, step * lam, data_term, u_min, u_max, alpha0, alpha1);
  }
  ctx->launches += 1 + (int64_t)iterations;
  if ((rc = launch_err(ctx, "tgv"))) return rc;
  double* wfin[2] = {sets[iterations & 1].w1, sets[iterations & 1].w2};
  double* ufin = sets[iterations & 1].u;
  if (w_out) {  // (H, W, 2) interleaved
    CK(cudaMemcpy2DAsync(w_out, 2 * sizeof(double), wfin[0], sizeof(double), sizeof(double), N,
                         cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpy2DAsync(w_out + 1, 2 * sizeof(double), wfin[1], sizeof(double), sizeof(double),
                         N, cudaMemcpyDeviceToHost, s));
  }
  return d2h_sync(ctx, u_out, ufin, B);
}

}  // extern "C"

// =========================================================================
// evr_group: one sensor split into row bands over several contexts (one per
// GPU, or several on one GPU), the megapixel configuration of SURVEY.md
// 8(e).  Every band runs the streaming step list in lock step; after each
// step the boundary rows its neighbours need travel as device-to-device
// (peer, over NVLink between GPUs) copies ordered by CUDA events:
//   after NORM / TVP : u_bar  of a band's first row -> the band above's halo below
//   after TVD        : py     of a band's last row  -> the band below's halo above
//   after TVFIN      : t      both ways (the metric's ty and the halo-row q)
//   after METRIC/PDD : p1..p3 of a band's last row  -> the band below's halo above
//   after PDP        : v      of a band's first row -> the band above's halo below
// No reduction happens inside the iterations; rel_change folds the bands'
// partial sums on the host.  Every boundary rule uses global row indices,
// so the result is bit-identical to the single-context run.
// =========================================================================
struct evr_group {
  int n = 0, H = 0, W = 0, prec = EVR_PREC_F64;
  // fused list: the iteration kernels read the neighbours' halo rows in place
  // (needs peer access between neighbouring GPUs); else split list + copies
  bool fused = true;
  // the whole per-packet step list of all bands as one CUDA graph (launched
  // on band 0's stream; cross-band / cross-device order from captured events)
  cudaGraphExec_t graph = nullptr;
  bool graph_failed = false;
  std::vector<int64_t> graph_launches, graph_cap;
  std::vector<cudaEvent_t> fork;  // per band: graph fork / join / host-order events
  std::vector<evr_ctx*> band;
  std::vector<int> y0;
  std::vector<cudaEvent_t> done, copied;
  evr_config cfg{};
  bool cfg_set = false;
  std::string err;
};

namespace {

void drop_group_graph(evr_group* g) {
  if (g && g->graph) {
    cudaSetDevice(g->band[0]->device);
    cudaGraphExecDestroy(g->graph);
    g->graph = nullptr;
  }
}

int gfail(evr_group* g, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (g) g->err = buf;
  return code;
}

#define GCK(call)                                                                      \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return gfail(grp, EVR_ERR_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

#define GBAND(b, rc_expr)                                                              \
  do {                                                                                 \
    int rc_ = (rc_expr);                                                               \
    if (rc_) return gfail(grp, rc_, "band %d: %s", (b), grp->band[b]->err.c_str());   \
  } while (0)

// copy one row of `field` (T elements) from band src local row rs into band
// dst local row rd, on dst's stream after src's last step
int copy_row(evr_group* grp, int dst, int rd, int src, int rs, int field) {
  evr_ctx* D = grp->band[dst];
  evr_ctx* S = grp->band[src];
  const size_t es = grp->prec == EVR_PREC_F64 ? 8 : 4;
  char* dp = D->slab + D->field_stride * field + (size_t)rd * grp->W * es;
  const char* sp = S->slab + S->field_stride * field + (size_t)rs * grp->W * es;
  GCK(cudaSetDevice(D->device));
  GCK(cudaStreamWaitEvent(D->stream, grp->done[src], 0));
  // unified addressing: a peer (NVLink) copy across GPUs, a D2D copy on one;
  // unlike cudaMemcpyPeerAsync it can be captured into the group's graph
  GCK(cudaMemcpyAsync(dp, sp, grp->W * es, cudaMemcpyDefault, D->stream));
  return EVR_OK;
}

// halo exchanges that follow a step (see the table above)
int exchange_after(evr_group* grp, int kind) {
  const int n = grp->n;
  auto from_below = [&](int field) -> int {  // first own row of b+1 -> halo below of b
    for (int b = 0; b + 1 < n; ++b) {
      int rc = copy_row(grp, b, grp->band[b]->own_hi + 1, b + 1, grp->band[b + 1]->own_lo, field);
      if (rc) return rc;
    }
    return EVR_OK;
  };
  auto from_above = [&](int field) -> int {  // last own row of b-1 -> halo above of b
    for (int b = 1; b < n; ++b) {
      int rc = copy_row(grp, b, 0, b - 1, grp->band[b - 1]->own_hi, field);
      if (rc) return rc;
    }
    return EVR_OK;
  };
  int rc = EVR_OK;
  switch (kind) {
    case ST_NORM:
    case ST_TVP:
      rc = from_below(F_TUB);
      break;
    case ST_TVD:
      rc = from_above(F_TPY);
      break;
    case ST_TVFIN:
    case ST_TVFINF:  // the metric's slopes read the neighbours' denoised rows
      if (!(rc = from_above(F_T))) rc = from_below(F_T);
      break;
    case ST_METRIC:
    case ST_PDD:
      for (int f : {F_P1, F_P2, F_P3})
        if ((rc = from_above(f))) break;
      break;
    case ST_PDP:
      rc = from_below(F_V);
      break;
    default:
      break;
  }
  return rc;
}

template <class T> int group_packet(evr_group* grp) {
  // fused bands run the tiles too (K rows of each neighbour read in place)
  // when every band has at least K own rows
  int tk = grp->fused ? tile_k(grp->prec) : 1;
  for (const evr_ctx* c : grp->band)
    if (c->own_hi - c->own_lo + 1 < tk) tk = 1;
  const std::vector<Step> steps = packet_steps(grp->cfg, 2, grp->fused, tk);
  const int n = grp->n;
  for (const Step& st : steps) {
    for (int b = 0; b < n; ++b) {
      evr_ctx* ctx = grp->band[b];
      GCK(cudaSetDevice(ctx->device));
      // neighbours must have copied this band's rows before it overwrites them
      if (b > 0) GCK(cudaStreamWaitEvent(ctx->stream, grp->copied[b - 1], 0));
      if (b + 1 < n) GCK(cudaStreamWaitEvent(ctx->stream, grp->copied[b + 1], 0));
      ctx->launches += launch_step<T>(ctx, st);
      GBAND(b, launch_err(ctx, "group step"));
      GCK(cudaEventRecord(grp->done[b], ctx->stream));
    }
    int rc = exchange_after(grp, st.kind);
    if (rc) return rc;
    for (int b = 0; b < n; ++b) {
      GCK(cudaSetDevice(grp->band[b]->device));
      GCK(cudaEventRecord(grp->copied[b], grp->band[b]->stream));
    }
  }
  return EVR_OK;
}

// host order: every band stream (staging copies) before `dst`
int group_order(evr_group* grp, cudaStream_t dst, int dst_dev) {
  for (int b = 0; b < grp->n; ++b) {
    evr_ctx* c = grp->band[b];
    if (c->stream == dst) continue;
    GCK(cudaSetDevice(c->device));
    GCK(cudaEventRecord(grp->fork[b], c->stream));
    GCK(cudaSetDevice(dst_dev));
    GCK(cudaStreamWaitEvent(dst, grp->fork[b], 0));
  }
  return EVR_OK;
}

// Capture the step list of all bands once (fork from band 0's stream, join
// back into it) and replay it per packet; the eager loop is the fallback
// when capture is refused (e.g. a driver without multi-device capture).
int group_run(evr_group* grp) {
  evr_ctx* c0 = grp->band[0];
  for (int b = 0; b < grp->n; ++b)  // staging buffers baked into the graph
    if (grp->graph && grp->graph_cap[b] != grp->band[b]->ev_cap) drop_group_graph(grp);
  if (!grp->graph && !grp->graph_failed) {
    std::vector<int64_t> before(grp->n);
    for (int b = 0; b < grp->n; ++b) before[b] = grp->band[b]->launches;
    GCK(cudaSetDevice(c0->device));
    cudaGraph_t g = nullptr;
    bool ok = cudaStreamBeginCapture(c0->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    int rc = EVR_OK;
    if (ok) {
      GCK(cudaEventRecord(grp->fork[0], c0->stream));
      for (int b = 0; b < grp->n; ++b) {
        evr_ctx* c = grp->band[b];
        cudaSetDevice(c->device);
        if (b > 0) ok &= cudaStreamWaitEvent(c->stream, grp->fork[0], 0) == cudaSuccess;
        ok &= cudaEventRecord(grp->copied[b], c->stream) == cudaSuccess;
      }
      if (ok)
        rc = grp->prec == EVR_PREC_F64 ? group_packet<double>(grp) : group_packet<float>(grp);
      for (int b = 1; b < grp->n && ok && !rc; ++b) {
        evr_ctx* c = grp->band[b];
        cudaSetDevice(c->device);
        ok &= cudaEventRecord(grp->done[b], c->stream) == cudaSuccess;
        cudaSetDevice(c0->device);
        ok &= cudaStreamWaitEvent(c0->stream, grp->done[b], 0) == cudaSuccess;
      }
      cudaSetDevice(c0->device);
      ok &= cudaStreamEndCapture(c0->stream, &g) == cudaSuccess;
      ok = ok && !rc && cudaGraphInstantiate(&grp->graph, g, 0) == cudaSuccess;
      if (g) cudaGraphDestroy(g);
    }
    cudaGetLastError();
    grp->graph_launches.assign(grp->n, 0);
    grp->graph_cap.assign(grp->n, 0);
    for (int b = 0; b < grp->n; ++b) {
      grp->graph_launches[b] = grp->band[b]->launches - before[b];
      grp->band[b]->launches = before[b];
      grp->graph_cap[b] = grp->band[b]->ev_cap;
    }
    if (!ok || rc) {  // capture refused: run (and keep running) the eager loop
      if (grp->graph) cudaGraphExecDestroy(grp->graph);
      grp->graph = nullptr;
      grp->graph_failed = true;
    }
  }
  if (!grp->graph)
    return grp->prec == EVR_PREC_F64 ? group_packet<double>(grp) : group_packet<float>(grp);
  int rc = group_order(grp, c0->stream, c0->device);  // staging copies first
  if (rc) return rc;
  GCK(cudaSetDevice(c0->device));
  GCK(cudaGraphLaunch(grp->graph, c0->stream));
  GCK(cudaEventRecord(grp->fork[0], c0->stream));
  for (int b = 0; b < grp->n; ++b) {  // later per-band work after the graph
    evr_ctx* c = grp->band[b];
    c->launches += grp->graph_launches[b];
    if (b == 0) continue;
    GCK(cudaSetDevice(c->device));
    GCK(cudaStreamWaitEvent(c->stream, grp->fork[0], 0));
  }
  return EVR_OK;
}

}  // namespace

extern "C" {

int evr_group_create(evr_group** out, int n_bands, const int* devices, int height, int width,
                     int precision) {
  if (!out || n_bands < 1 || height < 2 || width < 2 || n_bands > height)
    return EVR_ERR_INVALID;
  evr_group* grp = new evr_group();
  grp->n = n_bands;
  grp->H = height;
  grp->W = width;
  grp->prec = precision;
  for (int b = 0; b < n_bands; ++b) {
    const int y0 = (int)((int64_t)height * b / n_bands);
    const int y1 = (int)((int64_t)height * (b + 1) / n_bands);
    const int dev = devices ? devices[b] : 0;
    evr_ctx* ctx = nullptr;
    int rc = evr_create(&ctx, dev, y1 - y0 + 2, width, precision);
    if (rc) {
      evr_group_destroy(grp);
      return rc;
    }
    ctx->banded = true;
    ctx->row0 = y0 - 1;
    ctx->Htot = height;
    ctx->own_lo = 1;
    ctx->own_hi = y1 - y0;
    grp->band.push_back(ctx);
    grp->y0.push_back(y0);
    cudaSetDevice(dev);
    cudaEvent_t e1, e2;
    cudaEventCreateWithFlags(&e1, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&e2, cudaEventDisableTiming);
    cudaEventRecord(e2, ctx->stream);
    grp->done.push_back(e1);
    grp->copied.push_back(e2);
    cudaEvent_t e3;
    cudaEventCreateWithFlags(&e3, cudaEventDisableTiming);
    grp->fork.push_back(e3);
  }
  // peer access between neighbouring GPUs (NVLink); same-device bands need none
  for (int b = 0; b + 1 < n_bands; ++b) {
    const int d0 = grp->band[b]->device, d1 = grp->band[b + 1]->device;
    if (d0 == d1) continue;
    int ok = 0;
    cudaDeviceCanAccessPeer(&ok, d0, d1);
    if (ok) {
      cudaSetDevice(d0);
      cudaDeviceEnablePeerAccess(d1, 0);
      cudaSetDevice(d1);
      cudaDeviceEnablePeerAccess(d0, 0);
      cudaGetLastError();  // already-enabled is fine
    } else {
      grp->fused = false;  // no peer loads: halo rows travel as copies
    }
  }
  if (const char* e = getenv("EVR_GROUP_SPLIT"))  // A/B and test hook: split list + copies
    if (e[0] == '1') grp->fused = false;
  if (grp->fused)
    for (int b = 0; b < n_bands; ++b) {
      grp->band[b]->nb_up = b > 0 ? grp->band[b - 1] : nullptr;
      grp->band[b]->nb_dn = b + 1 < n_bands ? grp->band[b + 1] : nullptr;
    }
  *out = grp;
  return EVR_OK;
}

void evr_group_destroy(evr_group* grp) {
  if (!grp) return;
  drop_group_graph(grp);
  for (size_t b = 0; b < grp->band.size(); ++b) {
    cudaSetDevice(grp->band[b]->device);
    if (b < grp->done.size()) cudaEventDestroy(grp->done[b]);
    if (b < grp->copied.size()) cudaEventDestroy(grp->copied[b]);
    if (b < grp->fork.size()) cudaEventDestroy(grp->fork[b]);
    evr_destroy(grp->band[b]);
  }
  delete grp;
}

const char* evr_group_last_error(const evr_group* grp) {
  return grp ? grp->err.c_str() : "null group";
}

int evr_group_band(evr_group* grp, int b, int* y0, int* y1, int* device) {
  if (!grp || b < 0 || b >= grp->n) return EVR_ERR_INVALID;
  if (y0) *y0 = grp->y0[b];
  if (y1) *y1 = grp->y0[b] + grp->band[b]->own_hi;
  if (device) *device = grp->band[b]->device;
  return EVR_OK;
}

int evr_group_set_config(evr_group* grp, const evr_config* cfg) {
  if (!grp || !cfg) return EVR_ERR_INVALID;
  if (cfg->convergence_tol > 0)
    return gfail(grp, EVR_ERR_UNSUPPORTED, "banded solve runs fixed iterations only");
  evr_config c = *cfg;
  c.engine = EVR_ENGINE_STREAMING;
  for (int b = 0; b < grp->n; ++b) GBAND(b, evr_set_config(grp->band[b], &c));
  grp->cfg = c;
  grp->cfg_set = true;
  drop_group_graph(grp);
  return EVR_OK;
}

int evr_group_init_state(evr_group* grp) {
  if (!grp) return EVR_ERR_INVALID;
  for (int b = 0; b < grp->n; ++b) GBAND(b, evr_init_state(grp->band[b]));
  return EVR_OK;
}

// full-sensor host arrays; band b reads / writes its own rows
int evr_group_set_state(evr_group* grp, const double* u, const double* f, const int64_t* raw,
                        const double* p) {
  if (!grp) return EVR_ERR_INVALID;
  for (int b = 0; b < grp->n; ++b) {
    const int64_t o = (int64_t)grp->y0[b] * grp->W;
    GBAND(b, evr_set_state(grp->band[b], u ? u + o : nullptr, f ? f + o : nullptr,
                           raw ? raw + o : nullptr, p ? p + 3 * o : nullptr));
  }
  return EVR_OK;
}

int evr_group_get_state(evr_group* grp, double* u, double* f, int64_t* raw, double* p) {
  if (!grp) return EVR_ERR_INVALID;
  for (int b = 0; b < grp->n; ++b) {
    const int64_t o = (int64_t)grp->y0[b] * grp->W;
    GBAND(b, evr_get_state(grp->band[b], u ? u + o : nullptr, f ? f + o : nullptr,
                           raw ? raw + o : nullptr, p ? p + 3 * o : nullptr));
  }
  return EVR_OK;
}

int evr_group_process_packet(evr_group* grp, const evr_event* events, int64_t n, double window,
                             evr_solve_info* info) {
  if (!grp) return EVR_ERR_INVALID;
  if (!grp->cfg_set) return gfail(grp, EVR_ERR_INVALID, "evr_group_set_config has not been called");
  if (n <= 0 || !events) return gfail(grp, EVR_ERR_INVALID, "empty packet");
  for (int b = 0; b < grp->n; ++b) {
    evr_ctx* ctx = grp->band[b];
    cudaSetDevice(ctx->device);
    GBAND(b, stage_host_packet(ctx, events, n, window));
  }
  int rc = group_run(grp);
  if (rc) return rc;
  double d = 0.0, o = 0.0;
  int iters = 0;
  for (int b = 0; b < grp->n; ++b) {
    evr_ctx* ctx = grp->band[b];
    GCK(cudaSetDevice(ctx->device));
    double sums[2];
    GCK(cudaMemcpyAsync(sums, ctx->d_scalar + 2, sizeof sums, cudaMemcpyDeviceToHost, ctx->stream));
    GCK(cudaMemcpyAsync(ctx->h_info, ctx->d_info, sizeof(evr_solve_info), cudaMemcpyDeviceToHost,
                        ctx->stream));
    GCK(cudaStreamSynchronize(ctx->stream));
    GBAND(b, check_err_flag(ctx));
    d += sums[0];
    o += sums[1];
    iters = ctx->h_info->iterations;
  }
  if (info) {
    const double den = std::sqrt(o);
    info->iterations = iters;
    info->rel_change = std::sqrt(d) / (den > 1e-30 ? den : 1e-30);
  }
  return EVR_OK;
}

int evr_group_get_frame(evr_group* grp, double* u_out) {
  return evr_group_get_state(grp, u_out, nullptr, nullptr, nullptr);
}

int64_t evr_group_launch_count(const evr_group* grp) {
  int64_t n = 0;
  if (grp)
    for (auto* c : grp->band) n += c->launches;
  return n;
}

}  // extern "C"
