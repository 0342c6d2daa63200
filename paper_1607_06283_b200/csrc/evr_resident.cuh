// evr_resident.cuh -- the resident engine: ONE persistent kernel per event
// packet, the whole of process_packet (pipeline.py:142-171) in one launch.
//
// Decomposition.  CTA b of a cooperative grid (<= 1 CTA per SM) owns the
// row band [r0, r1) of the sensor (full width, equal band heights).  Every
// per-pixel field of the band -- plus one halo row above (r0-1) and one
// below (r1) -- lives in a private frame of planes in shared memory
// (PLANES_SMEM; the global-memory frame form is retired, `frames` stays
// unused).  Global memory outside the frame is touched only to load the state at the start, to exchange two
// boundary rows per iteration, and to write the state back at the end.
//
// Thread mapping.  Thread t owns sensor column(s) j = t, t+NT, ... and walks
// its column's band rows CH at a time, every input of a chunk gathered into
// registers first, so the rows' float64 div/sqrt chains are independent
// instructions the scheduler overlaps (ILP = CH).
//
// One neighbour exchange per iteration.  Each iteration recomputes on its
// halo rows what it would otherwise have to wait for a second time
// (SURVEY.md Appendix A.6, B.8-B.9):
//   TV-L1 (dual first): the dual update is also run on halo row r0-1, so
//     the primal needs no fresh px/py from the CTA above; only u_bar of the
//     neighbours' boundary rows is exchanged.
//   KL primal-dual (primal first): the primal (u+, v) is also run on halo
//     row r1, so the dual needs no fresh v from the CTA below; only p1..p3
//     of the neighbours' boundary rows are exchanged.
// Recomputed halo values are bit-identical to the owner's (same inputs,
// same operation order), so the band decomposition leaves every result
// bit-identical to the single-domain reference.
//
// Exchange protocol (per iteration).  The thread that produces a boundary
// value stores it at once as 64-bit words of {32-bit payload, 32-bit
// (packet, step) tag}; the neighbour polls its halo words until the tags
// match.  A 64-bit store is single-copy atomic, so no fence or flag is
// needed: one L2 round trip, ping-pong slots by step parity, two CTA
// barriers per iteration.  A release/acquire progress flag per CTA is used
// only once per packet (before the metric reads the neighbours' surface).
//
// q = A^T p (solve.py:149-158) is kept in two planes and refreshed right
// after each pixel's dual update.  Ingest is fused (evr_ingest.cuh): every
// CTA applies the packet's events of rows [r0-1, r1] in stream order to its
// private copies of f and of the surface; raw timestamps of its own rows go
// straight to global memory (idempotent for the neighbours).
#pragma once

#include <cstdint>

#include "evr_ingest.cuh"
#include "evr_kernels.cuh"
#include "evr_math.cuh"

namespace evr {

template <class T> struct ResArgs {
  const PacketHdr* hdr;
  double* f;
  int64_t* raw;
  T *u, *p1, *p2, *p3;           // state planes (global)
  T *t, *tx, *ty, *G, *sg;       // surface / metric planes (global, debug view)
  T* xchg;                       // tagged boundary words [2][nb][2][3][W][1|2]
  T* frames;                     // PLANES_GMEM: per-CTA plane frames
  unsigned long long* flags;     // [nb] release/acquire progress words
  double* part;                  // [2*nb] rel_change partials
  unsigned* ticket;              // last-CTA election for the final sum
  evr_solve_info* info;
  int* err;
  unsigned long long* trace;     // optional [nb][256] phase timestamps (ns)
  const int* perm;               // k_resident_col: band of CTA blockIdx.x (null = identity)
  unsigned long long* rx;        // k_resident_col, tol > 0: tagged rel_change partials [2][nb][4]
  double tol;                    // convergence_tol (k_resident_col: > 0 = early stop on device)
  int H, W, nb, R;
  int tv_iters, pd_iters, manifold;
  double t_scale, c_pos, c_neg, u_min, u_max;
  T tau, sigma, tl, tv_step, shrink, t_scaleT, uminT, umaxT;
};

// plane indices of a CTA's frame
enum : int {
  RP_U = 0, RP_P1, RP_P2, RP_P3, RP_A11, RP_A12, RP_A22, RP_A31, RP_A32, RP_SG, RP_FB, RP_V,
  RP_QX, RP_QY, RP_COUNT,
  // TV-L1 planes alias the coefficient planes (dead until the metric phase)
  RP_T0 = RP_A11, RP_TU = RP_A12, RP_TUB = RP_A22, RP_TPX = RP_A31, RP_TPY = RP_A32,
  // the binary64 copy of f (ingest .. metric) aliases V (and QX for float)
  RP_F64 = RP_V
};

enum : int { PLANES_SMEM = 0, PLANES_GMEM = 1, PLANES_REG = 2, PLANES_COL = 3 };

__host__ __device__ inline int resident_plane_stride(int R, int W) {
  return ((R + 2) * W + 3) / 4 * 4;
}

// bytes of one CTA's frame of planes
template <class T> __host__ __device__ inline size_t resident_frame_bytes(int R, int W) {
  return (size_t)resident_plane_stride(R, W) * RP_COUNT * sizeof(T);
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// 64-bit words of {payload, tag} for one boundary value
template <class T> struct LLWords;
template <> struct LLWords<float> {
  static constexpr int N = 1;
  __device__ static void pack(float v, unsigned tag, unsigned long long* w) {
    w[0] = ((unsigned long long)tag << 32) | __float_as_uint(v);
  }
  __device__ static float unpack(const unsigned long long* w) {
    return __uint_as_float((unsigned)w[0]);
  }
};
template <> struct LLWords<double> {
  static constexpr int N = 2;
  __device__ static void pack(double v, unsigned tag, unsigned long long* w) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    w[0] = ((unsigned long long)tag << 32) | (bits & 0xffffffffull);
    w[1] = ((unsigned long long)tag << 32) | (bits >> 32);
  }
  __device__ static double unpack(const unsigned long long* w) {
    return __longlong_as_double((long long)((w[1] << 32) | (w[0] & 0xffffffffull)));
  }
};

// one element global -> frame; asynchronous (LDGSTS) when the frame is
// shared memory
template <int MS, class T> __device__ __forceinline__ void copy_in(T* dst, const T* src) {
  if (MS == PLANES_SMEM) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(d), "l"(src), "n"(sizeof(T))
                 : "memory");
  } else {
    *dst = *src;
  }
}

struct Band {
  int base, extra;
  __host__ __device__ __forceinline__ int rows(int b) const { return base + (b < extra ? 1 : 0); }
  __host__ __device__ __forceinline__ int start(int b) const {
    return b * base + (b < extra ? b : extra);
  }
  __host__ __device__ __forceinline__ int of_row(int r) const {
    const int big = extra * (base + 1);
    return r < big ? r / (base + 1) : extra + (r - big) / base;
  }
};

// Chunks of CH local rows (lr = global row - r0 + 1) of [lo, hi]; inside a
// chunk k = 0..CH-1 is fully unrolled and row rb+k exists iff rb+k <= hi.
#define EVR_CHUNKS(rb, lo, hi) for (int rb = (lo); rb <= (hi); rb += CH)
#define EVR_K(k) _Pragma("unroll") for (int k = 0; k < CH; ++k)
#define EVR_K1(k) _Pragma("unroll") for (int k = 0; k <= CH; ++k)

template <class T, int NT, int CH, int MS>
__global__ void __launch_bounds__(NT, 1) k_resident(const ResArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[64];
  const int tid = threadIdx.x;
  const int b = blockIdx.x;
  const int H = a.H, W = a.W;
  const Band band{H / a.nb, H % a.nb};
  const int Rb = band.rows(b);
  const int r0 = band.start(b);
  const int r1 = r0 + Rb;
  const bool has_up = r0 > 0, has_dn = r1 < H;
  const int lo_halo = has_up ? 0 : 1;
  const int hi_halo = has_dn ? Rb + 1 : Rb;
  const size_t PS = (size_t)resident_plane_stride(a.R, W);
  T* pl = MS == PLANES_SMEM ? reinterpret_cast<T*>(smem_raw)
                            : a.frames + (size_t)b * RP_COUNT * PS;
  T* const U = pl + RP_U * PS;
  T* const P1 = pl + RP_P1 * PS;
  T* const P2 = pl + RP_P2 * PS;
  T* const P3 = pl + RP_P3 * PS;
  T* const A11 = pl + RP_A11 * PS;
  T* const A12 = pl + RP_A12 * PS;
  T* const A22 = pl + RP_A22 * PS;
  T* const A31 = pl + RP_A31 * PS;
  T* const A32 = pl + RP_A32 * PS;
  T* const SG = pl + RP_SG * PS;
  T* const FB = pl + RP_FB * PS;
  T* const V = pl + RP_V * PS;
  T* const QX = pl + RP_QX * PS;
  T* const QY = pl + RP_QY * PS;
  T* const T0 = pl + RP_T0 * PS;
  T* const TU = pl + RP_TU * PS;
  T* const TUB = pl + RP_TUB * PS;
  T* const TPX = pl + RP_TPX * PS;
  T* const TPY = pl + RP_TPY * PS;
  T* const TD = QY;  // denoised surface (TV-L1 end .. metric), QY idle then
  double* const F64 = reinterpret_cast<double*>(pl + RP_F64 * PS);

  const PacketHdr* hdr = a.hdr;
  const evr_event* __restrict__ ev = reinterpret_cast<const evr_event*>(hdr + 1);
  const int64_t n_ev = hdr->n;
  const double now = (double)hdr->now;
  const double window = hdr->window;
  const unsigned long long epoch = (unsigned long long)hdr->seq << 24;
  const unsigned tag_base = (unsigned)hdr->seq << 16;
  constexpr int NWD = LLWords<T>::N;
  const size_t xside = (size_t)3 * W * NWD;       // words of one side of one CTA
  const size_t xslot = (size_t)a.nb * 2 * xside;  // words of one ping-pong slot
  unsigned long long* const xw = reinterpret_cast<unsigned long long*>(a.xchg);
  auto gk_of = [&](int r, int j) { return (int64_t)(r0 - 1 + r) * W + j; };

  // optional phase timeline (diagnostics): globaltimer at phase marks
  int tmark = 0;
  auto mark = [&]() {
    if (a.trace && tid == 0 && tmark < 256) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
      a.trace[(size_t)b * 256 + tmark] = t;
    }
    ++tmark;
  };
  mark();

  // boundary value (r, j) of `field` goes to the CTA above (r == 1) and / or
  // below (r == Rb) as tagged words
  auto ll_put = [&](int step, int r, int j, int field, T v) {
    unsigned long long w[NWD];
    LLWords<T>::pack(v, tag_base + (unsigned)step, w);
    unsigned long long* base = xw + (step & 1) * xslot + (size_t)b * 2 * xside;
    if (r == 1) {
      unsigned long long* d = base + ((size_t)field * W + j) * NWD;
#pragma unroll
      for (int k = 0; k < NWD; ++k) st_relaxed_u64(d + k, w[k]);
    }
    if (r == Rb) {
      unsigned long long* d = base + xside + ((size_t)field * W + j) * NWD;
#pragma unroll
      for (int k = 0; k < NWD; ++k) st_relaxed_u64(d + k, w[k]);
    }
  };
  // halo rows <- neighbours' boundary rows of `step` (both sides of a column
  // polled together); for the dual field also refresh q = A^T p there
  auto ll_fetch = [&](int step, T* d0, T* d1, T* d2, int nf) {
    const unsigned want = tag_base + (unsigned)step;
    const unsigned long long* slot = xw + (step & 1) * xslot;
    const unsigned long long* up_src = slot + (size_t)(b - 1) * 2 * xside + xside;  // last row
    const unsigned long long* dn_src = slot + (size_t)(b + 1) * 2 * xside;          // first row
    for (int j = tid; j < W; j += NT) {
      unsigned long long w[2][3][NWD];
      bool ready;
      do {
        ready = true;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (s == 0 ? !has_up : !has_dn) continue;
          const unsigned long long* src = (s == 0 ? up_src : dn_src) + (size_t)j * NWD;
#pragma unroll
          for (int f = 0; f < 3; ++f) {
            if (f >= nf) break;
#pragma unroll
            for (int q = 0; q < NWD; ++q) {
              w[s][f][q] = ld_relaxed_u64(src + (size_t)f * W * NWD + q);
              ready &= (unsigned)(w[s][f][q] >> 32) == want;
            }
          }
        }
      } while (!ready);
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        if (s == 0 ? !has_up : !has_dn) continue;
        const int l = (s == 0 ? 0 : Rb + 1) * W + j;
        const T v0 = LLWords<T>::unpack(w[s][0]);
        d0[l] = v0;
        if (nf > 1) {
          const T v1 = LLWords<T>::unpack(w[s][1]), v2 = LLWords<T>::unpack(w[s][2]);
          d1[l] = v1;
          d2[l] = v2;
          T qx, qy;
          q_of(Coef<T>{A11[l], A12[l], A22[l], A31[l], A32[l]}, v0, v1, v2, qx, qy);
          QX[l] = qx;
          QY[l] = qy;
        }
      }
    }
    __syncthreads();
  };
  // whole-CTA progress flag (once per packet, not per iteration)
  auto flag_publish = [&](int step) {
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release_u64(&a.flags[b], epoch | (unsigned long long)step);
    }
  };
  auto flag_wait = [&](int b_lo, int b_hi, int step) {
    const unsigned long long target = epoch | (unsigned long long)step;
    const int nwait = b_hi - b_lo + 1;
    if (tid < nwait && b_lo + tid != b)
      while (ld_acquire_u64(&a.flags[b_lo + tid]) < target) __nanosleep(20);
    __syncthreads();
  };

  // ---------------------------------------------------------------- load --
  for (int j = tid; j < W; j += NT) {
    EVR_CHUNKS(rb, lo_halo, hi_halo) {
      int64_t rv[CH];
      double fv[CH];
      EVR_K(k) {
        const int r = rb + k;
        if (r > hi_halo) continue;
        const int64_t gk = gk_of(r, j);
        const int l = r * W + j;
        // warm-start u, p into their planes (idle until the solve); async
        // for shared frames, in flight during ingest and TV-L1
        if (r >= 1) copy_in<MS>(U + l, a.u + gk);
        copy_in<MS>(P1 + l, a.p1 + gk);
        copy_in<MS>(P2 + l, a.p2 + gk);
        copy_in<MS>(P3 + l, a.p3 + gk);
        rv[k] = a.manifold ? a.raw[gk] : 0;
        fv[k] = r >= 1 ? a.f[gk] : 0.0;
      }
      EVR_K(k) {
        const int r = rb + k;
        if (r > hi_halo) continue;
        const int l = r * W + j;
        if (a.manifold) {
          const T v = (T)normalize_at((double)rv[k], now, a.t_scale, window);
          T0[l] = v;
          TU[l] = v;
          TUB[l] = v;
          TPX[l] = T(0);
          TPY[l] = T(0);
        }
        if (r >= 1) F64[l] = fv[k];
      }
    }
  }
  if (MS == PLANES_SMEM) asm volatile("cp.async.commit_group;" ::: "memory");
  __syncthreads();

  // -------------------------------------------------------------- ingest --
  // apply_event (pipeline.py:114-121) for the events of rows [r0-1, r1]
  {
    __shared__ IngestShared<NT> ingest_sm;
    const int row_lo = r0 - 1 + lo_halo;
    ordered_ingest<NT>(
        ev, n_ev, H, W, row_lo, r0 - 1 + hi_halo, a.c_pos, a.c_neg, a.u_min, a.u_max, ingest_sm,
        b == 0 ? a.err : nullptr,
        [&](int lp) { return lp + lo_halo * W >= W ? F64[lp + lo_halo * W] : 0.0; },
        [&](int lp, double v, int64_t t) {
          const int l = lp + lo_halo * W;
          const int lr = l / W;
          if (lr >= 1) F64[l] = v;
          if (a.manifold) {
            const T tv = (T)normalize_at((double)t, now, a.t_scale, window);
            T0[l] = tv;
            TU[l] = tv;
            TUB[l] = tv;
          }
          if (lr >= 1 && lr <= Rb) a.raw[(int64_t)(r0 - 1) * W + l] = t;
        });
  }
  mark();  // 1: loaded + ingested

  // ------------------------------------------------------------ TV-L1 ----
  // denoise_timestamps (surface.py:146-196), one exchange per iteration
  int step = 0;
  if (a.manifold) {
    for (int it = 0; it < a.tv_iters; ++it) {
      const bool pub = it < a.tv_iters - 1;
      if (it > 0) ll_fetch(step, TUB, nullptr, nullptr, 1);  // u_bar of step `it`
      mark();
      // dual ascent + projection (surface.py:168-183), own rows + halo above
      for (int j = tid; j < W; j += NT) {
        EVR_CHUNKS(rb, lo_halo, Rb) {
          T ub[CH + 1], ubr[CH], px[CH], py[CH];
          EVR_K1(k) {
            if (rb + k <= hi_halo) ub[k] = TUB[(rb + k) * W + j];
          }
          EVR_K(k) {
            const int l = (rb + k) * W + j;
            if (rb + k > Rb) continue;
            ubr[k] = j < W - 1 ? TUB[l + 1] : T(0);
            px[k] = TPX[l];
            py[k] = TPY[l];
          }
          EVR_K(k) {
            const int r = rb + k;
            if (r > Rb) continue;
            const T dx = j < W - 1 ? ubr[k] - ub[k] : T(0);
            const T dy = r0 - 1 + r < H - 1 ? ub[k + 1] - ub[k] : T(0);
            tv_dual_step(dx, dy, a.tv_step, px[k], py[k]);
          }
          EVR_K(k) {
            if (rb + k > Rb) continue;
            TPX[(rb + k) * W + j] = px[k];
            TPY[(rb + k) * W + j] = py[k];
          }
        }
      }
      __syncthreads();
      // primal + L1 shrink (surface.py:185-193), own rows; boundary rows go
      // out to the neighbours as soon as they are computed
      for (int j = tid; j < W; j += NT) {
        EVR_CHUNKS(rb, 1, Rb) {
          T pyc[CH + 1], pxc[CH], pxl[CH], tu[CH], t0[CH];  // pyc[k] = row rb-1+k
          EVR_K1(k) {
            const int r = rb - 1 + k;
            if (r >= lo_halo && r <= Rb) pyc[k] = TPY[r * W + j];
          }
          EVR_K(k) {
            const int l = (rb + k) * W + j;
            if (rb + k > Rb) continue;
            pxc[k] = TPX[l];
            pxl[k] = j > 0 ? TPX[l - 1] : T(0);
            tu[k] = TU[l];
            t0[k] = T0[l];
          }
          EVR_K(k) {
            const int r = rb + k;
            if (r > Rb) continue;
            const int gi = r0 - 1 + r;
            const T d = div_at(pxc[k], pxl[k], pyc[k + 1], gi > 0 ? pyc[k] : T(0), gi, j, H, W);
            T ub;
            const T un = tv_primal_step(d, tu[k], t0[k], a.tv_step, a.shrink, ub);
            TU[r * W + j] = un;
            TUB[r * W + j] = ub;
            if (pub) ll_put(step + 1, r, j, 0, ub);
          }
        }
      }
      // no barrier: the next fetch only writes halo rows of u_bar, which
      // this primal does not read
      if (pub) ++step;
    }
    __syncthreads();
    // np.clip(u, 0, t_scale) (surface.py:195) -> global t and the TD plane
    for (int j = tid; j < W; j += NT)
      for (int r = 1; r <= Rb; ++r) {
        const T td = vclip(TU[r * W + j], T(0), a.t_scaleT);
        a.t[gk_of(r, j)] = td;
        TD[r * W + j] = td;
      }
  }
  // all rows of the denoised surface this band's metric reads are final
  const int s_met = a.tv_iters + 1;
  flag_publish(s_met);
  if (a.manifold) {
    flag_wait(band.of_row(has_up ? r0 - 1 : r0), band.of_row(r1 + 1 < H ? r1 + 1 : H - 1), s_met);
    for (int j = tid; j < W; j += NT) {  // neighbours' denoised rows r0-1, r1
      if (has_up) TD[j] = __ldcg(a.t + gk_of(0, j));
      if (has_dn) TD[(Rb + 1) * W + j] = __ldcg(a.t + gk_of(Rb + 1, j));
    }
  }
  step = s_met;
  if (MS == PLANES_SMEM) asm volatile("cp.async.wait_all;" ::: "memory");  // warm start landed
  __syncthreads();

  mark();
  // ------------------------------------------------------------ metric ---
  // compute_metric + coeffs (surface.py:81-90, :199-205), solver constants
  for (int j = tid; j < W; j += NT)
    for (int r = lo_halo; r <= hi_halo; ++r) {
      const int l = r * W + j;
      const int gi = r0 - 1 + r;
      T gx = T(0), gy = T(0);
      if (a.manifold) {
        const T tc = TD[l];
        gx = j < W - 1 ? TD[l + 1] - tc : T(0);
        if (gi < H - 1) gy = (r <= Rb ? TD[l + W] : __ldcg(a.t + gk_of(r + 1, j))) - tc;
      }
      const T g = metric_G(gx, gy);
      const T s = Arith<T>::sqrt(g);
      const Coef<T> c = coeffs_of(gx, gy, g);
      A11[l] = c.a11;
      A12[l] = c.a12;
      A22[l] = c.a22;
      A31[l] = c.a31;
      A32[l] = c.a32;
      SG[l] = s;
      if (r >= 1) FB[l] = T(4) * (a.tl * s) * (T)F64[l];
      if (r >= 1 && r <= Rb) {
        const int64_t gk = gk_of(r, j);
        a.tx[gk] = gx;
        a.ty[gk] = gy;
        a.G[gk] = g;
        a.sg[gk] = s;
      }
    }
  __syncthreads();  // F64 (aliasing V / QX) and TD (QY) are dead from here on
  for (int j = tid; j < W; j += NT)
    for (int r = lo_halo; r <= hi_halo; ++r) {
      const int l = r * W + j;
      T qx, qy;
      q_of(Coef<T>{A11[l], A12[l], A22[l], A31[l], A32[l]}, P1[l], P2[l], P3[l], qx, qy);
      QX[l] = qx;
      QY[l] = qy;
    }
  __syncthreads();

  // ------------------------------------------------------- primal-dual ---
  // primal_dual_solve (solve.py:207-261), warm start from the state
  mark();
  double rd = 0.0, ro = 0.0;
  for (int it = 0; it < a.pd_iters; ++it) {
    const bool last = it == a.pd_iters - 1;
    if (it > 0) ll_fetch(step, P1, P2, P3, 3);  // p of the previous step (+ q)
    mark();
    // KL prox + over-relaxation (solve.py:234-252), own rows + halo below
    for (int j = tid; j < W; j += NT) {
      EVR_CHUNKS(rb, 1, hi_halo) {
        T qyc[CH + 1], qxc[CH], qxl[CH], uu[CH], sgv[CH], fbv[CH];  // qyc[k] = row rb-1+k
        EVR_K1(k) {
          const int r = rb - 1 + k;
          if (r >= lo_halo && r <= hi_halo) qyc[k] = QY[r * W + j];
        }
        EVR_K(k) {
          const int l = (rb + k) * W + j;
          if (rb + k > hi_halo) continue;
          qxc[k] = QX[l];
          qxl[k] = j > 0 ? QX[l - 1] : T(0);
          uu[k] = U[l];
          sgv[k] = SG[l];
          fbv[k] = FB[l];
        }
        EVR_K(k) {
          const int r = rb + k;
          if (r > hi_halo) continue;
          const int gi = r0 - 1 + r;
          const T d = div_at(qxc[k], qxl[k], qyc[k + 1], gi > 0 ? qyc[k] : T(0), gi, j, H, W);
          const T uk = uu[k];
          const T nu = kl_primal(d, uk, a.tl * sgv[k], fbv[k], a.tau, a.uminT, a.umaxT);
          V[r * W + j] = Arith<T>::mad(nu, T(2), -uk);
          U[r * W + j] = nu;
          if (last && r <= Rb) {
            const double e = (double)nu - (double)uk;
            rd += e * e;
            ro += (double)uk * (double)uk;
          }
        }
      }
    }
    mark();  // primal issued (thread 0)
    __syncthreads();
    mark();  // primal done
    // dual ascent + ball projection (solve.py:170-201), own rows; refresh q;
    // boundary rows go out to the neighbours as soon as they are computed
    for (int j = tid; j < W; j += NT) {
      EVR_CHUNKS(rb, 1, Rb) {
        T vv[CH + 1], vr[CH], p1[CH], p2[CH], p3[CH], sgv[CH];  // vv[k] = row rb+k
        Coef<T> c[CH];
        EVR_K1(k) {
          if (rb + k <= hi_halo) vv[k] = V[(rb + k) * W + j];
        }
        EVR_K(k) {
          const int l = (rb + k) * W + j;
          if (rb + k > Rb) continue;
          vr[k] = j < W - 1 ? V[l + 1] : T(0);
          p1[k] = P1[l];
          p2[k] = P2[l];
          p3[k] = P3[l];
          sgv[k] = SG[l];
          c[k] = Coef<T>{A11[l], A12[l], A22[l], A31[l], A32[l]};
        }
        EVR_K(k) {
          const int r = rb + k;
          if (r > Rb) continue;
          const T gx = j < W - 1 ? vr[k] - vv[k] : T(0);
          const T gy = r0 - 1 + r < H - 1 ? vv[k + 1] - vv[k] : T(0);
          dual_step(c[k], a.sigma, gx, gy, sgv[k], p1[k], p2[k], p3[k]);
        }
        EVR_K(k) {
          const int r = rb + k;
          if (r > Rb) continue;
          const int l = r * W + j;
          P1[l] = p1[k];
          P2[l] = p2[k];
          P3[l] = p3[k];
          T qx, qy;
          q_of(c[k], p1[k], p2[k], p3[k], qx, qy);
          QX[l] = qx;
          QY[l] = qy;
          if (!last) {
            ll_put(step + 1, r, j, 0, p1[k]);
            ll_put(step + 1, r, j, 1, p2[k]);
            ll_put(step + 1, r, j, 2, p3[k]);
          }
        }
      }
    }
    // no barrier: the next fetch only writes halo rows of p / q, which this
    // dual step does not read
    mark();  // dual issued (thread 0)
    if (!last) ++step;
  }
  if (a.pd_iters < 2) {
    // neighbours may still be loading our rows of u / p as halos
    flag_publish(s_met + 1);
    flag_wait(has_up ? b - 1 : b, has_dn ? b + 1 : b, s_met + 1);
  }
  __syncthreads();
  mark();

  // ---------------------------------------------------------- epilogue ---
  // state.u = u+, state.p, state.f = copy(u+) (pipeline.py:167-170)
  for (int j = tid; j < W; j += NT)
    for (int r = 1; r <= Rb; ++r) {
      const int l = r * W + j;
      const int64_t gk = gk_of(r, j);
      const T v = U[l];
      a.u[gk] = v;
      a.f[gk] = (double)v;
      a.p1[gk] = P1[l];
      a.p2[gk] = P2[l];
      a.p3[gk] = P3[l];
    }

  // rel_change = |u+ - u| / max(|u|, 1e-30) (solve.py:246-249): fixed-order
  // block tree, per-CTA partials, last CTA folds them in index order
  const double sd = block_sum<NT>(rd, red);
  const double so = block_sum<NT>(ro, red);
  __shared__ bool is_last;
  if (tid == 0) {
    a.part[2 * b] = sd;
    a.part[2 * b + 1] = so;
    __threadfence();
    is_last = atomicAdd(a.ticket, 1u) == (unsigned)(a.nb - 1);
  }
  __syncthreads();
  if (is_last) {
    __threadfence();
    double d = 0.0, o = 0.0;
    for (int k = tid; k < a.nb; k += NT) {
      d += __ldcg(a.part + 2 * k);
      o += __ldcg(a.part + 2 * k + 1);
    }
    d = block_sum<NT>(d, red);
    o = block_sum<NT>(o, red);
    if (tid == 0) {
      const double den = sqrt(o);
      a.info->rel_change = sqrt(d) / (den > 1e-30 ? den : 1e-30);
      a.info->iterations = a.pd_iters;
      *a.ticket = 0u;
    }
  }
}

#undef EVR_CHUNKS
#undef EVR_K
#undef EVR_K1

}  // namespace evr
