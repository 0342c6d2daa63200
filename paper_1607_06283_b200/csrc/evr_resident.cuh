// evr_resident.cuh -- the resident engine: ONE persistent kernel per event
// packet, the whole of process_packet (pipeline.py:142-171) on chip.
//
// Decomposition.  CTA b of a cooperative grid (<= 1 CTA per SM) owns the
// row band [r0, r1) of the sensor (full width, equal band heights).  Every
// per-pixel field of the band lives in shared memory together with one halo
// row above (r0-1) and one below (r1); global memory is touched only to
// load the state at the start, to exchange two boundary rows per iteration,
// and to write the state back at the end.
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
// bit-identical to the single-domain reference.  Boundary rows go through
// a ping-pong buffer in global memory (L2) and a per-CTA release/acquire
// flag; a CTA waits only for its two neighbours, never for the grid.
//
// q = A^T p (solve.py:149-158) is kept in two planes and refreshed right
// after each pixel's dual update, so the primal's divergence reads its
// left / upper neighbours' q instead of recomputing them.
//
// Ingest is fused: every CTA scans the packet and applies the events of
// rows [r0-1, r1] with the same ordered, sort-grouped walk as k_ingest
// (evr_ingest.cuh) to its private copies of f and of the surface
// (duplicates compound in order, last timestamp wins); raw timestamps of
// its own rows go straight to global memory (idempotent for neighbours).
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
  T* xchg;                       // [2][nb][2][3][W] boundary rows
  unsigned long long* flags;     // [nb] release/acquire progress words
  double* part;                  // [2*nb] rel_change partials
  unsigned* ticket;              // last-CTA election for the final sum
  evr_solve_info* info;
  int* err;
  unsigned long long* trace;     // optional [nb][256] phase timestamps (ns)
  int H, W, nb, R;
  unsigned wdiv;                 // ceil(2^32 / W): q / W == __umulhi(q, wdiv)
  int tv_iters, pd_iters, manifold;
  double t_scale, c_pos, c_neg, u_min, u_max;
  T tau, sigma, tl, tv_step, shrink, t_scaleT, uminT, umaxT;
};

// plane indices in shared memory
enum : int {
  RP_U = 0, RP_P1, RP_P2, RP_P3, RP_A11, RP_A12, RP_A22, RP_A31, RP_A32, RP_SG, RP_FB, RP_V,
  RP_QX, RP_QY, RP_COUNT,
  // TV-L1 planes alias the coefficient planes (dead until the metric phase)
  RP_T0 = RP_A11, RP_TU = RP_A12, RP_TUB = RP_A22, RP_TPX = RP_A31, RP_TPY = RP_A32,
  // the binary64 copy of f (ingest .. metric) aliases V (and QX for float)
  RP_F64 = RP_V
};

__host__ __device__ inline int resident_plane_stride(int R, int W) {
  return ((R + 2) * W + 3) / 4 * 4;
}

template <class T> __host__ __device__ inline size_t resident_smem_bytes(int R, int W) {
  return (size_t)resident_plane_stride(R, W) * RP_COUNT * sizeof(T) + 64 * sizeof(double);
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

// Low-latency boundary-row exchange: every 64-bit word carries 32 payload
// bits and a 32-bit tag naming the (packet, step) that wrote it.  A 64-bit
// store is single-copy atomic, so a reader that sees the expected tag also
// sees the payload -- no fence, no separate flag, one L2 round trip.
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

// one element global -> shared, asynchronous (LDGSTS)
template <class T> __device__ __forceinline__ void cp_async_elem(T* dst, const T* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(d), "l"(src), "n"(sizeof(T))
               : "memory");
}

struct Band {
  int base, extra;
  __device__ __forceinline__ int rows(int b) const { return base + (b < extra ? 1 : 0); }
  __device__ __forceinline__ int start(int b) const { return b * base + (b < extra ? b : extra); }
  __device__ __forceinline__ int of_row(int r) const {
    const int big = extra * (base + 1);
    return r < big ? r / (base + 1) : extra + (r - big) / base;
  }
};

template <class T, int NT>
__global__ void __launch_bounds__(NT, 1) k_resident(const ResArgs<T> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int b = blockIdx.x;
  const int H = a.H, W = a.W;
  const Band band{H / a.nb, H % a.nb};
  const int Rb = band.rows(b);
  const int r0 = band.start(b);
  const int r1 = r0 + Rb;
  const bool has_up = r0 > 0, has_dn = r1 < H;
  const size_t PS = (size_t)resident_plane_stride(a.R, W);
  T* pl = reinterpret_cast<T*>(smem_raw);
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
  double* const F64 = reinterpret_cast<double*>(pl + RP_F64 * PS);
  double* const red = reinterpret_cast<double*>(pl + RP_COUNT * PS);

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

  // rows [lo, hi] of the local frame (lr = global row - r0 + 1), flat loop
#define EVR_FOR_ROWS(lo, hi)                                              \
  for (int q_ = tid, n_ = ((hi) - (lo) + 1) * W; q_ < n_; q_ += NT) {      \
    const int lr = (lo) + (int)__umulhi((unsigned)q_, a.wdiv);             \
    const int j = q_ - (lr - (lo)) * W;                                    \
    const int gi = r0 - 1 + lr;                                            \
    const int l = lr * W + j;
#define EVR_GK const int64_t gk = (int64_t)gi * W + j;
#define EVR_END_ROWS }

  // optional phase timeline (diagnostics): globaltimer at phase marks
  int tmark = 0;
  auto mark = [&]() {
    if (a.trace && tid == 0 && tmark < 256) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.trace[(size_t)b * 256 + tmark] = t;
    }
    ++tmark;
  };
  mark();

  const int lo_halo = has_up ? 0 : 1;
  const int hi_halo = has_dn ? Rb + 1 : Rb;

  // boundary-row publish: the thread that produced (lr, j) of the first /
  // last own row stores it as tagged words for the CTA above / below
  auto ll_put = [&](int step, int lr, int j, int field, T v) {
    unsigned long long w[NWD];
    LLWords<T>::pack(v, tag_base + (unsigned)step, w);
    unsigned long long* base = xw + (step & 1) * xslot + (size_t)b * 2 * xside;
    if (lr == 1) {
      unsigned long long* d = base + ((size_t)field * W + j) * NWD;
#pragma unroll
      for (int k = 0; k < NWD; ++k) st_relaxed_u64(d + k, w[k]);
    }
    if (lr == Rb) {
      unsigned long long* d = base + xside + ((size_t)field * W + j) * NWD;
#pragma unroll
      for (int k = 0; k < NWD; ++k) st_relaxed_u64(d + k, w[k]);
    }
  };
  // halo rows <- neighbours' boundary rows of `step`, polling the tags; for
  // the dual field also refresh q = A^T p there (coefficients cover halos)
  auto ll_fetch = [&](int step, T* d0, T* d1, T* d2, int nf) {
    const unsigned want = tag_base + (unsigned)step;
    const unsigned long long* slot = xw + (step & 1) * xslot;
    for (int k = tid; k < 2 * W; k += NT) {
      const bool up = k < W;
      const int j = up ? k : k - W;
      if (up ? !has_up : !has_dn) continue;
      // the CTA above sent its last row (side 1), the one below its first
      const unsigned long long* src =
          slot + (size_t)(up ? b - 1 : b + 1) * 2 * xside + (up ? xside : 0) + (size_t)j * NWD;
      unsigned long long w[3][NWD];
      bool ready;
      do {
        ready = true;
        for (int f = 0; f < nf; ++f)
#pragma unroll
          for (int q = 0; q < NWD; ++q) {
            w[f][q] = ld_relaxed_u64(src + (size_t)f * W * NWD + q);
            ready &= (unsigned)(w[f][q] >> 32) == want;
          }
      } while (!ready);
      const int l = up ? j : (Rb + 1) * W + j;
      const T v0 = LLWords<T>::unpack(w[0]);
      d0[l] = v0;
      if (nf > 1) {
        const T v1 = LLWords<T>::unpack(w[1]), v2 = LLWords<T>::unpack(w[2]);
        d1[l] = v1;
        d2[l] = v2;
        T qx, qy;
        q_of(Coef<T>{A11[l], A12[l], A22[l], A31[l], A32[l]}, v0, v1, v2, qx, qy);
        QX[l] = qx;
        QY[l] = qy;
      }
    }
    __syncthreads();
  };
  // whole-CTA progress flag (used once per packet, not per iteration)
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
  // warm-start u, p: asynchronous copies straight into their (idle until
  // the solve) planes, in flight during ingest and TV-L1
  EVR_FOR_ROWS(lo_halo, hi_halo)
    EVR_GK
    if (lr >= 1) cp_async_elem(U + l, a.u + gk);
    cp_async_elem(P1 + l, a.p1 + gk);
    cp_async_elem(P2 + l, a.p2 + gk);
    cp_async_elem(P3 + l, a.p3 + gk);
  EVR_END_ROWS
  asm volatile("cp.async.commit_group;" ::: "memory");
  // raw timestamps -> surface heights, f -> binary64 plane; loads batched
  // KB deep per thread so their latencies overlap
  {
    constexpr int KB = 4;
    const int n_ = (hi_halo - lo_halo + 1) * W;
    for (int q0 = tid; q0 < n_; q0 += NT * KB) {
      int64_t rv[KB];
      double fv[KB];
#pragma unroll
      for (int k = 0; k < KB; ++k) {
        const int q = q0 + k * NT;
        if (q < n_) {
          const int lr = lo_halo + (int)__umulhi((unsigned)q, a.wdiv);
          const int j = q - (lr - lo_halo) * W;
          const int64_t gk = (int64_t)(r0 - 1 + lr) * W + j;
          rv[k] = a.manifold ? a.raw[gk] : 0;
          fv[k] = lr >= 1 ? a.f[gk] : 0.0;
        }
      }
#pragma unroll
      for (int k = 0; k < KB; ++k) {
        const int q = q0 + k * NT;
        if (q < n_) {
          const int lr = lo_halo + (int)__umulhi((unsigned)q, a.wdiv);
          const int l = lr * W + (q - (lr - lo_halo) * W);
          if (a.manifold) {
            const T v = (T)normalize_at((double)rv[k], now, a.t_scale, window);
            T0[l] = v;
            TU[l] = v;
            TUB[l] = v;
            TPX[l] = T(0);
            TPY[l] = T(0);
          }
          if (lr >= 1) F64[l] = fv[k];
        }
      }
    }
  }
  __syncthreads();

  // -------------------------------------------------------------- ingest --
  // apply_event (pipeline.py:114-121) for the events of rows [r0-1, r1]:
  // private copies of f / the surface, raw of own rows straight to global
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
      EVR_FOR_ROWS(lo_halo, Rb)  // dual, own rows + halo row above
        const T dx = j < W - 1 ? TUB[l + 1] - TUB[l] : T(0);
        const T dy = gi < H - 1 ? TUB[l + W] - TUB[l] : T(0);
        T px = TPX[l], py = TPY[l];
        tv_dual_step(dx, dy, a.tv_step, px, py);
        TPX[l] = px;
        TPY[l] = py;
      EVR_END_ROWS
      __syncthreads();
      EVR_FOR_ROWS(1, Rb)  // primal, own rows; boundary rows go out at once
        const T d = div_at(TPX[l], j > 0 ? TPX[l - 1] : T(0), TPY[l], gi > 0 ? TPY[l - W] : T(0),
                           gi, j, H, W);
        T ub;
        const T un = tv_primal_step(d, TU[l], T0[l], a.tv_step, a.shrink, ub);
        TU[l] = un;
        TUB[l] = ub;
        if (pub) ll_put(step + 1, lr, j, 0, ub);
      EVR_END_ROWS
      // no barrier: the next fetch only writes halo rows of u_bar, which
      // this primal does not read
      if (pub) ++step;
    }
    __syncthreads();
    // np.clip(u, 0, t_scale) (surface.py:195) -> global t (own rows) and
    // the TD plane (QY is idle until the solve)
    EVR_FOR_ROWS(1, Rb)
      EVR_GK
      const T td = vclip(TU[l], T(0), a.t_scaleT);
      a.t[gk] = td;
      QY[l] = td;
    EVR_END_ROWS
  }
  // all rows of the denoised surface this band's metric reads are final
  const int s_met = a.tv_iters + 1;
  flag_publish(s_met);
  if (a.manifold) {
    flag_wait(band.of_row(has_up ? r0 - 1 : r0), band.of_row(r1 + 1 < H ? r1 + 1 : H - 1), s_met);
    // neighbours' denoised rows r0-1 and r1 into the TD plane
    for (int k = tid; k < 2 * W; k += NT) {
      const bool up = k < W;
      const int j = up ? k : k - W;
      if (up ? has_up : has_dn) {
        const int lr = up ? 0 : Rb + 1;
        QY[lr * W + j] = __ldcg(a.t + (int64_t)(r0 - 1 + lr) * W + j);
      }
    }
  }
  step = s_met;
  asm volatile("cp.async.wait_all;" ::: "memory");  // warm-start u, p landed
  __syncthreads();

  mark();
  // ------------------------------------------------------------ metric ---
  // compute_metric + coeffs (surface.py:81-90, :199-205), solver constants
  T* const TD = QY;
  EVR_FOR_ROWS(lo_halo, hi_halo)
    EVR_GK
    T gx = T(0), gy = T(0);
    if (a.manifold) {
      const T tc = TD[l];
      gx = j < W - 1 ? TD[l + 1] - tc : T(0);
      if (gi < H - 1) gy = (lr <= Rb ? TD[l + W] : __ldcg(a.t + gk + W)) - tc;
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
    if (lr >= 1) FB[l] = T(4) * (a.tl * s) * (T)F64[l];
    if (lr >= 1 && lr <= Rb) {
      a.tx[gk] = gx;
      a.ty[gk] = gy;
      a.G[gk] = g;
      a.sg[gk] = s;
    }
  EVR_END_ROWS
  __syncthreads();  // F64 (aliasing V / QX) and TD (QY) are dead from here on
  EVR_FOR_ROWS(lo_halo, hi_halo)
    T qx, qy;
    q_of(Coef<T>{A11[l], A12[l], A22[l], A31[l], A32[l]}, P1[l], P2[l], P3[l], qx, qy);
    QX[l] = qx;
    QY[l] = qy;
  EVR_END_ROWS
  __syncthreads();

  // ------------------------------------------------------- primal-dual ---
  // primal_dual_solve (solve.py:207-261), warm start from the state
  mark();
  double rd = 0.0, ro = 0.0;
  for (int it = 0; it < a.pd_iters; ++it) {
    const bool last = it == a.pd_iters - 1;
    if (it > 0) ll_fetch(step, P1, P2, P3, 3);  // p of the previous step (+ q)
    mark();
    EVR_FOR_ROWS(1, hi_halo)  // primal + over-relaxation, own rows + halo below
      const T d = div_at(QX[l], j > 0 ? QX[l - 1] : T(0), QY[l], gi > 0 ? QY[l - W] : T(0), gi,
                         j, H, W);
      const T uk = U[l];
      const T nu = kl_primal(d, uk, a.tl * SG[l], FB[l], a.tau, a.uminT, a.umaxT);
      V[l] = nu * T(2) - uk;
      U[l] = nu;
      if (last && lr <= Rb) {
        const double e = (double)nu - (double)uk;
        rd += e * e;
        ro += (double)uk * (double)uk;
      }
    EVR_END_ROWS
    __syncthreads();
    EVR_FOR_ROWS(1, Rb)  // dual ascent + ball projection, own rows; refresh q
      const T gx = j < W - 1 ? V[l + 1] - V[l] : T(0);
      const T gy = gi < H - 1 ? V[l + W] - V[l] : T(0);
      const Coef<T> c{A11[l], A12[l], A22[l], A31[l], A32[l]};
      T q1 = P1[l], q2 = P2[l], q3 = P3[l];
      dual_step(c, a.sigma, gx, gy, SG[l], q1, q2, q3);
      P1[l] = q1;
      P2[l] = q2;
      P3[l] = q3;
      T qx, qy;
      q_of(c, q1, q2, q3, qx, qy);
      QX[l] = qx;
      QY[l] = qy;
      if (!last) {
        ll_put(step + 1, lr, j, 0, q1);
        ll_put(step + 1, lr, j, 1, q2);
        ll_put(step + 1, lr, j, 2, q3);
      }
    EVR_END_ROWS
    // no barrier: the next fetch only writes halo rows of p / q, which this
    // dual step does not read
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
  EVR_FOR_ROWS(1, Rb)
    EVR_GK
    const T v = U[l];
    a.u[gk] = v;
    a.f[gk] = (double)v;
    a.p1[gk] = P1[l];
    a.p2[gk] = P2[l];
    a.p3[gk] = P3[l];
  EVR_END_ROWS
#undef EVR_FOR_ROWS
#undef EVR_GK
#undef EVR_END_ROWS

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

}  // namespace evr
