// evr_resident_col.cuh -- the resident engine for narrow bands: one thread
// per sensor column, the column's rows of the band in registers.
//
// Same decomposition, exchange protocol and operation order as k_resident
// (evr_resident.cuh: CTA b of a cooperative grid owns rows [b*RB, b*RB+RB),
// one tagged-word neighbour exchange per iteration, halo half-steps
// recomputed), specialised for the shapes AUTO sends to the resident engine:
// W <= NT and a compile-time band height RB (1 or 2 rows on B200's 148 SMs
// up to 296-row sensors).  Thread j keeps every per-pixel field of column j
// -- TV-L1 {u, u_bar, px, py, t0}, then solver {u, p1..p3, q, v} and the
// metric constants -- for local rows 0 (halo above) .. RB+1 (halo below) in
// registers, fully unrolled over the rows; shared memory carries only the
// one row value a half-step needs from the column to its left or right
// (qx / v, px / u_bar, the denoised surface) plus the ingest targets.
// Against the plane-frame kernel this removes the per-access address
// arithmetic and bounds tests that dominated its instruction stream
// (profiles/r01_summary.md), leaving the float64 arithmetic itself.
//
// Bands: every band has RB rows except possibly the last (the only one
// with no band below), so the halo-below row is always register RB+1.
#pragma once

#include <cstdint>

#include "evr_fastdp.cuh"
#include "evr_ingest.cuh"
#include "evr_kernels.cuh"
#include "evr_math.cuh"
#include "evr_resident.cuh"

namespace evr {

// Halo words of one column and side: 4 slots (p1, p2, p3, spare) of NWD
// tagged 64-bit words, contiguous, so a thread moves its column's whole dual
// in 256-bit accesses (1 for float, 2 for double); the single TV-L1 value
// per column is packed densely instead.
__device__ __forceinline__ void st_v4(unsigned long long* d, const unsigned long long* w) {
  asm volatile("st.relaxed.gpu.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(d), "l"(w[0]),
               "l"(w[1]), "l"(w[2]), "l"(w[3])
               : "memory");
}
__device__ __forceinline__ void ld_v4(const unsigned long long* s, unsigned long long* w) {
  asm volatile("ld.relaxed.gpu.global.v4.u64 {%0, %1, %2, %3}, [%4];"
               : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3])
               : "l"(s)
               : "memory");
}
__device__ __forceinline__ void st_v2(unsigned long long* d, const unsigned long long* w) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(d), "l"(w[0]), "l"(w[1])
               : "memory");
}
__device__ __forceinline__ void ld_v2(const unsigned long long* s, unsigned long long* w) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
               : "=l"(w[0]), "=l"(w[1])
               : "l"(s)
               : "memory");
}
// words [0, n) of a column's slots, n = NWD (one value) or 4 * NWD (all)
template <int N> __device__ __forceinline__ void st_words(unsigned long long* d,
                                                         const unsigned long long* w) {
  if constexpr (N == 1) st_relaxed_u64(d, w[0]);
  else if constexpr (N == 2) st_v2(d, w);
  else {
#pragma unroll
    for (int k = 0; k < N; k += 4) st_v4(d + k, w + k);
  }
}
template <int N> __device__ __forceinline__ void ld_words(const unsigned long long* s,
                                                         unsigned long long* w) {
  if constexpr (N == 1) w[0] = ld_relaxed_u64(s);
  else if constexpr (N == 2) ld_v2(s, w);
  else {
#pragma unroll
    for (int k = 0; k < N; k += 4) ld_v4(s + k, w + k);
  }
}

// dynamic shared memory of k_resident_col: f (binary64), the normalised
// surface, and two row-exchange planes, each (RB + 2) x W
template <class T> __host__ __device__ inline size_t resident_col_smem(int RB, int W) {
  const size_t n = (size_t)(RB + 2) * W;
  return n * sizeof(double) + 3 * n * sizeof(T) + 64;
}

template <class T, int NT, int RB>
__global__ void __launch_bounds__(NT, 1) k_resident_col(const ResArgs<T> a) {
  constexpr int NR = RB + 2;  // local rows: 0 = halo above, 1..RB own, RB+1 = halo below
  constexpr bool kFast = sizeof(T) == 8;  // float64: branch-free fast paths (evr_fastdp.cuh)
#ifndef EVR_SKIP_UNIT
#define EVR_SKIP_UNIT 1
#endif
  constexpr bool kSkipUnit = EVR_SKIP_UNIT;  // skip p / 1 when the whole warp is inside the ball
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[64];
  const int tid = threadIdx.x;
  const int b = a.perm ? a.perm[blockIdx.x] : (int)blockIdx.x;  // this CTA's band
  const int H = a.H, W = a.W;
  const int r0 = b * RB;  // first own row; local row r is global row r0 - 1 + r
  const int Rb = min(RB, H - r0);
  const bool has_up = r0 > 0, has_dn = r0 + RB < H;  // has_dn implies Rb == RB
  const int lo = has_up ? 0 : 1, hi = has_dn ? RB + 1 : Rb;
  const int j = tid;
  const bool col = j < W;
  // right / left neighbour columns, clamped into the sensor (the value read
  // at an edge, or by an idle thread j >= W, is never used)
  const int jc = min(j, W - 1);
  const int jr = jc < W - 1 ? jc + 1 : jc;
  const int jl = jc > 0 ? jc - 1 : jc;
  auto live = [&](int r) { return r >= lo && r <= hi; };

  const size_t NP = (size_t)NR * W;
  double* const F64 = reinterpret_cast<double*>(smem_raw);
  T* const TT = reinterpret_cast<T*>(F64 + NP);
  T* const XA = TT + NP;
  T* const XB = XA + NP;

  const PacketHdr* hdr = a.hdr;
  const evr_event* __restrict__ ev = reinterpret_cast<const evr_event*>(hdr + 1);
  const int64_t n_ev = hdr->n;
  const double now = (double)hdr->now;
  const double window = hdr->window;
  const unsigned long long epoch = (unsigned long long)hdr->seq << 24;
  const unsigned tag_base = (unsigned)hdr->seq << 16;
  constexpr int NWD = LLWords<T>::N;
  constexpr int NCW = 4 * NWD;                     // words of one column and side
  const size_t xside = (size_t)W * NCW;             // words of one side of one CTA
  const size_t xslot = (size_t)a.nb * 2 * xside;
  unsigned long long* const xw = reinterpret_cast<unsigned long long*>(a.xchg);
  auto gk_of = [&](int r) { return (int64_t)(r0 - 1 + r) * W + j; };

  int tmark = 0;
  const bool tracing = a.trace != nullptr && tid == 0;
  auto mark = [&]() {
    if (tracing) {
      if (tmark < 255) {  // slot 255: the SM id
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
        a.trace[(size_t)b * 256 + tmark] = t;
      }
      ++tmark;
    }
  };
  mark();
  if (tracing) {  // the SM this band runs on (slot 255 of the timeline)
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    a.trace[(size_t)b * 256 + 255] = smid;
  }

  // boundary values of local row r (1 = first own row -> the band above,
  // Rb = last own row -> the band below) as tagged words: nv = 1 (u_bar) or
  // 3 (p1, p2, p3) values in the column's slots
  auto ll_put = [&](int step, int r, int nv, T v0, T v1, T v2) {
    EVR_ASSERT(col && b < a.nb && (r == 1 || r == Rb));
    unsigned long long w[NCW];
    const unsigned tag = tag_base + (unsigned)step;
    LLWords<T>::pack(v0, tag, w);
    unsigned long long* side = xw + (step & 1) * xslot + (size_t)b * 2 * xside;
    if (nv == 1) {  // one value per column, densely packed (TV-L1)
      if (r == 1) st_words<NWD>(side + (size_t)j * NWD, w);
      if (r == Rb) st_words<NWD>(side + xside + (size_t)j * NWD, w);
      return;
    }
    unsigned long long* base = side + (size_t)j * NCW;
    LLWords<T>::pack(v1, tag, w + NWD);
    LLWords<T>::pack(v2, tag, w + 2 * NWD);
    LLWords<T>::pack(v2, tag, w + 3 * NWD);  // spare slot: keeps the access 256-bit
    if (r == 1) st_words<NCW>(base, w);
    if (r == Rb) st_words<NCW>(base + xside, w);
  };
  // the neighbours' boundary values of `step` for this column: v[0][f] from
  // the band above (-> local row 0), v[1][f] from the band below (-> RB+1)
  auto ll_fetch = [&](int step, int nf, T (&v)[2][3]) {
    const unsigned want = tag_base + (unsigned)step;
    const unsigned long long* slot = xw + (step & 1) * xslot;
    const size_t jw = (size_t)j * (nf == 1 ? NWD : NCW);  // dense for one value
    const unsigned long long* src[2] = {slot + (size_t)(b - 1) * 2 * xside + xside + jw,
                                        slot + (size_t)(b + 1) * 2 * xside + jw};
    const bool on[2] = {has_up, has_dn};
    EVR_ASSERT((!has_up || b >= 1) && (!has_dn || b + 1 < a.nb));
    unsigned long long w[2][NCW];
    bool ready;
    if (!col) {
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int f = 0; f < 3; ++f) v[s][f] = T(0);
      return;
    }
    // poll the whole column (1-2 256-bit loads per side) until every tag
    // matches; measured faster on B200 than spinning on one sentinel word
    // first (one L2 round trip fewer), and than any backoff
    do {
      ready = true;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        if (!on[s]) continue;
        if (nf == 1) {
          ld_words<NWD>(src[s], w[s]);
#pragma unroll
          for (int q = 0; q < NWD; ++q) ready &= (unsigned)(w[s][q] >> 32) == want;
        } else {
          ld_words<NCW>(src[s], w[s]);
#pragma unroll
          for (int q = 0; q < 3 * NWD; ++q) ready &= (unsigned)(w[s][q] >> 32) == want;
        }
      }
    } while (!ready);
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int f = 0; f < 3; ++f)
        if (f < nf) v[s][f] = on[s] ? LLWords<T>::unpack(w[s] + f * NWD) : T(0);
  };
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
  if (col) {
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      if (!live(r)) continue;
      const int64_t gk = gk_of(r);
      F64[r * W + j] = r >= 1 ? a.f[gk] : 0.0;
      if (a.manifold) TT[r * W + j] = (T)normalize_at((double)a.raw[gk], now, a.t_scale, window);
    }
  }
  __syncthreads();

  // -------------------------------------------------------------- ingest --
  // apply_event (pipeline.py:114-121) for the events of rows [r0-1, r0+RB]
  {
    __shared__ IngestShared<NT> ingest_sm;
    ordered_ingest<NT>(
        ev, n_ev, H, W, r0 - 1 + lo, r0 - 1 + hi, a.c_pos, a.c_neg, a.u_min, a.u_max, ingest_sm,
        b == 0 ? a.err : nullptr,
        [&](int lp) { return lp + lo * W >= W ? F64[lp + lo * W] : 0.0; },
        [&](int lp, double v, int64_t t) {
          const int l = lp + lo * W;
          const int lr = l / W;
          if (lr >= 1) F64[l] = v;
          if (a.manifold) TT[l] = (T)normalize_at((double)t, now, a.t_scale, window);
          if (lr >= 1 && lr <= Rb) a.raw[(int64_t)(r0 - 1) * W + l] = t;
        });
  }
  __syncthreads();
  mark();

  // ------------------------------------------------------------ TV-L1 ----
  // denoise_timestamps (surface.py:146-196): dual on rows lo..Rb (the row
  // above recomputed), primal on the own rows, u_bar exchanged
  T td[NR + 1];  // denoised surface, rows 0..RB+2 (RB+2: below the halo)
#pragma unroll
  for (int r = 0; r <= NR; ++r) td[r] = T(0);
  int step = 0;
  if (a.manifold) {
    T tu[NR], tub[NR], px[NR], py[NR], t0[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const T v = col && live(r) ? TT[r * W + j] : T(0);
      t0[r] = v;
      tu[r] = v;
      tub[r] = v;
      px[r] = T(0);
      py[r] = T(0);
    }
    for (int it = 0; it < a.tv_iters; ++it) {
      const bool pub = it < a.tv_iters - 1;
      if (it > 0) {
        T h[2][3];
        ll_fetch(step, 1, h);
        tub[0] = h[0][0];
        tub[RB + 1] = h[1][0];
      }
      mark();
      if (col) {
#pragma unroll
        for (int r = 0; r <= RB; ++r) XB[r * W + j] = tub[r];
      }
      __syncthreads();
      {
        // every row branch-free (rows past the band compute unused values),
        // so the rows' latency chains overlap; float64 fast paths with a
        // rare IEEE redo (evr_fastdp.cuh)
        T dx[RB + 1], dy[RB + 1], nx[RB + 1], ny[RB + 1], nn[RB + 1];
        bool slow = false, proj = false;
#pragma unroll
        for (int r = 0; r <= RB; ++r) {
          const T ubr = XB[r * W + jr];
          dx[r] = j < W - 1 ? ubr - tub[r] : T(0);
          dy[r] = r0 - 1 + r < H - 1 ? tub[r + 1] - tub[r] : T(0);
          nx[r] = px[r];
          ny[r] = py[r];
          if constexpr (kFast) {
            nn[r] = tv_dual_pre_fx(dx[r], dy[r], a.tv_step, nx[r], ny[r], slow);
            proj |= nn[r] != T(1);
          } else {
            tv_dual_step(dx[r], dy[r], a.tv_step, nx[r], ny[r]);
          }
        }
        if constexpr (kFast) {
          if (!kSkipUnit || __any_sync(0xffffffffu, proj)) {  // warp-uniform: x / 1 == x otherwise
#pragma unroll
            for (int r = 0; r <= RB; ++r) fdp_div2(nx[r], ny[r], nn[r], slow);
          }
        }
        if (kFast && slow) {
#pragma unroll
          for (int r = 0; r <= RB; ++r) {
            nx[r] = px[r];
            ny[r] = py[r];
            tv_dual_step(dx[r], dy[r], a.tv_step, nx[r], ny[r]);
          }
        }
#pragma unroll
        for (int r = 0; r <= RB; ++r) {
          px[r] = nx[r];
          py[r] = ny[r];
          if (col) XA[r * W + j] = px[r];
        }
      }
      __syncthreads();
#pragma unroll
      for (int r = 1; r <= RB; ++r) {
        if (r > Rb) continue;
        const int gi = r0 - 1 + r;
        const T pxl = XA[r * W + jl];
        const T d = div_at(px[r], j > 0 ? pxl : T(0), py[r], gi > 0 ? py[r - 1] : T(0), gi, j, H, W);
        T ub;
        tu[r] = tv_primal_step(d, tu[r], t0[r], a.tv_step, a.shrink, ub);
        tub[r] = ub;
        if (pub && col) ll_put(step + 1, r, 1, ub, ub, ub);
      }
      if (pub) ++step;
    }
    // np.clip(u, 0, t_scale) (surface.py:195)
#pragma unroll
    for (int r = 1; r <= RB; ++r) {
      if (r > Rb) continue;
      td[r] = vclip(tu[r], T(0), a.t_scaleT);
      if (col) a.t[gk_of(r)] = td[r];
    }
  }
  // all rows of the denoised surface this band's metric reads are final
  const int s_met = a.tv_iters + 1;
  flag_publish(s_met);
  if (a.manifold) {
    const int last_row = min(r0 + RB + 1, H - 1);
    flag_wait(has_up ? b - 1 : b, min(a.nb - 1, last_row / RB), s_met);
    if (col) {
      if (has_up) td[0] = __ldcg(a.t + gk_of(0));
      if (has_dn) td[RB + 1] = __ldcg(a.t + gk_of(RB + 1));
      if (has_dn && r0 + RB + 1 < H) td[RB + 2] = __ldcg(a.t + gk_of(RB + 2));
#pragma unroll
      for (int r = 0; r < NR; ++r) XA[r * W + j] = td[r];
    }
  }
  step = s_met;
  __syncthreads();

  mark();
  // ------------------------------------------------------------ metric ---
  // compute_metric + coeffs (surface.py:81-90, :199-205), solver constants
  Coef<T> c[NR];
  T sg[NR], fb[NR], ysg[NR];
  T gxs[NR], gys[NR], gs[NR];
  {
    bool slow = false;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int gi = r0 - 1 + r;
      T gx = T(0), gy = T(0);
      if (a.manifold) {
        const T tr = XA[r * W + jr];
        gx = j < W - 1 ? tr - td[r] : T(0);
        gy = gi < H - 1 ? td[r + 1] - td[r] : T(0);
      }
      gxs[r] = gx;
      gys[r] = gy;
      gs[r] = metric_G(gx, gy);
      if constexpr (kFast) {  // shared reciprocal of G, branch-free sqrt
        c[r] = coeffs_fx(gx, gy, gs[r], slow);
        sg[r] = fdp_sqrt(gs[r], slow);
      } else {
        c[r] = coeffs_of(gx, gy, gs[r]);
        sg[r] = Arith<T>::sqrt(gs[r]);
      }
    }
    if (kFast && slow) {
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        c[r] = coeffs_of(gxs[r], gys[r], gs[r]);
        sg[r] = Arith<T>::sqrt(gs[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      if constexpr (kFast)
        ysg[r] = fdp_recip(sg[r]);  // the dual's divisor, constant over the solve
      else
        ysg[r] = T(1);
    }
  }
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const T gx = gxs[r], gy = gys[r];
    const T g = gs[r];
    const T s = sg[r];
    fb[r] = r >= 1 && col && live(r) ? T(4) * (a.tl * s) * (T)F64[r * W + j] : T(0);
    if (r >= 1 && r <= Rb && col) {
      const int64_t gk = gk_of(r);
      a.tx[gk] = gx;
      a.ty[gk] = gy;
      a.G[gk] = g;
      a.sg[gk] = s;
    }
  }

  __syncthreads();  // XA (the surface) is rewritten with q below

  // ------------------------------------------------------- primal-dual ---
  // primal_dual_solve (solve.py:207-261), warm start from the state; primal
  // on rows 1..hi (the row below recomputed), dual on the own rows, p
  // exchanged
  T u[NR], p1[NR], p2[NR], p3[NR], qx[NR], qy[NR], v[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const bool ok = col && live(r);
    const int64_t gk = gk_of(r);
    p1[r] = ok ? a.p1[gk] : T(0);
    p2[r] = ok ? a.p2[gk] : T(0);
    p3[r] = ok ? a.p3[gk] : T(0);
    u[r] = ok && r >= 1 ? a.u[gk] : T(0);
    q_of(c[r], p1[r], p2[r], p3[r], qx[r], qy[r]);
    v[r] = T(0);
  }
  mark();
  // convergence_tol > 0 (solve.py:246-258): rel_change of every iteration,
  // folded on the device -- each CTA publishes its partial sums after the
  // primal step as tagged words, runs the dual step, then reads all the
  // bands' partials and folds them in band order (the same bits in every
  // CTA, so every band takes the same stop decision after the same dual)
  const bool track = a.tol > 0.0;
  int iters_done = a.pd_iters;
  double rel_track = 0.0;
  __shared__ double rel_sh;
  auto fold_rel = [&](int it) {
    const unsigned want = tag_base + (unsigned)it;
    const unsigned long long* slot = a.rx + (size_t)(it & 1) * a.nb * 4;
    double d = 0.0, o = 0.0;
    for (int k = tid; k < a.nb; k += NT) {
      unsigned long long w[4];
      bool ready;
      do {
        ld_v4(slot + (size_t)k * 4, w);
        ready = (unsigned)(w[0] >> 32) == want && (unsigned)(w[1] >> 32) == want &&
                (unsigned)(w[2] >> 32) == want && (unsigned)(w[3] >> 32) == want;
      } while (!ready);
      d += LLWords<double>::unpack(w);
      o += LLWords<double>::unpack(w + 2);
    }
    d = block_sum<NT>(d, red);
    o = block_sum<NT>(o, red);
    if (tid == 0) {
      const double den = sqrt(o);
      rel_sh = sqrt(d) / (den > 1e-30 ? den : 1e-30);
    }
    __syncthreads();
    return rel_sh;
  };
  double rd = 0.0, ro = 0.0;
  for (int it = 0; it < a.pd_iters; ++it) {
    const bool last = it == a.pd_iters - 1;
    if (track) rd = ro = 0.0;
    if (it > 0) {  // p of the previous step on the halo rows (+ their q)
      T h[2][3];
      ll_fetch(step, 3, h);
      p1[0] = h[0][0];
      p2[0] = h[0][1];
      p3[0] = h[0][2];
      q_of(c[0], p1[0], p2[0], p3[0], qx[0], qy[0]);
      p1[RB + 1] = h[1][0];
      p2[RB + 1] = h[1][1];
      p3[RB + 1] = h[1][2];
      q_of(c[RB + 1], p1[RB + 1], p2[RB + 1], p3[RB + 1], qx[RB + 1], qy[RB + 1]);
    }
    mark();
    if (col) {
#pragma unroll
      for (int r = 1; r < NR; ++r) XA[r * W + j] = qx[r];
    }
    __syncthreads();
    // KL prox + over-relaxation (solve.py:234-252), all rows branch-free
    {
      T d[NR], nu[NR];
      bool slow = false;
#pragma unroll
      for (int r = 1; r < NR; ++r) {
        const int gi = r0 - 1 + r;
        const T qxl = XA[r * W + jl];
        d[r] = div_at(qx[r], j > 0 ? qxl : T(0), qy[r], gi > 0 ? qy[r - 1] : T(0), gi, j, H, W);
        if constexpr (kFast)
          nu[r] = kl_primal_fx(d[r], u[r], a.tl * sg[r], fb[r], a.tau, a.uminT, a.umaxT, slow);
        else
          nu[r] = kl_primal(d[r], u[r], a.tl * sg[r], fb[r], a.tau, a.uminT, a.umaxT);
      }
      if (kFast && slow) {
#pragma unroll
        for (int r = 1; r < NR; ++r)
          nu[r] = kl_primal(d[r], u[r], a.tl * sg[r], fb[r], a.tau, a.uminT, a.umaxT);
      }
#pragma unroll
      for (int r = 1; r < NR; ++r) {
        const T uk = u[r];
        v[r] = Arith<T>::mad(nu[r], T(2), -uk);
        u[r] = nu[r];
        if ((last || track) && r <= Rb && col) {
          const double e = (double)nu[r] - (double)uk;
          rd += e * e;
          ro += (double)uk * (double)uk;
        }
        if (col) XB[r * W + j] = v[r];
      }
    }
    mark();
    if (track) {  // this band's partials of iteration it (block_sum syncs the CTA)
      const double sd = block_sum<NT>(rd, red);
      const double so = block_sum<NT>(ro, red);
      if (tid == 0) {
        unsigned long long w[4];
        LLWords<double>::pack(sd, tag_base + (unsigned)it, w);
        LLWords<double>::pack(so, tag_base + (unsigned)it, w + 2);
        st_v4(a.rx + ((size_t)(it & 1) * a.nb + b) * 4, w);
      }
    }
    __syncthreads();
    mark();
    // dual ascent + ball projection (solve.py:170-201); boundary rows go out
    // to the neighbours as soon as they are computed
    {
      T gx[RB + 1], gy[RB + 1], n1[RB + 1], n2[RB + 1], n3[RB + 1], nn[RB + 1];
      bool slow = false, proj = false;
#pragma unroll
      for (int r = 1; r <= RB; ++r) {
        const T vr = XB[r * W + jr];
        gx[r] = j < W - 1 ? vr - v[r] : T(0);
        gy[r] = r0 - 1 + r < H - 1 ? v[r + 1] - v[r] : T(0);
        n1[r] = p1[r];
        n2[r] = p2[r];
        n3[r] = p3[r];
        if constexpr (kFast) {
          nn[r] = dual_pre_fx_r(c[r], a.sigma, gx[r], gy[r], sg[r], ysg[r], n1[r], n2[r], n3[r],
                                slow);
          proj |= nn[r] != T(1);
        } else {
          dual_step(c[r], a.sigma, gx[r], gy[r], sg[r], n1[r], n2[r], n3[r]);
        }
      }
      if constexpr (kFast) {
        if (!kSkipUnit || __any_sync(0xffffffffu, proj)) {  // warp-uniform: q / 1 == q otherwise
#pragma unroll
          for (int r = 1; r <= RB; ++r) fdp_div3(n1[r], n2[r], n3[r], nn[r], slow);
        }
      }
      if (kFast && slow) {
#pragma unroll
        for (int r = 1; r <= RB; ++r) {
          n1[r] = p1[r];
          n2[r] = p2[r];
          n3[r] = p3[r];
          dual_step(c[r], a.sigma, gx[r], gy[r], sg[r], n1[r], n2[r], n3[r]);
        }
      }
#pragma unroll
      for (int r = 1; r <= RB; ++r) {
        p1[r] = n1[r];
        p2[r] = n2[r];
        p3[r] = n3[r];
        q_of(c[r], p1[r], p2[r], p3[r], qx[r], qy[r]);
        if (!last && col && r <= Rb) {
          ll_put(step + 1, r, 3, p1[r], p2[r], p3[r]);
        }
      }
    }
    mark();
    if (track) {
      rel_track = fold_rel(it);
      if (rel_track < a.tol) {  // solve.py:257-258, after the dual step
        iters_done = it + 1;
        break;
      }
    }
    if (!last) ++step;
  }
  if (iters_done < 2) {
    // neighbours may still be loading our rows of u / p as halos
    flag_publish(s_met + 1);
    flag_wait(has_up ? b - 1 : b, has_dn ? b + 1 : b, s_met + 1);
  }
  mark();

  // ---------------------------------------------------------- epilogue ---
  // state.u = u+, state.p, state.f = copy(u+) (pipeline.py:167-170)
  if (col) {
#pragma unroll
    for (int r = 1; r <= RB; ++r) {
      if (r > Rb) continue;
      const int64_t gk = gk_of(r);
      a.u[gk] = u[r];
      a.f[gk] = (double)u[r];
      a.p1[gk] = p1[r];
      a.p2[gk] = p2[r];
      a.p3[gk] = p3[r];
    }
  }

  if (track) {  // every CTA holds the folded rel_change of the last iteration
    if (b == 0 && tid == 0) {
      a.info->rel_change = rel_track;
      a.info->iterations = iters_done;
    }
    mark();
    return;
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
  mark();  // kernel end (after the epilogue and the rel_change fold)
}

}  // namespace evr
