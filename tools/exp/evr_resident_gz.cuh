// evr_resident_gz.cuh -- EXPERIMENT (measured and rejected, not built into
// the library; profiles/r02_tile64_experiments.md): the resident engine for
// one-row bands with a two-row ghost zone, one neighbour exchange every
// second iteration.  Bit-exact (the whole GPU suite passed with it enabled),
// but DVS128 float64 0.201 vs 0.151 ms per packet: with one warp per
// scheduler the extra rows of the first sub-iteration cost issue slots, not
// just latency.  Built against evr_capi.cu through a ResidentGzKernel table
// and a `resident_uses_gz` switch in resident_enqueue (removed with it).
//
// Same decomposition and arithmetic as k_resident_col<T, NT, 1>
// (evr_resident_col.cuh: CTA b owns sensor row b, one thread per column,
// every per-pixel field in registers), but each CTA keeps the rows b-2 .. b+2
// and recomputes the two rows on either side itself, so the tagged-word
// exchange through L2 -- the dominant cost at DVS128 size (timeline: 0.62 of
// 1.40 us per primal-dual iteration) -- happens once per two iterations:
//
//   TV-L1 (surface.py:167-193), after a fetch all rows b-2 .. b+2 valid:
//     A: dual on rows b-2 .. b+1, primal on b-1 .. b+1
//     B: dual on rows b-1 .. b,   primal on b
//   primal-dual (solve.py:233-252):
//     A: primal on rows b-1 .. b+2, dual on b-1 .. b+1
//     B: primal on rows b .. b+1,   dual on b
// Every value a CTA keeps is computed by the reference's operation sequence
// from values that are themselves exact, so results stay bit-identical.
// After B the CTA publishes its row's state (TV-L1: u_bar, px, py, u;
// primal-dual: p1, p2, p3, u, qx, qy) as tagged 64-bit words in a slot
// indexed by sensor row; the fetch takes from rows b-2 / b-1 / b+1 / b+2
// only the values the next A reads (b-2: u_bar, px, py / qy; b-1, b+1: all
// four / p, u; b+2: u_bar / u, qx, qy).
//
// The row outside this CTA's own that only feeds a boundary rule (rows off
// the sensor) computes values nobody reads, as in k_resident_col.  Early stop
// (convergence_tol > 0) needs the per-iteration fold of k_resident_col; this
// kernel runs fixed-iteration solves only (the host picks it for tol == 0).
#pragma once

#include <cstdint>

#include "../../paper_1607_06283_b200/csrc/evr_fastdp.cuh"
#include "../../paper_1607_06283_b200/csrc/evr_ingest.cuh"
#include "../../paper_1607_06283_b200/csrc/evr_kernels.cuh"
#include "../../paper_1607_06283_b200/csrc/evr_math.cuh"
#include "../../paper_1607_06283_b200/csrc/evr_resident.cuh"
#include "../../paper_1607_06283_b200/csrc/evr_resident_col.cuh"

namespace evr {

// dynamic shared memory: f (binary64) and the normalised surface for rows
// b-2 .. b+2, two row-exchange planes for rows b-2 .. b+3
template <class T> __host__ __device__ inline size_t resident_gz_smem(int W) {
  return (size_t)5 * W * sizeof(double) + (size_t)5 * W * sizeof(T) + (size_t)12 * W * sizeof(T) +
         64;
}

template <class T, int NT>
__global__ void __launch_bounds__(NT, 1) k_resident_gz(const ResArgs<T> a) {
  constexpr bool kFast = sizeof(T) == 8;
  constexpr int NWD = LLWords<T>::N;
  constexpr int NQ = 6 * NWD;  // words of one row slot: six values
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[64];
  const int tid = threadIdx.x;
  const int b = a.perm ? a.perm[blockIdx.x] : (int)blockIdx.x;  // this CTA's row
  const int H = a.H, W = a.W;
  const int j = tid;
  const bool col = j < W;
  const int jc = min(j, W - 1);
  const int jr = jc < W - 1 ? jc + 1 : jc;
  const int jl = jc > 0 ? jc - 1 : jc;
  // local row r (0 .. 4) is sensor row b - 2 + r; own row = 2
  auto gi_of = [&](int r) { return b - 2 + r; };
  auto live = [&](int r) { return b - 2 + r >= 0 && b - 2 + r < H; };
  const int lo = max(0, 2 - b), hi = min(4, H + 1 - b);  // live local rows

  double* const F64 = reinterpret_cast<double*>(smem_raw);  // [5][W]
  T* const TT = reinterpret_cast<T*>(F64 + 5 * W);           // [5][W]
  T* const XA = TT + 5 * W;                                  // [6][W]
  T* const XB = XA + 6 * W;                                  // [6][W]

  const PacketHdr* hdr = a.hdr;
  const evr_event* __restrict__ ev = reinterpret_cast<const evr_event*>(hdr + 1);
  const int64_t n_ev = hdr->n;
  const double now = (double)hdr->now;
  const double window = hdr->window;
  const unsigned long long epoch = (unsigned long long)hdr->seq << 24;
  const unsigned tag_base = (unsigned)hdr->seq << 16;
  const size_t xslot = (size_t)H * W * NQ;  // one parity of the row slots
  unsigned long long* const xw = reinterpret_cast<unsigned long long*>(a.xchg);
  auto gk_of = [&](int r) { return (int64_t)(b - 2 + r) * W + j; };

  // publish this CTA's row: values v[0 .. 5] tagged with `step`
  auto put = [&](int step, const T (&v)[6]) {
    unsigned long long w[NQ];
    const unsigned tag = tag_base + (unsigned)step;
#pragma unroll
    for (int k = 0; k < 6; ++k) LLWords<T>::pack(v[k], tag, w + k * NWD);
    unsigned long long* d = xw + (step & 1) * xslot + ((size_t)b * W + j) * NQ;
    if constexpr (NQ % 4 == 0) {
#pragma unroll
      for (int k = 0; k < NQ; k += 4) st_v4(d + k, w + k);
    } else {
#pragma unroll
      for (int k = 0; k < NQ; k += 2) st_v2(d + k, w + k);
    }
  };
  // fetch values [v0, v0 + nv) of the row slots of local rows 0, 1, 3, 4
  // (sensor rows b-2, b-1, b+1, b+2; rows off the sensor skipped)
  auto fetch = [&](int step, const int (&v0)[4], const int (&nv)[4], T (&out)[4][4]) {
    if (!col) return;
    const unsigned want = tag_base + (unsigned)step;
    const unsigned long long* slot = xw + (step & 1) * xslot;
    constexpr int rows[4] = {0, 1, 3, 4};
    bool on[4];
    const unsigned long long* src[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      on[q] = live(rows[q]);
      src[q] = slot + ((size_t)(on[q] ? gi_of(rows[q]) : 0) * W + j) * NQ;
    }
    unsigned long long w[4][4 * NWD];
    bool ready;
    do {
      ready = true;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (!on[q]) continue;
#pragma unroll
        for (int k = 0; k < 4 * NWD; ++k) {
          if (k < nv[q] * NWD) {
            w[q][k] = ld_relaxed_u64(src[q] + v0[q] * NWD + k);
            ready &= (unsigned)(w[q][k] >> 32) == want;
          }
        }
      }
    } while (!ready);
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (on[q] && k < nv[q]) out[q][k] = LLWords<T>::unpack(w[q] + k * NWD);
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
    for (int r = 0; r < 5; ++r) {
      if (!live(r)) continue;
      const int64_t gk = gk_of(r);
      F64[r * W + j] = r >= 1 ? a.f[gk] : 0.0;
      if (a.manifold) TT[r * W + j] = (T)normalize_at((double)a.raw[gk], now, a.t_scale, window);
    }
  }
  __syncthreads();

  // -------------------------------------------------------------- ingest --
  // apply_event (pipeline.py:114-121) for the events of rows b-2+lo .. b-2+hi
  {
    __shared__ IngestShared<NT> ingest_sm;
    ordered_ingest<NT>(
        ev, n_ev, H, W, b - 2 + lo, b - 2 + hi, a.c_pos, a.c_neg, a.u_min, a.u_max, ingest_sm,
        b == 0 ? a.err : nullptr,
        [&](int lp) { return lp + lo * W >= W ? F64[lp + lo * W] : 0.0; },
        [&](int lp, double v, int64_t t) {
          const int l = lp + lo * W;
          const int lr = l / W;
          if (lr >= 1) F64[l] = v;
          if (a.manifold) TT[l] = (T)normalize_at((double)t, now, a.t_scale, window);
          if (lr == 2) a.raw[(int64_t)b * W + (l - 2 * W)] = t;
        });
  }
  __syncthreads();

  // ------------------------------------------------------------ TV-L1 ----
  // denoise_timestamps (surface.py:146-196), cold start
  T td[6];  // denoised surface, rows b-2 .. b+3
#pragma unroll
  for (int r = 0; r < 6; ++r) td[r] = T(0);
  int step = 0;
  if (a.manifold) {
    // row 0: u_bar, px, py; rows 1..3 (index m = r - 1): all; row 4: u_bar
    T ub0, px0 = T(0), py0 = T(0), ub4;
    T tu[3], tub[3], px[3], py[3], t0[3];
    ub0 = col && live(0) ? TT[j] : T(0);
    ub4 = col && live(4) ? TT[4 * W + j] : T(0);
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const T v = col && live(m + 1) ? TT[(m + 1) * W + j] : T(0);
      t0[m] = v;
      tu[m] = v;
      tub[m] = v;
      px[m] = T(0);
      py[m] = T(0);
    }
    // dual ascent + projection of one row (surface.py:168-183), branch-free
    // fast paths with the IEEE redo of k_resident_col
    auto tv_duals = [&](auto rows_c, T* dxs, T* dys, T* nxs, T* nys, T* pxs, T* pys) {
      constexpr int NRW = decltype(rows_c)::value;
      T nn[NRW];
      bool slow = false, proj = false;
#pragma unroll
      for (int k = 0; k < NRW; ++k) {
        nxs[k] = pxs[k];
        nys[k] = pys[k];
        if constexpr (kFast) {
          nn[k] = tv_dual_pre_fx(dxs[k], dys[k], a.tv_step, nxs[k], nys[k], slow);
          proj |= nn[k] != T(1);
        } else {
          tv_dual_step(dxs[k], dys[k], a.tv_step, nxs[k], nys[k]);
        }
      }
      if constexpr (kFast) {
        if (__any_sync(0xffffffffu, proj)) {
#pragma unroll
          for (int k = 0; k < NRW; ++k) fdp_div2(nxs[k], nys[k], nn[k], slow);
        }
        if (slow) {
#pragma unroll
          for (int k = 0; k < NRW; ++k) {
            nxs[k] = pxs[k];
            nys[k] = pys[k];
            tv_dual_step(dxs[k], dys[k], a.tv_step, nxs[k], nys[k]);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < NRW; ++k) {
        pxs[k] = nxs[k];
        pys[k] = nys[k];
      }
      (void)nn;
      (void)slow;
      (void)proj;
    };
    for (int it = 0; it < a.tv_iters; ++it) {
      const bool A = (it & 1) == 0;
      if (it > 0 && A) {
        T h[4][4];
        fetch(step, {0, 0, 0, 0}, {3, 4, 4, 1}, h);
        if (col) {
          if (live(0)) ub0 = h[0][0], px0 = h[0][1], py0 = h[0][2];
          if (live(1)) tub[0] = h[1][0], px[0] = h[1][1], py[0] = h[1][2], tu[0] = h[1][3];
          if (live(3)) tub[2] = h[2][0], px[2] = h[2][1], py[2] = h[2][2], tu[2] = h[2][3];
          if (live(4)) ub4 = h[3][0];
        }
      }
      if (A) {
        if (col) {
          XB[j] = ub0;
#pragma unroll
          for (int m = 0; m < 3; ++m) XB[(m + 1) * W + j] = tub[m];
        }
        __syncthreads();
        // dual on rows 0..3
        T dx[4], dy[4], nx[4], ny[4], pxa[4], pya[4];
        const T ubr[4] = {ub0, tub[0], tub[1], tub[2]};
        const T ubd[4] = {tub[0], tub[1], tub[2], ub4};
        int gis[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          gis[k] = gi_of(k);
          const T ubR = XB[k * W + jr];
          dx[k] = j < W - 1 ? ubR - ubr[k] : T(0);
          dy[k] = gis[k] < H - 1 ? ubd[k] - ubr[k] : T(0);
          pxa[k] = k == 0 ? px0 : px[k - 1];
          pya[k] = k == 0 ? py0 : py[k - 1];
        }
        tv_duals(std::integral_constant<int, 4>{}, dx, dy, nx, ny, pxa, pya);
        px0 = pxa[0];
        py0 = pya[0];
#pragma unroll
        for (int m = 0; m < 3; ++m) {
          px[m] = pxa[m + 1];
          py[m] = pya[m + 1];
          if (col) XA[(m + 1) * W + j] = px[m];
        }
        __syncthreads();
        // primal on rows 1..3
#pragma unroll
        for (int m = 0; m < 3; ++m) {
          const int gi = gi_of(m + 1);
          const T pxl = XA[(m + 1) * W + jl];
          const T pyu = m == 0 ? py0 : py[m - 1];
          const T d = div_at(px[m], j > 0 ? pxl : T(0), py[m], gi > 0 ? pyu : T(0), gi, j, H, W);
          T ub;
          tu[m] = tv_primal_step(d, tu[m], t0[m], a.tv_step, a.shrink, ub);
          tub[m] = ub;
        }
      } else {
        if (col) {
          XB[W + j] = tub[0];
          XB[2 * W + j] = tub[1];
        }
        __syncthreads();
        // dual on rows 1..2
        T dx[2], dy[2], nx[2], ny[2], pxa[2], pya[2];
        const T ubr[2] = {tub[0], tub[1]};
        const T ubd[2] = {tub[1], tub[2]};
        int gis[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          gis[k] = gi_of(k + 1);
          const T ubR = XB[(k + 1) * W + jr];
          dx[k] = j < W - 1 ? ubR - ubr[k] : T(0);
          dy[k] = gis[k] < H - 1 ? ubd[k] - ubr[k] : T(0);
          pxa[k] = px[k];
          pya[k] = py[k];
        }
        tv_duals(std::integral_constant<int, 2>{}, dx, dy, nx, ny, pxa, pya);
        px[0] = pxa[0];
        py[0] = pya[0];
        px[1] = pxa[1];
        py[1] = pya[1];
        if (col) XA[2 * W + j] = px[1];
        __syncthreads();
        // primal on row 2 (own)
        {
          const int gi = b;
          const T pxl = XA[2 * W + jl];
          const T d = div_at(px[1], j > 0 ? pxl : T(0), py[1], gi > 0 ? py[0] : T(0), gi, j, H, W);
          T ub;
          tu[1] = tv_primal_step(d, tu[1], t0[1], a.tv_step, a.shrink, ub);
          tub[1] = ub;
        }
        if (it < a.tv_iters - 1) {
          if (col) put(step + 1, {tub[1], px[1], py[1], tu[1], T(0), T(0)});
          ++step;
        }
      }
    }
    // np.clip(u, 0, t_scale) (surface.py:195)
    td[2] = vclip(tu[1], T(0), a.t_scaleT);
    if (col) a.t[gk_of(2)] = td[2];
  }
  // every row of the denoised surface this row's metrics read is final
  const int s_met = a.tv_iters + 1;
  flag_publish(s_met);
  if (a.manifold) {
    flag_wait(max(b - 2, 0), min(a.nb - 1, b + 3), s_met);
    if (col) {
#pragma unroll
      for (int r = 0; r < 6; ++r) {
        if (r == 2) continue;
        const int gi = b - 2 + r;
        if (gi >= 0 && gi < H) td[r] = __ldcg(a.t + (int64_t)gi * W + j);
      }
#pragma unroll
      for (int r = 0; r < 6; ++r) XA[r * W + j] = td[r];
    }
  }
  step = s_met;
  __syncthreads();

  // ------------------------------------------------------------ metric ---
  // compute_metric + coeffs (surface.py:81-90, :199-205) on rows 0..4
  Coef<T> cm[5];
  T sgm[5];
  {
    T gxs[5], gys[5], gs[5];
    bool slow = false;
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      const int gi = gi_of(r);
      T gx = T(0), gy = T(0);
      if (a.manifold) {
        const T tr = XA[r * W + jr];
        gx = j < W - 1 ? tr - td[r] : T(0);
        gy = gi < H - 1 ? td[r + 1] - td[r] : T(0);
      }
      gxs[r] = gx;
      gys[r] = gy;
      gs[r] = metric_G(gx, gy);
      if constexpr (kFast) {
        cm[r] = coeffs_fx(gx, gy, gs[r], slow);
        sgm[r] = fdp_sqrt(gs[r], slow);
      } else {
        cm[r] = coeffs_of(gx, gy, gs[r]);
        sgm[r] = Arith<T>::sqrt(gs[r]);
      }
    }
    if (kFast && slow) {
#pragma unroll
      for (int r = 0; r < 5; ++r) {
        cm[r] = coeffs_of(gxs[r], gys[r], gs[r]);
        sgm[r] = Arith<T>::sqrt(gs[r]);
      }
    }
    if (col) {
      const int64_t gk = gk_of(2);
      a.tx[gk] = gxs[2];
      a.ty[gk] = gys[2];
      a.G[gk] = gs[2];
      a.sg[gk] = sgm[2];
    }
  }
  __syncthreads();  // XA (the surface) is rewritten with q below

  // ------------------------------------------------------- primal-dual ---
  // primal_dual_solve (solve.py:207-261), warm start from the state
  // rows 1..3 (m = r - 1): everything; row 0: qy; row 4: u, qx, qy, sqrtG, 4 beta f
  T u[3], p1[3], p2[3], p3[3], qx[3], qy[3], v[3], sg[3], ysg[3], fb[3];
  Coef<T> c[3];
  T qy0, u4, qx4, qy4, sg4, fb4, v4 = T(0);
  {
    T P[5][3];
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      const bool ok = col && live(r);
      const int64_t gk = gk_of(r);
      P[r][0] = ok ? a.p1[gk] : T(0);
      P[r][1] = ok ? a.p2[gk] : T(0);
      P[r][2] = ok ? a.p3[gk] : T(0);
    }
    T qxt, qyt;
    q_of(cm[0], P[0][0], P[0][1], P[0][2], qxt, qy0);
    q_of(cm[4], P[4][0], P[4][1], P[4][2], qx4, qy4);
    (void)qxt;
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      c[m] = cm[m + 1];
      sg[m] = sgm[m + 1];
      p1[m] = P[m + 1][0];
      p2[m] = P[m + 1][1];
      p3[m] = P[m + 1][2];
      const bool ok = col && live(m + 1);
      u[m] = ok ? a.u[gk_of(m + 1)] : T(0);
      fb[m] = ok ? T(4) * (a.tl * sg[m]) * (T)F64[(m + 1) * W + j] : T(0);
      if constexpr (kFast)
        ysg[m] = fdp_recip(sg[m]);  // the dual's divisor, constant over the solve
      else
        ysg[m] = T(1);
      q_of(c[m], p1[m], p2[m], p3[m], qx[m], qy[m]);
    }
    sg4 = sgm[4];
    const bool ok4 = col && live(4);
    u4 = ok4 ? a.u[gk_of(4)] : T(0);
    fb4 = ok4 ? T(4) * (a.tl * sg4) * (T)F64[4 * W + j] : T(0);
  }
  double rd = 0.0, ro = 0.0;
  // KL prox + over-relaxation on a row (solve.py:234-245)
  auto primal_rows = [&](auto n_c, T* d, T* uu, const T* sgs, const T* fbs, T* nu) {
    constexpr int N = decltype(n_c)::value;
    bool slow = false;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      if constexpr (kFast)
        nu[k] = kl_primal_fx(d[k], uu[k], a.tl * sgs[k], fbs[k], a.tau, a.uminT, a.umaxT, slow);
      else
        nu[k] = kl_primal(d[k], uu[k], a.tl * sgs[k], fbs[k], a.tau, a.uminT, a.umaxT);
    }
    if (kFast && slow) {
#pragma unroll
      for (int k = 0; k < N; ++k)
        nu[k] = kl_primal(d[k], uu[k], a.tl * sgs[k], fbs[k], a.tau, a.uminT, a.umaxT);
    }
    (void)slow;
  };
  // dual ascent + ball projection on rows m0 .. m0 + N - 1 (solve.py:170-201)
  auto dual_rows = [&](auto m0_c, auto n_c) {
    constexpr int M0 = decltype(m0_c)::value, N = decltype(n_c)::value;
    T gx[N], gy[N], n1[N], n2[N], n3[N], nn[N];
    bool slow = false, proj = false;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const int m = M0 + k;
      const int gi = gi_of(m + 1);
      const T vr = XB[(m + 1) * W + jr];
      const T vd = m < 2 ? v[m + 1] : v4;
      gx[k] = j < W - 1 ? vr - v[m] : T(0);
      gy[k] = gi < H - 1 ? vd - v[m] : T(0);
      n1[k] = p1[m];
      n2[k] = p2[m];
      n3[k] = p3[m];
      if constexpr (kFast) {
        nn[k] = dual_pre_fx_r(c[m], a.sigma, gx[k], gy[k], sg[m], ysg[m], n1[k], n2[k], n3[k], slow);
        proj |= nn[k] != T(1);
      } else {
        dual_step(c[m], a.sigma, gx[k], gy[k], sg[m], n1[k], n2[k], n3[k]);
      }
    }
    if constexpr (kFast) {
      if (__any_sync(0xffffffffu, proj)) {
#pragma unroll
        for (int k = 0; k < N; ++k) fdp_div3(n1[k], n2[k], n3[k], nn[k], slow);
      }
      if (slow) {
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const int m = M0 + k;
          n1[k] = p1[m];
          n2[k] = p2[m];
          n3[k] = p3[m];
          dual_step(c[m], a.sigma, gx[k], gy[k], sg[m], n1[k], n2[k], n3[k]);
        }
      }
    }
    (void)nn;
    (void)slow;
    (void)proj;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const int m = M0 + k;
      p1[m] = n1[k];
      p2[m] = n2[k];
      p3[m] = n3[k];
      q_of(c[m], p1[m], p2[m], p3[m], qx[m], qy[m]);
    }
  };
  for (int it = 0; it < a.pd_iters; ++it) {
    const bool last = it == a.pd_iters - 1;
    const bool A = (it & 1) == 0;
    if (it > 0 && A) {
      T h[4][4];
      fetch(step, {5, 0, 0, 3}, {1, 4, 4, 3}, h);
      if (col) {
        if (live(0)) qy0 = h[0][0];
        if (live(1)) {
          p1[0] = h[1][0], p2[0] = h[1][1], p3[0] = h[1][2], u[0] = h[1][3];
          q_of(c[0], p1[0], p2[0], p3[0], qx[0], qy[0]);
        }
        if (live(3)) {
          p1[2] = h[2][0], p2[2] = h[2][1], p3[2] = h[2][2], u[2] = h[2][3];
          q_of(c[2], p1[2], p2[2], p3[2], qx[2], qy[2]);
        }
        if (live(4)) u4 = h[3][0], qx4 = h[3][1], qy4 = h[3][2];
      }
    }
    if (A) {
      if (col) {
#pragma unroll
        for (int m = 0; m < 3; ++m) XA[(m + 1) * W + j] = qx[m];
        XA[4 * W + j] = qx4;
      }
      __syncthreads();
      // primal on rows 1..4
      T d[4], uu[4], sgs[4], fbs[4], nu[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int gi = gi_of(k + 1);
        const T qxl = XA[(k + 1) * W + jl];
        const T qxc = k < 3 ? qx[k] : qx4;
        const T qyc = k < 3 ? qy[k] : qy4;
        const T qyu = k == 0 ? qy0 : qy[k - 1];
        d[k] = div_at(qxc, j > 0 ? qxl : T(0), qyc, gi > 0 ? qyu : T(0), gi, j, H, W);
        uu[k] = k < 3 ? u[k] : u4;
        sgs[k] = k < 3 ? sg[k] : sg4;
        fbs[k] = k < 3 ? fb[k] : fb4;
      }
      primal_rows(std::integral_constant<int, 4>{}, d, uu, sgs, fbs, nu);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const T vk = Arith<T>::mad(nu[k], T(2), -uu[k]);
        if (k == 1 && last && col) {
          const double e = (double)nu[k] - (double)uu[k];
          rd += e * e;
          ro += (double)uu[k] * (double)uu[k];
        }
        if (k < 3) {
          v[k] = vk;
          u[k] = nu[k];
        } else {
          v4 = vk;
          u4 = nu[k];
        }
        if (col) XB[(k + 1) * W + j] = vk;
      }
      __syncthreads();
      dual_rows(std::integral_constant<int, 0>{}, std::integral_constant<int, 3>{});
    } else {
      if (col) {
        XA[2 * W + j] = qx[1];
        XA[3 * W + j] = qx[2];
      }
      __syncthreads();
      // primal on rows 2..3
      T d[2], uu[2], sgs[2], fbs[2], nu[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int m = k + 1;
        const int gi = gi_of(m + 1);
        const T qxl = XA[(m + 1) * W + jl];
        d[k] = div_at(qx[m], j > 0 ? qxl : T(0), qy[m], gi > 0 ? qy[m - 1] : T(0), gi, j, H, W);
        uu[k] = u[m];
        sgs[k] = sg[m];
        fbs[k] = fb[m];
      }
      primal_rows(std::integral_constant<int, 2>{}, d, uu, sgs, fbs, nu);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int m = k + 1;
        v[m] = Arith<T>::mad(nu[k], T(2), -uu[k]);
        if (k == 0 && last && col) {
          const double e = (double)nu[k] - (double)uu[k];
          rd += e * e;
          ro += (double)uu[k] * (double)uu[k];
        }
        u[m] = nu[k];
        if (col) XB[(m + 1) * W + j] = v[m];
      }
      __syncthreads();
      dual_rows(std::integral_constant<int, 1>{}, std::integral_constant<int, 1>{});
      if (!last) {
        if (col) put(step + 1, {p1[1], p2[1], p3[1], u[1], qx[1], qy[1]});
        ++step;
      }
    }
  }
  if (a.pd_iters <= 2) {
    // no exchange ran: rows b-2 .. b+2 may still be loading our p / u
    flag_publish(s_met + 1);
    flag_wait(max(b - 2, 0), min(a.nb - 1, b + 2), s_met + 1);
  }

  // ---------------------------------------------------------- epilogue ---
  // state.u = u+, state.p, state.f = copy(u+) (pipeline.py:167-170)
  if (col) {
    const int64_t gk = gk_of(2);
    a.u[gk] = u[1];
    a.f[gk] = (double)u[1];
    a.p1[gk] = p1[1];
    a.p2[gk] = p2[1];
    a.p3[gk] = p3[1];
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
    double dd = 0.0, oo = 0.0;
    for (int k = tid; k < a.nb; k += NT) {
      dd += __ldcg(a.part + 2 * k);
      oo += __ldcg(a.part + 2 * k + 1);
    }
    dd = block_sum<NT>(dd, red);
    oo = block_sum<NT>(oo, red);
    if (tid == 0) {
      const double den = sqrt(oo);
      a.info->rel_change = sqrt(dd) / (den > 1e-30 ? den : 1e-30);
      a.info->iterations = a.pd_iters;
      *a.ticket = 0u;
    }
  }
}

}  // namespace evr
