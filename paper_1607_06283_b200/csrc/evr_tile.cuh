// evr_tile.cuh -- temporally blocked iteration kernels of the streaming
// engine: K TV-L1 or K primal-dual iterations per launch.
//
// One iteration of either solver reads each pixel's neighbours at distance
// one (TV-L1: u_bar right / below for the dual, px left and py above for the
// primal; primal-dual: q = A^T p left / above for the primal, v right /
// below for the dual), so K iterations over a tile need K halo pixels on
// every side.  A CTA loads a region of 32 columns x G*RPT rows of the packed
// state (+ constants) into registers, runs K iterations on chip and stores
// the (32 - 2K) x (G*RPT - 2K) interior; the halo pixels it computes on the
// way are the neighbours' (recomputed bit-identically, never stored).
//
// Layout on chip: warp g owns region rows [g*RPT, (g+1)*RPT), lane l region
// column l; a thread keeps its RPT pixels' state and constants in registers.
// Horizontal neighbours come from warp shuffles (lane 0 / 31 are halo
// columns, so their missing neighbour only spoils values nobody keeps);
// vertical ones from the thread's own rows, and at a warp's first / last row
// from the adjacent warp through one shared-memory row (2 CTA barriers per
// iteration).  Global traffic per pixel and iteration falls from one state
// read + constants read + state write per iteration (k_pd_march) to that
// once per K iterations, x the halo overhead.
//
// Boundary rules (div_at, the last-row / last-column zero differences) go by
// global pixel coordinates, so a pixel inside the sensor never reads a value
// from outside it: region pixels beyond the sensor load the clamped pixel
// and compute values nobody reads.  Every pixel runs exactly the reference
// operation sequence of k_tv_march / k_pd_march, so results are bit-identical
// to the one-iteration-per-launch kernels.
#pragma once

#include <type_traits>

#include "evr_cluster.cuh"
#include "evr_fastdp.cuh"
#include "evr_kernels.cuh"

#ifndef EVR_F32_INTERIOR
#define EVR_F32_INTERIOR 1  // float32 tiles also take the interior instance
#endif

namespace evr {

// TV-L1 (surface.py:167-193), K iterations: dual ascent + projection, then
// divergence + L1 shrink + over-relaxation.  f0 is the t plane.
// Band contexts (evr_group, BANDED): the tiles cover the band's own rows
// [y0, y1) and read the K rows either side from the neighbour bands'
// buffers in place (MarchRows::at; peer memory across GPUs); out is
// indexed like in.own.
template <class T, int K, int RPT, int G, int MINB, bool BANDED>
__global__ void __launch_bounds__(32 * G, MINB)
k_tv_tile(const MarchRows<Q4<T>> in, const MarchRows<T> f0, Q4<T>* __restrict__ out, int H,
          int W, T sigma, T tau, T shrink, int early) {
  constexpr int RH = G * RPT, TIW = 32 - 2 * K, TIH = RH - 2 * K;
  __shared__ T ub_top[G][32];  // u_bar of each warp's first row
  __shared__ T py_bot[G][32];  // py of each warp's last row
  const int l = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int y0 = BANDED ? in.y0 : 0, y1 = BANDED ? in.y1 : H;
  const int rlo = max(y0 - K, 0), rhi = min(y1 + K, H) - 1;  // rows a tile may read
  const int gj = (int)blockIdx.x * TIW - K + l;
  const int gi0 = y0 + (int)blockIdx.y * TIH - K + g * RPT;
  const int jc = min(max(gj, 0), W - 1);
  T u[RPT], ub[RPT], px[RPT], py[RPT], f[RPT];
  // a band's warps whose rows are all its own skip the neighbour selects
  const bool inner = !BANDED || (gi0 >= y0 && gi0 + RPT <= y1);
  auto load_f = [&](auto banded) {
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int gr = min(max(gi0 + r, rlo), rhi);
      if constexpr (decltype(banded)::value) f[r] = f0.template at<true>(gr, jc, W);
      else f[r] = f0.at_own(gr, jc, W);
    }
  };
  auto load_s = [&](auto banded) {
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int gr = min(max(gi0 + r, rlo), rhi);
      Q4<T> q;
      if constexpr (decltype(banded)::value) q = in.template at<true>(gr, jc, W);
      else q = in.at_own(gr, jc, W);
      u[r] = q.x;
      ub[r] = q.y;
      px[r] = q.z;
      py[r] = q.w;
    }
  };
  // early: the surface t was written at least two launches ago, so its
  // loads overlap the previous launch's tail (as k_pd_tile's constants)
  const bool pre = !BANDED && sizeof(T) == 8 && early;  // float32: measured no gain
  if (pre) load_f(std::false_type{});
  pdl_wait_and_release();
  if (inner) {  // warp-uniform: a band's warps away from its edges skip the selects
    if (!pre) load_f(std::false_type{});
    load_s(std::false_type{});
  } else if constexpr (BANDED) {
    load_f(std::true_type{});
    load_s(std::true_type{});
  }
  // CTA-uniform: a tile whose whole region lies inside the sensor, one pixel
  // away from its edges, runs the iterations without boundary tests (the
  // reference's interior branch at every pixel, div_at's last else: same
  // operations, same bits)
  const int ry0 = gi0 - g * RPT, rx0 = (int)blockIdx.x * TIW - K;
  const bool interior = ry0 >= 1 && ry0 + RH <= H - 1 && rx0 >= 1 && rx0 + 32 <= W - 1;
  auto iterate = [&](auto interior_c) {
    constexpr bool IN = decltype(interior_c)::value;
    const bool XR = IN || gj < W - 1;
    auto YD = [&](int gi) { return IN || gi < H - 1; };
    auto DIV = [&](T xc, T xl, T yc, T yu, int gi) {
      if constexpr (IN) return (xc - xl) + (yc - yu);
      else return div_at(xc, gj > 0 ? xl : T(0), yc, gi > 0 ? yu : T(0), gi, gj, H, W);
    };
#pragma unroll 1
    for (int it = 0; it < K; ++it) {
      ub_top[g][l] = ub[0];
      __syncthreads();
      const T ub_below = ub_top[g < G - 1 ? g + 1 : g][l];
      if constexpr (sizeof(T) == 8) {
        // float64: branch-free fast div / sqrt so the rows' latency chains
        // overlap (evr_fastdp.cuh; rare out-of-range rows redone with IEEE)
        T dx[RPT], dy[RPT], nx[RPT], ny[RPT], nn[RPT];
        bool slow = false, proj = false;
  #pragma unroll
        for (int r = 0; r < RPT; ++r) {  // dual (surface.py:168-183)
          const int gi = gi0 + r;
          const T ub_r = __shfl_down_sync(0xffffffffu, ub[r], 1);
          const T ub_n = r < RPT - 1 ? ub[r + 1] : ub_below;
          dx[r] = XR ? ub_r - ub[r] : T(0);
          dy[r] = YD(gi) ? ub_n - ub[r] : T(0);
          nx[r] = px[r];
          ny[r] = py[r];
          nn[r] = tv_dual_pre_fx(dx[r], dy[r], sigma, nx[r], ny[r], slow);
          proj |= nn[r] != T(1);
        }
        if (__any_sync(0xffffffffu, proj)) {
  #pragma unroll
          for (int r = 0; r < RPT; ++r) fdp_div2(nx[r], ny[r], nn[r], slow);
        }
        if (slow) {
  #pragma unroll
          for (int r = 0; r < RPT; ++r) {
            nx[r] = px[r];
            ny[r] = py[r];
            tv_dual_step(dx[r], dy[r], sigma, nx[r], ny[r]);
          }
        }
  #pragma unroll
        for (int r = 0; r < RPT; ++r) {
          px[r] = nx[r];
          py[r] = ny[r];
        }
      } else {
  #pragma unroll
        for (int r = 0; r < RPT; ++r) {  // dual (surface.py:168-183)
          const int gi = gi0 + r;
          const T ub_r = __shfl_down_sync(0xffffffffu, ub[r], 1);
          const T ub_n = r < RPT - 1 ? ub[r + 1] : ub_below;
          const T dx = XR ? ub_r - ub[r] : T(0);
          const T dy = YD(gi) ? ub_n - ub[r] : T(0);
          tv_dual_step(dx, dy, sigma, px[r], py[r]);
        }
      }
      py_bot[g][l] = py[RPT - 1];
      __syncthreads();
      const T py_above = py_bot[g > 0 ? g - 1 : g][l];
  #pragma unroll
      for (int r = 0; r < RPT; ++r) {  // primal (surface.py:185-193)
        const int gi = gi0 + r;
        const T pxl = __shfl_up_sync(0xffffffffu, px[r], 1);
        const T pyu = r > 0 ? py[r - 1] : py_above;
        const T d = DIV(px[r], pxl, py[r], pyu, gi);
        T ubar;
        u[r] = tv_primal_step(d, u[r], f[r], tau, shrink, ubar);
        ub[r] = ubar;
      }
    }
  };
  // (float32 alone measured slower with the second instance, C3 0.614 ->
  // 0.620 ms; together with EVR_F32_MINMAX / SIGFOLD it is 0.585 -> 0.548)
  if ((sizeof(T) == 8 || EVR_F32_INTERIOR) && interior)
    iterate(std::true_type{});
  else
    iterate(std::false_type{});
  if (l < K || l >= 32 - K || gj >= W) return;
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int R = g * RPT + r, gi = gi0 + r;
    if (R >= K && R < RH - K && gi < y1)
      out[(int64_t)(gi - y0 + (BANDED ? in.olo : 0)) * W + gj] = Q4<T>{u[r], ub[r], px[r], py[r]};
  }
}

// Manifold-TV + KL primal-dual (solve.py:233-252), K iterations: q = A^T p,
// divergence, KL prox + over-relaxation, dual ascent + ball projection.
// The metric constants of the region are loaded once (M: MetricPackF32
// recomputes the matrix from the slopes, MetricPackF64 reads it) and stay
// in registers for the K iterations.  DT, the data term of the primal step
// (float64 operator solves): 0 = KL (packed slots beta, 4 beta f), 1 = ROF
// (rof_manifold_solve, solve.py:285-287: slots 1 / (1 + w), w f), 2 = L1
// (slots w = tau lam sqrtG, f; the soft shrink of k_l1_primal).
//
// Clustered form (CX x CY > 1, launched with cluster dims {CX, CY}): the
// region is the cluster's, CX*32 columns x CY*G*RPT rows, one 32 x G*RPT
// block per CTA, and only its outer edge is halo.  Inside the cluster a
// half-step's one missing neighbour value crosses to the adjacent CTA
// through DSMEM: q of the right / lower edge into the right / lower CTA
// before the primal, v of the left / upper edge into the left / upper CTA
// before the dual, each st.async counting its bytes off the receiver's
// mbarrier.  One buffer per direction suffices: a CTA sends its next value
// into a neighbour only after receiving the neighbour's reply to the last.
enum : int { DT_KL = 0, DT_ROF = 1, DT_L1 = 2 };
template <class T, int K, int RPT, int G, int MINB, class M, bool BANDED, int DT = DT_KL,
          bool PREV = false, int CX = 1, int CY = 1>
__global__ void __launch_bounds__(32 * G, MINB)
k_pd_tile(const MarchRows<Q4<T>> in, const __grid_constant__ M m, Q4<T>* __restrict__ out, int H, int W, T tau,
          T sigma, T umin, T umax, int early, T* __restrict__ prev) {
  constexpr bool CL = CX * CY > 1;
  constexpr int RH = G * RPT, CW = 32 * CX, CH = RH * CY, TIW = CW - 2 * K, TIH = CH - 2 * K;
  __shared__ T qy_bot[G][32];  // qy of each warp's last row
  __shared__ T v_top[G][32];   // v of each warp's first row
  __shared__ T x_qx[CL ? RH : 1], x_qy[CL ? 32 : 1];  // from the left / upper CTA
  __shared__ T x_vr[CL ? RH : 1], x_vb[CL ? 32 : 1];  // from the right / lower CTA
  __shared__ uint64_t x_bar[2];                       // primal-in, dual-in
  const int l = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int cx = CL ? (int)blockIdx.x % CX : 0, cy = CL ? (int)blockIdx.y % CY : 0;
  const int y0 = BANDED ? in.y0 : 0, y1 = BANDED ? in.y1 : H;
  const int rlo = max(y0 - K, 0), rhi = min(y1 + K, H) - 1;
  const int gj = (int)blockIdx.x / CX * TIW - K + cx * 32 + l;
  const int gi0 = y0 + (int)blockIdx.y / CY * TIH - K + cy * RH + g * RPT;
  // bytes each half-step receives (0: an outer side of the cluster)
  const unsigned in_p = (cx > 0 ? RH * sizeof(T) : 0) + (cy > 0 ? 32 * sizeof(T) : 0);
  const unsigned in_d = (cx < CX - 1 ? RH * sizeof(T) : 0) + (cy < CY - 1 ? 32 * sizeof(T) : 0);
  unsigned to_r = 0, to_b = 0, to_l = 0, to_a = 0;  // mapped slot bases in the neighbours
  unsigned me = 0;
  if constexpr (CL) {
    me = cl_rank();
    EVR_ASSERT(me == (unsigned)(cx + cy * CX));
    if (threadIdx.x == 0) {
      cl_bar_init(&x_bar[0]);
      cl_bar_init(&x_bar[1]);
      cl_fence_init();
    }
    cl_arrive();  // released; waited for after the loads, before the first send
    if (cx < CX - 1) to_r = cl_map(smem_addr(x_qx), me + 1);
    if (cy < CY - 1) to_b = cl_map(smem_addr(x_qy), me + CX);
    if (cx > 0) to_l = cl_map(smem_addr(x_vr), me - 1);
    if (cy > 0) to_a = cl_map(smem_addr(x_vb), me - CX);
  }
  const int jc = min(max(gj, 0), W - 1);
  T p1[RPT], p2[RPT], p3[RPT], u[RPT];
  Coef<T> cf[RPT];
  T sg[RPT], beta[RPT], fb[RPT];
  T ysg[sizeof(T) == 8 ? RPT : 1];  // float64: refined 1 / sqrtG, hoisted
  typename M::Raw craw[RPT];
  const bool inner = !BANDED || (gi0 >= y0 && gi0 + RPT <= y1);
  auto load_c = [&](auto banded) {
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int gr = min(max(gi0 + r, rlo), rhi);
      if constexpr (decltype(banded)::value) craw[r] = m.template load<true>(gr, y1, jc, W);
      else craw[r] = m.load_own(gr, in.y0, in.olo, jc, W);
    }
  };
  auto load_s = [&](auto banded) {
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int gr = min(max(gi0 + r, rlo), rhi);
      Q4<T> q;
      if constexpr (decltype(banded)::value) q = in.template at<true>(gr, jc, W);
      else q = in.at_own(gr, jc, W);
      p1[r] = q.x;
      p2[r] = q.y;
      p3[r] = q.z;
      u[r] = q.w;
    }
  };
  // early: the constants were packed at least two launches ago (every
  // launch of the list passes its griddepcontrol.wait before releasing the
  // next), so their loads go out before this launch's dependency wait and
  // overlap the previous launch's tail; the state waits for it
  const bool pre = !BANDED && sizeof(T) == 8 && early;  // float32: measured no gain
  if constexpr (M::kTma) {
    // TMA form (whole sensor, float64): the region's constants and state come
    // in as two 2-D boxes (RH rows x 32 pixels; the box's part off the sensor
    // is zero-filled and never read) issued by one thread, the constants
    // before the dependency wait when early
    static_assert(!BANDED && !CL && sizeof(T) == 8, "TMA tiles: whole-sensor float64");
    extern __shared__ __align__(128) unsigned char tma_dyn[];
    Q4<T>* const s_st = reinterpret_cast<Q4<T>*>(tma_dyn);  // RH x 32 quads
    Q4<T>* const s_c = s_st + RH * 32;                     // RH x 32 x 2 quads
    __shared__ uint64_t t_bar;
    const int x0 = gj - l, yr0 = gi0 - g * RPT;
    if (threadIdx.x == 0) {
      cl_bar_init(&t_bar);
      cl_fence_init();
      cl_expect(&t_bar, RH * 32 * 3 * sizeof(Q4<T>));
      if (pre) tma_load_2d(s_c, &m.tc, 8 * x0, yr0, &t_bar);
    }
    pdl_wait_and_release();
    if (threadIdx.x == 0) {
      if (!pre) tma_load_2d(s_c, &m.tc, 8 * x0, yr0, &t_bar);
      tma_load_2d(s_st, &m.ts, 4 * x0, yr0, &t_bar);
    }
    __syncthreads();  // the barrier's init before anyone waits on it
    cl_wait(&t_bar, 0);
    // a region pixel off the sensor takes its clamped pixel (inside the box),
    // as the global-load form does: its halo values stay finite, so no warp
    // drops to the IEEE slow paths
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int k = (min(max(gi0 + r, 0), H - 1) - yr0) * 32 + (jc - x0);
      const Q4<T> q = s_st[k];
      p1[r] = q.x;
      p2[r] = q.y;
      p3[r] = q.z;
      u[r] = q.w;
      craw[r] = typename M::Raw{s_c[2 * k], s_c[2 * k + 1]};
    }
  } else {
    if (pre) load_c(std::false_type{});
    pdl_wait_and_release();
    if (inner) {  // warp-uniform: a band's warps away from its edges skip the selects
      if (!pre) load_c(std::false_type{});
      load_s(std::false_type{});
    } else if constexpr (BANDED) {
      load_c(std::true_type{});
      load_s(std::true_type{});
    }
  }
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    m.finish(craw[r], cf[r], sg[r], beta[r], fb[r]);
    if constexpr (sizeof(T) == 8) ysg[r] = fdp_recip(sg[r]);
  }
  const int ry0 = gi0 - g * RPT, rx0 = (int)blockIdx.x / CX * TIW - K + cx * 32;
  const bool interior = ry0 >= 1 && ry0 + RH <= H - 1 && rx0 >= 1 && rx0 + 32 <= W - 1;
  if constexpr (CL) cl_sync_wait();  // every CTA's barriers initialised
  // the kept pixels: the cluster region's interior
  auto keep_col = [&] { return cx * 32 + l >= K && cx * 32 + l < CW - K && gj < W; };
  auto keep_row = [&](int r) {
    const int R = cy * RH + g * RPT + r;
    return R >= K && R < CH - K;
  };
  auto iterate = [&](auto interior_c) {
    constexpr bool IN = decltype(interior_c)::value;
    const bool XR = IN || gj < W - 1;
    auto YD = [&](int gi) { return IN || gi < H - 1; };
    auto DIV = [&](T xc, T xl, T yc, T yu, int gi) {
      if constexpr (IN) return (xc - xl) + (yc - yu);
      else return div_at(xc, gj > 0 ? xl : T(0), yc, gi > 0 ? yu : T(0), gi, gj, H, W);
    };
#pragma unroll 1
    for (int it = 0; it < K; ++it) {
      if (PREV && it == K - 1) {  // the final launch: u before the last iteration
        if (keep_col()) {  // (k_unpack_rel's rel_change)
  #pragma unroll
          for (int r = 0; r < RPT; ++r) {
            const int gi = gi0 + r;
            if (keep_row(r) && gi < y1)
              prev[(int64_t)(gi - y0 + (BANDED ? in.olo : 0)) * W + gj] = u[r];
          }
        }
      }
      T qx[RPT], qy[RPT], v[RPT];
  #pragma unroll
      for (int r = 0; r < RPT; ++r) q_of(cf[r], p1[r], p2[r], p3[r], qx[r], qy[r]);
      qy_bot[g][l] = qy[RPT - 1];
      if constexpr (CL) {
        if (to_r && l == 31) {
          const unsigned bar = cl_map(smem_addr(&x_bar[0]), me + 1);
  #pragma unroll
          for (int r = 0; r < RPT; ++r) cl_send(to_r + (g * RPT + r) * sizeof(T), qx[r], bar);
        }
        if (to_b && g == G - 1)
          cl_send(to_b + l * sizeof(T), qy[RPT - 1], cl_map(smem_addr(&x_bar[0]), me + CX));
      }
      __syncthreads();
      T qy_above = qy_bot[g > 0 ? g - 1 : g][l];
      if constexpr (CL) {
        if (in_p) {
          if (threadIdx.x == 0) cl_expect(&x_bar[0], in_p);
          cl_wait(&x_bar[0], it & 1);
        }
        if (g == 0 && cy > 0) qy_above = x_qy[l];
      }
      {
        T d[RPT], nu[RPT];
        bool slow = false;
  #pragma unroll
        for (int r = 0; r < RPT; ++r) {  // primal (solve.py:233-245)
          const int gi = gi0 + r;
          T qxl = __shfl_up_sync(0xffffffffu, qx[r], 1);
          if (CL && l == 0 && cx > 0) qxl = x_qx[g * RPT + r];
          const T qyu = r > 0 ? qy[r - 1] : qy_above;
          d[r] = DIV(qx[r], qxl, qy[r], qyu, gi);
          if constexpr (DT == DT_ROF) {
            nu[r] = rof_primal(d[r], u[r], fb[r], beta[r], tau);  // fb = w f, beta = 1 / (1 + w)
          } else if constexpr (DT == DT_L1) {
            const T t1 = Arith<T>::mad(d[r], tau, u[r]);  // fb = f, beta = w
            nu[r] = t1 - vclip(t1 - fb[r], -beta[r], beta[r]);
          } else if constexpr (sizeof(T) == 8) {
            nu[r] = kl_primal_fx(d[r], u[r], beta[r], fb[r], tau, umin, umax, slow);
          } else {
            nu[r] = kl_primal(d[r], u[r], beta[r], fb[r], tau, umin, umax);
          }
        }
        if (DT == DT_KL && sizeof(T) == 8 && slow) {
  #pragma unroll
          for (int r = 0; r < RPT; ++r) nu[r] = kl_primal(d[r], u[r], beta[r], fb[r], tau, umin, umax);
        }
  #pragma unroll
        for (int r = 0; r < RPT; ++r) {
          v[r] = Arith<T>::mad(nu[r], T(2), -u[r]);
          u[r] = nu[r];
        }
      }
      v_top[g][l] = v[0];
      if constexpr (CL) {
        if (to_l && l == 0) {
          const unsigned bar = cl_map(smem_addr(&x_bar[1]), me - 1);
  #pragma unroll
          for (int r = 0; r < RPT; ++r) cl_send(to_l + (g * RPT + r) * sizeof(T), v[r], bar);
        }
        if (to_a && g == 0)
          cl_send(to_a + l * sizeof(T), v[0], cl_map(smem_addr(&x_bar[1]), me - CX));
      }
      __syncthreads();
      T v_below = v_top[g < G - 1 ? g + 1 : g][l];
      if constexpr (CL) {
        if (in_d) {
          if (threadIdx.x == 0) cl_expect(&x_bar[1], in_d);
          cl_wait(&x_bar[1], it & 1);
        }
        if (g == G - 1 && cy < CY - 1) v_below = x_vb[l];
      }
      if constexpr (sizeof(T) == 8) {
        T gx[RPT], gy[RPT], n1[RPT], n2[RPT], n3[RPT], nn[RPT];
        bool slow = false, proj = false;
  #pragma unroll
        for (int r = 0; r < RPT; ++r) {  // dual (solve.py:246-252)
          const int gi = gi0 + r;
          T vr = __shfl_down_sync(0xffffffffu, v[r], 1);
          if (CL && l == 31 && cx < CX - 1) vr = x_vr[g * RPT + r];
          const T vd = r < RPT - 1 ? v[r + 1] : v_below;
          gx[r] = XR ? vr - v[r] : T(0);
          gy[r] = YD(gi) ? vd - v[r] : T(0);
          n1[r] = p1[r];
          n2[r] = p2[r];
          n3[r] = p3[r];
          nn[r] = dual_pre_fx_r(cf[r], sigma, gx[r], gy[r], sg[r], ysg[r], n1[r], n2[r], n3[r],
                                slow);
          proj |= nn[r] != T(1);
        }
        if (__any_sync(0xffffffffu, proj)) {
  #pragma unroll
          for (int r = 0; r < RPT; ++r) fdp_div3(n1[r], n2[r], n3[r], nn[r], slow);
        }
        if (slow) {
  #pragma unroll
          for (int r = 0; r < RPT; ++r) {
            n1[r] = p1[r];
            n2[r] = p2[r];
            n3[r] = p3[r];
            dual_step(cf[r], sigma, gx[r], gy[r], sg[r], n1[r], n2[r], n3[r]);
          }
        }
  #pragma unroll
        for (int r = 0; r < RPT; ++r) {
          p1[r] = n1[r];
          p2[r] = n2[r];
          p3[r] = n3[r];
        }
      } else {
  #pragma unroll
        for (int r = 0; r < RPT; ++r) {  // dual (solve.py:246-252)
          const int gi = gi0 + r;
          T vr = __shfl_down_sync(0xffffffffu, v[r], 1);
          if (CL && l == 31 && cx < CX - 1) vr = x_vr[g * RPT + r];
          const T vd = r < RPT - 1 ? v[r + 1] : v_below;
          const T gx = XR ? vr - v[r] : T(0);
          const T gy = YD(gi) ? vd - v[r] : T(0);
          dual_step(cf[r], sigma, gx, gy, sg[r], p1[r], p2[r], p3[r]);
        }
      }
    }
  };
  // (float32 alone measured slower with the second instance, C3 0.614 ->
  // 0.620 ms; together with EVR_F32_MINMAX / SIGFOLD it is 0.585 -> 0.548)
  if ((sizeof(T) == 8 || EVR_F32_INTERIOR) && interior)
    iterate(std::true_type{});
  else
    iterate(std::false_type{});
  if (!keep_col()) return;
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int gi = gi0 + r;
    if (keep_row(r) && gi < y1)
      out[(int64_t)(gi - y0 + (BANDED ? in.olo : 0)) * W + gj] = Q4<T>{p1[r], p2[r], p3[r], u[r]};
  }
}

}  // namespace evr
