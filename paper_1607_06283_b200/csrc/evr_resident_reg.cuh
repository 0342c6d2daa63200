// evr_resident_reg.cuh -- resident engine, float32, for sensors whose band
// frames do not fit shared memory (1280x720 at real time, 640x480).
//
// Same decomposition, exchange protocol and phase order as k_resident
// (evr_resident.cuh: row bands, one CTA per SM, one tagged-word exchange of
// boundary rows per iteration); what changes is where the per-pixel fields
// live:
//   registers : u, p1, p2, p3 (solver state) and u, f0 (TV-L1) of the
//               thread's own columns -- only their owner ever reads them;
//   shared    : the fields neighbours read -- v, q_x, q_y (solver),
//               u_bar, p_x, p_y (TV-L1, aliased) -- plus t_x, t_y and fb;
//   recomputed: G, sqrt(G) and the 3x2 metric matrix, from (t_x, t_y) at
//               each use with the float engine's own operations
//               (metric_G; a_k = num_k / G as num_k * rcp(G), which is what
//               __fdividef compiles to), so every value equals the
//               shared-memory float engine's bit for bit.
// Six float planes of (R+2) rows instead of fourteen: a 1280-wide band of
// 5 rows is 215 KB.
#pragma once

#include <cstdint>

#include "evr_ingest.cuh"
#include "evr_kernels.cuh"
#include "evr_math.cuh"
#include "evr_resident.cuh"

namespace evr {

enum : int { SR_V = 0, SR_QX, SR_QY, SR_TX, SR_TY, SR_FB, SR_COUNT };

__host__ __device__ inline size_t resident_reg_frame_bytes(int R, int W) {
  return (size_t)resident_plane_stride(R, W) * SR_COUNT * sizeof(float);
}

#define EVR_CS(cs) _Pragma("unroll") for (int cs = 0; cs < CS; ++cs)
#define EVR_R(r) _Pragma("unroll") for (int r = 0; r < RM + 2; ++r)

template <int NT, int CS, int RM>
__global__ void __launch_bounds__(NT, 1) k_resident_reg(const ResArgs<float> a) {
  using T = float;
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
  T* pl = reinterpret_cast<T*>(smem_raw);
  T* const V = pl + SR_V * PS;
  T* const QX = pl + SR_QX * PS;
  T* const QY = pl + SR_QY * PS;
  T* const TX = pl + SR_TX * PS;
  T* const TY = pl + SR_TY * PS;
  T* const FB = pl + SR_FB * PS;
  T* const TUB = V;   // TV-L1 planes alias the solver's exchange planes
  T* const TPX = QX;
  T* const TPY = QY;
  T* const TD = QY;   // denoised surface, TV-L1 end .. metric
  double* const F64 = reinterpret_cast<double*>(TX);  // ingest .. metric (TX, TY)

  const PacketHdr* hdr = a.hdr;
  const evr_event* __restrict__ ev = reinterpret_cast<const evr_event*>(hdr + 1);
  const int64_t n_ev = hdr->n;
  const double now = (double)hdr->now;
  const double window = hdr->window;
  const unsigned long long epoch = (unsigned long long)hdr->seq << 24;
  const unsigned tag_base = (unsigned)hdr->seq << 16;
  const size_t xside = (size_t)3 * W;
  const size_t xslot = (size_t)a.nb * 2 * xside;
  unsigned long long* const xw = reinterpret_cast<unsigned long long*>(a.xchg);
  auto gk_of = [&](int r, int j) { return (int64_t)(r0 - 1 + r) * W + j; };
  auto col = [&](int cs) { return tid + cs * NT; };
  auto live = [&](int r, int lo, int hi) { return r >= lo && r <= hi; };

  auto ll_put = [&](int step, int r, int j, int field, T v) {
    unsigned long long w[1];
    LLWords<T>::pack(v, tag_base + (unsigned)step, w);
    unsigned long long* base = xw + (step & 1) * xslot + (size_t)b * 2 * xside + (size_t)field * W + j;
    if (r == 1) st_relaxed_u64(base, w[0]);
    if (r == Rb) st_relaxed_u64(base + xside, w[0]);
  };
  // poll the neighbours' boundary words of `step` for column j: out[side][field]
  auto ll_get = [&](int step, int j, int nf, T out[2][3]) {
    const unsigned want = tag_base + (unsigned)step;
    const unsigned long long* slot = xw + (step & 1) * xslot;
    const unsigned long long* src[2] = {slot + (size_t)(b - 1) * 2 * xside + xside + j,
                                        slot + (size_t)(b + 1) * 2 * xside + j};
    unsigned long long w[2][3];
    bool ready;
    do {
      ready = true;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        if (s == 0 ? !has_up : !has_dn) continue;
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          if (f >= nf) break;
          w[s][f] = ld_relaxed_u64(src[s] + (size_t)f * W);
          ready &= (unsigned)(w[s][f] >> 32) == want;
        }
      }
    } while (!ready);
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int f = 0; f < 3; ++f) out[s][f] = LLWords<T>::unpack(&w[s][f]);
  };
  int tmark = 0;  // optional phase timeline, same marks as k_resident
  auto mark = [&]() {
    if (a.trace && tid == 0 && tmark < 256) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
      a.trace[(size_t)b * 256 + tmark] = t;
    }
    ++tmark;
  };
  mark();
  auto flag_publish = [&](int step) {
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release_u64(&a.flags[b], epoch | (unsigned long long)step);
    }
  };
  auto flag_wait = [&](int b_lo, int b_hi, int step) {
    const unsigned long long target = epoch | (unsigned long long)step;
    if (tid < b_hi - b_lo + 1 && b_lo + tid != b)
      while (ld_acquire_u64(&a.flags[b_lo + tid]) < target) __nanosleep(20);
    __syncthreads();
  };

  // per-thread state of the owned columns, local rows 0 .. RM+1
  T tu[CS][RM + 2], t0[CS][RM + 2];
  T u[CS][RM + 2], p1[CS][RM + 2], p2[CS][RM + 2], p3[CS][RM + 2];

  // ---------------------------------------------------------------- load --
  EVR_CS(cs) {
    const int j = col(cs);
    if (j >= W) continue;
    int64_t rv[RM + 2];
    double fv[RM + 2];
    EVR_R(r) {
      if (!live(r, lo_halo, hi_halo)) continue;
      const int64_t gk = gk_of(r, j);
      rv[r] = a.manifold ? a.raw[gk] : 0;
      fv[r] = r >= 1 ? a.f[gk] : 0.0;
    }
    EVR_R(r) {
      if (!live(r, lo_halo, hi_halo)) continue;
      const int l = r * W + j;
      if (a.manifold) {
        TUB[l] = (T)normalize_at((double)rv[r], now, a.t_scale, window);
        TPX[l] = T(0);
        TPY[l] = T(0);
      }
      if (r >= 1) F64[l] = fv[r];
    }
  }
  __syncthreads();

  // -------------------------------------------------------------- ingest --
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
          if (a.manifold) TUB[l] = (T)normalize_at((double)t, now, a.t_scale, window);
          if (lr >= 1 && lr <= Rb) a.raw[(int64_t)(r0 - 1) * W + l] = t;
        });
  }
  mark();
  // TV-L1 cold start u = u_bar = f0 = t (surface.py:161-165)
  EVR_CS(cs) {
    const int j = col(cs);
    EVR_R(r) {
      if (j < W && live(r, lo_halo, hi_halo) && a.manifold) {
        tu[cs][r] = TUB[r * W + j];
        t0[cs][r] = tu[cs][r];
      }
    }
  }

  // ------------------------------------------------------------ TV-L1 ----
  int step = 0;
  if (a.manifold) {
    for (int it = 0; it < a.tv_iters; ++it) {
      const bool pub = it < a.tv_iters - 1;
      if (it > 0) {
        EVR_CS(cs) {
          const int j = col(cs);
          if (j >= W) continue;
          T h[2][3];
          ll_get(step, j, 1, h);
          if (has_up) TUB[j] = h[0][0];
          if (has_dn) TUB[(Rb + 1) * W + j] = h[1][0];
        }
        __syncthreads();
      }
      mark();
      // dual ascent + projection (surface.py:168-183), own rows + halo above
      EVR_CS(cs) {
        const int j = col(cs);
        if (j >= W) continue;
        T ub[RM + 2], ubr[RM + 2], px[RM + 2], py[RM + 2];
        EVR_R(r) {
          const int l = r * W + j;
          if (live(r, lo_halo, hi_halo)) ub[r] = TUB[l];
          if (live(r, lo_halo, Rb)) {
            ubr[r] = j < W - 1 ? TUB[l + 1] : T(0);
            px[r] = TPX[l];
            py[r] = TPY[l];
          }
        }
        EVR_R(r) {
          if (!live(r, lo_halo, Rb)) continue;
          const T dx = j < W - 1 ? ubr[r] - ub[r] : T(0);
          const T dy = r0 - 1 + r < H - 1 ? ub[r < RM + 1 ? r + 1 : r] - ub[r] : T(0);
          tv_dual_step(dx, dy, a.tv_step, px[r], py[r]);
          TPX[r * W + j] = px[r];
          TPY[r * W + j] = py[r];
        }
      }
      __syncthreads();
      // primal + L1 shrink (surface.py:185-193), own rows
      EVR_CS(cs) {
        const int j = col(cs);
        if (j >= W) continue;
        T pyc[RM + 2], pxc[RM + 2], pxl[RM + 2];
        EVR_R(r) {
          const int l = r * W + j;
          if (live(r, lo_halo, Rb)) pyc[r] = TPY[l];
          if (live(r, 1, Rb)) {
            pxc[r] = TPX[l];
            pxl[r] = j > 0 ? TPX[l - 1] : T(0);
          }
        }
        EVR_R(r) {
          if (!live(r, 1, Rb)) continue;
          const int gi = r0 - 1 + r;
          const T d = div_at(pxc[r], pxl[r], pyc[r], gi > 0 ? pyc[r > 0 ? r - 1 : 0] : T(0), gi,
                             j, H, W);
          T ubv;
          tu[cs][r] = tv_primal_step(d, tu[cs][r], t0[cs][r], a.tv_step, a.shrink, ubv);
          TUB[r * W + j] = ubv;
          if (pub) ll_put(step + 1, r, j, 0, ubv);
        }
      }
      if (pub) ++step;
    }
    __syncthreads();
    // np.clip(u, 0, t_scale) (surface.py:195) -> global t and TD
    EVR_CS(cs) {
      const int j = col(cs);
      EVR_R(r) {
        if (j >= W || !live(r, 1, Rb)) continue;
        const T td = vclip(tu[cs][r], T(0), a.t_scaleT);
        a.t[gk_of(r, j)] = td;
        TD[r * W + j] = td;
      }
    }
  }
  const int s_met = a.tv_iters + 1;
  flag_publish(s_met);
  if (a.manifold) {
    flag_wait(band.of_row(has_up ? r0 - 1 : r0), band.of_row(r1 + 1 < H ? r1 + 1 : H - 1), s_met);
    for (int j = tid; j < W; j += NT) {
      if (has_up) TD[j] = __ldcg(a.t + gk_of(0, j));
      if (has_dn) TD[(Rb + 1) * W + j] = __ldcg(a.t + gk_of(Rb + 1, j));
    }
  }
  step = s_met;
  __syncthreads();

  mark();
  // ------------------------------------------------------------ metric ---
  // surface slopes of pixel (r, j) from TD (row below the halo from L2)
  auto slopes = [&](int r, int j, T& gx, T& gy) {
    gx = T(0);
    gy = T(0);
    if (!a.manifold) return;
    const int l = r * W + j;
    const T tc = TD[l];
    gx = j < W - 1 ? TD[l + 1] - tc : T(0);
    if (r0 - 1 + r < H - 1) gy = (r <= Rb ? TD[l + W] : __ldcg(a.t + gk_of(r + 1, j))) - tc;
  };
  // pass 1: solver constant fb (reads F64), debug planes, warm-start u, p
  EVR_CS(cs) {
    const int j = col(cs);
    if (j >= W) continue;
    EVR_R(r) {
      if (!live(r, lo_halo, hi_halo)) continue;
      const int l = r * W + j;
      const int64_t gk = gk_of(r, j);
      T gx, gy;
      slopes(r, j, gx, gy);
      const T g = metric_G(gx, gy);
      const T s = Arith<T>::sqrt(g);
      if (r >= 1) {
        FB[l] = T(4) * (a.tl * s) * (T)F64[l];
        u[cs][r] = a.u[gk];
        p1[cs][r] = a.p1[gk];
        p2[cs][r] = a.p2[gk];
        p3[cs][r] = a.p3[gk];
      }
      if (r >= 1 && r <= Rb) {
        a.tx[gk] = gx;
        a.ty[gk] = gy;
        a.G[gk] = g;
        a.sg[gk] = s;
      }
    }
  }
  __syncthreads();  // F64 (aliasing TX, TY) is dead
  // pass 2: the slopes themselves (TD still intact)
  EVR_CS(cs) {
    const int j = col(cs);
    if (j >= W) continue;
    EVR_R(r) {
      if (!live(r, lo_halo, hi_halo)) continue;
      T gx, gy;
      slopes(r, j, gx, gy);
      TX[r * W + j] = gx;
      TY[r * W + j] = gy;
    }
  }
  __syncthreads();  // TD (aliasing QY) is dead
  // pass 3: q = A^T p of the warm start (halo-above p straight from L2)
  EVR_CS(cs) {
    const int j = col(cs);
    if (j >= W) continue;
    EVR_R(r) {
      if (!live(r, lo_halo, hi_halo)) continue;
      const int l = r * W + j;
      const MetricPx m = metric_px(TX[l], TY[l]);
      T qx, qy;
      if (r >= 1) {
        q_of(m.c, p1[cs][r], p2[cs][r], p3[cs][r], qx, qy);
      } else {
        const int64_t gk = gk_of(r, j);
        q_of(m.c, a.p1[gk], a.p2[gk], a.p3[gk], qx, qy);
      }
      QX[l] = qx;
      QY[l] = qy;
    }
  }
  __syncthreads();

  // ------------------------------------------------------- primal-dual ---
  mark();
  double rd = 0.0, ro = 0.0;
  for (int it = 0; it < a.pd_iters; ++it) {
    const bool last = it == a.pd_iters - 1;
    if (it > 0) {
      // neighbours' p rows -> halo registers, their q -> QX / QY
      EVR_CS(cs) {
        const int j = col(cs);
        if (j >= W) continue;
        T h[2][3];
        ll_get(step, j, 3, h);
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (s == 0 ? !has_up : !has_dn) continue;
          const int r = s == 0 ? 0 : Rb + 1;
          const int l = r * W + j;
          const MetricPx m = metric_px(TX[l], TY[l]);
          T qx, qy;
          q_of(m.c, h[s][0], h[s][1], h[s][2], qx, qy);
          QX[l] = qx;
          QY[l] = qy;
          // keep the halo-below dual for the primal recompute (local row Rb+1)
          if (s == 1) {
            EVR_R(rr) {
              if (rr == Rb + 1) {
                p1[cs][rr] = h[1][0];
                p2[cs][rr] = h[1][1];
                p3[cs][rr] = h[1][2];
              }
            }
          }
        }
      }
      __syncthreads();
    }
    mark();
    // KL prox + over-relaxation (solve.py:234-252), own rows + halo below
    EVR_CS(cs) {
      const int j = col(cs);
      if (j >= W) continue;
      T qyc[RM + 2], qxc[RM + 2], qxl[RM + 2];
      EVR_R(r) {
        const int l = r * W + j;
        if (live(r, lo_halo, hi_halo)) qyc[r] = QY[l];
        if (live(r, 1, hi_halo)) {
          qxc[r] = QX[l];
          qxl[r] = j > 0 ? QX[l - 1] : T(0);
        }
      }
      EVR_R(r) {
        if (!live(r, 1, hi_halo)) continue;
        const int l = r * W + j;
        const int gi = r0 - 1 + r;
        const T d = div_at(qxc[r], qxl[r], qyc[r], gi > 0 ? qyc[r > 0 ? r - 1 : 0] : T(0), gi, j,
                           H, W);
        const T sg = Arith<T>::sqrt(metric_G(TX[l], TY[l]));
        const T uk = u[cs][r];
        const T nu = kl_primal(d, uk, a.tl * sg, FB[l], a.tau, a.uminT, a.umaxT);
        V[l] = Arith<T>::mad(nu, T(2), -uk);
        u[cs][r] = nu;
        if (last && r <= Rb) {
          const double e = (double)nu - (double)uk;
          rd += e * e;
          ro += (double)uk * (double)uk;
        }
      }
    }
    mark();  // primal issued (thread 0)
    __syncthreads();
    mark();  // primal done
    // dual ascent + ball projection (solve.py:170-201), own rows; refresh q
    EVR_CS(cs) {
      const int j = col(cs);
      if (j >= W) continue;
      T vv[RM + 2], vr[RM + 2];
      EVR_R(r) {
        const int l = r * W + j;
        if (live(r, 1, hi_halo)) vv[r] = V[l];
        if (live(r, 1, Rb)) vr[r] = j < W - 1 ? V[l + 1] : T(0);
      }
      EVR_R(r) {
        if (!live(r, 1, Rb)) continue;
        const int l = r * W + j;
        const T gx = j < W - 1 ? vr[r] - vv[r] : T(0);
        const T gy = r0 - 1 + r < H - 1 ? vv[r < RM + 1 ? r + 1 : r] - vv[r] : T(0);
        const MetricPx m = metric_px(TX[l], TY[l]);
        dual_step(m.c, a.sigma, gx, gy, m.sg, p1[cs][r], p2[cs][r], p3[cs][r]);
        T qx, qy;
        q_of(m.c, p1[cs][r], p2[cs][r], p3[cs][r], qx, qy);
        QX[l] = qx;
        QY[l] = qy;
        if (!last) {
          ll_put(step + 1, r, j, 0, p1[cs][r]);
          ll_put(step + 1, r, j, 1, p2[cs][r]);
          ll_put(step + 1, r, j, 2, p3[cs][r]);
        }
      }
    }
    mark();  // dual issued (thread 0)
    if (!last) ++step;
  }
  if (a.pd_iters < 2) {
    flag_publish(s_met + 1);
    flag_wait(has_up ? b - 1 : b, has_dn ? b + 1 : b, s_met + 1);
  }
  __syncthreads();

  // ---------------------------------------------------------- epilogue ---
  EVR_CS(cs) {
    const int j = col(cs);
    EVR_R(r) {
      if (j >= W || !live(r, 1, Rb)) continue;
      const int64_t gk = gk_of(r, j);
      a.u[gk] = u[cs][r];
      a.f[gk] = (double)u[cs][r];
      a.p1[gk] = p1[cs][r];
      a.p2[gk] = p2[cs][r];
      a.p3[gk] = p3[cs][r];
    }
  }
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

#undef EVR_CS
#undef EVR_R

}  // namespace evr
