// evr_kernels.cuh -- streaming-engine kernels (one launch per half-step,
// fields in HBM / L2) and the operator-level kernels of the C ABI.
//
// Layout in device memory: every per-pixel field is its own row-major (H, W)
// plane (SoA), 256-byte aligned, so a warp's 32 consecutive columns are one
// coalesced 128 / 256-byte transaction.  The dual field p lives as three
// planes p1, p2, p3 (the reference's _Loop keeps the same split,
// solve.py:133-135); the interleaved (H, W, 3) host layout is converted at
// the ABI boundary only.
#pragma once

#include <cuda.h>  // CUtensorMap

#include <cstdint>

#include "evr_ingest.cuh"
#include "evr_math.cuh"
#include "../../include/evr.h"

namespace evr {

// Per-packet scalars the host writes before each packet, so one captured
// CUDA graph serves every packet.
struct PacketHdr {
  int64_t n;        // events in the packet
  int64_t now;      // events[-1].timestamp (pipeline.py:160)
  double window;    // surface window (pipeline.py:128-132)
  int64_t seq;      // packet sequence number
};

template <class T> struct CoefPlanes {
  T *a11, *a12, *a22, *a31, *a32;
  __device__ __forceinline__ Coef<T> at(int64_t k) const {
    return Coef<T>{a11[k], a12[k], a22[k], a31[k], a32[k]};
  }
};

#define EVR_2D_INDEX                                   \
  const int j = blockIdx.x * blockDim.x + threadIdx.x; \
  const int i = blockIdx.y * blockDim.y + threadIdx.y; \
  if (i >= H || j >= W) return;                        \
  const int64_t k = (int64_t)i * W + j;

// Rows [ilo, ihi] of a context's planes, local row i being global sensor row
// row0 + i of a Htot-row sensor.  A whole-sensor context has row0 = 0 and
// Htot = its height; a band context (evr_group) keeps one halo row above and
// below its own rows, and every boundary rule of the reference is applied
// by GLOBAL row index.
struct Geo {
  int W, row0, Htot, ilo, ihi;
};
#define EVR_GEO_INDEX                                                         \
  const int j = blockIdx.x * blockDim.x + threadIdx.x;                        \
  const int i = g.ilo + (int)(blockIdx.y * blockDim.y + threadIdx.y);         \
  if (i > g.ihi || j >= g.W) return;                                          \
  const int W = g.W;                                                          \
  const int gi = g.row0 + i;                                                  \
  const int64_t k = (int64_t)i * W + j;

// ---------------------------------------------------------------- ingest --
// apply_event (pipeline.py:114-121) for every event of the packet, bit-exact
// including duplicates (evr_ingest.cuh): CTA b owns rows
// [b*rows_per, (b+1)*rows_per) and applies the packet's events of those rows
// in stream order; no two CTAs touch the same pixel.
template <int NT>
__global__ void __launch_bounds__(NT)
k_ingest(const PacketHdr* __restrict__ hdr, double* __restrict__ f, int64_t* __restrict__ raw,
         int Htot, int W, int y0, int nrows, int rows_per, double c_pos, double c_neg,
         double u_min, double u_max, int* err) {
  __shared__ IngestShared<NT> sm;
  // the packet's events follow the header in the staging buffer
  const evr_event* __restrict__ ev = reinterpret_cast<const evr_event*>(hdr + 1);
  // f / raw point at global row y0; this CTA takes global rows [row_lo, row_hi]
  const int row_lo = y0 + blockIdx.x * rows_per;
  const int row_hi = min(y0 + nrows, row_lo + rows_per) - 1;
  double* fb = f + (int64_t)(row_lo - y0) * W;
  int64_t* rb = raw + (int64_t)(row_lo - y0) * W;
  ordered_ingest<NT>(
      ev, hdr->n, Htot, W, row_lo, row_hi, c_pos, c_neg, u_min, u_max, sm,
      blockIdx.x == 0 ? err : nullptr, [&](int lp) { return fb[lp]; },
      [&](int lp, double v, int64_t t) {
        fb[lp] = v;
        rb[lp] = t;
      });
}

// ------------------------------------------------------------- surface --
// normalize_timestamps (surface.py:130-143) fused with the TV-L1 cold start
// (surface.py:161-165: u = u_bar = t, px = py = 0).
template <class T>
__global__ void k_normalize_tvinit(const int64_t* __restrict__ raw,
                                   const PacketHdr* __restrict__ hdr, double t_scale,
                                   T* t, T* tu, T* tub, T* tpx, T* tpy, int64_t N) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  const T v = (T)normalize_at((double)raw[k], (double)hdr->now, t_scale, hdr->window);
  t[k] = v;
  tu[k] = v;
  tub[k] = v;
  tpx[k] = T(0);
  tpy[k] = T(0);
}

// TV-L1 dual half-step (surface.py:168-183)
template <class T>
__global__ void k_tv_dual(const T* __restrict__ ub, T* __restrict__ px, T* __restrict__ py, Geo g,
                          T sigma) {
  EVR_GEO_INDEX
  const T dx = j < W - 1 ? ub[k + 1] - ub[k] : T(0);
  const T dy = gi < g.Htot - 1 ? ub[k + W] - ub[k] : T(0);
  T a = px[k], b = py[k];
  tv_dual_step(dx, dy, sigma, a, b);
  px[k] = a;
  py[k] = b;
}

// TV-L1 primal half-step (surface.py:185-193)
template <class T>
__global__ void k_tv_primal(const T* __restrict__ px, const T* __restrict__ py, T* u, T* ub,
                            const T* __restrict__ f0, Geo g, T tau, T shrink) {
  EVR_GEO_INDEX
  const T d = div_at(px[k], j > 0 ? px[k - 1] : T(0), py[k], gi > 0 ? py[k - W] : T(0), gi, j,
                     g.Htot, W);
  T ubar;
  const T un = tv_primal_step(d, u[k], f0[k], tau, shrink, ubar);
  u[k] = un;
  ub[k] = ubar;
}

// np.clip(u, 0, t_scale) after the TV-L1 loop (surface.py:195)
template <class T>
__global__ void k_tv_finish(const T* __restrict__ u, T* __restrict__ t, T t_scale, int64_t N) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  t[k] = vclip(u[k], T(0), t_scale);
}

// compute_metric (surface.py:199-205) + MetricField.coeffs (surface.py:81-90)
// + the solver constants beta = (tau*lam)*sqrtG, fb = (4*beta)*f
// (solve.py:227-228).  `flat` gives flat_metric (surface.py:208-211).
template <class T>
__global__ void k_metric_setup(const T* __restrict__ t, const double* __restrict__ f, T* tx,
                               T* ty, T* G, T* sg, CoefPlanes<T> c, T* beta, T* fb, Geo g,
                               T tl, int flat) {
  EVR_GEO_INDEX
  T gx = T(0), gy = T(0);
  if (!flat) {
    gx = j < W - 1 ? t[k + 1] - t[k] : T(0);
    gy = gi < g.Htot - 1 ? t[k + W] - t[k] : T(0);
  }
  const T det = metric_G(gx, gy);
  const T s = Arith<T>::sqrt(det);
  const Coef<T> a = coeffs_of(gx, gy, det);
  tx[k] = gx;
  ty[k] = gy;
  G[k] = det;
  sg[k] = s;
  c.a11[k] = a.a11;
  c.a12[k] = a.a12;
  c.a22[k] = a.a22;
  c.a31[k] = a.a31;
  c.a32[k] = a.a32;
  const T b = tl * s;
  beta[k] = b;
  fb[k] = T(4) * b * (T)f[k];
}

// Solver set-up from a caller-supplied MetricField (operator API):
// coefficients from (tx, ty, G) and beta/fb from sqrtG as given.
template <class T>
__global__ void k_solver_setup(const T* __restrict__ tx, const T* __restrict__ ty,
                               const T* __restrict__ G, const T* __restrict__ sg,
                               const double* __restrict__ f, CoefPlanes<T> c, T* beta, T* fb,
                               int64_t N, T tl, int rof) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  const Coef<T> a = coeffs_of(tx[k], ty[k], G[k]);
  c.a11[k] = a.a11;
  c.a12[k] = a.a12;
  c.a22[k] = a.a22;
  c.a31[k] = a.a31;
  c.a32[k] = a.a32;
  const T b = tl * sg[k];
  if (rof) {  // solve.py:278-280: w, wf = w*f, inv = 1/(1+w)
    beta[k] = T(1) / (T(1) + b);
    fb[k] = b * (T)f[k];
  } else {
    beta[k] = b;
    fb[k] = T(4) * b * (T)f[k];
  }
}

// ------------------------------------------------------------ solver --
// q = A^T p at pixel k
template <class T>
__device__ __forceinline__ void q_at(const CoefPlanes<T>& c, const T* p1, const T* p2,
                                     const T* p3, int64_t k, T& qx, T& qy) {
  q_of(c.at(k), p1[k], p2[k], p3[k], qx, qy);
}

// descent point div(A^T p) at global (gi, j) (solve.py:144-167, without
// *tau + u); the row above is local k - W
template <class T>
__device__ __forceinline__ T div_q(const CoefPlanes<T>& c, const T* p1, const T* p2,
                                   const T* p3, int gi, int j, int Htot, int W, int64_t k) {
  T qx, qy, qxl = T(0), qyu = T(0), dummy;
  q_at(c, p1, p2, p3, k, qx, qy);
  if (j > 0) q_at(c, p1, p2, p3, k - 1, qxl, dummy);
  if (gi > 0) q_at(c, p1, p2, p3, k - W, dummy, qyu);
  return div_at(qx, qxl, qy, qyu, gi, j, Htot, W);
}

// KL primal half-step + over-relaxation (solve.py:234-252)
template <class T>
__global__ void k_pd_primal(const T* __restrict__ p1, const T* __restrict__ p2,
                            const T* __restrict__ p3, CoefPlanes<T> c,
                            const T* __restrict__ u, const T* __restrict__ beta,
                            const T* __restrict__ fb, T* __restrict__ un, T* __restrict__ v,
                            Geo g, T tau, T umin, T umax) {
  EVR_GEO_INDEX
  const T d = div_q(c, p1, p2, p3, gi, j, g.Htot, W, k);
  const T uk = u[k];
  const T nu = kl_primal(d, uk, beta[k], fb[k], tau, umin, umax);
  un[k] = nu;
  v[k] = Arith<T>::mad(nu, T(2), -uk);
}

// ROF primal half-step + over-relaxation (solve.py:283-291); beta holds
// inv = 1/(1+w) and fb holds wf = w*f for this variant.
template <class T>
__global__ void k_rof_primal(const T* __restrict__ p1, const T* __restrict__ p2,
                             const T* __restrict__ p3, CoefPlanes<T> c,
                             const T* __restrict__ u, const T* __restrict__ inv,
                             const T* __restrict__ wf, T* __restrict__ un, T* __restrict__ v,
                             Geo g, T tau) {
  EVR_GEO_INDEX
  const T d = div_q(c, p1, p2, p3, gi, j, g.Htot, W, k);
  const T uk = u[k];
  const T nu = rof_primal(d, uk, wf[k], inv[k], tau);
  un[k] = nu;
  v[k] = Arith<T>::mad(nu, T(2), -uk);
}

// ---- variants the reference does not ship (parity unpinned; the CPU
// oracle oracle/evr_oracle.c evo_l1_solve / evo_tgv_solve restates them in
// this operation order): the L1 data term and second-order manifold TGV.

// data-term prox of the descent point t1 with beta = (tau*lam)*sqrtG:
// kind 0 = KL (box), 1 = ROF, 2 = L1 (soft shrink toward f)
template <class T>
__device__ __forceinline__ T data_prox(int kind, T t1, T f, T beta, T umin, T umax) {
  if (kind == 0) {
    const T s = t1 - beta;
    return vclip((s + Arith<T>::sqrt(Arith<T>::mad(s, s, (T(4) * beta) * f))) * T(0.5), umin,
                 umax);
  }
  if (kind == 1) return Arith<T>::mad(beta, f, t1) * Arith<T>::div(T(1), T(1) + beta);
  const T g = vclip(t1 - f, -beta, beta);
  return t1 - g;
}

// manifold TV + L1 data term: rof_manifold_solve's primal with the L1 prox
template <class T>
__global__ void k_l1_primal(const T* __restrict__ p1, const T* __restrict__ p2,
                            const T* __restrict__ p3, CoefPlanes<T> c,
                            const T* __restrict__ u, const T* __restrict__ sg,
                            const double* __restrict__ f, T* __restrict__ un, T* __restrict__ v,
                            Geo g, T tau, T tl) {
  EVR_GEO_INDEX
  const T d = div_q(c, p1, p2, p3, gi, j, g.Htot, W, k);
  const T uk = u[k];
  const T nu = data_prox(2, Arith<T>::mad(d, tau, uk), (T)f[k], tl * sg[k], T(0), T(0));
  un[k] = nu;
  v[k] = Arith<T>::mad(nu, T(2), -uk);
}

// One TGV iteration in one launch.  Primal half-step: u+ = prox_D(div(A^T p)
// tau + u), w+ = w + (A^T p + div_sym Q) tau, over-relaxed u_bar = v and
// w_bar = b, on the pixel and, recomputed bit-identically, on its right and
// lower neighbours (the values the dual reads there).  Dual half-step on the
// pixel: p = proj_{alpha1 sqrtG}(p + sigma A (grad u_bar - w_bar)), Q =
// proj_{alpha0}(Q + sigma E w_bar), |Q|^2 = q11^2 + q22^2 + 2 q12^2.  Every field is ping-ponged (set in
// -> set out), so the neighbours' reads of set `in` never race this launch's
// writes; the intermediate planes v, w_bar of the split form disappear.
template <class T> struct TgvSet {
  T *u, *w1, *w2, *p1, *p2, *p3, *q11, *q22, *q12;
};
// Block (32, 8): the primal runs once per pixel of the block's 32 x 8 tile
// plus its right column and lower row (33 x 9, the halo recomputed), into
// shared memory; the dual then reads its right / lower neighbours there.
template <class T>
__global__ void __launch_bounds__(256) k_tgv_iter(const TgvSet<T> in, TgvSet<T> out,
                                                  CoefPlanes<T> c, const T* __restrict__ sg,
                                                  const double* __restrict__ f, Geo g, T tau,
                                                  T sigma, T tl, int kind, T umin, T umax,
                                                  T alpha0, T alpha1) {
  __shared__ T sv[9][33], sb1[9][33], sb2[9][33];
  const int W = g.W, H = g.Htot;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int j0 = blockIdx.x * 32, i0 = g.ilo + (int)blockIdx.y * 8;
  // primal at local row ii, column jj (inside the sensor)
  auto primal = [&](int ii, int jj, T& nu, T& vv, T& n1, T& n2, T& b1, T& b2) {
    const int64_t kk = (int64_t)ii * W + jj;
    const int gii = g.row0 + ii;
    T qx, qy, qxl = T(0), qyu = T(0), dummy;
    q_at(c, in.p1, in.p2, in.p3, kk, qx, qy);
    if (jj > 0) q_at(c, in.p1, in.p2, in.p3, kk - 1, qxl, dummy);
    if (gii > 0) q_at(c, in.p1, in.p2, in.p3, kk - W, dummy, qyu);
    const T d = div_at(qx, qxl, qy, qyu, gii, jj, H, W);
    const T uk = in.u[kk];
    nu = data_prox(kind, Arith<T>::mad(d, tau, uk), (T)f[kk], tl * sg[kk], umin, umax);
    vv = Arith<T>::mad(nu, T(2), -uk);
    const T e1 = div_at(in.q11[kk], jj > 0 ? in.q11[kk - 1] : T(0), in.q12[kk],
                        gii > 0 ? in.q12[kk - W] : T(0), gii, jj, H, W);
    const T e2 = div_at(in.q12[kk], jj > 0 ? in.q12[kk - 1] : T(0), in.q22[kk],
                        gii > 0 ? in.q22[kk - W] : T(0), gii, jj, H, W);
    const T w1 = in.w1[kk], w2 = in.w2[kk];
    n1 = Arith<T>::mad(qx + e1, tau, w1);
    n2 = Arith<T>::mad(qy + e2, tau, w2);
    b1 = Arith<T>::mad(n1, T(2), -w1);
    b2 = Arith<T>::mad(n2, T(2), -w2);
  };
  const int i = i0 + ty, j = j0 + tx;
  const bool own = i <= g.ihi && j < W;
  T nu = T(0), n1 = T(0), n2 = T(0), t0, t1, t2;
  if (own) primal(i, j, nu, sv[ty][tx], n1, n2, sb1[ty][tx], sb2[ty][tx]);
  if (tx < 8) {  // the column right of the tile
    const int ii = i0 + tx, jj = j0 + 32;
    if (ty == 0 && ii <= g.ihi && jj < W && g.row0 + ii < H)
      primal(ii, jj, t0, sv[tx][32], t1, t2, sb1[tx][32], sb2[tx][32]);
  }
  if (ty == 7) {  // the row below the tile (the corner is never read)
    const int ii = i0 + 8;
    if (ii <= g.ihi && g.row0 + ii < H && j < W)
      primal(ii, j, t0, sv[8][tx], t1, t2, sb1[8][tx], sb2[8][tx]);
  }
  __syncthreads();
  if (!own) return;
  const int64_t k = (int64_t)i * W + j;
  const int gi = g.row0 + i;
  const bool xr = j < W - 1, yd = gi < H - 1;
  out.u[k] = nu;
  out.w1[k] = n1;
  out.w2[k] = n2;
  const T v = sv[ty][tx], b1 = sb1[ty][tx], b2 = sb2[ty][tx];
  const T vr = xr ? sv[ty][tx + 1] : T(0), b1r = xr ? sb1[ty][tx + 1] : T(0);
  const T b2r = xr ? sb2[ty][tx + 1] : T(0);
  const T vd = yd ? sv[ty + 1][tx] : T(0), b1d = yd ? sb1[ty + 1][tx] : T(0);
  const T b2d = yd ? sb2[ty + 1][tx] : T(0);
  // dual
  const T gx = (xr ? vr - v : T(0)) - b1;
  const T gy = (yd ? vd - v : T(0)) - b2;
  const Coef<T> a = c.at(k);
  const T s11 = sigma * a.a11, s12 = sigma * a.a12, s22 = sigma * a.a22;
  const T s31 = sigma * a.a31, s32 = sigma * a.a32;
  const T q1 = Arith<T>::mad(s12, gy, Arith<T>::mad(s11, gx, in.p1[k]));
  const T q2 = Arith<T>::mad(s22, gy, Arith<T>::mad(s12, gx, in.p2[k]));
  const T q3 = Arith<T>::mad(s32, gy, Arith<T>::mad(s31, gx, in.p3[k]));
  T n = Arith<T>::sqrt(Arith<T>::mad(q3, q3, Arith<T>::mad(q2, q2, q1 * q1)));
  n = vmax(Arith<T>::div(n, alpha1 * sg[k]), T(1));
  out.p1[k] = Arith<T>::div(q1, n);
  out.p2[k] = Arith<T>::div(q2, n);
  out.p3[k] = Arith<T>::div(q3, n);
  const T e11 = xr ? b1r - b1 : T(0);
  const T e22 = yd ? b2d - b2 : T(0);
  const T e12 = ((yd ? b1d - b1 : T(0)) + (xr ? b2r - b2 : T(0))) * T(0.5);
  const T qa = Arith<T>::mad(sigma, e11, in.q11[k]);
  const T qb = Arith<T>::mad(sigma, e22, in.q22[k]);
  const T qd = Arith<T>::mad(sigma, e12, in.q12[k]);
  T mq = Arith<T>::sqrt(Arith<T>::mad(qd * qd, T(2), Arith<T>::mad(qb, qb, qa * qa)));
  mq = vmax(Arith<T>::div(mq, alpha0), T(1));
  out.q11[k] = Arith<T>::div(qa, mq);
  out.q22[k] = Arith<T>::div(qb, mq);
  out.q12[k] = Arith<T>::div(qd, mq);
}

// dual ascent + ball projection (solve.py:170-201)
template <class T>
__global__ void k_pd_dual(const T* __restrict__ v, T* __restrict__ p1, T* __restrict__ p2,
                          T* __restrict__ p3, CoefPlanes<T> c, const T* __restrict__ sg, Geo g,
                          T sigma) {
  EVR_GEO_INDEX
  const T gx = j < W - 1 ? v[k + 1] - v[k] : T(0);
  const T gy = gi < g.Htot - 1 ? v[k + W] - v[k] : T(0);
  T a = p1[k], b = p2[k], d = p3[k];
  dual_step(c.at(k), sigma, gx, gy, sg[k], a, b, d);
  p1[k] = a;
  p2[k] = b;
  p3[k] = d;
}

// ------------------------------------------------- fused iterations --
// One launch per iteration (streaming engine, whole-sensor contexts).  Each
// warp owns a strip of kStrip = 30 columns x RY rows; its 32 lanes cover the
// strip plus one column either side, and the warp marches down the rows
// keeping the previous row in registers.  Horizontal neighbours come from
// warp shuffles, vertical ones from the march, so the half-step a
// neighbouring strip also needs (the TV-L1 dual on the left column / row
// above; the KL primal on the right column / row
// below) is recomputed, bit-identically, instead of exchanged.  Fields are
// ping-ponged between iterations so neighbours read iteration k while
// iteration k+1 is written.  No shared memory, no block barrier.
constexpr int kStrip = 30;

// Programmatic dependent launch: the iteration kernels are launched with
// programmatic stream serialization, so the next iteration's CTAs are
// resident and waiting while this one drains; griddepcontrol.wait blocks
// until the previous grid has completed and its writes are visible (a
// no-op for a normal launch).
__device__ __forceinline__ void pdl_wait_and_release() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// The fused iterations keep their changing fields interleaved, one 16-byte
// (float) / 32-byte (double) quad per pixel, so a warp row is one vector
// load / store per field group instead of one access per plane:
//   TV-L1:        TvQ = {u, u_bar, px, py}        (ping-pong), f0 = the t plane
//   primal-dual:  PdQ = {p1, p2, p3, u}           (ping-pong)
//                 constants: float  {tx, ty, fb, 0} (matrix recomputed)
//                            double {a11, a12, a22, a31}, {a32, sqrtG, beta, fb}
// k_pack_solver / k_unpack_solver convert to and from the planes the rest of
// the engine (state I/O, operator API, host loop) uses.
template <class T> struct alignas(4 * sizeof(T)) Q4 {
  T x, y, z, w;
};
// read-only (non-coherent) loads of the packed quads: the iteration kernels
// read ping-pong set a and write set a ^ 1, so nothing they read is written
// while they run
__device__ __forceinline__ Q4<float> ldg(const Q4<float>* p) {
  const float4 v = __ldg(reinterpret_cast<const float4*>(p));
  return Q4<float>{v.x, v.y, v.z, v.w};
}
// (a 32-byte quad stays one plain 256-bit load)
__device__ __forceinline__ Q4<double> ldg(const Q4<double>* p) { return *p; }
__device__ __forceinline__ float ldg(const float* p) { return __ldg(p); }
__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }

// Row sources of a march kernel.  A context owns global sensor rows
// [y0, y1), global row gr living at local row gr - y0 + olo of `own` (E
// elements per pixel).  A whole-sensor context is y0 = 0, y1 = H, olo = 0.
// A band (evr_group) reads the one row on each side its recomputed halo
// half-steps need -- the last row of the band above (y0 - 1) and the first
// row of the band below (y1) -- in place from the neighbours' buffers: peer
// memory over NVLink when the bands sit on different GPUs, so the halo
// exchange is part of the iteration kernel itself.
// Bounds-checked builds (-DEVR_CHECKS=1, tools/build_variants.sh): device
// asserts on the indices every iteration kernel reads through MarchRows and
// on the resident engine's exchange slots; a failing check traps the
// context (the stand-in for compute-sanitizer, closed on this GPU pool)
#ifndef EVR_CHECKS
#define EVR_CHECKS 0
#endif
#define EVR_ASSERT(c)                                                                  \
  do {                                                                                 \
    if (EVR_CHECKS && !(c)) {                                                          \
      printf("EVR_CHECKS failed: %s (%s:%d) block %d thread %d\n", #c, __FILE__,        \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                             \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)

template <class Q> struct MarchRows {
  const Q* own;
  const Q* up;  // row y0 - 1 of the band above (BANDED only; the tile kernels
                // also read rows y0 - K .. y0 - 2 at negative row offsets)
  const Q* dn;  // row y1 of the band below (BANDED only; tiles: .. y1 + K - 1)
  int y0, y1, olo, E;
  // element of global row gr (a band's own rows or K rows either side)
  // own row gr (32-bit offsets; the caller knows gr is in [y0, y1))
  __device__ __forceinline__ Q at_own(int gr, int jc, int W) const {
    EVR_ASSERT(gr >= y0 && gr < y1 && jc >= 0 && jc < W);
    return ldg(own + ((gr - y0 + olo) * W + jc));
  }
  template <bool BANDED> __device__ __forceinline__ Q at(int gr, int jc, int W) const {
    EVR_ASSERT(jc >= 0 && jc < W);
    if constexpr (BANDED) {
      // up to 4 rows (the largest tile K) either side, from a neighbour that exists
      EVR_ASSERT(gr >= y0 - 4 && gr < y1 + 4 && (gr >= y0 || up) && (gr < y1 || dn));
      return ldg(gr < y0   ? up + ((int64_t)(gr - y0 + 1) * W + jc)
                 : gr >= y1 ? dn + ((int64_t)(gr - y1) * W + jc)
                            : own + ((int64_t)(gr - y0 + olo) * W + jc));
    } else {
      EVR_ASSERT(gr >= y0 && gr < y1);
      return ldg(own + (gr * W + jc));
    }
  }
};

struct Strip {
  int j, i0, lane;
  bool inb, own, live;
};
// warp strips over the context's own rows [y0, y1)
template <int RY>
__device__ __forceinline__ Strip strip_of(int y0, int y1, int W) {
  Strip s;
  s.lane = threadIdx.x & 31;
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nsx = (W + kStrip - 1) / kStrip;
  const int sx = w % nsx, sy = w / nsx;
  s.i0 = y0 + sy * RY;
  s.live = s.i0 < y1;
  s.j = sx * kStrip - 1 + s.lane;
  s.inb = s.j >= 0 && s.j < W;
  s.own = s.lane >= 1 && s.lane <= kStrip && s.j < W;
  return s;
}

// TV-L1 iteration (surface.py:167-193): dual ascent + projection on rows
// i0-1 .. i0+RY-1, primal + L1 shrink + over-relaxation on the owned rows.
// Loads go to the clamped pixel so they are unconditional and are issued D
// rows ahead of the arithmetic (software pipeline over the unrolled march);
// out-of-sensor lanes / rows compute values nobody reads and store nothing.
// H is the sensor height (boundary rules by global row); f0 and out are
// indexed like in.own.
template <class T, int RY, int D, bool BANDED>
__global__ void __launch_bounds__(128)
k_tv_march(const Q4<T>* __restrict__ own, const MarchRows<Q4<T>> in, const T* __restrict__ f0,
           Q4<T>* __restrict__ out, int H, int W, T sigma, T tau, T shrink) {
  const int y1 = BANDED ? in.y1 : H;  // end of the own rows (global)
  const Strip s = strip_of<RY>(BANDED ? in.y0 : 0, y1, W);
  pdl_wait_and_release();
  if (!s.live) return;  // whole warp
  const int j = s.j;
  const int jc = min(max(j, 0), W - 1);
  const int rlo = BANDED ? max(in.y0 - 1, 0) : 0, rhi = BANDED ? min(y1, H - 1) : H - 1;
  auto grow = [&](int rr) { return min(max(s.i0 - 1 + rr, rlo), rhi); };
  // offset of global row gr in the context's own buffers (32-bit for a
  // whole sensor, the hot case)
  auto local = [&](int gr) {
    if constexpr (BANDED) return (int64_t)(gr - in.y0 + in.olo) * W;
    else return gr * W;
  };
  constexpr int NR = RY + 2;  // rows i0-1 .. i0+RY (the last one: u_bar only)
  Q4<T> q[NR];
  T f[NR];
  auto load = [&](int rr) {
    const int gr = grow(rr);
    if constexpr (BANDED) {
      q[rr] = gr < in.y0 ? in.up[jc] : gr >= y1 ? in.dn[jc] : own[local(gr) + jc];
      if (rr >= 1 && rr < NR - 1) f[rr] = f0[local(min(gr, y1 - 1)) + jc];
    } else {
      const int kc = gr * W + jc;
      q[rr] = own[kc];
      if (rr >= 1 && rr < NR - 1) f[rr] = f0[kc];
    }
  };
#pragma unroll
  for (int rr = 0; rr < D && rr < NR; ++rr) load(rr);
  T pyn_up = T(0);
#pragma unroll
  for (int rr = 0; rr < NR - 1; ++rr) {
    if (rr + D < NR) load(rr + D);
    const int r = s.i0 - 1 + rr;
    const T ub_c = q[rr].y, ub_n = q[rr + 1].y;
    T pxn = q[rr].z, pyn = q[rr].w;
    const T ub_r = __shfl_down_sync(0xffffffffu, ub_c, 1);
    const T dx = j < W - 1 ? ub_r - ub_c : T(0);
    const T dy = r < H - 1 ? ub_n - ub_c : T(0);
    tv_dual_step(dx, dy, sigma, pxn, pyn);
    const T pxl = __shfl_up_sync(0xffffffffu, pxn, 1);
    if (rr >= 1 && r < y1 && s.own) {
      const T d = div_at(pxn, j > 0 ? pxl : T(0), pyn, r > 0 ? pyn_up : T(0), r, j, H, W);
      T ubar;
      const T un = tv_primal_step(d, q[rr].x, f[rr], tau, shrink, ubar);
      out[local(r) + j] = Q4<T>{un, ubar, pxn, pyn};
    }
    pyn_up = pyn;
  }
}

// metric inputs of the primal-dual iteration, from the packed constants
struct MetricPackF32 {
  static constexpr bool kTma = false;
  const Q4<float>* __restrict__ c;  // {tx, ty, fb, 0}, the context's own rows
  MarchRows<Q4<float>> rows;        // a band's neighbour rows
  float tl;                         // tau * lam (solve.py:227)
  using Raw = Q4<float>;
  template <bool BANDED>
  __device__ __forceinline__ Raw load(int gr, int y1, int jc, int W) const {
    if constexpr (BANDED)
      return ldg(gr < rows.y0 ? rows.up + ((int64_t)(gr - rows.y0 + 1) * W + jc)
                 : gr >= y1   ? rows.dn + ((int64_t)(gr - y1) * W + jc)
                              : c + ((int64_t)(gr - rows.y0 + rows.olo) * W + jc));
    else
      return ldg(c + (gr * W + jc));
  }
  __device__ __forceinline__ Raw load_own(int gr, int y0, int olo, int jc, int W) const {
    return ldg(c + ((gr - y0 + olo) * W + jc));
  }
  __device__ __forceinline__ void finish(const Raw& r, Coef<float>& cf, float& sg, float& beta,
                                         float& fb) const {
    const MetricPx m = metric_px(r.x, r.y);  // bit-identical to k_metric_setup's planes
    cf = m.c;
    sg = m.sg;
    beta = tl * m.sg;
    fb = r.z;
  }
};
struct MetricPackF64 {
  static constexpr bool kTma = false;
  const Q4<double>* __restrict__ c;  // {a11, a12, a22, a31}, {a32, sqrtG, beta, fb}
  MarchRows<Q4<double>> rows;        // a band's neighbour rows (E = 2)
  struct Raw {
    Q4<double> a, b;
  };
  template <bool BANDED>
  __device__ __forceinline__ Raw load(int gr, int y1, int jc, int W) const {
    if constexpr (BANDED) {
      const Q4<double>* p = gr < rows.y0 ? rows.up + 2 * ((int64_t)(gr - rows.y0 + 1) * W + jc)
                            : gr >= y1   ? rows.dn + 2 * ((int64_t)(gr - y1) * W + jc)
                                         : c + 2 * ((int64_t)(gr - rows.y0 + rows.olo) * W + jc);
      return Raw{ldg(p), ldg(p + 1)};
    } else {
      const int k = gr * W + jc;
      return Raw{ldg(c + 2 * k), ldg(c + 2 * k + 1)};
    }
  }
  __device__ __forceinline__ Raw load_own(int gr, int y0, int olo, int jc, int W) const {
    const int k = (gr - y0 + olo) * W + jc;
    return Raw{ldg(c + 2 * k), ldg(c + 2 * k + 1)};
  }
  __device__ __forceinline__ void finish(const Raw& r, Coef<double>& cf, double& sg,
                                         double& beta, double& fb) const {
    cf = Coef<double>{r.a.x, r.a.y, r.a.z, r.a.w, r.b.x};
    sg = r.b.y;
    beta = r.b.z;
    fb = r.b.w;
  }
};
// MetricPackF64 plus TMA descriptors of the packed constants (tc: 8 doubles
// per pixel) and of the launch's input state (ts: 4 doubles per pixel), whole
// sensor; a tile kernel taking it loads its region with two 2-D tensor copies
// into shared memory (k_pd_tile's TMA form)
struct MetricPackF64Tma : MetricPackF64 {
  static constexpr bool kTma = true;
  CUtensorMap tc, ts;
};
template <class T> struct MetricPack;
template <> struct MetricPack<float> { using type = MetricPackF32; };
template <> struct MetricPack<double> { using type = MetricPackF64; };

// primal-dual iteration (solve.py:233-252): q = A^T p on rows i0-1 .. i0+RY,
// KL prox + over-relaxation on rows i0 .. i0+RY, dual ascent + ball
// projection on the owned rows one row behind the primal, then the row's
// {p, u} quad is stored; loads pipelined D rows ahead as in k_tv_march.
template <class T, int RY, int D, class M, bool BANDED>
__global__ void __launch_bounds__(128)
k_pd_march(const Q4<T>* __restrict__ own, const MarchRows<Q4<T>> in, M m,
           Q4<T>* __restrict__ out, int H, int W, T tau, T sigma, T umin, T umax,
           const int* __restrict__ stop = nullptr) {
  const int y1 = BANDED ? in.y1 : H;  // end of the own rows (global)
  const Strip s = strip_of<RY>(BANDED ? in.y0 : 0, y1, W);
  pdl_wait_and_release();
  if (stop && *stop) return;  // convergence_tol reached (k_relchange): the iteration is skipped
  if (!s.live) return;  // whole warp
  const int j = s.j;
  const int jc = min(max(j, 0), W - 1);
  const int rlo = BANDED ? max(in.y0 - 1, 0) : 0, rhi = BANDED ? min(y1, H - 1) : H - 1;
  auto grow = [&](int rr) { return min(max(s.i0 - 1 + rr, rlo), rhi); };
  auto local = [&](int gr) {
    if constexpr (BANDED) return (int64_t)(gr - in.y0 + in.olo) * W;
    else return gr * W;
  };
  constexpr int NR = RY + 2;  // rows i0-1 .. i0+RY
  Q4<T> q[NR];
  typename M::Raw c[NR];
  auto load = [&](int rr) {
    const int gr = grow(rr);
    if constexpr (BANDED) {
      q[rr] = gr < in.y0 ? in.up[jc] : gr >= y1 ? in.dn[jc] : own[local(gr) + jc];
    } else {
      q[rr] = own[gr * W + jc];
    }
    c[rr] = m.template load<BANDED>(gr, y1, jc, W);
  };
#pragma unroll
  for (int rr = 0; rr < D && rr < NR; ++rr) load(rr);
  T qy_up = T(0), v_up = T(0), sg_up = T(1), nu_up = T(0);
  Coef<T> cf_up{T(0), T(0), T(0), T(0), T(0)};
#pragma unroll
  for (int rr = 0; rr < NR; ++rr) {
    if (rr + D < NR) load(rr + D);
    const int r = s.i0 - 1 + rr;
    Coef<T> cf;
    T sg, beta, fb, qx, qy, v = T(0), nu = T(0);
    m.finish(c[rr], cf, sg, beta, fb);
    q_of(cf, q[rr].x, q[rr].y, q[rr].z, qx, qy);
    const T qxl = __shfl_up_sync(0xffffffffu, qx, 1);
    if (rr >= 1) {
      const T d = div_at(qx, j > 0 ? qxl : T(0), qy, r > 0 ? qy_up : T(0), r, j, H, W);
      const T uk = q[rr].w;
      nu = kl_primal(d, uk, beta, fb, tau, umin, umax);
      v = Arith<T>::mad(nu, T(2), -uk);
    }
    const T vr = __shfl_down_sync(0xffffffffu, v_up, 1);
    if (rr >= 2 && r - 1 < y1 && s.own) {
      T a = q[rr - 1].x, b = q[rr - 1].y, cc = q[rr - 1].z;
      const T gx = j < W - 1 ? vr - v_up : T(0);
      const T gy = r - 1 < H - 1 ? v - v_up : T(0);
      dual_step(cf_up, sigma, gx, gy, sg_up, a, b, cc);
      out[local(r - 1) + j] = Q4<T>{a, b, cc, nu_up};
    }
    qy_up = qy;
    v_up = v;
    nu_up = nu;
    cf_up = cf;
    sg_up = sg;
  }
}

// normalize_timestamps (surface.py:130-143) + the TV-L1 cold start
// (surface.py:161-165) into the packed state
template <class T>
__global__ void k_normalize_pack(const int64_t* __restrict__ raw,
                                 const PacketHdr* __restrict__ hdr, double t_scale,
                                 T* __restrict__ t, Q4<T>* __restrict__ q, int64_t N) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  const T v = (T)normalize_at((double)raw[k], (double)hdr->now, t_scale, hdr->window);
  t[k] = v;
  q[k] = Q4<T>{v, v, T(0), T(0)};
}

// np.clip(u, 0, t_scale) from the packed TV-L1 state (surface.py:195)
template <class T>
__global__ void k_tv_finish_packed(const Q4<T>* __restrict__ q, T* __restrict__ t, T t_scale,
                                   int64_t N) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  t[k] = vclip(q[k].x, T(0), t_scale);
}

// Whole-sensor fused list, one launch instead of three: the end of TV-L1
// (np.clip(u, 0, t_scale), surface.py:195) on the packed TV state, the
// metric (compute_metric + coeffs, surface.py:81-90, :199-205, exactly
// k_metric_setup's operations: a pixel's slopes read its right / lower
// neighbours' clipped u) and the packing of the solver state and
// constants.  Writes the t, tx, ty, G, sqrtG planes (state views); the
// coefficient planes stay unwritten -- only the packed constants feed the
// tiles.  flat: the metric of a disabled manifold (tx = ty = 0).
template <class T>
__global__ void k_metric_pack(const Q4<T>* __restrict__ tvq, const double* __restrict__ f,
                              const T* __restrict__ p1, const T* __restrict__ p2,
                              const T* __restrict__ p3, const T* __restrict__ u,
                              T* __restrict__ t, T* __restrict__ tx, T* __restrict__ ty,
                              T* __restrict__ G, T* __restrict__ sgp, Q4<T>* __restrict__ st,
                              Q4<T>* __restrict__ cst, int H, int W, T t_scale, T tl, int flat) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= H || j >= W) return;
  const int64_t k = (int64_t)i * W + j;
  T gx = T(0), gy = T(0);
  if (!flat) {
    const T tk = vclip(tvq[k].x, T(0), t_scale);
    t[k] = tk;
    gx = j < W - 1 ? vclip(tvq[k + 1].x, T(0), t_scale) - tk : T(0);
    gy = i < H - 1 ? vclip(tvq[k + W].x, T(0), t_scale) - tk : T(0);
  }
  const T det = metric_G(gx, gy);
  const T s = Arith<T>::sqrt(det);
  tx[k] = gx;
  ty[k] = gy;
  G[k] = det;
  sgp[k] = s;
  const T b = tl * s;
  const T fb = T(4) * b * (T)f[k];
  st[k] = Q4<T>{p1[k], p2[k], p3[k], u[k]};
  if constexpr (sizeof(T) == 4) {
    cst[k] = Q4<T>{gx, gy, fb, T(0)};
  } else {
    const Coef<T> a = coeffs_of(gx, gy, det);
    cst[2 * k] = Q4<T>{a.a11, a.a12, a.a22, a.a31};
    cst[2 * k + 1] = Q4<T>{a.a32, s, b, fb};
  }
}

// planes -> packed solver state + constants (after k_metric_setup)
template <class T>
__global__ void k_pack_solver(const T* __restrict__ p1, const T* __restrict__ p2,
                              const T* __restrict__ p3, const T* __restrict__ u,
                              const T* __restrict__ tx, const T* __restrict__ ty,
                              CoefPlanes<T> c, const T* __restrict__ sg,
                              const T* __restrict__ beta, const T* __restrict__ fb,
                              Q4<T>* __restrict__ st, Q4<T>* __restrict__ cst, int64_t N,
                              const double* __restrict__ fslot = nullptr) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  st[k] = Q4<T>{p1[k], p2[k], p3[k], u[k]};
  if constexpr (sizeof(T) == 4) {
    cst[k] = Q4<T>{tx[k], ty[k], fb[k], T(0)};
  } else {
    // fslot: the L1 data term keeps f itself in the last slot
    cst[2 * k] = Q4<T>{c.a11[k], c.a12[k], c.a22[k], c.a31[k]};
    cst[2 * k + 1] = Q4<T>{c.a32[k], sg[k], beta[k], fslot ? (T)fslot[k] : fb[k]};
  }
}

// packed solver state -> p, u planes and f = u (pipeline.py:165)
template <class T>
__global__ void k_unpack_solver(const Q4<T>* __restrict__ st, T* __restrict__ p1,
                                T* __restrict__ p2, T* __restrict__ p3, T* __restrict__ u,
                                double* __restrict__ f, int64_t N,
                                const Q4<T>* __restrict__ st_odd = nullptr,
                                const evr_solve_info* __restrict__ info = nullptr) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  // early stop: the set holding the last executed iteration is decided on
  // the device (iterations n -> set n & 1)
  const Q4<T> q = (st_odd && (info->iterations & 1)) ? st_odd[k] : st[k];
  p1[k] = q.x;
  p2[k] = q.y;
  p3[k] = q.z;
  u[k] = q.w;
  f[k] = (double)q.w;
}

// --------------------------------------------------------- reductions --
// Deterministic two-pass reductions (fixed tree): pass 1 writes one partial
// per block, pass 2 (one block) folds the partials in index order.
template <int NT>
__device__ __forceinline__ double block_sum(double x, double* sh) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = x;
  __syncthreads();
  x = threadIdx.x < NT / 32 ? sh[threadIdx.x] : 0.0;
  if (wid == 0)
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
  return x;
}

// rel_change = |u+ - u| / max(|u|, 1e-30) (solve.py:246-249) in one launch:
// each CTA writes its partial sums of (un-u)^2 and u^2 in a fixed order, the
// last CTA to take the ticket folds the partials in index order and resets
// the ticket (deterministic: the same bits every run)
template <class T, int NT>
__global__ void __launch_bounds__(NT)
k_relchange(const T* __restrict__ un, const T* __restrict__ u, int64_t N, double* part,
            int stride, unsigned* ticket, evr_solve_info* info, int iterations, double* sums,
            double tol = 0.0, int* stop = nullptr, double* hist = nullptr) {
  __shared__ double sh[NT / 32];
  __shared__ bool last;
  pdl_wait_and_release();
  // early stop (solve.py:257-258): once an iteration's rel_change fell below
  // tol, the remaining iterations and their rel_change launches are no-ops
  // (every CTA reads the flag before the last CTA of the stopping launch
  // can write it)
  if (stop && *stop) return;
  double d = 0.0, o = 0.0;
  for (int64_t k = (int64_t)blockIdx.x * NT + threadIdx.x; k < N; k += (int64_t)gridDim.x * NT) {
    const double a = (double)un[k * stride], b = (double)u[k * stride];
    d += (a - b) * (a - b);
    o += b * b;
  }
  d = block_sum<NT>(d, sh);
  o = block_sum<NT>(o, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = d;
    part[2 * blockIdx.x + 1] = o;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int nb = (int)gridDim.x;
  d = 0.0;
  o = 0.0;
  for (int b = threadIdx.x; b < nb; b += NT) {
    d += __ldcg(part + 2 * b);
    o += __ldcg(part + 2 * b + 1);
  }
  d = block_sum<NT>(d, sh);
  o = block_sum<NT>(o, sh);
  if (threadIdx.x == 0) {
    const double den = sqrt(o);
    const double rel = sqrt(d) / (den > 1e-30 ? den : 1e-30);
    info->rel_change = rel;
    info->iterations = iterations;
    if (hist) hist[iterations - 1] = rel;  // per-iteration trace, read back once
    sums[0] = d;  // evr_group folds the bands' sums
    sums[1] = o;
    *ticket = 0u;
    if (stop && rel < tol) *stop = 1;
  }
}

// Whole-sensor fused list: the epilogue (state.u = u, state.p, state.f =
// copy(u), pipeline.py:167-170) from the packed set holding the last
// iteration, fused with rel_change of that iteration (solve.py:246-249:
// |u_M - u_{M-1}| / max(|u_{M-1}|, 1e-30)) against the u_{M-1} plane the
// final tile left (k_pd_tile's `prev`); per-CTA partials, the last CTA
// folds them in index order (as k_relchange).
template <class T, int NT>
__global__ void __launch_bounds__(NT)
k_unpack_rel(const Q4<T>* __restrict__ q, const T* __restrict__ uprev, T* __restrict__ p1,
             T* __restrict__ p2, T* __restrict__ p3, T* __restrict__ u,
             double* __restrict__ f, int64_t N, double* part, unsigned* ticket,
             evr_solve_info* info, int iterations) {
  __shared__ double sh[NT / 32];
  __shared__ bool last;
  pdl_wait_and_release();
  double d = 0.0, o = 0.0;
  for (int64_t k = (int64_t)blockIdx.x * NT + threadIdx.x; k < N; k += (int64_t)gridDim.x * NT) {
    const Q4<T> v = q[k];
    p1[k] = v.x;
    p2[k] = v.y;
    p3[k] = v.z;
    u[k] = v.w;
    f[k] = (double)v.w;
    const double a = (double)v.w, b = (double)uprev[k];
    d += (a - b) * (a - b);
    o += b * b;
  }
  d = block_sum<NT>(d, sh);
  o = block_sum<NT>(o, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = d;
    part[2 * blockIdx.x + 1] = o;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int nb = (int)gridDim.x;
  d = 0.0;
  o = 0.0;
  for (int b = threadIdx.x; b < nb; b += NT) {
    d += __ldcg(part + 2 * b);
    o += __ldcg(part + 2 * b + 1);
  }
  d = block_sum<NT>(d, sh);
  o = block_sum<NT>(o, sh);
  if (threadIdx.x == 0) {
    const double den = sqrt(o);
    info->rel_change = sqrt(d) / (den > 1e-30 ? den : 1e-30);
    info->iterations = iterations;
    *ticket = 0u;
  }
}

// energy (solve.py:111-118) partials: tv = sqrt(G * |S u|^2), data term
template <class T, int NT>
__global__ void __launch_bounds__(NT)
k_energy_partial(const T* __restrict__ u, const double* __restrict__ f, CoefPlanes<T> c,
                 const T* __restrict__ G, const T* __restrict__ sg, int H, int W,
                 double* __restrict__ part) {
  __shared__ double sh[NT / 32];
  double tv = 0.0, data = 0.0;
  const int64_t N = (int64_t)H * W;
  for (int64_t k = (int64_t)blockIdx.x * NT + threadIdx.x; k < N; k += (int64_t)gridDim.x * NT) {
    const int i = (int)(k / W), j = (int)(k - (int64_t)i * W);
    const T ux = j < W - 1 ? u[k + 1] - u[k] : T(0);
    const T uy = i < H - 1 ? u[k + W] - u[k] : T(0);
    const Coef<T> a = c.at(k);
    const T s0 = a.a11 * ux + a.a12 * uy;
    const T s1 = a.a12 * ux + a.a22 * uy;
    const T s2 = a.a31 * ux + a.a32 * uy;
    const T s = s0 * s0 + s1 * s1 + s2 * s2;
    tv += (double)sqrt(G[k] * s);
    const double uk = (double)u[k];
    data += (uk - f[k] * log(uk)) * (double)sg[k];
  }
  tv = block_sum<NT>(tv, sh);
  data = block_sum<NT>(data, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = tv;
    part[2 * blockIdx.x + 1] = data;
  }
}

template <int NT>
__global__ void __launch_bounds__(NT)
k_energy_final(const double* __restrict__ part, int nb, double lam, double* out) {
  __shared__ double sh[NT / 32];
  double tv = 0.0, data = 0.0;
  for (int b = threadIdx.x; b < nb; b += NT) {
    tv += part[2 * b];
    data += part[2 * b + 1];
  }
  tv = block_sum<NT>(tv, sh);
  data = block_sum<NT>(data, sh);
  if (threadIdx.x == 0) *out = tv + lam * data;
}

// ---------------------------------------------------------- epilogue --
// process_packet re-anchor (pipeline.py:167-170): u <- u+, f <- copy(u+)
template <class T>
__global__ void k_epilogue(const T* __restrict__ un, T* __restrict__ u, double* __restrict__ f,
                           int64_t N) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  const T v = un[k];
  if (un != u) u[k] = v;
  f[k] = (double)v;
}

// ------------------------------------------------------ conversions --
template <class S, class D>
__global__ void k_convert(const S* __restrict__ s, D* __restrict__ d, int64_t N) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < N) d[k] = (D)s[k];
}

template <class T>
__global__ void k_fill(T* __restrict__ d, T v, int64_t N) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < N) d[k] = v;
}

// (H, W, 3) interleaved double <-> three planes
template <class T>
__global__ void k_aos_to_planes(const double* __restrict__ aos, T* p1, T* p2, T* p3, int64_t N) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  p1[k] = (T)aos[3 * k];
  p2[k] = (T)aos[3 * k + 1];
  p3[k] = (T)aos[3 * k + 2];
}

template <class T>
__global__ void k_planes_to_aos(const T* __restrict__ p1, const T* __restrict__ p2,
                                const T* __restrict__ p3, double* aos, int64_t N) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  aos[3 * k] = (double)p1[k];
  aos[3 * k + 1] = (double)p2[k];
  aos[3 * k + 2] = (double)p3[k];
}

// to_gray (pgm.py:14-22): floor(255*(u-lo)/(hi-lo) + 0.5), clipped, uint8
template <class T>
__global__ void k_to_gray(const T* __restrict__ u, double lo, double hi, uint8_t* out, int64_t N) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  // scaled = 255.0 * (image - u_min) / (u_max - u_min), left to right
  const double s = 255.0 * ((double)u[k] - lo) / (hi - lo);
  out[k] = (uint8_t)vclip(floor(s + 0.5), 0.0, 255.0);
}

// ------------------------------------------------- operator kernels --
// grad_x / grad_y (surface.py:93-104)
__global__ void k_op_grad(const double* __restrict__ u, double* gx, double* gy, int H, int W) {
  EVR_2D_INDEX
  gx[k] = j < W - 1 ? u[k + 1] - u[k] : 0.0;
  gy[k] = i < H - 1 ? u[k + W] - u[k] : 0.0;
}

// div_xy (surface.py:107-121); negate for surface_gradient_adjoint
__global__ void k_op_div(const double* __restrict__ qx, const double* __restrict__ qy,
                         double* out, int H, int W, int negate) {
  EVR_2D_INDEX
  const double d = div_at(qx[k], j > 0 ? qx[k - 1] : 0.0, qy[k], i > 0 ? qy[k - W] : 0.0, i, j,
                          H, W);
  out[k] = negate ? -d : d;
}

// q = A^T p from interleaved p (surface.py:249-251)
__global__ void k_op_q(const double* __restrict__ p, CoefPlanes<double> c, double* qx,
                       double* qy, int64_t N) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  q_of(c.at(k), p[3 * k], p[3 * k + 1], p[3 * k + 2], qx[k], qy[k]);
}

// surface_gradient (surface.py:214-236) -> interleaved (H, W, 3)
__global__ void k_op_surface_gradient(const double* __restrict__ u, CoefPlanes<double> c,
                                      double* out, int H, int W) {
  EVR_2D_INDEX
  const double ux = j < W - 1 ? u[k + 1] - u[k] : 0.0;
  const double uy = i < H - 1 ? u[k + W] - u[k] : 0.0;
  const Coef<double> a = c.at(k);
  out[3 * k] = a.a11 * ux + a.a12 * uy;
  out[3 * k + 1] = a.a12 * ux + a.a22 * uy;
  out[3 * k + 2] = a.a31 * ux + a.a32 * uy;
}

// prox_data (solve.py:88-100)
__global__ void k_op_prox_data(const double* __restrict__ ub, const double* __restrict__ f,
                               const double* __restrict__ sg, double tl, double umin,
                               double umax, double* out, int64_t N) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  const double beta = tl * sg[k];
  const double s = ub[k] - beta;
  const double root = 0.5 * (s + sqrt(s * s + 4.0 * beta * f[k]));
  out[k] = vclip(root, umin, umax);
}

// prox_dual (solve.py:103-108)
__global__ void k_op_prox_dual(const double* __restrict__ p, const double* __restrict__ sg,
                               double* out, int64_t N) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  const double a = p[3 * k], b = p[3 * k + 1], c = p[3 * k + 2];
  const double nrm = sqrt(a * a + b * b + c * c);
  const double s = vmax(1.0, nrm / sg[k]);
  out[3 * k] = a / s;
  out[3 * k + 1] = b / s;
  out[3 * k + 2] = c / s;
}

// coefficient planes from caller-supplied (tx, ty, G)
__global__ void k_op_coeffs(const double* __restrict__ tx, const double* __restrict__ ty,
                            const double* __restrict__ G, CoefPlanes<double> c, int64_t N) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  const Coef<double> a = coeffs_of(tx[k], ty[k], G[k]);
  c.a11[k] = a.a11;
  c.a12[k] = a.a12;
  c.a22[k] = a.a22;
  c.a31[k] = a.a31;
  c.a32[k] = a.a32;
}

// compute_metric fields only (surface.py:199-205)
__global__ void k_op_metric(const double* __restrict__ t, double* tx, double* ty, double* G,
                            double* sg, int H, int W) {
  EVR_2D_INDEX
  const double gx = j < W - 1 ? t[k + 1] - t[k] : 0.0;
  const double gy = i < H - 1 ? t[k + W] - t[k] : 0.0;
  const double g = metric_G(gx, gy);
  tx[k] = gx;
  ty[k] = gy;
  G[k] = g;
  sg[k] = sqrt(g);
}

// normalize_timestamps on a float64 raw map (surface.py:141-142)
__global__ void k_op_normalize(const double* __restrict__ raw, double now, double t_scale,
                               double window, double* t, int64_t N) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  t[k] = normalize_at(raw[k], now, t_scale, window);
}

}  // namespace evr
