// evr_math.cuh -- per-pixel arithmetic of the hot path, shared by every
// engine (streaming kernels, resident persistent kernel, operator kernels).
//
// Each function is one pixel's worth of a reference stage, written in the
// reference's exact operation order.  The translation
// unit is compiled with -fmad=false and every binary64 a*b+c is spelled
// __dmul_rn + __dadd_rn, so with T = double every result is bit-identical to
// numpy float64: IEEE div.rn / sqrt.rn, no contraction.
// Scalars (tau, sigma, tau*lam, c+-, ...) come from the host already
// rounded exactly as the reference computes them; none is re-derived here.
#pragma once

#include <cstdint>
#include <type_traits>

// float32 instruction-count switches (each keeps the float engine inside
// its tolerance and every float kernel on the same arithmetic; float64 is
// untouched).  With EVR_F32_INTERIOR (evr_tile.cuh), measured on B200:
// C3 f32 0.615 -> 0.548 ms, C4 0.198 -> 0.185, C5 1.588 -> 1.443
// (profiles/r01f/experiments.md)
#ifndef EVR_F32_MINMAX
#define EVR_F32_MINMAX 1  // vmax / vmin as one FMNMX instead of FSETP + FSEL
#endif
#ifndef EVR_F32_SIGFOLD
#define EVR_F32_SIGFOLD 1  // dual: sigma * g once per axis, not sigma * a_ij
#endif

namespace evr {

// np.minimum / np.maximum / np.clip on non-NaN data
template <class T> __device__ __forceinline__ T vmax(T a, T b) {
  if constexpr (EVR_F32_MINMAX && std::is_same<T, float>::value) return fmaxf(a, b);
  else return b > a ? b : a;
}
template <class T> __device__ __forceinline__ T vmin(T a, T b) {
  if constexpr (EVR_F32_MINMAX && std::is_same<T, float>::value) return fminf(a, b);
  else return b < a ? b : a;
}
template <class T> __device__ __forceinline__ T vclip(T x, T lo, T hi) {
  return vmin(vmax(x, lo), hi);
}

// Division / square root of the iteration kernels.  binary64: IEEE div.rn /
// sqrt.rn (the bit-exact engine).  binary32: the hardware approximations
// (MUFU-based, ~2 ulp), which keep the float engine well inside its 1e-4
// log-intensity tolerance at a fraction of the instruction count.
template <class T> struct Arith;
//
// mad(a, b, c) is the reference's `a * b + c`: binary64 rounds the product
// and the sum separately (numpy never fuses), binary32 issues one FFMA --
// half the FP instructions of the iteration kernels, and more accurate.
template <> struct Arith<double> {
  static __device__ __forceinline__ double div(double a, double b) { return a / b; }
  static __device__ __forceinline__ double sqrt(double x) { return ::sqrt(x); }
  static __device__ __forceinline__ double mad(double a, double b, double c) {
    return __dadd_rn(__dmul_rn(a, b), c);
  }
};
// The .ftz forms are single MUFU ops (+ FMUL for the quotient); without
// .ftz ptxas wraps each in a subnormal range test and rescale.  The float
// engine's operands (u in [u_min, u_max], slopes, duals in the unit ball)
// are never subnormal where it matters.
template <> struct Arith<float> {
  static __device__ __forceinline__ float div(float a, float b) {
    float r;
    asm("div.approx.ftz.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
  }
  static __device__ __forceinline__ float mad(float a, float b, float c) {
    return __fmaf_rn(a, b, c);
  }
  static __device__ __forceinline__ float sqrt(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
  }
};

template <class T> struct Coef { T a11, a12, a22, a31, a32; };

// MetricField.coeffs (surface.py:81-90)
template <class T>
__device__ __forceinline__ Coef<T> coeffs_of(T tx, T ty, T G) {
  Coef<T> c;
  c.a11 = Arith<T>::div(Arith<T>::mad(ty, ty, T(1)), G);
  c.a12 = Arith<T>::div(-(tx * ty), G);
  c.a22 = Arith<T>::div(Arith<T>::mad(tx, tx, T(1)), G);
  c.a31 = Arith<T>::div(tx, G);
  c.a32 = Arith<T>::div(ty, G);
  return c;
}

// compute_metric (surface.py:202-205): G = 1 + tx*tx + ty*ty, left to right
template <class T> __device__ __forceinline__ T metric_G(T tx, T ty) {
  return Arith<T>::mad(ty, ty, Arith<T>::mad(tx, tx, T(1)));
}

// float32 metric matrix and sqrt(G) of one pixel from its surface slopes,
// recomputed on the fly: G once, one MUFU.RCP shared by the five quotients
// (__fdividef(a, G) == a * rcp(G)), bit-identical to k_metric_setup's planes
struct MetricPx {
  Coef<float> c;
  float sg;
};
__device__ __forceinline__ MetricPx metric_px(float tx, float ty) {
  const float G = metric_G(tx, ty);
  const float r = Arith<float>::div(1.0f, G);  // MUFU.RCP(G)
  MetricPx m;
  m.c.a11 = Arith<float>::mad(ty, ty, 1.0f) * r;
  m.c.a12 = -(tx * ty) * r;
  m.c.a22 = Arith<float>::mad(tx, tx, 1.0f) * r;
  m.c.a31 = tx * r;
  m.c.a32 = ty * r;
  m.sg = Arith<float>::sqrt(G);
  return m;
}

// div_xy (surface.py:107-121) at (i, j): x part (qx here / qx left), then the
// y part (qy here / qy above) added into it.  qx[:, W-1], qy[H-1, :] unused.
template <class T>
__device__ __forceinline__ T div_at(T qx_c, T qx_l, T qy_c, T qy_u, int i, int j,
                                    int H, int W) {
  if constexpr (sizeof(T) == 4) {
    // binary32 (callers pass qx_l = 0 on the first column, qy_u = 0 on the
    // first row): one select per axis; the last-column / last-row forms
    // 0 - qx_l, 0 - qy_u equal -qx_l, -qy_u up to the sign of a zero, which
    // never reaches u (t1 = d * tau + u)
    const T d = (j < W - 1 ? qx_c : T(0)) - qx_l;
    return d + ((i < H - 1 ? qy_c : T(0)) - qy_u);
  }
  T d;
  if (j == 0)
    d = qx_c;
  else if (j == W - 1)
    d = -qx_l;
  else
    d = qx_c - qx_l;
  if (i == 0)
    d = d + qy_c;
  else if (i == H - 1)
    d = d - qy_u;
  else
    d = d + (qy_c - qy_u);
  return d;
}

// _Loop.descent_point q = A^T p (solve.py:149-158)
template <class T>
__device__ __forceinline__ void q_of(const Coef<T>& c, T p1, T p2, T p3, T& qx, T& qy) {
  qx = Arith<T>::mad(c.a31, p3, Arith<T>::mad(c.a12, p2, c.a11 * p1));
  qy = Arith<T>::mad(c.a32, p3, Arith<T>::mad(c.a22, p2, c.a12 * p1));
}

// primal_dual_solve KL prox (solve.py:235-242): t1 = div*tau + u;
// s = t1 - beta; clip((s + sqrt(s*s + 4 beta f)) * 0.5)
template <class T>
__device__ __forceinline__ T kl_primal(T divq, T u, T beta, T fb, T tau, T umin, T umax) {
  const T t1 = Arith<T>::mad(divq, tau, u);
  const T s = t1 - beta;
  const T r = (s + Arith<T>::sqrt(Arith<T>::mad(s, s, fb))) * T(0.5);
  return vclip(r, umin, umax);
}

// rof_manifold_solve primal (solve.py:285-287): ((div*tau + u) + wf) * inv
template <class T>
__device__ __forceinline__ T rof_primal(T divq, T u, T wf, T inv, T tau) {
  return (Arith<T>::mad(divq, tau, u) + wf) * inv;
}

// _Loop.dual_ascent (solve.py:175-201) at one pixel; gx, gy are the forward
// differences of the over-relaxed point (0 on the last column / row).
template <class T>
__device__ __forceinline__ void dual_step(const Coef<T>& c, T sigma, T gx, T gy, T sqrtG,
                                          T& p1, T& p2, T& p3) {
  T q1, q2, q3;
  if constexpr (EVR_F32_SIGFOLD && sizeof(T) == 4) {
    // binary32: p + A (sigma g), 2 products instead of the 5 sigma * a_ij
    const T sx = sigma * gx, sy = sigma * gy;
    q1 = Arith<T>::mad(c.a12, sy, Arith<T>::mad(c.a11, sx, p1));
    q2 = Arith<T>::mad(c.a22, sy, Arith<T>::mad(c.a12, sx, p2));
    q3 = Arith<T>::mad(c.a32, sy, Arith<T>::mad(c.a31, sx, p3));
  } else {
    const T s11 = sigma * c.a11, s12 = sigma * c.a12, s22 = sigma * c.a22;
    const T s31 = sigma * c.a31, s32 = sigma * c.a32;
    q1 = Arith<T>::mad(s12, gy, Arith<T>::mad(s11, gx, p1));
    q2 = Arith<T>::mad(s22, gy, Arith<T>::mad(s12, gx, p2));
    q3 = Arith<T>::mad(s32, gy, Arith<T>::mad(s31, gx, p3));
  }
  T n = Arith<T>::sqrt(Arith<T>::mad(q3, q3, Arith<T>::mad(q2, q2, q1 * q1)));
  if constexpr (sizeof(T) == 4) {
    // binary32: a * rcp(b) unconditionally (no selects; rcp(1) == 1)
    n = vmax(Arith<T>::div(n, sqrtG), T(1));
    p1 = Arith<T>::div(q1, n);
    p2 = Arith<T>::div(q2, n);
    p3 = Arith<T>::div(q3, n);
    return;
  }
  if (sqrtG != T(1)) n = Arith<T>::div(n, sqrtG);  // x / 1 == x exactly
  n = vmax(n, T(1));
  if (n != T(1)) {  // interior point: p / 1 == p exactly
    p1 = Arith<T>::div(q1, n);
    p2 = Arith<T>::div(q2, n);
    p3 = Arith<T>::div(q3, n);
  } else {
    p1 = q1;
    p2 = q2;
    p3 = q3;
  }
}

// denoise_timestamps dual ascent + unit-ball projection (surface.py:168-183)
template <class T>
__device__ __forceinline__ void tv_dual_step(T dx, T dy, T sigma, T& px, T& py) {
  const T a = Arith<T>::mad(dx, sigma, px);
  const T b = Arith<T>::mad(dy, sigma, py);
  const T n = vmax(Arith<T>::sqrt(Arith<T>::mad(b, b, a * a)), T(1));
  if constexpr (sizeof(T) == 4) {  // binary32: unconditional a * rcp(n)
    px = Arith<T>::div(a, n);
    py = Arith<T>::div(b, n);
    return;
  }
  if (n != T(1)) {
    px = Arith<T>::div(a, n);
    py = Arith<T>::div(b, n);
  } else {
    px = a;
    py = b;
  }
}

// denoise_timestamps primal step with L1 soft shrink (surface.py:185-193);
// returns u+, writes the over-relaxed u_bar = u+ * 2 - u
template <class T>
__device__ __forceinline__ T tv_primal_step(T divp, T u, T f0, T tau, T shrink, T& ubar) {
  const T t1 = Arith<T>::mad(divp, tau, u);
  const T g = vclip(t1 - f0, -shrink, shrink);
  const T un = t1 - g;
  ubar = Arith<T>::mad(un, T(2), -u);  // un * 2 is exact: same bits either way
  return un;
}

// normalize_timestamps (surface.py:141-142), evaluated in float64
__device__ __forceinline__ double normalize_at(double raw, double now, double t_scale,
                                               double window) {
  const double age = vclip(now - raw, 0.0, window);
  return t_scale * (1.0 - age / window);
}

}  // namespace evr
