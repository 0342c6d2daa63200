// evr_math.cuh -- per-pixel arithmetic of the hot path, shared by every
// engine (streaming kernels, resident persistent kernel, operator kernels).
//
// Each function is one pixel's worth of a reference stage, written in the
// reference's exact operation order.  The translation
// unit is compiled with -fmad=false, so with T = double every result is
// bit-identical to numpy float64: IEEE div.rn / sqrt.rn, no contraction.
// Scalars (tau, sigma, tau*lam, c+-, ...) come from the host already
// rounded exactly as the reference computes them; none is re-derived here.
#pragma once

#include <cstdint>

namespace evr {

// np.minimum / np.maximum / np.clip on non-NaN data
template <class T> __device__ __forceinline__ T vmax(T a, T b) { return b > a ? b : a; }
template <class T> __device__ __forceinline__ T vmin(T a, T b) { return b < a ? b : a; }
template <class T> __device__ __forceinline__ T vclip(T x, T lo, T hi) {
  return vmin(vmax(x, lo), hi);
}

// Division / square root of the iteration kernels.  binary64: IEEE div.rn /
// sqrt.rn (the bit-exact engine).  binary32: the hardware approximations
// (MUFU-based, ~2 ulp), which keep the float engine well inside its 1e-4
// log-intensity tolerance at a fraction of the instruction count.
template <class T> struct Arith;
template <> struct Arith<double> {
  static __device__ __forceinline__ double div(double a, double b) { return a / b; }
  static __device__ __forceinline__ double sqrt(double x) { return ::sqrt(x); }
};
template <> struct Arith<float> {
  static __device__ __forceinline__ float div(float a, float b) { return __fdividef(a, b); }
  static __device__ __forceinline__ float sqrt(float x) {
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
  }
};

template <class T> struct Coef { T a11, a12, a22, a31, a32; };

// MetricField.coeffs (surface.py:81-90)
template <class T>
__device__ __forceinline__ Coef<T> coeffs_of(T tx, T ty, T G) {
  Coef<T> c;
  c.a11 = Arith<T>::div(T(1) + ty * ty, G);
  c.a12 = Arith<T>::div(-(tx * ty), G);
  c.a22 = Arith<T>::div(T(1) + tx * tx, G);
  c.a31 = Arith<T>::div(tx, G);
  c.a32 = Arith<T>::div(ty, G);
  return c;
}

// compute_metric (surface.py:202-205): G = 1 + tx*tx + ty*ty, left to right
template <class T> __device__ __forceinline__ T metric_G(T tx, T ty) {
  return T(1) + tx * tx + ty * ty;
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
  m.c.a11 = (1.0f + ty * ty) * r;
  m.c.a12 = -(tx * ty) * r;
  m.c.a22 = (1.0f + tx * tx) * r;
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
  qx = c.a11 * p1 + c.a12 * p2 + c.a31 * p3;
  qy = c.a12 * p1 + c.a22 * p2 + c.a32 * p3;
}

// primal_dual_solve KL prox (solve.py:235-242): t1 = div*tau + u;
// s = t1 - beta; clip((s + sqrt(s*s + 4 beta f)) * 0.5)
template <class T>
__device__ __forceinline__ T kl_primal(T divq, T u, T beta, T fb, T tau, T umin, T umax) {
  const T t1 = divq * tau + u;
  const T s = t1 - beta;
  const T r = (s + Arith<T>::sqrt(s * s + fb)) * T(0.5);
  return vclip(r, umin, umax);
}

// rof_manifold_solve primal (solve.py:285-287): ((div*tau + u) + wf) * inv
template <class T>
__device__ __forceinline__ T rof_primal(T divq, T u, T wf, T inv, T tau) {
  return (divq * tau + u + wf) * inv;
}

// _Loop.dual_ascent (solve.py:175-201) at one pixel; gx, gy are the forward
// differences of the over-relaxed point (0 on the last column / row).
template <class T>
__device__ __forceinline__ void dual_step(const Coef<T>& c, T sigma, T gx, T gy, T sqrtG,
                                          T& p1, T& p2, T& p3) {
  const T s11 = sigma * c.a11, s12 = sigma * c.a12, s22 = sigma * c.a22;
  const T s31 = sigma * c.a31, s32 = sigma * c.a32;
  const T q1 = p1 + s11 * gx + s12 * gy;
  const T q2 = p2 + s12 * gx + s22 * gy;
  const T q3 = p3 + s31 * gx + s32 * gy;
  T n = Arith<T>::sqrt(q1 * q1 + q2 * q2 + q3 * q3);
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
  const T a = px + dx * sigma;
  const T b = py + dy * sigma;
  const T n = vmax(Arith<T>::sqrt(a * a + b * b), T(1));
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
  const T t1 = divp * tau + u;
  const T g = vclip(t1 - f0, -shrink, shrink);
  const T un = t1 - g;
  ubar = un * T(2) - u;
  return un;
}

// normalize_timestamps (surface.py:141-142), evaluated in float64
__device__ __forceinline__ double normalize_at(double raw, double now, double t_scale,
                                               double window) {
  const double age = vclip(now - raw, 0.0, window);
  return t_scale * (1.0 - age / window);
}

}  // namespace evr
