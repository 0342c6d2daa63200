// pdmath_probe.cu -- how fast is the float64 primal-dual arithmetic alone?
// (diagnostic, GPU)
//
// The per-pixel operation sequence of k_pd_tile<f64, DT_KL> (q = A^T p,
// divergence, KL prox through kl_primal_fx, over-relaxation, dual ascent
// through dual_pre_fx_r, the projection through fdp_div3, the slow-path
// flags) on register-resident pixels, with the neighbour values taken from
// the thread's own rows instead of shuffles / shared memory and no barriers,
// loads or stores inside the loop.  Time per pixel-iteration against the
// tile's (40.0 us per C3 launch / 4.61 M computed pixel-iterations) says how
// much of the tile's cost is the arithmetic itself.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false \
//        -I paper_1607_06283_b200/csrc -o tools/pdmath_probe tools/pdmath_probe.cu
#include <cstdio>

#include "evr_fastdp.cuh"
#include "evr_math.cuh"

using namespace evr;

template <int R, int MINB>
__global__ void __launch_bounds__(256, MINB) k_math(double* out, int iters, double tau, double sigma,
                                                    int proj_every) {
  double p1[R], p2[R], p3[R], u[R], sg[R], ysg[R], beta[R], fb[R];
  Coef<double> cf[R];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const double s = 1e-3 * ((t * 7 + r * 13) % 97);
    p1[r] = 0.3 + s;
    p2[r] = -0.2 + s;
    p3[r] = 0.1 - s;
    u[r] = 1.5 + s;
    const double tx = 0.05 + s, ty = -0.03 + s, G = 1.0 + tx * tx + ty * ty;
    cf[r] = Coef<double>{(1.0 + ty * ty) / G, -(tx * ty) / G, (1.0 + tx * tx) / G, tx / G, ty / G};
    sg[r] = sqrt(G);
    ysg[r] = fdp_recip(sg[r]);
    beta[r] = 0.19 * sg[r];
    fb[r] = 4.0 * beta[r] * (1.4 + s);
  }
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    double qx[R], qy[R], v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) q_of(cf[r], p1[r], p2[r], p3[r], qx[r], qy[r]);
    {
      double d[R], nu[R];
      bool slow = false;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double qxl = qx[(r + 1) % R], qyu = qy[(r + R - 1) % R];
        d[r] = (qx[r] - qxl) + (qy[r] - qyu);
        nu[r] = kl_primal_fx(d[r], u[r], beta[r], fb[r], tau, 1.0, 2.0, slow);
      }
      if (slow) {
#pragma unroll
        for (int r = 0; r < R; ++r) nu[r] = kl_primal(d[r], u[r], beta[r], fb[r], tau, 1.0, 2.0);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        v[r] = Arith<double>::mad(nu[r], 2.0, -u[r]);
        u[r] = nu[r];
      }
    }
    {
      double gx[R], gy[R], n1[R], n2[R], n3[R], nn[R];
      bool slow = false, proj = false;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double vr = v[(r + 1) % R], vd = v[(r + R - 1) % R];
        gx[r] = vr - v[r];
        gy[r] = vd - v[r];
        n1[r] = p1[r];
        n2[r] = p2[r];
        n3[r] = p3[r];
        nn[r] = dual_pre_fx_r(cf[r], sigma, gx[r], gy[r], sg[r], ysg[r], n1[r], n2[r], n3[r], slow);
        proj |= nn[r] != 1.0;
      }
      if (__any_sync(0xffffffffu, proj) || (proj_every && it % proj_every == 0)) {
#pragma unroll
        for (int r = 0; r < R; ++r) fdp_div3(n1[r], n2[r], n3[r], proj_every ? 1.25 : nn[r], slow);
      }
      if (slow) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          n1[r] = p1[r];
          n2[r] = p2[r];
          n3[r] = p3[r];
          dual_step(cf[r], sigma, gx[r], gy[r], sg[r], n1[r], n2[r], n3[r]);
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        p1[r] = n1[r];
        p2[r] = n2[r];
        p3[r] = n3[r];
      }
    }
  }
  double acc = 0.0;
#pragma unroll
  for (int r = 0; r < R; ++r) acc += p1[r] + p2[r] + p3[r] + u[r];
  out[t] = acc;
}

template <int R, int MINB> void run(double* out, int ctas, int iters, int proj_every) {
  const double tau = 0.2705980500730985, sigma = tau;
  k_math<R, MINB><<<ctas, 256>>>(out, 2, tau, sigma, proj_every);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_math<R, MINB><<<ctas, 256>>>(out, iters, tau, sigma, proj_every);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double pix_it = (double)ctas * 256 * R * iters;
  printf("R=%d MINB=%d ctas=%d proj_every=%d: %.3f ms, %.3f ps per pixel-iteration (%s)\n", R, MINB,
         ctas, proj_every, ms, ms * 1e9 / pix_it, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 8 * 256 * sizeof(double));
  const int iters = 2000;
  for (int pe : {0, 1}) {
    run<3, 2>(out, 296, iters, pe);
    run<3, 2>(out, 296 * 4, iters / 4, pe);
    run<2, 3>(out, 444, iters, pe);
    run<4, 2>(out, 296, iters, pe);
    run<6, 1>(out, 148, iters, pe);
    run<1, 4>(out, 592, iters, pe);
  }
  printf("tile reference: k_pd_tile<f64,K=3> 40.0 us / (2000 CTAs x 768 pixels x 3) = %.3f ps\n",
         40.0e6 / (2000.0 * 768 * 3));
  return 0;
}
