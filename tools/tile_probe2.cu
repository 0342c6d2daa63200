#define EVR_PROBE_NOLOAD 1
#include "evr_tile64.cuh"
#include <cstdio>
using namespace evr;
using Q = Q4<double>;
int main() {
  int H = 720, W = 1280; int64_t N = (int64_t)H * W;
  Q *a, *b, *c; cudaMalloc(&a, N * 32); cudaMalloc(&b, N * 32); cudaMalloc(&c, N * 64);
  cudaMemset(a, 0, N*32); cudaMemset(c, 0, N*64);
  MarchRows<Q> r{a, nullptr, nullptr, 0, H, 0, 1};
  MarchRows<Q> rc{c, nullptr, nullptr, 0, H, 0, 2};
  double tau = 0.27, tl = 0.19; long long lo = 0x3ff0000000000000LL, hi = 0x4000000000000000LL;
  PdScalars S{tau, tau, tl, 1.0, 2.0, lo, hi};
  auto run = [&](const char* name, auto kern, dim3 grid, int threads, MetricPackF64 m, int K) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    kern<<<grid, threads>>>(r, m, b, H, W, S); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) kern<<<grid, threads>>>(r, m, b, H, W, S);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-40s %8.2f us/launch %s\n", name, ms * 50, cudaGetErrorString(cudaGetLastError()));
  };
  MetricPackF64 mload{c, rc}, mnone{nullptr, rc};
  dim3 g3((W + 25) / 26, (H + 25) / 26), g0(W / 32, H / 32);
  run("K3 RPT4 G8 MINB2 load+compute", k_pd_tile64<3, 4, 8, 2, 1, false>, g3, 256, mload, 3);
  run("K3 RPT4 G8 MINB2 compute only", k_pd_tile64<3, 4, 8, 2, 1, false>, g3, 256, mnone, 3);
  run("K0 RPT4 G8 MINB2 load+store (no halo)", k_pd_tile64<0, 4, 8, 2, 1, false>, g0, 256, mload, 0);
  run("K1 RPT4 G8 MINB2 compute only", k_pd_tile64<1, 4, 8, 2, 1, false>, dim3((W+29)/30,(H+29)/30), 256, mnone, 1);
  run("K3 RPT4 G8 MINB1 compute only", k_pd_tile64<3, 4, 8, 1, 1, false>, g3, 256, mnone, 3);
  run("K3 RPT8 G8 MINB1 compute only", k_pd_tile64<3, 8, 8, 1, 1, false>, dim3((W + 25) / 26, (H + 57) / 58), 256, mnone, 3);
  run("K3 RPT2 G16 MINB2 compute only", k_pd_tile64<3, 2, 16, 2, 1, false>, g3, 512, mnone, 3);
  run("K3 RPT2 G8 MINB4 compute only", k_pd_tile64<3, 2, 8, 4, 1, false>, dim3((W + 25) / 26, (H + 9) / 10), 256, mnone, 3);
  return 0;
}
