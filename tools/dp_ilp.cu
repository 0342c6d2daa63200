// Diagnostic: float64 throughput vs chains per thread (ILP) and warps per SM,
// pure DFMA and DFMA interleaved with one integer op each.
#include <cstdio>
template <int ILP, int MIX>
__global__ void k(double* out, int n) {
  double a[ILP];
  unsigned m[ILP];
  for (int i = 0; i < ILP; ++i) a[i] = 1.0 + threadIdx.x * 1e-9 + i, m[i] = threadIdx.x + i;
  const double b = 0.999999, c = 1e-7;
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      a[i] = fma(a[i], b, c);
      if (MIX) m[i] = m[i] * 3u + (unsigned)it;
    }
  }
  double s = 0;
  for (int i = 0; i < ILP; ++i) s += a[i] + m[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int ILP, int MIX> void run(int warps_per_sm) {
  double* o;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 32 * warps_per_sm;
  cudaMalloc(&o, sizeof(double) * sms * threads);
  const int n = 1 << 14;
  k<ILP, MIX><<<sms, threads>>>(o, n);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<ILP, MIX><<<sms, threads>>>(o, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = (double)sms * threads * n * ILP;
  printf("ILP %d mix %d warps/SM %2d: %6.2f Tdfma/s\n", ILP, MIX, warps_per_sm, ops / (ms * 1e-3) / 1e12);
  cudaFree(o);
}
int main() {
  for (int w : {8, 16, 32}) {
    run<1, 0>(w); run<2, 0>(w); run<4, 0>(w); run<8, 0>(w);
    run<1, 1>(w); run<2, 1>(w); run<4, 1>(w); run<8, 1>(w);
  }
  return 0;
}
