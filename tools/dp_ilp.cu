// Diagnostic: float64 throughput vs chains per thread (ILP) and warps per SM,
// pure DFMA and DFMA interleaved with one integer op each.
#include <cstdio>
template <int ILP, int MIX, class T = double>
__global__ void k(T* out, int n) {
  T a[ILP];
  unsigned m[ILP];
  for (int i = 0; i < ILP; ++i) a[i] = 1.0 + threadIdx.x * 1e-9 + i, m[i] = threadIdx.x + i;
  const T b = (T)0.999999, c = (T)1e-7;
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      a[i] = fma(a[i], b, c);
      if (MIX) m[i] = m[i] * 3u + (unsigned)it;
    }
  }
  T s = 0;
  for (int i = 0; i < ILP; ++i) s += a[i] + (T)m[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int ILP, int MIX, class T = double> void run(int warps_per_sm) {
  T* o;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 32 * warps_per_sm;
  cudaMalloc(&o, sizeof(T) * sms * threads);
  const int n = 1 << 14;
  k<ILP, MIX, T><<<sms, threads>>>(o, n);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<ILP, MIX, T><<<sms, threads>>>(o, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = (double)sms * threads * n * ILP;
  printf("%s ILP %d mix %d warps/SM %2d: %6.2f T fma/s\n", sizeof(T) == 8 ? "f64" : "f32", ILP,
         MIX, warps_per_sm, ops / (ms * 1e-3) / 1e12);
  cudaFree(o);
}
int main() {
  for (int w : {8, 16, 32}) {
    run<1, 0>(w); run<2, 0>(w); run<4, 0>(w); run<8, 0>(w);
    run<1, 1>(w); run<2, 1>(w); run<4, 1>(w); run<8, 1>(w);
    run<4, 0, float>(w); run<8, 0, float>(w); run<8, 1, float>(w);
  }
  return 0;
}
