// Diagnostic: throughput of the float64 MUFU seeds (MUFU.RSQ64H / RCP64H)
// against the float32 MUFU.RSQ, independent chains, full occupancy.
#include <cstdio>
template <int OP, int ILP>
__global__ void k(double* out, int n) {
  double a[ILP];
  float b[ILP];
  for (int i = 0; i < ILP; ++i) a[i] = 1.5 + threadIdx.x * 1e-7 + i, b[i] = 1.5f + i;
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      if (OP == 0) asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(a[i]));
      if (OP == 1) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(a[i]));
      if (OP == 2) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(b[i]));
      if (OP == 3) asm volatile("add.f64 %0, %0, %0;" : "+d"(a[i]));
    }
  }
  double s = 0;
  for (int i = 0; i < ILP; ++i) s += a[i] + b[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int OP> void run(const char* name) {
  double* o;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 1024, blocks = sms * 2, n = 4096;
  cudaMalloc(&o, sizeof(double) * blocks * threads);
  k<OP, 8><<<blocks, threads>>>(o, n);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<OP, 8><<<blocks, threads>>>(o, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = (double)blocks * threads * n * 8;
  printf("%-22s %8.3f T lane-ops/s  = %6.2f lanes/clk/SM at 1.965 GHz\n", name, ops / (ms * 1e-3) / 1e12,
         ops / (ms * 1e-3) / 1.965e9 / sms);
  cudaFree(o);
}
int main() {
  run<0>("rsqrt.approx.ftz.f64");
  run<1>("rcp.approx.ftz.f64");
  run<2>("rsqrt.approx.ftz.f32");
  run<3>("add.f64");
  return 0;
}
