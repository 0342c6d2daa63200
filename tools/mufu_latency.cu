// Diagnostic: dependent-chain latency (cycles) of the float64 MUFU seeds
// against the float32 MUFU.RSQ and a DADD, one warp, clock64 around the chain.
#include <cstdio>
template <int OP>
__global__ void k(double* out, long long* cyc, int n) {
  double a = 1.5 + threadIdx.x * 1e-7;
  float b = 1.5f;
  const long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
    if (OP == 0) asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(a));
    if (OP == 1) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(a));
    if (OP == 2) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(b));
    if (OP == 3) asm volatile("add.f64 %0, %0, %0;" : "+d"(a));
    if (OP == 4) asm volatile("shfl.sync.up.b32 %0, %0, 1, 0, -1;" : "+f"(b));
  }
  const long long t1 = clock64();
  out[threadIdx.x] = a + b;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
template <int OP> void run(const char* name) {
  double* o;
  long long* c;
  cudaMalloc(&o, 32 * sizeof(double));
  cudaMalloc(&c, sizeof(long long));
  const int n = 1 << 14;
  k<OP><<<1, 32>>>(o, c, n);
  k<OP><<<1, 32>>>(o, c, n);
  long long h;
  cudaMemcpy(&h, c, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-24s %6.1f cycles per dependent op\n", name, (double)h / n);
}
int main() {
  run<0>("MUFU.RSQ64H (f64 seed)");
  run<1>("MUFU.RCP64H (f64 seed)");
  run<2>("MUFU.RSQ (f32)");
  run<3>("DADD");
  run<4>("SHFL.UP");
  return 0;
}
