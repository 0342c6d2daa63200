// Diagnostic: latency / throughput of float64 and float32 ops on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o dp_latency dp_latency.cu
#include <cstdio>

template <int OP, class T>
__global__ void chain(T* out, T x, int n, long long* cyc) {
  T a = x + threadIdx.x * 1e-9, b = x * 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (OP == 0) a = a + b;
    if (OP == 1) a = a * b;
    if (OP == 2) a = sqrt(a);
    if (OP == 3) a = b / a;
    if (OP == 4) a = fma(a, b, b);
  }
  long long t1 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = a;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int OP, class T> void run(const char* name, int blocks, int threads) {
  T* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(T) * blocks * threads);
  cudaMalloc(&cyc, 8);
  const int n = 4096;
  chain<OP, T><<<blocks, threads>>>(out, (T)1.0000001, n, cyc);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  chain<OP, T><<<blocks, threads>>>(out, (T)1.0000001, n, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double ops = (double)blocks * threads * n;
  printf("%-12s %5d x %4d: %7.2f cyc/op (1 thread chain)  %9.1f Gop/s\n", name, blocks, threads,
         (double)c / n, ops / (ms * 1e6));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int cfg = 0; cfg < 2; ++cfg) {
    const int B = cfg ? 148 * 4 : 1, T = cfg ? 512 : 32;
    run<0, double>("dadd", B, T);
    run<1, double>("dmul", B, T);
    run<4, double>("dfma", B, T);
    run<2, double>("dsqrt.rn", B, T);
    run<3, double>("ddiv.rn", B, T);
    run<0, float>("fadd", B, T);
    run<2, float>("fsqrt.rn", B, T);
    run<3, float>("fdiv.rn", B, T);
  }
  return 0;
}
