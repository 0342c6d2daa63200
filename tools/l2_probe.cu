// Diagnostic: effective bandwidth of repeated passes over a working set of
// S MB (read-only, and read + write of half of it) -- where the L2 stops
// holding it.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const double4* __restrict__ a, long n, double* out) {
  double s = 0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    double4 v = a[i];
    s += v.x + v.w;
  }
  if (s == 12345.678) *out = s;
}
__global__ void rw(const double4* __restrict__ a, double4* __restrict__ b, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    double4 v = a[i];
    v.x += 1.0;
    b[i] = v;
  }
}
int main() {
  double4 *a, *b; double* o;
  size_t maxb = 512ull << 20;
  cudaMalloc(&a, maxb); cudaMalloc(&b, maxb); cudaMalloc(&o, 8);
  cudaMemset(a, 0, maxb); cudaMemset(b, 0, maxb);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mb : {16, 32, 48, 64, 80, 96, 112, 128, 160, 256, 512}) {
    long n = ((long)mb << 20) / 32;
    for (int w = 0; w < 3; ++w) rd<<<sms * 8, 256>>>(a, n, o);
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) rd<<<sms * 8, 256>>>(a, n, o);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double bw = 20.0 * mb * 1048576.0 / (ms * 1e-3) / 1e12;
    long n2 = n / 2;  // read half, write half: the same bytes moved
    for (int w = 0; w < 3; ++w) rw<<<sms * 8, 256>>>(a, b, n2);
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) rw<<<sms * 8, 256>>>(a, b, n2);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double bw2 = 20.0 * mb * 1048576.0 / (ms * 1e-3) / 1e12;
    printf("working set %4d MB: read %6.2f TB/s   read+write %6.2f TB/s\n", mb, bw, bw2);
  }
  return 0;
}
