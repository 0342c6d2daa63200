// Diagnostic microbenchmark of ordered-ingest strategies (not product code).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o ingest_bench ingest_bench.cu
#include <cub/block/block_radix_sort.cuh>
#include <cstdio>
#include <cstdlib>
#include <vector>

struct Ev { long long t; int x; short y; short pol; };

// V1: leader scan (as k_ingest)
__global__ void __launch_bounds__(1024) v1(const Ev* ev, int n, double* f, long long* raw, int W) {
  __shared__ int spix[1024];
  const int tid = threadIdx.x;
  for (int base = 0; base < n; base += 1024) {
    const int m = min(1024, n - base);
    int pix = -1 - tid;
    if (tid < m) pix = ev[base + tid].y * W + ev[base + tid].x;
    spix[tid] = pix;
    __syncthreads();
    if (tid < m) {
      bool leader = true;
      for (int j = tid - 1; j >= 0; --j)
        if (spix[j] == pix) { leader = false; break; }
      if (leader) {
        double v = f[pix];
        int last = tid;
        for (int j = tid; j < m; ++j) {
          if (spix[j] != pix) continue;
          const double c = ev[base + j].pol > 0 ? 1.16 : 0.86;
          v = v * c;
          if (1.0 > v) v = 1.0;
          if (2.0 < v) v = 2.0;
          last = j;
        }
        f[pix] = v;
        raw[pix] = ev[base + last].t;
      }
    }
    __syncthreads();
  }
}

// V2: block radix sort of (pix << 10 | idx), segment leaders walk their run
__global__ void __launch_bounds__(1024) v2(const Ev* ev, int n, double* f, long long* raw, int W) {
  using Sort = cub::BlockRadixSort<unsigned long long, 1024, 1>;
  __shared__ typename Sort::TempStorage tmp;
  __shared__ unsigned long long skey[1024];
  const int tid = threadIdx.x;
  for (int base = 0; base < n; base += 1024) {
    const int m = min(1024, n - base);
    unsigned long long key[1];
    key[0] = tid < m ? ((unsigned long long)(ev[base + tid].y * W + ev[base + tid].x) << 11) | tid
                     : ~0ull;
    Sort(tmp).Sort(key);
    skey[tid] = key[0];
    __syncthreads();
    if (tid < m) {
      const unsigned long long pix = key[0] >> 11;
      const bool head = tid == 0 || (skey[tid - 1] >> 11) != pix;
      if (head) {
        double v = f[pix];
        int last = 0;
        for (int s = tid; s < m && (skey[s] >> 11) == pix; ++s) {
          const int j = (int)(skey[s] & 2047);
          const double c = ev[base + j].pol > 0 ? 1.16 : 0.86;
          v = v * c;
          if (1.0 > v) v = 1.0;
          if (2.0 < v) v = 2.0;
          last = j;
        }
        f[pix] = v;
        raw[pix] = ev[base + last].t;
      }
    }
    __syncthreads();
  }
}

int main() {
  const int W = 346, H = 260, N = W * H;
  double* f; long long* raw; Ev* d;
  cudaMalloc(&f, N * 8); cudaMalloc(&raw, N * 8); cudaMalloc(&d, 8192 * sizeof(Ev));
  std::vector<double> hf(N, 1.5);
  for (int hot = 0; hot < 2; ++hot)
    for (int n : {100, 500, 1000, 4000}) {
      std::vector<Ev> h(n);
      srand(1);
      for (int i = 0; i < n; ++i) h[i] = Ev{i, rand() % W, (short)(hot ? rand() % 2 : rand() % H), (short)(rand() % 2 ? 1 : -1)};
      cudaMemcpy(d, h.data(), n * sizeof(Ev), cudaMemcpyHostToDevice);
      for (int v = 1; v <= 2; ++v) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaMemcpy(f, hf.data(), N * 8, cudaMemcpyHostToDevice);
        for (int w = 0; w < 3; ++w) (v == 1 ? v1 : v2)<<<1, 1024>>>(d, n, f, raw, W);
        cudaEventRecord(a);
        for (int r = 0; r < 10; ++r) (v == 1 ? v1 : v2)<<<1, 1024>>>(d, n, f, raw, W);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("hot=%d n=%5d v%d: %9.2f us  (%s)\n", hot, n, v, ms * 100.f, cudaGetErrorString(cudaGetLastError()));
      }
    }
  return 0;
}
