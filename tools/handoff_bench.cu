// handoff_bench.cu -- one-way latency of a tagged-word handoff between two
// CTAs through L2 (the resident engine's neighbour exchange), diagnostic.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/hb tools/handoff_bench.cu
// CTA a and CTA b ping-pong ROUNDS times on one 64-bit word each way;
// prints ns per one-way handoff for several CTA pairs (same die / far die
// is decided by the hardware's SM placement of the CTA ids).
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

constexpr int ROUNDS = 2000;

__global__ void pingpong(unsigned long long* words, int a, int b, unsigned long long* out) {
  if (threadIdx.x != 0) return;
  unsigned smid;
  asm("mov.u32 %0, %%smid;" : "=r"(smid));
  if (blockIdx.x != a && blockIdx.x != b) return;
  const bool first = blockIdx.x == a;
  unsigned long long* mine = words + (first ? 0 : 32);
  unsigned long long* theirs = words + (first ? 32 : 0);
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int r = 1; r <= ROUNDS; ++r) {
    if (first) {
      st_relaxed(mine, r);
      while (ld_relaxed(theirs) != (unsigned long long)r) {
      }
    } else {
      while (ld_relaxed(theirs) != (unsigned long long)r) {
      }
      st_relaxed(mine, r);
    }
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (first) {
    out[0] = t1 - t0;
    out[1] = smid;
  } else {
    out[2] = smid;
  }
}

int main() {
  unsigned long long *w, *o, h[3];
  cudaMalloc(&w, 64 * sizeof(unsigned long long));
  cudaMalloc(&o, 3 * sizeof(unsigned long long));
  const int pairs[][2] = {{0, 1}, {0, 2}, {0, 74}, {0, 147}, {10, 90}, {64, 65}};
  for (const auto& p : pairs) {
    cudaMemset(w, 0, 64 * sizeof(unsigned long long));
    void* args[] = {&w, (void*)&p[0], (void*)&p[1], &o};
    cudaLaunchCooperativeKernel((void*)pingpong, 148, 32, args, 0, 0);
    cudaDeviceSynchronize();
    cudaMemcpy(h, o, sizeof h, cudaMemcpyDeviceToHost);
    printf("CTAs %3d,%3d (SM %3llu,%3llu): %.1f ns per one-way handoff\n", p[0], p[1], h[1], h[2],
           (double)h[0] / (2.0 * ROUNDS));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
