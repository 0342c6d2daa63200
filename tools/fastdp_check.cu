// fastdp_check.cu -- GPU check that evr_fastdp.cuh's branch-free binary64
// division / square root equal the IEEE operators bit for bit wherever they
// report the fast path valid (diagnostic; build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false \
//        -o /tmp/fastdp_check tools/fastdp_check.cu && /tmp/fastdp_check [rounds]).
// Operands: full-range random bit patterns, the magnitudes of this path
// (norms, metric determinants, |p| <= a few), and near-square / near-exact
// quotients that sit next to rounding boundaries.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>

#include "../paper_1607_06283_b200/csrc/evr_fastdp.cuh"

using namespace evr;

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}
__device__ __forceinline__ double unit(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

// kind 0: arbitrary finite bits; 1: path magnitudes; 2: near-boundary
__device__ void operands(uint64_t i, int kind, double& a, double& b) {
  const uint64_t h1 = mix(i * 2 + 1), h2 = mix(i * 2 + 2), h3 = mix(i ^ 0x9e3779b97f4a7c15ull);
  if (kind == 0) {
    a = __longlong_as_double((long long)h1);
    b = __longlong_as_double((long long)h2);
  } else if (kind == 1) {
    a = (unit(h1) * 2.0 - 1.0) * exp2((double)((int)(h3 % 40) - 30));
    b = 1.0 + unit(h2) * exp2((double)((int)((h3 >> 8) % 24) - 12));
  } else {
    // a = b * q (+- a few ulps) for short q: quotients next to ties
    b = 1.0 + unit(h2);
    const double q = (double)(1 + (h1 % 4096)) * 0x1.0p-12;
    a = __longlong_as_double(__double_as_longlong(b * q) + (long long)(h3 % 5) - 2);
  }
}

__device__ unsigned long long g_ex[3][8][2];
__device__ unsigned g_nex[3];
__device__ void note(int op, double a, double b) {
  const unsigned k = atomicAdd(&g_nex[op], 1u);
  if (k < 8) {
    g_ex[op][k][0] = __double_as_longlong(a);
    g_ex[op][k][1] = __double_as_longlong(b);
  }
}

__global__ void check(uint64_t base, int kind, unsigned long long* bad, unsigned long long* slow_n) {
  const uint64_t i = base + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double a, b;
  operands(i, kind, a, b);
  unsigned long long nbad = 0, nslow = 0;
  // division
  {
    bool slow = false;
    const double q = fdp_div(a, b, slow);
    const double r = a / b;
    if (slow) ++nslow;
    else if (__double_as_longlong(q) != __double_as_longlong(r) && !(q != q && r != r)) {
      ++nbad;
      note(0, a, b);
    }
  }
  // shared reciprocal for three numerators
  {
    bool oka;
    const double y = fdp_recip(b);
    const double a2 = a * 0.75, a3 = -a * 1.3125;
    const double n[3] = {a, a2, a3};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double q = fdp_quot(n[k], b, y, oka);
      const double r = n[k] / b;
      if (!oka) continue;
      if (__double_as_longlong(q) != __double_as_longlong(r) && !(q != q && r != r)) {
        ++nbad;
        note(1, n[k], b);
      }
    }
  }
  // square root of |a| and of a*a + b*b style sums
  {
    const double xs[2] = {fabs(a), __fma_rn(a, a, b * b)};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      bool slow = false;
      const double s = fdp_sqrt(xs[k], slow);
      const double r = sqrt(xs[k]);
      if (slow) ++nslow;
      else if (__double_as_longlong(s) != __double_as_longlong(r) && !(s != s && r != r)) {
        ++nbad;
        note(2, xs[k], 0.0);
      }
    }
  }
  if (nbad) atomicAdd(bad, nbad);
  if (nslow) atomicAdd(slow_n, nslow);
}

int main(int argc, char** argv) {
  const int rounds = argc > 1 ? atoi(argv[1]) : 64;
  unsigned long long *d, h[2];
  cudaMalloc(&d, 2 * sizeof(unsigned long long));
  const int threads = 256, blocks = 148 * 64;
  const uint64_t per = (uint64_t)threads * blocks;
  for (int kind = 0; kind < 3; ++kind) {
    cudaMemset(d, 0, 2 * sizeof(unsigned long long));
    for (int r = 0; r < rounds; ++r) check<<<blocks, threads>>>(per * r, kind, d, d + 1);
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("kind %d: %llu operand sets, mismatches %llu, slow-path verdicts %llu\n", kind,
           (unsigned long long)(per * rounds), h[0], h[1]);
  }
  unsigned long long ex[3][8][2];
  unsigned nex[3];
  cudaMemcpyFromSymbol(ex, g_ex, sizeof ex);
  cudaMemcpyFromSymbol(nex, g_nex, sizeof nex);
  for (int op = 0; op < 3; ++op) {
    printf("op %d (%s): %u mismatches\n", op, op == 0 ? "div" : op == 1 ? "shared div" : "sqrt", nex[op]);
    for (int k = 0; k < 8 && k < (int)nex[op]; ++k) {
      double a, b;
      memcpy(&a, &ex[op][k][0], 8);
      memcpy(&b, &ex[op][k][1], 8);
      printf("   a=%a b=%a\n", a, b);
    }
  }
  const cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  return 0;
}
