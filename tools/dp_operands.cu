// dp_operands.cu -- float64 instruction rate when every operand is a distinct,
// changing register (diagnostic, GPU).
//
// tools/dp_ilp.cu reaches 18.37 T DFMA/s with fma(a[i], b, c): b and c are
// loop-invariant, so the operand reuse cache supplies two of the three
// 64-bit operands.  The solver's float64 stream reads 2-3 distinct live
// registers per instruction.  This measures DADD / DMUL / DFMA chains whose
// operands all change every iteration, at the tile's shape (16 warps per
// SM) and at 32 warps per SM, ILP 2-8.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false \
//        -o tools/dp_operands tools/dp_operands.cu
#include <cstdio>

// OP 0: a[i] = a[i] + b[j]; b[i] = b[i] * a[k]   (two-operand DADD / DMUL)
// OP 1: a[i] = fma(a[i], b[j], c[k]), rotating   (three distinct operands)
// OP 2: a[i] = fma(a[i], b, c) with b, c fixed   (dp_ilp's case, for reference)
template <int ILP, int OP>
__global__ void k(double* out, int n) {
  double a[ILP], b[ILP], c[ILP];
  for (int i = 0; i < ILP; ++i) {
    a[i] = 1.0 + threadIdx.x * 1e-9 + i * 1e-3;
    b[i] = 0.9999999 - i * 1e-9;
    c[i] = 1e-9 * (i + 1);
  }
  const double bf = 0.999999, cf = 1e-7;
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      if constexpr (OP == 0) {
        a[i] = __dadd_rn(a[i], c[(i + 1) % ILP]);
        b[i] = __dmul_rn(b[i], b[(i + 2) % ILP]);
        c[i] = __dadd_rn(c[i], -c[(i + 3) % ILP]);
      } else if constexpr (OP == 1) {
        a[i] = fma(a[i], b[(i + 1) % ILP], c[(i + 2) % ILP]);
        b[i] = fma(b[i], c[(i + 1) % ILP], a[(i + 3) % ILP] * 1e-30);
        c[i] = fma(c[i], a[(i + 2) % ILP] * 1e-30, b[(i + 3) % ILP] * 1e-30);
      } else {
        a[i] = fma(a[i], bf, cf);
        b[i] = fma(b[i], bf, cf);
        c[i] = fma(c[i], bf, cf);
      }
    }
  }
  double s = 0;
  for (int i = 0; i < ILP; ++i) s += a[i] + b[i] + c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int ILP, int OP> void run(int warps_per_sm) {
  double* o;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 32 * warps_per_sm;
  cudaMalloc(&o, sizeof(double) * sms * threads);
  const int n = 1 << 13;
  k<ILP, OP><<<sms, threads>>>(o, n);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<ILP, OP><<<sms, threads>>>(o, n);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  // instructions per inner step: OP 0 three, OP 1 three DFMA (+ the DMULs by
  // 1e-30: two more in b, three in c -> counted), OP 2 three
  const double per = OP == 1 ? 3.0 + 4.0 : 3.0;
  const double ops = (double)sms * threads * n * ILP * per;
  printf("OP %d ILP %d warps/SM %2d: %6.2f T float64 instr/s (%s)\n", OP, ILP, warps_per_sm,
         ops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(o);
}

int main() {
  for (int w : {16, 32}) {
    run<2, 0>(w); run<4, 0>(w); run<8, 0>(w);
    run<2, 1>(w); run<4, 1>(w);
    run<2, 2>(w); run<4, 2>(w); run<8, 2>(w);
  }
  return 0;
}
