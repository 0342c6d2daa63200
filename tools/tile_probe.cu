// Diagnostic: float64 tile kernels, generation 1 (evr_tile.cuh) vs
// generation 2 (evr_tile64.cuh) on synthetic C3-sized state: bitwise
// agreement after a chain of launches and time per launch (CUDA events).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false \
//        --expt-relaxed-constexpr -I tools/exp -I paper_1607_06283_b200/csrc -o tools/tile_probe tools/tile_probe.cu
//   tools/tile_probe [H W launches]
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <random>
#include <vector>

#include "evr_tile64.cuh"

using namespace evr;
using Q = Q4<double>;

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));     \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

__global__ void k_recip(const Q* c, Q* c2, int64_t N) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= N) return;
  Q a = c[2 * k], b = c[2 * k + 1];
  c2[2 * k] = a;
  c2[2 * k + 1] = Q{b.x, b.y, fdp_recip(b.y), b.w};
}

static int H = 720, W = 1280, NL = 33;
static const double tau = 1.0 / std::sqrt(8.0 + 4.0 * std::sqrt(2.0)), sigma = tau;
static const double lam = 180.0 / 255.0, tl = tau * lam;

template <class F> float time_it(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / reps;
}

MarchRows<Q> rows(const Q* p, int E) {
  MarchRows<Q> r;
  r.own = p;
  r.up = r.dn = nullptr;
  r.y0 = 0;
  r.y1 = H;
  r.olo = 0;
  r.E = E;
  return r;
}

int main(int argc, char** argv) {
  if (argc > 2) H = atoi(argv[1]), W = atoi(argv[2]);
  if (argc > 3) NL = atoi(argv[3]);
  const int64_t N = (int64_t)H * W;
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U(0, 1);
  std::normal_distribution<double> Nd(0, 1);
  std::vector<Q> st(N), cst(2 * N), tv(N);
  std::vector<double> f0(N);
  for (int64_t k = 0; k < N; ++k) {
    const bool flat = U(rng) < 0.8;
    const double tx = flat ? 0.0 : 0.4 * Nd(rng), ty = flat ? 0.0 : 0.4 * Nd(rng);
    const double G = (1.0 + tx * tx) + ty * ty, sg = std::sqrt(G);
    const double f = 1.0 + U(rng);
    const double beta = tl * sg;
    cst[2 * k] = Q{(1.0 + ty * ty) / G, -(tx * ty) / G, (1.0 + tx * tx) / G, tx / G};
    cst[2 * k + 1] = Q{ty / G, sg, beta, 4.0 * beta * f};
    st[k] = Q{0.3 * Nd(rng), 0.3 * Nd(rng), 0.3 * Nd(rng), 1.0 + U(rng)};
    const double t = U(rng) < 0.8 ? 0.0 : 3.0 * U(rng);
    f0[k] = t;
    tv[k] = Q{t, t, 0.3 * Nd(rng), 0.3 * Nd(rng)};
  }
  Q *d_st[2], *d_c, *d_c2, *d_tv[2];
  double* d_f0;
  for (int i = 0; i < 2; ++i) {
    CK(cudaMalloc(&d_st[i], N * sizeof(Q)));
    CK(cudaMalloc(&d_tv[i], N * sizeof(Q)));
  }
  CK(cudaMalloc(&d_c, 2 * N * sizeof(Q)));
  CK(cudaMalloc(&d_c2, 2 * N * sizeof(Q)));
  CK(cudaMalloc(&d_f0, N * sizeof(double)));
  CK(cudaMemcpy(d_c, cst.data(), 2 * N * sizeof(Q), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_f0, f0.data(), N * sizeof(double), cudaMemcpyHostToDevice));
  k_recip<<<(N + 255) / 256, 256>>>(d_c, d_c2, N);
  CK(cudaDeviceSynchronize());
  long long lo, hi;
  { const double a = 1.0, b = 2.0; memcpy(&lo, &a, 8); memcpy(&hi, &b, 8); }

  // ---- reference: generation-1 kernels (K = 3, RPT 4, G 8, 2 CTAs / SM)
  auto reset = [&]() {
    CK(cudaMemcpy(d_st[0], st.data(), N * sizeof(Q), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_tv[0], tv.data(), N * sizeof(Q), cudaMemcpyHostToDevice));
  };
  std::vector<Q> ref_pd(N), ref_tv(N), got(N);
  MetricPackF64 m1{d_c, rows(d_c, 2)};
  MetricPackF64 m2{d_c2, rows(d_c2, 2)};
  MarchRows<double> fr;
  fr.own = d_f0;
  fr.up = fr.dn = nullptr;
  fr.y0 = 0;
  fr.y1 = H;
  fr.olo = 0;
  fr.E = 1;
  const double tvs = 1.0 / std::sqrt(8.0), shrink = tvs * 1.0;
  const PdScalars S{tau, sigma, tl, 1.0, 2.0, lo, hi};
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);

  auto gen1_pd = [&](int K, int a) {
    constexpr int G = 8, RPT = 4;
    const int TIW = 32 - 2 * K, TIH = G * RPT - 2 * K;
    dim3 grid((W + TIW - 1) / TIW, (H + TIH - 1) / TIH);
    if (K == 3)
      k_pd_tile<double, 3, RPT, G, 2, MetricPackF64, false><<<grid, 32 * G>>>(
          rows(d_st[a], 1), m1, d_st[a ^ 1], H, W, tau, sigma, 1.0, 2.0, 0, (double*)nullptr);
    else
      k_pd_tile<double, 4, RPT, G, 2, MetricPackF64, false><<<grid, 32 * G>>>(
          rows(d_st[a], 1), m1, d_st[a ^ 1], H, W, tau, sigma, 1.0, 2.0, 0, (double*)nullptr);
  };
  auto gen1_tv = [&](int K, int a) {
    constexpr int G = 8, RPT = 4;
    const int TIW = 32 - 2 * K, TIH = G * RPT - 2 * K;
    dim3 grid((W + TIW - 1) / TIW, (H + TIH - 1) / TIH);
    if (K == 3)
      k_tv_tile<double, 3, RPT, G, 2, false><<<grid, 32 * G>>>(rows(d_tv[a], 1), fr, d_tv[a ^ 1], H,
                                                               W, tvs, tvs, shrink, 0);
    else
      k_tv_tile<double, 4, RPT, G, 2, false><<<grid, 32 * G>>>(rows(d_tv[a], 1), fr, d_tv[a ^ 1], H,
                                                               W, tvs, tvs, shrink, 0);
  };
  reset();
  for (int i = 0; i < NL; ++i) gen1_pd(3, i & 1);
  for (int i = 0; i < NL; ++i) gen1_tv(3, i & 1);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(ref_pd.data(), d_st[NL & 1], N * sizeof(Q), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ref_tv.data(), d_tv[NL & 1], N * sizeof(Q), cudaMemcpyDeviceToHost));
  printf("sensor %dx%d, %d launches\n", W, H, NL);
  printf("%-44s %9.2f us/launch\n", "gen1 k_pd_tile K3 RPT4 G8 MINB2",
         time_it([&] { gen1_pd(3, 0); }, 20));
  printf("%-44s %9.2f us/launch\n", "gen1 k_tv_tile K3 RPT4 G8 MINB2",
         time_it([&] { gen1_tv(3, 0); }, 20));

  auto check = [&](const char* name, int tvk, auto launch, int K) {
    reset();
    for (int i = 0; i < NL; ++i) launch(i & 1);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(got.data(), (tvk ? d_tv : d_st)[NL & 1], N * sizeof(Q), cudaMemcpyDeviceToHost));
    const std::vector<Q>& ref = tvk ? ref_tv : ref_pd;
    int64_t bad = 0;
    for (int64_t k = 0; k < N; ++k) bad += memcmp(&got[k], &ref[k], sizeof(Q)) != 0;
    const float us = time_it([&] { launch(0); }, 20);
    printf("%-44s %9.2f us/launch  %6.2f us/iter  mismatches %lld\n", name, us, us / K,
           (long long)bad);
  };
#define PD2(K, RPT, G, MINB, CPL)                                                               \
  check("gen2 pd K" #K " RPT" #RPT " G" #G " MINB" #MINB " CPL" #CPL, 0,                     \
        [&](int a) {                                                                           \
          const int TIW = 32 * CPL - 2 * K, TIH = G * RPT - 2 * K;                             \
          dim3 grid((W + TIW - 1) / TIW, (H + TIH - 1) / TIH);                                 \
          k_pd_tile64<K, RPT, G, MINB, CPL, false><<<grid, 32 * G>>>(                          \
              rows(d_st[a], 1), m2, d_st[a ^ 1], H, W, S);      \
        },                                                                                     \
        K)
#define TV2(K, RPT, G, MINB, CPL)                                                               \
  check("gen2 tv K" #K " RPT" #RPT " G" #G " MINB" #MINB " CPL" #CPL, 1,                     \
        [&](int a) {                                                                           \
          const int TIW = 32 * CPL - 2 * K, TIH = G * RPT - 2 * K;                             \
          dim3 grid((W + TIW - 1) / TIW, (H + TIH - 1) / TIH);                                 \
          k_tv_tile64<K, RPT, G, MINB, CPL, false><<<grid, 32 * G>>>(                          \
              rows(d_tv[a], 1), fr, d_tv[a ^ 1], H, W, tvs, tvs, shrink, 0);                      \
        },                                                                                     \
        K)
#define PDP(K, RPT, G, MINB)                                                                    \
  {                                                                                            \
    auto kern = k_pd_tile64p<K, RPT, G, MINB>;                                                 \
    const int smem = G * RPT * 32 * 96 + 16;                                                   \
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));         \
    const int TIW = 32 - 2 * K, TIH = G * RPT - 2 * K;                                         \
    const int ntx = (W + TIW - 1) / TIW, nt = ntx * ((H + TIH - 1) / TIH);                     \
    for (int mult = 1; mult <= MINB; ++mult) {                                                 \
      const int grid = std::min(nt, sms * mult);                                               \
      char name[96];                                                                           \
      snprintf(name, sizeof name, "gen2p pd K%d RPT%d G%d MINB%d grid %d", K, RPT, G, MINB, grid); \
      check(name, 0,                                                                           \
            [&](int a) {                                                                       \
              kern<<<grid, 32 * G, smem>>>(d_st[a], d_c2, d_st[a ^ 1], H, W, ntx, nt, S);     \
            },                                                                                 \
            K);                                                                                \
      CK(cudaGetLastError());                                                                  \
    }                                                                                          \
  }
#define PDS(K, RPT, G, MINB, NB)                                                               \
  {                                                                                            \
    auto kern = k_pd_tile64s<K, RPT, G, MINB, NB>;                                             \
    const int smem = G * RPT * 32 * 64;                                                        \
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));         \
    const int TIW = 32 - 2 * K, TIH = G * RPT - 2 * K;                                         \
    dim3 grid((W + TIW - 1) / TIW, (H + TIH - 1) / TIH);                                       \
    check("gen2s pd K" #K " RPT" #RPT " G" #G " MINB" #MINB " NB" #NB, 0,                      \
          [&](int a) { kern<<<grid, 32 * G, smem>>>(d_st[a], d_c2, d_st[a ^ 1], H, W, S); }, K); \
    CK(cudaGetLastError());                                                                    \
  }
#define TV1(K, RPT, G, MINB)                                                                   \
  check("gen1 tv K" #K " RPT" #RPT " G" #G " MINB" #MINB, 1,                                   \
        [&](int a) {                                                                           \
          const int TIW = 32 - 2 * K, TIH = G * RPT - 2 * K;                                   \
          dim3 grid((W + TIW - 1) / TIW, (H + TIH - 1) / TIH);                                 \
          k_tv_tile<double, K, RPT, G, MINB, false><<<grid, 32 * G>>>(rows(d_tv[a], 1), fr,   \
                                                                    d_tv[a ^ 1], H, W, tvs,   \
                                                                    tvs, shrink, 0);          \
        },                                                                                     \
        K)
#define PD1(K, RPT, G, MINB)                                                                   \
  check("gen1 pd K" #K " RPT" #RPT " G" #G " MINB" #MINB, 0,                                   \
        [&](int a) {                                                                           \
          const int TIW = 32 - 2 * K, TIH = G * RPT - 2 * K;                                   \
          dim3 grid((W + TIW - 1) / TIW, (H + TIH - 1) / TIH);                                 \
          k_pd_tile<double, K, RPT, G, MINB, MetricPackF64, false><<<grid, 32 * G>>>(          \
              rows(d_st[a], 1), m1, d_st[a ^ 1], H, W, tau, sigma, 1.0, 2.0, 0, (double*)nullptr);                  \
        },                                                                                     \
        K)
  PD1(3, 3, 8, 2);
#define PDG(K, RPT, OFF)                                                                       \
  {                                                                                            \
    auto kern = k_pd_tile64pg<K, RPT>;                                                         \
    const int smem = 2 * 8 * RPT * 32 * 96;                                                    \
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));         \
    const int TIW = 32 - 2 * K, TIH = 8 * RPT - 2 * K;                                         \
    const int ntx = (W + TIW - 1) / TIW, nt = ntx * ((H + TIH - 1) / TIH);                     \
    check("gen2pg pd K" #K " RPT" #RPT " offset " #OFF, 0,                                     \
          [&](int a) { kern<<<sms, 512, smem>>>(d_st[a], d_c2, d_st[a ^ 1], H, W, ntx, nt, S, OFF); }, \
          K);                                                                                  \
    CK(cudaGetLastError());                                                                    \
  }
  PDG(3, 3, 0);
  PDG(3, 3, 1);
  PDG(3, 3, 2);
  PDG(3, 3, 3);
  PDG(3, 4, 1);
  return 0;
}
