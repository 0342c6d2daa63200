// evr_simulate.cu -- GPU event simulator: the events a
// log-intensity frame stack produces under the comparator model of
// simulate.py:51-103 (generate_events), sorted by (t, y, x, polarity).
//
// One thread per pixel walks the frame intervals in order -- the pixel's
// running reference level is its only state -- counting its crossings
// (pass 1), then, at its offset from an exclusive scan, writing each
// crossing as a 64-bit sort key {t - t_first : 30 | y : 16 | x : 16 |
// polarity : 1} (pass 2); a device radix sort orders the keys exactly as the
// reference's lexsort((p, x, y, t)) and a last pass unpacks them into
// evr_event records.  Every float64 step repeats the reference's own
// operation order (compiled with -fmad=false, IEEE division, rint =
// round-half-even), so the stream is bit-identical to the reference given
// the same log frames (the host takes np.log, simulate.py:60).
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "../../include/evr.h"

namespace {

constexpr double kCrossingEps = 1e-9;  // simulate.py:20
constexpr int kNT = 256;

// crossings of one pixel in one frame interval (simulate.py:80-84)
__device__ __forceinline__ void crossings(double l1, double ref, double dp, double dn,
                                          int64_t& n_pos, int64_t& n_neg) {
  const double a = floor(__dadd_rn(__ddiv_rn(__dsub_rn(l1, ref), dp), kCrossingEps));
  const double b = floor(__dadd_rn(__ddiv_rn(__dsub_rn(ref, l1), dn), kCrossingEps));
  n_pos = a > 0.0 ? (int64_t)a : 0;
  n_neg = b > 0.0 ? (int64_t)b : 0;
}

// rint(t0 + (level - l0) / (l1 - l0) * (t1 - t0)) (simulate.py:68-70)
__device__ __forceinline__ int64_t crossing_time(double level, double l0, double l1, int64_t t0,
                                                 int64_t t1) {
  const double frac = __ddiv_rn(__dsub_rn(level, l0), __dsub_rn(l1, l0));
  return (int64_t)rint(__dadd_rn((double)t0, __dmul_rn(frac, (double)(t1 - t0))));
}

__device__ __forceinline__ unsigned long long sim_key(int64_t t, int64_t t_first, int y, int x,
                                                      int pol) {
  return ((unsigned long long)(t - t_first) << 33) | ((unsigned long long)y << 17) |
         ((unsigned long long)x << 1) | (pol > 0 ? 1ull : 0ull);
}

// EMIT = false: per-pixel crossing count; EMIT = true: keys at `offset`
template <bool EMIT>
__global__ void __launch_bounds__(kNT)
k_sim_walk(const double* __restrict__ L, const int64_t* __restrict__ ts, int n, int64_t N, int W,
           double dp, double dn, int64_t* __restrict__ count, const int64_t* __restrict__ offset,
           unsigned long long* __restrict__ keys) {
  const int64_t pix = (int64_t)blockIdx.x * kNT + threadIdx.x;
  if (pix >= N) return;
  const int y = (int)(pix / W), x = (int)(pix - (int64_t)y * W);
  double ref = L[pix];  // log_frames[0] (simulate.py:65)
  int64_t total = 0, o = EMIT ? offset[pix] : 0;
  for (int k = 0; k + 1 < n; ++k) {
    const double l0 = L[(int64_t)k * N + pix], l1 = L[(int64_t)(k + 1) * N + pix];
    int64_t n_pos, n_neg;
    crossings(l1, ref, dp, dn, n_pos, n_neg);
    if (EMIT) {
      const int64_t t0 = ts[k], t1 = ts[k + 1];
      for (int64_t j = 1; j <= n_pos; ++j)
        keys[o++] = sim_key(crossing_time(__dadd_rn(ref, __dmul_rn((double)j, dp)), l0, l1, t0, t1),
                            ts[0], y, x, +1);
      for (int64_t j = 1; j <= n_neg; ++j)
        keys[o++] = sim_key(crossing_time(__dsub_rn(ref, __dmul_rn((double)j, dn)), l0, l1, t0, t1),
                            ts[0], y, x, -1);
    }
    total += n_pos + n_neg;
    // ref += n_pos * dp - n_neg * dn (simulate.py:93)
    ref = __dadd_rn(ref, __dsub_rn(__dmul_rn((double)n_pos, dp), __dmul_rn((double)n_neg, dn)));
  }
  if (!EMIT) count[pix] = total;
}

__global__ void k_sim_unpack(const unsigned long long* __restrict__ keys, int64_t n,
                             int64_t t_first, evr_event* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x;
  if (i >= n) return;
  const unsigned long long k = keys[i];
  evr_event e;
  e.t = t_first + (int64_t)(k >> 33);
  e.x = (int32_t)((k >> 1) & 0xffff);
  e.y = (int16_t)((k >> 17) & 0xffff);
  e.polarity = (k & 1) ? 1 : -1;
  out[i] = e;
}

}  // namespace

struct evr_sim {
  int device = 0;
  cudaStream_t stream = nullptr;
  double* L = nullptr;
  int64_t* ts = nullptr;
  int64_t* count = nullptr;  // per pixel, then exclusive offsets
  int64_t* offset = nullptr;
  unsigned long long* keys[2] = {nullptr, nullptr};
  evr_event* events = nullptr;
  void* temp = nullptr;
  size_t cap_L = 0, cap_count = 0, cap_offset = 0, cap_k0 = 0, cap_k1 = 0, cap_ev = 0;
  size_t cap_temp = 0;
  int cap_n = 0;
  int64_t n_events = 0;
  std::string err;
};

namespace {

int sim_fail(evr_sim* s, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (s) s->err = buf;
  return code;
}

#define SIM_CK(call)                                                                     \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return sim_fail(s, e_ == cudaErrorMemoryAllocation ? EVR_ERR_OOM : EVR_ERR_CUDA,   \
                      "%s failed: %s", #call, cudaGetErrorString(e_));                   \
  } while (0)

template <class T> int grow(evr_sim* s, T** p, size_t& cap, size_t want) {
  if (want <= cap) return EVR_OK;
  cudaFree(*p);
  *p = nullptr;
  cap = 0;
  SIM_CK(cudaMalloc(p, want * sizeof(T)));
  cap = want;
  return EVR_OK;
}

}  // namespace

extern "C" {

int evr_sim_create(evr_sim** out, int device) {
  if (!out) return EVR_ERR_INVALID;
  evr_sim* s = new evr_sim();
  s->device = device;
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete s;
    return EVR_ERR_CUDA;
  }
  *out = s;
  return EVR_OK;
}

void evr_sim_destroy(evr_sim* s) {
  if (!s) return;
  cudaSetDevice(s->device);
  if (s->stream) cudaStreamSynchronize(s->stream);
  cudaFree(s->L);
  cudaFree(s->ts);
  cudaFree(s->count);
  cudaFree(s->offset);
  cudaFree(s->keys[0]);
  cudaFree(s->keys[1]);
  cudaFree(s->events);
  cudaFree(s->temp);
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
}

const char* evr_sim_last_error(const evr_sim* s) { return s ? s->err.c_str() : "null simulator"; }

int evr_sim_generate(evr_sim* s, const double* log_frames, const int64_t* frame_ts, int n, int H,
                     int W, double dp, double dn, int64_t* n_events) {
  if (!s) return EVR_ERR_INVALID;
  if (!log_frames || !frame_ts || n < 2 || H < 1 || W < 1)
    return sim_fail(s, EVR_ERR_INVALID, "need a (n>=2, h, w) log-frame stack");
  if (!(dp > 0) || !(dn > 0))
    return sim_fail(s, EVR_ERR_INVALID, "thresholds must be positive, got dp=%g, dn=%g", dp, dn);
  if (H > 32767 || W > 65535)
    return sim_fail(s, EVR_ERR_UNSUPPORTED, "sensor %dx%d beyond the packed event key", W, H);
  for (int k = 0; k + 1 < n; ++k)
    if (frame_ts[k + 1] <= frame_ts[k])
      return sim_fail(s, EVR_ERR_INVALID, "frame timestamps must be strictly increasing");
  if (frame_ts[n - 1] - frame_ts[0] >= (int64_t(1) << 30))
    return sim_fail(s, EVR_ERR_UNSUPPORTED, "frame time span beyond the packed event key");
  if (cudaSetDevice(s->device) != cudaSuccess) return sim_fail(s, EVR_ERR_CUDA, "cudaSetDevice");
  int rc;
  const int64_t N = (int64_t)H * W;
  if ((rc = grow(s, &s->L, s->cap_L, (size_t)n * N))) return rc;
  if ((size_t)n > (size_t)s->cap_n) {
    cudaFree(s->ts);
    s->ts = nullptr;
    SIM_CK(cudaMalloc(&s->ts, sizeof(int64_t) * n));
    s->cap_n = n;
  }
  if ((rc = grow(s, &s->count, s->cap_count, (size_t)N))) return rc;
  if ((rc = grow(s, &s->offset, s->cap_offset, (size_t)N))) return rc;
  cudaStream_t st = s->stream;
  SIM_CK(cudaMemcpyAsync(s->L, log_frames, sizeof(double) * n * N, cudaMemcpyHostToDevice, st));
  SIM_CK(cudaMemcpyAsync(s->ts, frame_ts, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
  const unsigned grid = (unsigned)((N + kNT - 1) / kNT);
  k_sim_walk<false><<<grid, kNT, 0, st>>>(s->L, s->ts, n, N, W, dp, dn, s->count, nullptr,
                                          nullptr);
  // exclusive offsets + total
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, s->count, s->offset, N, st);
  if (tb > s->cap_temp) {
    cudaFree(s->temp);
    s->temp = nullptr;
    SIM_CK(cudaMalloc(&s->temp, tb));
    s->cap_temp = tb;
  }
  SIM_CK(cub::DeviceScan::ExclusiveSum(s->temp, tb, s->count, s->offset, N, st));
  int64_t last_off = 0, last_cnt = 0;
  SIM_CK(cudaMemcpyAsync(&last_off, s->offset + N - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  SIM_CK(cudaMemcpyAsync(&last_cnt, s->count + N - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  SIM_CK(cudaStreamSynchronize(st));
  const int64_t total = last_off + last_cnt;
  s->n_events = total;
  if (n_events) *n_events = total;
  if (total == 0) return EVR_OK;
  if ((rc = grow(s, &s->keys[0], s->cap_k0, (size_t)total))) return rc;
  if ((rc = grow(s, &s->keys[1], s->cap_k1, (size_t)total))) return rc;
  if ((rc = grow(s, &s->events, s->cap_ev, (size_t)total))) return rc;
  k_sim_walk<true><<<grid, kNT, 0, st>>>(s->L, s->ts, n, N, W, dp, dn, nullptr, s->offset,
                                         s->keys[0]);
  // 30 time bits + 33 coordinate bits
  cub::DoubleBuffer<unsigned long long> db(s->keys[0], s->keys[1]);
  tb = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tb, db, total, 0, 63, st);
  if (tb > s->cap_temp) {
    cudaFree(s->temp);
    s->temp = nullptr;
    SIM_CK(cudaMalloc(&s->temp, tb));
    s->cap_temp = tb;
  }
  SIM_CK(cub::DeviceRadixSort::SortKeys(s->temp, tb, db, total, 0, 63, st));
  int64_t t_first = frame_ts[0];
  k_sim_unpack<<<(unsigned)((total + kNT - 1) / kNT), kNT, 0, st>>>(db.Current(), total, t_first,
                                                                   s->events);
  SIM_CK(cudaGetLastError());
  SIM_CK(cudaStreamSynchronize(st));
  return EVR_OK;
}

int evr_sim_events(evr_sim* s, evr_event* out, int64_t cap) {
  if (!s || (!out && cap > 0)) return EVR_ERR_INVALID;
  if (cap < s->n_events)
    return sim_fail(s, EVR_ERR_RANGE, "buffer of %lld events for %lld", (long long)cap,
                    (long long)s->n_events);
  if (s->n_events == 0) return EVR_OK;
  SIM_CK(cudaSetDevice(s->device));
  SIM_CK(cudaMemcpyAsync(out, s->events, sizeof(evr_event) * s->n_events, cudaMemcpyDeviceToHost,
                         s->stream));
  SIM_CK(cudaStreamSynchronize(s->stream));
  return EVR_OK;
}

int evr_sim_device_events(evr_sim* s, const evr_event** dev_events, int64_t* n) {
  if (!s || !dev_events || !n) return EVR_ERR_INVALID;
  *dev_events = s->events;
  *n = s->n_events;
  return EVR_OK;
}

}  // extern "C"
