// evr_ingest.cuh -- ordered, bit-exact event ingest (apply_event,
// pipeline.py:114-121; update_timestamp_map, surface.py:124-127).
//
// The reference applies events one by one: f[y,x] = clamp(f[y,x] * c) and
// raw[y,x] = t, so duplicates at one pixel compound in stream order with a
// clamp after every step and the last timestamp wins.  Multiply-then-clamp
// does not commute, hence the device must preserve the per-pixel order.
//
// A CTA takes the packet in chunks of NT events.  Events of the rows it is
// responsible for get the 32-bit key (local pixel << log2(NT)) | lane, one
// cub block radix sort groups them by pixel with the stream order kept
// inside each group, and the first lane of every group walks its group
// applying the events in order.  Cost per chunk is one sort of NT keys plus
// the longest duplicate run, independent of how the events cluster; chunks
// are ordered by CTA barriers.
#pragma once

#include <cub/block/block_radix_sort.cuh>
#include <cstdint>

#include "../../include/evr.h"

namespace evr {

template <int NT> struct IngestSort {
  static constexpr int LOG_NT = NT == 1024 ? 10 : NT == 512 ? 9 : NT == 256 ? 8 : 7;
  static_assert((1 << LOG_NT) == NT, "NT must be 128, 256, 512 or 1024");
  using Sort = cub::BlockRadixSort<uint32_t, NT, 1>;
  struct Storage {
    typename Sort::TempStorage sort;
    uint32_t keys[NT];
  };
};

__host__ __device__ inline int bits_for(uint32_t v) {
  int b = 0;
  while ((1u << b) < v && b < 32) ++b;
  return b;
}

// Apply the packet's events of global rows [row_lo, row_hi] in stream order.
//   load(lp) -> double   current f at local pixel lp = (row - row_lo) * W + x
//   store(lp, f, t)      final f and last timestamp of a touched pixel
// Every thread of the CTA must call this (it contains barriers).
template <int NT, class Load, class Store>
__device__ __forceinline__ void ordered_ingest(const evr_event* __restrict__ ev, int64_t n, int H,
                                               int W, int row_lo, int row_hi, double c_pos,
                                               double c_neg, double u_min, double u_max,
                                               typename IngestSort<NT>::Storage& sm, int* err,
                                               Load load, Store store) {
  using S = IngestSort<NT>;
  constexpr uint32_t NONE = 0xffffffffu;
  const int tid = threadIdx.x;
  const uint32_t npix = (uint32_t)(row_hi - row_lo + 1) * (uint32_t)W;
  const int end_bit = S::LOG_NT + bits_for(npix + 1);
  for (int64_t base = 0; base < n; base += NT) {
    uint32_t key[1] = {NONE};
    if (base + tid < n) {
      const evr_event e = ev[base + tid];
      if (e.x >= 0 && e.x < W && e.y >= 0 && e.y < H) {
        if (e.y >= row_lo && e.y <= row_hi)
          key[0] = ((uint32_t)((e.y - row_lo) * W + e.x) << S::LOG_NT) | (uint32_t)tid;
      } else if (err) {
        atomicOr(err, 1);
      }
    }
    typename S::Sort(sm.sort).Sort(key, 0, end_bit < 32 ? end_bit : 32);
    sm.keys[tid] = key[0];
    __syncthreads();
    const uint32_t k = key[0];
    if (k != NONE && (end_bit >= 32 || k < (1u << end_bit))) {
      const uint32_t lp = k >> S::LOG_NT;
      if (tid == 0 || (sm.keys[tid - 1] >> S::LOG_NT) != lp) {
        double v = load((int)lp);
        int64_t last_t = 0;
        for (int s = tid; s < NT; ++s) {
          const uint32_t ks = sm.keys[s];
          if (ks == NONE || (ks >> S::LOG_NT) != lp) break;
          const evr_event e = ev[base + (ks & (NT - 1))];
          v = v * (e.polarity > 0 ? c_pos : c_neg);
          if (u_min > v) v = u_min;  // Python max(value, u_min)
          if (u_max < v) v = u_max;  // Python min(.., u_max)
          last_t = e.t;
        }
        store((int)lp, v, last_t);
      }
    }
    __syncthreads();
  }
}

}  // namespace evr
