// evr_ingest.cuh -- ordered, bit-exact event ingest (apply_event,
// pipeline.py:114-121; update_timestamp_map, surface.py:124-127).
//
// The reference applies events one by one: f[y,x] = clamp(f[y,x] * c) and
// raw[y,x] = t, so duplicates at one pixel compound in stream order with a
// clamp after every step and the last timestamp wins.  Multiply-then-clamp
// does not commute, hence the device must preserve the per-pixel order.
//
// A CTA owns a range of rows and takes the packet in chunks of NT events:
//   1. every thread tests one event; the events of the CTA's rows are
//      compacted, in stream order, into a shared list (warp ballots + a
//      prefix over the per-warp counts);
//   2. warp 0 walks the list 32 entries at a time: __match_any_sync groups
//      equal pixels, the lowest lane of each group applies the group's
//      events in lane (= stream) order, and consecutive 32-entry windows run
//      in program order, so a pixel's duplicates compound exactly as in the
//      sequential reference.
// A row band sees a small share of the packet, so the walk is a handful of
// warp steps; a band that receives the whole packet costs n/32 of them.
#pragma once

#include <cstdint>

#include "../../include/evr.h"

namespace evr {

template <int NT> struct IngestShared {
  int pix[NT];    // local pixel of each kept event
  int idx[NT];    // its index inside the chunk
  int wcount[NT / 32];
};

// Apply the packet's events of global rows [row_lo, row_hi] in stream order.
//   load(lp) -> double   current f at local pixel lp = (row - row_lo) * W + x
//   store(lp, f, t)      final f and last timestamp of a touched pixel
// Every thread of the CTA must call this (it contains barriers).
template <int NT, class Load, class Store>
__device__ __forceinline__ void ordered_ingest(const evr_event* __restrict__ ev, int64_t n, int H,
                                               int W, int row_lo, int row_hi, double c_pos,
                                               double c_neg, double u_min, double u_max,
                                               IngestShared<NT>& sm, int* err, Load load,
                                               Store store) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int64_t base = 0; base < n; base += NT) {
    bool keep = false;
    int lp = 0;
    if (base + tid < n) {
      const evr_event e = ev[base + tid];
      if (e.x >= 0 && e.x < W && e.y >= 0 && e.y < H) {
        if (e.y >= row_lo && e.y <= row_hi) {
          keep = true;
          lp = (e.y - row_lo) * W + e.x;
        }
      } else if (err) {
        atomicOr(err, 1);
      }
    }
    const unsigned ball = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) sm.wcount[wid] = __popc(ball);
    __syncthreads();
    int off = 0, m = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
      const int c = sm.wcount[w];
      off += w < wid ? c : 0;
      m += c;
    }
    if (keep) {
      const int pos = off + __popc(ball & ((1u << lane) - 1u));
      sm.pix[pos] = lp;
      sm.idx[pos] = tid;
    }
    __syncthreads();
    if (wid == 0) {
      for (int s = 0; s < m; s += 32) {
        const int k = s + lane;
        const bool act = k < m;
        const unsigned live = __ballot_sync(0xffffffffu, act);
        if (act) {
          const int pix = sm.pix[k];
          const unsigned grp = __match_any_sync(live, pix);
          if (lane == __ffs(grp) - 1) {
            double v = load(pix);
            int64_t last_t = 0;
            for (unsigned g = grp; g; g &= g - 1) {
              const evr_event e = ev[base + sm.idx[s + __ffs(g) - 1]];
              v = v * (e.polarity > 0 ? c_pos : c_neg);
              if (u_min > v) v = u_min;  // Python max(value, u_min)
              if (u_max < v) v = u_max;  // Python min(.., u_max)
              last_t = e.t;
            }
            store(pix, v, last_t);
          }
        }
        __syncwarp();
      }
    }
    __syncthreads();
  }
}

}  // namespace evr
