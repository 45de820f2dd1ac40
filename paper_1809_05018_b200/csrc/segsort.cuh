// segsort.cuh -- warp-level sort / unique building blocks shared by the
// device structure builders (hoods.cu, structure.cu): the sort_by_key +
// unique pairs of proj/include/dpmrf/dpp/kernels.hpp restricted to short
// segments, where one warp owns a segment and the data never leaves
// registers (<= 32 keys) or the warp's shared-memory slice (<= 1024 keys).
#pragma once

#include "common.cuh"

namespace dpmrf_b200 {

constexpr uint32_t kPad = 0xFFFFFFFFu;  // sorts last; never a valid id

// Ascending bitonic sort of one key per lane (32 keys) with shuffles.
__device__ __forceinline__ uint32_t warp_bitonic32(uint32_t x, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
      const bool up = (lane & k) == 0;
      const bool lower = (lane & j) == 0;
      x = (lower == up) ? min(x, y) : max(x, y);
    }
  }
  return x;
}

// Unique-compacts a sorted run held in lanes (chunk of 32); returns the
// number written.  valid: lane holds an element; prev_last/has_prev: the last
// key of the previous chunk of the same run.
__device__ __forceinline__ uint32_t warp_unique_chunk(uint32_t x, bool valid, uint32_t prev_last,
                                                      bool has_prev, uint32_t* out, int lane) {
  uint32_t left = __shfl_up_sync(0xffffffffu, x, 1);
  if (lane == 0) left = prev_last;
  const bool keep = valid && ((lane == 0 && !has_prev) || x != left);
  const unsigned mask = __ballot_sync(0xffffffffu, keep);
  if (keep) out[__popc(mask & ((1u << lane) - 1u))] = x;
  return __popc(mask);
}

// Ascending bitonic sort of b[0, P) (P a power of two) by the threads
// [0, nthreads) of `sync`'s group; sync() orders the passes.
template <class Sync>
__device__ __forceinline__ void bitonic_sort(uint32_t* b, uint64_t P, uint32_t tid,
                                             uint32_t nthreads, Sync sync) {
  for (uint64_t k = 2; k <= P; k <<= 1) {
    for (uint64_t j = k >> 1; j > 0; j >>= 1) {
      for (uint64_t i = tid; i < P; i += nthreads) {
        const uint64_t l = i ^ j;
        if (l > i) {
          const uint32_t xi = b[i], xl = b[l];
          const bool asc = (i & k) == 0;
          if ((xi > xl) == asc) {
            b[i] = xl;
            b[l] = xi;
          }
        }
      }
      sync();
    }
  }
}

// Unique of the sorted b[0, n) into out by one warp; returns the count.
__device__ __forceinline__ uint32_t warp_unique_sorted(const uint32_t* b, uint32_t n,
                                                       uint32_t* out, int lane) {
  uint32_t written = 0, last = 0;
  for (uint32_t base = 0; base < n; base += 32) {
    const uint32_t i = base + lane;
    const uint32_t x = i < n ? b[i] : kPad;
    written += warp_unique_chunk(x, i < n, last, base > 0, out + written, lane);
    last = __shfl_sync(0xffffffffu, x, 31);
  }
  return written;
}

// Sort + unique of one short segment held by a G-lane group of the warp
// (G in {2, 4, ..., 32}; every lane of the warp calls this; lane l = lane % G
// holds key x, kPad for none).  Returns the segment's unique count; keep /
// rank tell a lane whether and where (within the segment) its key goes.
template <int G>
__device__ __forceinline__ uint32_t group_sort_unique(uint32_t& x, int lane, bool& keep,
                                                      uint32_t& rank) {
  static_assert(G >= 2 && G <= 32 && (G & (G - 1)) == 0, "group width");
  const int l = lane & (G - 1);
#pragma unroll
  for (int k = 2; k <= G; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
      const bool up = (l & k) == 0;
      const bool lower = (l & j) == 0;
      x = (lower == up) ? min(x, y) : max(x, y);
    }
  }
  const uint32_t left = __shfl_up_sync(0xffffffffu, x, 1, G);
  keep = x != kPad && (l == 0 || x != left);
  const unsigned all = __ballot_sync(0xffffffffu, keep);
  const unsigned gmask = G == 32 ? 0xffffffffu : ((1u << G) - 1u);
  const unsigned seg = (all >> (lane & ~(G - 1))) & gmask;
  rank = __popc(seg & ((1u << l) - 1u));
  return __popc(seg);
}

}  // namespace dpmrf_b200
