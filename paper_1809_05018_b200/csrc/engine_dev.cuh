// engine_dev.cuh -- device helpers shared by the MAP kernels (engine.cu) and
// the M-step / EM tail (mstep.cu): launch shapes, the EM/MAP skip state, the
// executed-iteration bookkeeping and the small-graph label scatter that the
// last fused MAP launch runs in its extra blocks.  Internal header.
#pragma once

#include "engine.cuh"

namespace dpmrf_b200 {
namespace {
constexpr int kVtxThreads = 256;
constexpr int kHoodThreads = 256;

// The per-MAP-iteration counters live behind a small EM state block in the
// same allocation: unconv[kEmDone] != 0 once the EM loop has stopped on the
// device (optimize.cpp:71 evaluated by k_em_epilogue), which turns every
// later kernel of the device-resident EM loop into a no-op.
constexpr int kEmDone = -4, kEmPending = -3, kEmCount = -2;

__device__ __forceinline__ bool em_skipped(const uint32_t* unconv) {
  return unconv && unconv[kEmDone] != 0;
}

__device__ __forceinline__ bool map_iter_skipped(const uint32_t* unconv, int t, int fixed) {
  // optimize.cpp:59 -- the MAP loop stops after an iteration whose flags are
  // all set.  Iteration t runs iff no earlier iteration had zero unconverged
  // hoods; skipped iterations leave their counter at 0 so the chain holds.
  return unconv[kEmDone] != 0 || (!fixed && t > 0 && unconv[t - 1] == 0);
}

// Label histogram of this block's 256 new labels -> out[0..M) (the M-step's
// per-tile counts; M == 2 needs just two block-wide counts).  Every thread
// of the block must call it.
__device__ __forceinline__ void block_label_counts(uint32_t* __restrict__ out, uint32_t M,
                                                   bool valid, uint32_t label) {
  if (M == 2) {
    const int ones = __syncthreads_count(valid && label == 1u);
    const int all = __syncthreads_count(valid);
    if (threadIdx.x == 0) {
      out[0] = uint32_t(all - ones);
      out[1] = uint32_t(ones);
    }
    return;
  }
  __shared__ uint32_t hist[kMaxLabels + 1];
  for (uint32_t i = threadIdx.x; i < M; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  if (valid) atomicAdd(&hist[label], 1u);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < M; i += blockDim.x) out[i] = hist[i];
  __syncthreads();
}

constexpr int kTileThreads = 256;
constexpr int kTileVerts = kTileThreads;  // == kVtxThreads: vertex blocks are label tiles

__device__ __forceinline__ int executed_iters(const uint32_t* unconv, int map_max, int fixed) {
  if (fixed) return map_max;
  for (int t = 0; t < map_max; ++t)
    if (unconv[t] == 0) return t + 1;
  return map_max;
}

// The same number, read while the hood pass of the last iteration is still
// running (the tail blocks of the last fused launch): iteration map_max-1 ran
// unless an earlier counter was zero, and the loop ends after it either way,
// so its own (in-flight) counter is never needed.
__device__ __forceinline__ int executed_iters_known(const uint32_t* unconv, int map_max,
                                                    int fixed) {
  if (fixed) return map_max;
  for (int t = 0; t + 1 < map_max; ++t)
    if (unconv[t] == 0) return t + 1;
  return map_max;
}

template <bool kKnown = false>
__device__ __forceinline__ int final_iters(const uint32_t* unconv, int map_max, int fixed) {
  return kKnown ? executed_iters_known(unconv, map_max, fixed)
                : executed_iters(unconv, map_max, fixed);
}

template <bool kKnown = false>
__device__ __forceinline__ const uint8_t* final_labels(const uint8_t* even, const uint8_t* odd,
                                                       const uint32_t* unconv, int map_max,
                                                       int fixed) {
  if (!unconv) return even;
  return (final_iters<kKnown>(unconv, map_max, fixed) & 1) ? odd : even;
}

// Counts of the final labels per 256-vertex tile: the buffer written by the
// last executed vertex pass (iteration T-1 -> slot (T-1)&1), or slot 0 when
// the counts were produced by k_label_tiles<0> (standalone update_parameters).
template <bool kKnown = false>
__device__ __forceinline__ const uint32_t* final_counts(const uint32_t* counts, uint32_t tiles,
                                                        uint32_t M, const uint32_t* unconv,
                                                        int map_max, int fixed) {
  if (!unconv) return counts;
  const int T = final_iters<kKnown>(unconv, map_max, fixed);
  return counts + uint64_t((T - 1) & 1) * tiles * M;
}


// Small graphs (tiles * M <= kSelfScanMax): k_tile_offsets folded into the
// scatter -- every block sums the label counts of the tiles before it (and of
// all tiles, for the label starts) itself, block 0 publishes the layout.
// One launch less per EM iteration where launches, not bytes, dominate.
constexpr uint32_t kSelfScanMax = 8192;

// smem: [kWarps x M] | base[M] | start[M] | red[2 kWarps]
inline size_t scatter_small_smem(uint32_t M) {
  return ((kTileThreads / 32) * M + 2 * M + 2 * (kTileThreads / 32)) * sizeof(uint32_t);
}

template <bool kKnown>
__device__ __forceinline__ void label_scatter_small_body(
    const uint8_t* lab_even, const uint8_t* lab_odd, const uint32_t* unconv,
    const uint32_t* count_sel, int map_max, int fixed, uint32_t R, uint32_t M, uint64_t Hs,
    const double* __restrict__ mean, const uint32_t* __restrict__ counts_buf, uint32_t tiles,
    uint32_t* __restrict__ layout, double* __restrict__ x, uint32_t tile, uint32_t* wcnt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kWarps = kTileThreads / 32;
  uint32_t* base_s = wcnt + kWarps * M;
  uint32_t* start_s = base_s + M;
  uint32_t* red = start_s + M;
  const uint32_t* tc = final_counts<kKnown>(counts_buf, tiles, M, count_sel, map_max, fixed);
  for (uint32_t l = 0; l < M; ++l) {  // prefix (tiles before this one) and total of label l
    uint32_t pre = 0, tot = 0;
    for (uint32_t i = threadIdx.x; i < tiles; i += kTileThreads) {
      const uint32_t c = tc[uint64_t(i) * M + l];
      tot += c;
      pre += i < tile ? c : 0u;
    }
    pre = __reduce_add_sync(0xffffffffu, pre);
    tot = __reduce_add_sync(0xffffffffu, tot);
    if (lane == 0) {
      red[warp] = pre;
      red[kWarps + warp] = tot;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t p = 0, q = 0;
      for (int w = 0; w < kWarps; ++w) {
        p += red[w];
        q += red[kWarps + w];
      }
      base_s[l] = p;
      start_s[l] = q;  // (total; turned into label starts below)
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    uint32_t s = 0, lf = 0;
    for (uint32_t l = 0; l < M; ++l) {
      const uint32_t n = start_s[l];
      if (tile == 0) {
        layout[l] = n;
        layout[M + l] = s;
        layout[2 * M + 1 + l] = lf;
      }
      start_s[l] = s;
      s += n;
      lf += (n + kFoldLeaf - 1) / kFoldLeaf;
    }
    if (tile == 0) {
      layout[2 * M] = s;
      layout[3 * M + 1] = lf;
      layout[3 * M + 2] = lf + uint32_t((Hs + kFoldLeaf - 1) / kFoldLeaf);
    }
  }
  const uint8_t* lab = final_labels<kKnown>(lab_even, lab_odd, unconv, map_max, fixed);
  for (uint32_t i = threadIdx.x; i < kWarps * M; i += kTileThreads) wcnt[i] = 0;
  __syncthreads();
  const uint64_t v = uint64_t(tile) * kTileVerts + threadIdx.x;
  const bool valid = v < R;
  const uint32_t l = valid ? lab[v] : 0xFFFFFFFFu;
  const unsigned peers = __match_any_sync(0xffffffffu, l);
  const uint32_t rank_in_warp = __popc(peers & ((1u << lane) - 1u));
  if (valid && rank_in_warp == 0) wcnt[warp * M + l] = __popc(peers);
  __syncthreads();
  if (valid) {
    uint32_t before = 0;
    for (int w = 0; w < warp; ++w) before += wcnt[w * M + l];
    x[start_s[l] + base_s[l] + before + rank_in_warp] = mean[v];
  }
}


}  // namespace
}  // namespace dpmrf_b200
