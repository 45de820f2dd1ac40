// fold_trees.cuh -- the pairwise tree of dpp::fold_range (kernels.hpp:45-51)
// over leaf partials, on the device (internal; engine.cu's M-step folds).
// Bottom-up adjacent pairing with an odd last element carried up unchanged
// == the reference's split at bit_floor(n-1); every node covers an aligned
// power-of-two block, so a block's own tree is exactly a node of the whole
// tree and the levels can be split across registers, lanes, warps.
#pragma once

#include "common.cuh"

namespace dpmrf_b200 {

constexpr uint32_t kTreeChunk = 1024;  // a chunk's root == the level-10 node

// The pairwise tree of kernels.hpp:45-51 (bottom-up adjacent pairing, an odd
// last element carried up unchanged == the split at bit_floor(n-1)) over
// e[0, r) in registers (B a power of two, r <= B); the root ends in e[0].
template <int B>
__device__ __forceinline__ double regs_tree(double (&e)[B], uint32_t r) {
#pragma unroll
  for (int w = B; w > 1; w /= 2) {
    const uint32_t pr = r / 2;
#pragma unroll
    for (int j = 0; j < w / 2; ++j) {
      const double s = __dadd_rn(e[2 * j], e[2 * j + 1]);
      e[j] = uint32_t(j) < pr ? s : ((uint32_t(j) == pr && (r & 1u)) ? e[2 * j] : e[j]);
    }
    r = pr + (r & 1u);
  }
  return e[0];
}


__device__ __forceinline__ double lanes_tree(double v, uint32_t m) {
  const uint32_t lane = threadIdx.x & 31;
  while (m > 1) {
    const uint32_t pr = m / 2;
    const double a = __shfl_sync(0xffffffffu, v, (2 * lane) & 31);
    const double b = __shfl_sync(0xffffffffu, v, (2 * lane + 1) & 31);
    const double c = __shfl_sync(0xffffffffu, v, (m - 1) & 31);
    v = lane < pr ? __dadd_rn(a, b) : ((lane == pr && (m & 1u)) ? c : v);
    m = pr + (m & 1u);
  }
  return __shfl_sync(0xffffffffu, v, 0);
}

// cnt <= 32 * B: lane l holds the aligned block p[l*B, l*B + B) (a warp
// reads one contiguous span); the block's own tree is exactly a node of the
// series' tree, so the lanes reduce their blocks in registers and the <= 32
// block roots finish with shuffles.
template <int B, bool kGlobal>
__device__ __forceinline__ double warp_tree_regs(const double* p, uint32_t cnt) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t lo = lane * B;
  const uint32_t r = cnt > lo ? min(cnt - lo, uint32_t(B)) : 0u;
  double e[B];
#pragma unroll
  for (int k = 0; k < B; ++k)
    e[k] = uint32_t(k) < r ? (kGlobal ? __ldcg(p + lo + k) : p[lo + k]) : 0.0;
  return lanes_tree(regs_tree<B>(e, r), (cnt + B - 1) / B);
}

// Root of the tree over p[0, cnt), 1 <= cnt <= 1024 (kGlobal: p in global
// memory, read through L2), by one warp; every lane gets it.  Up to 256
// elements straight into registers; beyond, coalesced into the warp's
// shared scratch q (kTreeScratch doubles, rows padded to 33) and back out as
// one aligned 32-block per lane.
constexpr uint32_t kTreeScratch = 32 * 33;

template <bool kGlobal>
__device__ double warp_tree(const double* p, uint32_t cnt, double* q) {
  if (cnt <= 32) return warp_tree_regs<1, kGlobal>(p, cnt);
  if (cnt <= 64) return warp_tree_regs<2, kGlobal>(p, cnt);
  if (cnt <= 128) return warp_tree_regs<4, kGlobal>(p, cnt);
  if (cnt <= 256) return warp_tree_regs<8, kGlobal>(p, cnt);
  const uint32_t lane = threadIdx.x & 31;
  {
    double t[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) {  // (all loads in flight at once)
      const uint32_t j = uint32_t(k) * 32 + lane;
      t[k] = j < cnt ? (kGlobal ? __ldcg(p + j) : p[j]) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 32; ++k) q[k * 33 + lane] = t[k];  // element 32k + l of block k
  }
  __syncwarp();
  const uint32_t lo = lane * 32;
  const uint32_t r = cnt > lo ? min(cnt - lo, 32u) : 0u;
  double e[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) e[k] = q[lane * 33 + k];
  __syncwarp();
  return lanes_tree(regs_tree<32>(e, r), (cnt + 31) / 32);
}

// warp_tree for cnt <= 512 without scratch: up to 16 partials per lane in
// registers (the same aligned blocks, so the same tree).
template <bool kGlobal>
__device__ __forceinline__ double warp_tree512(const double* p, uint32_t cnt) {
  if (cnt <= 32) return warp_tree_regs<1, kGlobal>(p, cnt);
  if (cnt <= 64) return warp_tree_regs<2, kGlobal>(p, cnt);
  if (cnt <= 128) return warp_tree_regs<4, kGlobal>(p, cnt);
  if (cnt <= 256) return warp_tree_regs<8, kGlobal>(p, cnt);
  return warp_tree_regs<16, kGlobal>(p, cnt);
}

// warp_tree for cnt <= 1024 without scratch: the two aligned 512-halves are
// the level-9 nodes, paired at level 10 when both exist.
template <bool kGlobal>
__device__ __forceinline__ double warp_tree1024(const double* p, uint32_t cnt) {
  if (cnt <= 512) return warp_tree512<kGlobal>(p, cnt);
  const double lo = warp_tree512<kGlobal>(p, 512);
  return __dadd_rn(lo, warp_tree512<kGlobal>(p + 512, cnt - 512));
}

// The whole series' tree by the block: aligned 1024-partial chunks (a
// chunk's root is exactly the level-10 node of the series' tree) by the
// warps in parallel, roots in shared memory, then the tree over the roots
// (in 1024-root chunks again if needed; roots holds >= ceil(cnt/1024)).
// Called by every thread; returns the root to every thread.
__device__ double block_series_tree(const double* __restrict__ p, uint32_t cnt, double* roots,
                                    double* qw) {
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (cnt <= kTreeChunk) {  // one warp; the block takes it from shared memory
    if (warp == 0) {
      const double r = warp_tree<true>(p, cnt, qw);
      if (lane == 0) roots[0] = r;
    }
  } else {
    uint32_t nch = (cnt + kTreeChunk - 1) / kTreeChunk;
    for (uint32_t c = warp; c < nch; c += nw) {
      const double r =
          warp_tree<true>(p + uint64_t(c) * kTreeChunk, min(kTreeChunk, cnt - c * kTreeChunk), qw);
      if (lane == 0) roots[c] = r;
    }
    __syncthreads();
    while (nch > 1) {  // roots of roots: aligned 1024-chunks again
      const uint32_t nn = (nch + kTreeChunk - 1) / kTreeChunk;
      double r = 0.0;
      if (warp < nn)
        r = warp_tree<false>(roots + warp * kTreeChunk, min(kTreeChunk, nch - warp * kTreeChunk), qw);
      __syncthreads();
      if (warp < nn && lane == 0) roots[warp] = r;
      __syncthreads();
      nch = nn;
    }
  }
  __syncthreads();
  const double r = roots[0];
  __syncthreads();
  return r;
}

}  // namespace dpmrf_b200
