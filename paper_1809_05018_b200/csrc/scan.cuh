// scan.cuh -- device-wide exclusive scan of u32 (offsets_from_counts /
// scan_exclusive of proj/include/dpmrf/dpp/kernels.hpp:144-173, :351-357).
// Integer scans are exact, so any combination order reproduces the
// reference's wrap-around u32 recurrence bit for bit.
#pragma once

#include "common.cuh"

namespace dpmrf_b200 {

// Reusable scratch for the multi-level scan.
struct ScanWorkspace {
  DevBuf<uint32_t> level[4];
};

// out[i] = sum(in[0..i)), out may alias in.  If total != nullptr, *total
// (device pointer) receives the full sum.  n may be 0.
void exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, uint32_t* total,
                        ScanWorkspace& ws, cudaStream_t stream);

// Block-wide exclusive scan helper for kernels (blockDim.x multiple of 32, <= 1024).
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* smem_warp,
                                                         uint32_t* block_total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < nw ? smem_warp[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) smem_warp[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  const uint32_t warp_base = warp ? smem_warp[warp - 1] : 0u;
  if (block_total) *block_total = smem_warp[nw - 1];
  const uint32_t r = warp_base + x - v;
  __syncthreads();
  return r;
}

}  // namespace dpmrf_b200
