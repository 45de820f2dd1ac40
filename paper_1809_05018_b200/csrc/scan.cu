// scan.cu -- three-phase (reduce / scan-of-partials / downsweep) device scan.
#include "scan.cuh"

namespace dpmrf_b200 {

namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kTile = kScanThreads * kScanItems;  // 2048 elements per block

__global__ void __launch_bounds__(kScanThreads) k_tile_sums(const uint32_t* __restrict__ in,
                                                            uint64_t n, uint32_t* __restrict__ sums) {
  __shared__ uint32_t warp_sums[kScanThreads / 32];
  const uint64_t base = uint64_t(blockIdx.x) * kTile;
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t idx = base + uint64_t(i) * kScanThreads + threadIdx.x;
    if (idx < n) acc += in[idx];
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) warp_sums[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t w = threadIdx.x < kScanThreads / 32 ? warp_sums[threadIdx.x] : 0u;
    for (int o = 16; o > 0; o >>= 1) w += __shfl_down_sync(0xffffffffu, w, o);
    if (threadIdx.x == 0) sums[blockIdx.x] = w;
  }
}

// Scans one tile per block; each thread owns kScanItems CONSECUTIVE elements.
__global__ void __launch_bounds__(kScanThreads) k_tile_scan(const uint32_t* in, uint32_t* out,
                                                            uint64_t n,
                                                            const uint32_t* __restrict__ tile_base,
                                                            uint32_t* total) {
  __shared__ uint32_t warp_sums[kScanThreads / 32];
  const uint64_t base = uint64_t(blockIdx.x) * kTile + uint64_t(threadIdx.x) * kScanItems;
  uint32_t v[kScanItems];
  uint32_t local = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t idx = base + i;
    v[i] = idx < n ? in[idx] : 0u;
    local += v[i];
  }
  uint32_t block_total;
  uint32_t run = block_exclusive_scan(local, warp_sums, &block_total);
  if (tile_base) run += tile_base[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t idx = base + i;
    if (idx < n) out[idx] = run;
    run += v[i];
  }
  if (total && blockIdx.x == gridDim.x - 1 && threadIdx.x == kScanThreads - 1) *total = run;
}

void scan_level(const uint32_t* in, uint32_t* out, uint64_t n, uint32_t* total, ScanWorkspace& ws,
                int depth, cudaStream_t stream) {
  const uint64_t tiles = (n + kTile - 1) / kTile;
  if (tiles <= 1) {
    k_tile_scan<<<1, kScanThreads, 0, stream>>>(in, out, n, nullptr, total);
    CK_LAUNCH();
    return;
  }
  if (depth >= 4) fail(DPMRF_INTERNAL_ERROR, "scan: input too large");
  uint32_t* sums = ws.level[depth].ensure(tiles);
  k_tile_sums<<<grid_for(tiles, 1), kScanThreads, 0, stream>>>(in, n, sums);
  CK_LAUNCH();
  scan_level(sums, sums, tiles, nullptr, ws, depth + 1, stream);
  k_tile_scan<<<static_cast<unsigned>(tiles), kScanThreads, 0, stream>>>(in, out, n, sums, total);
  CK_LAUNCH();
}

}  // namespace

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, uint32_t* total,
                        ScanWorkspace& ws, cudaStream_t stream) {
  if (n == 0) {
    if (total) CK(cudaMemsetAsync(total, 0, sizeof(uint32_t), stream));
    return;
  }
  scan_level(in, out, n, total, ws, 0, stream);
}

}  // namespace dpmrf_b200
