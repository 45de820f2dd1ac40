// labelmap.cu -- validate_label_map (proj/src/graph/label_map.cpp:38-78) on
// the device, for the label maps that feed build_region_graph (SURVEY.md
// section 8(f) item 4: the RLM1 reader validates every map it reads).
//
// The reference checks (1) every id in [0, max] is used -- reporting the
// lowest unused id -- and (2) each region is one 4-connected component -- a
// serial union-find over same-id right / down pixel pairs, then a scan that
// reports the region of the first pixel whose root differs from its
// region's first root.  Here: a lock-free union-find over the pixel grid
// (parents only ever point to smaller indices; a union links the larger root
// under the smaller with atomicMin and retries on contention), a flattening
// pass, and two min-reductions that name exactly the id / pixel the
// reference's scans would reach first (the first pixel in scan order that is
// not in its region's first pixel's component does not depend on how the
// union-find picked its roots), so the error messages match.
#include <algorithm>
#include <string>

#include "context.cuh"

namespace dpmrf_b200 {
namespace {

constexpr int kLmThreads = 256;

__global__ void k_lm_init(const uint32_t* __restrict__ region, uint64_t n, uint32_t* parent,
                          uint32_t* max_id) {
  uint32_t m = 0;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    parent[i] = uint32_t(i);
    m = max(m, region[i]);
  }
  m = __reduce_max_sync(0xFFFFFFFFu, m);
  if ((threadIdx.x & 31) == 0) atomicMax(max_id, m);
}

// used[id] for ids < nused (ids beyond n cannot all be used: see the host).
__global__ void k_lm_used(const uint32_t* __restrict__ region, uint64_t n, uint8_t* used,
                          uint64_t nused) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t id = region[i];
    if (id < nused) used[id] = 1;
  }
}

__global__ void k_lm_lowest_unused(const uint8_t* __restrict__ used, uint64_t nused,
                                   uint32_t* lowest) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nused; i += stride)
    if (!used[i]) atomicMin(lowest, uint32_t(i));
}

// Path halving during the unions: the shortcut is written with atomicMin, so
// a parent only ever decreases and never undoes a concurrent relink (every
// relinked node's old parent is united with its new one by the relinking
// thread, so shortcuts stay inside the node's final set).
__device__ __forceinline__ uint32_t lm_find(uint32_t* parent, uint32_t x) {
  for (;;) {
    const uint32_t p = __ldcg(parent + x);
    if (p == x) return x;
    const uint32_t g = __ldcg(parent + p);
    if (g != p) atomicMin(parent + x, g);
    x = g;
  }
}

// Read-only root walk (the flattening pass: each thread rewrites only its own
// entry, to its root, so a concurrent walk through it still ends at a root).
__device__ __forceinline__ uint32_t lm_root(const uint32_t* parent, uint32_t x) {
  for (;;) {
    const uint32_t p = __ldcg(parent + x);
    if (p == x) return x;
    x = p;
  }
}

__device__ __forceinline__ void lm_unite(uint32_t* parent, uint32_t a, uint32_t b) {
  for (;;) {
    a = lm_find(parent, a);
    b = lm_find(parent, b);
    if (a == b) return;
    if (a > b) {
      const uint32_t t = a;
      a = b;
      b = t;
    }
    const uint32_t old = atomicMin(parent + b, a);
    if (old == b) return;  // b was a root and now hangs under a
    b = old;               // b was linked meanwhile: retry from there
  }
}

__global__ void k_lm_union(const uint32_t* __restrict__ region, uint32_t w, uint32_t h,
                           uint32_t* parent) {
  const uint64_t n = uint64_t(w) * h;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t x = uint32_t(i % w), y = uint32_t(i / w);
    const uint32_t id = region[i];
    if (x + 1 < w && region[i + 1] == id) lm_unite(parent, uint32_t(i), uint32_t(i + 1));
    if (y + 1 < h && region[i + w] == id) lm_unite(parent, uint32_t(i), uint32_t(i + w));
  }
}

// roots, and each region's first pixel (scan order)
__global__ void k_lm_flatten(const uint32_t* __restrict__ region, uint64_t n, uint32_t* parent,
                             uint32_t* first) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    parent[i] = lm_root(parent, uint32_t(i));
    atomicMin(first + region[i], uint32_t(i));
  }
}

// the first pixel (scan order) outside its region's first pixel's component
__global__ void k_lm_check(const uint32_t* __restrict__ region, uint64_t n,
                           const uint32_t* __restrict__ parent, const uint32_t* __restrict__ first,
                           uint32_t* bad) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    if (parent[i] != parent[first[region[i]]]) atomicMin(bad, uint32_t(i));
}

unsigned lm_grid(uint64_t n) {
  return unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n + kLmThreads - 1) / kLmThreads,
                                                           uint64_t(16) * kNumSMs)));
}

}  // namespace

uint32_t validate_label_map_device(dpmrf_context* ctx, uint32_t w, uint32_t h,
                                   const uint32_t* region) {
  const uint64_t n = uint64_t(w) * h;
  if (n == 0) fail(DPMRF_INPUT_ERROR, "label map: empty");
  if (n > 0xFFFFFFFFull) fail(DPMRF_INPUT_ERROR, "label map: too large");
  cudaStream_t s = ctx->stream;
  uint32_t* parent = ctx->lm_parent.ensure(n);
  uint32_t* st = ctx->lm_state.ensure(4);  // max id, lowest unused, first bad pixel
  const uint32_t init[4] = {0u, 0xFFFFFFFFu, 0xFFFFFFFFu, 0u};
  CK(cudaMemcpyAsync(st, init, sizeof init, cudaMemcpyHostToDevice, s));
  k_lm_init<<<lm_grid(n), kLmThreads, 0, s>>>(region, n, parent, st);
  CK_LAUNCH();
  uint32_t max_id = 0;
  CK(cudaMemcpyAsync(&max_id, st, 4, cudaMemcpyDeviceToHost, s));
  ctx->sync();
  const uint64_t num = uint64_t(max_id) + 1;
  // n pixels use at most n ids: with num > n some id <= n is unused, so the
  // lowest unused id is found among the first min(num, n + 1)
  const uint64_t nused = std::min<uint64_t>(num, n + 1);
  uint8_t* used = ctx->lm_used.ensure(nused);
  CK(cudaMemsetAsync(used, 0, nused, s));
  k_lm_used<<<lm_grid(n), kLmThreads, 0, s>>>(region, n, used, nused);
  CK_LAUNCH();
  k_lm_lowest_unused<<<lm_grid(nused), kLmThreads, 0, s>>>(used, nused, st + 1);
  CK_LAUNCH();
  uint32_t lowest = 0xFFFFFFFFu;
  CK(cudaMemcpyAsync(&lowest, st + 1, 4, cudaMemcpyDeviceToHost, s));
  ctx->sync();
  if (lowest != 0xFFFFFFFFu)
    fail(DPMRF_INPUT_ERROR, "label map: region id " + std::to_string(lowest) + " unused");
  // every id < num is used, so num <= n
  uint32_t* first = ctx->lm_first.ensure(num);
  CK(cudaMemsetAsync(first, 0xFF, num * sizeof(uint32_t), s));
  k_lm_union<<<lm_grid(n), kLmThreads, 0, s>>>(region, w, h, parent);
  CK_LAUNCH();
  k_lm_flatten<<<lm_grid(n), kLmThreads, 0, s>>>(region, n, parent, first);
  CK_LAUNCH();
  k_lm_check<<<lm_grid(n), kLmThreads, 0, s>>>(region, n, parent, first, st + 2);
  CK_LAUNCH();
  uint32_t bad = 0xFFFFFFFFu;
  CK(cudaMemcpyAsync(&bad, st + 2, 4, cudaMemcpyDeviceToHost, s));
  ctx->sync();
  if (bad != 0xFFFFFFFFu) {
    uint32_t id = 0;
    CK(cudaMemcpy(&id, region + bad, 4, cudaMemcpyDeviceToHost));
    fail(DPMRF_INPUT_ERROR, "label map: region " + std::to_string(id) + " is not 4-connected");
  }
  return uint32_t(num);
}

}  // namespace dpmrf_b200
