// partition.cu -- vertex-range partitioned optimize (one giant slice over
// several GPUs).
//
// The reference runs optimize() (proj/src/mrf/optimize.cpp:31-74) over one
// address space.  Here the region graph is cut into `world` contiguous vertex
// ranges (row bands of the superpixel grid; multiples of the 256-vertex tile)
// and the series (nonempty hoods) into as many contiguous ranges.  Every
// partition keeps the whole static structure resident (it is small next to
// 180 GB) and the per-vertex / per-series arrays globally indexed, but runs
// the MAP kernels only over what it owns:
//
//   per MAP iteration t        vertex pass (own vertices)
//                              halo: labels + minima its neighbors' owners /
//                                    hoods need (exact [lo, hi] windows per
//                                    (source, destination) pair, planned once)
//                              hood pass (own series; NCCL groups fold the
//                                    interior series while the halo exchange
//                                    runs on a side stream, the boundary
//                                    series after it)
//                              sum of the unconverged-hood counters
//   per EM iteration           distributed M-step (k_part_*): own label
//                              counts -> allgather; own vertices scattered
//                              into their segments of the label-grouped x;
//                              head fragments (<= 1023 values per label) ->
//                              allgather; own leaves folded (both passes),
//                              leaf partials -> allgather; the same trees
//                              and EM bookkeeping on every rank.  The own
//                              hood-series leaves (the row folded into
//                              1024-element leaves on the rank that owns
//                              them) -> allgather.
//   after the EM loop          the labels, gathered once.
//
// Everything runs in stream order with the device-side early exit of the
// single-GPU path (skipped iterations still move their -- stale but never
// read -- halos, so the schedule is static and capturable).  Every leaf is
// folded whole, in order, on one rank and every tree sees the same partials,
// so the results are bit-identical to dpmrf_optimize.  Per EM at 16384^2 / 8
// ranks a rank receives ~0.3 MB (counts, 16 KB of heads per rank, leaf
// partials) instead of the 5.5 MB label gather plus a full-R regroup.
//
// Transports: NCCL (one process per GPU; libnccl.so.2 loaded at run time,
// grouped ncclSend/ncclRecv for the halos, ncclAllReduce for the counters,
// in-place ncclAllGather per EM) or local (all partitions in one context on
// one device; device-to-device copies and a counter-sum kernel -- the same
// schedule without NVLink, which is how one GPU tests the partition logic).
#include <dlfcn.h>
#include <cstdlib>
#include <nccl.h>  // types and enums only; every symbol comes from dlsym

#include <algorithm>
#include <cmath>
#include <functional>
#include <initializer_list>
#include <cstring>
#include <memory>
#include <vector>

#include "context.cuh"
#include "scan.cuh"

using namespace dpmrf_b200;

void dpmrf_b200_set_error(const char* msg);

namespace {

constexpr int kMaxParts = 64;

// ---- NCCL, resolved at run time ------------------------------------------------
struct Nccl {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;

  static Nccl& get() {
    static Nccl n;
    if (!n.lib) n.load();
    return n;
  }
  void load() {
    // DPMRF_NCCL_LIB: another library with the same entry points (the test
    // suite's in-process multi-rank shim, tests/nccl_shim).  RTLD_LOCAL: the
    // symbols are used through dlsym only, and must not shadow the NCCL a
    // later-loaded library (libtorch_cuda) links against.
    const char* alt = std::getenv("DPMRF_NCCL_LIB");
    // an NCCL the process already loaded (e.g. by PyTorch) is reused as is
    void* h = alt && alt[0] ? dlopen(alt, RTLD_NOW | RTLD_LOCAL)
                            : dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL | RTLD_NOLOAD);
    if (!h && !(alt && alt[0])) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h && !(alt && alt[0])) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) fail(DPMRF_NCCL_ERROR, std::string("cannot load libnccl.so.2: ") + dlerror());
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p) fail(DPMRF_NCCL_ERROR, std::string("libnccl.so.2 lacks ") + name);
      return p;
    };
    GetUniqueId = reinterpret_cast<decltype(GetUniqueId)>(sym("ncclGetUniqueId"));
    CommInitRank = reinterpret_cast<decltype(CommInitRank)>(sym("ncclCommInitRank"));
    CommDestroy = reinterpret_cast<decltype(CommDestroy)>(sym("ncclCommDestroy"));
    AllReduce = reinterpret_cast<decltype(AllReduce)>(sym("ncclAllReduce"));
    AllGather = reinterpret_cast<decltype(AllGather)>(sym("ncclAllGather"));
    Send = reinterpret_cast<decltype(Send)>(sym("ncclSend"));
    Recv = reinterpret_cast<decltype(Recv)>(sym("ncclRecv"));
    GroupStart = reinterpret_cast<decltype(GroupStart)>(sym("ncclGroupStart"));
    GroupEnd = reinterpret_cast<decltype(GroupEnd)>(sym("ncclGroupEnd"));
    GetErrorString = reinterpret_cast<decltype(GetErrorString)>(sym("ncclGetErrorString"));
    lib = h;
  }
  void check(ncclResult_t r, const char* what) const {
    if (r != ncclSuccess)
      fail(DPMRF_NCCL_ERROR, std::string(what) + " failed: " + GetErrorString(r));
  }
};
#define NK(call) nccl.check((call), #call)

// ---- halo plan ----------------------------------------------------------------------
struct Bounds {
  int W;
  uint32_t vb[kMaxParts + 1];
  uint64_t hb[kMaxParts + 1];
};

__device__ __forceinline__ int part_of_vertex(const Bounds& b, uint32_t v) {
  int lo = 0, hi = b.W - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (b.vb[mid] <= v) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ int part_of_series(const Bounds& b, uint64_t h) {
  int lo = 0, hi = b.W - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (b.hb[mid] <= h) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// win[(s * W + d) * 4 + {0,1}] = [lo, hi] of the source-s vertices whose labels
// destination d's vertex pass reads (discord over neighbors, engine.cpp:74-86);
// {2,3} = the source-s vertices whose minima d's hood pass folds.
__global__ void k_halo_plan(Bounds b, const uint32_t* __restrict__ g_off,
                            const uint32_t* __restrict__ g_nbr, uint32_t R,
                            const uint32_t* __restrict__ s_off, const uint32_t* __restrict__ h_mem,
                            uint64_t Hs, uint32_t* win) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  const uint64_t i0 = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (uint64_t v = i0; v < R; v += stride) {
    const int d = part_of_vertex(b, uint32_t(v));
    for (uint32_t a = g_off[v]; a < g_off[v + 1]; ++a) {
      const uint32_t u = g_nbr[a];
      const int s = part_of_vertex(b, u);
      if (s == d) continue;
      atomicMin(&win[(s * b.W + d) * 4 + 0], u);
      atomicMax(&win[(s * b.W + d) * 4 + 1], u);
    }
  }
  for (uint64_t h = i0; h < Hs; h += stride) {
    const int d = part_of_series(b, h);
    for (uint32_t j = s_off[h]; j < s_off[h + 1]; ++j) {
      const uint32_t m = h_mem[j];
      const int s = part_of_vertex(b, m);
      if (s == d) continue;
      atomicMin(&win[(s * b.W + d) * 4 + 2], m);
      atomicMax(&win[(s * b.W + d) * 4 + 3], m);
    }
  }
}

__global__ void k_win_init(uint32_t* win, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) win[i] = (i & 1) ? 0u : 0xFFFFFFFFu;
}

// Local transport: the sum of every partition's counter t, written back to all.
struct CounterPtrs {
  uint32_t* p[kMaxParts];
};
__global__ void k_sum_counters(CounterPtrs c, int W, int t) {
  pdl_wait();
  if (threadIdx.x != 0) return;
  uint32_t s = 0;
  for (int r = 0; r < W; ++r) s += c.p[r][t];
  for (int r = 0; r < W; ++r) c.p[r][t] = s;
}

// ---- distributed M-step ----------------------------------------------------------------
// update_parameters (engine.cpp:193-223) without gathering the labels: the
// label-grouped array x is the stable sort of ALL region means by label, so
// rank r's vertices form, per label l, the contiguous segment
// [label_start[l] + off_r[l], + n_r[l]) of x (off_r[l] = the counts of the
// ranks before it).  Each rank scatters its own vertices there, owns the
// 1024-element leaves of x that START in its segments, and folds them
// (fold_leaf, kernels.hpp:37-42) -- a leaf straddling into the next ranks'
// segments reads their "head" fragments (<= 1023 elements per label, up to
// the next leaf boundary), which are allgathered.  The leaf partials are
// allgathered too and every rank runs the same trees.  Per EM and rank this
// exchanges M counts, M x 1024 head values and its leaf partials instead of
// all R labels, and nobody regroups vertices it does not own.
constexpr uint32_t kPartLPB = 8;  // leaves per fold block (one chain per leaf)

// (the EM skip flag and the final-label buffer, as engine_dev.cuh's
// em_skipped / final_labels: unconv[-4] = EM loop stopped; the last executed
// MAP iteration T selects the buffer by parity)
__device__ __forceinline__ bool part_em_skipped(const uint32_t* unconv) {
  return unconv && unconv[-4] != 0;
}
__device__ __forceinline__ const uint8_t* part_final_labels(const uint8_t* even, const uint8_t* odd,
                                                            const uint32_t* unconv, int map_max,
                                                            int fixed) {
  int T = map_max;
  if (!fixed)
    for (int t = 0; t < map_max; ++t)
      if (unconv[t] == 0) {
        T = t + 1;
        break;
      }
  return (T & 1) ? odd : even;
}

// per-rank metadata written by k_part_layout (u32):
//   [0, M)   off_r[l]      this rank's offset inside label l's segment of x
//   [M, 2M)  own_first[l]  first owned leaf of label l (index within the label)
//   [2M,3M)  own_end[l]    one past the last owned leaf
//   [3M,4M)  own_base[l]   ordinal of own_first[l] among this rank's owned leaves
//   [4M]     owned leaves in total
__device__ __forceinline__ uint32_t head_len(uint32_t off, uint32_t n) {
  const uint32_t to_boundary = (kFoldLeaf - off % kFoldLeaf) % kFoldLeaf;
  return min(n, to_boundary);
}

// own label counts (stable tile ranks as k_label_counts) + per-tile counts
__global__ void __launch_bounds__(256)
    k_part_count(const uint8_t* lab_even, const uint8_t* lab_odd, const uint32_t* unconv,
                 int map_max, int fixed, uint32_t vb, uint32_t ve, uint32_t M,
                 uint32_t* __restrict__ tile_counts, uint32_t* __restrict__ cnt) {
  extern __shared__ uint32_t wcnt[];  // [warp][M]
  pdl_wait();
  if (part_em_skipped(unconv)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint8_t* lab = part_final_labels(lab_even, lab_odd, unconv, map_max, fixed);
  for (uint32_t i = threadIdx.x; i < 8 * M; i += 256) wcnt[i] = 0;
  __syncthreads();
  const uint32_t v = vb + blockIdx.x * 256 + threadIdx.x;
  const bool valid = v < ve;
  const uint32_t l = valid ? lab[v] : 0xFFFFFFFFu;
  const unsigned peers = __match_any_sync(0xffffffffu, l);
  if (valid && __popc(peers & ((1u << lane) - 1u)) == 0) wcnt[warp * M + l] = __popc(peers);
  __syncthreads();
  for (uint32_t q = threadIdx.x; q < M; q += 256) {
    uint32_t c = 0;
    for (int w = 0; w < 8; ++w) c += wcnt[w * M + q];
    tile_counts[uint64_t(blockIdx.x) * M + q] = c;
    if (c) atomicAdd(&cnt[q], c);
  }
}

// global layout (n | label_start | leaf_start, as the one-device M-step) and
// this rank's metadata, from the gathered counts allcnt[W][M]
__global__ void k_part_layout(const uint32_t* __restrict__ allcnt, int W, int r, uint32_t M,
                              uint64_t Hs, const uint32_t* unconv, uint32_t* __restrict__ layout,
                              uint32_t* __restrict__ meta) {
  pdl_wait();
  if (part_em_skipped(unconv) || threadIdx.x != 0) return;
  uint32_t* n = layout;
  uint32_t* label_start = layout + M;
  uint32_t* leaf_start = layout + 2 * M + 1;
  uint32_t s = 0, lf = 0, owned = 0;
  for (uint32_t l = 0; l < M; ++l) {
    uint32_t tot = 0, off = 0;
    for (int q = 0; q < W; ++q) {
      if (q < r) off += allcnt[q * M + l];
      tot += allcnt[q * M + l];
    }
    n[l] = tot;
    label_start[l] = s;
    leaf_start[l] = lf;
    s += tot;
    lf += (tot + kFoldLeaf - 1) / kFoldLeaf;
    const uint32_t mine = allcnt[r * M + l];
    // leaves j with off <= 1024 j < off + mine
    const uint32_t first = (off + kFoldLeaf - 1) / kFoldLeaf;
    const uint32_t end = mine ? (off + mine + kFoldLeaf - 1) / kFoldLeaf : first;
    meta[l] = off;
    meta[M + l] = first;
    meta[2 * M + l] = end > first ? end : first;
    meta[3 * M + l] = owned;
    owned += end > first ? end - first : 0;
  }
  label_start[M] = s;
  leaf_start[M] = lf;
  leaf_start[M + 1] = lf + uint32_t((Hs + kFoldLeaf - 1) / kFoldLeaf);
  meta[4 * M] = owned;
}

// x positions of this rank's tiles: label_start + off_r + the counts of its
// earlier tiles (one block, chunks of 1024 tiles)
__global__ void __launch_bounds__(1024)
    k_part_tile_base(const uint32_t* __restrict__ tile_counts, uint32_t tiles, uint32_t M,
                     const uint32_t* unconv, const uint32_t* __restrict__ layout,
                     const uint32_t* __restrict__ meta, uint32_t* __restrict__ tile_base) {
  __shared__ uint32_t warp_sums[32];
  __shared__ uint32_t carry_s;
  pdl_wait();
  if (part_em_skipped(unconv)) return;
  for (uint32_t l = 0; l < M; ++l) {
    uint32_t carry = layout[M + l] + meta[l];
    for (uint32_t c0 = 0; c0 < tiles; c0 += 1024) {
      const uint32_t i = c0 + threadIdx.x;
      const uint32_t v = i < tiles ? tile_counts[uint64_t(i) * M + l] : 0u;
      uint32_t total = 0;
      const uint32_t ex = block_exclusive_scan(v, warp_sums, &total);
      if (i < tiles) tile_base[uint64_t(i) * M + l] = carry + ex;
      carry += total;
      __syncthreads();
    }
  }
  (void)carry_s;
}

// stable scatter of this rank's region means into x, one WARP per 256-vertex
// tile (eight tiles per block), as k_label_scatter_warp (mstep.cu): the warp
// walks its tile in vertex order with running per-label counts in shared
// memory; tile_base holds each tile's absolute start per label
__global__ void __launch_bounds__(256)
    k_part_scatter(const uint8_t* lab_even, const uint8_t* lab_odd, const uint32_t* unconv,
                   int map_max, int fixed, uint32_t vb, uint32_t ve, uint32_t M,
                   const double* __restrict__ mean, const uint32_t* __restrict__ tile_base,
                   double* __restrict__ x) {
  extern __shared__ uint32_t run_all[];  // [warp][M]
  constexpr int kIters = 256 / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t tile = uint64_t(blockIdx.x) * 8 + warp;
  uint32_t* run = run_all + warp * M;
  for (uint32_t l = lane; l < M; l += 32) run[l] = 0;
  const uint64_t v0 = vb + tile * 256 + lane;
  double mv[kIters];
#pragma unroll
  for (int i = 0; i < kIters; ++i) {  // (means are static: before the wait)
    const uint64_t v = v0 + 32 * i;
    mv[i] = v < ve ? mean[v] : 0.0;
  }
  pdl_wait();
  if (part_em_skipped(unconv)) return;
  const uint8_t* lab = part_final_labels(lab_even, lab_odd, unconv, map_max, fixed);
  uint32_t lv[kIters];
#pragma unroll
  for (int i = 0; i < kIters; ++i) {
    const uint64_t v = v0 + 32 * i;
    lv[i] = v < ve ? lab[v] : 0xFFFFFFFFu;
  }
  const uint32_t* tb = tile_base + tile * M;
  __syncwarp();
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < kIters; ++i) {
    const uint32_t l = lv[i];
    const unsigned peers = __match_any_sync(0xffffffffu, l);
    const uint32_t rank = __popc(peers & lt);
    if (l != 0xFFFFFFFFu) x[tb[l] + run[l] + rank] = mv[i];
    __syncwarp();
    if (l != 0xFFFFFFFFu && rank == 0) run[l] += __popc(peers);
    __syncwarp();
  }
}

// this rank's head fragments -> heads[l * 1024 ...] (its allgather slot)
__global__ void k_part_pack_heads(const double* __restrict__ x, const uint32_t* unconv,
                                  const uint32_t* __restrict__ layout,
                                  const uint32_t* __restrict__ allcnt, int r, uint32_t M,
                                  const uint32_t* __restrict__ meta, double* __restrict__ heads) {
  pdl_wait();
  if (part_em_skipped(unconv)) return;
  for (uint32_t l = blockIdx.x; l < M; l += gridDim.x) {
    const uint32_t off = meta[l], len = head_len(off, allcnt[r * M + l]);
    const uint64_t base = uint64_t(layout[M + l]) + off;
    for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) heads[uint64_t(l) * kFoldLeaf + i] = x[base + i];
  }
}

// the later ranks' head fragments into x (the straddling leaves this rank owns)
__global__ void k_part_unpack_heads(const double* __restrict__ heads, const uint32_t* unconv,
                                    const uint32_t* __restrict__ layout,
                                    const uint32_t* __restrict__ allcnt, int W, int r, uint32_t M,
                                    double* __restrict__ x) {
  pdl_wait();
  if (part_em_skipped(unconv)) return;
  for (uint32_t ql = blockIdx.x; ql < uint32_t(W) * M; ql += gridDim.x) {
    const int q = int(ql / M);
    const uint32_t l = ql % M;
    if (q <= r) continue;
    uint32_t off = 0;
    for (int p = 0; p < q; ++p) off += allcnt[p * M + l];
    const uint32_t len = head_len(off, allcnt[q * M + l]);
    const uint64_t base = uint64_t(layout[M + l]) + off;
    const double* src = heads + (uint64_t(q) * M + l) * kFoldLeaf;
    for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) x[base + i] = src[i];
  }
}

// fold this rank's owned leaves (kSq: (x - mu)^2, engine.cpp:213-217) ->
// pk[ordinal] (the allgather slot) and partials[global leaf]
template <bool kSq>
__global__ void __launch_bounds__(256)
    k_part_fold(const double* __restrict__ x, const uint32_t* unconv,
                const uint32_t* __restrict__ layout, const uint32_t* __restrict__ meta,
                uint32_t M, const double* __restrict__ params, double* __restrict__ pk,
                double* __restrict__ partials) {
  extern __shared__ double stage[];  // kPartLPB x (kFoldLeaf + 1)
  __shared__ uint64_t src_s[kPartLPB];
  __shared__ uint32_t len_s[kPartLPB], leaf_s[kPartLPB];
  __shared__ double mu_s[kPartLPB];
  pdl_wait();
  if (part_em_skipped(unconv)) return;
  const uint32_t owned = meta[4 * M];
  const uint32_t o0 = blockIdx.x * kPartLPB;
  if (o0 >= owned) return;
  if (threadIdx.x < kPartLPB) {
    const uint32_t o = o0 + threadIdx.x;
    uint32_t len = 0;
    if (o < owned) {
      uint32_t l = 0;  // the label whose owned ordinals [own_base, + count) hold o
      while (o >= meta[3 * M + l] + (meta[2 * M + l] - meta[M + l])) ++l;
      const uint32_t j = meta[M + l] + (o - meta[3 * M + l]);
      const uint32_t n = layout[l];
      const uint64_t b = uint64_t(j) * kFoldLeaf;
      len = static_cast<uint32_t>(n - b < kFoldLeaf ? n - b : uint64_t(kFoldLeaf));
      src_s[threadIdx.x] = uint64_t(layout[M + l]) + b;
      leaf_s[threadIdx.x] = layout[2 * M + 1 + l] + j;
      mu_s[threadIdx.x] = kSq ? params[l] : 0.0;
    }
    len_s[threadIdx.x] = len;
  }
  __syncthreads();
  constexpr uint32_t kStride = kFoldLeaf + 1;
  for (uint32_t f = threadIdx.x; f < kPartLPB * kFoldLeaf; f += blockDim.x) {
    const uint32_t j = f / kFoldLeaf, i = f % kFoldLeaf;
    if (i < len_s[j]) {
      double v = __ldcg(x + src_s[j] + i);
      if (kSq) {
        const double d = __dsub_rn(v, mu_s[j]);
        v = __dmul_rn(d, d);
      }
      stage[j * kStride + i] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x < kPartLPB && len_s[threadIdx.x]) {
    const double* v = stage + threadIdx.x * kStride;
    double acc = v[0];
    for (uint32_t i = 1; i < len_s[threadIdx.x]; ++i) acc = __dadd_rn(acc, v[i]);
    pk[o0 + threadIdx.x] = acc;
    partials[leaf_s[threadIdx.x]] = acc;
  }
}

// every rank's owned-leaf partials (pk[q][ordinal]) -> partials[global leaf]
__global__ void k_part_unpack_partials(const double* __restrict__ pk, uint64_t chunk_l,
                                       const uint32_t* unconv, const uint32_t* __restrict__ layout,
                                       const uint32_t* __restrict__ allcnt, int W, int r,
                                       uint32_t M, double* __restrict__ partials) {
  pdl_wait();
  if (part_em_skipped(unconv)) return;
  for (int q = blockIdx.x; q < W; q += gridDim.x) {
    if (q == r) continue;
    uint32_t ord = 0;
    for (uint32_t l = 0; l < M; ++l) {
      uint32_t off = 0;
      for (int p = 0; p < q; ++p) off += allcnt[p * M + l];
      const uint32_t mine = allcnt[q * M + l];
      const uint32_t first = (off + kFoldLeaf - 1) / kFoldLeaf;
      const uint32_t end = mine ? (off + mine + kFoldLeaf - 1) / kFoldLeaf : first;
      const uint32_t cnt = end > first ? end - first : 0;
      for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x)
        partials[layout[2 * M + 1 + l] + first + i] = pk[uint64_t(q) * chunk_l + ord + i];
      ord += cnt;
    }
  }
}

// ---- per-partition device state ---------------------------------------------------
struct Part {
  int r = 0;
  uint32_t vb = 0, ve = 0;
  uint64_t hb = 0, he = 0;
  // [ia, ib) of the owned series: hoods whose members are all owned (their
  // hood pass runs while the halo exchange is in flight)
  uint64_t ia = 0, ib = 0;
  DevBuf<uint8_t> lab[2], lab_full;
  // hpart: the hood-energy series' leaf partials of every rank (W x chunkH/1024)
  DevBuf<double> minE, hist, hpart, params, em_out, terms, em_rec, em_hist;
  DevBuf<uint32_t> state;  // [em_done, pending, em_count, pad | unconv[map_max]]
  DevBuf<uint8_t> eq;      // equal-run counts of the window test (owned series)
  // distributed M-step: gathered label counts [W][M], this rank's metadata,
  // head fragments [W][M][1024], owned-leaf partials [W][chunk_l]
  DevBuf<uint32_t> allcnt, meta;
  DevBuf<double> heads, pk;
  MStepBuffers ms;
  MapArgs a{};
  EmEpilogueArgs ep{};
};

struct Window {
  uint32_t lo, hi;
  bool empty() const { return lo > hi; }
  uint64_t count() const { return empty() ? 0 : uint64_t(hi) - lo + 1; }
};

}  // namespace

struct dpmrf_group {
  dpmrf_context* ctx = nullptr;
  int world = 1;
  int rank = -1;  // -1: local group (every partition in this process)
  ncclComm_t comm = nullptr;
  std::vector<std::unique_ptr<Part>> parts;
  // plan (per structure generation)
  bool planned = false;
  uint64_t plan_gen = 0;
  uint32_t chunkV = 0;
  uint64_t chunkH = 0;
  std::vector<Window> lab_win, min_win;  // [s * W + d]
  uint64_t halo_bytes = 0, gather_bytes = 0;
  // halo exchange on its own stream, overlapping the interior hood pass
  cudaStream_t cs = nullptr;
  cudaEvent_t ev_v = nullptr, ev_x = nullptr;
  // split hood pass (interior during the exchange, boundary after): NCCL
  // groups; local groups only with DPMRF_GROUP_SPLIT=1 (one device gains
  // nothing from the overlap and pays two more launches per iteration)
  bool split = true;
  // CUDA graph of one EM iteration (device loop; local groups)
  bool use_graph = true;
  std::vector<uint64_t> graph_key;
  cudaGraphExec_t graph = nullptr;
  uint64_t graph_kernels = 0;
  void drop_graph() {
    if (graph) cudaGraphExecDestroy(graph);
    graph = nullptr;
    graph_key.clear();
  }
  bool local() const { return rank < 0; }
};

namespace {

template <class F>
dpmrf_status guarded(F&& f) {
  try {
    f();
    return DPMRF_OK;
  } catch (const Error& e) {
    dpmrf_b200_set_error(e.what());
    return e.status;
  } catch (const std::bad_alloc&) {
    dpmrf_b200_set_error("host allocation failed");
    return DPMRF_INTERNAL_ERROR;
  } catch (const std::exception& e) {
    dpmrf_b200_set_error(e.what());
    return DPMRF_INTERNAL_ERROR;
  }
}

void need(bool c, dpmrf_status s, const char* m) {
  if (!c) fail(s, m);
}

// The owned series whose members all lie in the owned vertex range form an
// interior range [ia, ib): every boundary hood below mid moves ia past it,
// every boundary hood at or above mid moves ib below it (exact for any
// partition shape; row bands give thin boundary strips at both ends).
__global__ void k_interior(const uint32_t* __restrict__ s_off, const uint32_t* __restrict__ h_mem,
                           uint32_t hb, uint32_t he, uint32_t vb, uint32_t ve, uint32_t* out) {
  const uint32_t mid = hb + (he - hb) / 2;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t h = hb + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; h < he; h += stride) {
    bool boundary = false;
    for (uint32_t j = s_off[h]; j < s_off[h + 1] && !boundary; ++j) {
      const uint32_t m = h_mem[j];
      boundary = m < vb || m >= ve;
    }
    if (!boundary) continue;
    if (h < mid) atomicMax(&out[0], uint32_t(h) + 1);
    else atomicMin(&out[1], uint32_t(h));
  }
}

// upper bound of the leaves a rank owns in the distributed M-step
uint64_t owned_leaf_cap(const dpmrf_group* g, uint32_t M) {
  return (uint64_t(g->chunkV) + kFoldLeaf - 1) / kFoldLeaf + M + 1;
}

// Ranges + halo windows for the context's current structure.
void plan(dpmrf_group* g) {
  dpmrf_context* ctx = g->ctx;
  ctx->prepare();
  if (g->planned && g->plan_gen == ctx->generation) return;
  const int W = g->world;
  const uint32_t R = ctx->R;
  const uint64_t Hs = ctx->Hs;
  // vertex ranges: equal multiples of the 256-vertex tile (row bands of the
  // row-major superpixel grid); series ranges: equal multiples of the
  // 1024-element fold leaf.  Equal chunks make the allgathers plain
  // in-place ncclAllGather calls (the last chunk is padded).
  const uint64_t cv = (uint64_t(R) + W - 1) / W;
  g->chunkV = static_cast<uint32_t>(std::max<uint64_t>(256, (cv + 255) / 256 * 256));
  const uint64_t ch = (Hs + W - 1) / W;
  g->chunkH = std::max<uint64_t>(kFoldLeaf, (ch + kFoldLeaf - 1) / kFoldLeaf * kFoldLeaf);
  Bounds b{};
  b.W = W;
  for (int r = 0; r <= W; ++r) {
    b.vb[r] = static_cast<uint32_t>(std::min<uint64_t>(uint64_t(r) * g->chunkV, R));
    b.hb[r] = std::min<uint64_t>(uint64_t(r) * g->chunkH, Hs);
  }
  for (auto& p : g->parts) {
    p->vb = b.vb[p->r];
    p->ve = b.vb[p->r + 1];
    p->hb = b.hb[p->r];
    p->he = b.hb[p->r + 1];
  }
  const int nwin = W * W * 4;
  uint32_t* win = ctx->tmp_u32[5].ensure(nwin);
  cudaStream_t st = ctx->stream;
  k_win_init<<<grid_for(nwin, 256), 256, 0, st>>>(win, nwin);
  CK_LAUNCH();
  const uint32_t* s_off = ctx->series_alias ? ctx->h_off.get() : ctx->s_off_buf.get();
  const uint64_t n = std::max<uint64_t>(R, Hs);
  const unsigned grid = std::min<unsigned>(grid_for(n ? n : 1, 256), 8 * kNumSMs);
  k_halo_plan<<<grid, 256, 0, st>>>(b, ctx->g_off.get(), ctx->g_nbr.get(), R, s_off,
                                    ctx->h_mem.get(), Hs, win);
  CK_LAUNCH();
  std::vector<uint32_t> hw(nwin);
  CK(cudaMemcpyAsync(hw.data(), win, nwin * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  ctx->sync();
  g->lab_win.assign(W * W, Window{1, 0});
  g->min_win.assign(W * W, Window{1, 0});
  g->halo_bytes = 0;
  for (int s = 0; s < W; ++s)
    for (int d = 0; d < W; ++d) {
      const int i = s * W + d;
      g->lab_win[i] = Window{hw[i * 4 + 0], hw[i * 4 + 1]};
      g->min_win[i] = Window{hw[i * 4 + 2], hw[i * 4 + 3]};
      if (g->local() || s == g->rank)
        g->halo_bytes += g->lab_win[i].count() + 8 * g->min_win[i].count();
    }
  const int mine = g->local() ? 0 : g->rank;
  (void)mine;
  // per EM and receiving rank (distributed M-step): the other ranks' label
  // counts, hood-series leaf partials, head fragments and owned-leaf
  // partials of both passes (the labels are gathered once per optimize)
  {
    const uint64_t M = ctx->trace_M ? ctx->trace_M : 2;
    const uint64_t per = 4 * M + 8 * (g->chunkH / kFoldLeaf) + 8 * M * kFoldLeaf +
                         2 * 8 * owned_leaf_cap(g, uint32_t(M));
    g->gather_bytes = (g->local() ? uint64_t(W) : 1) * (W - 1) * per;
  }
  // interior series ranges (one small D2H per partition, planning time only)
  {
    uint32_t* io = ctx->tmp_u32[4].ensure(2 * W);
    std::vector<uint32_t> init(2 * W);
    for (auto& pp : g->parts) {
      init[2 * pp->r] = uint32_t(pp->hb);
      init[2 * pp->r + 1] = uint32_t(pp->he);
    }
    CK(cudaMemcpyAsync(io, init.data(), init.size() * 4, cudaMemcpyHostToDevice, st));
    for (auto& pp : g->parts) {
      if (pp->he > pp->hb)
        k_interior<<<std::min<unsigned>(grid_for(pp->he - pp->hb, 256), 8 * kNumSMs), 256, 0, st>>>(
            s_off, ctx->h_mem.get(), uint32_t(pp->hb), uint32_t(pp->he), pp->vb, pp->ve,
            io + 2 * pp->r);
      CK_LAUNCH();
    }
    std::vector<uint32_t> res(2 * W);
    CK(cudaMemcpyAsync(res.data(), io, res.size() * 4, cudaMemcpyDeviceToHost, st));
    ctx->sync();
    for (auto& pp : g->parts) {
      pp->ia = res[2 * pp->r];
      pp->ib = std::max<uint64_t>(res[2 * pp->r + 1], pp->ia);
    }
  }
  g->planned = true;
  g->plan_gen = ctx->generation;
  g->drop_graph();
}

// ---- the schedule --------------------------------------------------------------
// Labels (u8, buffer b) and minima of iteration t's vertex pass to the
// partitions that read them.
void exchange_halo(dpmrf_group* g, int b, cudaStream_t st) {
  const int W = g->world;
  if (W == 1) return;
  if (g->local()) {
    for (int s = 0; s < W; ++s)
      for (int d = 0; d < W; ++d) {
        if (s == d) continue;
        const Window lw = g->lab_win[s * W + d], mw = g->min_win[s * W + d];
        Part& ps = *g->parts[s];
        Part& pd = *g->parts[d];
        if (!lw.empty())
          CK(cudaMemcpyAsync(pd.lab[b].get() + lw.lo, ps.lab[b].get() + lw.lo, lw.count(),
                             cudaMemcpyDeviceToDevice, st));
        if (!mw.empty())
          CK(cudaMemcpyAsync(pd.minE.get() + mw.lo, ps.minE.get() + mw.lo, 8 * mw.count(),
                             cudaMemcpyDeviceToDevice, st));
      }
    return;
  }
  Nccl& nccl = Nccl::get();
  Part& p = *g->parts[0];
  const int me = g->rank;
  NK(nccl.GroupStart());
  for (int o = 0; o < W; ++o) {
    if (o == me) continue;
    const Window ls = g->lab_win[me * W + o], ms = g->min_win[me * W + o];  // me -> o
    const Window lr = g->lab_win[o * W + me], mr = g->min_win[o * W + me];  // o -> me
    if (!ls.empty())
      NK(nccl.Send(p.lab[b].get() + ls.lo, ls.count(), ncclUint8, o, g->comm, st));
    if (!ms.empty())
      NK(nccl.Send(p.minE.get() + ms.lo, ms.count(), ncclFloat64, o, g->comm, st));
    if (!lr.empty())
      NK(nccl.Recv(p.lab[b].get() + lr.lo, lr.count(), ncclUint8, o, g->comm, st));
    if (!mr.empty())
      NK(nccl.Recv(p.minE.get() + mr.lo, mr.count(), ncclFloat64, o, g->comm, st));
  }
  NK(nccl.GroupEnd());
}

// Unconverged-hood counter of iteration t summed over the partitions, so the
// early exit (optimize.cpp:59) is decided on the whole slice.
void sum_counters(dpmrf_group* g, int t, cudaStream_t st, uint64_t* k) {
  const int W = g->world;
  if (W == 1) return;
  if (g->local()) {
    CounterPtrs c{};
    for (int r = 0; r < W; ++r) c.p[r] = g->parts[r]->a.unconv;
    launch_pdl(k_sum_counters, dim3(1), dim3(32), 0, st, c, W, t);
    ++*k;
    return;
  }
  Nccl& nccl = Nccl::get();
  uint32_t* u = g->parts[0]->a.unconv + t;
  NK(nccl.AllReduce(u, u, 1, ncclUint32, ncclSum, g->comm, st));
}

// Per-rank slots of `count` elements assembled on every partition: slot r of
// buf(part r) -> slot r of buf(every part) (in-place ncclAllGather; device
// copies on the local transport).  Several buffers go in one NCCL group.
struct SlotBuf {
  std::function<void*(Part&)> buf;
  uint64_t count;
  ncclDataType_t type;
  size_t elem;
};
void gather_slots(dpmrf_group* g, std::initializer_list<SlotBuf> bufs, cudaStream_t st) {
  const int W = g->world;
  if (W == 1) return;
  if (g->local()) {
    for (const SlotBuf& b : bufs)
      for (int sp = 0; sp < W; ++sp)
        for (int d = 0; d < W; ++d) {
          if (sp == d || !b.count) continue;
          const uint64_t bytes = b.count * b.elem;
          CK(cudaMemcpyAsync(static_cast<char*>(b.buf(*g->parts[d])) + sp * bytes,
                             static_cast<char*>(b.buf(*g->parts[sp])) + sp * bytes, bytes,
                             cudaMemcpyDeviceToDevice, st));
        }
    return;
  }
  Nccl& nccl = Nccl::get();
  Part& p = *g->parts[0];
  NK(nccl.GroupStart());
  for (const SlotBuf& b : bufs) {
    char* base = static_cast<char*>(b.buf(p));
    NK(nccl.AllGather(base + g->rank * b.count * b.elem, base, b.count, b.type, g->comm, st));
  }
  NK(nccl.GroupEnd());
}

bool run_partitioned(dpmrf_group* g, const dpmrf_optimizer_config* cfg, const dpmrf_run_options& o,
                     bool device_loop, uint32_t* labels_out, double* mu_out, double* sigma_out) {
  dpmrf_context* ctx = g->ctx;
  const int fixed = (o.flags & DPMRF_RUN_FIXED_WORK) ? 1 : 0;
  cudaStream_t st = ctx->stream;
  const uint32_t M = cfg->num_labels;
  const uint32_t R = ctx->R;
  const int L = cfg->convergence_window;
  const int map_max = cfg->map_max_iters;
  const int em_max = cfg->em_max_iters;
  const int W = g->world;

  ctx->trace.clear();
  ctx->trace_level = o.trace_level;
  ctx->trace_M = M;
  const uint32_t fallbacks = ctx->stats.device_log_fallbacks;
  ctx->stats = dpmrf_run_stats{};
  ctx->stats.device_log_fallbacks = fallbacks;
  ctx->stats.device_loop = device_loop;
  uint64_t launches = 0;

  std::vector<double> mu(M), sigma(M);
  initial_params(M, cfg->rng_seed, mu.data(), sigma.data());
  plan(g);  // (also prepares the structure)
  const uint64_t Hs = ctx->Hs;
  const uint64_t padV = uint64_t(g->chunkV) * W, padH = g->chunkH * W;
  const uint64_t rec_stride = 3 + 3 * uint64_t(M);
  const int ring = L + 1;
  const bool packed = !(o.flags & DPMRF_RUN_CSR);
  for (auto& pp : g->parts) {
    Part& p = *pp;
    p.lab[0].ensure(padV);
    p.lab[1].ensure(padV);
    p.lab_full.ensure(padV);
    MapArgs& a = p.a;
    a = MapArgs{};
    a.g_off = ctx->g_off.get();
    a.g_nbr = ctx->g_nbr.get();
    a.mean = ctx->g_mean.get();
    a.cover = ctx->cover.get();
    a.s_off = ctx->series_alias ? ctx->h_off.get() : ctx->s_off_buf.get();
    a.h_mem = ctx->h_mem.get();
    a.R = R;
    a.Hs = Hs;
    a.v_begin = p.vb;
    a.v_end = p.ve;
    a.h_begin = p.hb;
    a.h_end = p.he;
    a.M = M;
    a.beta = cfg->beta;
    a.tol = cfg->convergence_tol;
    a.L = L;
    a.ring = ring;
    a.fixed = fixed;
    a.adj_k = packed ? ctx->adj_k : 0;
    a.adj_pk = ctx->adj_pk.get();
    a.hood_k = packed ? ctx->hood_k : 0;
    a.hood_base = ctx->hood_base.get();
    a.hood_pk = ctx->hood_pk.get();
    a.terms = p.terms.ensure(3 * M);
    a.minE = p.minE.ensure(R ? R : 1);
    a.hist = p.hist.ensure(uint64_t(ring) * (Hs ? Hs : 1));
    a.flags = nullptr;
    a.eq = a.hood_k ? p.eq.ensure(Hs ? Hs : 1) : nullptr;
    uint32_t* state = p.state.ensure(uint64_t(map_max) + 4);
    a.unconv = state + 4;
    a.tile_counts = nullptr;  // the distributed M-step counts its own labels
    a.tiles = label_tiles(R);
    p.hpart.ensure(padH / kFoldLeaf);
    p.params.ensure(2 * M);
    p.em_out.ensure(2 + 2 * M);
    p.em_rec.ensure(uint64_t(em_max ? em_max : 1) * rec_stride);
    p.em_hist.ensure(uint64_t(em_max ? em_max : 1));
    mstep_reserve(p.ms, R, M, Hs);
    p.allcnt.ensure(uint64_t(W) * M);
    p.meta.ensure(4 * uint64_t(M) + 1);
    p.heads.ensure(uint64_t(W) * M * kFoldLeaf);
    p.pk.ensure(uint64_t(W) * owned_leaf_cap(g, M));
    EmEpilogueArgs& ep = p.ep;
    ep = EmEpilogueArgs{};
    ep.unconv = a.unconv;
    ep.map_max = map_max;
    ep.fixed = fixed;
    ep.L = L;
    ep.tol = cfg->convergence_tol;
    ep.lab0 = p.lab[0].get();
    ep.lab1 = p.lab[1].get();
    ep.R = R;
    ep.M = M;
    ep.em_out = p.em_out.get();
    ep.em_hist = p.em_hist.get();
    ep.em_rec = p.em_rec.get();
    ep.terms = p.terms.get();
  }
  double* h_terms = ctx->h_terms.ensure(3 * M);
  double* h_em = ctx->h_em.ensure(2 + 2 * M);
  double* h_rec = ctx->h_rec.ensure(uint64_t(em_max ? em_max : 1) * rec_stride + 4);

  CK(cudaEventRecord(ctx->ev_begin, st));
  for (auto& pp : g->parts) {
    Part& p = *pp;
    launch_init_labels(p.lab[0].get(), R, M, cfg->rng_seed, st);  // every rank: all R labels
    ++launches;
    CK(cudaMemsetAsync(p.state.get(), 0, 4 * sizeof(uint32_t), st));
    CK(cudaMemcpyAsync(p.params.get(), mu.data(), M * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(p.params.get() + M, sigma.data(), M * 8, cudaMemcpyHostToDevice, st));
  }
  const uint8_t* result = g->parts[0]->lab[0].get();  // em_max == 0: the initial labels

  if (em_max > 0) {
    result = g->parts[0]->lab_full.get();
    int final_buf = 0;  // label buffer holding the final labels (device loop: 0)
    uint64_t em_kernels = 0;
    auto enqueue_em = [&](int parity) {
      uint64_t k = 0;
      for (auto& pp : g->parts) {
        Part& p = *pp;
        if (device_loop) {
          launch_em_prologue(p.a.unconv, map_max, st);
          ++k;
        } else {
          CK(cudaMemcpyAsync(const_cast<double*>(p.a.terms), h_terms, 3 * M * 8,
                             cudaMemcpyHostToDevice, st));
          CK(cudaMemsetAsync(p.a.unconv, 0, map_max * sizeof(uint32_t), st));
        }
      }
      for (int t = 0; t < map_max; ++t) {
        const int bin = (parity + t) & 1, bout = bin ^ 1;
        for (auto& pp : g->parts) {
          launch_vertex_argmin(pp->a, pp->lab[bin].get(), pp->lab[bout].get(), t, st);
          ++k;
        }
        if (W > 1 && !g->split) {
          exchange_halo(g, bout, st);
          for (auto& pp : g->parts) {
            launch_hood_sums(pp->a, t, st);
            ++k;
          }
        } else {
        if (W > 1) {
          // exchange on the side stream; interior hoods meanwhile, boundary
          // hoods once the halos have landed
          CK(cudaEventRecord(g->ev_v, st));
          CK(cudaStreamWaitEvent(g->cs, g->ev_v, 0));
          exchange_halo(g, bout, g->cs);
          CK(cudaEventRecord(g->ev_x, g->cs));
        }
        for (auto& pp : g->parts) {
          if (pp->ib > pp->ia) {
            MapArgs ai = pp->a;
            ai.h_begin = pp->ia;
            ai.h_end = pp->ib;
            launch_hood_sums(ai, t, st);
            ++k;
          }
        }
        if (W > 1) CK(cudaStreamWaitEvent(st, g->ev_x, 0));
        for (auto& pp : g->parts) {
          if (pp->ia > pp->hb) {
            MapArgs lo = pp->a;
            lo.h_end = pp->ia;
            launch_hood_sums(lo, t, st);
            ++k;
          }
          if (pp->he > pp->ib) {
            MapArgs hi = pp->a;
            hi.h_begin = pp->ib;
            launch_hood_sums(hi, t, st);
            ++k;
          }
        }
        }
        // The summed counter decides the MAP early exit (optimize.cpp:59);
        // fixed-work runs never read it (executed_iters == map_max), so they
        // skip one latency-bound collective per MAP iteration.
        if (!fixed) sum_counters(g, t, st, &k);
      }
      // ---- distributed M-step (see k_part_count .. k_part_unpack_partials) ----
      const uint64_t cap_l = owned_leaf_cap(g, M);
      const size_t wsm = 8 * M * sizeof(uint32_t);
      for (auto& pp : g->parts) {
        Part& p = *pp;
        const uint32_t ntiles = (p.ve - p.vb + 255) / 256;
        const uint8_t* le = p.lab[parity].get();
        const uint8_t* lo_ = p.lab[parity ^ 1].get();
        CK(cudaMemsetAsync(p.allcnt.get() + uint64_t(p.r) * M, 0, M * sizeof(uint32_t), st));
        if (ntiles) {
          launch_pdl(k_part_count, dim3(ntiles), dim3(256), wsm, st, le, lo_,
                     (const uint32_t*)p.a.unconv, map_max, fixed, p.vb, p.ve, M,
                     p.ms.counts.get(), p.allcnt.get() + uint64_t(p.r) * M);
          ++k;
        }
        launch_row_leaves(p.a.hist, ring, Hs, p.a.unconv, map_max, fixed, p.hb, p.he,
                          p.hpart.get() + p.hb / kFoldLeaf, st);
        ++k;
      }
      gather_slots(g, {SlotBuf{[](Part& q) -> void* { return q.allcnt.get(); }, M, ncclUint32, 4},
                       SlotBuf{[](Part& q) -> void* { return q.hpart.get(); },
                               g->chunkH / kFoldLeaf, ncclFloat64, 8}},
                   st);
      for (auto& pp : g->parts) {
        Part& p = *pp;
        const uint32_t ntiles = (p.ve - p.vb + 255) / 256;
        const uint32_t* u = p.a.unconv;
        launch_pdl(k_part_layout, dim3(1), dim3(32), 0, st, (const uint32_t*)p.allcnt.get(), W,
                   p.r, M, Hs, u, p.ms.layout.get(), p.meta.get());
        launch_pdl(k_part_tile_base, dim3(1), dim3(1024), 0, st, (const uint32_t*)p.ms.counts.get(),
                   ntiles, M, u, (const uint32_t*)p.ms.layout.get(), (const uint32_t*)p.meta.get(),
                   p.ms.tile_base.get());
        k += 2;
        if (ntiles) {
          launch_pdl(k_part_scatter, dim3((ntiles + 7) / 8), dim3(256), wsm, st,
                     (const uint8_t*)p.lab[parity].get(), (const uint8_t*)p.lab[parity ^ 1].get(),
                     u, map_max, fixed, p.vb, p.ve, M, (const double*)p.a.mean,
                     (const uint32_t*)p.ms.tile_base.get(), p.ms.x.get());
          ++k;
        }
        launch_pdl(k_part_pack_heads, dim3(std::min<uint32_t>(M, 64)), dim3(256), 0, st,
                   (const double*)p.ms.x.get(), u, (const uint32_t*)p.ms.layout.get(),
                   (const uint32_t*)p.allcnt.get(), p.r, M, (const uint32_t*)p.meta.get(),
                   p.heads.get() + uint64_t(p.r) * M * kFoldLeaf);
        ++k;
      }
      gather_slots(g, {SlotBuf{[](Part& q) -> void* { return q.heads.get(); },
                               uint64_t(M) * kFoldLeaf, ncclFloat64, 8}},
                   st);
      for (auto& pp : g->parts) {
        Part& p = *pp;
        launch_pdl(k_part_unpack_heads, dim3(std::min<uint32_t>(W * M, 256)), dim3(256), 0, st,
                   (const double*)p.heads.get(), (const uint32_t*)p.a.unconv,
                   (const uint32_t*)p.ms.layout.get(), (const uint32_t*)p.allcnt.get(), W, p.r, M,
                   p.ms.x.get());
        ++k;
      }
      // per pass (sum, then (x - mu)^2): owned leaves, gathered partials, the
      // same trees on every rank (the same bits everywhere)
      const size_t fsm = size_t(kPartLPB) * (kFoldLeaf + 1) * sizeof(double);
      ensure_dynamic_smem(k_part_fold<false>, fsm);
      ensure_dynamic_smem(k_part_fold<true>, fsm);
      const unsigned fgrid = grid_for(cap_l, kPartLPB);
      for (int pass = 0; pass < 2; ++pass) {
        for (auto& pp : g->parts) {
          Part& p = *pp;
          launch_pdl(pass ? k_part_fold<true> : k_part_fold<false>, dim3(fgrid), dim3(256), fsm,
                     st, (const double*)p.ms.x.get(), (const uint32_t*)p.a.unconv,
                     (const uint32_t*)p.ms.layout.get(), (const uint32_t*)p.meta.get(), M,
                     (const double*)p.params.get(), p.pk.get() + uint64_t(p.r) * cap_l,
                     p.ms.partials.get());
          ++k;
        }
        gather_slots(g, {SlotBuf{[](Part& q) -> void* { return q.pk.get(); }, cap_l,
                                 ncclFloat64, 8}},
                     st);
        for (auto& pp : g->parts) {
          Part& p = *pp;
          launch_pdl(k_part_unpack_partials, dim3(std::min<int>(W, 64)), dim3(256), 0, st,
                     (const double*)p.pk.get(), cap_l, (const uint32_t*)p.a.unconv,
                     (const uint32_t*)p.ms.layout.get(), (const uint32_t*)p.allcnt.get(), W, p.r,
                     M, p.ms.partials.get());
          launch_fold_trees(pass == 1, M, Hs, p.a.unconv, map_max, fixed, p.params.get(),
                            p.em_out.get(), p.ms, p.hpart.get(), st);
          k += 2;
        }
      }
      for (auto& pp : g->parts) {
        Part& p = *pp;
        if (device_loop) {
          launch_em_epilogue(p.ep, st);
          ++k;
        }
      }
      if (!device_loop)
        CK(cudaMemcpyAsync(h_em, g->parts[0]->em_out.get(), (2 + 2 * M) * 8,
                           cudaMemcpyDeviceToHost, st));
      em_kernels = k;
    };
    auto host_terms = [&] {  // make_label_terms (model.hpp:48-60) with the host's std::log
      for (uint32_t l = 0; l < M; ++l) {
        h_terms[l] = mu[l];
        h_terms[M + l] = 2.0 * (sigma[l] * sigma[l]);
        h_terms[2 * M + l] = std::log(sigma[l]);
      }
    };
    ctx->stats.graphs = 0;
    if (device_loop) {
      host_terms();
      for (auto& pp : g->parts)
        CK(cudaMemcpyAsync(pp->terms.get(), h_terms, 3 * M * 8, cudaMemcpyHostToDevice, st));
      const bool use_graph = g->use_graph && g->local() && !(o.flags & DPMRF_RUN_NO_GRAPH);
      if (use_graph) {
        std::vector<uint64_t> key = {ctx->generation, R, Hs, M, uint64_t(L), uint64_t(map_max),
                                     uint64_t(fixed), uint64_t(packed)};
        uint64_t bits;
        std::memcpy(&bits, &cfg->beta, 8);
        key.push_back(bits);
        std::memcpy(&bits, &cfg->convergence_tol, 8);
        key.push_back(bits);
        for (auto& pp : g->parts) {
          Part& p = *pp;
          for (const void* q :
               {(const void*)p.lab[0].get(), (const void*)p.lab[1].get(),
                (const void*)p.lab_full.get(), (const void*)p.minE.get(),
                (const void*)p.hist.get(), (const void*)p.hpart.get(),
                (const void*)p.params.get(), (const void*)p.em_out.get(),
                (const void*)p.terms.get(), (const void*)p.em_rec.get(),
                (const void*)p.em_hist.get(), (const void*)p.state.get(),
                (const void*)p.ms.counts.get(), (const void*)p.ms.x.get(),
                (const void*)p.ms.partials.get(), (const void*)p.ms.layout.get(),
                (const void*)p.ms.tile_base.get()})
            key.push_back(reinterpret_cast<uintptr_t>(q));
        }
        if (!g->graph || key != g->graph_key) {
          g->drop_graph();
          cudaGraph_t gr = nullptr;
          CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
          try {
            enqueue_em(0);
          } catch (...) {
            cudaStreamEndCapture(st, &gr);
            if (gr) cudaGraphDestroy(gr);
            throw;
          }
          CK(cudaStreamEndCapture(st, &gr));
          CK(cudaGraphInstantiate(&g->graph, gr, 0));
          CK(cudaGraphDestroy(gr));
          g->graph_key = key;
          g->graph_kernels = em_kernels;
        }
        for (int em = 0; em < em_max; ++em) CK(cudaGraphLaunch(g->graph, st));
        em_kernels = g->graph_kernels;
        ctx->stats.graphs = 1;
      } else {
        for (int em = 0; em < em_max; ++em) enqueue_em(0);
      }
      Part& p0 = *g->parts[0];
      CK(cudaMemcpyAsync(h_rec, p0.state.get(), 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(h_rec + 4, p0.em_rec.get(), uint64_t(em_max) * rec_stride * 8,
                         cudaMemcpyDeviceToHost, st));
      ctx->sync();
      uint32_t hstate[4];
      std::memcpy(hstate, h_rec, sizeof hstate);
      const int em_count = static_cast<int>(hstate[2]);
      const double* rec = h_rec + 4;
      for (int e = 0; e + 1 < em_count; ++e)
        for (uint32_t l = 0; l < M; ++l) {
          const double sg = rec[e * rec_stride + 3 + M + l];
          const double dev = rec[e * rec_stride + 3 + 2 * M + l];
          const double host = std::log(sg);
          if (std::memcmp(&dev, &host, sizeof host) != 0) return false;
        }
      launches += uint64_t(em_max) * em_kernels;
      for (int e = 0; e < em_count; ++e) {
        const double* r = rec + e * rec_stride;
        ctx->stats.map_iters_total += static_cast<int>(r[1]);
        if (o.trace_level >= DPMRF_TRACE_EM) {
          dpmrf_context::EmRecord er;
          er.map_iters = static_cast<int>(r[1]);
          er.total = r[0];
          er.converged = r[2] != 0.0;
          er.mu.assign(r + 3, r + 3 + M);
          er.sigma.assign(r + 3 + M, r + 3 + 2 * M);
          ctx->trace.push_back(std::move(er));
        }
        if (e == em_count - 1) {
          mu.assign(r + 3, r + 3 + M);
          sigma.assign(r + 3 + M, r + 3 + 2 * M);
        }
      }
      ctx->stats.em_iters = em_count;
    } else {
      int cur = 0;
      std::vector<double> em_hist;
      for (int em = 0; em < em_max; ++em) {
        host_terms();
        enqueue_em(cur);
        launches += em_kernels;
        ctx->sync();
        const int T = static_cast<int>(h_em[1]);
        const double total = h_em[0];
        std::memcpy(mu.data(), h_em + 2, M * 8);
        std::memcpy(sigma.data(), h_em + 2 + M, M * 8);
        cur = (cur + T) & 1;
        ctx->stats.map_iters_total += T;
        em_hist.push_back(total);  // EM-level window, optimize.cpp:66-69
        uint8_t conv = 0;
        const size_t rows = em_hist.size();
        if (rows >= size_t(L) + 1) {
          conv = 1;
          for (int i = 1; i <= L; ++i)
            if (!(std::fabs(total - em_hist[rows - 1 - i]) < cfg->convergence_tol)) {
              conv = 0;
              break;
            }
        }
        if (o.trace_level >= DPMRF_TRACE_EM) {
          dpmrf_context::EmRecord er;
          er.map_iters = T;
          er.total = total;
          er.converged = conv;
          er.mu = mu;
          er.sigma = sigma;
          ctx->trace.push_back(std::move(er));
        }
        ctx->stats.em_iters = em + 1;
        if (conv && !fixed) break;
      }
      final_buf = cur;
    }
    // the labels are gathered once, after the EM loop (every rank's owned range)
    for (auto& pp : g->parts) {
      Part& p = *pp;
      if (p.ve > p.vb)
        CK(cudaMemcpyAsync(p.lab_full.get() + p.vb, p.lab[final_buf].get() + p.vb, p.ve - p.vb,
                           cudaMemcpyDeviceToDevice, st));
    }
    gather_slots(g, {SlotBuf{[](Part& q) -> void* { return q.lab_full.get(); }, g->chunkV,
                             ncclUint8, 1}},
                 st);
    ctx->stats.series = Hs;
  }
  uint32_t* l32 = ctx->labels32.ensure(R);
  launch_u8_to_u32(result, l32, R, st);
  ++launches;
  CK(cudaEventRecord(ctx->ev_end, st));
  if (labels_out && R)
    CK(cudaMemcpyAsync(labels_out, l32, uint64_t(R) * 4, cudaMemcpyDeviceToHost, st));
  ctx->sync();
  float total_ms = 0.f;
  CK(cudaEventElapsedTime(&total_ms, ctx->ev_begin, ctx->ev_end));
  ctx->stats.optimize_ms = total_ms;
  ctx->stats.kernel_launches = launches;
  if (mu_out) std::memcpy(mu_out, mu.data(), M * 8);
  if (sigma_out) std::memcpy(sigma_out, sigma.data(), M * 8);
  return true;
}

}  // namespace

// ---- C ABI -----------------------------------------------------------------------
extern "C" dpmrf_status dpmrf_nccl_unique_id(uint8_t id[128]) {
  return guarded([&] {
    need(id != nullptr, DPMRF_INVALID_ARGUMENT, "null id");
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
    Nccl& nccl = Nccl::get();
    ncclUniqueId u;
    NK(nccl.GetUniqueId(&u));
    std::memcpy(id, &u, sizeof u);
  });
}

namespace {
void init_side_stream(dpmrf_group* g) {
  CK(cudaStreamCreateWithFlags(&g->cs, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&g->ev_v, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&g->ev_x, cudaEventDisableTiming));
}
}  // namespace

extern "C" dpmrf_status dpmrf_group_create_nccl(dpmrf_context* ctx, const uint8_t id[128],
                                                int rank, int world, dpmrf_group** out) {
  return guarded([&] {
    need(ctx && id && out, DPMRF_INVALID_ARGUMENT, "null argument");
    ContextLock lock_(ctx);
    need(world >= 1 && world <= kMaxParts, DPMRF_INVALID_ARGUMENT, "world must be in [1, 64]");
    need(rank >= 0 && rank < world, DPMRF_INVALID_ARGUMENT, "rank out of range");
    ctx->bind();
    Nccl& nccl = Nccl::get();
    auto g = std::make_unique<dpmrf_group>();
    g->ctx = ctx;
    g->world = world;
    g->rank = rank;
    g->use_graph = false;  // NCCL calls are enqueued directly (no capture)
    if (const char* e = std::getenv("DPMRF_GROUP_GRAPH")) g->use_graph = e[0] == '1';
    // DPMRF_GROUP_SPLIT=0: one hood pass after the exchange (no overlap)
    if (const char* e = std::getenv("DPMRF_GROUP_SPLIT")) g->split = e[0] != '0';
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    NK(nccl.CommInitRank(&g->comm, world, u, rank));
    auto p = std::make_unique<Part>();
    p->r = rank;
    g->parts.push_back(std::move(p));
    init_side_stream(g.get());
    *out = g.release();
  });
}

extern "C" dpmrf_status dpmrf_group_create_local(dpmrf_context* ctx, int world,
                                                 dpmrf_group** out) {
  return guarded([&] {
    need(ctx && out, DPMRF_INVALID_ARGUMENT, "null argument");
    ContextLock lock_(ctx);
    need(world >= 1 && world <= kMaxParts, DPMRF_INVALID_ARGUMENT, "world must be in [1, 64]");
    ctx->bind();
    auto g = std::make_unique<dpmrf_group>();
    g->ctx = ctx;
    g->world = world;
    g->rank = -1;
    if (const char* e = std::getenv("DPMRF_NO_GRAPH")) g->use_graph = e[0] == '0';
    const char* sp = std::getenv("DPMRF_GROUP_SPLIT");
    g->split = sp && sp[0] == '1';
    for (int r = 0; r < world; ++r) {
      auto p = std::make_unique<Part>();
      p->r = r;
      g->parts.push_back(std::move(p));
    }
    init_side_stream(g.get());
    *out = g.release();
  });
}

extern "C" void dpmrf_group_destroy(dpmrf_group* g) {
  if (!g) return;
  cudaSetDevice(g->ctx->device);
  cudaStreamSynchronize(g->ctx->stream);
  g->drop_graph();
  if (g->cs) {
    cudaStreamSynchronize(g->cs);
    cudaStreamDestroy(g->cs);
  }
  if (g->ev_v) cudaEventDestroy(g->ev_v);
  if (g->ev_x) cudaEventDestroy(g->ev_x);
  if (g->comm) {
    Nccl& nccl = Nccl::get();
    nccl.CommDestroy(g->comm);
  }
  delete g;
}

extern "C" dpmrf_status dpmrf_group_info_get(dpmrf_group* g, dpmrf_group_info* out) {
  return guarded([&] {
    need(g && out, DPMRF_INVALID_ARGUMENT, "null argument");
    ContextLock lock_(g->ctx);  // plan() prepares the context and uses its scratch + stream
    g->ctx->bind();
    plan(g);
    dpmrf_group_info i{};
    i.world = g->world;
    i.rank = g->rank;
    const Part& p = *g->parts[0];
    i.vertex_begin = p.vb;
    i.vertex_end = p.ve;
    i.series_begin = p.hb;
    i.series_end = p.he;
    i.halo_bytes_per_map = g->halo_bytes;
    i.gather_bytes_per_em = g->gather_bytes;
    *out = i;
  });
}

extern "C" dpmrf_status dpmrf_optimize_partitioned(dpmrf_group* g,
                                                   const dpmrf_optimizer_config* cfg,
                                                   const dpmrf_run_options* opts,
                                                   uint32_t* labels_out, double* mu_out,
                                                   double* sigma_out) {
  return guarded([&] {
    need(g && cfg, DPMRF_INVALID_ARGUMENT, "null argument");
    const dpmrf_run_options o = opts ? *opts : dpmrf_run_options{0, DPMRF_TRACE_EM};
    check_config(*cfg, (o.flags & DPMRF_RUN_MULTILABEL) != 0);
    need(o.trace_level <= DPMRF_TRACE_EM, DPMRF_INVALID_ARGUMENT,
         "partitioned optimize records the EM trace only (trace level NONE or EM)");
    dpmrf_context* ctx = g->ctx;
    ContextLock lock_(ctx);  // the group runs on its context's stream and inputs
    need(ctx->has_graph, DPMRF_INVALID_ARGUMENT, "no region graph uploaded");
    need(ctx->has_hoods, DPMRF_INVALID_ARGUMENT, "no neighborhoods uploaded");
    ctx->bind();
    const bool device_loop = ctx->use_device_loop && !(o.flags & DPMRF_RUN_HOST_LOG) &&
                             cfg->em_max_iters > 0;
    if (device_loop) {
      if (run_partitioned(g, cfg, o, true, labels_out, mu_out, sigma_out)) return;
      ++ctx->stats.device_log_fallbacks;
    }
    run_partitioned(g, cfg, o, false, labels_out, mu_out, sigma_out);
  });
}
