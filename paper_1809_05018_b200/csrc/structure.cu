// structure.cu -- the inputs of the optimization phase built on the device
// (SURVEY.md §8(f) items 1 and 2).  Integer set / integer-sum work: the
// results are bit-identical to the reference whatever the order of the
// atomics, because every output is either a sorted set or an exact integer.
//
// build_region_graph (proj/src/graph/region_graph.cpp:10-73).  The reference
// emits two directed u64 keys per 4-adjacent pixel pair in different regions
// (2.04 M keys at 2560^2, ~150 M at 16384^2), sorts them all, uniques them,
// splits them by source into the CSR, and gets region sizes / sums from a
// second sort + reduce_by_key over all pixels.  Here:
//   1. k_boundary_tiles<0>: one 1024-thread block per 32x32 pixel tile.  The
//      tile's boundary pairs go into a shared-memory hash set (a boundary
//      crossing many pixel pairs of the tile is kept once), its regions into
//      a shared-memory (size, sum) table flushed with one global atomic per
//      (tile, region).  Out: the number of unique pairs per tile.
//   2. exclusive scan over tiles; k_boundary_tiles<1> rebuilds each tile's
//      set and writes its unique undirected pairs into the tile's range.
//   3. k_pair_degrees -> scan -> k_pair_fill: both orientations of every pair
//      bucketed by source region (counting sort, any order inside a bucket).
//   4. k_seg_sort_unique: one warp per region sorts + uniques its bucket in
//      registers (<= 32 keys) or its shared-memory slice (<= 1024); longer
//      buckets go to one block each (k_big_segments).  The sorted, unique,
//      self-loop-free list == the reference's sort + unique + split by source.
//   5. scan of the unique counts -> offsets; k_compact_segments -> neighbors;
//      k_region_means: mean = double(sum) / double(size) (region_graph.cpp:66-71).
//
// enumerate_maximal_cliques (proj/src/graph/cliques.cpp:53-106).  The same
// level-synchronous lexicographic extension: level k holds every k-clique as
// an ascending member list (stride k) in lexicographic order; per clique one
// thread intersects the members' adjacency lists (driven by the shortest
// list, binary search in the others: common_neighbors, cliques.cpp:16-27),
// marks the clique maximal when the intersection is empty, and (second pass)
// appends its children -- candidates above the last member, ascending -- at
// its scanned offset, which keeps the next level lexicographically sorted.
// canonical_sort (cliques.cpp:30-49) over the mixed-length union of the
// per-level maximal lists is a rank computation: a clique's final position is
// its index in its own (sorted) level plus, for every other level, the
// number of that level's cliques that precede it lexicographically (binary
// search); no two maximal cliques are prefixes of each other, so ranks are
// distinct.
#include <algorithm>
#include <memory>
#include <vector>

#include "context.cuh"
#include "segsort.cuh"

namespace dpmrf_b200 {

namespace {

constexpr int kTile = 32;                       // 32 x 32 pixels per block
constexpr int kTileThreads = kTile * kTile;     // one thread per pixel
constexpr uint32_t kPairSlots = 4096;           // <= 2 pairs per pixel: load <= 1/2
constexpr uint32_t kRegSlots = 2048;            // <= 1024 regions per tile: load <= 1/2
constexpr unsigned long long kEmpty64 = ~0ull;
constexpr uint32_t kEmpty32 = ~0u;
constexpr uint32_t kSegWarps = 8;               // warps per block in k_seg_sort_unique
constexpr uint32_t kSegSmem = 1024;             // keys per warp in shared memory
constexpr int kMaxCliqueSize = 64;

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

// Inserts key into the shared-memory set; true iff this call inserted it.
// The table is never more than half full, so probing terminates.
__device__ __forceinline__ bool set_insert(unsigned long long* tab, unsigned long long key) {
  uint32_t i = mix32(uint32_t(key) ^ mix32(uint32_t(key >> 32))) & (kPairSlots - 1);
  while (true) {
    const unsigned long long prev = atomicCAS(&tab[i], kEmpty64, key);
    if (prev == kEmpty64) return true;
    if (prev == key) return false;
    i = (i + 1) & (kPairSlots - 1);
  }
}

// Pass 0: unique boundary pairs per tile + region (size, sum) accumulation.
// Pass 1: the same pairs written to the tile's range of `pairs`.
// err bit 0: a region id >= R.
template <int kPass>
__global__ void __launch_bounds__(kTileThreads)
    k_boundary_tiles(const uint32_t* __restrict__ reg, const uint8_t* __restrict__ px, uint32_t w,
                     uint32_t h, uint32_t R, uint32_t* __restrict__ tile_cnt,
                     const uint32_t* __restrict__ tile_off, unsigned long long* __restrict__ pairs,
                     uint32_t* __restrict__ rsize, unsigned long long* __restrict__ rsum,
                     uint32_t* __restrict__ err) {
  extern __shared__ unsigned long long smem[];
  unsigned long long* ptab = smem;                                   // kPairSlots
  uint32_t* rkey = reinterpret_cast<uint32_t*>(smem + kPairSlots);   // kRegSlots
  uint32_t* rcnt = rkey + kRegSlots;                                 // kRegSlots
  uint32_t* rsm = rcnt + kRegSlots;                                  // kRegSlots (tile sum < 2^18)
  __shared__ uint32_t warp_tmp[32];
  const uint32_t tid = threadIdx.x;
  const uint64_t tile = uint64_t(blockIdx.y) * gridDim.x + blockIdx.x;
  for (uint32_t i = tid; i < kPairSlots; i += kTileThreads) ptab[i] = kEmpty64;
  if (kPass == 0)
    for (uint32_t i = tid; i < kRegSlots; i += kTileThreads) {
      rkey[i] = kEmpty32;
      rcnt[i] = 0;
      rsm[i] = 0;
    }
  __syncthreads();
  const uint32_t x = blockIdx.x * kTile + (tid & (kTile - 1));
  const uint32_t y = blockIdx.y * kTile + (tid / kTile);
  // (Folding pixel runs with __match_any_sync before the shared-memory
  // atomics measured slower: three warp matches per pixel cost more than
  // the atomics they save.)
  unsigned long long k1 = kEmpty64, k2 = kEmpty64;
  if (x < w && y < h) {
    const uint64_t i = uint64_t(y) * w + x;
    const uint32_t a = reg[i];
    if (a >= R) {
      if (kPass == 0) atomicOr(err, 1u);
    } else {
      if (kPass == 0) {
        uint32_t s = mix32(a) & (kRegSlots - 1);
        while (true) {
          const uint32_t prev = atomicCAS(&rkey[s], kEmpty32, a);
          if (prev == kEmpty32 || prev == a) break;
          s = (s + 1) & (kRegSlots - 1);
        }
        atomicAdd(&rcnt[s], 1u);
        atomicAdd(&rsm[s], uint32_t(px[i]));
      }
      // right and down arcs cover every 4-adjacent pixel pair once (region_graph.cpp:21-26)
      if (x + 1 < w) {
        const uint32_t b = reg[i + 1];
        if (b != a && b < R) {
          const unsigned long long key = (uint64_t(min(a, b)) << 32) | max(a, b);
          if (set_insert(ptab, key)) k1 = key;
        }
      }
      if (y + 1 < h) {
        const uint32_t b = reg[i + w];
        if (b != a && b < R) {
          const unsigned long long key = (uint64_t(min(a, b)) << 32) | max(a, b);
          if (set_insert(ptab, key)) k2 = key;
        }
      }
    }
  }
  const uint32_t nn = (k1 != kEmpty64) + (k2 != kEmpty64);
  if (kPass == 0) {
    const int c1 = __syncthreads_count(nn >= 1);
    const int c2 = __syncthreads_count(nn == 2);
    if (tid == 0) tile_cnt[tile] = uint32_t(c1 + c2);
    for (uint32_t s = tid; s < kRegSlots; s += kTileThreads) {
      const uint32_t r = rkey[s];
      if (r != kEmpty32) {
        atomicAdd(&rsize[r], rcnt[s]);
        atomicAdd(&rsum[r], static_cast<unsigned long long>(rsm[s]));
      }
    }
  } else {
    const uint32_t pos = tile_off[tile] + block_exclusive_scan(nn, warp_tmp, nullptr);
    uint32_t o = 0;
    if (k1 != kEmpty64) pairs[pos + o++] = k1;
    if (k2 != kEmpty64) pairs[pos + o] = k2;
  }
}

__global__ void k_pair_degrees(const unsigned long long* __restrict__ pairs, uint64_t P,
                               uint32_t* __restrict__ deg) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const unsigned long long k = pairs[i];
  atomicAdd(&deg[uint32_t(k >> 32)], 1u);
  atomicAdd(&deg[uint32_t(k)], 1u);
}

__global__ void k_pair_fill(const unsigned long long* __restrict__ pairs, uint64_t P,
                            const uint32_t* __restrict__ boff, uint32_t* __restrict__ fill,
                            uint32_t* __restrict__ bucket) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const unsigned long long k = pairs[i];
  const uint32_t a = uint32_t(k >> 32), b = uint32_t(k);
  bucket[boff[a] + atomicAdd(&fill[a], 1u)] = b;
  bucket[boff[b] + atomicAdd(&fill[b], 1u)] = a;
}

// In-place sort + unique of every segment [off[v], off[v+1]) of keys with at
// most kSegSmem keys; ucnt[v] = unique count.  Longer segments are appended to
// `big` (count in big_n) and left to k_big_segments.
__global__ void __launch_bounds__(kSegWarps * 32)
    k_seg_sort_unique(uint32_t* __restrict__ keys, const uint32_t* __restrict__ off, uint32_t n_seg,
                      uint32_t* __restrict__ ucnt, uint32_t* __restrict__ big,
                      uint32_t* __restrict__ big_n) {
  __shared__ uint32_t buf[kSegWarps][kSegSmem];
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const uint64_t v = uint64_t(blockIdx.x) * kSegWarps + wi;
  if (v >= n_seg) return;
  const uint32_t lo = off[v], n = off[v + 1] - lo;
  uint32_t* seg = keys + lo;
  if (n <= 32) {
    uint32_t x = lane < int(n) ? seg[lane] : kPad;
    x = warp_bitonic32(x, lane);
    const uint32_t u = warp_unique_chunk(x, lane < int(n), 0, false, seg, lane);
    if (lane == 0) ucnt[v] = u;
    return;
  }
  if (n > kSegSmem) {
    if (lane == 0) big[atomicAdd(big_n, 1u)] = static_cast<uint32_t>(v);
    return;
  }
  uint32_t* b = buf[wi];
  uint32_t P = 64;
  while (P < n) P <<= 1;
  for (uint32_t i = lane; i < P; i += 32) b[i] = i < n ? seg[i] : kPad;
  __syncwarp();
  bitonic_sort(b, P, lane, 32, [] { __syncwarp(); });
  const uint32_t u = warp_unique_sorted(b, n, seg, lane);
  if (lane == 0) ucnt[v] = u;
}

// Buckets of <= G keys (every grid / brick region): G lanes per region sort +
// unique in registers; kPass 0 -> unique counts, kPass 1 -> the neighbors at
// the scanned offsets (no separate compaction).
template <int G, int kPass>
__global__ void __launch_bounds__(256)
    k_bucket_small(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ off,
                   uint32_t n_seg, uint32_t* __restrict__ ucnt,
                   const uint32_t* __restrict__ out_off, uint32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int l = lane & (G - 1);
  const uint64_t v = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) / G;
  uint32_t x = kPad;
  if (v < n_seg) {
    const uint32_t lo = off[v], n = off[v + 1] - lo;
    if (uint32_t(l) < n) x = keys[lo + l];
  }
  bool keep;
  uint32_t rank;
  const uint32_t u = group_sort_unique<G>(x, lane, keep, rank);
  if (v >= n_seg) return;
  if (kPass == 0) {
    if (l == 0) ucnt[v] = u;
  } else if (keep) {
    out[out_off[v] + rank] = x;
  }
}

template <int G>
void bucket_small(const uint32_t* keys, const uint32_t* off, uint32_t n, uint32_t* ucnt,
                  const uint32_t* out_off, uint32_t* out, int pass, cudaStream_t st) {
  const unsigned grid = grid_for(uint64_t(n) * G, 256);
  if (pass == 0) k_bucket_small<G, 0><<<grid, 256, 0, st>>>(keys, off, n, ucnt, out_off, out);
  else k_bucket_small<G, 1><<<grid, 256, 0, st>>>(keys, off, n, ucnt, out_off, out);
  CK_LAUNCH();
}

__global__ void k_max_u32(const uint32_t* __restrict__ x, uint64_t n, uint32_t* __restrict__ out) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t v = i < n ? x[i] : 0u;
  const uint32_t m = __reduce_max_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

// One block per long segment: bitonic sort in a power-of-two scratch slice.
__global__ void __launch_bounds__(1024)
    k_big_segments(uint32_t* __restrict__ keys, const uint32_t* __restrict__ off,
                   const uint32_t* __restrict__ big, const uint64_t* __restrict__ tmp_off,
                   uint32_t* __restrict__ tmp, uint32_t* __restrict__ ucnt) {
  const uint32_t v = big[blockIdx.x];
  const uint32_t lo = off[v], n = off[v + 1] - lo;
  uint32_t* b = tmp + tmp_off[blockIdx.x];
  const uint64_t P = tmp_off[blockIdx.x + 1] - tmp_off[blockIdx.x];
  for (uint64_t i = threadIdx.x; i < P; i += blockDim.x) b[i] = i < n ? keys[lo + i] : kPad;
  __syncthreads();
  bitonic_sort(b, P, threadIdx.x, blockDim.x, [] { __syncthreads(); });
  if (threadIdx.x >= 32) return;
  const uint32_t u = warp_unique_sorted(b, n, keys + lo, threadIdx.x);
  if (threadIdx.x == 0) ucnt[v] = u;
}

// out[dst_off[v] + j] = keys[src_off[v] + j], j < dst_off[v+1] - dst_off[v]; warp per segment.
__global__ void k_compact_segments(const uint32_t* __restrict__ keys,
                                   const uint32_t* __restrict__ src_off,
                                   const uint32_t* __restrict__ dst_off, uint32_t n_seg,
                                   uint32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t v = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (v >= n_seg) return;
  const uint32_t src = src_off[v], dst = dst_off[v], n = dst_off[v + 1] - dst;
  for (uint32_t i = lane; i < n; i += 32) out[dst + i] = keys[src + i];
}

// region_mean = double(integer sum) / double(size) (region_graph.cpp:66-71).
// err bit 1: a region with no pixels (the label map was not validated).
__global__ void k_region_means(const uint32_t* __restrict__ rsize,
                               const unsigned long long* __restrict__ rsum, uint32_t R,
                               double* __restrict__ mean, uint32_t* __restrict__ err) {
  const uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const uint32_t n = rsize[r];
  if (n == 0) {
    atomicOr(err, 2u);
    mean[r] = 0.0;
    return;
  }
  mean[r] = __ddiv_rn(static_cast<double>(rsum[r]), static_cast<double>(n));
}

// ---- maximal cliques ------------------------------------------------------------

__device__ __forceinline__ bool adj_contains(const uint32_t* __restrict__ g_off,
                                             const uint32_t* __restrict__ g_nbr, uint32_t v,
                                             uint32_t u) {
  uint32_t lo = g_off[v], hi = g_off[v + 1];
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    const uint32_t x = g_nbr[mid];
    if (x == u) return true;
    if (x < u) lo = mid + 1;
    else hi = mid;
  }
  return false;
}

// Level 1 (every vertex is a 1-clique): maximal iff isolated; children are
// the edges (v, u), u > v.  cnt[v] = children, flag[v] = maximal.
__global__ void k_clique_level1(const uint32_t* __restrict__ g_off,
                                const uint32_t* __restrict__ g_nbr, uint32_t R,
                                uint32_t* __restrict__ cnt, uint32_t* __restrict__ flag) {
  const uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= R) return;
  const uint32_t lo = g_off[v], hi = g_off[v + 1];
  uint32_t a = lo, b = hi;  // first neighbor > v (upper_bound, cliques.cpp:79)
  while (a < b) {
    const uint32_t mid = (a + b) >> 1;
    if (g_nbr[mid] <= v) a = mid + 1;
    else b = mid;
  }
  cnt[v] = hi - a;
  flag[v] = lo == hi;
}

__global__ void k_clique_level1_write(const uint32_t* __restrict__ g_off,
                                      const uint32_t* __restrict__ g_nbr, uint32_t R,
                                      const uint32_t* __restrict__ child_off,
                                      uint32_t* __restrict__ next) {
  const uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= R) return;
  uint32_t pos = child_off[v];
  for (uint32_t s = g_off[v]; s < g_off[v + 1]; ++s) {
    const uint32_t u = g_nbr[s];
    if (u <= v) continue;
    next[2ull * pos] = uint32_t(v);
    next[2ull * pos + 1] = u;
    ++pos;
  }
}

// Level k >= 2.  kPass 0: cnt[i] = children, flag[i] = maximal (common
// neighborhood empty).  kPass 1: children written at child_off[i].
template <int kPass>
__global__ void k_clique_level(const uint32_t* __restrict__ F, uint64_t fk, int k,
                               const uint32_t* __restrict__ g_off,
                               const uint32_t* __restrict__ g_nbr, uint32_t* __restrict__ cnt,
                               uint32_t* __restrict__ flag, const uint32_t* __restrict__ child_off,
                               uint32_t* __restrict__ next) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= fk) return;
  const uint32_t* m = F + i * k;
  // drive the intersection with the shortest adjacency list
  int jd = 0;
  uint32_t best = g_off[m[0] + 1] - g_off[m[0]];
  for (int j = 1; j < k; ++j) {
    const uint32_t d = g_off[m[j] + 1] - g_off[m[j]];
    if (d < best) {
      best = d;
      jd = j;
    }
  }
  const uint32_t last = m[k - 1];
  const uint32_t d0 = g_off[m[jd]], d1 = g_off[m[jd] + 1];
  uint32_t all = 0, hi = 0;
  uint64_t pos = kPass == 1 ? uint64_t(child_off[i]) : 0;
  for (uint32_t s = d0; s < d1; ++s) {
    const uint32_t u = g_nbr[s];
    bool common = true;
    for (int j = 0; j < k && common; ++j)
      if (j != jd) common = adj_contains(g_off, g_nbr, m[j], u);
    if (!common) continue;  // (members drop out: no self-loops)
    ++all;
    if (u > last) {
      if (kPass == 1) {
        uint32_t* c = next + pos * (k + 1);
        for (int j = 0; j < k; ++j) c[j] = m[j];
        c[k] = u;
        ++pos;
      }
      ++hi;
    }
  }
  if (kPass == 0) {
    cnt[i] = hi;
    flag[i] = all == 0;
  }
}

// Copies the flagged cliques (stride k) of a level, in order, to out.
__global__ void k_clique_compact(const uint32_t* __restrict__ F, uint64_t fk, int k,
                                 const uint32_t* __restrict__ flag,
                                 const uint32_t* __restrict__ pos, uint32_t* __restrict__ out) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= fk || !flag[i]) return;
  for (int j = 0; j < k; ++j) out[uint64_t(pos[i]) * k + j] = F[i * k + j];
}

__global__ void k_clique_isolated(uint32_t R, const uint32_t* __restrict__ flag,
                                  const uint32_t* __restrict__ pos, uint32_t* __restrict__ out) {
  const uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v < R && flag[v]) out[pos[v]] = static_cast<uint32_t>(v);
}

struct LevelDesc {
  const uint32_t* data;  // count x k members, lexicographically sorted
  uint64_t count;
  uint64_t base;         // index of this level's first clique in the flat per-level order
  int k;
};
constexpr int kMaxLevels = kMaxCliqueSize;
struct Levels {
  LevelDesc l[kMaxLevels];
  int n;
};

// std::lexicographical_compare(a, a+ka, b, b+kb)
__device__ __forceinline__ bool lex_less(const uint32_t* a, int ka, const uint32_t* b, int kb) {
  const int n = ka < kb ? ka : kb;
  for (int j = 0; j < n; ++j) {
    if (a[j] < b[j]) return true;
    if (b[j] < a[j]) return false;
  }
  return ka < kb;
}

// rank of every maximal clique in the canonical order (cliques.cpp:30-49);
// size_at[rank] = k, src[rank] = (level, index) packed as the flat index.
__global__ void k_clique_rank(Levels L, uint64_t total, uint32_t* __restrict__ size_at,
                              unsigned long long* __restrict__ src_at) {
  const uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= total) return;
  int lv = 0;
  while (lv + 1 < L.n && g >= L.l[lv + 1].base) ++lv;
  const uint64_t i = g - L.l[lv].base;
  const int k = L.l[lv].k;
  const uint32_t* x = L.l[lv].data + i * k;
  uint64_t rank = i;
  for (int o = 0; o < L.n; ++o) {
    if (o == lv) continue;
    const LevelDesc& d = L.l[o];
    uint64_t lo = 0, hi = d.count;  // number of d's cliques lexicographically below x
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (lex_less(d.data + mid * d.k, d.k, x, k)) lo = mid + 1;
      else hi = mid;
    }
    rank += lo;
  }
  size_at[rank] = static_cast<uint32_t>(k);
  src_at[rank] = g;
}

__global__ void k_clique_emit(Levels L, uint64_t total, const uint32_t* __restrict__ c_off,
                              const unsigned long long* __restrict__ src_at,
                              uint32_t* __restrict__ c_mem) {
  const uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= total) return;
  const uint64_t g = src_at[r];
  int lv = 0;
  while (lv + 1 < L.n && g >= L.l[lv + 1].base) ++lv;
  const int k = L.l[lv].k;
  const uint32_t* x = L.l[lv].data + (g - L.l[lv].base) * k;
  for (int j = 0; j < k; ++j) c_mem[c_off[r] + j] = x[j];
}

template <class T>
T d2h(const T* p, cudaStream_t st) {
  T v;
  CK(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return v;
}

}  // namespace

// Sort + unique every segment of keys in place; ucnt[v] receives the counts.
void segmented_sort_unique(uint32_t* keys, const uint32_t* off, uint32_t n_seg, uint32_t* ucnt,
                           DevBuf<uint32_t>& big_buf, cudaStream_t st) {
  if (!n_seg) return;
  uint32_t* big = big_buf.ensure(uint64_t(n_seg) + 1);
  uint32_t* big_n = big + n_seg;
  CK(cudaMemsetAsync(big_n, 0, 4, st));
  k_seg_sort_unique<<<grid_for(n_seg, kSegWarps), kSegWarps * 32, 0, st>>>(keys, off, n_seg, ucnt,
                                                                          big, big_n);
  CK_LAUNCH();
  const uint32_t nb = d2h(big_n, st);
  if (!nb) return;
  // rare: segments longer than kSegSmem keys (very high-degree regions)
  std::vector<uint32_t> ids(nb), offs(uint64_t(n_seg) + 1);
  CK(cudaMemcpyAsync(ids.data(), big, nb * 4ull, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(offs.data(), off, (uint64_t(n_seg) + 1) * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::vector<uint64_t> toff{0};
  for (uint32_t v : ids) {
    uint64_t P = 1;
    while (P < offs[v + 1] - offs[v]) P <<= 1;
    toff.push_back(toff.back() + P);
  }
  DevBuf<uint32_t> d_ids, tmp;
  DevBuf<unsigned long long> d_toff;
  CK(cudaMemcpyAsync(d_ids.ensure(nb), ids.data(), nb * 4ull, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_toff.ensure(toff.size()), toff.data(), toff.size() * 8,
                     cudaMemcpyHostToDevice, st));
  k_big_segments<<<nb, 1024, 0, st>>>(keys, off, d_ids.get(),
                                      reinterpret_cast<const uint64_t*>(d_toff.get()),
                                      tmp.ensure(toff.back()), ucnt);
  CK_LAUNCH();
  CK(cudaStreamSynchronize(st));  // (scratch is freed on return)
}

void build_region_graph_device(dpmrf_context* ctx, uint32_t w, uint32_t h, const uint8_t* px,
                               const uint32_t* reg, uint32_t R) {
  cudaStream_t st = ctx->stream;
  const uint32_t tx = (w + kTile - 1) / kTile, ty = (h + kTile - 1) / kTile;
  const uint64_t tiles = uint64_t(tx) * ty;
  if (tiles >= (1ull << 32) - 1) fail(DPMRF_INVALID_ARGUMENT, "region graph: image too large");
  uint32_t* tile_cnt = ctx->st_u32[0].ensure(tiles + 1);
  uint32_t* err = ctx->st_u32[1].ensure(uint64_t(R) * 4 + 8);  // err | size | deg | fill | ucnt
  uint32_t* rsize = err + 2;
  uint32_t* deg = rsize + R;
  uint32_t* fill = deg + R;
  uint32_t* ucnt = fill + R;
  uint32_t* boff = ctx->st_u32[2].ensure(uint64_t(R) + 1);
  unsigned long long* rsum = ctx->st_u64[0].ensure(R);
  CK(cudaMemsetAsync(err, 0, (uint64_t(R) * 4 + 8) * 4, st));
  CK(cudaMemsetAsync(rsum, 0, uint64_t(R) * 8, st));
  const size_t smem = kPairSlots * 8 + 3 * kRegSlots * 4;
  ensure_dynamic_smem(k_boundary_tiles<0>, smem);
  const dim3 grid(tx, ty);
  k_boundary_tiles<0><<<grid, kTileThreads, smem, st>>>(reg, px, w, h, R, tile_cnt, nullptr,
                                                        nullptr, rsize, rsum, err);
  CK_LAUNCH();
  exclusive_scan_u32(tile_cnt, tile_cnt, tiles, tile_cnt + tiles, ctx->scan, st);
  const uint32_t e0 = d2h(err, st);
  if (e0 & 1u) fail(DPMRF_OUT_OF_RANGE, "region graph: region id >= num_regions");
  const uint64_t P = d2h(tile_cnt + tiles, st);
  unsigned long long* pairs = ctx->st_u64[1].ensure(P);
  if (P)
    k_boundary_tiles<1><<<grid, kTileThreads, kPairSlots * 8, st>>>(
        reg, px, w, h, R, nullptr, tile_cnt, pairs, nullptr, nullptr, nullptr);
  CK_LAUNCH();
  if (P >= (1ull << 31)) fail(DPMRF_INVALID_ARGUMENT, "region graph: too many boundary pairs");
  if (P) {
    k_pair_degrees<<<grid_for(P, 256), 256, 0, st>>>(pairs, P, deg);
    CK_LAUNCH();
  }
  exclusive_scan_u32(deg, boff, R, boff + R, ctx->scan, st);
  uint32_t* bucket = ctx->st_u32[3].ensure(2 * P);
  uint32_t* dmax = err + 1;  // (err[1] is free scratch)
  if (P) {
    k_pair_fill<<<grid_for(P, 256), 256, 0, st>>>(pairs, P, boff, fill, bucket);
    CK_LAUNCH();
    k_max_u32<<<grid_for(R, 256), 256, 0, st>>>(deg, R, dmax);
    CK_LAUNCH();
  }
  const uint32_t max_bucket = d2h(dmax, st);
  uint32_t* g_off = ctx->g_off.ensure(uint64_t(R) + 1);
  const int G = max_bucket <= 8 ? 8 : (max_bucket <= 16 ? 16 : (max_bucket <= 32 ? 32 : 0));
  auto small = [&](int pass, uint32_t* out) {
    if (G == 8) bucket_small<8>(bucket, boff, R, ucnt, g_off, out, pass, st);
    else if (G == 16) bucket_small<16>(bucket, boff, R, ucnt, g_off, out, pass, st);
    else bucket_small<32>(bucket, boff, R, ucnt, g_off, out, pass, st);
  };
  if (G) small(0, nullptr);
  else segmented_sort_unique(bucket, boff, R, ucnt, ctx->st_u32[4], st);
  exclusive_scan_u32(ucnt, g_off, R, g_off + R, ctx->scan, st);
  const uint64_t A = d2h(g_off + R, st);
  uint32_t* g_nbr = ctx->g_nbr.ensure(A);
  if (R) {
    if (G) {
      small(1, g_nbr);
    } else {
      k_compact_segments<<<grid_for(uint64_t(R) * 32, 256), 256, 0, st>>>(bucket, boff, g_off,
                                                                           R, g_nbr);
      CK_LAUNCH();
    }
    k_region_means<<<grid_for(R, 256), 256, 0, st>>>(rsize, rsum, R, ctx->g_mean.ensure(R), err);
    CK_LAUNCH();
  }
  CK(cudaMemcpyAsync(ctx->g_size.ensure(R), rsize, uint64_t(R) * 4, cudaMemcpyDeviceToDevice, st));
  const uint32_t e1 = d2h(err, st);
  if (e1 & 2u) fail(DPMRF_INPUT_ERROR, "region graph: label map not validated (unused region id)");
  ctx->R = R;
  ctx->A = A;
}

void enumerate_maximal_cliques_device(dpmrf_context* ctx) {
  cudaStream_t st = ctx->stream;
  const uint32_t R = ctx->R;
  const uint32_t* g_off = ctx->g_off.get();
  const uint32_t* g_nbr = ctx->g_nbr.get();
  // per-level maximal cliques (context scratch: no allocation once warm)
  std::vector<uint32_t*> lv_data;
  std::vector<uint64_t> lv_count;
  std::vector<int> lv_k;
  DevBuf<uint32_t>* front = ctx->cl_tmp;  // [0], [1]
  DevBuf<uint32_t>& cnt = ctx->cl_tmp[2];
  DevBuf<uint32_t>& flag = ctx->cl_tmp[3];
  DevBuf<uint32_t>& pos = ctx->cl_tmp[4];
  auto level_buf = [&](uint64_t n) {
    const size_t i = lv_data.size();
    if (ctx->cl_level.size() <= i) ctx->cl_level.push_back(std::make_unique<DevBuf<uint32_t>>());
    return ctx->cl_level[i]->ensure(n);
  };
  if (R == 0) {
    ctx->C = ctx->CS = 0;
    CK(cudaMemsetAsync(ctx->c_off.ensure(1), 0, 4, st));
    ctx->c_mem.ensure(1);
    return;
  }
  // ---- level 1 ----
  {
    uint32_t* c = cnt.ensure(uint64_t(R) + 1);
    uint32_t* f = flag.ensure(uint64_t(R) + 1);
    uint32_t* p = pos.ensure(uint64_t(R) + 1);
    k_clique_level1<<<grid_for(R, 256), 256, 0, st>>>(g_off, g_nbr, R, c, f);
    CK_LAUNCH();
    exclusive_scan_u32(c, c, R, c + R, ctx->scan, st);
    exclusive_scan_u32(f, p, R, p + R, ctx->scan, st);
    const uint64_t n_max = d2h(p + R, st), n_next = d2h(c + R, st);
    if (n_max) {
      // isolated vertices: singleton cliques, already in order
      uint32_t* d = level_buf(n_max);
      k_clique_isolated<<<grid_for(R, 256), 256, 0, st>>>(R, f, p, d);
      CK_LAUNCH();
      lv_data.push_back(d);
      lv_count.push_back(n_max);
      lv_k.push_back(1);
    }
    uint32_t* nx = front[0].ensure(2 * n_next);
    if (n_next) {
      k_clique_level1_write<<<grid_for(R, 256), 256, 0, st>>>(g_off, g_nbr, R, c, nx);
      CK_LAUNCH();
    }
    uint64_t fk = n_next;
    int cur = 0;
    for (int k = 2; fk; ++k) {
      if (k > kMaxCliqueSize) fail(DPMRF_INVALID_ARGUMENT, "maximal cliques: clique too large");
      if (fk >= (1ull << 32) - 1) fail(DPMRF_INVALID_ARGUMENT, "maximal cliques: frontier too large");
      const uint32_t* F = front[cur].get();
      uint32_t* cc = cnt.ensure(fk + 1);
      uint32_t* ff = flag.ensure(fk + 1);
      uint32_t* pp = pos.ensure(fk + 1);
      k_clique_level<0><<<grid_for(fk, 256), 256, 0, st>>>(F, fk, k, g_off, g_nbr, cc, ff,
                                                           nullptr, nullptr);
      CK_LAUNCH();
      exclusive_scan_u32(cc, cc, fk, cc + fk, ctx->scan, st);
      exclusive_scan_u32(ff, pp, fk, pp + fk, ctx->scan, st);
      const uint64_t nm = d2h(pp + fk, st), nn = d2h(cc + fk, st);
      if (nm) {
        uint32_t* d = level_buf(nm * k);
        k_clique_compact<<<grid_for(fk, 256), 256, 0, st>>>(F, fk, k, ff, pp, d);
        CK_LAUNCH();
        lv_data.push_back(d);
        lv_count.push_back(nm);
        lv_k.push_back(k);
      }
      if (nn) {
        uint32_t* nx2 = front[cur ^ 1].ensure(nn * (k + 1));
        k_clique_level<1><<<grid_for(fk, 256), 256, 0, st>>>(F, fk, k, g_off, g_nbr, nullptr,
                                                             nullptr, cc, nx2);
        CK_LAUNCH();
      }
      CK(cudaStreamSynchronize(st));  // before the next level reuses cnt/flag/pos
      cur ^= 1;
      fk = nn;
    }
  }
  // ---- canonical order over all levels ----
  Levels L{};
  L.n = static_cast<int>(lv_data.size());
  uint64_t total = 0, members = 0;
  for (int i = 0; i < L.n; ++i) {
    L.l[i] = LevelDesc{lv_data[i], lv_count[i], total, lv_k[i]};
    total += lv_count[i];
    members += lv_count[i] * lv_k[i];
  }
  if (total >= (1ull << 32) - 1 || members >= (1ull << 32))
    fail(DPMRF_INVALID_ARGUMENT, "maximal cliques: too many cliques");
  uint32_t* c_off = ctx->c_off.ensure(total + 1);
  uint32_t* c_mem = ctx->c_mem.ensure(members);
  if (total) {
    unsigned long long* sa = ctx->st_u64[2].ensure(total);
    k_clique_rank<<<grid_for(total, 256), 256, 0, st>>>(L, total, c_off, sa);
    CK_LAUNCH();
    exclusive_scan_u32(c_off, c_off, total, c_off + total, ctx->scan, st);
    k_clique_emit<<<grid_for(total, 256), 256, 0, st>>>(L, total, c_off, sa, c_mem);
    CK_LAUNCH();
    CK(cudaStreamSynchronize(st));
  } else {
    CK(cudaMemsetAsync(c_off, 0, 4, st));
  }
  ctx->C = total;
  ctx->CS = members;
  CK(cudaStreamSynchronize(st));
}

}  // namespace dpmrf_b200
