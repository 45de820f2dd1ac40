// hoods.cu -- build_neighborhoods on the device (north_star item 1).
//
// Reference: proj/src/graph/neighborhoods.cpp:10-57.  The reference writes
// one u64 key (clique << 32 | vertex) per candidate (each clique member plus
// its graph neighbors), sorts ALL keys globally, uniques them and rebuilds the
// offsets.  Sorting by (clique, vertex) only ever orders candidates WITHIN a
// clique, so the device version sorts each clique's candidate list on its own:
//   1. count    : per clique, sum over members of 1 + degree   (neighborhoods.cpp:23-25)
//   2. scan     : candidate offsets                            (:26)
//   3. sort     : one warp per clique -- register bitonic sort via shuffles
//                 for <= 32 candidates (every grid / brick hood), a
//                 shared-memory bitonic sort for <= 1024, and a block-wide
//                 global-memory bitonic sort beyond that; duplicates are
//                 dropped with a ballot compaction              (:40-41)
//   4. scan     : hood offsets from the unique counts          (:49-52)
//   5. compact  : members                                     (:44-48)
// source_clique is the identity (:53-55).
#include <algorithm>
#include <vector>

#include "context.cuh"
#include "segsort.cuh"

namespace dpmrf_b200 {

namespace {

constexpr int kWarpsPerBlock = 8;
constexpr uint32_t kSmemCap = 1024;  // candidates per warp in the shared-memory path

__global__ void k_count_candidates(const uint32_t* __restrict__ c_off,
                                   const uint32_t* __restrict__ c_mem, uint64_t C,
                                   const uint32_t* __restrict__ g_off, uint32_t R,
                                   uint32_t* __restrict__ cnt, uint32_t* err,
                                   unsigned long long* max_cnt) {
  const uint64_t c = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  uint64_t n = 0;
  if (c < C) {
    bool bad = false;
    for (uint32_t s = c_off[c]; s < c_off[c + 1]; ++s) {
      const uint32_t m = c_mem[s];
      if (m >= R) {
        bad = true;
        break;
      }
      n += 1 + (g_off[m + 1] - g_off[m]);
    }
    if (bad) {
      atomicOr(err, 1u);
      n = 0;
    }
    cnt[c] = static_cast<uint32_t>(n);
  }
  // one atomic per warp (a single contended address otherwise serializes C atomics)
  const uint32_t n32 = n > 0xFFFFFFFFull ? 0xFFFFFFFFu : uint32_t(n);
  const uint32_t wmax = __reduce_max_sync(0xffffffffu, n32);
  if ((threadIdx.x & 31) == 0 && wmax) atomicMax(max_cnt, static_cast<unsigned long long>(wmax));
}

// Hoods with <= G candidates (every grid / brick hood): G lanes per clique.
// Lanes j < k load member j, its adjacency base and length; a segment scan
// of the lengths places candidate l (members in order, each followed by its
// neighbors, neighborhoods.cpp:31-36); the group sorts + uniques in
// registers.  kPass 0 writes the unique counts, kPass 1 the members at the
// scanned hood offsets -- no candidate scratch, no compaction pass.
template <int G, int kPass>
__global__ void __launch_bounds__(256)
    k_hood_small(const uint32_t* __restrict__ c_off, const uint32_t* __restrict__ c_mem,
                 uint64_t C, const uint32_t* __restrict__ g_off,
                 const uint32_t* __restrict__ g_nbr, uint32_t* __restrict__ uniq,
                 const uint32_t* __restrict__ h_off, uint32_t* __restrict__ members) {
  const int lane = threadIdx.x & 31;
  const int l = lane & (G - 1);
  const uint64_t c = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) / G;
  const bool cv = c < C;
  uint32_t lo = 0, k = 0;
  if (cv) {
    lo = c_off[c];
    k = c_off[c + 1] - lo;  // <= candidates <= G
  }
  uint32_t m = 0, base = 0, len = 0;
  if (cv && uint32_t(l) < k) {
    m = c_mem[lo + l];
    base = g_off[m];
    len = 1 + (g_off[m + 1] - base);
  }
  uint32_t incl = len;
#pragma unroll
  for (int o = 1; o < G; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o, G);
    if (l >= o) incl += y;
  }
  const uint32_t start = incl - len;
  const uint32_t kmax = __reduce_max_sync(0xffffffffu, k);
  uint32_t x = kPad;
  for (uint32_t j = 0; j < kmax; ++j) {
    const uint32_t sj = __shfl_sync(0xffffffffu, start, j, G);
    const uint32_t lj = __shfl_sync(0xffffffffu, len, j, G);
    const uint32_t mj = __shfl_sync(0xffffffffu, m, j, G);
    const uint32_t bj = __shfl_sync(0xffffffffu, base, j, G);
    if (j < k && uint32_t(l) >= sj && uint32_t(l) < sj + lj)
      x = uint32_t(l) == sj ? mj : g_nbr[bj + (uint32_t(l) - sj - 1)];
  }
  bool keep;
  uint32_t rank;
  const uint32_t u = group_sort_unique<G>(x, lane, keep, rank);
  if (!cv) return;
  if (kPass == 0) {
    if (l == 0) uniq[c] = u;
  } else if (keep) {
    members[h_off[c] + rank] = x;
  }
}

template <int G>
void launch_hood_small(const uint32_t* c_off, const uint32_t* c_mem, uint64_t C,
                       const uint32_t* g_off, const uint32_t* g_nbr, uint32_t* uniq,
                       uint32_t* h_off, uint32_t* members, int pass, cudaStream_t st) {
  const unsigned grid = grid_for(C * G, 256);
  if (pass == 0)
    k_hood_small<G, 0><<<grid, 256, 0, st>>>(c_off, c_mem, C, g_off, g_nbr, uniq, h_off, members);
  else
    k_hood_small<G, 1><<<grid, 256, 0, st>>>(c_off, c_mem, C, g_off, g_nbr, uniq, h_off, members);
  CK_LAUNCH();
}

void hood_small(int G, const uint32_t* c_off, const uint32_t* c_mem, uint64_t C,
                const uint32_t* g_off, const uint32_t* g_nbr, uint32_t* uniq, uint32_t* h_off,
                uint32_t* members, int pass, cudaStream_t st) {
  switch (G) {
    case 8: launch_hood_small<8>(c_off, c_mem, C, g_off, g_nbr, uniq, h_off, members, pass, st); break;
    case 16: launch_hood_small<16>(c_off, c_mem, C, g_off, g_nbr, uniq, h_off, members, pass, st); break;
    default: launch_hood_small<32>(c_off, c_mem, C, g_off, g_nbr, uniq, h_off, members, pass, st); break;
  }
}

// Position p of clique c's candidate list: member, then its neighbors, in
// member order (neighborhoods.cpp:31-36).
__device__ __forceinline__ uint32_t candidate_at(const uint32_t* c_mem, uint32_t lo, uint32_t hi,
                                                 const uint32_t* g_off, const uint32_t* g_nbr,
                                                 uint32_t p) {
  for (uint32_t s = lo; s < hi; ++s) {
    const uint32_t m = c_mem[s];
    const uint32_t deg = g_off[m + 1] - g_off[m];
    if (p == 0) return m;
    if (p <= deg) return g_nbr[g_off[m] + p - 1];
    p -= 1 + deg;
  }
  return kPad;
}

// Sort + unique of every clique with <= kSmemCap candidates; larger ones are
// left to k_big_clique (uniq written there).
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    k_sort_unique(const uint32_t* __restrict__ c_off, const uint32_t* __restrict__ c_mem,
                  uint64_t C, const uint32_t* __restrict__ g_off,
                  const uint32_t* __restrict__ g_nbr, const uint32_t* __restrict__ cnt,
                  const uint32_t* __restrict__ cand_off, uint32_t* __restrict__ scratch,
                  uint32_t* __restrict__ uniq) {
  __shared__ uint32_t buf[kWarpsPerBlock][kSmemCap];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t c = uint64_t(blockIdx.x) * kWarpsPerBlock + w;
  if (c >= C) return;
  const uint32_t n = cnt[c];
  const uint32_t lo = c_off[c], hi = c_off[c + 1];
  uint32_t* out = scratch + cand_off[c];
  if (n <= 32) {
    uint32_t x = lane < int(n) ? candidate_at(c_mem, lo, hi, g_off, g_nbr, lane) : kPad;
    x = warp_bitonic32(x, lane);
    const uint32_t u = warp_unique_chunk(x, lane < int(n), 0, false, out, lane);
    if (lane == 0) uniq[c] = u;
    return;
  }
  if (n > kSmemCap) return;  // k_big_clique
  uint32_t* b = buf[w];
  // gather: the warp walks the members; each member's segment is copied by lanes
  uint32_t pos = 0;
  for (uint32_t s = lo; s < hi; ++s) {
    const uint32_t m = c_mem[s];
    const uint32_t a0 = g_off[m], deg = g_off[m + 1] - a0;
    if (lane == 0) b[pos] = m;
    for (uint32_t i = lane; i < deg; i += 32) b[pos + 1 + i] = g_nbr[a0 + i];
    pos += 1 + deg;
  }
  uint32_t P = 64;
  while (P < n) P <<= 1;
  for (uint32_t i = n + lane; i < P; i += 32) b[i] = kPad;
  __syncwarp();
  bitonic_sort(b, P, lane, 32, [] { __syncwarp(); });
  const uint32_t written = warp_unique_sorted(b, n, out, lane);
  if (lane == 0) uniq[c] = written;
}

// One block per oversized clique: bitonic sort in a global scratch region.
__global__ void __launch_bounds__(1024)
    k_big_clique(const uint32_t* __restrict__ big, const uint64_t* __restrict__ big_tmp_off,
                 const uint32_t* __restrict__ c_off, const uint32_t* __restrict__ c_mem,
                 const uint32_t* __restrict__ g_off, const uint32_t* __restrict__ g_nbr,
                 const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ cand_off,
                 uint32_t* __restrict__ scratch, uint32_t* __restrict__ tmp,
                 uint32_t* __restrict__ uniq) {
  const uint32_t c = big[blockIdx.x];
  const uint32_t n = cnt[c];
  uint32_t* b = tmp + big_tmp_off[blockIdx.x];
  const uint64_t P = big_tmp_off[blockIdx.x + 1] - big_tmp_off[blockIdx.x];
  uint32_t pos = 0;
  for (uint32_t s = c_off[c]; s < c_off[c + 1]; ++s) {
    const uint32_t m = c_mem[s];
    const uint32_t a0 = g_off[m], deg = g_off[m + 1] - a0;
    if (threadIdx.x == 0) b[pos] = m;
    for (uint32_t i = threadIdx.x; i < deg; i += blockDim.x) b[pos + 1 + i] = g_nbr[a0 + i];
    pos += 1 + deg;
  }
  for (uint64_t i = n + threadIdx.x; i < P; i += blockDim.x) b[i] = kPad;
  __syncthreads();
  bitonic_sort(b, P, threadIdx.x, blockDim.x, [] { __syncthreads(); });
  // unique, in order, by warp 0
  if (threadIdx.x >= 32) return;
  const uint32_t written = warp_unique_sorted(b, n, scratch + cand_off[c], threadIdx.x);
  if (threadIdx.x == 0) uniq[c] = written;
}

__global__ void k_compact_members(const uint32_t* __restrict__ scratch,
                                  const uint32_t* __restrict__ cand_off,
                                  const uint32_t* __restrict__ h_off, uint64_t C,
                                  uint32_t* __restrict__ members) {
  const int lane = threadIdx.x & 31;
  const uint64_t c = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (c >= C) return;
  const uint32_t src = cand_off[c], dst = h_off[c], n = h_off[c + 1] - dst;
  for (uint32_t i = lane; i < n; i += 32) members[dst + i] = scratch[src + i];
}

}  // namespace

void build_neighborhoods_device(dpmrf_context* ctx, uint64_t C, const uint32_t* c_off_host,
                                const uint32_t* c_mem_host) {
  cudaStream_t st = ctx->stream;
  const uint64_t CS = c_off_host[C];
  uint32_t* c_off = ctx->tmp_u32[0].ensure(C + 1);
  uint32_t* c_mem = ctx->tmp_u32[1].ensure(CS);
  CK(cudaMemcpyAsync(c_off, c_off_host, (C + 1) * 4, cudaMemcpyHostToDevice, st));
  if (CS) CK(cudaMemcpyAsync(c_mem, c_mem_host, CS * 4, cudaMemcpyHostToDevice, st));
  build_neighborhoods_from(ctx, C, c_off, c_mem);
}

// Same, from device-resident cliques (e.g. dpmrf_enumerate_maximal_cliques).
void build_neighborhoods_from(dpmrf_context* ctx, uint64_t C, const uint32_t* c_off,
                              const uint32_t* c_mem) {
  cudaStream_t st = ctx->stream;
  uint32_t* cnt = ctx->tmp_u32[2].ensure(C + 1);
  uint32_t* cand_off = ctx->tmp_u32[3].ensure(C + 1);
  uint32_t* err = ctx->prep_err.ensure(2);
  unsigned long long* maxc = ctx->tmp_u64[0].ensure(1);
  CK(cudaMemsetAsync(err, 0, 8, st));
  CK(cudaMemsetAsync(maxc, 0, 8, st));
  if (C) {
    k_count_candidates<<<grid_for(C, 256), 256, 0, st>>>(c_off, c_mem, C, ctx->g_off.get(),
                                                         ctx->R, cnt, err, maxc);
    CK_LAUNCH();
  }
  uint32_t h_err = 0, h_total = 0;
  unsigned long long h_max = 0;
  CK(cudaMemcpyAsync(&h_err, err, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&h_max, maxc, 8, cudaMemcpyDeviceToHost, st));
  ctx->sync();
  if (h_err) fail(DPMRF_OUT_OF_RANGE, "build_neighborhoods: clique member >= num_vertices");
  if (h_max <= 32) {  // every hood fits a lane group: two register passes, no scratch
    const int G = h_max <= 8 ? 8 : (h_max <= 16 ? 16 : 32);
    uint32_t* uniq = ctx->tmp_u32[5].ensure(C + 1);
    uint32_t* h_off = ctx->h_off.ensure(C + 1);
    if (C) hood_small(G, c_off, c_mem, C, ctx->g_off.get(), ctx->g_nbr.get(), uniq, h_off,
                      nullptr, 0, st);
    exclusive_scan_u32(uniq, h_off, C, h_off + C, ctx->scan, st);
    uint32_t S = 0;
    CK(cudaMemcpyAsync(&S, h_off + C, 4, cudaMemcpyDeviceToHost, st));
    ctx->sync();
    uint32_t* members = ctx->h_mem.ensure(S);
    if (C) hood_small(G, c_off, c_mem, C, ctx->g_off.get(), ctx->g_nbr.get(), uniq, h_off,
                      members, 1, st);
    ctx->H = C;
    ctx->S = S;
    ctx->sync();
    return;
  }
  exclusive_scan_u32(cnt, cand_off, C, cand_off + C, ctx->scan, st);
  CK(cudaMemcpyAsync(&h_total, cand_off + C, 4, cudaMemcpyDeviceToHost, st));
  ctx->sync();
  uint32_t* scratch = ctx->tmp_u32[4].ensure(h_total);
  uint32_t* uniq = ctx->tmp_u32[5].ensure(C + 1);
  if (C) {
    k_sort_unique<<<grid_for(C, kWarpsPerBlock), kWarpsPerBlock * 32, 0, st>>>(
        c_off, c_mem, C, ctx->g_off.get(), ctx->g_nbr.get(), cnt, cand_off, scratch, uniq);
    CK_LAUNCH();
  }
  if (h_max > kSmemCap) {
    // rare: hoods with > 1024 candidates (very high-degree regions)
    std::vector<uint32_t> h_cnt(C);
    CK(cudaMemcpyAsync(h_cnt.data(), cnt, C * 4, cudaMemcpyDeviceToHost, st));
    ctx->sync();
    std::vector<uint32_t> big;
    std::vector<uint64_t> toff{0};
    for (uint64_t c = 0; c < C; ++c)
      if (h_cnt[c] > kSmemCap) {
        uint64_t P = 1;
        while (P < h_cnt[c]) P <<= 1;
        big.push_back(static_cast<uint32_t>(c));
        toff.push_back(toff.back() + P);
      }
    DevBuf<uint32_t> big_list;
    DevBuf<unsigned long long> big_off;
    DevBuf<uint32_t> big_tmp;
    uint32_t* bl = big_list.ensure(big.size());
    auto* bo = reinterpret_cast<uint64_t*>(big_off.ensure(toff.size()));
    uint32_t* bt = big_tmp.ensure(toff.back());
    CK(cudaMemcpyAsync(bl, big.data(), big.size() * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(bo, toff.data(), toff.size() * 8, cudaMemcpyHostToDevice, st));
    k_big_clique<<<static_cast<unsigned>(big.size()), 1024, 0, st>>>(
        bl, bo, c_off, c_mem, ctx->g_off.get(), ctx->g_nbr.get(), cnt, cand_off, scratch, bt,
        uniq);
    CK_LAUNCH();
    ctx->sync();
  }
  uint32_t* h_off = ctx->h_off.ensure(C + 1);
  exclusive_scan_u32(uniq, h_off, C, h_off + C, ctx->scan, st);
  uint32_t S = 0;
  CK(cudaMemcpyAsync(&S, h_off + C, 4, cudaMemcpyDeviceToHost, st));
  ctx->sync();
  uint32_t* members = ctx->h_mem.ensure(S);
  if (C) {
    k_compact_members<<<grid_for(C * 32, 256), 256, 0, st>>>(scratch, cand_off, h_off, C,
                                                             members);
    CK_LAUNCH();
  }
  ctx->H = C;
  ctx->S = S;
  ctx->sync();
}

}  // namespace dpmrf_b200
