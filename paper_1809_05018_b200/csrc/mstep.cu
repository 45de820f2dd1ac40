// mstep.cu -- sm_100a kernels of the M-step and the EM tail of the
// optimization phase: the stable grouping of region means by label (tile
// counts + scatter), the fixed-topology leaf folds and pairwise trees of
// update_parameters (proj/src/mrf/engine.cpp:193-223) and of the total energy
// (dpp::reduce, kernels.hpp:124-139; optimize.cpp:64-65), the EM record /
// window / next label terms with the device log (optimize.cpp:60-71,
// model.hpp:48-60), and the partitioned run's per-rank folds.
#include <algorithm>
#include <cstdlib>

#include "engine_dev.cuh"
#include "fold_trees.cuh"

namespace dpmrf_b200 {

namespace {



// Phase probe (build with EXTRA=-DDPMRF_PROBE only): %globaltimer stamps of
// the M-step folds, per block (entry, after pdl_wait, staged, chain done) and
// for the ticket block (ticket, trees done, end); read by dpmrf_probe_read.
#ifdef DPMRF_PROBE
__device__ unsigned long long g_probe_blk[2][256][8];
__device__ unsigned long long g_probe_tail[2][4];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PROBE_BLK(k, i) \
  do { if (threadIdx.x == 0 && blockIdx.x < 256) g_probe_blk[k][blockIdx.x][i] = gtimer(); } while (0)
#define PROBE_BLK_T(k, i) \
  do { if (blockIdx.x < 256) g_probe_blk[k][blockIdx.x][i] = gtimer(); } while (0)
#define PROBE_TAIL(k, i) do { if (threadIdx.x == 0) g_probe_tail[k][i] = gtimer(); } while (0)
#else
#define PROBE_BLK(k, i) do {} while (0)
#define PROBE_BLK_T(k, i) do {} while (0)
#define PROBE_TAIL(k, i) do {} while (0)
#endif

// ---------------------------------------------------------------------------
// M-step: stable grouping of region means by label + fixed-topology folds.
//   update_parameters  engine.cpp:193-223 (sort_by_key stable, reduce_by_key
//                      fold_range per run, kernels.hpp:226-253)
//   dpp::reduce        kernels.hpp:124-139 (total energy, optimize.cpp:64-65)
// Launches per EM iteration: the grouping (k_label_scatter_small, or
// k_tile_chunks / k_tile_offsets / k_label_scatter_warp on large graphs), then the
// folds: k_fold_sum_ldg + k_fold_sq_cluster (few leaves), k_mstep_stream
// (many leaves), each finishing with the pairwise trees.  The per-tile label counts come from the
// last executed vertex pass (double-buffered by iteration parity).
// ---------------------------------------------------------------------------
// Label counts per 256-vertex tile (when the vertex pass did not count
// them): __match_any_sync groups the warp's lanes by label, per-warp counts
// in shared memory are summed per tile.
__global__ void __launch_bounds__(kTileThreads)
    k_label_counts(const uint8_t* lab_even, const uint8_t* lab_odd, const uint32_t* unconv,
                   int map_max, int fixed, uint32_t R, uint32_t M,
                   uint32_t* __restrict__ tile_counts) {
  extern __shared__ uint32_t wcnt[];  // [warp][M]
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kWarps = kTileThreads / 32;
  if (em_skipped(unconv)) return;
  const uint8_t* lab = final_labels(lab_even, lab_odd, unconv, map_max, fixed);
  for (uint32_t i = threadIdx.x; i < kWarps * M; i += kTileThreads) wcnt[i] = 0;
  __syncthreads();
  const uint64_t tile = blockIdx.x;
  const uint64_t v = tile * kTileVerts + threadIdx.x;
  const bool valid = v < R;
  const uint32_t l = valid ? lab[v] : 0xFFFFFFFFu;
  const unsigned peers = __match_any_sync(0xffffffffu, l);
  const uint32_t rank_in_warp = __popc(peers & ((1u << lane) - 1u));
  if (valid && rank_in_warp == 0) wcnt[warp * M + l] = __popc(peers);
  __syncthreads();
  for (uint32_t q = threadIdx.x; q < M; q += kTileThreads) {
    uint32_t c = 0;
    for (int w = 0; w < kWarps; ++w) c += wcnt[w * M + q];
    tile_counts[tile * M + q] = c;
  }
}

// Stable grouping of the region means by label (== stable sort_by_key of the
// labels, engine.cpp:201) with one WARP per 256-vertex tile (eight tiles per
// block): the warp walks its tile in vertex order, 32 at a time; a lane's
// position is its label's start + the tile's offset for that label + the
// warp's running count of that label + its rank among the lanes of the same
// label (__match_any_sync).  The running counts live in shared memory, so the
// stable rank needs no block barrier; the tile's means and labels are loaded
// up front (eight independent loads per lane in flight).  (One block per tile
// with a per-warp count exchange: 41.8 us at 16384^2; this: M-step -15 us/EM.)
constexpr int kScatterIters = kTileVerts / 32;
__global__ void __launch_bounds__(kTileThreads)
    k_label_scatter_warp(const uint8_t* lab_even, const uint8_t* lab_odd, const uint32_t* unconv,
                         int map_max, int fixed, uint32_t R, uint32_t M,
                         const double* __restrict__ mean, const uint32_t* __restrict__ tile_base,
                         const uint32_t* __restrict__ layout, double* __restrict__ x) {
  extern __shared__ uint32_t run_all[];  // [warp][M]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t tile = uint64_t(blockIdx.x) * (kTileThreads / 32) + warp;
  uint32_t* run = run_all + warp * M;
  for (uint32_t l = lane; l < M; l += 32) run[l] = 0;
  const uint64_t v0 = tile * kTileVerts + lane;
  double mv[kScatterIters];
#pragma unroll
  for (int i = 0; i < kScatterIters; ++i) {  // (means are static: before the wait)
    const uint64_t v = v0 + 32 * i;
    mv[i] = v < R ? mean[v] : 0.0;
  }
  pdl_wait();
  if (em_skipped(unconv)) return;
  const uint8_t* lab = final_labels(lab_even, lab_odd, unconv, map_max, fixed);
  uint32_t lv[kScatterIters];
#pragma unroll
  for (int i = 0; i < kScatterIters; ++i) {
    const uint64_t v = v0 + 32 * i;
    lv[i] = v < R ? lab[v] : 0xFFFFFFFFu;
  }
  const uint32_t* label_start = layout + M;
  const uint32_t* tb = tile_base + tile * M;
  __syncwarp();
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < kScatterIters; ++i) {
    const uint32_t l = lv[i];
    const unsigned peers = __match_any_sync(0xffffffffu, l);
    const uint32_t rank = __popc(peers & lt);
    if (l != 0xFFFFFFFFu) x[label_start[l] + tb[l] + run[l] + rank] = mv[i];
    __syncwarp();
    if (l != 0xFFFFFFFFu && rank == 0) run[l] += __popc(peers);
    __syncwarp();
  }
}

__global__ void __launch_bounds__(kTileThreads)
    k_label_scatter_small(const uint8_t* lab_even, const uint8_t* lab_odd,
                          const uint32_t* unconv, const uint32_t* count_sel, int map_max,
                          int fixed, uint32_t R, uint32_t M, uint64_t Hs,
                          const double* __restrict__ mean, const uint32_t* __restrict__ counts_buf,
                          uint32_t tiles, uint32_t* __restrict__ layout, double* __restrict__ x) {
  extern __shared__ uint32_t wcnt[];
  pdl_wait();
  if (em_skipped(unconv)) return;
  label_scatter_small_body<false>(lab_even, lab_odd, unconv, count_sel, map_max, fixed, R, M, Hs,
                                  mean, counts_buf, tiles, layout, x, blockIdx.x, wcnt);
}

// Single block: per-label exclusive scan over tiles; label starts; leaf layout.
// layout = n[M] | label_start[M+1] | leaf_start[M+2] (series M = hood energies)
// Large graphs: per-label tile offsets with two many-block kernels (one
// block per 1024 tiles): k_tile_chunks sums each chunk's counts per label,
// k_tile_offsets adds the preceding chunks' sums to a block scan of its own
// tiles.  Integer sums -- any order gives the same offsets.
// layout = n[M] | label_start[M+1] | leaf_start[M+2] (series M = hood energies)
constexpr uint32_t kTileChunk = 1024;

__device__ __forceinline__ uint32_t block_sum_1024(uint32_t v, uint32_t* red) {
  v = __reduce_add_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  uint32_t t = 0;
  if (threadIdx.x < 32) t = __reduce_add_sync(0xffffffffu, threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0u);
  if (threadIdx.x == 0) red[32] = t;
  __syncthreads();
  const uint32_t r = red[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(1024)
    k_tile_chunks(const uint32_t* __restrict__ counts_buf, const uint32_t* __restrict__ unconv,
                  int map_max, int fixed, uint32_t tiles, uint32_t M,
                  uint32_t* __restrict__ chunk_sum) {
  __shared__ uint32_t red[33];
  pdl_wait();
  if (em_skipped(unconv)) return;
  const uint32_t* tc = final_counts(counts_buf, tiles, M, unconv, map_max, fixed);
  const uint64_t i = uint64_t(blockIdx.x) * kTileChunk + threadIdx.x;
  for (uint32_t l = 0; l < M; ++l) {
    const uint32_t c = i < tiles ? tc[i * M + l] : 0u;
    const uint32_t s = block_sum_1024(c, red);
    if (threadIdx.x == 0) chunk_sum[uint64_t(blockIdx.x) * M + l] = s;
  }
}

__global__ void __launch_bounds__(1024)
    k_tile_offsets(const uint32_t* __restrict__ counts_buf, const uint32_t* __restrict__ unconv,
                   int map_max, int fixed, uint32_t* __restrict__ tile_base, uint32_t tiles,
                   uint32_t M, uint64_t Hs, uint32_t* __restrict__ layout,
                   const uint32_t* __restrict__ chunk_sum, uint32_t nchunks) {
  __shared__ uint32_t warp_sums[32];
  __shared__ uint32_t red[33];
  pdl_wait();
  if (em_skipped(unconv)) return;
  const uint32_t* tc = final_counts(counts_buf, tiles, M, unconv, map_max, fixed);
  const uint64_t i = uint64_t(blockIdx.x) * kTileChunk + threadIdx.x;
  for (uint32_t l = 0; l < M; ++l) {
    uint32_t pre = 0, tot = 0;  // preceding chunks / all chunks of label l
    for (uint32_t c = threadIdx.x; c < nchunks; c += blockDim.x) {
      const uint32_t v = chunk_sum[uint64_t(c) * M + l];
      tot += v;
      pre += c < blockIdx.x ? v : 0u;
    }
    pre = block_sum_1024(pre, red);
    tot = block_sum_1024(tot, red);
    const uint32_t cnt = i < tiles ? tc[i * M + l] : 0u;
    const uint32_t ex = block_exclusive_scan(cnt, warp_sums, nullptr);
    if (i < tiles) tile_base[i * M + l] = pre + ex;
    if (blockIdx.x == 0 && threadIdx.x == 0) layout[l] = tot;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    __threadfence_block();
    uint32_t* label_start = layout + M;
    uint32_t* leaf_start = layout + 2 * M + 1;
    uint32_t s = 0, lf = 0;
    for (uint32_t l = 0; l < M; ++l) {
      label_start[l] = s;
      leaf_start[l] = lf;
      s += layout[l];
      lf += (layout[l] + kFoldLeaf - 1) / kFoldLeaf;
    }
    label_start[M] = s;
    leaf_start[M] = lf;
    lf += uint32_t((Hs + kFoldLeaf - 1) / kFoldLeaf);
    leaf_start[M + 1] = lf;
  }
}

__device__ __forceinline__ uint32_t series_of(const uint32_t* leaf_start, uint32_t nseries,
                                              uint32_t leaf) {
  uint32_t s = 0;
  while (s + 1 < nseries && leaf >= leaf_start[s + 1]) ++s;
  return s;
}

// Leaf folds (fold_leaf, kernels.hpp:37-42): each 1024-element leaf is a
// strictly sequential left fold seeded by its first element -- the chain of
// dependent adds cannot be reassociated without changing bits.  Leaf
// partials combine with the pairwise tree of kernels.hpp:45-51 (bottom-up
// adjacent pairing == the split at bit_floor(n-1), fold_trees.cuh).
// kLeavesPerBlock: leaves per block of k_row_leaves (the partitioned run's
// hood-series leaves, staged by the whole block, one chain per leaf).
#ifndef DPMRF_LEAVES_PER_BLOCK
#define DPMRF_LEAVES_PER_BLOCK 8
#endif
constexpr int kLeavesPerBlock = DPMRF_LEAVES_PER_BLOCK;
constexpr int kLeafStride = kFoldLeaf + 1;

// EM bookkeeping after the M-step (one warp): record the EM log, apply the
// EM-level window (optimize.cpp:66-71) and write the next EM's label terms
// with the device log (make_label_terms, model.hpp:48-60).  merged: called
// from the sq-pass tail of the device-resident loop, which also stops the
// loop directly and re-arms the MAP counters for the next EM (no separate
// prologue / epilogue launches); otherwise the stop is left pending for
// k_em_prologue.
// What em_record reads from global state that does not depend on the
// M-step's results: loaded by the sq-pass tail before its trees, so those
// round trips overlap the tree instead of following it.
constexpr int kPrefetchWin = 8;
struct EmPrefetch {
  int T;
  uint32_t e;
  double hist[kPrefetchWin];  // em_hist[e - 1 - i]
};

__device__ __forceinline__ void em_prefetch(const EmEpilogueArgs& a, EmPrefetch* pf) {
  pf->T = executed_iters(a.unconv, a.map_max, a.fixed);
  const uint32_t e = a.unconv[kEmCount];
  pf->e = e;
  for (int i = 1; i <= a.L && i <= kPrefetchWin; ++i)
    pf->hist[i - 1] = int(e) >= i ? a.em_hist[e - i] : 0.0;
}

// log c_k of log_fast (common.cuh), per device, built once (init_log_table).
__device__ LogTable g_log_table;

__global__ void k_init_log_table() {
  const int k = threadIdx.x;
  if (k < kLogTable) {
    const dd_t r = log_dd(0.75 + k * 0.0078125);
    g_log_table.hi[k] = r.hi;
    g_log_table.lo[k] = r.lo;
  }
}

// vals: this EM's [total, T, mu(M), sigma(M)] -- a.em_out, or the caller's
// shared-memory copy (saves the global round trip).
__device__ void em_record(const EmEpilogueArgs& a, bool merged, const EmPrefetch* pf = nullptr,
                          const double* thi = g_log_table.hi, const double* tlo = g_log_table.lo,
                          const double* vals = nullptr) {
  const int lane = threadIdx.x & 31;
  const int T = pf ? pf->T : executed_iters(a.unconv, a.map_max, a.fixed);
  const uint32_t e = pf ? pf->e : a.unconv[kEmCount];
  const uint32_t M = a.M;
  if (!vals) vals = a.em_out;
  double* rec = a.em_rec + uint64_t(e) * (3 + 3 * M);
  for (uint32_t l = lane; l < M; l += 32) {  // one lane per label evaluates the device log
    const double mu = vals[2 + l], sg = vals[2 + M + l];
    const double ls = log_fast(sg, thi, tlo);
    rec[3 + l] = mu;
    rec[3 + M + l] = sg;
    rec[3 + 2 * M + l] = ls;
    a.terms[l] = mu;
    a.terms[M + l] = __dmul_rn(2.0, __dmul_rn(sg, sg));
    a.terms[2 * M + l] = ls;
  }
  __syncwarp();
  if (lane != 0) return;
  const double total = vals[0];
  a.em_hist[e] = total;
  uint32_t conv = 0;
  if (int(e) + 1 >= a.L + 1) {
    conv = 1;
    for (int i = 1; i <= a.L; ++i) {
      const double prev = pf && i <= kPrefetchWin ? pf->hist[i - 1] : a.em_hist[e - i];
      if (!(fabs(__dsub_rn(total, prev)) < a.tol)) conv = 0;
    }
  }
  rec[0] = total;
  rec[1] = static_cast<double>(T);
  rec[2] = static_cast<double>(conv);
  a.unconv[kEmCount] = e + 1;
  if (conv && !a.fixed) a.unconv[merged ? kEmDone : kEmPending] = 1;
  if (merged)
    for (int t = 0; t < a.map_max; ++t) a.unconv[t] = 0;
}

// Trees only (the partitioned run): every rank folded its own leaves and the
// partials were gathered into `partials` (label series, global leaf order)
// and hood_parts (the hood-energy series); one block runs the pairwise trees
// of kernels.hpp:45-51 (block_series_tree) and publishes mu (sum pass) or
// sigma and the EM output (sq pass), exactly as the one-device M-step.
template <bool kSq>
__global__ void __launch_bounds__(256)
    k_fold_trees(const uint32_t* __restrict__ layout, uint32_t M,
                 const uint32_t* __restrict__ unconv, int map_max, int fixed, double* params,
                 const double* __restrict__ partials, const double* __restrict__ hood_parts,
                 double* em_out) {
  extern __shared__ double scratch[];  // roots (root_cap) | 8 warps x kTreeScratch
  __shared__ uint32_t lay[4 * kMaxLabels + 4];
  pdl_wait();
  if (em_skipped(unconv)) return;
  for (uint32_t i = threadIdx.x; i < 4 * M + 4; i += blockDim.x) lay[i] = layout[i];
  __syncthreads();
  const uint32_t* n = lay;
  const uint32_t* leaf_start = lay + 2 * M + 1;
  const uint32_t nch_max = (leaf_start[M + 1] + kFoldLeaf - 1) / kFoldLeaf + 1;
  double* roots = scratch;
  double* qw = scratch + (nch_max + 1) / 2 * 2 + (threadIdx.x >> 5) * kTreeScratch;
  for (uint32_t s = 0; s < (kSq ? M : M + 1); ++s) {
    const uint32_t cnt = leaf_start[s + 1] - leaf_start[s];
    const double* p = s < M ? partials + leaf_start[s] : hood_parts;
    const double folded = cnt ? block_series_tree(p, cnt, roots, qw) : 0.0;
    if (threadIdx.x != 0) continue;
    if (s < M) {
      if (n[s] != 0) {  // empty labels keep their previous parameters (engine.cpp:209-220)
        const double count = static_cast<double>(n[s]);
        if (!kSq) {
          params[s] = __ddiv_rn(folded, count);
        } else {
          const double sd = __dsqrt_rn(__ddiv_rn(folded, count));
          params[M + s] = sd < kSigmaFloor ? kSigmaFloor : sd;
        }
      }
      if (kSq) {  // the final pass publishes (mu, sigma) of every label
        em_out[2 + s] = params[s];
        em_out[2 + M + s] = params[M + s];
      }
    } else {
      // total energy: dpp::reduce(..., 0.0) -> identity only for empty input
      em_out[0] = cnt == 0 ? 0.0 : folded;
      em_out[1] = static_cast<double>(unconv ? executed_iters(unconv, map_max, fixed) : 0);
    }
  }
}


// ---------------------------------------------------------------------------
// M-step folds, TMA-fed (the single-device path; k_fold_trees above serves the
// partitioned schedule's distributed folds).
//   k_fold_sum: lane j < kLPB of a one-warp block owns leaf blockIdx*kLPB + j
//     of the sum pass (the label series of x, then the hood-energy series).
//     It fetches the leaf with two cp.async.bulk copies (halves, one mbarrier
//     each: no thread-issued loads compete with the chain's shared-memory
//     reads) and starts the dependent left fold (fold_leaf,
//     kernels.hpp:37-42) as soon as the first half has landed.  No tail: the
//     grid releases the sq pass at once (griddepcontrol.launch_dependents).
//   k_fold_sq: fetches its label leaves of x BEFORE griddepcontrol.wait (x
//     and the layout come from the MAP launches, complete by then); after
//     the wait every block evaluates mu of its own labels from the sum-pass
//     partials (the pairwise tree of kernels.hpp:45-51, redundantly per
//     block, instead of a serial last-block tail between the passes), folds
//     (x - mu)^2 (engine.cpp:213-217), and the last block (ticket) runs the
//     sigma and total-energy trees, publishes the parameters and records the
//     EM iteration (em_record).
// Leaves are fetched as the 16-byte-aligned superset of [src, src + len):
// rows start at an even double, the data at offset 0 or 1; x and the
// hood-energy ring are allocated with 2 doubles of slack for the round-up.
// ---------------------------------------------------------------------------
constexpr uint32_t kFoldPitch = kFoldLeaf + 2;  // doubles per staged leaf (16-B rows)
constexpr uint32_t kFoldHalf = kFoldLeaf / 2;
constexpr int kSqThreads = 128;

struct FoldArgs {
  const double* x;         // R region means grouped by label (stable)
  const uint32_t* layout;  // n[M] | label_start[M+1] | leaf_start[M+2]
  uint32_t M;
  const double* hist;      // hood-energy ring (ring x Hs)
  uint64_t Hs;
  int ring;
  const uint32_t* unconv;  // nullptr: standalone update_parameters
  int map_max;
  int fixed;
  double* params;          // mu[M] | sigma[M]: previous in, new out
  double* partials;        // sum-pass leaf partials (all series)
  double* sq_partials;     // sq-pass leaf partials (label series)
  double* em_out;          // [total, T, mu(M), sigma(M)]
  uint32_t* done;          // sq-pass ticket (re-armed by the last block)
  EmEpilogueArgs ep;
  int merged;
  uint32_t root_cap;       // shared chunk-root slots of the sq pass (>= all series' chunks)
  // Many-leaf graphs: chunk roots folded by the passes themselves (nullptr:
  // the trees read the leaf partials).  A chunk is an aligned run of 1024
  // leaves of one series; its root is exactly the level-10 node of the
  // series' tree (fold_trees.cuh), so a series' root is the tree over its
  // chunk roots.
  double* roots_sum;       // chunk roots of the sum pass (all series)
  double* roots_sq;        // chunk roots of the sq pass (label series)
  uint32_t* tickets;       // per chunk: leaves folded so far (sum | sq halves; self re-arming)
};

constexpr uint32_t kMaxChunks = 8192;  // chunk tickets per pass

// first chunk of series s: the chunks of the series before it
__device__ __forceinline__ uint32_t chunk_base(const uint32_t* leaf_start, uint32_t s) {
  uint32_t b = 0;
  for (uint32_t i = 0; i < s; ++i) b += (leaf_start[i + 1] - leaf_start[i] + kFoldLeaf - 1) / kFoldLeaf;
  return b;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait0(uint64_t* bar) {
  uint32_t ok = 0;
  uint32_t spins = 0;
  while (!ok) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar))
        : "memory");
    if (!ok && ++spins > (1u << 26)) __trap();  // a lost copy: fail loudly, never hang
  }
}

// Issue the fetch of leaf [src, src + len) into row; returns the data offset
// (0|1) and the staged length in doubles of the first half (*n0).
__device__ __forceinline__ uint32_t fetch_leaf(double* row, const double* src, uint32_t len,
                                               uint64_t* bar2, uint32_t* n0_out) {
  const uint32_t off = (reinterpret_cast<uintptr_t>(src) & 15u) ? 1u : 0u;
  const double* base = src - off;
  const uint32_t n = (off + len + 1u) & ~1u;
  const uint32_t n0 = n < kFoldHalf ? n : kFoldHalf;
  mbar_expect(&bar2[0], n0 * 8u);
  bulk_g2s(row, base, n0 * 8u, &bar2[0]);
  if (n > n0) {
    mbar_expect(&bar2[1], (n - n0) * 8u);
    bulk_g2s(row + n0, base + n0, (n - n0) * 8u, &bar2[1]);
  }
  *n0_out = n0;
  return off;
}

#ifndef DPMRF_FOLD_V2
#define DPMRF_FOLD_V2 1
#endif
constexpr bool kFoldV2 = DPMRF_FOLD_V2 != 0;  // 16-byte shared-memory loads in the chains

// Left fold of term(v[i]) over [i, end) onto acc, software-pipelined: the
// next 16 operands are read from shared memory while 16 dependent adds retire
// (kFoldV2: as 8 16-byte loads, after peeling one element to 16-byte
// alignment; the adds keep their order, so the bits are the same).
template <bool kSq>
__device__ __forceinline__ double fold_span(const double* v, uint32_t i, uint32_t end, double acc,
                                            double mu) {
  auto term = [&](double x) {
    if (kSq) {
      const double d = __dsub_rn(x, mu);
      return __dmul_rn(d, d);
    }
    return x;
  };
  constexpr int kG = 16;
  if (kFoldV2) {
    if (i < end && (reinterpret_cast<uintptr_t>(v + i) & 15u)) acc = __dadd_rn(acc, term(v[i++]));
    constexpr int kP = kG / 2;
    double2 cur[kP], nxt[kP];
    if (i + kG <= end) {
      const double2* w = reinterpret_cast<const double2*>(v + i);
#pragma unroll
      for (int j = 0; j < kP; ++j) cur[j] = w[j];
      while (i + 2 * kG <= end) {
#pragma unroll
        for (int j = 0; j < kP; ++j) nxt[j] = w[kP + j];
#pragma unroll
        for (int j = 0; j < kP; ++j) {
          acc = __dadd_rn(acc, term(cur[j].x));
          acc = __dadd_rn(acc, term(cur[j].y));
        }
#pragma unroll
        for (int j = 0; j < kP; ++j) cur[j] = nxt[j];
        w += kP;
        i += kG;
      }
#pragma unroll
      for (int j = 0; j < kP; ++j) {
        acc = __dadd_rn(acc, term(cur[j].x));
        acc = __dadd_rn(acc, term(cur[j].y));
      }
      i += kG;
    }
    for (; i < end; ++i) acc = __dadd_rn(acc, term(v[i]));
    return acc;
  }
  double cur[kG], nxt[kG];
  if (i + kG <= end) {
#pragma unroll
    for (int j = 0; j < kG; ++j) cur[j] = v[i + j];
    while (i + 2 * kG <= end) {
#pragma unroll
      for (int j = 0; j < kG; ++j) nxt[j] = v[i + kG + j];
#pragma unroll
      for (int j = 0; j < kG; ++j) acc = __dadd_rn(acc, term(cur[j]));
#pragma unroll
      for (int j = 0; j < kG; ++j) cur[j] = nxt[j];
      i += kG;
    }
#pragma unroll
    for (int j = 0; j < kG; ++j) acc = __dadd_rn(acc, term(cur[j]));
    i += kG;
  }
  for (; i < end; ++i) acc = __dadd_rn(acc, term(v[i]));
  return acc;
}

// fold_span<true> with the squares of the next group computed while the
// current group's dependent adds retire (the terms are independent of acc)
__device__ __forceinline__ double fold_span_sq(const double* v, uint32_t i, uint32_t end,
                                               double acc, double mu) {
  auto term = [&](double x) {
    const double d = __dsub_rn(x, mu);
    return __dmul_rn(d, d);
  };
  constexpr int kG = 16;
  if (kFoldV2) {
    if (i < end && (reinterpret_cast<uintptr_t>(v + i) & 15u)) acc = __dadd_rn(acc, term(v[i++]));
    constexpr int kP = kG / 2;
    double cur[kG];
    double2 nxt[kP];
    if (i + kG <= end) {
      const double2* w = reinterpret_cast<const double2*>(v + i);
#pragma unroll
      for (int j = 0; j < kP; ++j) {
        const double2 t = w[j];
        cur[2 * j] = term(t.x);
        cur[2 * j + 1] = term(t.y);
      }
      while (i + 2 * kG <= end) {
#pragma unroll
        for (int j = 0; j < kP; ++j) nxt[j] = w[kP + j];
#pragma unroll
        for (int j = 0; j < kP; ++j) {
          acc = __dadd_rn(acc, cur[2 * j]);
          cur[2 * j] = term(nxt[j].x);
          acc = __dadd_rn(acc, cur[2 * j + 1]);
          cur[2 * j + 1] = term(nxt[j].y);
        }
        w += kP;
        i += kG;
      }
#pragma unroll
      for (int j = 0; j < kG; ++j) acc = __dadd_rn(acc, cur[j]);
      i += kG;
    }
    for (; i < end; ++i) acc = __dadd_rn(acc, term(v[i]));
    return acc;
  }
  double cur[kG], nxt[kG];
  if (i + kG <= end) {
#pragma unroll
    for (int j = 0; j < kG; ++j) cur[j] = term(v[i + j]);
    while (i + 2 * kG <= end) {
#pragma unroll
      for (int j = 0; j < kG; ++j) nxt[j] = v[i + kG + j];
#pragma unroll
      for (int j = 0; j < kG; ++j) {
        acc = __dadd_rn(acc, cur[j]);
        cur[j] = term(nxt[j]);
      }
      i += kG;
    }
#pragma unroll
    for (int j = 0; j < kG; ++j) acc = __dadd_rn(acc, cur[j]);
    i += kG;
  }
  for (; i < end; ++i) acc = __dadd_rn(acc, term(v[i]));
  return acc;
}

// fold_leaf over a fetched row: the first half as soon as it lands, then the
// rest.  len >= 1.
template <bool kSq>
__device__ __forceinline__ double fold_fetched(const double* row, uint32_t off, uint32_t len,
                                               uint32_t n0, uint64_t* bar2, double mu) {
  const double* v = row + off;
  const uint32_t first_end = min(len, n0 - off);
  mbar_wait0(&bar2[0]);
  if ((threadIdx.x & 31) == 0) PROBE_BLK_T(kSq, 4);
  double acc = v[0];
  if (kSq) {
    const double d = __dsub_rn(acc, mu);
    acc = __dmul_rn(d, d);
  }
  acc = fold_span<kSq>(v, 1, first_end, acc, mu);
  if ((threadIdx.x & 31) == 0) PROBE_BLK_T(kSq, 5);
  if (len > first_end) {
    mbar_wait0(&bar2[1]);
    acc = fold_span<kSq>(v, first_end, len, acc, mu);
  }
  return acc;
}

// Called by one whole warp after its lanes wrote their leaf partials (lane
// holds `leaf` when valid): count the leaves into their chunks; the warp
// whose leaves complete a chunk folds that chunk's root (the tree over its
// <= 1024 partials, read through L2) and re-arms the chunk's ticket.  With
// series counters (sc), the warp completing a series' last chunk also folds
// the series root (the tree over its chunk roots) and hands it to
// on_series(s, root) on lane 0.
struct NoSeries {
  __device__ void operator()(uint32_t, double) const {}
};
template <class F = NoSeries>
__device__ void chunk_tickets(const uint32_t* leaf_start, uint32_t nseries, uint32_t leaf,
                              bool valid, const double* parts, double* roots, uint32_t* tickets,
                              double* q, uint32_t* sc = nullptr, F on_series = F{}) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t gch = 0xFFFFFFFFu, base = 0, len = 0, sr = 0;
  if (valid) {
    sr = series_of(leaf_start, nseries, leaf);
    const uint32_t qi = (leaf - leaf_start[sr]) / kFoldLeaf;
    gch = chunk_base(leaf_start, sr) + qi;
    base = leaf_start[sr] + qi * kFoldLeaf;
    len = min(kFoldLeaf, leaf_start[sr + 1] - base);
  }
  __threadfence();  // (each lane's partial) before the tickets
  const uint32_t grp = __match_any_sync(0xffffffffu, gch);
  bool last = false;
  if (valid && uint32_t(__ffs(grp) - 1) == lane) {
    const uint32_t c = __popc(grp);
    last = atomicAdd(&tickets[gch], c) + c == len;
  }
  uint32_t lasts = __ballot_sync(0xffffffffu, last);
  if (lasts) __threadfence();
  while (lasts) {
    const int src = __ffs(lasts) - 1;
    lasts &= lasts - 1;
    const uint32_t g = __shfl_sync(0xffffffffu, gch, src);
    const uint32_t b = __shfl_sync(0xffffffffu, base, src);
    const uint32_t n = __shfl_sync(0xffffffffu, len, src);
    const uint32_t s = __shfl_sync(0xffffffffu, sr, src);
    const double r = q ? warp_tree<true>(parts + b, n, q) : warp_tree1024<true>(parts + b, n);
    uint32_t series_done = 0;
    if (lane == 0) {
      roots[g] = r;
      tickets[g] = 0;
      if (sc) {
        __threadfence();
        const uint32_t nch = (leaf_start[s + 1] - leaf_start[s] + kFoldLeaf - 1) / kFoldLeaf;
        series_done = atomicAdd(&sc[s], 1u) + 1 == nch;
      }
    }
    if (__shfl_sync(0xffffffffu, series_done, 0)) {
      __threadfence();
      const uint32_t nch = (leaf_start[s + 1] - leaf_start[s] + kFoldLeaf - 1) / kFoldLeaf;
      const double root = q ? warp_tree<true>(roots + chunk_base(leaf_start, s), nch, q)
                            : warp_tree1024<true>(roots + chunk_base(leaf_start, s), nch);
      if (lane == 0) {
        on_series(s, root);
        sc[s] = 0;
      }
    }
  }
}

// Sum pass for few leaves (one block per SM): the warp stages its leaves with
// 16-byte loads (first halves, then the second halves in flight while the
// chains fold the first) -- the freshly scattered x lands faster this way
// than through bulk copies (measured: a bulk copy of a just-written x leaf
// can take ~2.8 us, the same copy again ~0.3 us).
template <int kLPB>
__global__ void __launch_bounds__(32) k_fold_sum_ldg(FoldArgs a) {
  extern __shared__ __align__(16) double stage[];  // kLPB x kFoldPitch
  const uint32_t lane = threadIdx.x;
  PROBE_BLK(0, 0);
  pdl_wait();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  PROBE_BLK(0, 1);
  const uint32_t M = a.M;
  // The layout, the skip flag and the MAP counters in ONE round trip (a lane
  // per word) when they fit a warp, instead of a chain of dependent loads
  // (skip flag -> leaf bounds -> series bounds) before the leaves' addresses.
  const uint32_t nlay = 4 * M + 4;
  const bool in_warp = nlay <= 32 && a.map_max <= 32;
  uint32_t lw = 0, cw = 1, done = 0;
  if (in_warp) {
    if (lane < nlay) lw = a.layout[lane];
    if (a.unconv) {
      done = a.unconv[kEmDone];
      if (!a.fixed && lane < uint32_t(a.map_max)) cw = a.unconv[lane];
    }
  } else {
    done = a.unconv ? a.unconv[kEmDone] : 0u;
  }
  if (done) return;
  auto lay = [&](uint32_t i) {
    return in_warp ? __shfl_sync(0xffffffffu, lw, i) : a.layout[i];
  };
  const uint32_t total = lay(3 * M + 2);  // leaf_start[M + 1]
  const double2* base[kLPB];
  uint32_t len[kLPB], off[kLPB], n2[kLPB];
  int T = 0;
  if (a.unconv) {
    if (!in_warp || a.fixed) {
      T = executed_iters(a.unconv, a.map_max, a.fixed);
    } else {  // executed_iters: one past the first zero counter, else map_max
      const uint32_t z = __ballot_sync(0xffffffffu, lane < uint32_t(a.map_max) && cw == 0);
      T = z ? __ffs(z) : a.map_max;
    }
  }
#pragma unroll
  for (int j = 0; j < kLPB; ++j) {
    const uint32_t leaf = blockIdx.x * kLPB + j;
    len[j] = 0;
    off[j] = 0;
    n2[j] = 0;
    base[j] = nullptr;
    if (leaf < total) {
      uint32_t sr = 0;  // series_of over leaf_start = layout[2M+1 ..]
      while (sr < M && leaf >= lay(2 * M + 2 + sr)) ++sr;
      const uint64_t b = uint64_t(leaf - lay(2 * M + 1 + sr)) * kFoldLeaf;
      const double* src;
      uint64_t slen;
      if (sr < M) {
        src = a.x + lay(M + sr) + b;
        slen = lay(sr);
      } else {  // the hood-energy row of the last executed MAP iteration (optimize.cpp:64-65)
        src = a.hist + uint64_t((T - 1) % a.ring) * a.Hs + b;
        slen = a.Hs;
      }
      const uint64_t rem = slen - b;
      len[j] = static_cast<uint32_t>(rem < kFoldLeaf ? rem : uint64_t(kFoldLeaf));
      off[j] = (reinterpret_cast<uintptr_t>(src) & 15u) ? 1u : 0u;
      base[j] = reinterpret_cast<const double2*>(src - off[j]);
      n2[j] = (off[j] + len[j] + 1u) / 2u;  // 16-byte vectors, <= 513
    }
  }
  constexpr uint32_t kH2 = kFoldHalf / 2;  // vectors in the first part (256)
  {
    double2 r[kLPB][kH2 / 32];
#pragma unroll
    for (int j = 0; j < kLPB; ++j)
#pragma unroll
      for (int q = 0; q < int(kH2 / 32); ++q) {
        const uint32_t i = q * 32 + lane;
        r[j][q] = i < n2[j] ? __ldcg(base[j] + i) : make_double2(0.0, 0.0);
      }
#pragma unroll
    for (int j = 0; j < kLPB; ++j)
#pragma unroll
      for (int q = 0; q < int(kH2 / 32); ++q)
        reinterpret_cast<double2*>(stage + j * kFoldPitch)[q * 32 + lane] = r[j][q];
  }
  __syncwarp();
  PROBE_BLK_T(0, 2);
  constexpr int kQ2 = (kFoldPitch / 2 - kH2 + 31) / 32;  // second-part vectors per lane (9)
  double2 r2[kLPB][kQ2];
#pragma unroll
  for (int j = 0; j < kLPB; ++j)
#pragma unroll
    for (int q = 0; q < kQ2; ++q) {
      const uint32_t i = kH2 + q * 32 + lane;
      r2[j][q] = i < n2[j] ? __ldcg(base[j] + i) : make_double2(0.0, 0.0);
    }
  // the chains fold the first parts while the second parts are in flight
  uint32_t my_len = 0, my_off = 0;
#pragma unroll
  for (int j = 0; j < kLPB; ++j)
    if (lane == uint32_t(j)) {
      my_len = len[j];
      my_off = off[j];
    }
  const double* v = stage + lane * kFoldPitch + my_off;
  const uint32_t first_end = min(my_len, kFoldHalf - my_off);
  double acc = 0.0;
#ifdef DPMRF_PROBE
  const long long c0 = clock64();
  const unsigned long long g0 = gtimer();
#endif
  if (my_len) acc = fold_span<false>(v, 1, first_end, v[0], 0.0);
#ifdef DPMRF_PROBE
  const long long c1 = clock64();
  const unsigned long long g1 = gtimer();
  if (lane == 0 && blockIdx.x < 256) {
    g_probe_blk[0][blockIdx.x][6] = static_cast<unsigned long long>(c1 - c0);
    g_probe_blk[0][blockIdx.x][7] = g1 - g0;
  }
#endif
  if ((lane & 31) == 0) PROBE_BLK_T(0, 5);
#pragma unroll
  for (int j = 0; j < kLPB; ++j)
#pragma unroll
    for (int q = 0; q < kQ2; ++q) {
      const uint32_t i = kH2 + q * 32 + lane;
      if (i < kFoldPitch / 2) reinterpret_cast<double2*>(stage + j * kFoldPitch)[i] = r2[j][q];
    }
  __syncwarp();
  if (my_len) {
    if (my_len > first_end) acc = fold_span<false>(v, first_end, my_len, acc, 0.0);
    a.partials[blockIdx.x * kLPB + lane] = acc;
  }
  PROBE_BLK_T(0, 3);
}

template <int kLPB>
__global__ void __launch_bounds__(32) k_fold_sum(FoldArgs a) {
  extern __shared__ __align__(16) double stage[];  // kLPB x kFoldPitch
  __shared__ __align__(8) uint64_t bar[kLPB][2];
  const uint32_t lane = threadIdx.x;
  if (lane < kLPB) {
    mbar_init1(&bar[lane][0]);
    mbar_init1(&bar[lane][1]);
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  PROBE_BLK(0, 0);
  pdl_wait();
  // release the sq pass now: its blocks fetch their x leaves while this grid folds
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  PROBE_BLK(0, 1);
  if (em_skipped(a.unconv)) return;
  const uint32_t M = a.M;
  const uint32_t* n = a.layout;
  const uint32_t* label_start = a.layout + M;
  const uint32_t* leaf_start = a.layout + 2 * M + 1;
  const uint32_t leaf = blockIdx.x * kLPB + lane;
  const bool valid = lane < kLPB && leaf < leaf_start[M + 1];
  if (valid) {
    const uint32_t sr = series_of(leaf_start, M + 1, leaf);
    const uint64_t b = uint64_t(leaf - leaf_start[sr]) * kFoldLeaf;
    const double* src;
    uint64_t slen;
    if (sr < M) {
      src = a.x + label_start[sr] + b;
      slen = n[sr];
    } else {  // the hood-energy row of the last executed MAP iteration (optimize.cpp:64-65)
      const int T = executed_iters(a.unconv, a.map_max, a.fixed);
      src = a.hist + uint64_t((T - 1) % a.ring) * a.Hs + b;
      slen = a.Hs;
    }
    const uint64_t rem = slen - b;
    const uint32_t len = static_cast<uint32_t>(rem < kFoldLeaf ? rem : uint64_t(kFoldLeaf));
    double* row = stage + lane * kFoldPitch;
    uint32_t n0;
    const uint32_t off = fetch_leaf(row, src, len, bar[lane], &n0);
    PROBE_BLK_T(0, 2);
    a.partials[leaf] = fold_fetched<false>(row, off, len, n0, bar[lane], 0.0);
    PROBE_BLK_T(0, 3);
  }
  if (a.roots_sum) {
    __syncwarp();  // (the stage is free: every chain is done)
    chunk_tickets(leaf_start, M + 1, leaf, valid, a.partials, a.roots_sum, a.tickets, stage);
  }
}

template <int kLPB>
__global__ void __launch_bounds__(kSqThreads) k_fold_sq(FoldArgs a) {
  extern __shared__ __align__(16) double stage[];  // kLPB x kFoldPitch | root_cap | 4 x scratch
  __shared__ __align__(8) uint64_t bar[kLPB][2];
  __shared__ uint32_t sr_s[kLPB], len_s[kLPB], off_s[kLPB], n0_s[kLPB];
  __shared__ double mu_s[kLPB];
  __shared__ uint32_t lay[4 * kMaxLabels + 4];  // the layout, read once
  __shared__ double root_s[kMaxLabels + 1];
  __shared__ double mu_all[kMaxLabels];
  __shared__ EmPrefetch pf;
  __shared__ double lt_s[2 * kLogTable];  // log_fast's table, read before the wait
  __shared__ bool last;
  double* roots = stage + kLPB * kFoldPitch;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr uint32_t kWarps = kSqThreads / 32;
  double* qw = roots + a.root_cap + warp * kTreeScratch;  // this warp's tree scratch
  const uint32_t M = a.M;
  const uint32_t* n = lay;
  const uint32_t* label_start = lay + M;
  const uint32_t* leaf_start = lay + 2 * M + 1;
  const uint32_t first = blockIdx.x * kLPB;
  if (tid < kLPB) {
    mbar_init1(&bar[tid][0]);
    mbar_init1(&bar[tid][1]);
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  // before the wait: x, the layout, the skip flag and the MAP counters are
  // the MAP launches' (complete once the sum pass released this grid); the
  // EM history is the previous EM's
  const bool skipped = em_skipped(a.unconv);
  for (uint32_t i = tid; i < 4 * M + 4; i += kSqThreads) lay[i] = a.layout[i];
  for (uint32_t i = tid; i < 2 * kLogTable; i += kSqThreads)
    lt_s[i] = i < kLogTable ? g_log_table.hi[i] : g_log_table.lo[i - kLogTable];
  if (a.merged && !skipped && tid == kSqThreads - 32) em_prefetch(a.ep, &pf);
  __syncthreads();
  PROBE_BLK(1, 0);
  if (!skipped && tid < kLPB) {
    const uint32_t leaf = first + tid;
    uint32_t len = 0;
    if (leaf < leaf_start[M]) {
      const uint32_t sr = series_of(leaf_start, M, leaf);
      const uint64_t b = uint64_t(leaf - leaf_start[sr]) * kFoldLeaf;
      const uint64_t rem = n[sr] - b;
      len = static_cast<uint32_t>(rem < kFoldLeaf ? rem : uint64_t(kFoldLeaf));
      sr_s[tid] = sr;
      off_s[tid] = fetch_leaf(stage + tid * kFoldPitch, a.x + label_start[sr] + b, len, bar[tid],
                              &n0_s[tid]);
    }
    len_s[tid] = len;
  }
  pdl_wait();  // the sum pass is complete: its partials are visible
  PROBE_BLK(1, 1);
  if (skipped) return;  // (uniform: no block takes a ticket)
  __syncthreads();
  // mu of this block's labels (consecutive series s_lo..s_hi) from the
  // sum-pass partials, one warp per label; the block holding a label's
  // first leaf publishes it
  if (len_s[0] != 0) {
    const uint32_t s_lo = sr_s[0];
    uint32_t s_hi = s_lo;
    for (int j = 1; j < kLPB; ++j)
      if (len_s[j] != 0) s_hi = sr_s[j];
    auto publish = [&](uint32_t s, double folded) {  // (one thread)
      const double mu = __ddiv_rn(folded, static_cast<double>(n[s]));
      root_s[s - s_lo] = mu;
      if (leaf_start[s] >= first && leaf_start[s] < first + kLPB) a.params[s] = mu;
    };
    bool short_series = true;
    for (uint32_t s = s_lo; s <= s_hi; ++s)
      short_series = short_series && leaf_start[s + 1] - leaf_start[s] <= kFoldLeaf;
    if (a.roots_sum) {  // the sum pass folded the chunk roots: a short tree per label
      for (uint32_t s = s_lo + warp; s <= s_hi; s += kWarps) {
        const uint32_t cnt = leaf_start[s + 1] - leaf_start[s];
        if (cnt == 0) continue;
        const double folded = warp_tree<true>(a.roots_sum + chunk_base(leaf_start, s),
                                              (cnt + kFoldLeaf - 1) / kFoldLeaf, qw);
        if (lane == 0) publish(s, folded);
      }
    } else if (short_series) {
      for (uint32_t s = s_lo + warp; s <= s_hi; s += kWarps) {
        const uint32_t cnt = leaf_start[s + 1] - leaf_start[s];
        if (cnt == 0) continue;  // (a label without leaves is held by no block)
        const double folded = warp_tree<true>(a.partials + leaf_start[s], cnt, qw);
        if (lane == 0) publish(s, folded);
      }
    } else {
      for (uint32_t s = s_lo; s <= s_hi; ++s) {
        const uint32_t cnt = leaf_start[s + 1] - leaf_start[s];
        if (cnt == 0) continue;
        const double folded = block_series_tree(a.partials + leaf_start[s], cnt, roots, qw);
        if (tid == 0) publish(s, folded);
      }
    }
    __syncthreads();
    if (tid < kLPB && len_s[tid] != 0) mu_s[tid] = root_s[sr_s[tid] - s_lo];
  }
  __syncthreads();
  PROBE_BLK(1, 2);
  // the terms (x - mu)^2 (engine.cpp:213-217) by the whole block, in place;
  // the chains then fold plain sums (one dependent DADD per element)
#pragma unroll
  for (int j = 0; j < kLPB; ++j) {
    if (len_s[j] == 0) continue;
    mbar_wait0(&bar[j][0]);
    if (len_s[j] > n0_s[j] - off_s[j]) mbar_wait0(&bar[j][1]);
    double* v = stage + j * kFoldPitch + off_s[j];
    const double mu = mu_s[j];
    for (uint32_t i = tid; i < len_s[j]; i += kSqThreads) {
      const double d = __dsub_rn(v[i], mu);
      v[i] = __dmul_rn(d, d);
    }
  }
  __syncthreads();
  if (tid < kLPB && len_s[tid] != 0) {
    const double* v = stage + tid * kFoldPitch + off_s[tid];
    a.sq_partials[first + tid] = fold_span<false>(v, 1, len_s[tid], v[0], 0.0);
    if (tid == 0) PROBE_BLK_T(1, 3);
  }
  if (a.roots_sq && warp == 0)
    chunk_tickets(leaf_start, M, first + tid, tid < kLPB && len_s[tid] != 0, a.sq_partials,
                  a.roots_sq, a.tickets + kMaxChunks, qw);
  if (a.merged && (executed_iters(a.unconv, a.map_max, a.fixed) & 1)) {
    // device-resident loop: the next EM starts from buffer 0, so an odd
    // number of MAP iterations leaves the committed labels to move back
    // (read by the next launch: the kernel boundary orders it)
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    const uint64_t words = a.ep.R / 4;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(a.ep.lab1);
    uint32_t* dst = reinterpret_cast<uint32_t*>(a.ep.lab0);
    const uint64_t g = uint64_t(blockIdx.x) * blockDim.x + tid;
    for (uint64_t w = g; w < words; w += stride) dst[w] = src[w];
    for (uint64_t v = words * 4 + g; v < a.ep.R; v += stride) a.ep.lab0[v] = a.ep.lab1[v];
  }
  // ---- last block: sigma + total-energy trees, parameters, EM record ----
  if (warp == 0) __threadfence();  // (warp 0 wrote the partials and the mu)
  __syncthreads();
  if (tid == 0) last = atomicAdd(a.done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  PROBE_TAIL(1, 0);
  const uint32_t nseries = M + 1;
  auto series_ptr = [&](uint32_t s) {
    return s < M ? a.sq_partials + leaf_start[s] : a.partials + leaf_start[M];
  };
  auto series_cnt = [&](uint32_t s) {
    return s < M ? leaf_start[s + 1] - leaf_start[s] : leaf_start[M + 1] - leaf_start[M];
  };
  // every label's mu (published by the blocks above; empty labels keep the
  // previous one), loaded beside the trees' partials
  for (uint32_t s = tid; s < M; s += kSqThreads) mu_all[s] = __ldcg(a.params + s);
  PROBE_TAIL(0, 2);
  bool all_short = true;
  for (uint32_t s = 0; s < nseries; ++s) all_short = all_short && series_cnt(s) <= kFoldLeaf;
  if (a.roots_sum && a.roots_sq) {
    // the passes folded every chunk root: one warp per series over its roots
    for (uint32_t s = warp; s < nseries; s += kWarps) {
      const uint32_t cnt = series_cnt(s);
      const double r = cnt ? warp_tree<true>((s < M ? a.roots_sq : a.roots_sum) +
                                                 chunk_base(leaf_start, s),
                                             (cnt + kFoldLeaf - 1) / kFoldLeaf, qw)
                           : 0.0;
      if (lane == 0) root_s[s] = r;
    }
  } else if (all_short) {  // one warp per series, all at once
    for (uint32_t s = warp; s < nseries; s += kWarps) {
      const uint32_t cnt = series_cnt(s);
      const double r = cnt ? warp_tree<true>(series_ptr(s), cnt, qw) : 0.0;
      if (lane == 0) root_s[s] = r;
    }
  } else {
    // every series' aligned 1024-partial chunks by the warps at once (a
    // chunk's root is the level-10 node of its series' tree), then one warp
    // per series over its chunk roots
    uint32_t total_chunks = 0;
    for (uint32_t s = 0; s < nseries; ++s) total_chunks += (series_cnt(s) + kFoldLeaf - 1) / kFoldLeaf;
    for (uint32_t c = warp; c < total_chunks; c += kWarps) {
      uint32_t s = 0, base = 0;
      while (c >= base + (series_cnt(s) + kFoldLeaf - 1) / kFoldLeaf) {
        base += (series_cnt(s) + kFoldLeaf - 1) / kFoldLeaf;
        ++s;
      }
      const uint32_t q = c - base, cnt = series_cnt(s);
      const double r = warp_tree<true>(series_ptr(s) + uint64_t(q) * kFoldLeaf,
                                       min(kFoldLeaf, cnt - q * kFoldLeaf), qw);
      if (lane == 0) roots[c] = r;
    }
    __syncthreads();
    PROBE_TAIL(0, 0);
    uint32_t base = 0;
    for (uint32_t s = 0; s < nseries; ++s) {
      const uint32_t nch = (series_cnt(s) + kFoldLeaf - 1) / kFoldLeaf;
      if (warp == s % kWarps) {
        const double r = nch ? warp_tree<false>(roots + base, nch, qw) : 0.0;
        if (lane == 0) root_s[s] = r;
      }
      base += nch;
    }
  }
  __syncthreads();
  for (uint32_t s = tid; s < nseries; s += kSqThreads) {
    const double folded = root_s[s];
    if (s < M) {
      double sg = a.params[M + s];
      if (n[s] != 0) {  // empty labels keep their previous parameters (engine.cpp:209-220)
        const double sd = __dsqrt_rn(__ddiv_rn(folded, static_cast<double>(n[s])));
        sg = sd < kSigmaFloor ? kSigmaFloor : sd;
        a.params[M + s] = sg;
      }
      a.em_out[2 + s] = mu_all[s];
      a.em_out[2 + M + s] = sg;
    } else {
      // total energy: dpp::reduce(..., 0.0) -> identity only for empty input
      a.em_out[0] = series_cnt(M) == 0 ? 0.0 : folded;
      a.em_out[1] = static_cast<double>(a.unconv ? executed_iters(a.unconv, a.map_max, a.fixed) : 0);
    }
  }
  __syncthreads();
  PROBE_TAIL(1, 1);
  if (a.merged && tid < 32) em_record(a.ep, true, &pf, lt_s, lt_s + kLogTable);
  if (tid == 0) *a.done = 0;  // re-arm the ticket for the next launch
  PROBE_TAIL(1, 2);
}

// ---------------------------------------------------------------------------
// k_fold_sq_cluster: the sq pass and the EM tail as ONE thread-block cluster
// of kClCtas CTAs, for graphs with few label leaves (2560^2: ~100).  Same
// arithmetic and fetch schedule as k_fold_sq, but the cross-block combine
// runs through distributed shared memory instead of a global ticket: each
// CTA pushes its sq partials, and the mu of every label whose first leaf it
// holds, into CTA 0's shared memory (st.shared::cluster); one cluster
// barrier; CTA 0 then runs the sigma trees and the EM record straight from
// shared memory.  CTA 0's last warp folds the total-energy tree (series M of
// the sum pass) while the chains run, so it is off the critical path.
// ---------------------------------------------------------------------------
#ifndef DPMRF_CL_THREADS
#define DPMRF_CL_THREADS 128
#endif
#ifndef DPMRF_CL_BLOCKSQ
#define DPMRF_CL_BLOCKSQ 0
#endif
constexpr int kClCtas = 8;
constexpr int kClThreads = DPMRF_CL_THREADS;
constexpr bool kClBlockSq = DPMRF_CL_BLOCKSQ != 0;
#ifndef DPMRF_CL_SQPIPE
#define DPMRF_CL_SQPIPE 1
#endif
constexpr bool kClSqPipe = DPMRF_CL_SQPIPE != 0;  // squares one group ahead of the adds
constexpr uint32_t kClMaxPer = 24;  // staged label leaves per CTA

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// store v into CTA `cta`'s copy of the shared variable *p (same layout in every CTA)
__device__ __forceinline__ void st_cluster(double* p, uint32_t cta, double v) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(p)), "r"(cta));
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}

__global__ void __launch_bounds__(kClThreads) k_fold_sq_cluster(FoldArgs a, uint32_t per,
                                                                uint32_t sq_cap) {
  extern __shared__ __align__(16) double stage[];  // per x kFoldPitch | sqp[sq_cap] | scratch
  __shared__ __align__(8) uint64_t bar[kClMaxPer][2];
  __shared__ uint32_t sr_s[kClMaxPer], len_s[kClMaxPer], off_s[kClMaxPer], n0_s[kClMaxPer];
  __shared__ double mu_s[kClMaxPer];
  __shared__ uint32_t lay[4 * kMaxLabels + 4];
  __shared__ double root_s[kMaxLabels + 1];
  __shared__ double vals[2 + 2 * kMaxLabels];  // CTA 0: [total, T, mu(M), sigma(M)]
  __shared__ double mu_pub[kMaxLabels];         // CTA 0: mu pushed by the label's first CTA
  __shared__ EmPrefetch pf;
  __shared__ double lt_s[2 * kLogTable];
  double* sqp = stage + per * kFoldPitch;  // CTA 0: sq partials of every label leaf
  double* qw = sqp + sq_cap;               // CTA 0's last warp: tree scratch
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr uint32_t kWarps = kClThreads / 32;
  const uint32_t rank = cluster_ctarank();
  const uint32_t M = a.M;
  const uint32_t* n = lay;
  const uint32_t* label_start = lay + M;
  const uint32_t* leaf_start = lay + 2 * M + 1;
  const uint32_t first = rank * per;
  PROBE_BLK(1, 0);
  if (tid < per) {
    mbar_init1(&bar[tid][0]);
    mbar_init1(&bar[tid][1]);
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  // (every CTA of the cluster has started before anyone writes remote
  // shared memory: arrive now, wait after the grid dependency)
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  // before the wait (as k_fold_sq): x, the layout, the skip flag and the MAP
  // counters are the MAP launches'; params and the EM history the previous EM's
  const bool skipped = em_skipped(a.unconv);  // (the same value in every CTA)
  for (uint32_t i = tid; i < 4 * M + 4; i += kClThreads) lay[i] = a.layout[i];
  if (rank == 0) {
    for (uint32_t i = tid; i < 2 * kLogTable; i += kClThreads)
      lt_s[i] = i < kLogTable ? g_log_table.hi[i] : g_log_table.lo[i - kLogTable];
    // a label without vertices keeps its parameters (engine.cpp:209-220)
    for (uint32_t l = tid; l < M; l += kClThreads) {
      vals[2 + l] = a.params[l];
      vals[2 + M + l] = a.params[M + l];
    }
    if (a.merged && !skipped && tid == 32) em_prefetch(a.ep, &pf);
  }
  __syncthreads();
  if (!skipped && tid < per) {
    const uint32_t leaf = first + tid;
    uint32_t len = 0;
    if (leaf < leaf_start[M]) {
      const uint32_t sr = series_of(leaf_start, M, leaf);
      const uint64_t b = uint64_t(leaf - leaf_start[sr]) * kFoldLeaf;
      const uint64_t rem = n[sr] - b;
      len = static_cast<uint32_t>(rem < kFoldLeaf ? rem : uint64_t(kFoldLeaf));
      sr_s[tid] = sr;
      off_s[tid] = fetch_leaf(stage + tid * kFoldPitch, a.x + label_start[sr] + b, len, bar[tid],
                              &n0_s[tid]);
    }
    len_s[tid] = len;
  }
  pdl_wait();  // the sum pass is complete: its partials are visible
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  PROBE_BLK(1, 1);
  if (skipped) return;  // (uniform over the cluster)
  __syncthreads();
  const int T = executed_iters(a.unconv, a.map_max, a.fixed);
  // mu of this CTA's labels from the sum-pass partials, one warp per label
  if (per && len_s[0] != 0) {
    const uint32_t s_lo = sr_s[0];
    uint32_t s_hi = s_lo;
    for (uint32_t j = 1; j < per; ++j)
      if (len_s[j] != 0) s_hi = sr_s[j];
    for (uint32_t s = s_lo + warp; s <= s_hi; s += kWarps) {
      const uint32_t cnt = leaf_start[s + 1] - leaf_start[s];
      if (cnt == 0) continue;  // (a label without leaves is held by no CTA)
      const double folded = warp_tree512<true>(a.partials + leaf_start[s], cnt);
      if (lane == 0) {
        const double mu = __ddiv_rn(folded, static_cast<double>(n[s]));
        root_s[s - s_lo] = mu;
        if (leaf_start[s] >= first && leaf_start[s] < first + per) st_cluster(&mu_pub[s], 0, mu);
      }
    }
    __syncthreads();
    if (tid < per && len_s[tid] != 0) mu_s[tid] = root_s[sr_s[tid] - s_lo];
  }
  __syncthreads();
  if (kClBlockSq) {
    // the terms (x - mu)^2 (engine.cpp:213-217) by the whole CTA, in place
    for (uint32_t j = 0; j < per; ++j) {
      if (len_s[j] == 0) continue;
      mbar_wait0(&bar[j][0]);
      if (len_s[j] > n0_s[j] - off_s[j]) mbar_wait0(&bar[j][1]);
      double* v = stage + j * kFoldPitch + off_s[j];
      const double mu = mu_s[j];
#pragma unroll 4
      for (uint32_t i = tid; i < len_s[j]; i += kClThreads) {
        const double d = __dsub_rn(v[i], mu);
        v[i] = __dmul_rn(d, d);
      }
    }
    __syncthreads();
  }
  PROBE_BLK(1, 2);
  if (warp == 0) {
    // the dependent chains (fold_leaf) over (x - mu)^2 (engine.cpp:213-217),
    // one lane per staged leaf (kClBlockSq: squared above; else the squares
    // are computed in the chain, off its dependent path)
    if (tid < per && len_s[tid] != 0) {
      const double* v = stage + tid * kFoldPitch + off_s[tid];
      double r;
      if (kClBlockSq) {
        r = fold_span<false>(v, 1, len_s[tid], v[0], 0.0);
      } else {
        mbar_wait0(&bar[tid][0]);
        if (len_s[tid] > n0_s[tid] - off_s[tid]) mbar_wait0(&bar[tid][1]);
        const double mu = mu_s[tid];
        const double d0 = __dsub_rn(v[0], mu);
        r = kClSqPipe ? fold_span_sq(v, 1, len_s[tid], __dmul_rn(d0, d0), mu)
                      : fold_span<true>(v, 1, len_s[tid], __dmul_rn(d0, d0), mu);
      }
      st_cluster(&sqp[first + tid], 0, r);
    }
    PROBE_BLK_T(1, 3);
  } else {
    if (rank == 0 && warp == kWarps - 1) {
      // total energy: dpp::reduce(..., 0.0) over the last executed MAP row
      // (optimize.cpp:64-65) -- identity only for empty input
      const uint32_t cnt = leaf_start[M + 1] - leaf_start[M];
      const double r = cnt ? warp_tree<true>(a.partials + leaf_start[M], cnt, qw) : 0.0;
      if (lane == 0) {
        vals[0] = r;
        vals[1] = static_cast<double>(T);
      }
    }
    if (a.merged && (T & 1)) {
      // device-resident loop: the next EM starts from buffer 0, so an odd
      // number of MAP iterations moves the committed labels back
      const uint64_t stride = uint64_t(kClCtas) * (kClThreads - 32);
      const uint64_t g = uint64_t(rank) * (kClThreads - 32) + (tid - 32);
      const uint64_t words = a.ep.R / 4;
      const uint32_t* src = reinterpret_cast<const uint32_t*>(a.ep.lab1);
      uint32_t* dst = reinterpret_cast<uint32_t*>(a.ep.lab0);
      for (uint64_t w = g; w < words; w += stride) dst[w] = src[w];
      for (uint64_t v = words * 4 + g; v < a.ep.R; v += stride) a.ep.lab0[v] = a.ep.lab1[v];
    }
  }
  cluster_sync_all();  // every sq partial and mu is in CTA 0's shared memory
  if (rank != 0) return;
  PROBE_TAIL(1, 0);
  for (uint32_t s = warp; s < M; s += kWarps) {
    const uint32_t cnt = leaf_start[s + 1] - leaf_start[s];
    if (cnt == 0) continue;  // empty labels keep their previous parameters
    const double folded = warp_tree512<false>(sqp + leaf_start[s], cnt);
    if (lane == 0) {
      vals[2 + s] = mu_pub[s];
      const double sd = __dsqrt_rn(__ddiv_rn(folded, static_cast<double>(n[s])));
      vals[2 + M + s] = sd < kSigmaFloor ? kSigmaFloor : sd;
    }
  }
  __syncthreads();
  for (uint32_t i = tid; i < 2 + 2 * M; i += kClThreads) {
    a.em_out[i] = vals[i];
    if (i >= 2) a.params[i - 2] = vals[i];
  }
  PROBE_TAIL(1, 1);
  if (a.merged && tid < 32) em_record(a.ep, true, &pf, lt_s, lt_s + kLogTable, vals);
  PROBE_TAIL(1, 2);
}

// ---------------------------------------------------------------------------
// k_mstep_stream: both M-step passes of many-leaf graphs (16384^2: ~16 000
// sum-pass leaves) as ONE persistent kernel.  Lane j < C of a one-warp block
// is a chain that walks the leaves gid, gid + G*C, ... (gid = block*C + j);
// each leaf streams through the lane's ring of NS shared-memory slots in
// kQuarter-double parts (one cp.async.bulk + one mbarrier per slot), the next
// parts in flight while the chain folds the current one, so every SM
// keeps ~30 chains busy instead of running whole-leaf waves.  After each
// round the warp counts its leaves into their chunks (chunk_tickets): the
// warp completing a chunk folds its root, the warp completing a series folds
// the series root and publishes mu (sum pass), sigma (sq pass) or the total
// energy.  Between the passes every block waits at a grid barrier (the grid
// is sized by occupancy, so all blocks are resident), then folds (x - mu)^2
// (engine.cpp:213-217) -- x read again, largely from L2.  The last block
// (ticket) completes the EM output and record.
// ---------------------------------------------------------------------------
#ifndef DPMRF_STREAM_C
#define DPMRF_STREAM_C 16
#endif
#ifndef DPMRF_STREAM_NS
#define DPMRF_STREAM_NS 3
#endif
#ifndef DPMRF_STREAM_W
#define DPMRF_STREAM_W 1
#endif
constexpr int kStreamChains = DPMRF_STREAM_C;  // chains (lanes) per warp
constexpr int kStreamWarps = DPMRF_STREAM_W;   // warps per block (independent rings)

constexpr int kStreamSlots = DPMRF_STREAM_NS;  // ring slots per chain
#ifndef DPMRF_STREAM_Q
#define DPMRF_STREAM_Q 128  // (128: 4 one-warp blocks per SM, one per scheduler; 256
                            //  fits only 2 -- D: M-step 136.6 -> 122 us/EM, +1%)
#endif
constexpr uint32_t kQuarter = DPMRF_STREAM_Q;  // doubles per streamed part of a leaf
constexpr uint32_t kParts = kFoldLeaf / kQuarter;  // parts per leaf (power of two)
static_assert(kParts * kQuarter == kFoldLeaf && (kParts & (kParts - 1)) == 0 && kQuarter % 16 == 0,
              "a leaf streams in equal power-of-two parts");
constexpr uint32_t kSlotPitch = kQuarter + 2;  // doubles per slot (16-byte aligned superset)
#ifndef DPMRF_STREAM_PFENCE
#define DPMRF_STREAM_PFENCE 1
#endif
constexpr bool kStreamProxyFence = DPMRF_STREAM_PFENCE != 0;

struct StreamCounters {  // zeroed once; re-armed by the kernel itself
  uint32_t gen;     // launches completed (the ready flags of launch g read g + 1)
  uint32_t done;    // blocks finished
  uint32_t ready[kMaxLabels];             // per label: mu published (== gen + 1)
  uint32_t series[2 * (kMaxLabels + 1)];  // chunks completed per series (sum | sq)
};

__device__ __forceinline__ void mbar_wait_par(uint64_t* bar, uint32_t par) {
  uint32_t ok = 0, spins = 0;
  while (!ok) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(par)
        : "memory");
    if (!ok && ++spins > (1u << 26)) __trap();  // a lost copy: fail loudly, never hang
  }
}

struct StreamView {
  const uint32_t* n;
  const uint32_t* label_start;
  const uint32_t* leaf_start;
  const double* x;
  const double* hood_row;
  uint64_t Hs;
  uint32_t M;
  // leaf -> [src, src + len) of its series, and the series
  __device__ __forceinline__ uint32_t span(bool sq, uint32_t leaf, const double*& src,
                                           uint32_t& len) const {
    const uint32_t sr = series_of(leaf_start, sq ? M : M + 1, leaf);
    const uint64_t b = uint64_t(leaf - leaf_start[sr]) * kFoldLeaf;
    const uint64_t slen = sr < M ? n[sr] : Hs;
    src = (sr < M ? x + label_start[sr] : hood_row) + b;
    const uint64_t rem = slen - b;
    len = static_cast<uint32_t>(rem < kFoldLeaf ? rem : uint64_t(kFoldLeaf));
    return sr;
  }
};

// One task stream per chain: tasks 0..nsum-1 are the sum-pass leaves (label
// series, then the hood-energy series), tasks nsum.. the sq-pass leaves;
// chain c takes tasks c, c + S, c + 2S, ... (S chains in the grid), so every
// chain folds the same number of leaves (+-1) and no grid barrier separates
// the passes: an sq task first waits for its label's mu flag (published by
// the warp completing that label's sum series -- long done by then, the
// label leaves come first).
template <int C, int W, int NS>
__device__ void stream_tasks(const FoldArgs& a, const StreamView& v, double* ring,
                             uint64_t* bars, StreamCounters* cnt, uint32_t gen) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t M = a.M;
  const uint32_t stride = gridDim.x * W * C;
  // sq tasks start at P: after every sum task, and in a later round than
  // every label leaf, so no round of any warp both folds a label leaf and
  // waits for a mu (a warp never waits on its own round: deadlock-free)
  const uint32_t nsum = v.leaf_start[M + 1], nlab = v.leaf_start[M];
  const uint32_t P = max(nsum, (nlab + stride - 1) / stride * stride);
  const uint32_t ntask = P + nlab;
  const uint32_t g0 = (blockIdx.x * W + warp) * C;
  const uint32_t gid = g0 + lane;
  const uint32_t rounds = ntask > g0 ? (ntask - g0 + stride - 1) / stride : 0u;
  uint32_t ph = 0;  // this chain's slot parities
  // task -> fetched span
  auto task_span = [&](uint32_t t, const double*& src, uint32_t& len) -> uint32_t {
    return t < nsum ? v.span(false, t, src, len) : v.span(true, t - P, src, len);
  };
  // the span of the task being fetched, cached across its quarters
  uint32_t ct = 0xFFFFFFFFu, clen = 0;
  const double* csrc = nullptr;
  auto issue = [&](uint32_t pos) {
    if (lane >= uint32_t(C)) return;
    const uint32_t k = pos / kParts, qq = pos % kParts;
    if (k >= rounds) return;
    const uint32_t t = gid + k * stride;
    if (t >= ntask || (t >= nsum && t < P)) return;
    if (t != ct) {
      task_span(t, csrc, clen);
      ct = t;
    }
    const double* src = csrc;
    const uint32_t len = clen;
    if (qq * kQuarter >= len) return;
    const double* s0 = src + qq * kQuarter;
    const uint32_t n = min(kQuarter, len - qq * kQuarter);
    const uint32_t off = (reinterpret_cast<uintptr_t>(s0) & 15u) ? 1u : 0u;
    const uint32_t nd = (off + n + 1u) & ~1u;
    uint64_t* b = bars + (pos % NS);
    mbar_expect(b, nd * 8u);
    bulk_g2s(ring + (pos % NS) * kSlotPitch, s0 - off, nd * 8u, b);
  };
  for (uint32_t p = 0; p < uint32_t(NS); ++p) issue(p);
  for (uint32_t k = 0; k < rounds; ++k) {
    const uint32_t t = gid + k * stride;
    const bool has = lane < uint32_t(C) && t < ntask && (t < nsum || t >= P);
    const bool sq = t >= P;
    double acc = 0.0, mu = 0.0;
    const double* src = nullptr;
    uint32_t len = 0;
    if (has) {
      const uint32_t sr = task_span(t, src, len);
      if (sq) {  // this label's mu (engine.cpp:207-208) must be published
        uint32_t seen = 0, spins = 0;
        for (;;) {
          asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(seen) : "l"(&cnt->ready[sr]) : "memory");
          if (seen == gen + 1) break;
          __nanosleep(128);
          if (++spins > (1u << 26)) __trap();
        }
        mu = __ldcg(a.params + sr);
      }
    }
#pragma unroll 1
    for (uint32_t qq = 0; qq < kParts; ++qq) {
      const uint32_t pos = kParts * k + qq;
      if (has && qq * kQuarter < len) {
        const uint32_t slot = pos % NS;
        mbar_wait_par(bars + slot, (ph >> slot) & 1u);
        ph ^= 1u << slot;
        const double* s0 = src + qq * kQuarter;
        const uint32_t n = min(kQuarter, len - qq * kQuarter);
        const double* w =
            ring + slot * kSlotPitch + ((reinterpret_cast<uintptr_t>(s0) & 15u) ? 1 : 0);
        if (sq) {
          if (qq == 0) {
            const double d = __dsub_rn(w[0], mu);
            acc = fold_span_sq(w, 1, n, __dmul_rn(d, d), mu);
          } else {
            acc = fold_span_sq(w, 0, n, acc, mu);
          }
        } else {
          acc = fold_span<false>(w, qq == 0 ? 1 : 0, n, qq == 0 ? w[0] : acc, 0.0);
        }
      }
      // the slot is free again: refill it with the quarter NS positions ahead
      if (kStreamProxyFence) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(pos + NS);
    }
    if (has) {
      if (sq) a.sq_partials[t - P] = acc;
      else a.partials[t] = acc;
    }
    __syncwarp();
    // chunk / series tickets of this round's sum leaves, then its sq leaves
    if (__any_sync(0xffffffffu, has && !sq))
      chunk_tickets(v.leaf_start, M + 1, t, has && !sq, a.partials, a.roots_sum, a.tickets,
                    nullptr, cnt->series, [&](uint32_t s, double root) {
                      if (s < M) {
                        a.params[s] = __ddiv_rn(root, static_cast<double>(v.n[s]));
                        __threadfence();
                        asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(&cnt->ready[s]),
                                     "r"(gen + 1)
                                     : "memory");
                      } else {
                        a.em_out[0] = root;  // total energy (optimize.cpp:64-65)
                      }
                    });
    if (__any_sync(0xffffffffu, has && sq))
      chunk_tickets(v.leaf_start, M, t - P, has && sq, a.sq_partials, a.roots_sq,
                    a.tickets + kMaxChunks, nullptr, cnt->series + (kMaxLabels + 1),
                    [&](uint32_t s, double root) {
                      const double sd = __dsqrt_rn(__ddiv_rn(root, static_cast<double>(v.n[s])));
                      a.params[M + s] = sd < kSigmaFloor ? kSigmaFloor : sd;
                    });
  }
}

template <int C, int W, int NS>
__global__ void __launch_bounds__(32 * W) k_mstep_stream(FoldArgs a, StreamCounters* cnt) {
  extern __shared__ __align__(16) double sm[];  // W x C x NS x kSlotPitch
  __shared__ __align__(8) uint64_t bar[W * C][NS];
  __shared__ uint32_t lay[4 * kMaxLabels + 4];
  __shared__ uint32_t last;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (lane < uint32_t(C))
    for (int k = 0; k < NS; ++k) mbar_init1(&bar[warp * C + lane][k]);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  PROBE_BLK(0, 0);
  pdl_wait();
  PROBE_BLK(0, 1);
  if (em_skipped(a.unconv)) return;
  const uint32_t M = a.M;
  for (uint32_t i = tid; i < 4 * M + 4; i += 32 * W) lay[i] = a.layout[i];
  const uint32_t gen = cnt->gen;  // (advanced by the previous launch's last block)
  __syncthreads();
  const int T = a.unconv ? executed_iters(a.unconv, a.map_max, a.fixed) : 0;
  StreamView v{lay, lay + M, lay + 2 * M + 1, a.x,
               a.hist && T > 0 ? a.hist + uint64_t((T - 1) % a.ring) * a.Hs : nullptr, a.Hs, M};
  const uint32_t chain = warp * C + (lane < uint32_t(C) ? lane : 0u);
  stream_tasks<C, W, NS>(a, v, sm + chain * NS * kSlotPitch, &bar[chain][0], cnt, gen);
  PROBE_BLK(0, 4);
  if (a.merged && (T & 1)) {
    // device-resident loop: the next EM starts from buffer 0, so an odd
    // number of MAP iterations moves the committed labels back
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    const uint64_t words = a.ep.R / 4;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(a.ep.lab1);
    uint32_t* dst = reinterpret_cast<uint32_t*>(a.ep.lab0);
    const uint64_t g = uint64_t(blockIdx.x) * blockDim.x + tid;
    for (uint64_t w = g; w < words; w += stride) dst[w] = src[w];
    for (uint64_t x = words * 4 + g; x < a.ep.R; x += stride) a.ep.lab0[x] = a.ep.lab1[x];
  }
  // ---- last block: the EM output [total, T, mu, sigma] and record ----
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    last = atomicAdd(&cnt->done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || warp != 0) return;
  __threadfence();
  PROBE_TAIL(0, 0);
  if (lane == 0) {
    // dpp::reduce(..., 0.0): identity only for empty input
    if (v.leaf_start[M + 1] == v.leaf_start[M]) a.em_out[0] = 0.0;
    a.em_out[1] = static_cast<double>(T);
    cnt->done = 0;
    cnt->gen = gen + 1;  // (this launch's ready flags read gen + 1)
  }
  // (labels without vertices keep their previous parameters, engine.cpp:209-220)
  for (uint32_t s = lane; s < M; s += 32) {
    a.em_out[2 + s] = __ldcg(a.params + s);
    a.em_out[2 + M + s] = __ldcg(a.params + M + s);
  }
  __syncwarp();
  if (a.merged) em_record(a.ep, true);
  PROBE_TAIL(0, 1);
}

// ---------------------------------------------------------------------------
// Device-resident EM loop (no host round trip between EM iterations).
// k_em_prologue arms the MAP counters and folds the previous epilogue's stop
// decision into the state (so every kernel of this EM sees one value);
// k_em_epilogue moves the committed labels back to buffer 0, records the EM
// log, applies the EM-level window (optimize.cpp:66-71) and writes the label
// terms of the next EM with the device log (make_label_terms, model.hpp:48-60).
// ---------------------------------------------------------------------------
__global__ void k_em_prologue(uint32_t* unconv, int map_max) {
  pdl_wait();
  if (threadIdx.x == 0 && unconv[kEmPending]) unconv[kEmDone] = 1;
  for (int t = threadIdx.x; t < map_max; t += blockDim.x) unconv[t] = 0;
}

__global__ void k_em_epilogue(EmEpilogueArgs a) {
  pdl_wait();
  if (a.unconv[kEmDone]) return;
  const int T = executed_iters(a.unconv, a.map_max, a.fixed);
  if (T & 1) {  // the last MAP iteration left the committed labels in buffer 1
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < a.R; v += stride)
      a.lab0[v] = a.lab1[v];
  }
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;
  em_record(a, false);
}

// Partitioned optimize: this rank's leaves of the hood-energy series (its
// series range starts on a leaf boundary) folded from the last executed MAP
// row -- fold_leaf, kernels.hpp:37-42 -- into out[leaf - first_leaf], so the
// per-EM exchange carries H/1024 partials instead of the H-element row.
__global__ void __launch_bounds__(256)
    k_row_leaves(const double* __restrict__ hist, int ring, uint64_t Hs,
                 const uint32_t* __restrict__ unconv, int map_max, int fixed, uint64_t hb,
                 uint64_t he, double* __restrict__ out) {
  extern __shared__ double stage[];  // kLeavesPerBlock x kLeafStride
  __shared__ uint32_t len_s[kLeavesPerBlock];
  pdl_wait();
  if (em_skipped(unconv)) return;
  const int T = executed_iters(unconv, map_max, fixed);
  const double* row = hist + uint64_t((T - 1) % ring) * Hs;
  const uint64_t first = hb / kFoldLeaf + uint64_t(blockIdx.x) * kLeavesPerBlock;
  const uint64_t nleaf = (he + kFoldLeaf - 1) / kFoldLeaf;
  if (threadIdx.x < kLeavesPerBlock) {
    const uint64_t leaf = first + threadIdx.x;
    uint32_t len = 0;
    if (leaf < nleaf) {
      const uint64_t rem = he - leaf * kFoldLeaf;
      len = static_cast<uint32_t>(rem < kFoldLeaf ? rem : uint64_t(kFoldLeaf));
    }
    len_s[threadIdx.x] = len;
  }
  __syncthreads();
  for (uint32_t f = threadIdx.x; f < kLeavesPerBlock * kFoldLeaf; f += blockDim.x) {
    const uint32_t j = f / kFoldLeaf, i = f % kFoldLeaf;
    stage[j * kLeafStride + i] = i < len_s[j] ? __ldcg(row + (first + j) * kFoldLeaf + i) : 0.0;
  }
  __syncthreads();
  if (threadIdx.x < kLeavesPerBlock && len_s[threadIdx.x]) {
    const double* v = stage + threadIdx.x * kLeafStride;
    double acc = v[0];
    for (uint32_t i = 1; i < len_s[threadIdx.x]; ++i) acc = __dadd_rn(acc, v[i]);
    out[first + threadIdx.x - hb / kFoldLeaf] = acc;
  }
}

__global__ void k_log_cr(const double* x, double* out, uint64_t n) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = log_fast(x[i], g_log_table.hi, g_log_table.lo);
}


// update_parameters on caller labels: u32 -> u8 with the range check
__global__ void k_u32_to_u8_checked(const uint32_t* __restrict__ in, uint8_t* __restrict__ out,
                                    uint64_t n, uint32_t M, uint32_t* err) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t l = in[i];
  if (l >= M) {
    atomicOr(err, 1u);
    out[i] = 0;
  } else {
    out[i] = static_cast<uint8_t>(l);
  }
}

}  // namespace

namespace {

void mstep_core(const double* mean, uint32_t R, uint32_t M, const uint8_t* lab_even,
                const uint8_t* lab_odd, const uint32_t* unconv, int map_max, int fixed,
                const double* hist, uint64_t Hs, int ring, double* params, double* em_out,
                MStepBuffers& mb, cudaStream_t s, uint64_t* launches, bool counts_ready,
                bool scattered, const EmEpilogueArgs* ep, const double* hood_parts) {
  mstep_reserve(mb, R, M, Hs);
  const uint32_t tiles = static_cast<uint32_t>((uint64_t(R) + kTileVerts - 1) / kTileVerts);
  uint32_t* counts = mb.counts.get();
  uint32_t* tile_base = mb.tile_base.get();
  uint32_t* layout = mb.layout.get();
  double* x = mb.x.get();
  const uint64_t max_leaves = (uint64_t(R) + kFoldLeaf - 1) / kFoldLeaf + M +
                              (Hs + kFoldLeaf - 1) / kFoldLeaf + 1;
  double* partials = mb.partials.get();
  const size_t smem = (kTileThreads / 32) * M * sizeof(uint32_t);
  uint64_t n = 0;
  if (scattered) {
    // the grouping already ran beside the last hood pass (launch_map_fused)
  } else if (tiles && !counts_ready) {
    k_label_counts<<<tiles, kTileThreads, smem, s>>>(lab_even, lab_odd, unconv, map_max, fixed,
                                                     R, M, counts);
    CK_LAUNCH();
    ++n;
  }
  if (scattered) {
  } else if (tiles && uint64_t(tiles) * M <= kSelfScanMax) {
    const size_t smem_s = scatter_small_smem(M);
    launch_pdl(k_label_scatter_small, dim3(tiles), dim3(kTileThreads), smem_s, s, lab_even,
               lab_odd, unconv, counts_ready ? unconv : (const uint32_t*)nullptr, map_max, fixed,
               R, M, Hs, mean, (const uint32_t*)counts, tiles, layout, x);
    ++n;
  } else {
    const uint32_t nchunks = (tiles + kTileChunk - 1) / kTileChunk;
    uint32_t* chunk_sum = mb.chunk_sum.ensure(uint64_t(nchunks ? nchunks : 1) * M);
    const uint32_t* sel = counts_ready ? unconv : nullptr;
    if (nchunks) {
      launch_pdl(k_tile_chunks, dim3(nchunks), dim3(1024), 0, s, (const uint32_t*)counts, sel,
                 map_max, fixed, tiles, M, chunk_sum);
      ++n;
    }
    launch_pdl(k_tile_offsets, dim3(nchunks ? nchunks : 1), dim3(1024), 0, s,
               (const uint32_t*)counts, sel, map_max, fixed, tile_base, tiles, M, Hs, layout,
               (const uint32_t*)chunk_sum, nchunks);
    ++n;
  }
  if (!scattered && tiles && uint64_t(tiles) * M > kSelfScanMax) {
    constexpr uint32_t kTilesPerBlock = kTileThreads / 32;
    launch_pdl(k_label_scatter_warp, dim3((tiles + kTilesPerBlock - 1) / kTilesPerBlock),
               dim3(kTileThreads), smem, s, lab_even, lab_odd, unconv, map_max, fixed, R, M, mean,
               (const uint32_t*)tile_base, (const uint32_t*)layout, x);
    ++n;
  }
  // few leaves (2560^2: ~300): 2 per block, one block per SM -- latency;
  // many (16384^2: ~16 000): 8 per sum block / 4 per sq block (three blocks
  // per SM by shared memory) -- enough chains in flight for HBM
  const bool few = max_leaves <= uint64_t(4) * kNumSMs;
  const uint64_t label_leaves = (uint64_t(R) + kFoldLeaf - 1) / kFoldLeaf + M;
  const EmEpilogueArgs epv = ep ? *ep : EmEpilogueArgs{};
  {
    // chunk roots: every series' 1024-partial chunks at once in the tail
    const uint64_t chunks = (label_leaves + kFoldLeaf - 1) / kFoldLeaf + M +
                            ((Hs + kFoldLeaf - 1) / kFoldLeaf + kFoldLeaf - 1) / kFoldLeaf + 1;
    if (chunks > 8192) fail(DPMRF_INVALID_ARGUMENT, "M-step: series too long for the fold trees");
    const uint32_t root_cap = static_cast<uint32_t>((chunks + 31) / 32 * 32);
    FoldArgs fa{x,       layout,        M,     hist,      Hs,
                ring,    unconv,        map_max, fixed,   params,
                partials, mb.sq_partials.get(), em_out, mb.done.get() + 1, epv,
                ep ? 1 : 0, root_cap, nullptr, nullptr, nullptr};
    const uint64_t hood_leaves = (Hs + kFoldLeaf - 1) / kFoldLeaf;
    if (few && mb.cluster_sq && label_leaves <= uint64_t(kClCtas) * kClMaxPer &&
        hood_leaves <= kFoldLeaf) {
      // the sq pass + EM tail as one cluster (distributed shared memory)
      constexpr int kS = 2;
      const size_t ss = size_t(kS) * kFoldPitch * sizeof(double);
      const uint32_t per = static_cast<uint32_t>((label_leaves + kClCtas - 1) / kClCtas);
      const uint32_t sq_cap = static_cast<uint32_t>((label_leaves + 1) / 2 * 2);
      const size_t sc = (size_t(per) * kFoldPitch + sq_cap + kTreeScratch) * sizeof(double);
      ensure_dynamic_smem(k_fold_sum_ldg<kS>, ss);
      ensure_dynamic_smem(k_fold_sq_cluster, sc);
      launch_pdl(k_fold_sum_ldg<kS>, dim3(grid_for(max_leaves, kS)), dim3(32), ss, s, fa);
      launch_pdl_cluster(k_fold_sq_cluster, dim3(kClCtas), dim3(kClThreads), sc, kClCtas, s, fa,
                         per, sq_cap);
    } else if (few) {
      constexpr int kS = 2, kQ = 2;
      const size_t ss = size_t(kS) * kFoldPitch * sizeof(double);
      const size_t sq = (size_t(kQ) * kFoldPitch + root_cap + (kSqThreads / 32) * kTreeScratch) *
                        sizeof(double);
      ensure_dynamic_smem(k_fold_sum_ldg<kS>, ss);
      ensure_dynamic_smem(k_fold_sq<kQ>, sq);
      launch_pdl(k_fold_sum_ldg<kS>, dim3(grid_for(max_leaves, kS)), dim3(32), ss, s, fa);
      launch_pdl(k_fold_sq<kQ>, dim3(grid_for(label_leaves, kQ)), dim3(kSqThreads), sq, s, fa);
    } else if (mb.stream && label_leaves <= uint64_t(kFoldLeaf) * kFoldLeaf &&
               hood_leaves <= uint64_t(kFoldLeaf) * kFoldLeaf && chunks <= kMaxChunks) {
      // both passes + the EM tail in one persistent streaming kernel
      fa.roots_sum = mb.roots.get();
      fa.roots_sq = mb.roots.get() + kMaxChunks;
      fa.tickets = mb.tickets.get();
      constexpr int kC = kStreamChains, kW = kStreamWarps, kNS = kStreamSlots;
      const size_t sm = size_t(kW) * kC * kNS * kSlotPitch * sizeof(double);
      ensure_dynamic_smem(k_mstep_stream<kC, kW, kNS>, sm);
      static int per_sm[64] = {0};  // resident blocks per SM, per device
      int dev = 0;
      CK(cudaGetDevice(&dev));
      if (!per_sm[dev & 63])
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[dev & 63],
                                                         k_mstep_stream<kC, kW, kNS>, 32 * kW, sm));
      const uint64_t need = (max_leaves + label_leaves + kC * kW - 1) / (kC * kW);
      const unsigned grid = static_cast<unsigned>(
          std::max<uint64_t>(1, std::min<uint64_t>(need, uint64_t(per_sm[dev & 63]) * kNumSMs)));
      launch_pdl(k_mstep_stream<kC, kW, kNS>, dim3(grid), dim3(32 * kW), sm, s, fa,
                 reinterpret_cast<StreamCounters*>(mb.stream_cnt.get()));
      n -= 1;  // (one launch for both passes)
    } else {
      constexpr int kS = 8, kQ = 4;
      // chunk roots folded by the passes (series of <= 1024 chunks)
      if (label_leaves <= uint64_t(kFoldLeaf) * kFoldLeaf && hood_leaves <= uint64_t(kFoldLeaf) * kFoldLeaf &&
          chunks <= kMaxChunks) {
        fa.roots_sum = mb.roots.get();
        fa.roots_sq = mb.roots.get() + kMaxChunks;
        fa.tickets = mb.tickets.get();
      }
      const size_t ss = size_t(kS) * kFoldPitch * sizeof(double);
      const size_t sq = (size_t(kQ) * kFoldPitch + root_cap + (kSqThreads / 32) * kTreeScratch) *
                        sizeof(double);
      ensure_dynamic_smem(k_fold_sum<kS>, ss);
      ensure_dynamic_smem(k_fold_sq<kQ>, sq);
      launch_pdl(k_fold_sum<kS>, dim3(grid_for(max_leaves, kS)), dim3(32), ss, s, fa);
      launch_pdl(k_fold_sq<kQ>, dim3(grid_for(label_leaves, kQ)), dim3(kSqThreads), sq, s, fa);
    }
    n += 2;
  }
  if (launches) *launches += n;
}

}  // namespace

uint32_t label_tiles(uint32_t R) {
  return static_cast<uint32_t>((uint64_t(R) + kTileVerts - 1) / kTileVerts);
}

void launch_mstep(const double* mean, uint32_t R, uint32_t M, const uint8_t* lab_even,
                  const uint8_t* lab_odd, const double* hist, uint64_t Hs, int ring,
                  const uint32_t* unconv, int map_max, int fixed, double* params, double* em_out,
                  MStepBuffers& mb, cudaStream_t s, uint64_t* launches, bool counts_ready,
                  bool scattered, const EmEpilogueArgs* ep, const double* hood_parts) {
  mstep_core(mean, R, M, lab_even, lab_odd, unconv, map_max, fixed, hist, Hs, ring, params,
             em_out, mb, s, launches, counts_ready, scattered, ep, hood_parts);
}

void launch_fold_trees(bool sq, uint32_t M, uint64_t Hs, const uint32_t* unconv, int map_max,
                       int fixed, double* params, double* em_out, MStepBuffers& mb,
                       const double* hood_parts, cudaStream_t s) {
  (void)Hs;
  const uint64_t leaves = mb.partials.cap;  // >= every series' leaves
  const size_t smem = (((leaves + kFoldLeaf - 1) / kFoldLeaf + 2) / 2 * 2 + 8 * kTreeScratch) *
                      sizeof(double);
  if (sq) {
    ensure_dynamic_smem(k_fold_trees<true>, smem);
    launch_pdl(k_fold_trees<true>, dim3(1), dim3(256), smem, s, (const uint32_t*)mb.layout.get(),
               M, unconv, map_max, fixed, params, (const double*)mb.partials.get(), hood_parts,
               em_out);
  } else {
    ensure_dynamic_smem(k_fold_trees<false>, smem);
    launch_pdl(k_fold_trees<false>, dim3(1), dim3(256), smem, s, (const uint32_t*)mb.layout.get(),
               M, unconv, map_max, fixed, params, (const double*)mb.partials.get(), hood_parts,
               em_out);
  }
}

void launch_em_prologue(uint32_t* unconv, int map_max, cudaStream_t s) {
  launch_pdl(k_em_prologue, dim3(1), dim3(256), 0, s, unconv, map_max);
}

void launch_em_epilogue(const EmEpilogueArgs& a, cudaStream_t s) {
  const unsigned g = std::min<unsigned>(grid_for(a.R ? a.R : 1, 256), 4 * kNumSMs);
  launch_pdl(k_em_epilogue, dim3(g), dim3(256), 0, s, a);
}

void launch_row_leaves(const double* hist, int ring, uint64_t Hs, const uint32_t* unconv,
                       int map_max, int fixed, uint64_t hb, uint64_t he, double* out,
                       cudaStream_t s) {
  if (he <= hb) return;
  const uint64_t nl = (he + kFoldLeaf - 1) / kFoldLeaf - hb / kFoldLeaf;
  const size_t smem = size_t(kLeavesPerBlock) * kLeafStride * sizeof(double);
  ensure_dynamic_smem(k_row_leaves, smem);
  launch_pdl(k_row_leaves, dim3(grid_for(nl, kLeavesPerBlock)), dim3(256), smem, s, hist, ring,
             Hs, unconv, map_max, fixed, hb, he, out);
}

void init_log_table() {
  static std::mutex mu;
  static std::set<int> done;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (done.count(dev)) return;
  k_init_log_table<<<1, 128>>>();
  CK_LAUNCH();
  CK(cudaDeviceSynchronize());
  done.insert(dev);
}

void launch_log_cr(const double* x, double* out, uint64_t n, cudaStream_t s) {
  if (!n) return;
  k_log_cr<<<grid_for(n, 256), 256, 0, s>>>(x, out, n);
  CK_LAUNCH();
}

void mstep_reserve(MStepBuffers& mb, uint32_t R, uint32_t M, uint64_t Hs) {
  const uint32_t tiles = label_tiles(R);
  const uint32_t tiles_g = tiles ? tiles : 1;
  mb.counts.ensure(2 * uint64_t(tiles_g) * M);
  mb.tile_base.ensure(uint64_t(tiles_g) * M);
  mb.chunk_sum.ensure(((uint64_t(tiles_g) + kTileChunk - 1) / kTileChunk) * M);
  mb.layout.ensure(4 * M + 4);
  mb.x.ensure(uint64_t(R) + 2);  // (+2: the folds fetch 16-byte-aligned supersets)
  mb.partials.ensure((uint64_t(R) + kFoldLeaf - 1) / kFoldLeaf + M + (Hs + kFoldLeaf - 1) / kFoldLeaf + 1);
  mb.sq_partials.ensure((uint64_t(R) + kFoldLeaf - 1) / kFoldLeaf + M);
  if (!mb.done.get()) {
    CK(cudaMalloc(reinterpret_cast<void**>(&mb.done.p), 2 * sizeof(uint32_t)));
    mb.done.cap = 2;
    CK(cudaMemset(mb.done.p, 0, 2 * sizeof(uint32_t)));  // tickets re-arm themselves after
  }
  if (!mb.tickets.get()) {  // chunk tickets of both passes (zero; re-armed by their folders)
    CK(cudaMalloc(reinterpret_cast<void**>(&mb.tickets.p), 2 * kMaxChunks * sizeof(uint32_t)));
    mb.tickets.cap = 2 * kMaxChunks;
    CK(cudaMemset(mb.tickets.p, 0, 2 * kMaxChunks * sizeof(uint32_t)));
    mb.roots.ensure(2 * kMaxChunks);
  }
  if (!mb.stream_cnt.get()) {
    const size_t words = (sizeof(StreamCounters) + 3) / 4;
    CK(cudaMalloc(reinterpret_cast<void**>(&mb.stream_cnt.p), words * sizeof(uint32_t)));
    mb.stream_cnt.cap = words;
    CK(cudaMemset(mb.stream_cnt.p, 0, words * sizeof(uint32_t)));
  }
}

void launch_update_parameters_u32(const double* mean, uint32_t R, uint32_t M,
                                  const uint32_t* labels, double* params, MStepBuffers& mb,
                                  DevBuf<uint8_t>& lab_tmp, cudaStream_t s) {
  uint8_t* lab = lab_tmp.ensure(R);
  uint32_t* e = mb.err.ensure(1);
  CK(cudaMemsetAsync(e, 0, sizeof(uint32_t), s));
  if (R) {
    k_u32_to_u8_checked<<<grid_for(R, 256), 256, 0, s>>>(labels, lab, R, M, e);
    CK_LAUNCH();
  }
  uint32_t h_err = 0;
  CK(cudaMemcpyAsync(&h_err, e, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (h_err) fail(DPMRF_INVALID_ARGUMENT, "update_parameters: label out of range");
  if (R == 0) return;
  double* eo = mb.em_scratch.ensure(2 + 2 * M);
  mstep_core(mean, R, M, lab, lab, nullptr, 1, 1, nullptr, 0, 1, params, eo, mb, s, nullptr,
             /*counts_ready=*/false, /*scattered=*/false, nullptr, nullptr);
}

}  // namespace dpmrf_b200

#ifdef DPMRF_PROBE
extern "C" int dpmrf_probe_read(unsigned long long* blk, unsigned long long* tail) {
  if (cudaMemcpyFromSymbol(blk, dpmrf_b200::g_probe_blk, sizeof(dpmrf_b200::g_probe_blk)) !=
      cudaSuccess)
    return 1;
  return cudaMemcpyFromSymbol(tail, dpmrf_b200::g_probe_tail, sizeof(dpmrf_b200::g_probe_tail)) !=
         cudaSuccess;
}
#endif
