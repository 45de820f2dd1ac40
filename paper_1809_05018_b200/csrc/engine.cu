// engine.cu -- sm_100a kernels of the EM/MAP optimization phase.
//
// Reference: proj/src/mrf/optimize.cpp:31-74 and the step functions of
// proj/src/mrf/engine.cpp.  The reference replicates every hood slot once per
// label (M*S elements), sorts by slot, reduces by key, then sorts by vertex to
// pick each vertex's lowest-hood slot.  Because the replicated energy of an
// element depends only on (vertex, label) (engine.cpp:96-110: the Potts term
// counts GRAPH neighbors, not hood neighbors), every slot of a vertex carries
// the same minimum and argmin, so the sort/reduce/sort chain collapses to one
// per-vertex argmin (bit-identical; SURVEY.md key finding 1).  The hood sums
// then gather the per-vertex minima in slot order.
//
// The M-step folds and the EM tail live in mstep.cu; the helpers both use
// are in engine_dev.cuh.
#include <algorithm>

#include "engine_dev.cuh"
#include "scan.cuh"

namespace dpmrf_b200 {

namespace {

// ---------------------------------------------------------------------------
// Per-vertex energies + argmin + label commit.
//   discord_counts       engine.cpp:74-86   (labels frozen at iteration start)
//   compute_energies     engine.cpp:88-113  (label_energy order, model.hpp:66-72)
//   min_label_energies   engine.cpp:115-145 (ties -> smaller label: strict <)
//   update_labels        engine.cpp:171-191 (uncovered vertices keep labels)
// ---------------------------------------------------------------------------
template <int MT>
__device__ __forceinline__ uint32_t vertex_body(uint32_t v, const uint32_t* __restrict__ g_off,
                                            const uint32_t* __restrict__ g_nbr,
                                            const double* __restrict__ mean,
                                            const uint8_t* __restrict__ cover,
                                            const uint8_t* __restrict__ lab_in,
                                            uint8_t* __restrict__ lab_out,
                                            double* __restrict__ minE, uint32_t M_rt,
                                            const double* __restrict__ terms, double beta) {
  const uint8_t old = lab_in[v];
  if (!cover[v]) {
    lab_out[v] = old;
    return old;
  }
  const uint32_t M = MT > 0 ? uint32_t(MT) : M_rt;
  const uint32_t lo = g_off[v], hi = g_off[v + 1];
  const uint32_t deg = hi - lo;
  const double x = mean[v];
  double best;
  uint32_t best_l;
  if constexpr (MT == 2) {
    // labels are {0,1}: discord(0) = #neighbors labeled 1, discord(1) = deg - that
    uint32_t ones = 0;
    uint32_t a = lo;
    for (; a + 4 <= hi; a += 4) {
      const uint32_t u0 = g_nbr[a], u1 = g_nbr[a + 1], u2 = g_nbr[a + 2], u3 = g_nbr[a + 3];
      ones += uint32_t(lab_in[u0]) + uint32_t(lab_in[u1]) + uint32_t(lab_in[u2]) +
              uint32_t(lab_in[u3]);
    }
    for (; a < hi; ++a) ones += lab_in[g_nbr[a]];
    const double e0 = label_energy(x, terms[0], terms[2], terms[4], beta, ones);
    const double e1 = label_energy(x, terms[1], terms[3], terms[5], beta, deg - ones);
    best = e0;
    best_l = 0;
    if (e1 < best) {
      best = e1;
      best_l = 1;
    }
  } else if constexpr (MT > 0) {
    uint32_t cnt[MT];
#pragma unroll
    for (int l = 0; l < MT; ++l) cnt[l] = 0;
    for (uint32_t a = lo; a < hi; ++a) {
      const uint32_t c = lab_in[g_nbr[a]];
#pragma unroll
      for (int l = 0; l < MT; ++l) cnt[l] += (c == uint32_t(l));
    }
    best = label_energy(x, terms[0], terms[MT], terms[2 * MT], beta, deg - cnt[0]);
    best_l = 0;
#pragma unroll
    for (int l = 1; l < MT; ++l) {
      const double e = label_energy(x, terms[l], terms[MT + l], terms[2 * MT + l], beta,
                                    deg - cnt[l]);
      if (e < best) {
        best = e;
        best_l = l;
      }
    }
  } else {
    best = 0.0;
    best_l = 0;
    for (uint32_t l = 0; l < M; ++l) {
      uint32_t same = 0;
      for (uint32_t a = lo; a < hi; ++a) same += (lab_in[g_nbr[a]] == l);
      const double e = label_energy(x, terms[l], terms[M + l], terms[2 * M + l], beta, deg - same);
      if (l == 0 || e < best) {
        best = e;
        best_l = l;
      }
    }
  }
  minE[v] = best;
  lab_out[v] = static_cast<uint8_t>(best_l);
  return best_l;
}

template <int MT>
__global__ void __launch_bounds__(kVtxThreads)
    k_vertex_argmin(const uint32_t* __restrict__ g_off, const uint32_t* __restrict__ g_nbr,
                    const double* __restrict__ mean, const uint8_t* __restrict__ cover,
                    const uint8_t* __restrict__ lab_in, uint8_t* __restrict__ lab_out,
                    double* __restrict__ minE, uint32_t R, uint32_t M_rt,
                    const double* __restrict__ terms, double beta,
                    const uint32_t* __restrict__ unconv, int t, int fixed,
                    uint32_t* __restrict__ tile_counts, uint32_t tiles, uint32_t v_begin) {
  pdl_wait();
  if (map_iter_skipped(unconv, t, fixed)) return;
  const uint32_t v = v_begin + blockIdx.x * kVtxThreads + threadIdx.x;
  const bool valid = v < R;  // R = end of the owned range
  uint32_t lab = 0;
  if (valid) lab = vertex_body<MT>(v, g_off, g_nbr, mean, cover, lab_in, lab_out, minE, M_rt, terms, beta);
  const uint32_t M = MT > 0 ? uint32_t(MT) : M_rt;
  if (tile_counts && blockIdx.x < tiles)
    block_label_counts(tile_counts + (uint64_t(t & 1) * tiles + blockIdx.x) * M, M, valid, lab);
}

// ---------------------------------------------------------------------------
// Hood energy sums + convergence window.
//   neighborhood_energy_sums  engine.cpp:147-152 (fold_range in slot order)
//   check_convergence         engine.cpp:154-169 (!(|last-prev| < tol) -> 0)
//   all_set                   optimize.cpp:25-27 (block count -> one atomic)
// ---------------------------------------------------------------------------
__device__ __noinline__ double hood_fold_long(const uint32_t* __restrict__ h_mem,
                                              const double* __restrict__ minE, uint32_t lo,
                                              uint32_t hi) {
  // fold_range for more than kFoldLeaf slots: leaves + pairwise tree.
  TreeStack<double, AddOp> st;
  for (uint32_t b = lo; b < hi; b += kFoldLeaf) {
    const uint32_t e = min(hi, b + kFoldLeaf);
    double acc = minE[h_mem[b]];
    for (uint32_t s = b + 1; s < e; ++s) acc = __dadd_rn(acc, minE[h_mem[s]]);
    st.push(acc, AddOp{});
  }
  return st.finish(AddOp{});
}

// Hood h of iteration t; returns 1 if NOT converged (0 for h >= Hs).
__device__ __forceinline__ int hood_body(uint64_t h, const uint32_t* __restrict__ s_off,
                                         const uint32_t* __restrict__ h_mem,
                                         const double* __restrict__ minE,
                                         double* __restrict__ hist, uint8_t* __restrict__ flags,
                                         uint64_t Hs, int t, int L, int ring, double tol) {
  if (h >= Hs) return 0;
  // (hoisting the window loads and fully unrolling <= 16-slot hoods raised
  // register use to 64 and measured slower at both 2560^2 and 16384^2)
  const int R1 = ring;  // >= L+1 rows; == map_max rows when the full trace is kept
  const uint32_t lo = s_off[h], hi = s_off[h + 1];
  double sum;
  if (hi - lo <= kFoldLeaf) {
    sum = minE[h_mem[lo]];
    uint32_t s = lo + 1;
    for (; s + 4 <= hi; s += 4) {
      const double a0 = minE[h_mem[s]], a1 = minE[h_mem[s + 1]];
      const double a2 = minE[h_mem[s + 2]], a3 = minE[h_mem[s + 3]];
      sum = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(sum, a0), a1), a2), a3);
    }
    for (; s < hi; ++s) sum = __dadd_rn(sum, minE[h_mem[s]]);
  } else {
    sum = hood_fold_long(h_mem, minE, lo, hi);
  }
  hist[uint64_t(t % R1) * Hs + h] = sum;
  int ok = 0;
  if (t >= L) {
    ok = 1;
    for (int i = 1; i <= L; ++i) {
      const double prev = hist[uint64_t((t - i) % R1) * Hs + h];
      if (!(fabs(__dsub_rn(sum, prev)) < tol)) {
        ok = 0;
        break;
      }
    }
  }
  if (flags) flags[uint64_t(t) * Hs + h] = static_cast<uint8_t>(ok);
  return !ok;
}

__global__ void __launch_bounds__(kHoodThreads)
    k_hood_sums(const uint32_t* __restrict__ s_off, const uint32_t* __restrict__ h_mem,
                const double* __restrict__ minE, double* __restrict__ hist,
                uint8_t* __restrict__ flags, uint64_t Hs, int t, int L, int ring, double tol,
                uint32_t* __restrict__ unconv, int fixed, uint64_t h_begin, uint64_t h_end) {
  pdl_wait();
  if (map_iter_skipped(unconv, t, fixed)) return;
  const uint64_t h = h_begin + uint64_t(blockIdx.x) * kHoodThreads + threadIdx.x;
  const int not_conv =
      h < h_end ? hood_body(h, s_off, h_mem, minE, hist, flags, Hs, t, L, ring, tol) : 0;
  const int block_unconv = __syncthreads_count(not_conv);
  if (threadIdx.x == 0 && block_unconv) atomicAdd(&unconv[t], uint32_t(block_unconv));
}

__global__ void k_init_labels(uint8_t* lab, uint32_t R, uint32_t M, uint64_t seed) {
  const uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= R) return;
  // draw 2M+v of the init_random stream (engine.cpp:29: mu, sigma, then labels)
  lab[v] = static_cast<uint8_t>(splitmix_draw(seed, 2ull * M + v) % M);
}

__global__ void k_u8_to_u32(const uint8_t* __restrict__ in, uint32_t* __restrict__ out,
                            uint64_t n) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}

// ---- structure preparation -------------------------------------------------
__global__ void k_validate(const uint32_t* __restrict__ g_off, const uint32_t* __restrict__ g_nbr,
                           uint32_t R, uint64_t A, const uint32_t* __restrict__ h_off,
                           const uint32_t* __restrict__ h_mem, uint64_t H, uint64_t S,
                           uint32_t* err, uint32_t* empty_hoods) {
  const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  uint32_t e = 0, empties = 0;
  for (uint64_t i = tid; i < S; i += stride)
    if (h_mem[i] >= R) e |= 1u;
  for (uint64_t i = tid; i < A; i += stride)
    if (g_nbr[i] >= R) e |= 2u;
  for (uint64_t h = tid; h < H; h += stride) {
    const uint32_t a = h_off[h], b = h_off[h + 1];
    if (b < a) e |= 4u;
    empties += (a == b);
  }
  for (uint64_t v = tid; v < R; v += stride)
    if (g_off[v + 1] < g_off[v]) e |= 8u;
  if (tid == 0) {
    if (h_off[0] != 0 || h_off[H] != S) e |= 4u;
    if (g_off[0] != 0 || g_off[R] != A) e |= 8u;
  }
  if (e) atomicOr(err, e);
  if (empties) atomicAdd(empty_hoods, empties);
}

// (runs before prepare() has checked the members: out-of-range ones skipped)
__global__ void k_cover(const uint32_t* __restrict__ h_mem, uint64_t S, uint8_t* cover,
                        uint32_t R) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < S; i += stride) {
    const uint32_t m = h_mem[i];
    if (m < R) cover[m] = 1;
  }
}

__global__ void k_nonempty_flags(const uint32_t* __restrict__ h_off, uint64_t H, uint32_t* f) {
  const uint64_t h = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (h < H) f[h] = h_off[h + 1] != h_off[h];
}

__global__ void k_compact_offsets(const uint32_t* __restrict__ h_off, uint64_t H, uint64_t S,
                                  const uint32_t* __restrict__ pos, uint32_t* s_off) {
  const uint64_t h = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (h < H && h_off[h + 1] != h_off[h]) s_off[pos[h]] = h_off[h];
  if (h == 0) s_off[pos[H]] = static_cast<uint32_t>(S);
}

}  // namespace

// ---- launchers -----------------------------------------------------------------
#ifndef DPMRF_FUSED_MINB
#define DPMRF_FUSED_MINB 8  // 8 x 256 threads per SM: caps the fused kernel at 32 registers
#endif
namespace {
// The 2-label, <= 8-slot instance fits 32 registers without spilling, so it
// runs 8 blocks per SM.
// The config C instances (5 labels) at 8 blocks per SM: 32 registers and a
// 40-byte spill, one wave of 2048 threads per SM (2560^2 brick: 12.8 k vs
// 12.5 k EM-it/s at 5 blocks / 48 registers, 12.4 k at 6 / 40; before the
// round-2 instruction diet 5 blocks won); the other wide instances keep the
// compiler's choice.
#ifndef DPMRF_FUSED_MINB_M5
#define DPMRF_FUSED_MINB_M5 8
#endif
#ifndef DPMRF_FUSED_MINB_VP2
#define DPMRF_FUSED_MINB_VP2 8
#endif
#ifndef DPMRF_ACT_MINB
#define DPMRF_ACT_MINB 8
#endif
constexpr int fused_min_blocks(int mt, int kh, int vp = 1, bool act = false) {
  return act ? DPMRF_ACT_MINB
             : (mt == 2 && kh == 8 ? (vp == 2 ? DPMRF_FUSED_MINB_VP2 : DPMRF_FUSED_MINB)
                                   : (mt == 5 ? DPMRF_FUSED_MINB_M5 : 1));
}
#ifndef DPMRF_HOIST_MEAN
#define DPMRF_HOIST_MEAN 0
#endif
// The static region mean is read before griddepcontrol.wait on the
// one-vertex instances (2560^2: part of the +10% of the index diet); the
// two-vertex instance reads it after the wait (hoisting both means costs it
// spills: 16384^2 662 vs 675 EM-it/s).
constexpr bool kHoistMean = DPMRF_HOIST_MEAN != 0;
constexpr int kWinRegs = 3;  // window rows held in registers (default L = 3)
#ifndef DPMRF_ACT_BLOCKS
#define DPMRF_ACT_BLOCKS (8 * 148)
#endif
constexpr uint32_t kActBlocks = DPMRF_ACT_BLOCKS;  // blocks per list-driven pass
#ifdef DPMRF_PROBE
// processed vertices / series per MAP iteration in active-set runs (probe builds)
__device__ unsigned long long g_act_probe[2][64];
#define ACT_PROBE(k, t) atomicAdd(&g_act_probe[k][(t) & 63], 1ull)
#else
#define ACT_PROBE(k, t) do {} while (0)
#endif
#ifndef DPMRF_VP2_MIN
#define DPMRF_VP2_MIN (1u << 20)
#endif
constexpr uint32_t kVertsPerThreadMin = DPMRF_VP2_MIN;  // owned vertices for 2 per thread
template <int MT, int K>
__global__ void __launch_bounds__(kVtxThreads)
    k_vertex_packed(MapArgs a, const uint8_t* __restrict__ lab_in, uint8_t* __restrict__ lab_out,
                    int t);
template <int K>
__global__ void __launch_bounds__(kHoodThreads) k_hood_packed(MapArgs a, int t);
template <int MT, int KV, int KH, int VP, bool kAct = false>
__global__ void __launch_bounds__(kVtxThreads, fused_min_blocks(MT, KH, VP, kAct))
    k_map_fused(MapArgs a, const uint8_t* __restrict__ lab_in, uint8_t* __restrict__ lab_out,
                const double* __restrict__ minE_prev, double* __restrict__ minE_cur, int t,
                uint32_t nh, uint32_t nv, ScatterArgs sc);
}  // namespace


bool map_fused_supported(const MapArgs& a) { return a.adj_k && a.hood_k; }

// The fused layouts with an active-set instance: the grid graphs with two
// labels (configs A, B, D, E) and the brick graphs with five (config C).
bool map_active_supported(const MapArgs& a) {
  // (brick graphs with five labels keep changing labels in every EM
  // iteration: their flags stay dense and the dense loop is faster -- 12.8 k
  // vs 5.9 k EM-it/s at 2560^2 -- so they keep the dense loop)
  return map_fused_supported(a) && a.M == 2 && a.adj_k == 4 && a.hood_k == 8;
}

namespace {
// The launch's copy of the arguments with the ring rows of hood iteration th.
MapArgs with_rows(const MapArgs& a, int th) {
  MapArgs r = a;
  const int R1 = a.ring > 0 ? a.ring : 1;
  r.row_t = th >= 0 ? th % R1 : 0;
  r.row_p = th >= 1 ? (th - 1) % R1 : 0;
  return r;
}
}  // namespace

bool mstep_tail_fusable(uint32_t R, uint32_t M) {
  const uint64_t tiles = (uint64_t(R) + kTileVerts - 1) / kTileVerts;
  return tiles && tiles * M <= kSelfScanMax;
}

void launch_map_fused(const MapArgs& a, const uint8_t* lab_in, uint8_t* lab_out,
                      const double* minE_prev, double* minE_cur, int t, int map_max,
                      cudaStream_t s, const ScatterArgs* sc) {
  const int sel = (a.M == 2 ? 0 : 4) + (a.adj_k == 8 ? 2 : 0) + (a.hood_k == 16 ? 1 : 0);
  const bool k12 = a.hood_k == 12;  // brick hoods (<= 13 slots)
  // Two vertices per thread on large graphs (+4% at 16384^2: more loads in
  // flight per thread); one on small ones, where the extra per-thread
  // latency shows (-3% at 2560^2).
  const int vp = sel == 0 && a.v_end - a.v_begin >= kVertsPerThreadMin ? 2 : 1;
  const uint32_t nh = t >= 1 ? grid_for(a.h_end - a.h_begin, kHoodThreads) : 0u;
  const uint32_t nv =
      t < map_max ? grid_for(a.v_end - a.v_begin, uint64_t(kVtxThreads) * vp) : 0u;
  const bool tail = sc && t == map_max;
  const uint32_t ns = tail ? sc->tiles : 0u;
  const ScatterArgs scv = tail ? *sc : ScatterArgs{};
  const size_t smem = tail ? scatter_small_smem(sc->M) : 0;
  const dim3 g(nh + nv + ns), blk(kVtxThreads);
  MapArgs ar = with_rows(a, t - 1);
  // fixed work: only the last vertex pass's label counts are ever read (by
  // the M-step's grouping), so the other passes skip their block counts
  if (a.fixed && t != map_max - 1) ar.tile_counts = nullptr;
  if (a.act_vflag) {  // active-set instances (map_active_supported)
    // list-driven passes: a fixed grid of kActBlocks blocks (per pass)
    const bool sh = t - 1 >= 1, sv = t >= 2 && !ar.tile_counts;
    const uint32_t nh2 = t >= 1 ? (sh ? std::min<uint32_t>(kActBlocks, grid_for(a.h_end - a.h_begin, kHoodThreads))
                                      : grid_for(a.h_end - a.h_begin, kHoodThreads)) : 0u;
    const uint32_t nv2 = t < map_max ? (sv ? std::min<uint32_t>(kActBlocks, grid_for(a.v_end - a.v_begin, kVtxThreads))
                                           : grid_for(a.v_end - a.v_begin, uint64_t(kVtxThreads) * vp)) : 0u;
    const dim3 g2(nh2 + nv2 + ns);
#define MFA(MT, KV, KH, VP)                                                                 \
  launch_pdl(k_map_fused<MT, KV, KH, VP, true>, g2, blk, smem, s, ar, lab_in, lab_out,       \
             minE_prev, minE_cur, t, nh2, nv2, scv)
    if (vp == 2) MFA(2, 4, 8, 2);
    else MFA(2, 4, 8, 1);
#undef MFA
    return;
  }
#define MF4(MT, KV, KH, VP)                                                              \
  launch_pdl(k_map_fused<MT, KV, KH, VP>, g, blk, smem, s, ar, lab_in, lab_out, minE_prev,  \
             minE_cur, t, nh, nv, scv)
#define MF(MT, KV, KH) MF4(MT, KV, KH, 1)
  if (a.M == 5 && a.adj_k == 8 && a.hood_k == 16) {  // config C's layout: label loop unrolled
    MF(5, 8, 16);
    return;
  }
  if (k12) {
    if (a.M == 5 && a.adj_k == 8) MF(5, 8, 12);  // config C
    else if (a.M == 2) {
      if (a.adj_k == 4) MF(2, 4, 12);
      else MF(2, 8, 12);
    } else {
      if (a.adj_k == 4) MF(0, 4, 12);
      else MF(0, 8, 12);
    }
    return;
  }
  switch (sel) {
    case 0:
      if (vp == 2)
        MF4(2, 4, 8, 2);
      else
        MF(2, 4, 8);
      break;
    case 1: MF(2, 4, 16); break;
    case 2: MF(2, 8, 8); break;
    case 3: MF(2, 8, 16); break;
    case 4: MF(0, 4, 8); break;
    case 5: MF(0, 4, 16); break;
    case 6: MF(0, 8, 8); break;
    default: MF(0, 8, 16); break;
  }
#undef MF
#undef MF4
}

void launch_vertex_argmin(const MapArgs& a, const uint8_t* lab_in, uint8_t* lab_out, int t,
                          cudaStream_t s) {
  const dim3 g(grid_for(a.v_end - a.v_begin, kVtxThreads)), blk(kVtxThreads);
  if (a.adj_k) {
    if (a.M == 2) {
      if (a.adj_k == 4) launch_pdl(k_vertex_packed<2, 4>, g, blk, 0, s, a, lab_in, lab_out, t);
      else launch_pdl(k_vertex_packed<2, 8>, g, blk, 0, s, a, lab_in, lab_out, t);
    } else {
      if (a.adj_k == 4) launch_pdl(k_vertex_packed<0, 4>, g, blk, 0, s, a, lab_in, lab_out, t);
      else launch_pdl(k_vertex_packed<0, 8>, g, blk, 0, s, a, lab_in, lab_out, t);
    }
    return;
  }
#define VA_ARGS                                                                                \
  a.g_off, a.g_nbr, a.mean, a.cover, lab_in, lab_out, a.minE, a.v_end, a.M, a.terms, a.beta, \
      a.unconv, t, a.fixed, a.tile_counts, a.tiles, a.v_begin
  switch (a.M) {
    case 2: launch_pdl(k_vertex_argmin<2>, g, blk, 0, s, VA_ARGS); break;
    case 3: launch_pdl(k_vertex_argmin<3>, g, blk, 0, s, VA_ARGS); break;
    case 4: launch_pdl(k_vertex_argmin<4>, g, blk, 0, s, VA_ARGS); break;
    case 5: launch_pdl(k_vertex_argmin<5>, g, blk, 0, s, VA_ARGS); break;
    case 6: launch_pdl(k_vertex_argmin<6>, g, blk, 0, s, VA_ARGS); break;
    case 7: launch_pdl(k_vertex_argmin<7>, g, blk, 0, s, VA_ARGS); break;
    case 8: launch_pdl(k_vertex_argmin<8>, g, blk, 0, s, VA_ARGS); break;
    default: launch_pdl(k_vertex_argmin<0>, g, blk, 0, s, VA_ARGS); break;
  }
#undef VA_ARGS
}

void launch_hood_sums(const MapArgs& a, int t, cudaStream_t s) {
  const dim3 g(grid_for(a.h_end - a.h_begin, kHoodThreads)), blk(kHoodThreads);
  if (a.hood_k) {
    const MapArgs ar = with_rows(a, t);
    if (a.hood_k == 8) launch_pdl(k_hood_packed<8>, g, blk, 0, s, ar, t);
    else if (a.hood_k == 12) launch_pdl(k_hood_packed<12>, g, blk, 0, s, ar, t);
    else launch_pdl(k_hood_packed<16>, g, blk, 0, s, ar, t);
    return;
  }
  launch_pdl(k_hood_sums, g, blk, 0, s, a.s_off, a.h_mem, (const double*)a.minE, a.hist,
               a.flags, a.Hs, t, a.L, a.ring, a.tol, a.unconv, a.fixed, a.h_begin, a.h_end);
}

namespace {

// ---------------------------------------------------------------------------
// Packed-layout MAP kernels.  The region graph and hoods are static for the
// whole optimization, so they are re-laid out once (launch_pack_*) for HBM:
// a vertex's neighbor list becomes K int16 deltas (one 8/16-byte vector load,
// no offsets lookup) and a hood becomes its first member plus K u16 deltas
// (one u32 + one/two 16-byte vector loads).  Per MAP iteration at 16384^2 this
// moves ~45% fewer bytes than the u32 CSR (offsets + ids).  The arithmetic and
// the fold order are exactly those of vertex_body / hood_body: discord counts
// are integers, and hood members stay in ascending (slot) order.
// ---------------------------------------------------------------------------
template <int K>
__device__ __forceinline__ void load_i16(const int16_t* __restrict__ p, int16_t (&d)[K]) {
  static_assert(K == 4 || K == 8, "adjacency pack width");
  if constexpr (K == 4) {
    const uint2 w = *reinterpret_cast<const uint2*>(p);
    const uint32_t u[2] = {w.x, w.y};
#pragma unroll
    for (int i = 0; i < 4; ++i) d[i] = static_cast<int16_t>(u[i >> 1] >> (16 * (i & 1)));
  } else {
    const uint4 w = *reinterpret_cast<const uint4*>(p);
    const uint32_t u[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] = static_cast<int16_t>(u[i >> 1] >> (16 * (i & 1)));
  }
}

// Vertex pass over P vertices per thread (v, v + 256, ...: block blk covers
// the P label tiles P*blk .. P*blk + P-1).  All structure loads of the P
// vertices are issued before their label gathers.
// The static structure (packed adjacency, cover flags) is read BEFORE
// griddepcontrol.wait -- it never changes during optimize, so the loads
// overlap the predecessor's drain -- and the skip decision (the previous
// iteration's unconverged counter) is read beside the first dependent loads
// rather than ahead of them: one memory round trip less per launch.
// Energies of every label (label_energy, model.hpp:66-72, in that order) and
// the argmin with ties to the smaller label (engine.cpp:115-145: strict <).
template <int MT, int K>
__device__ __forceinline__ void vertex_argmin_packed(const MapArgs& a, uint32_t M, double x,
                                                     const uint8_t (&nb)[K], uint32_t deg,
                                                     double& best, uint32_t& best_l) {
  const double* T = a.terms;
  if constexpr (MT == 2) {
    uint32_t ones = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) ones += (nb[k] == 1);
    const double e0 = label_energy(x, T[0], T[2], T[4], a.beta, ones);
    const double e1 = label_energy(x, T[1], T[3], T[5], a.beta, deg - ones);
    best = e0;
    best_l = 0;
    if (e1 < best) {
      best = e1;
      best_l = 1;
    }
  } else {
    best = 0.0;
    best_l = 0;
    for (uint32_t l = 0; l < M; ++l) {
      uint32_t same = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) same += (nb[k] == l);
      const double e = label_energy(x, T[l], T[M + l], T[2 * M + l], a.beta, deg - same);
      if (l == 0 || e < best) {
        best = e;
        best_l = l;
      }
    }
  }
}

// Active-set flag slices (rows padded to 16 bytes: the sparse passes read
// 16 flags per thread with one vector load).
__device__ __forceinline__ uint64_t act_vpitch(const MapArgs& a) { return (uint64_t(a.R) + 15) & ~15ull; }
__device__ __forceinline__ uint64_t act_hpitch(const MapArgs& a) { return (a.Hs + 15) & ~15ull; }
__device__ __forceinline__ uint8_t* act_vflags(const MapArgs& a, int t) {
  return a.act_vflag + uint64_t(t & 1) * act_vpitch(a);
}
__device__ __forceinline__ uint8_t* act_hflags(const MapArgs& a, int t) {
  return a.act_hflag + uint64_t(t & 1) * act_hpitch(a);
}

__device__ __forceinline__ uint32_t act_vtiles(const MapArgs& a) { return (a.R + 255) / 256; }
__device__ __forceinline__ uint32_t act_htiles(const MapArgs& a) {
  return static_cast<uint32_t>((a.Hs + 255) / 256);
}
// list counters of iteration t of the current EM: [0] vertex tiles, [1] series tiles
__device__ __forceinline__ uint32_t* act_counts(const MapArgs& a, int t) {
  const uint32_t e = a.unconv[kEmCount];
  return a.act_cnt + 2 * (uint64_t(e) * a.act_stride + t);
}
// flag item idx for iteration t (vertex: k = 0, series: k = 1) and list its tile
__device__ __forceinline__ void act_flag(const MapArgs& a, int k, int t, uint32_t idx) {
  uint8_t* items = k == 0 ? act_vflags(a, t) : act_hflags(a, t);
  if (items[idx]) return;  // (its tile is listed already)
  items[idx] = 1;
  const uint32_t tile = idx >> 8;
  const uint32_t nt = k == 0 ? act_vtiles(a) : act_htiles(a);
  uint32_t* tiles = (k == 0 ? a.act_vtile : a.act_htile) + uint64_t(t & 1) * nt;
  // (a plain read first: a tile's 256 items must not all hit one atomic)
  if (*reinterpret_cast<volatile uint32_t*>(&tiles[tile]) == 0u &&
      atomicExch(&tiles[tile], 1u) == 0u) {
    uint32_t* list = (k == 0 ? a.act_vlist : a.act_hlist) + uint64_t(t & 1) * nt;
    list[atomicAdd(act_counts(a, t) + k, 1u)] = tile;
  }
}

// After vertex v of iteration t (t >= 1) computed (best, best_l) from its
// old label: who is evaluated next.  A new label re-evaluates the neighbors
// (their discord counts) and v (the label double buffer); a new minimum v
// (the minima double buffer) and -- once the hood pass is flag-driven
// (t > L) -- every series v is in.
template <int K>
__device__ __forceinline__ void act_mark(const MapArgs& a, int t, uint32_t v, const int16_t (&d)[K],
                                         uint32_t old, uint32_t best_l, double best,
                                         double prev) {
  const bool lab_changed = best_l != old;
  const bool min_changed = __double_as_longlong(prev) != __double_as_longlong(best);
  if (lab_changed || min_changed) act_flag(a, 0, t + 1, v);
  if (lab_changed) {
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (d[k] != INT16_MIN)
        act_flag(a, 0, t + 1, v + static_cast<uint32_t>(static_cast<int32_t>(d[k])));
  }
  if (min_changed)
    for (uint32_t i = a.inv_off[v]; i < a.inv_off[v + 1]; ++i) act_flag(a, 1, t, a.inv_ser[i]);
}

template <int MT, int K, int P = 1, bool kAct = false>
__device__ __forceinline__ void vertex_packed_body(const MapArgs& a,
                                                   const uint8_t* __restrict__ lab_in,
                                                   uint8_t* __restrict__ lab_out,
                                                   double* __restrict__ minE, int t,
                                                   uint32_t blk, int skip_t,
                                                   const double* __restrict__ minE_prev = nullptr) {
  const uint32_t M = MT > 0 ? uint32_t(MT) : a.M;
  const uint32_t v0 = a.v_begin + blk * (kVtxThreads * P) + threadIdx.x;
  // active-set (a.act_vflag): iterations 0 and 1 evaluate every vertex (new
  // label terms; the minima double buffer is stale from the last EM), later
  // ones only the flagged vertices, whose structure is read once the flag
  // is known
  constexpr bool act = kAct;
  const bool sparse = act && t >= 2;
  int16_t d[P][K];
  uint8_t old[P], cov[P], run[P];
  double xs[P];
#pragma unroll
  for (int j = 0; j < P; ++j) {
    const uint32_t v = v0 + j * kVtxThreads;
    xs[j] = 0.0;
    run[j] = 1;
    if (v < a.v_end && !sparse) {
      load_i16<K>(a.adj_pk + uint64_t(v) * K, d[j]);
      cov[j] = a.cover[v];
      if (kHoistMean || P == 1) xs[j] = a.mean[v];
    }
  }
  pdl_wait();
  uint8_t* vcur = act ? act_vflags(a, t) : nullptr;
  if (kAct) {
    // this pass consumes the tiles of parity t; the first pass of an EM also
    // clears parity 1 (left over from the previous EM)
    const uint32_t nt = act_vtiles(a);
    if (threadIdx.x == 0)
#pragma unroll
      for (int j = 0; j < P; ++j) {
        const uint32_t tile = blk * P + j;
        if (tile < nt) {
          a.act_vtile[uint64_t(t & 1) * nt + tile] = 0;
          if (t == 0) a.act_vtile[nt + tile] = 0;
        }
      }
    if (t == 0) {
#pragma unroll
      for (int j = 0; j < P; ++j) {
        const uint32_t v = v0 + j * kVtxThreads;
        if (v < a.v_end) act_vflags(a, 1)[v] = 0;
      }
      // the series flags and tiles of parity 1 (marked from the next launch
      // on; parity 0 is cleared by the dense hood pass of iteration 0)
      const uint64_t nthreads =
          uint64_t((a.v_end - a.v_begin + kVtxThreads * P - 1) / (kVtxThreads * P)) * kVtxThreads;
      const uint64_t g = uint64_t(blk) * kVtxThreads + threadIdx.x;
      uint8_t* h1 = act_hflags(a, 1);
      for (uint64_t h = g; h < a.Hs; h += nthreads) h1[h] = 0;
      const uint32_t ht = act_htiles(a);
      for (uint64_t k = g; k < ht; k += nthreads) a.act_htile[ht + k] = 0;
    }
  }
#pragma unroll
  for (int j = 0; j < P; ++j) {
    const uint32_t v = v0 + j * kVtxThreads;
    if (v < a.v_end) {
      if (act) {
        run[j] = !sparse || vcur[v];
        if (run[j]) vcur[v] = 0;
        if (sparse && run[j]) {
          load_i16<K>(a.adj_pk + uint64_t(v) * K, d[j]);
          cov[j] = a.cover[v];
          if (kHoistMean || P == 1) xs[j] = a.mean[v];
        }
      }
      // (a vertex not re-evaluated keeps its label: the output buffer holds it)
      old[j] = run[j] ? lab_in[v] : lab_out[v];
    }
  }
  if (map_iter_skipped(a.unconv, skip_t, a.fixed)) return;  // uniform over the grid
  uint32_t nl[P];
#pragma unroll
  for (int j = 0; j < P; ++j) {
    const uint32_t v = v0 + j * kVtxThreads;
    nl[j] = 0;
    if (v >= a.v_end) continue;
    if (!run[j]) {
      nl[j] = old[j];
      continue;
    }
    if (!cov[j]) {
      lab_out[v] = old[j];
      nl[j] = old[j];
      continue;
    }
    uint8_t nb[K];
    uint32_t deg = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const bool ok = d[j][k] != INT16_MIN;
      deg += ok;
      // (u32 wrap-around: v + d is a vertex id whenever the slot is present)
      nb[k] = ok ? lab_in[v + static_cast<uint32_t>(static_cast<int32_t>(d[j][k]))]
                 : uint8_t(0xFF);
    }
    const double x = kHoistMean || P == 1 ? xs[j] : a.mean[v];
    double best;
    uint32_t best_l;
    vertex_argmin_packed<MT, K>(a, M, x, nb, deg, best, best_l);
    minE[v] = best;
    lab_out[v] = static_cast<uint8_t>(best_l);
    nl[j] = best_l;
    if (kAct && t >= 1) act_mark<K>(a, t, v, d[j], old[j], best_l, best, minE_prev[v]);
  }
  if (a.tile_counts) {
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const uint32_t tile = blk * P + j;
      if (tile < a.tiles)  // (uniform per block)
        block_label_counts(a.tile_counts + (uint64_t(t & 1) * a.tiles + tile) * M, M,
                           v0 + j * kVtxThreads < a.v_end, nl[j]);
    }
  }
}

template <int MT, int K>
__global__ void __launch_bounds__(kVtxThreads)
    k_vertex_packed(MapArgs a, const uint8_t* __restrict__ lab_in, uint8_t* __restrict__ lab_out,
                    int t) {
  vertex_packed_body<MT, K>(a, lab_in, lab_out, a.minE, t, blockIdx.x, t);
}

// A hood's K u16 deltas as K/2 words: 16-byte loads for K = 8 / 16, three
// 8-byte loads for K = 12 (rows of 24 bytes are only 8-byte aligned).
template <int K>
__device__ __forceinline__ void load_hood_row(const uint16_t* __restrict__ row,
                                              uint32_t (&u)[K / 2]) {
  if constexpr (K % 8 == 0) {
    const uint4* src = reinterpret_cast<const uint4*>(row);
#pragma unroll
    for (int q = 0; q < K / 8; ++q) {
      const uint4 w = src[q];
      u[4 * q] = w.x;
      u[4 * q + 1] = w.y;
      u[4 * q + 2] = w.z;
      u[4 * q + 3] = w.w;
    }
  } else {
    static_assert(K == 12, "hood pack width");
    const uint2* src = reinterpret_cast<const uint2*>(row);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const uint2 w = src[q];
      u[2 * q] = w.x;
      u[2 * q + 1] = w.y;
    }
  }
}

// One hood's sum (left fold of its members' minima in slot order,
// engine.cpp:147-152) + record + window test (engine.cpp:154-169); returns 1
// when the hood is not converged.
//
// The ring rows of iterations t and t-1 come precomputed with the launch
// (MapArgs::row_t / row_p, set by with_rows): no per-thread modulo, and the
// hood index stays 32-bit (one wide multiply-add per address).
template <int K>
__device__ __forceinline__ int hood_eval(const MapArgs& a, const double* __restrict__ minE, int t,
                                         uint32_t h, uint32_t base, const uint32_t (&u)[K / 2],
                                         const double* p1_over = nullptr,
                                         double* sum_out = nullptr, uint32_t* eq_out = nullptr) {
  const int R1 = a.ring;
  const int nwin = t >= a.L ? a.L : 0;
  double* __restrict__ row_t = a.hist + uint64_t(a.row_t) * a.Hs;
  const double* __restrict__ row_p = a.hist + uint64_t(a.row_p) * a.Hs;
  // Window test with an equal-run count: eq[h] = how many predecessors of
  // the previous row are bit-identical to it (a hood whose members' minima
  // did not change sums to the same bits).  Only row t-1 and the count are
  // read up front; an older row is read only when its comparison is not
  // already implied -- the previous comparison passed and the row is not
  // inside the equal run.  Same flags as reading every row (the skipped
  // comparisons are |x - x| = 0 < tol), 18 instead of 32 window bytes per
  // hood.
  // (a.eq is always set when the packed hood layout is in use)
  double p1 = 0.0;
  uint32_t e1 = 0;
  if (t >= 1) {
    p1 = p1_over ? *p1_over : row_p[h];
    e1 = a.eq[h];
  }
  double e[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {  // all gathers in flight before the fold
    const uint32_t dk = (u[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
    e[k] = dk != 0xFFFFu ? minE[base + dk] : 0.0;
  }
  // Absent slots add +0.0, which leaves every partial sum unchanged: a
  // minimum energy is never -0.0 (label_energy's q >= +0 and log sigma is
  // finite, so neither rounded sum can be -0), hence no partial sum is -0
  // and x + (+0) == x bit for bit (NaN stays the canonical NaN).  Same
  // bits as folding only the present members, without the selects.
  double sum = minE[base];
#pragma unroll
  for (int k = 0; k < K; ++k) sum = __dadd_rn(sum, e[k]);
  row_t[h] = sum;
  int ok = nwin > 0;
  const bool same = t >= 1 && sum == p1;  // (false for NaN)
  const uint32_t eq_new = same ? min(e1 + 1u, 255u) : 0u;
  a.eq[h] = static_cast<uint8_t>(eq_new);
  if (sum_out) *sum_out = sum;
  if (eq_out) *eq_out = eq_new;
  if (nwin) {
    if (!(fabs(__dsub_rn(sum, p1)) < a.tol)) {
      ok = 0;
    } else if (e1 + 1 < uint32_t(nwin)) {
      // rows t-1-e1 .. t-1 equal p1 (their comparisons are implied); read the rest
      int row = a.row_p - int(e1) - 1;  // row of iteration t - (e1 + 2)
      if (row < 0) row += R1;
      for (int i = int(e1) + 2; i <= nwin; ++i) {
        const double p = a.hist[uint64_t(row) * a.Hs + h];
        if (!(fabs(__dsub_rn(sum, p)) < a.tol)) {
          ok = 0;
          break;
        }
        row = row == 0 ? R1 - 1 : row - 1;
      }
    }
  }
  if (a.flags) a.flags[uint64_t(t) * a.Hs + h] = static_cast<uint8_t>(ok);
  return !ok;
}

// (static structure before griddepcontrol.wait, skip decision beside the
// first dependent loads -- see vertex_packed_body)
template <int K, bool kAct = false>
__device__ __forceinline__ void hood_packed_body(const MapArgs& a,
                                                 const double* __restrict__ minE, int t,
                                                 uint32_t blk, int skip_t) {
  static_assert(K == 8 || K == 12 || K == 16, "hood pack width");
  const uint32_t h = static_cast<uint32_t>(a.h_begin) + blk * kHoodThreads + threadIdx.x;
  const bool live = h < a.h_end;
  // active-set, after the window opened (t > L): only flagged series fold,
  // and their structure is read once the flag is known
  constexpr bool act = kAct;
  const bool sparse = act && t >= 1;
  uint32_t base = 0;
  uint32_t u[K / 2];
  if (live && !sparse) {
    base = a.hood_base[h];
    load_hood_row<K>(a.hood_pk + uint64_t(h) * K, u);
  }
  pdl_wait();
  int not_conv = 0;
  if (live) {
    if (map_iter_skipped(a.unconv, skip_t, a.fixed)) return;  // uniform over the grid
    if constexpr (!act) {
      not_conv = hood_eval<K>(a, minE, t, h, base, u);
    } else {
      uint8_t* flag = act_hflags(a, t) + h;
      const bool run = !sparse || *flag;
      if (threadIdx.x == 0) a.act_htile[uint64_t(t & 1) * act_htiles(a) + (h >> 8)] = 0;
      if (run) {
        *flag = 0;
        double over = 0.0;
        const double* p1o = nullptr;
        if (sparse) {
          base = a.hood_base[h];
          load_hood_row<K>(a.hood_pk + uint64_t(h) * K, u);
          if (a.act_lastp[h] != uint8_t(t - 1)) {
            // folded again after converged iterations: every window row
            // since equals its last sum (their ring slots are stale)
            over = a.act_hval[h];
            p1o = &over;
            int row = a.row_p;
            for (int i = 0; i < a.L; ++i) {
              a.hist[uint64_t(row) * a.Hs + h] = over;
              row = row == 0 ? a.ring - 1 : row - 1;
            }
          }
        }
        double sum;
        uint32_t eqn;
        not_conv = hood_eval<K>(a, minE, t, h, base, u, p1o, &sum, &eqn);
        a.act_hval[h] = sum;
        a.act_lastp[h] = static_cast<uint8_t>(t);
        // still open (not converged, or converged on a run shorter than the
        // window): fold again in the next iteration
        // (dense only at t = 0: a series whose sum then stays unchanged is
        // converged by iteration L without being folded again -- except a NaN
        // sum, or a non-positive tolerance, which never converge)
        if (isnan(sum) || !(a.tol > 0.0)) act_flag(a, 1, t + 1, h);
      }
    }
  }
  if (!live && map_iter_skipped(a.unconv, skip_t, a.fixed)) return;
  const int bu = __syncthreads_count(not_conv);
  if (threadIdx.x == 0 && bu) atomicAdd(&a.unconv[t], uint32_t(bu));
}

// ---- active-set sparse passes (t >= 2 vertices, t > L series) ----
// A fixed grid of blocks walks the iteration's work list (the 256-item tiles
// holding a flagged item, appended by act_flag during the previous launch):
// block b takes tiles b, b + G, ...; in a tile, each flagged item is
// evaluated by its own thread.  Few flagged tiles cost a few block
// iterations; all of them (the first EM) cost what the dense pass costs,
// without scheduling a block per tile.
template <int MT, int K>
__device__ __forceinline__ void vertex_active_item(const MapArgs& a,
                                                   const uint8_t* __restrict__ lab_in,
                                                   uint8_t* __restrict__ lab_out,
                                                   double* __restrict__ minE,
                                                   const double* __restrict__ minE_prev, int t,
                                                   uint32_t v) {
  const uint32_t M = MT > 0 ? uint32_t(MT) : a.M;
  int16_t d[K];
  load_i16<K>(a.adj_pk + uint64_t(v) * K, d);
  const uint8_t old = lab_in[v];
  if (!a.cover[v]) {
    lab_out[v] = old;
    return;
  }
  uint8_t nb[K];
  uint32_t deg = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const bool ok = d[k] != INT16_MIN;
    deg += ok;
    nb[k] = ok ? lab_in[v + static_cast<uint32_t>(static_cast<int32_t>(d[k]))] : uint8_t(0xFF);
  }
  double best;
  uint32_t best_l;
  vertex_argmin_packed<MT, K>(a, M, a.mean[v], nb, deg, best, best_l);
  minE[v] = best;
  lab_out[v] = static_cast<uint8_t>(best_l);
  act_mark<K>(a, t, v, d, old, best_l, best, minE_prev[v]);
}

template <int MT, int K>
__device__ __forceinline__ void vertex_list_body(const MapArgs& a,
                                                 const uint8_t* __restrict__ lab_in,
                                                 uint8_t* __restrict__ lab_out,
                                                 double* __restrict__ minE,
                                                 const double* __restrict__ minE_prev, int t,
                                                 uint32_t blk, uint32_t nblk, int skip_t) {
  pdl_wait();
  if (map_iter_skipped(a.unconv, skip_t, a.fixed)) return;  // uniform over the grid
  const uint32_t nt = act_vtiles(a);
  const uint32_t n = act_counts(a, t)[0];
  const uint32_t* list = a.act_vlist + uint64_t(t & 1) * nt;
  uint32_t* tiles = a.act_vtile + uint64_t(t & 1) * nt;
  uint8_t* vcur = act_vflags(a, t);
  for (uint32_t i = blk; i < n; i += nblk) {
    const uint32_t tile = list[i];
    if (threadIdx.x == 0) tiles[tile] = 0;
    const uint32_t v = tile * kVtxThreads + threadIdx.x;
    if (v < a.v_end && vcur[v]) {
      vcur[v] = 0;
      ACT_PROBE(0, t);
      vertex_active_item<MT, K>(a, lab_in, lab_out, minE, minE_prev, t, v);
    }
  }
}

// one flagged series of a sparse pass (t > L); returns 1 when not converged
template <int K>
__device__ __forceinline__ int hood_active_item(const MapArgs& a, const double* __restrict__ minE,
                                                int t, uint32_t h) {
  act_hflags(a, t)[h] = 0;
  ACT_PROBE(1, t);
  const uint32_t base = a.hood_base[h];
  uint32_t u[K / 2];
  load_hood_row<K>(a.hood_pk + uint64_t(h) * K, u);
  double over = 0.0;
  const double* p1o = nullptr;
  if (a.act_lastp[h] != uint8_t(t - 1)) {
    // folded again after converged iterations: every window row since
    // equals its last sum (their ring slots are stale)
    over = a.act_hval[h];
    p1o = &over;
    int row = a.row_p;
    for (int i = 0; i < a.L; ++i) {
      a.hist[uint64_t(row) * a.Hs + h] = over;
      row = row == 0 ? a.ring - 1 : row - 1;
    }
  }
  double sum;
  uint32_t eqn;
  const int nc = hood_eval<K>(a, minE, t, h, base, u, p1o, &sum, &eqn);
  a.act_hval[h] = sum;
  a.act_lastp[h] = static_cast<uint8_t>(t);
  // still open (not converged, or converged on a run shorter than the
  // window): fold again in the next iteration
  if (nc || eqn < uint32_t(a.L)) act_flag(a, 1, t + 1, h);
  return nc;
}

template <int K>
__device__ __forceinline__ void hood_list_body(const MapArgs& a, const double* __restrict__ minE,
                                               int t, uint32_t blk, uint32_t nblk, int skip_t) {
  pdl_wait();
  if (map_iter_skipped(a.unconv, skip_t, a.fixed)) return;  // uniform over the grid
  const uint32_t nt = act_htiles(a);
  const uint32_t n = act_counts(a, t)[1];
  const uint32_t* list = a.act_hlist + uint64_t(t & 1) * nt;
  uint32_t* tiles = a.act_htile + uint64_t(t & 1) * nt;
  const uint8_t* hcur = act_hflags(a, t);
  int cnt = 0;
  for (uint32_t i = blk; i < n; i += nblk) {
    const uint32_t tile = list[i];
    if (threadIdx.x == 0) tiles[tile] = 0;
    const uint32_t h = tile * kHoodThreads + threadIdx.x;
    if (h < a.h_end && hcur[h]) cnt += hood_active_item<K>(a, minE, t, h);
  }
  // unconverged series of this iteration (the early exit, optimize.cpp:59);
  // before the window opens (t < L) no series converges, folded or not
  if (t < a.L) {
    if (blk == 0 && threadIdx.x == 0 && a.h_end > a.h_begin)
      atomicAdd(&a.unconv[t], uint32_t(a.h_end - a.h_begin));
    return;
  }
  const int wsum = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0 && wsum) atomicAdd(&a.unconv[t], uint32_t(wsum));
}

template <int K>
__global__ void __launch_bounds__(kHoodThreads) k_hood_packed(MapArgs a, int t) {
  hood_packed_body<K>(a, a.minE, t, blockIdx.x, t);
}

// One kernel per MAP-iteration boundary: the hood pass of iteration t-1 and
// the vertex pass of iteration t read only what the vertex pass of t-1 wrote
// (its minima and committed labels), so they share a launch -- blocks
// [0, nh) fold hoods, the rest evaluate vertices.  The vertex pass of t runs
// speculatively whenever t-1 runs: if t-1 turns out to be the last
// iteration, the speculative pass only wrote buffers nothing reads any more
// (labels into the buffer t-1 consumed, minima into the other half of the
// double-buffered minima, label counts into the other parity slot).
template <int MT, int KV, int KH, int VP, bool kAct>
__global__ void __launch_bounds__(kVtxThreads, fused_min_blocks(MT, KH, VP, kAct))
    k_map_fused(MapArgs a, const uint8_t* __restrict__ lab_in, uint8_t* __restrict__ lab_out,
                const double* __restrict__ minE_prev, double* __restrict__ minE_cur, int t,
                uint32_t nh, uint32_t nv, ScatterArgs sc) {
  static_assert(kVtxThreads == kHoodThreads, "one block shape for both passes");
  static_assert(kVtxThreads == kTileThreads, "scatter tiles are vertex blocks");
  extern __shared__ uint32_t fused_smem[];
  if (blockIdx.x < nh) {
    if (kAct && t - 1 >= 1)
      hood_list_body<KH>(a, minE_prev, t - 1, blockIdx.x, nh, t - 1);
    else
      hood_packed_body<KH, kAct>(a, minE_prev, t - 1, blockIdx.x, t - 1);
  } else if (blockIdx.x >= nh + nv) {
    // last launch (t = map_max): the M-step's label scatter runs beside the
    // hood pass of the last iteration -- it reads only the committed labels
    // and label counts of the last vertex pass (see executed_iters_known)
    pdl_wait();
    if (!em_skipped(a.unconv))
      label_scatter_small_body<true>(sc.lab_even, sc.lab_odd, a.unconv, a.unconv, t, a.fixed,
                                     sc.R, sc.M, sc.Hs, sc.mean, sc.counts, sc.tiles, sc.layout,
                                     sc.x, blockIdx.x - nh - nv, fused_smem);
  } else if (kAct && t >= 2 && !a.tile_counts) {
    vertex_list_body<MT, KV>(a, lab_in, lab_out, minE_cur, minE_prev, t, blockIdx.x - nh, nv,
                             t > 0 ? t - 1 : 0);
  } else {
    vertex_packed_body<MT, KV, VP, kAct>(a, lab_in, lab_out, minE_cur, t, blockIdx.x - nh,
                                         t > 0 ? t - 1 : 0, minE_prev);
  }
}

// ---- vertex -> series index (active-set MAP) ----
// inv_off[v + 1] = number of series containing v; after the scan, the
// series ids of vertex v are inv_ser[inv_off[v] .. inv_off[v + 1]) (any order:
// the flags they set commute).
__global__ void k_inv_count(const uint32_t* __restrict__ s_off, const uint32_t* __restrict__ h_mem,
                            uint64_t Hs, uint32_t* __restrict__ cnt) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t h = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; h < Hs; h += stride)
    for (uint32_t j = s_off[h]; j < s_off[h + 1]; ++j) atomicAdd(&cnt[h_mem[j]], 1u);
}
__global__ void k_inv_fill(const uint32_t* __restrict__ s_off, const uint32_t* __restrict__ h_mem,
                           uint64_t Hs, uint32_t* __restrict__ cursor, uint32_t* __restrict__ ser) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t h = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; h < Hs; h += stride)
    for (uint32_t j = s_off[h]; j < s_off[h + 1]; ++j)
      ser[atomicAdd(&cursor[h_mem[j]], 1u)] = static_cast<uint32_t>(h);
}

// ---- pack builders ----
// Runs beside k_validate (one host sync for both), so every read is clamped
// to the array bounds: on an invalid CSR the stats are meaningless but safe,
// and prepare() fails on the validation result before using them.  Empty
// hoods do not move any maximum, so the raw hood offsets serve as well as the
// series offsets.
__global__ void k_pack_stats(const uint32_t* __restrict__ g_off, const uint32_t* __restrict__ g_nbr,
                             uint32_t R, uint64_t A, const uint32_t* __restrict__ s_off,
                             const uint32_t* __restrict__ h_mem, uint64_t Hs, uint64_t S,
                             uint32_t* stats) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  uint32_t deg = 0, dist = 0, size = 0, span = 0;
  for (uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < R; v += stride) {
    const uint32_t lo = g_off[v], hi = uint64_t(g_off[v + 1]) < A ? g_off[v + 1] : uint32_t(A);
    if (hi < lo) continue;
    deg = max(deg, hi - lo);
    for (uint32_t i = lo; i < hi; ++i) {
      const uint32_t u = g_nbr[i];
      dist = max(dist, u > v ? uint32_t(u - v) : uint32_t(v - u));
    }
  }
  for (uint64_t h = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; h < Hs; h += stride) {
    const uint32_t lo = s_off[h], hi = uint64_t(s_off[h + 1]) < S ? s_off[h + 1] : uint32_t(S);
    if (hi < lo) continue;
    size = max(size, hi - lo);
    if (hi > lo) {
      // the packed layout stores members as deltas from the first, so it
      // needs them ascending: an out-of-order hood disables it
      bool asc = true;
      for (uint32_t i = lo + 1; i < hi; ++i) asc &= h_mem[i] >= h_mem[i - 1];
      span = max(span, asc ? h_mem[hi - 1] - h_mem[lo] : 0xFFFFFFFFu);
    }
  }
  // one atomic per warp and statistic (not per thread: ~300k same-address
  // atomics cost more than the scan itself)
  deg = __reduce_max_sync(0xffffffffu, deg);
  dist = __reduce_max_sync(0xffffffffu, dist);
  size = __reduce_max_sync(0xffffffffu, size);
  span = __reduce_max_sync(0xffffffffu, span);
  if ((threadIdx.x & 31) == 0) {
    if (deg) atomicMax(stats + 0, deg);
    if (dist) atomicMax(stats + 1, dist);
    if (size) atomicMax(stats + 2, size);
    if (span) atomicMax(stats + 3, span);
  }
}

template <int K>
__global__ void k_pack_adjacency(const uint32_t* __restrict__ g_off,
                                 const uint32_t* __restrict__ g_nbr, uint32_t R,
                                 int16_t* __restrict__ out) {
  const uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= R) return;
  const uint32_t lo = g_off[v], hi = g_off[v + 1];
#pragma unroll
  for (int k = 0; k < K; ++k)
    out[v * K + k] = lo + k < hi ? static_cast<int16_t>(int64_t(g_nbr[lo + k]) - int64_t(v))
                                 : int16_t(INT16_MIN);
}

template <int K>
__global__ void k_pack_hoods(const uint32_t* __restrict__ s_off, const uint32_t* __restrict__ h_mem,
                             uint64_t Hs, uint32_t* __restrict__ base, uint16_t* __restrict__ out) {
  const uint64_t h = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (h >= Hs) return;
  const uint32_t lo = s_off[h], hi = s_off[h + 1];
  const uint32_t b = h_mem[lo];
  base[h] = b;
#pragma unroll
  for (int k = 0; k < K; ++k)
    out[h * K + k] = lo + 1 + k < hi ? static_cast<uint16_t>(h_mem[lo + 1 + k] - b) : uint16_t(0xFFFF);
}

// Packed layouts chosen ON THE DEVICE from the validation / statistics words
// [error bits, empty hoods, deg, dist, size, span] of the same prepare()
// batch -- the rule of choose_packing (capi.cu), so the host's sync finds the
// layouts already built.  Nothing is written when the inputs are invalid or
// (hoods) when empty hoods need the compacted series offsets.
__device__ __forceinline__ int dev_adj_k(const uint32_t* e) {
  if (e[0]) return 0;
  return e[3] <= 32767u ? (e[2] <= 4 ? 4 : (e[2] <= 8 ? 8 : 0)) : 0;
}
__device__ __forceinline__ int dev_hood_k(const uint32_t* e, uint64_t H, int use_k12) {
  if (e[0] || e[1]) return 0;
  if (!(e[5] < 0xFFFFu && H > 0 && H < (uint64_t(1) << 32) - 256)) return 0;
  return e[4] <= 9 ? 8 : (e[4] <= 13 && use_k12 ? 12 : (e[4] <= 17 ? 16 : 0));
}
__global__ void k_pack_adjacency_auto(const uint32_t* __restrict__ g_off,
                                      const uint32_t* __restrict__ g_nbr, uint32_t R,
                                      const uint32_t* e, int16_t* __restrict__ out) {
  const uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= R) return;
  const int K = dev_adj_k(e);
  if (K == 0) return;
  const uint32_t lo = g_off[v], hi = g_off[v + 1];
  for (int k = 0; k < K; ++k)
    out[v * K + k] = lo + k < hi ? static_cast<int16_t>(int64_t(g_nbr[lo + k]) - int64_t(v))
                                 : int16_t(INT16_MIN);
}
__global__ void k_pack_hoods_auto(const uint32_t* __restrict__ h_off,
                                  const uint32_t* __restrict__ h_mem, uint64_t H,
                                  const uint32_t* e, int use_k12, uint32_t* __restrict__ base,
                                  uint16_t* __restrict__ out) {
  const uint64_t h = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (h >= H) return;
  const int K = dev_hood_k(e, H, use_k12);
  if (K == 0) return;
  const uint32_t lo = h_off[h], hi = h_off[h + 1];
  const uint32_t b = h_mem[lo];
  base[h] = b;
  for (int k = 0; k < K; ++k)
    out[h * K + k] = lo + 1 + k < hi ? static_cast<uint16_t>(h_mem[lo + 1 + k] - b) : uint16_t(0xFFFF);
}

}  // namespace

void build_vertex_series(const uint32_t* s_off, const uint32_t* h_mem, uint64_t Hs, uint32_t R,
                         uint64_t S, uint32_t* inv_off, uint32_t* inv_ser, uint32_t* cursor,
                         ScanWorkspace& ws, cudaStream_t s) {
  CK(cudaMemsetAsync(inv_off, 0, (uint64_t(R) + 1) * sizeof(uint32_t), s));
  const unsigned g = std::min<unsigned>(grid_for(Hs ? Hs : 1, 256), 16 * kNumSMs);
  if (Hs) {
    k_inv_count<<<g, 256, 0, s>>>(s_off, h_mem, Hs, inv_off);
    CK_LAUNCH();
  }
  exclusive_scan_u32(inv_off, inv_off, uint64_t(R) + 1, nullptr, ws, s);
  CK(cudaMemcpyAsync(cursor, inv_off, uint64_t(R) * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
  if (Hs) {
    k_inv_fill<<<g, 256, 0, s>>>(s_off, h_mem, Hs, cursor, inv_ser);
    CK_LAUNCH();
  }
  (void)S;
}

void launch_pack_stats(const uint32_t* g_off, const uint32_t* g_nbr, uint32_t R, uint64_t A,
                       const uint32_t* s_off, const uint32_t* h_mem, uint64_t Hs, uint64_t S,
                       uint32_t* stats, cudaStream_t s) {
  const uint64_t work = std::max<uint64_t>(std::max<uint64_t>(R, Hs), 1);
  k_pack_stats<<<std::min<unsigned>(grid_for(work, 256), 8 * kNumSMs), 256, 0, s>>>(
      g_off, g_nbr, R, A, s_off, h_mem, Hs, S, stats);
  CK_LAUNCH();
}

void launch_pack_adjacency(const uint32_t* g_off, const uint32_t* g_nbr, uint32_t R, int k,
                           int16_t* out, cudaStream_t s) {
  if (!R) return;
  if (k == 4)
    k_pack_adjacency<4><<<grid_for(R, 256), 256, 0, s>>>(g_off, g_nbr, R, out);
  else
    k_pack_adjacency<8><<<grid_for(R, 256), 256, 0, s>>>(g_off, g_nbr, R, out);
  CK_LAUNCH();
}

void launch_pack_auto(const uint32_t* g_off, const uint32_t* g_nbr, uint32_t R,
                      const uint32_t* h_off, const uint32_t* h_mem, uint64_t H,
                      const uint32_t* stats6, int use_k12, int16_t* adj_out, uint32_t* hood_base,
                      uint16_t* hood_out, cudaStream_t s) {
  if (R) {
    k_pack_adjacency_auto<<<grid_for(R, 256), 256, 0, s>>>(g_off, g_nbr, R, stats6, adj_out);
    CK_LAUNCH();
  }
  if (H) {
    k_pack_hoods_auto<<<grid_for(H, 256), 256, 0, s>>>(h_off, h_mem, H, stats6, use_k12,
                                                       hood_base, hood_out);
    CK_LAUNCH();
  }
}

void launch_pack_hoods(const uint32_t* s_off, const uint32_t* h_mem, uint64_t Hs, int k,
                       uint32_t* base, uint16_t* out, cudaStream_t s) {
  if (!Hs) return;
  if (k == 8)
    k_pack_hoods<8><<<grid_for(Hs, 256), 256, 0, s>>>(s_off, h_mem, Hs, base, out);
  else if (k == 12)
    k_pack_hoods<12><<<grid_for(Hs, 256), 256, 0, s>>>(s_off, h_mem, Hs, base, out);
  else
    k_pack_hoods<16><<<grid_for(Hs, 256), 256, 0, s>>>(s_off, h_mem, Hs, base, out);
  CK_LAUNCH();
}



void launch_init_labels(uint8_t* lab, uint32_t R, uint32_t M, uint64_t seed, cudaStream_t s) {
  if (!R) return;
  k_init_labels<<<grid_for(R, 256), 256, 0, s>>>(lab, R, M, seed);
  CK_LAUNCH();
}

void launch_u8_to_u32(const uint8_t* in, uint32_t* out, uint64_t n, cudaStream_t s) {
  if (!n) return;
  k_u8_to_u32<<<grid_for(n, 256), 256, 0, s>>>(in, out, n);
  CK_LAUNCH();
}

void launch_validate(const uint32_t* g_off, const uint32_t* g_nbr, uint32_t R, uint64_t A,
                     const uint32_t* h_off, const uint32_t* h_mem, uint64_t H, uint64_t S,
                     uint32_t* err, uint32_t* empty_hoods, cudaStream_t s) {
  const uint64_t work = std::max<uint64_t>({S, A, H, uint64_t(R), 1});
  k_validate<<<std::min<unsigned>(grid_for(work, 256), 8 * kNumSMs), 256, 0, s>>>(
      g_off, g_nbr, R, A, h_off, h_mem, H, S, err, empty_hoods);
  CK_LAUNCH();
}

void launch_cover(const uint32_t* h_mem, uint64_t S, uint8_t* cover, uint32_t R, cudaStream_t s) {
  CK(cudaMemsetAsync(cover, 0, R ? R : 1, s));
  if (!S) return;
  k_cover<<<std::min<unsigned>(grid_for(S, 256), 8 * kNumSMs), 256, 0, s>>>(h_mem, S, cover, R);
  CK_LAUNCH();
}

void launch_series_offsets(const uint32_t* h_off, uint64_t H, uint64_t S, uint32_t* s_off,
                           DevBuf<uint32_t>& tmp, ScanWorkspace& ws, cudaStream_t s) {
  uint32_t* f = tmp.ensure(H + 1);
  if (H) {
    k_nonempty_flags<<<grid_for(H, 256), 256, 0, s>>>(h_off, H, f);
    CK_LAUNCH();
  }
  exclusive_scan_u32(f, f, H, f + H, ws, s);
  k_compact_offsets<<<grid_for(H ? H : 1, 256), 256, 0, s>>>(h_off, H, S, f, s_off);
  CK_LAUNCH();
}

}  // namespace dpmrf_b200

#ifdef DPMRF_PROBE
extern "C" int dpmrf_probe_read_act(unsigned long long* out) {  // [2][64], then zeroed
  if (cudaMemcpyFromSymbol(out, dpmrf_b200::g_act_probe, sizeof(dpmrf_b200::g_act_probe)) != cudaSuccess)
    return 1;
  unsigned long long z[2][64] = {};
  return cudaMemcpyToSymbol(dpmrf_b200::g_act_probe, z, sizeof z) != cudaSuccess;
}
#endif
