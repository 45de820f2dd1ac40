// engine.cuh -- host launchers of the optimization-phase kernels (internal).
#pragma once

#include "common.cuh"
#include "scan.cuh"

namespace dpmrf_b200 {

// Label terms live in HBM as [mu(M) | two_var(M) | log_sigma(M)], written by
// the host once per EM iteration (make_label_terms, model.hpp:48-60, keeps
// glibc's std::log for log_sigma).

struct MapArgs {
  const uint32_t* g_off;
  const uint32_t* g_nbr;
  const double* mean;
  const uint8_t* cover;
  const uint32_t* s_off;   // series offsets (nonempty hoods), Hs+1
  const uint32_t* h_mem;
  uint32_t R;
  uint64_t Hs;
  uint32_t M;
  double beta;
  double tol;
  int L;         // convergence_window
  int ring;      // rows of the hood-energy ring (L+1, or map_max for the full trace)
  int fixed;     // 1 = no early exit
  // Packed static structure (built once by launch_pack_*; k == 0: CSR only).
  //   adjacency: adj_k (4|8) int16 deltas u - v per vertex, INT16_MIN = none
  //   hoods: hood_base[h] = first (smallest) member, hood_pk[h*hood_k + j] =
  //          member(j+1) - base as u16, 0xFFFF = none (members stay ascending)
  const int16_t* adj_pk;
  int adj_k;
  const uint32_t* hood_base;
  const uint16_t* hood_pk;
  int hood_k;
  // Owned ranges (vertex-range partitioning; [0,R) and [0,Hs) on one GPU).
  // Arrays stay globally indexed; v_begin is a multiple of 256.
  uint32_t v_begin, v_end;
  uint64_t h_begin, h_end;
  const double* terms;
  double* minE;    // R
  double* hist;    // ring x Hs hood energies
  uint8_t* flags;  // map_max x Hs convergence flags (nullptr = not recorded)
  uint8_t* eq;     // Hs equal-run counts of the window test (packed hood pass; nullptr = off)
  uint32_t* unconv;  // per MAP iteration count of unconverged hoods
  uint32_t* tile_counts;  // 2 x tiles x M: label counts per 256-vertex tile, by iteration parity
  uint32_t tiles;
  // Per launch (set by the launchers from the hood iteration th): the ring
  // rows of iterations th and th-1, so no thread evaluates a modulo.
  int row_t, row_p;
  // Active-set MAP loop (DPMRF_RUN_ACTIVE_SET; act_vflag == nullptr: off).
  // An item is re-evaluated only when an input of it changed: a vertex when
  // a neighbor's label (or its own label / minimum, for the double buffers)
  // changed in the previous iteration, a series (nonempty hood) when a
  // member's minimum changed or its window test is still open.  The kernels
  // derive the per-iteration slices from the MAP iteration.
  uint8_t* act_vflag;        // 2 x R: vertex flags by iteration parity
  uint8_t* act_hflag;        // 2 x Hs: series flags by iteration parity
  double* act_hval;          // Hs: latest sum of every series
  uint8_t* act_lastp;        // Hs: MAP iteration a series was last folded in
  const uint32_t* inv_off;   // R + 1: vertex -> series CSR
  const uint32_t* inv_ser;   // S: the series containing each vertex
  // work lists of the sparse passes: 256-item tiles holding a flagged item,
  // appended once per (tile, parity) by whoever flags its first item
  uint32_t* act_vtile;       // 2 x vertex tiles: tile flagged (by parity)
  uint32_t* act_htile;       // 2 x series tiles
  uint32_t* act_vlist;       // 2 x vertex tiles: flagged tile ids (by parity)
  uint32_t* act_hlist;       // 2 x series tiles
  uint32_t* act_cnt;         // per (EM, MAP iteration): [vertex tiles, series tiles] listed
  int act_stride;            // map_max + 1
};

// Number of 256-vertex label tiles (== vertex-kernel blocks).
uint32_t label_tiles(uint32_t R);

// One MAP iteration = energies against the frozen labels + per-vertex argmin
// + label commit (engine.cpp:88-191 fused), then the hood
// sums + window test (engine.cpp:147-169).
void launch_vertex_argmin(const MapArgs& a, const uint8_t* lab_in, uint8_t* lab_out, int t,
                          cudaStream_t s);
void launch_hood_sums(const MapArgs& a, int t, cudaStream_t s);
// Fused MAP-iteration boundary (packed layouts only): launch t runs the hood
// pass of iteration t-1 and the vertex pass of iteration t (t = 0..map_max);
// the minima are double-buffered by iteration parity (minE_cur = vertex
// output of t, minE_prev = that of t-1).
bool map_fused_supported(const MapArgs& a);
struct EmEpilogueArgs {
  uint32_t* unconv;
  int map_max;
  int fixed;
  int L;
  double tol;
  uint8_t* lab0;
  const uint8_t* lab1;
  uint32_t R;
  uint32_t M;
  const double* em_out;  // [total, T, mu(M), sigma(M)] of this EM's M-step
  double* em_hist;       // em_max totals
  double* em_rec;        // em_max x (3 + 3M): total, T, conv, mu, sigma, device log(sigma)
  double* terms;         // next EM's [mu | 2 sigma^2 | log sigma]
};

// The M-step's stable grouping of region means by label, run by the extra
// blocks of the last fused MAP launch (t = map_max) on graphs whose label
// tiles fit the self-scanning scatter (mstep_tail_fusable).
struct ScatterArgs {
  const double* mean;
  const uint8_t* lab_even;
  const uint8_t* lab_odd;
  const uint32_t* counts;  // 2 x tiles x M (by MAP-iteration parity)
  uint32_t tiles;
  uint32_t R;
  uint32_t M;
  uint64_t Hs;
  uint32_t* layout;
  double* x;
};
bool mstep_tail_fusable(uint32_t R, uint32_t M);
bool map_active_supported(const MapArgs& a);
struct ScanWorkspace;
// vertex -> series CSR (inv_off R+1, inv_ser S) for the active-set MAP loop
void build_vertex_series(const uint32_t* s_off, const uint32_t* h_mem, uint64_t Hs, uint32_t R,
                         uint64_t S, uint32_t* inv_off, uint32_t* inv_ser, uint32_t* cursor,
                         ScanWorkspace& ws, cudaStream_t s);

void launch_map_fused(const MapArgs& a, const uint8_t* lab_in, uint8_t* lab_out,
                      const double* minE_prev, double* minE_cur, int t, int map_max,
                      cudaStream_t s, const ScatterArgs* sc = nullptr);
struct MStepBuffers {
  DevBuf<uint32_t> counts;       // 2 x tiles x M label counts (slot = MAP iteration parity)
  DevBuf<uint32_t> tile_base;    // tiles x M
  DevBuf<uint32_t> layout;       // n[M] | label_start[M+1] | leaf_start[M+2]
  DevBuf<double> x;              // R values grouped by label (stable)
  DevBuf<double> partials;       // leaf partials of all series (sum pass)
  DevBuf<double> sq_partials;    // leaf partials of the label series (sq pass)
  DevBuf<uint32_t> done;         // last-block tickets of the two leaf-fold kernels
  DevBuf<uint32_t> chunk_sum;    // per-1024-tile-chunk label counts (large graphs)
  DevBuf<uint32_t> err;
  DevBuf<double> em_scratch;
  DevBuf<double> roots;          // chunk roots of the sum | sq passes (many-leaf graphs)
  DevBuf<uint32_t> tickets;      // per-chunk leaf tickets of both passes
  DevBuf<uint32_t> stream_cnt;   // k_mstep_stream's grid barrier / series / block counters
  bool stream = true;            // many-leaf graphs: one persistent streaming fold (DPMRF_STREAM=0: two passes)
  bool cluster_sq = true;  // small graphs: sq pass + EM tail as one cluster (DPMRF_CLUSTER_SQ=0: off)
};

// update_parameters (engine.cpp:193-223) over the labels left by the last
// executed MAP iteration, plus the EM total energy (optimize.cpp:64-65) over
// that iteration's hood-energy row.  params (2M, device) is updated in
// place; em_out receives [total, map_iters, mu(M), sigma(M)].
void launch_mstep(const double* mean, uint32_t R, uint32_t M, const uint8_t* lab_even,
                  const uint8_t* lab_odd, const double* hist, uint64_t Hs, int ring,
                  const uint32_t* unconv, int map_max, int fixed, double* params, double* em_out,
                  MStepBuffers& mb, cudaStream_t s, uint64_t* launches,
                  bool counts_ready = true, bool scattered = false,
                  const EmEpilogueArgs* ep = nullptr, const double* hood_parts = nullptr);
// Partitioned optimize (distributed M-step, partition.cu): the pairwise trees
// in one block over the gathered label-series partials (mb.partials, global
// leaf order) and the hood-series partials.
void launch_fold_trees(bool sq, uint32_t M, uint64_t Hs, const uint32_t* unconv, int map_max,
                       int fixed, double* params, double* em_out, MStepBuffers& mb,
                       const double* hood_parts, cudaStream_t s);
// Partitioned optimize: fold this rank's leaves [hb/1024, ceil(he/1024)) of
// the last executed hood-energy row into out (hood_parts of launch_mstep).
void launch_row_leaves(const double* hist, int ring, uint64_t Hs, const uint32_t* unconv,
                       int map_max, int fixed, uint64_t hb, uint64_t he, double* out,
                       cudaStream_t s);

// Device-resident EM loop (see engine.cu).  unconv points 4 words into its
// allocation: [em_done, pending_done, em_count, pad | unconv[map_max]].

void launch_em_prologue(uint32_t* unconv, int map_max, cudaStream_t s);
void launch_em_epilogue(const EmEpilogueArgs& a, cudaStream_t s);
// log_cr over n values (diagnostics / tests of the device log).
void launch_log_cr(const double* x, double* out, uint64_t n, cudaStream_t s);
// Builds the per-device table of the EM loop's device log once (blocking).
void init_log_table();

// Allocates every M-step buffer up front (required before stream capture).
void mstep_reserve(MStepBuffers& mb, uint32_t R, uint32_t M, uint64_t Hs);

// Standalone update_parameters over caller labels (u32, validated < M).
void launch_update_parameters_u32(const double* mean, uint32_t R, uint32_t M,
                                  const uint32_t* labels, double* params, MStepBuffers& mb,
                                  DevBuf<uint8_t>& lab_tmp, cudaStream_t s);

void launch_init_labels(uint8_t* lab, uint32_t R, uint32_t M, uint64_t seed, cudaStream_t s);
void launch_u8_to_u32(const uint8_t* in, uint32_t* out, uint64_t n, cudaStream_t s);

// Structure preparation (once per graph/hoods pair).
// err bits: 1 = member out of range, 2 = neighbor out of range,
//           4 = hood offsets malformed, 8 = graph offsets malformed
void launch_validate(const uint32_t* g_off, const uint32_t* g_nbr, uint32_t R, uint64_t A,
                     const uint32_t* h_off, const uint32_t* h_mem, uint64_t H, uint64_t S,
                     uint32_t* err, uint32_t* empty_hoods, cudaStream_t s);
void launch_cover(const uint32_t* h_mem, uint64_t S, uint8_t* cover, uint32_t R, cudaStream_t s);
// Packing: stats[0] = max degree, [1] = max |u - v|, [2] = max hood size,
// [3] = max (last - first member) over the series hoods.
void launch_pack_stats(const uint32_t* g_off, const uint32_t* g_nbr, uint32_t R, uint64_t A,
                       const uint32_t* s_off, const uint32_t* h_mem, uint64_t Hs, uint64_t S,
                       uint32_t* stats, cudaStream_t s);
void launch_pack_adjacency(const uint32_t* g_off, const uint32_t* g_nbr, uint32_t R, int k,
                           int16_t* out, cudaStream_t s);
// the packed layouts with K chosen on the device from prepare()'s statistics
// words (as choose_packing); buffers sized for the largest K (8 / 16)
void launch_pack_auto(const uint32_t* g_off, const uint32_t* g_nbr, uint32_t R,
                      const uint32_t* h_off, const uint32_t* h_mem, uint64_t H,
                      const uint32_t* stats6, int use_k12, int16_t* adj_out, uint32_t* hood_base,
                      uint16_t* hood_out, cudaStream_t s);
void launch_pack_hoods(const uint32_t* s_off, const uint32_t* h_mem, uint64_t Hs, int k,
                       uint32_t* base, uint16_t* out, cudaStream_t s);
// Offsets of the nonempty hoods (the runs reduce_by_key sees, engine.cpp:150).
void launch_series_offsets(const uint32_t* h_off, uint64_t H, uint64_t S, uint32_t* s_off,
                           DevBuf<uint32_t>& tmp, ScanWorkspace& ws, cudaStream_t s);

}  // namespace dpmrf_b200
