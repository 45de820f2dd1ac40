// context.cuh -- the opaque dpmrf_context behind the C ABI (internal).
#pragma once

#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "engine.cuh"

struct dpmrf_context {
  int device = 0;
  cudaStream_t stream = nullptr;

  // ---- resident region graph (RegionGraph, region_graph.hpp:14-25) ----
  bool has_graph = false;
  uint32_t R = 0;
  uint64_t A = 0;
  dpmrf_b200::DevBuf<uint32_t> g_off, g_nbr;
  dpmrf_b200::DevBuf<double> g_mean;

  // region_size (region_graph.hpp:23): known only when the graph was built
  // on the device (dpmrf_build_region_graph); dpmrf_set_graph carries none.
  bool has_sizes = false;
  dpmrf_b200::DevBuf<uint32_t> g_size;

  // ---- device structure builders (structure.cu) ----
  // input image / label map of dpmrf_build_region_graph, and the resident
  // maximal cliques (CliqueSet, cliques.hpp:14-22) of the current graph
  bool has_cliques = false;
  uint64_t C = 0, CS = 0;
  dpmrf_b200::DevBuf<uint32_t> c_off, c_mem;
  dpmrf_b200::DevBuf<uint8_t> img_px, img_truth;
  dpmrf_b200::DevBuf<uint32_t> img_reg;
  dpmrf_b200::DevBuf<uint64_t> eval_counts;     // {tp, tn, fp, fn}
  dpmrf_b200::DevBuf<uint8_t> eval_a, eval_b;   // uploaded masks / the written-back mask
  dpmrf_b200::DevBuf<uint32_t> eval_labels;
  // validate_label_map scratch (labelmap.cu)
  dpmrf_b200::DevBuf<uint32_t> lm_parent, lm_state, lm_first, lm_region;
  dpmrf_b200::DevBuf<uint8_t> lm_used;
  uint32_t img_w = 0, img_h = 0, img_regions = 0;  // resident image / region map (synth.cu)
  bool has_image = false, has_regions = false;
  dpmrf_b200::HostBuf<unsigned long long> h_syn;
  dpmrf_b200::DevBuf<uint32_t> st_u32[6];
  dpmrf_b200::DevBuf<unsigned long long> st_u64[3];
  dpmrf_b200::DevBuf<uint32_t> cl_tmp[5];               // frontier x2, counts, flags, positions
  std::vector<std::unique_ptr<dpmrf_b200::DevBuf<uint32_t>>> cl_level;  // maximal cliques per level

  // ---- resident neighborhoods (NeighborhoodSet, neighborhoods.hpp:15-23) ----
  bool has_hoods = false;
  uint64_t H = 0, S = 0;
  dpmrf_b200::DevBuf<uint32_t> h_off, h_mem, h_src;

  // ---- derived per (graph, hoods) pair, built lazily on the device ----
  bool prepared = false;
  uint64_t generation = 0;         // bumped whenever the graph or hoods change
  dpmrf_status prep_status = DPMRF_OK;
  std::string prep_msg;
  uint64_t Hs = 0;                 // nonempty hoods = reduce_by_key runs
  bool series_alias = true;        // s_off == h_off (no empty hoods)
  dpmrf_b200::DevBuf<uint32_t> s_off_buf, prep_tmp, prep_err;
  dpmrf_b200::DevBuf<uint8_t> cover;  // vertex appears in >= 1 hood

  // ---- optimization buffers ----
  dpmrf_b200::DevBuf<uint8_t> lab[2];
  dpmrf_b200::DevBuf<double> minE, hist, terms, params, em_out;
  dpmrf_b200::DevBuf<uint8_t> flags, hood_eq;
  // active-set MAP loop (DPMRF_RUN_ACTIVE_SET): flags, latest series sums,
  // last-folded iterations, and the vertex -> series index (per generation)
  dpmrf_b200::DevBuf<uint8_t> act_vflag, act_hflag, act_lastp;
  dpmrf_b200::DevBuf<double> act_hval;
  dpmrf_b200::DevBuf<uint32_t> inv_off, inv_ser, inv_cursor;
  dpmrf_b200::DevBuf<uint32_t> act_vtile, act_htile, act_vlist, act_hlist, act_cnt;
  uint64_t inv_gen = ~0ull;
  dpmrf_b200::DevBuf<uint32_t> unconv, labels32;
  dpmrf_b200::MStepBuffers ms;
  dpmrf_b200::ScanWorkspace scan;
  dpmrf_b200::HostBuf<double> h_terms, h_em, h_row;
  dpmrf_b200::HostBuf<uint8_t> h_flags;

  // ---- step-API / hood-build scratch ----
  dpmrf_b200::DevBuf<uint32_t> tmp_u32[6];
  dpmrf_b200::DevBuf<double> tmp_f64[3];
  dpmrf_b200::DevBuf<uint8_t> tmp_u8[2];
  dpmrf_b200::DevBuf<unsigned long long> tmp_u64[2];

  // ---- trace of the last optimize (OptimizeResult.trace, engine.hpp:82-99) ----
  struct EmRecord {
    int32_t map_iters = 0;
    double total = 0.0;
    uint8_t converged = 0;
    std::vector<double> mu, sigma;
    std::vector<std::vector<double>> hood_energy;  // FULL trace only
    std::vector<std::vector<uint8_t>> hood_conv;
    int64_t row0 = -1;  // device-loop full trace: first host row (trace_rows)
  };
  std::vector<EmRecord> trace;
  // Full trace of the device-resident loop: every EM's MAP rows stashed in
  // HBM (trace_dev*), streamed by DMA on trace_stream into the caller's sink
  // or the library's pinned arena; EmRecord::row0 indexes those host rows.
  dpmrf_b200::DevBuf<double> trace_dev;
  dpmrf_b200::DevBuf<uint8_t> trace_devf;
  dpmrf_b200::HostBuf<double> trace_arena;
  dpmrf_b200::HostBuf<uint8_t> trace_arenaf;
  double* sink_e = nullptr;
  uint8_t* sink_f = nullptr;
  uint64_t sink_rows = 0, sink_stride = 0;
  const double* trace_rows = nullptr;    // host rows of the last run (sink or arena)
  const uint8_t* trace_rowsf = nullptr;
  uint64_t trace_stride = 0;
  cudaStream_t trace_stream = nullptr;
  std::vector<cudaEvent_t> trace_ev;
  cudaEvent_t trace_event(size_t i) {
    while (trace_ev.size() <= i) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      trace_ev.push_back(e);
    }
    return trace_ev[i];
  }
  int32_t trace_level = DPMRF_TRACE_NONE;
  uint32_t trace_M = 0;
  dpmrf_run_stats stats{};
  std::vector<cudaEvent_t> ev_pool;
  cudaEvent_t ev_begin = nullptr, ev_end = nullptr;

  cudaEvent_t event(size_t i) {
    while (ev_pool.size() <= i) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      ev_pool.push_back(e);
    }
    return ev_pool[i];
  }
  // ---- CUDA graphs of one EM iteration (one per label-buffer parity) ----
  struct GraphKey {
    uint64_t R, Hs;
    uint32_t M;
    int32_t L, map_max, fixed, timing, trace, mode;
    double beta, tol;
    const void* p[24];
    const void* p2[8];
    int32_t layout;
  };
  bool use_device_loop = true;  // EM iterations back to back on the device (DPMRF_HOST_LOG=1 off)
  dpmrf_b200::DevBuf<double> em_rec, em_hist;
  dpmrf_b200::HostBuf<double> h_rec;
  bool use_graphs = true;
  // hood pass of t-1 + vertex pass of t in one launch (packed layouts)
  bool use_fused = true;
  bool graph_valid = false;
  GraphKey graph_key{};
  cudaGraphExec_t graph_exec[2] = {nullptr, nullptr};
  uint64_t graph_kernels = 0;
  void drop_graphs() {
    for (auto& g : graph_exec)
      if (g) {
        cudaGraphExecDestroy(g);
        g = nullptr;
      }
    graph_valid = false;
  }

  // L2 residency for the per-vertex minima: the hood pass gathers them while
  // streaming ~8x more member bytes, which would otherwise evict them (at
  // 16384^2 the L2 hit rate of those gathers was 19%).  One persisting
  // access-policy window on the context stream (captured into graph nodes).
  const void* l2_window = nullptr;
  uint64_t l2_bytes = 0;
  bool use_l2_persist = true;
  void pin_in_l2(const void* base, uint64_t bytes) {
    if (!use_l2_persist || bytes < (8ull << 20)) return;  // small graphs stay in L2 anyway
    if (base == l2_window && bytes == l2_bytes) return;
    int max_persist = 0, max_window = 0;
    CK(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device));
    CK(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, device));
    if (max_persist <= 0 || max_window <= 0) return;
    const uint64_t win = bytes < uint64_t(max_window) ? bytes : uint64_t(max_window);
    const uint64_t carve = win < uint64_t(max_persist) ? win : uint64_t(max_persist);
    CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve));
    cudaStreamAttrValue attr{};
    attr.accessPolicyWindow.base_ptr = const_cast<void*>(base);
    attr.accessPolicyWindow.num_bytes = win;
    attr.accessPolicyWindow.hitRatio = float(double(carve) / double(win));
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    CK(cudaStreamSetAttribute(stream, cudaStreamAttributeAccessPolicyWindow, &attr));
    l2_window = base;
    l2_bytes = bytes;
  }

  void sync() { CK(cudaStreamSynchronize(stream)); }
  void bind() { CK(cudaSetDevice(device)); }

  // Every C-ABI entry point holds this for its whole call: calls on one
  // context from several host threads serialize (the reference's pool
  // serializes concurrent submissions, proj/src/dpp/backend.cpp:45); the
  // lock is recursive because entry points call each other.
  std::recursive_mutex mu;
  void prepare();  // validate + cover + series offsets + packed layouts (capi.cu)

  // ---- packed static structure (engine.cuh MapArgs::adj_k / hood_k) ----
  bool use_packed = true;
  bool use_k12 = true;  // 12-slot hood rows for <= 13-slot hoods (DPMRF_NO_K12=1: 16)
  int adj_k = 0, hood_k = 0;
  dpmrf_b200::DevBuf<int16_t> adj_pk;
  dpmrf_b200::DevBuf<uint32_t> hood_base;
  dpmrf_b200::DevBuf<uint16_t> hood_pk;
};

namespace dpmrf_b200 {
// Entry-point guard: a null context is DPMRF_INVALID_ARGUMENT, otherwise the
// context's mutex is held until the call returns.
struct ContextLock {
  std::unique_lock<std::recursive_mutex> lk;
  explicit ContextLock(dpmrf_context* c) {
    if (c == nullptr) fail(DPMRF_INVALID_ARGUMENT, "null context");
    lk = std::unique_lock<std::recursive_mutex>(c->mu);
  }
};
}  // namespace dpmrf_b200


namespace dpmrf_b200 {
// capi.cu
void check_config(const dpmrf_optimizer_config& c, bool multilabel);  // validate_config
void initial_params(uint32_t M, uint64_t seed, double* mu, double* sigma);  // init_random
// hoods.cu
void build_neighborhoods_device(dpmrf_context* ctx, uint64_t C, const uint32_t* c_off_host,
                                const uint32_t* c_mem_host);
void build_neighborhoods_from(dpmrf_context* ctx, uint64_t C, const uint32_t* c_off_dev,
                              const uint32_t* c_mem_dev);
// structure.cu
void build_region_graph_device(dpmrf_context* ctx, uint32_t width, uint32_t height,
                               const uint8_t* pixels_dev, const uint32_t* region_dev, uint32_t R);
void enumerate_maximal_cliques_device(dpmrf_context* ctx);
// synth.cu
uint32_t make_phantom_device(dpmrf_context* ctx, const dpmrf_phantom_spec& spec);
uint32_t oversegment_device(dpmrf_context* ctx, uint32_t block, bool brick);
// Evaluation (synth.cu): confusion of two device u8 masks; the segment
// write-back of device labels over the resident region map (mask: device
// buffer or nullptr), counted against the resident truth when with_truth.
void confusion_device(dpmrf_context* ctx, const uint8_t* pred, const uint8_t* truth, uint64_t n,
                      uint64_t counts[4]);
void segment_mask_device(dpmrf_context* ctx, const uint32_t* labels, uint32_t pore,
                         uint8_t* mask, bool with_truth, uint64_t counts[4]);
// validate_label_map (labelmap.cu) of a device label map: returns num_regions
// or fails with the reference's InputError message.
uint32_t validate_label_map_device(dpmrf_context* ctx, uint32_t width, uint32_t height,
                                   const uint32_t* region);
}  // namespace dpmrf_b200
