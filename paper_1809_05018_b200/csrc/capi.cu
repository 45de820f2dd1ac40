// capi.cu -- the C ABI (include/dpmrf_cuda.h): context, resident inputs and
// the optimize() driver.
//
// Driver shape (proj/src/mrf/optimize.cpp:31-74 re-planned for the device):
//   * the graph and neighborhoods stay resident in HBM across calls, re-laid
//     out once per upload by prepare() (validation + packed rows, one sync);
//   * one fused kernel per MAP-iteration boundary (hood pass of t-1 + vertex
//     pass of t), launched back to back with programmatic dependent launch and
//     NO host synchronization: the early exit of optimize.cpp:59 is evaluated
//     on the device from the previous iteration's unconverged-hood counter;
//   * the M-step, total energy, EM window and the next EM's label terms (a
//     correctly rounded device log) run on the device, one CUDA graph per EM,
//     all EM iterations enqueued at once; the host synchronizes once at the
//     end, checks every device log against the host libm (make_label_terms,
//     model.hpp:57) and reruns with host logs in the (not yet observed) case
//     of a difference -- so the energies stay bit-identical to the reference.
//   * the host-log loop (one sync per EM) remains for kernel timing and the
//     full per-MAP trace.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>

#include "context.cuh"

using namespace dpmrf_b200;

namespace {

thread_local std::string g_last_error;

template <class F>
dpmrf_status guarded(F&& f) {
  try {
    f();
    return DPMRF_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return DPMRF_INTERNAL_ERROR;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return DPMRF_INTERNAL_ERROR;
  } catch (...) {
    g_last_error = "unknown failure";
    return DPMRF_INTERNAL_ERROR;
  }
}

void need(bool cond, dpmrf_status s, const char* msg) {
  if (!cond) fail(s, msg);
}

// validate_config, proj/src/mrf/optimize.cpp:13-23 (num_labels relaxed to
// [1, 255] under DPMRF_RUN_MULTILABEL; labels are u8 in HBM).
void validate_config(const dpmrf_optimizer_config& c, bool multilabel) {
  if (multilabel) {
    if (c.num_labels < 1 || c.num_labels > uint32_t(kMaxLabels))
      fail(DPMRF_INPUT_ERROR, "num_labels must be in [1, 255]");
  } else if (c.num_labels != 2) {
    fail(DPMRF_INPUT_ERROR, "only 2 labels are supported");
  }
  if (c.em_max_iters < 0) fail(DPMRF_INPUT_ERROR, "em_max_iters must be >= 0");
  if (c.map_max_iters < 1) fail(DPMRF_INPUT_ERROR, "map_max_iters must be >= 1");
  if (c.convergence_window < 1) fail(DPMRF_INPUT_ERROR, "convergence_window must be >= 1");
  if (c.convergence_window >= c.map_max_iters)
    fail(DPMRF_INPUT_ERROR, "convergence_window must be < map_max_iters");
  if (!(c.convergence_tol > 0.0)) fail(DPMRF_INPUT_ERROR, "convergence_tol must be > 0");
  if (!(c.beta >= 0.0)) fail(DPMRF_INPUT_ERROR, "beta must be >= 0");
  if (c.map_max_iters > kMaxMapIters) fail(DPMRF_INPUT_ERROR, "map_max_iters too large");
}

double unit_of(uint64_t z) { return static_cast<double>(z >> 11) * 0x1.0p-53; }

// init_random's parameter draws, engine.cpp:33-34 (draws 0..2M-1).
void init_params(uint32_t M, uint64_t seed, double* mu, double* sigma) {
  for (uint32_t l = 0; l < M; ++l) mu[l] = 255.0 * unit_of(splitmix_draw(seed, l));
  for (uint32_t l = 0; l < M; ++l) {
    const double s = 255.0 * unit_of(splitmix_draw(seed, M + l));
    sigma[l] = s < kSigmaFloor ? kSigmaFloor : s;
  }
}

}  // namespace

void dpmrf_b200_set_error(const char* msg) { g_last_error = msg; }

namespace dpmrf_b200 {
void check_config(const dpmrf_optimizer_config& c, bool multilabel) { validate_config(c, multilabel); }
void initial_params(uint32_t M, uint64_t seed, double* mu, double* sigma) {
  init_params(M, seed, mu, sigma);
}
}  // namespace dpmrf_b200

// ---- structure preparation ---------------------------------------------------
// The packed-layout rule (host side; dev_adj_k / dev_hood_k in engine.cu are
// the same rule on the device): neighbor lists of <= 4 / 8 with |u - v| <
// 2^15 pack as int16 deltas; hoods of <= 9 / 13 / 17 ascending members
// spanning < 2^16 pack as u16 deltas from the first (the packed hood pass
// indexes hoods with 32 bits).
void choose_packing(const uint32_t* hs, uint64_t Hs, bool use_k12, int* adj_k, int* hood_k) {
  *adj_k = *hood_k = 0;
  if (hs[1] <= 32767u) *adj_k = hs[0] <= 4 ? 4 : (hs[0] <= 8 ? 8 : 0);
  if (hs[3] < 0xFFFFu && Hs > 0 && Hs < (uint64_t(1) << 32) - 256)
    *hood_k = hs[2] <= 9 ? 8 : (hs[2] <= 13 && use_k12 ? 12 : (hs[2] <= 17 ? 16 : 0));
}

void dpmrf_context::prepare() {
  if (prepared) {
    if (prep_status != DPMRF_OK) fail(prep_status, prep_msg);
    return;
  }
  need(has_graph, DPMRF_INVALID_ARGUMENT, "no region graph uploaded");
  need(has_hoods, DPMRF_INVALID_ARGUMENT, "no neighborhoods uploaded");
  // ONE batch and one host sync: validation, the packing statistics, the
  // cover flags and -- chosen on the device from those statistics -- the
  // packed layouts (buffers sized for the largest K).  Every kernel of the
  // batch clamps or skips what an invalid input would make unsafe; the
  // error bits are checked after the sync, before anything else runs.
  uint32_t* err = prep_err.ensure(6);  // [error bits, empty hoods | deg, dist, size, span]
  CK(cudaMemsetAsync(err, 0, 6 * sizeof(uint32_t), stream));
  launch_validate(g_off.get(), g_nbr.get(), R, A, h_off.get(), h_mem.get(), H, S, err, err + 1,
                  stream);
  const bool pack = use_packed && R > 0;
  const uint64_t Hp_max = (H + 255) / 256 * 256;
  if (pack) {
    launch_pack_stats(g_off.get(), g_nbr.get(), R, A, h_off.get(), h_mem.get(), H, S, err + 2,
                      stream);
    launch_pack_auto(g_off.get(), g_nbr.get(), R, h_off.get(), h_mem.get(), H, err, use_k12 ? 1 : 0,
                     adj_pk.ensure(uint64_t(R) * 8), hood_base.ensure(Hp_max ? Hp_max : 1),
                     hood_pk.ensure((Hp_max ? Hp_max : 1) * 16), stream);
  }
  launch_cover(h_mem.get(), S, cover.ensure(R), R, stream);
  uint32_t h_err[6];
  CK(cudaMemcpyAsync(h_err, err, sizeof h_err, cudaMemcpyDeviceToHost, stream));
  sync();
  prepared = true;
  prep_status = DPMRF_OK;
  if (h_err[0] & 1u) {
    prep_status = DPMRF_OUT_OF_RANGE;
    prep_msg = "gather: index out of range (hood member >= num_vertices)";
  } else if (h_err[0] & 2u) {
    prep_status = DPMRF_OUT_OF_RANGE;
    prep_msg = "region graph neighbor >= num_vertices";
  } else if (h_err[0] & 4u) {
    prep_status = DPMRF_INVALID_ARGUMENT;
    prep_msg = "neighborhood offsets are not a valid CSR";
  } else if (h_err[0] & 8u) {
    prep_status = DPMRF_INVALID_ARGUMENT;
    prep_msg = "region graph offsets are not a valid CSR";
  }
  if (prep_status != DPMRF_OK) fail(prep_status, prep_msg);
  const uint32_t empties = h_err[1];
  Hs = H - empties;
  series_alias = empties == 0;
  if (!series_alias) {
    launch_series_offsets(h_off.get(), H, S, s_off_buf.ensure(Hs + 1), prep_tmp, scan, stream);
  }
  // packed layouts when every neighbor list / hood fits (all grid and brick
  // oversegmentations do); otherwise the kernels read the CSR directly
  adj_k = hood_k = 0;
  if (pack) {
    choose_packing(h_err + 2, Hs, use_k12, &adj_k, &hood_k);
    // (the device built both layouts with this K already -- the hood rows
    //  only when no hood is empty; then they are built from the compacted
    //  series offsets here, rows padded to whole 256-hood tiles)
    if (hood_k && !series_alias) {
      const uint64_t Hp = (Hs + 255) / 256 * 256;
      launch_pack_hoods(s_off_buf.get(), h_mem.get(), Hs, hood_k, hood_base.ensure(Hp),
                        hood_pk.ensure(Hp * hood_k), stream);
    }
  }
  // (no sync: everything that reads these runs later on the same stream)
}

// ---- context -----------------------------------------------------------------
extern "C" dpmrf_status dpmrf_context_create(int device, dpmrf_context** out) {
  return guarded([&] {
    need(out != nullptr, DPMRF_INVALID_ARGUMENT, "out is null");
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    need(device >= 0 && device < n, DPMRF_INVALID_ARGUMENT, "no such CUDA device");
    auto* c = new dpmrf_context;
    c->device = device;
    if (const char* e = std::getenv("DPMRF_NO_GRAPH")) c->use_graphs = e[0] == '0';
    if (const char* e = std::getenv("DPMRF_NO_L2_PERSIST")) c->use_l2_persist = e[0] == '0';
    if (const char* e = std::getenv("DPMRF_NO_PDL")) pdl_enabled() = e[0] == '0';
    if (const char* e = std::getenv("DPMRF_HOST_LOG")) c->use_device_loop = e[0] == '0';
    if (const char* e = std::getenv("DPMRF_CSR")) c->use_packed = e[0] == '0';
    if (const char* e = std::getenv("DPMRF_NO_K12")) c->use_k12 = e[0] == '0';
    if (const char* e = std::getenv("DPMRF_UNFUSED")) c->use_fused = e[0] == '0';
    if (const char* e = std::getenv("DPMRF_CLUSTER_SQ")) c->ms.cluster_sq = e[0] != '0';
    if (const char* e = std::getenv("DPMRF_STREAM")) c->ms.stream = e[0] != '0';
    try {
      CK(cudaSetDevice(device));
      CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      CK(cudaEventCreate(&c->ev_begin));
      CK(cudaEventCreate(&c->ev_end));
      init_log_table();  // (once per device)
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

extern "C" void dpmrf_context_destroy(dpmrf_context* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->trace_stream) cudaStreamSynchronize(ctx->trace_stream);
  for (auto e : ctx->trace_ev) cudaEventDestroy(e);
  if (ctx->trace_stream) cudaStreamDestroy(ctx->trace_stream);
  if (ctx->ev_begin) cudaEventDestroy(ctx->ev_begin);
  if (ctx->ev_end) cudaEventDestroy(ctx->ev_end);
  ctx->drop_graphs();
  cudaStream_t s = ctx->stream;
  delete ctx;
  if (s) cudaStreamDestroy(s);
}

extern "C" const char* dpmrf_last_error(void) { return g_last_error.c_str(); }
extern "C" int dpmrf_abi_version(void) { return DPMRF_ABI_VERSION; }

// ---- resident inputs -----------------------------------------------------------
namespace {

// Asynchronous uploads on the context stream; the caller synchronizes before
// returning (the C ABI is externally synchronous: host buffers may be reused
// as soon as a call returns).
void upload_graph(dpmrf_context* ctx, uint32_t R, const uint32_t* offsets,
                  const uint32_t* neighbors, const double* region_mean) {
  need(offsets != nullptr, DPMRF_INVALID_ARGUMENT, "null argument");
  const uint64_t A = offsets[R];
  need(A == 0 || neighbors, DPMRF_INVALID_ARGUMENT, "neighbors is null");
  need(R == 0 || region_mean, DPMRF_INVALID_ARGUMENT, "region_mean is null");
  CK(cudaMemcpyAsync(ctx->g_off.ensure(uint64_t(R) + 1), offsets, (uint64_t(R) + 1) * 4,
                     cudaMemcpyHostToDevice, ctx->stream));
  if (A)
    CK(cudaMemcpyAsync(ctx->g_nbr.ensure(A), neighbors, A * 4, cudaMemcpyHostToDevice,
                       ctx->stream));
  else
    ctx->g_nbr.ensure(1);
  if (R)
    CK(cudaMemcpyAsync(ctx->g_mean.ensure(R), region_mean, uint64_t(R) * 8,
                       cudaMemcpyHostToDevice, ctx->stream));
  else
    ctx->g_mean.ensure(1);
  ctx->R = R;
  ctx->A = A;
  ctx->has_graph = true;
  ctx->has_sizes = ctx->has_cliques = false;
  ctx->prepared = false;
  ++ctx->generation;
}

void upload_hoods(dpmrf_context* ctx, uint64_t H, const uint32_t* offsets,
                  const uint32_t* members) {
  need(offsets != nullptr, DPMRF_INVALID_ARGUMENT, "null argument");
  const uint64_t S = offsets[H];
  need(S == 0 || members, DPMRF_INVALID_ARGUMENT, "members is null");
  CK(cudaMemcpyAsync(ctx->h_off.ensure(H + 1), offsets, (H + 1) * 4, cudaMemcpyHostToDevice,
                     ctx->stream));
  if (S)
    CK(cudaMemcpyAsync(ctx->h_mem.ensure(S), members, S * 4, cudaMemcpyHostToDevice,
                       ctx->stream));
  else
    ctx->h_mem.ensure(1);
  ctx->h_src.release();  // identity (neighborhoods.cpp:53-55)
  ctx->H = H;
  ctx->S = S;
  ctx->has_hoods = true;
  ctx->prepared = false;
  ++ctx->generation;
}

}  // namespace

extern "C" dpmrf_status dpmrf_set_graph(dpmrf_context* ctx, uint32_t R, const uint32_t* offsets,
                                        const uint32_t* neighbors, const double* region_mean) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(ctx != nullptr, DPMRF_INVALID_ARGUMENT, "null argument");
    ctx->bind();
    upload_graph(ctx, R, offsets, neighbors, region_mean);
    ctx->sync();
  });
}

extern "C" dpmrf_status dpmrf_set_hoods(dpmrf_context* ctx, uint64_t H, const uint32_t* offsets,
                                        const uint32_t* members) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(ctx != nullptr, DPMRF_INVALID_ARGUMENT, "null argument");
    ctx->bind();
    upload_hoods(ctx, H, offsets, members);
    ctx->sync();
  });
}

extern "C" dpmrf_status dpmrf_build_neighborhoods(dpmrf_context* ctx, uint64_t C,
                                                  const uint32_t* c_off, const uint32_t* c_mem,
                                                  uint32_t k, uint64_t* num_slots) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(ctx && c_off, DPMRF_INVALID_ARGUMENT, "null argument");
    if (k != 1) fail(DPMRF_INPUT_ERROR, "only 1-neighborhoods are supported");
    need(ctx->has_graph, DPMRF_INVALID_ARGUMENT, "no region graph uploaded");
    ctx->bind();
    build_neighborhoods_device(ctx, C, c_off, c_mem);
    ctx->has_hoods = true;
    ctx->prepared = false;
    ++ctx->generation;
    if (num_slots) *num_slots = ctx->S;
  });
}

extern "C" dpmrf_status dpmrf_get_hoods(dpmrf_context* ctx, uint64_t* H, uint64_t* S,
                                        uint32_t* offsets, uint32_t* members,
                                        uint32_t* source_clique) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(ctx && ctx->has_hoods, DPMRF_INVALID_ARGUMENT, "no neighborhoods");
    ctx->bind();
    if (H) *H = ctx->H;
    if (S) *S = ctx->S;
    if (offsets)
      CK(cudaMemcpyAsync(offsets, ctx->h_off.get(), (ctx->H + 1) * 4, cudaMemcpyDeviceToHost,
                         ctx->stream));
    if (members && ctx->S)
      CK(cudaMemcpyAsync(members, ctx->h_mem.get(), ctx->S * 4, cudaMemcpyDeviceToHost,
                         ctx->stream));
    ctx->sync();
    if (source_clique)
      for (uint64_t h = 0; h < ctx->H; ++h) source_clique[h] = static_cast<uint32_t>(h);
  });
}

// ---- device structure builders (structure.cu) ------------------------------------
extern "C" dpmrf_status dpmrf_build_region_graph(dpmrf_context* ctx, uint32_t w, uint32_t h,
                                                 const uint8_t* pixels, const uint32_t* region,
                                                 uint32_t R, uint64_t* num_adjacency) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(ctx, DPMRF_INVALID_ARGUMENT, "null argument");
    const uint64_t n = uint64_t(w) * h;
    need(n == 0 || (pixels && region), DPMRF_INVALID_ARGUMENT, "null image or label map");
    if (R == 0) fail(DPMRF_INPUT_ERROR, "region graph: label map not validated");
    ctx->bind();
    cudaStream_t st = ctx->stream;
    uint8_t* px = ctx->img_px.ensure(n);
    uint32_t* reg = ctx->img_reg.ensure(n);
    if (n) {
      CK(cudaMemcpyAsync(px, pixels, n, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(reg, region, n * 4, cudaMemcpyHostToDevice, st));
    }
    // the previous graph (and everything derived from it) is gone from here on
    ctx->has_graph = ctx->has_sizes = ctx->has_cliques = ctx->has_hoods = false;
    ctx->has_image = ctx->has_regions = false;  // (img_px / img_reg now hold these inputs)
    ctx->prepared = false;
    ++ctx->generation;
    build_region_graph_device(ctx, w, h, px, reg, R);
    ctx->has_graph = ctx->has_sizes = true;
    // the uploaded label map stays resident for dpmrf_segment_mask (no truth)
    ctx->img_w = w;
    ctx->img_h = h;
    ctx->img_regions = R;
    ctx->has_regions = true;
    if (num_adjacency) *num_adjacency = ctx->A;
  });
}

extern "C" dpmrf_status dpmrf_build_region_graph_device(dpmrf_context* ctx, uint32_t w,
                                                        uint32_t h, const uint8_t* pixels,
                                                        const uint32_t* region, uint32_t R,
                                                        uint64_t* num_adjacency) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(ctx, DPMRF_INVALID_ARGUMENT, "null argument");
    need(uint64_t(w) * h == 0 || (pixels && region), DPMRF_INVALID_ARGUMENT,
         "null image or label map");
    if (R == 0) fail(DPMRF_INPUT_ERROR, "region graph: label map not validated");
    ctx->bind();
    ctx->has_graph = ctx->has_sizes = ctx->has_cliques = ctx->has_hoods = false;
    ctx->prepared = false;
    ++ctx->generation;
    build_region_graph_device(ctx, w, h, pixels, region, R);
    ctx->has_graph = ctx->has_sizes = true;
    if (num_adjacency) *num_adjacency = ctx->A;
  });
}

extern "C" dpmrf_status dpmrf_make_phantom(dpmrf_context* ctx, const dpmrf_phantom_spec* spec,
                                           uint8_t* truth, uint8_t* image, uint32_t* host_ties) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(ctx && spec, DPMRF_INVALID_ARGUMENT, "null argument");
    ctx->bind();
    ctx->has_image = ctx->has_regions = false;
    const uint32_t ties = make_phantom_device(ctx, *spec);
    ctx->has_image = true;
    const uint64_t n = uint64_t(spec->width) * spec->height;
    if (truth) CK(cudaMemcpyAsync(truth, ctx->img_truth.get(), n, cudaMemcpyDeviceToHost, ctx->stream));
    if (image) CK(cudaMemcpyAsync(image, ctx->img_px.get(), n, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    if (host_ties) *host_ties = ties;
  });
}

extern "C" dpmrf_status dpmrf_validate_label_map(dpmrf_context* ctx, uint32_t width,
                                                 uint32_t height, const uint32_t* region,
                                                 uint32_t* num_regions) {
  return guarded([&] {
    ContextLock lock_(ctx);
    const uint64_t n = uint64_t(width) * height;
    need(num_regions && (n == 0 || region), DPMRF_INVALID_ARGUMENT, "null argument");
    ctx->bind();
    uint32_t* d = ctx->lm_region.ensure(n ? n : 1);
    if (n) CK(cudaMemcpyAsync(d, region, n * 4, cudaMemcpyHostToDevice, ctx->stream));
    *num_regions = validate_label_map_device(ctx, width, height, d);
  });
}

extern "C" dpmrf_status dpmrf_confusion(dpmrf_context* ctx, uint64_t n, const uint8_t* pred,
                                        const uint8_t* truth, uint64_t counts[4]) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(counts && (n == 0 || (pred && truth)), DPMRF_INVALID_ARGUMENT, "null argument");
    ctx->bind();
    uint8_t* a = ctx->eval_a.ensure(n ? n : 1);
    uint8_t* b = ctx->eval_b.ensure(n ? n : 1);
    if (n) {
      CK(cudaMemcpyAsync(a, pred, n, cudaMemcpyHostToDevice, ctx->stream));
      CK(cudaMemcpyAsync(b, truth, n, cudaMemcpyHostToDevice, ctx->stream));
    }
    confusion_device(ctx, a, b, n, counts);
  });
}

extern "C" dpmrf_status dpmrf_segment_mask(dpmrf_context* ctx, uint32_t num_vertices,
                                           const uint32_t* labels, const double* mu,
                                           uint8_t* mask, uint64_t counts[4]) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(labels && mu, DPMRF_INVALID_ARGUMENT, "null argument");
    need(ctx->has_regions, DPMRF_INVALID_ARGUMENT, "no resident label map (dpmrf_oversegment)");
    need(num_vertices == ctx->img_regions, DPMRF_INVALID_ARGUMENT,
         "labels do not match the resident label map's regions");
    need(!counts || ctx->has_image, DPMRF_INVALID_ARGUMENT,
         "no resident phantom truth (dpmrf_make_phantom)");
    ctx->bind();
    const uint64_t n = uint64_t(ctx->img_w) * ctx->img_h;
    uint32_t* d_lab = ctx->eval_labels.ensure(num_vertices ? num_vertices : 1);
    if (num_vertices)
      CK(cudaMemcpyAsync(d_lab, labels, uint64_t(num_vertices) * 4, cudaMemcpyHostToDevice,
                         ctx->stream));
    uint8_t* d_mask = mask ? ctx->eval_a.ensure(n ? n : 1) : nullptr;
    // the darker class (smaller mean) is the pore phase (main.cpp:157)
    const uint32_t pore = mu[0] <= mu[1] ? 0u : 1u;
    uint64_t c[4];
    segment_mask_device(ctx, d_lab, pore, d_mask, counts != nullptr, c);
    if (mask && n) {
      CK(cudaMemcpyAsync(mask, d_mask, n, cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
    }
    if (counts) std::memcpy(counts, c, sizeof c);
  });
}

extern "C" dpmrf_status dpmrf_oversegment(dpmrf_context* ctx, uint32_t block, int32_t brick,
                                          uint32_t* num_regions, uint32_t* region) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(ctx != nullptr, DPMRF_INVALID_ARGUMENT, "null argument");
    need(ctx->has_image, DPMRF_INVALID_ARGUMENT, "no resident image (dpmrf_make_phantom)");
    ctx->bind();
    const uint32_t R = oversegment_device(ctx, block, brick != 0);
    ctx->has_regions = true;
    if (region)
      CK(cudaMemcpyAsync(region, ctx->img_reg.get(), uint64_t(ctx->img_w) * ctx->img_h * 4,
                         cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    if (num_regions) *num_regions = R;
  });
}

extern "C" dpmrf_status dpmrf_build_region_graph_resident(dpmrf_context* ctx,
                                                          uint64_t* num_adjacency) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(ctx != nullptr, DPMRF_INVALID_ARGUMENT, "null argument");
    need(ctx->has_image && ctx->has_regions, DPMRF_INVALID_ARGUMENT,
         "no resident image / region map");
    ctx->bind();
    ctx->has_graph = ctx->has_sizes = ctx->has_cliques = ctx->has_hoods = false;
    ctx->prepared = false;
    ++ctx->generation;
    build_region_graph_device(ctx, ctx->img_w, ctx->img_h, ctx->img_px.get(), ctx->img_reg.get(),
                              ctx->img_regions);
    ctx->has_graph = ctx->has_sizes = true;
    if (num_adjacency) *num_adjacency = ctx->A;
  });
}

extern "C" dpmrf_status dpmrf_get_graph(dpmrf_context* ctx, uint32_t* R, uint64_t* A,
                                        uint32_t* offsets, uint32_t* neighbors, double* mean,
                                        uint32_t* size) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(ctx && ctx->has_graph, DPMRF_INVALID_ARGUMENT, "no region graph");
    need(!size || ctx->has_sizes, DPMRF_INVALID_ARGUMENT,
         "region sizes exist only for a graph built by dpmrf_build_region_graph");
    ctx->bind();
    cudaStream_t st = ctx->stream;
    if (R) *R = ctx->R;
    if (A) *A = ctx->A;
    if (offsets)
      CK(cudaMemcpyAsync(offsets, ctx->g_off.get(), (uint64_t(ctx->R) + 1) * 4,
                         cudaMemcpyDeviceToHost, st));
    if (neighbors && ctx->A)
      CK(cudaMemcpyAsync(neighbors, ctx->g_nbr.get(), ctx->A * 4, cudaMemcpyDeviceToHost, st));
    if (mean && ctx->R)
      CK(cudaMemcpyAsync(mean, ctx->g_mean.get(), uint64_t(ctx->R) * 8, cudaMemcpyDeviceToHost, st));
    if (size && ctx->R)
      CK(cudaMemcpyAsync(size, ctx->g_size.get(), uint64_t(ctx->R) * 4, cudaMemcpyDeviceToHost, st));
    ctx->sync();
  });
}

extern "C" dpmrf_status dpmrf_enumerate_maximal_cliques(dpmrf_context* ctx, uint64_t* C,
                                                        uint64_t* CS) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(ctx && ctx->has_graph, DPMRF_INVALID_ARGUMENT, "no region graph");
    ctx->bind();
    ctx->has_cliques = false;
    enumerate_maximal_cliques_device(ctx);
    ctx->has_cliques = true;
    if (C) *C = ctx->C;
    if (CS) *CS = ctx->CS;
  });
}

extern "C" dpmrf_status dpmrf_get_cliques(dpmrf_context* ctx, uint32_t* offsets,
                                          uint32_t* members) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(ctx && ctx->has_cliques, DPMRF_INVALID_ARGUMENT, "no cliques enumerated");
    ctx->bind();
    if (offsets)
      CK(cudaMemcpyAsync(offsets, ctx->c_off.get(), (ctx->C + 1) * 4, cudaMemcpyDeviceToHost,
                         ctx->stream));
    if (members && ctx->CS)
      CK(cudaMemcpyAsync(members, ctx->c_mem.get(), ctx->CS * 4, cudaMemcpyDeviceToHost,
                         ctx->stream));
    ctx->sync();
  });
}

extern "C" dpmrf_status dpmrf_build_neighborhoods_resident(dpmrf_context* ctx, uint32_t k,
                                                           uint64_t* num_slots) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(ctx, DPMRF_INVALID_ARGUMENT, "null argument");
    if (k != 1) fail(DPMRF_INPUT_ERROR, "only 1-neighborhoods are supported");
    need(ctx->has_graph, DPMRF_INVALID_ARGUMENT, "no region graph uploaded");
    need(ctx->has_cliques, DPMRF_INVALID_ARGUMENT, "no cliques enumerated");
    ctx->bind();
    build_neighborhoods_from(ctx, ctx->C, ctx->c_off.get(), ctx->c_mem.get());
    ctx->has_hoods = true;
    ctx->prepared = false;
    ++ctx->generation;
    if (num_slots) *num_slots = ctx->S;
  });
}

// ---- optimize ------------------------------------------------------------------
namespace {

// One optimize() run.  device_loop = true enqueues every EM iteration back to
// back with the EM bookkeeping and log(sigma) on the device (k_em_epilogue)
// and synchronizes once; it returns false if any device log differs from the
// host libm (the caller then reruns with host logs, device_loop = false,
// which synchronizes once per EM iteration exactly as make_label_terms).
bool run_optimize(dpmrf_context* ctx, const dpmrf_optimizer_config* cfg,
                  const dpmrf_run_options& o, bool device_loop, uint32_t* labels_out,
                  double* mu_out, double* sigma_out) {
  const int fixed = (o.flags & DPMRF_RUN_FIXED_WORK) ? 1 : 0;
  const bool timing = (o.flags & DPMRF_RUN_KERNEL_TIMING) != 0;
  cudaStream_t st = ctx->stream;
  const uint32_t M = cfg->num_labels;
  const uint32_t R = ctx->R;
  const int L = cfg->convergence_window;
  const int map_max = cfg->map_max_iters;
  const int em_max = cfg->em_max_iters;

  ctx->trace.clear();
  ctx->trace_rows = nullptr;
  ctx->trace_rowsf = nullptr;
  ctx->trace_level = o.trace_level;
  ctx->trace_M = M;
  const uint32_t fallbacks = ctx->stats.device_log_fallbacks;
  ctx->stats = dpmrf_run_stats{};
  ctx->stats.device_log_fallbacks = fallbacks;
  ctx->stats.device_loop = device_loop;
  uint64_t launches = 0;

  // init_random (engine.cpp:28-38): params on the host, labels on the device
  std::vector<double> mu(M), sigma(M);
  init_params(M, cfg->rng_seed, mu.data(), sigma.data());
  uint8_t* lab[2] = {ctx->lab[0].ensure(R), ctx->lab[1].ensure(R)};
  CK(cudaEventRecord(ctx->ev_begin, st));
  launch_init_labels(lab[0], R, M, cfg->rng_seed, st);
  launches += R ? 1 : 0;
  int cur = 0;

  if (em_max > 0) {
    ctx->prepare();
    const uint64_t Hs = ctx->Hs;
    MapArgs a{};
    a.g_off = ctx->g_off.get();
    a.g_nbr = ctx->g_nbr.get();
    a.mean = ctx->g_mean.get();
    a.cover = ctx->cover.get();
    a.s_off = ctx->series_alias ? ctx->h_off.get() : ctx->s_off_buf.get();
    a.h_mem = ctx->h_mem.get();
    a.R = R;
    a.Hs = Hs;
    a.v_begin = 0;
    a.v_end = R;
    a.h_begin = 0;
    a.h_end = Hs;
    a.M = M;
    a.beta = cfg->beta;
    a.tol = cfg->convergence_tol;
    const bool full = o.trace_level >= DPMRF_TRACE_FULL;
    a.L = L;
    a.ring = full ? map_max : L + 1;
    const bool fused_req = ctx->use_fused && !(o.flags & DPMRF_RUN_UNFUSED);
    a.fixed = fixed;
    const bool packed = !(o.flags & DPMRF_RUN_CSR);
    a.adj_k = packed ? ctx->adj_k : 0;
    a.adj_pk = ctx->adj_pk.get();
    a.hood_k = packed ? ctx->hood_k : 0;
    a.hood_base = ctx->hood_base.get();
    a.hood_pk = ctx->hood_pk.get();
    const bool fused = fused_req && map_fused_supported(a);
    a.terms = ctx->terms.ensure(3 * M);
    double* minE2 = ctx->minE.ensure(2 * uint64_t(R ? R : 1));
    ctx->pin_in_l2(minE2, uint64_t(R) * sizeof(double) * (fused ? 2 : 1));
    a.minE = minE2;
    a.hist = ctx->hist.ensure(uint64_t(a.ring) * Hs + 2);  // (+2: aligned leaf fetches)
    a.flags = full ? ctx->flags.ensure(uint64_t(map_max) * Hs) : nullptr;
    a.eq = a.hood_k ? ctx->hood_eq.ensure(Hs) : nullptr;  // (packed hood pass only)
    // active-set MAP loop (opt-in extension; include/dpmrf_cuda.h)
    const bool active = (o.flags & DPMRF_RUN_ACTIVE_SET) && fused && !full && Hs > 0 &&
                        device_loop && map_active_supported(a);
    if (active) {
      const uint64_t Rp = (uint64_t(R) + 15) & ~15ull, Hp = (Hs + 15) & ~15ull;  // 16-B rows
      a.act_vflag = ctx->act_vflag.ensure(2 * Rp);
      a.act_hflag = ctx->act_hflag.ensure(2 * Hp);
      a.act_hval = ctx->act_hval.ensure(Hs + 2);  // (+2: aligned leaf fetches in the M-step)
      a.act_lastp = ctx->act_lastp.ensure(Hs);
      if (ctx->inv_gen != ctx->generation) {
        const uint32_t* so = ctx->series_alias ? ctx->h_off.get() : ctx->s_off_buf.get();
        build_vertex_series(so, ctx->h_mem.get(), Hs, R, ctx->S, ctx->inv_off.ensure(uint64_t(R) + 1),
                            ctx->inv_ser.ensure(ctx->S ? ctx->S : 1), ctx->inv_cursor.ensure(R ? R : 1),
                            ctx->scan, st);
        CK(cudaMemsetAsync(a.act_vflag, 0, 2 * Rp, st));  // (padding bytes stay 0)
        CK(cudaMemsetAsync(a.act_hflag, 0, 2 * Hp, st));
        ctx->inv_gen = ctx->generation;
      }
      a.inv_off = ctx->inv_off.get();
      a.inv_ser = ctx->inv_ser.get();
      // work lists of the sparse passes (tile flags zero; re-armed by the passes)
      const uint64_t tv = (uint64_t(R) + 255) / 256, th = (Hs + 255) / 256;
      const bool fresh = !ctx->act_vtile.get() || ctx->act_vtile.cap < 2 * tv ||
                         !ctx->act_htile.get() || ctx->act_htile.cap < 2 * th;
      a.act_vtile = ctx->act_vtile.ensure(2 * tv);
      a.act_htile = ctx->act_htile.ensure(2 * th);
      if (fresh) {
        CK(cudaMemsetAsync(a.act_vtile, 0, 2 * tv * 4, st));
        CK(cudaMemsetAsync(a.act_htile, 0, 2 * th * 4, st));
      }
      a.act_vlist = ctx->act_vlist.ensure(2 * tv);
      a.act_hlist = ctx->act_hlist.ensure(2 * th);
      a.act_stride = map_max + 1;
      const uint64_t ncnt = 2 * uint64_t(std::max(em_max, 1)) * (map_max + 1);
      a.act_cnt = ctx->act_cnt.ensure(ncnt);
      CK(cudaMemsetAsync(a.act_cnt, 0, ncnt * 4, st));
    }
    ctx->stats.active_set = active ? 1 : 0;
    ctx->stats.packed_layout = uint32_t(a.adj_k * 100 + a.hood_k);
    // [em_done, pending_done, em_count, pad | per-MAP-iteration counters]
    uint32_t* state = ctx->unconv.ensure(uint64_t(map_max) + 4);
    a.unconv = state + 4;
    CK(cudaMemsetAsync(state, 0, 4 * sizeof(uint32_t), st));
    mstep_reserve(ctx->ms, R, M, Hs);  // before any capture: no allocation inside a graph
    a.tile_counts = ctx->ms.counts.get();
    a.tiles = label_tiles(R);
    double* params = ctx->params.ensure(2 * M);
    double* em_out = ctx->em_out.ensure(2 + 2 * M);
    double* h_terms = ctx->h_terms.ensure(3 * M);
    double* h_em = ctx->h_em.ensure(2 + 2 * M);
    const uint64_t rec_stride = 3 + 3 * uint64_t(M);
    double* em_rec = ctx->em_rec.ensure(uint64_t(em_max) * rec_stride);
    double* em_hist_d = ctx->em_hist.ensure(uint64_t(em_max));
    double* h_rec = ctx->h_rec.ensure(uint64_t(em_max) * rec_stride + 4);
    double* h_row = nullptr;
    uint8_t* h_flags = nullptr;
    if (a.flags) {
      h_row = ctx->h_row.ensure(uint64_t(map_max) * Hs);
      h_flags = ctx->h_flags.ensure(uint64_t(map_max) * Hs);
    }
    CK(cudaMemcpyAsync(params, mu.data(), M * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(params + M, sigma.data(), M * 8, cudaMemcpyHostToDevice, st));
    EmEpilogueArgs ep{};
    ep.unconv = a.unconv;
    ep.map_max = map_max;
    ep.fixed = fixed;
    ep.L = L;
    ep.tol = cfg->convergence_tol;
    ep.lab0 = lab[0];
    ep.lab1 = lab[1];
    ep.R = R;
    ep.M = M;
    ep.em_out = em_out;
    ep.em_hist = em_hist_d;
    ep.em_rec = em_rec;
    ep.terms = const_cast<double*>(a.terms);
    std::vector<double> em_hist;
    const size_t ev_per_em = timing ? size_t(3 * map_max + 6) : 0;
    for (size_t i = 0; i < ev_per_em; ++i) ctx->event(i);
    // Everything one EM iteration puts on the stream (no host sync inside).
    uint64_t em_kernels = 0;
    bool capturing = false;  // event records become graph nodes only when captured as external
    auto record = [&](size_t i) {
      if (!timing) return;
      if (capturing)
        CK(cudaEventRecordWithFlags(ctx->ev_pool[i], st, cudaEventRecordExternal));
      else
        CK(cudaEventRecord(ctx->ev_pool[i], st));
    };
    // Device loop over the fused path on graphs whose M-step scatter fits
    // the self-scanning kernel: the scatter joins the last fused launch and
    // the EM bookkeeping joins the sq-pass tail -- 3 launches fewer per EM
    // (no k_em_prologue / k_label_scatter_small / k_em_epilogue).
    const bool merged = device_loop && fused && mstep_tail_fusable(R, M);
    ScatterArgs sc{};
    sc.mean = a.mean;
    sc.counts = ctx->ms.counts.get();
    sc.tiles = label_tiles(R);
    sc.R = R;
    sc.M = M;
    sc.Hs = Hs;
    sc.layout = ctx->ms.layout.get();
    sc.x = ctx->ms.x.get();
    if (merged)  // the MAP counters of the first EM (later ones are re-armed by the tail)
      CK(cudaMemsetAsync(a.unconv, 0, map_max * sizeof(uint32_t), st));
    // active set: the first EM iteration (from random labels: nearly every
    // item changes) runs dense, the later ones flag-driven
    bool em_active = active;
    MapArgs a_dense = a;
    a_dense.act_vflag = nullptr;
    auto enqueue_em = [&](int parity) {
      uint64_t k = 0;
      size_t ev = 0;
      const MapArgs& am = em_active ? a : a_dense;
      sc.lab_even = lab[parity];
      sc.lab_odd = lab[parity ^ 1];
      if (merged) {
      } else if (device_loop) {
        launch_em_prologue(a.unconv, map_max, st);
        ++k;
      } else {
        CK(cudaMemcpyAsync(const_cast<double*>(a.terms), h_terms, 3 * M * 8,
                           cudaMemcpyHostToDevice, st));
        CK(cudaMemsetAsync(a.unconv, 0, map_max * sizeof(uint32_t), st));
        if (a.act_cnt)  // (the EM counter stays 0 on the host-log loop)
          CK(cudaMemsetAsync(a.act_cnt, 0, 2 * uint64_t(map_max + 1) * 4, st));
      }
      if (fused) {
        const uint64_t half = R ? R : 1;
        // timing: events around the whole chain of fused launches only, so
        // the PDL overlap between consecutive launches stays in the figure
        for (int t = 0; t <= map_max; ++t) {
          if (t == 0) record(ev++);
          launch_map_fused(am, lab[(parity + t) & 1], lab[(parity + t + 1) & 1],
                           minE2 + uint64_t((t + 1) & 1) * half, minE2 + uint64_t(t & 1) * half,
                           t, map_max, st, merged ? &sc : nullptr);
          k += 1;
        }
        record(ev++);
      } else {
        for (int t = 0; t < map_max; ++t) {
          const uint8_t* lin = lab[(parity + t) & 1];
          uint8_t* lout = lab[(parity + t + 1) & 1];
          record(ev++);
          launch_vertex_argmin(a, lin, lout, t, st);
          record(ev++);
          launch_hood_sums(a, t, st);
          record(ev++);
          k += 2;
        }
      }
      if (a.flags && Hs && !device_loop) {  // host-log full trace: this EM's MAP rows + flags
        CK(cudaMemcpyAsync(h_row, a.hist, uint64_t(map_max) * Hs * 8, cudaMemcpyDeviceToHost,
                           st));
        CK(cudaMemcpyAsync(h_flags, a.flags, uint64_t(map_max) * Hs, cudaMemcpyDeviceToHost,
                           st));
      }
      record(ev++);
      // (active set: the latest sum of every series, not the last ring row)
      launch_mstep(a.mean, R, M, lab[parity], lab[parity ^ 1], em_active ? a.act_hval : a.hist,
                   Hs, em_active ? 1 : a.ring, a.unconv,
                   map_max, fixed, params, em_out, ctx->ms, st, &k, /*counts_ready=*/true,
                   /*scattered=*/merged, merged ? &ep : nullptr);
      record(ev++);
      if (merged) {
      } else if (device_loop) {
        launch_em_epilogue(ep, st);
        ++k;
      } else {
        CK(cudaMemcpyAsync(h_em, em_out, (2 + 2 * M) * 8, cudaMemcpyDeviceToHost, st));
      }
      em_kernels = k;
    };
    // CUDA graphs of one EM iteration, captured once per shape and replayed
    // every EM iteration (one per label-buffer parity on the host-log path;
    // the device loop always restarts from buffer 0).
    const bool use_graph = ctx->use_graphs && !(o.flags & DPMRF_RUN_NO_GRAPH);
    ctx->stats.graphs = use_graph;
    if (use_graph) {
      dpmrf_context::GraphKey key{};
      key.R = R;
      key.Hs = Hs;
      key.M = M;
      key.L = L;
      key.map_max = map_max;
      key.fixed = fixed;
      key.timing = timing;
      key.mode = device_loop + 2 * fused;
      key.trace = o.trace_level;
      key.beta = cfg->beta;
      key.tol = cfg->convergence_tol;
      key.p[0] = lab[0];
      key.p[1] = lab[1];
      key.p[2] = a.minE;
      key.p[3] = a.hist;
      key.p[4] = a.flags;
      key.p[5] = a.unconv;
      key.p[6] = params;
      key.p[7] = h_em;
      key.p[8] = h_row;
      key.p[9] = a.s_off;
      key.p[10] = a.h_mem;
      key.p[11] = a.g_nbr;
      key.p[12] = ctx->ms.x.get();
      key.p[13] = ctx->ms.partials.get();
      key.p[14] = a.terms;
      key.p[15] = h_terms;
      key.p[16] = ctx->ms.counts.get();
      key.p[17] = ctx->ms.tile_base.get();
      key.p[18] = ctx->ms.layout.get();
      key.p[19] = em_rec;
      key.p[20] = h_flags;
      key.p[21] = a.cover;
      key.p[22] = a.g_off;
      key.p[23] = em_out;
      key.p2[0] = em_hist_d;
      key.p2[1] = a.mean;
      key.p2[2] = a.adj_pk;
      key.p2[3] = a.hood_pk;
      key.p2[4] = a.hood_base;
      key.layout = a.adj_k * 100 + a.hood_k + (active ? 100000 : 0);
      key.p2[5] = a.act_vflag;
      key.p2[6] = a.act_hval;
      key.p2[7] = a.act_cnt;  // (the tile / list buffers follow R and Hs)
      if (!ctx->graph_valid || std::memcmp(&key, &ctx->graph_key, sizeof key) != 0) {
        ctx->drop_graphs();
        // (device loop: [0] the EM graph, [1] the dense first EM of an
        //  active-set run; host-log loop: one graph per label parity)
        const int ngraphs = device_loop ? (active ? 2 : 1) : 2;
        for (int parity = 0; parity < ngraphs; ++parity) {
          cudaGraph_t g;
          em_active = active && !(device_loop && parity == 1);
          CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
          capturing = true;
          try {
            enqueue_em(device_loop ? 0 : parity);
          } catch (...) {
            capturing = false;
            cudaStreamEndCapture(st, &g);
            if (g) cudaGraphDestroy(g);
            throw;
          }
          capturing = false;
          CK(cudaStreamEndCapture(st, &g));
          CK(cudaGraphInstantiate(&ctx->graph_exec[parity], g, 0));
          CK(cudaGraphDestroy(g));
        }
        ctx->graph_kernels = em_kernels;
        ctx->graph_key = key;
        ctx->graph_valid = true;
      }
    }
    auto host_terms = [&] {  // make_label_terms (model.hpp:48-60) with the host's std::log
      for (uint32_t l = 0; l < M; ++l) {
        h_terms[l] = mu[l];
        h_terms[M + l] = 2.0 * (sigma[l] * sigma[l]);
        h_terms[2 * M + l] = std::log(sigma[l]);
      }
    };
    if (device_loop) {
      // ---- all EM iterations back to back, one synchronization ----
      host_terms();
      CK(cudaMemcpyAsync(const_cast<double*>(a.terms), h_terms, 3 * M * 8,
                         cudaMemcpyHostToDevice, st));
      // Full trace: after each EM its MAP rows (hood energies + flags) are
      // stashed in HBM (one slice per EM); fixed-work runs stream every
      // slice to the host on a side stream while later EMs compute, runs with
      // early exits copy the rows of the executed iterations after the loop.
      const uint64_t slice = uint64_t(map_max) * Hs;
      const bool stash = a.flags && Hs;
      double* dte = nullptr;
      uint8_t* dtf = nullptr;
      double* hte = nullptr;
      uint8_t* htf = nullptr;
      uint64_t pitch = Hs;
      if (stash) {
        dte = ctx->trace_dev.ensure(uint64_t(em_max) * slice);
        dtf = ctx->trace_devf.ensure(uint64_t(em_max) * slice);
        const uint64_t rows = uint64_t(em_max) * map_max;
        if (ctx->sink_e && ctx->sink_f && ctx->sink_rows >= rows && ctx->sink_stride >= Hs) {
          hte = ctx->sink_e;
          htf = ctx->sink_f;
          pitch = ctx->sink_stride;
        } else {
          hte = ctx->trace_arena.ensure(rows * Hs);
          htf = ctx->trace_arenaf.ensure(rows * Hs);
        }
        if (!ctx->trace_stream)
          CK(cudaStreamCreateWithFlags(&ctx->trace_stream, cudaStreamNonBlocking));
      }
      auto rows_d2h = [&](int e, uint64_t nrows, cudaStream_t cs) {
        if (!nrows) return;
        CK(cudaMemcpy2DAsync(hte + uint64_t(e) * map_max * pitch, pitch * 8, dte + e * slice,
                             Hs * 8, Hs * 8, nrows, cudaMemcpyDeviceToHost, cs));
        CK(cudaMemcpy2DAsync(htf + uint64_t(e) * map_max * pitch, pitch, dtf + e * slice, Hs, Hs,
                             nrows, cudaMemcpyDeviceToHost, cs));
      };
      for (int em = 0; em < em_max; ++em) {
        const bool first_dense = active && em == 0;
        if (use_graph) {
          CK(cudaGraphLaunch(ctx->graph_exec[first_dense ? 1 : 0], st));
        } else {
          em_active = active && !first_dense;
          enqueue_em(0);
        }
        if (stash) {
          CK(cudaMemcpyAsync(dte + em * slice, a.hist, slice * 8, cudaMemcpyDeviceToDevice, st));
          CK(cudaMemcpyAsync(dtf + em * slice, a.flags, slice, cudaMemcpyDeviceToDevice, st));
          if (fixed) {
            cudaEvent_t ev = ctx->trace_event(em);
            CK(cudaEventRecord(ev, st));
            CK(cudaStreamWaitEvent(ctx->trace_stream, ev, 0));
            rows_d2h(em, uint64_t(map_max), ctx->trace_stream);
          }
        }
      }
      CK(cudaMemcpyAsync(h_rec, state, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(h_rec + 4, em_rec, uint64_t(em_max) * rec_stride * 8,
                         cudaMemcpyDeviceToHost, st));
      ctx->sync();
      if (stash && fixed) CK(cudaStreamSynchronize(ctx->trace_stream));
      uint32_t hstate[4];
      std::memcpy(hstate, h_rec, sizeof hstate);
      const int em_count = static_cast<int>(hstate[2]);
      const double* rec = h_rec + 4;
      // every device log(sigma) that fed a later EM iteration must equal glibc's
      for (int e = 0; e + 1 < em_count; ++e)
        for (uint32_t l = 0; l < M; ++l) {
          const double sg = rec[e * rec_stride + 3 + M + l];
          const double dev = rec[e * rec_stride + 3 + 2 * M + l];
          const double host = std::log(sg);
          if (std::memcmp(&dev, &host, sizeof host) != 0) return false;
        }
      launches += uint64_t(em_count) * (use_graph ? ctx->graph_kernels : em_kernels);
      for (int e = 0; e < em_count; ++e) {
        const double* r = rec + e * rec_stride;
        const int T = static_cast<int>(r[1]);
        ctx->stats.map_iters_total += T;
        if (o.trace_level >= DPMRF_TRACE_EM) {
          dpmrf_context::EmRecord er;
          er.map_iters = T;
          er.total = r[0];
          er.converged = r[2] != 0.0;
          er.mu.assign(r + 3, r + 3 + M);
          er.sigma.assign(r + 3 + M, r + 3 + 2 * M);
          if (stash) {
            er.row0 = int64_t(e) * map_max;
            if (!fixed) rows_d2h(e, uint64_t(T), st);
          }
          ctx->trace.push_back(std::move(er));
        }
        if (e == em_count - 1) {
          mu.assign(r + 3, r + 3 + M);
          sigma.assign(r + 3 + M, r + 3 + 2 * M);
        }
      }
      ctx->stats.em_iters = em_count;
      if (stash) {
        ctx->trace_rows = hte;
        ctx->trace_rowsf = htf;
        ctx->trace_stride = pitch;
      }
      cur = 0;
    } else {
      for (int em = 0; em < em_max; ++em) {
        host_terms();
        if (use_graph) {
          CK(cudaGraphLaunch(ctx->graph_exec[cur], st));
          launches += ctx->graph_kernels;
        } else {
          enqueue_em(cur);
          launches += em_kernels;
        }
        ctx->sync();
        if (timing) {
          float ms = 0.f;
          size_t e = 0;
          if (fused) {
            CK(cudaEventElapsedTime(&ms, ctx->ev_pool[0], ctx->ev_pool[1]));
            ctx->stats.map_loop_ms += ms;
            ctx->stats.map_loop_launches += map_max + 1;
            e = 2;
          } else {
            for (int t = 0; t < map_max; ++t, e += 3) {
              CK(cudaEventElapsedTime(&ms, ctx->ev_pool[e], ctx->ev_pool[e + 1]));
              ctx->stats.vertex_kernel_ms += ms;
              CK(cudaEventElapsedTime(&ms, ctx->ev_pool[e + 1], ctx->ev_pool[e + 2]));
              ctx->stats.hood_kernel_ms += ms;
            }
            ctx->stats.vertex_launches += map_max;
            ctx->stats.hood_launches += map_max;
          }
          CK(cudaEventElapsedTime(&ms, ctx->ev_pool[e], ctx->ev_pool[e + 1]));
          ctx->stats.mstep_ms += ms;
        }
        const int T = static_cast<int>(h_em[1]);
        const double total = h_em[0];
        std::memcpy(mu.data(), h_em + 2, M * 8);
        std::memcpy(sigma.data(), h_em + 2 + M, M * 8);
        cur = (cur + T) & 1;
        ctx->stats.map_iters_total += T;
        // EM-level window (optimize.cpp:66-69): history never resets
        em_hist.push_back(total);
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
          dpmrf_context::EmRecord rec;
          rec.map_iters = T;
          rec.total = total;
          rec.converged = conv;
          rec.mu = mu;
          rec.sigma = sigma;
          if (a.flags) {
            rec.hood_energy.resize(T);
            rec.hood_conv.resize(T);
            for (int t = 0; t < T; ++t) {
              rec.hood_energy[t].assign(h_row + uint64_t(t) * Hs, h_row + uint64_t(t + 1) * Hs);
              rec.hood_conv[t].assign(h_flags + uint64_t(t) * Hs, h_flags + uint64_t(t + 1) * Hs);
            }
          }
          ctx->trace.push_back(std::move(rec));
        }
        ctx->stats.em_iters = em + 1;
        if (conv && !fixed) break;
      }
    }
    ctx->stats.series = Hs;
  }
  // labels out (u8 in HBM -> the reference's u32)
  uint32_t* l32 = ctx->labels32.ensure(R);
  launch_u8_to_u32(lab[cur], l32, R, st);
  launches += R ? 1 : 0;
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

namespace {

void optimize_resident(dpmrf_context* ctx, const dpmrf_optimizer_config* cfg,
                       const dpmrf_run_options* opts, uint32_t* labels_out, double* mu_out,
                       double* sigma_out);

}  // namespace

extern "C" dpmrf_status dpmrf_optimize(dpmrf_context* ctx, const dpmrf_optimizer_config* cfg,
                                       const dpmrf_run_options* opts, uint32_t* labels_out,
                                       double* mu_out, double* sigma_out) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(ctx && cfg, DPMRF_INVALID_ARGUMENT, "null argument");
    optimize_resident(ctx, cfg, opts, labels_out, mu_out, sigma_out);
  });
}

extern "C" dpmrf_status dpmrf_optimize_arrays(
    dpmrf_context* ctx, uint32_t R, const uint32_t* g_offsets, const uint32_t* g_neighbors,
    const double* region_mean, uint64_t H, const uint32_t* h_offsets, const uint32_t* h_members,
    const dpmrf_optimizer_config* cfg, const dpmrf_run_options* opts, uint32_t* labels_out,
    double* mu_out, double* sigma_out) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(ctx && cfg, DPMRF_INVALID_ARGUMENT, "null argument");
    ctx->bind();
    upload_graph(ctx, R, g_offsets, g_neighbors, region_mean);
    upload_hoods(ctx, H, h_offsets, h_members);
    // (the copies complete before optimize's first synchronization; the
    // host buffers are not touched after this call returns)
    optimize_resident(ctx, cfg, opts, labels_out, mu_out, sigma_out);
  });
}

namespace {

void optimize_resident(dpmrf_context* ctx, const dpmrf_optimizer_config* cfg,
                       const dpmrf_run_options* opts, uint32_t* labels_out, double* mu_out,
                       double* sigma_out) {
  {
    const dpmrf_run_options o = opts ? *opts : dpmrf_run_options{0, DPMRF_TRACE_FULL};
    validate_config(*cfg, (o.flags & DPMRF_RUN_MULTILABEL) != 0);
    need(ctx->has_graph, DPMRF_INVALID_ARGUMENT, "no region graph uploaded");
    ctx->bind();
    // The device-resident EM loop serves every trace level (the full trace's
    // rows are stashed in HBM per EM, up to kTraceStashBytes); per-kernel
    // timing uses the host-log loop.
    const bool full = o.trace_level >= DPMRF_TRACE_FULL;
    const double stash = full ? double(cfg->em_max_iters) * cfg->map_max_iters * ctx->H * 9.0 : 0;
    const bool device_loop = ctx->use_device_loop && !(o.flags & DPMRF_RUN_HOST_LOG) &&
                             !(o.flags & DPMRF_RUN_KERNEL_TIMING) && stash <= kTraceStashBytes &&
                             cfg->em_max_iters > 0;
    if (device_loop) {
      if (run_optimize(ctx, cfg, o, true, labels_out, mu_out, sigma_out)) return;
      ++ctx->stats.device_log_fallbacks;  // a device log(sigma) differed from glibc's
    }
    run_optimize(ctx, cfg, o, false, labels_out, mu_out, sigma_out);
  }
}

}  // namespace

extern "C" dpmrf_status dpmrf_trace_info(dpmrf_context* ctx, int32_t* em_iters, uint64_t* series) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(ctx != nullptr, DPMRF_INVALID_ARGUMENT, "null context");
    if (em_iters) *em_iters = static_cast<int32_t>(ctx->trace.size());
    if (series) *series = ctx->stats.series;
  });
}

extern "C" dpmrf_status dpmrf_trace_em(dpmrf_context* ctx, int32_t em, int32_t* map_iters,
                                       double* total, uint8_t* converged, double* mu,
                                       double* sigma) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(ctx && em >= 0 && size_t(em) < ctx->trace.size(), DPMRF_OUT_OF_RANGE,
         "no such EM iteration in the trace");
    const auto& r = ctx->trace[em];
    if (map_iters) *map_iters = r.map_iters;
    if (total) *total = r.total;
    if (converged) *converged = r.converged;
    if (mu) std::memcpy(mu, r.mu.data(), r.mu.size() * 8);
    if (sigma) std::memcpy(sigma, r.sigma.data(), r.sigma.size() * 8);
  });
}

extern "C" dpmrf_status dpmrf_set_trace_sink(dpmrf_context* ctx, double* hood_energy,
                                            uint8_t* converged, uint64_t rows,
                                            uint64_t row_stride) {
  return guarded([&] {
    ContextLock lock_(ctx);
    const bool on = hood_energy && converged;
    ctx->sink_e = on ? hood_energy : nullptr;
    ctx->sink_f = on ? converged : nullptr;
    ctx->sink_rows = on ? rows : 0;
    ctx->sink_stride = on ? row_stride : 0;
  });
}

extern "C" dpmrf_status dpmrf_trace_map(dpmrf_context* ctx, int32_t em, int32_t it,
                                        double* hood_energy, uint8_t* converged) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(ctx && em >= 0 && size_t(em) < ctx->trace.size(), DPMRF_OUT_OF_RANGE,
         "no such EM iteration in the trace");
    const auto& r = ctx->trace[em];
    if (r.row0 >= 0 && ctx->trace_rows) {  // device-loop full trace: host rows
      need(it >= 0 && it < r.map_iters, DPMRF_OUT_OF_RANGE, "no such MAP iteration in the trace");
      const uint64_t row = uint64_t(r.row0 + it) * ctx->trace_stride;
      const uint64_t n = ctx->stats.series;
      if (hood_energy) std::memcpy(hood_energy, ctx->trace_rows + row, n * 8);
      if (converged) std::memcpy(converged, ctx->trace_rowsf + row, n);
      return;
    }
    need(it >= 0 && size_t(it) < r.hood_energy.size(), DPMRF_OUT_OF_RANGE,
         "no such MAP iteration in the trace (needs DPMRF_TRACE_FULL)");
    if (hood_energy)
      std::memcpy(hood_energy, r.hood_energy[it].data(), r.hood_energy[it].size() * 8);
    if (converged) std::memcpy(converged, r.hood_conv[it].data(), r.hood_conv[it].size());
  });
}

extern "C" dpmrf_status dpmrf_get_stats(dpmrf_context* ctx, dpmrf_run_stats* out) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(ctx && out, DPMRF_INVALID_ARGUMENT, "null argument");
    *out = ctx->stats;
  });
}

extern "C" dpmrf_status dpmrf_debug_log(dpmrf_context* ctx, uint64_t n, const double* x,
                                        double* out) {
  return guarded([&] {
    ContextLock lock_(ctx);
    need(ctx && (n == 0 || (x && out)), DPMRF_INVALID_ARGUMENT, "null argument");
    ctx->bind();
    double* d = ctx->tmp_f64[0].ensure(2 * n);
    if (n) CK(cudaMemcpyAsync(d, x, n * 8, cudaMemcpyHostToDevice, ctx->stream));
    launch_log_cr(d, d + n, n, ctx->stream);
    if (n) CK(cudaMemcpyAsync(out, d + n, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
  });
}
