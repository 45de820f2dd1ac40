// steps.cu -- the step functions of proj/include/dpmrf/mrf/engine.hpp on the
// device, each behind its C ABI entry point (API parity with the reference's
// step-level interface; optimize() itself uses the fused kernels of
// engine.cu).
#include <cmath>
#include <cstring>
#include <vector>

#include "context.cuh"

using namespace dpmrf_b200;

namespace {

// ---- kernels -----------------------------------------------------------------
__global__ void k_init_labels_u32(uint32_t* lab, uint32_t R, uint32_t M, uint64_t seed) {
  const uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v < R) lab[v] = static_cast<uint32_t>(splitmix_draw(seed, 2ull * M + v) % M);
}

// replicate_by_label, engine.cpp:50-72: e = M*o + l*sz + j.
__global__ void k_replicate(const uint32_t* __restrict__ h_off, uint64_t H, uint32_t M,
                            uint32_t* tl, uint32_t* oi, uint32_t* hid, uint32_t* slot_hood) {
  const uint64_t h = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (h >= H) return;
  const uint64_t o = h_off[h], sz = h_off[h + 1] - o;
  for (uint64_t j = 0; j < sz; ++j) {
    if (slot_hood) slot_hood[o + j] = static_cast<uint32_t>(h);
    if (tl)
      for (uint32_t l = 0; l < M; ++l) {
        const uint64_t e = uint64_t(M) * o + uint64_t(l) * sz + j;
        tl[e] = l;
        oi[e] = static_cast<uint32_t>(o + j);
        hid[e] = static_cast<uint32_t>(h);
      }
  }
}

// discord_counts, engine.cpp:74-86.
__global__ void k_discord(const uint32_t* __restrict__ g_off, const uint32_t* __restrict__ g_nbr,
                          const uint32_t* __restrict__ labels, uint32_t R, uint32_t M,
                          uint32_t* __restrict__ out) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= uint64_t(M) * R) return;
  const uint32_t l = static_cast<uint32_t>(i / R), v = static_cast<uint32_t>(i % R);
  uint32_t c = 0;
  for (uint32_t a = g_off[v]; a < g_off[v + 1]; ++a) c += labels[g_nbr[a]] != l;
  out[i] = c;
}

// compute_energies, engine.cpp:88-113 (gathers bounds-checked -> out_of_range).
__global__ void k_energies(const uint32_t* __restrict__ g_off, const uint32_t* __restrict__ g_nbr,
                           const double* __restrict__ mean, const uint32_t* __restrict__ members,
                           uint64_t S, uint32_t R, const uint32_t* __restrict__ tl,
                           const uint32_t* __restrict__ oi, uint64_t E, uint32_t M,
                           const double* __restrict__ terms, const uint32_t* __restrict__ labels,
                           double beta, double* __restrict__ out, uint32_t* err) {
  const uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const uint32_t s = oi[e];
  if (s >= S) {
    atomicOr(err, 1u);
    return;
  }
  const uint32_t v = members[s];
  const uint32_t l = tl[e];
  if (v >= R || l >= M) {
    atomicOr(err, 1u);
    return;
  }
  uint32_t d = 0;
  for (uint32_t a = g_off[v]; a < g_off[v + 1]; ++a) d += labels[g_nbr[a]] != l;
  out[e] = label_energy(mean[v], terms[l], terms[M + l], terms[2 * M + l], beta, d);
}

// min_label_energies, engine.cpp:115-145.  For runs of at most kFoldLeaf
// replicas the keyed fold is a left fold with the keep-strictly-smaller op,
// i.e. "the FIRST element (in stable order) holding the minimum over the
// non-NaN elements, unless the first element itself is NaN" -- computed
// order-independently with atomics.
__device__ __forceinline__ unsigned long long ordered_key(double x) {
  if (x == 0.0) x = 0.0;  // -0.0 == +0.0 under operator<
  const unsigned long long b = __double_as_longlong(x);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_min_pass1(const uint32_t* __restrict__ oi, const double* __restrict__ en,
                            uint64_t E, uint64_t num_slots, uint32_t* __restrict__ count,
                            unsigned long long* __restrict__ first,
                            unsigned long long* __restrict__ minkey, uint32_t* err) {
  const uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const uint32_t k = oi[e];
  if (k >= num_slots) {
    atomicOr(err, 1u);
    return;
  }
  atomicAdd(&count[k], 1u);
  atomicMin(&first[k], static_cast<unsigned long long>(e));
  const double x = en[e];
  if (!isnan(x)) atomicMin(&minkey[k], ordered_key(x));
}

__global__ void k_min_pass2(const uint32_t* __restrict__ oi, const double* __restrict__ en,
                            uint64_t E, const unsigned long long* __restrict__ minkey,
                            unsigned long long* __restrict__ argfirst) {
  const uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const uint32_t k = oi[e];
  const double x = en[e];
  if (!isnan(x) && ordered_key(x) == minkey[k]) atomicMin(&argfirst[k], static_cast<unsigned long long>(e));
}

__global__ void k_min_pass3(const uint32_t* __restrict__ tl, const double* __restrict__ en,
                            uint64_t num_slots, const uint32_t* __restrict__ count,
                            const unsigned long long* __restrict__ first,
                            const unsigned long long* __restrict__ argfirst,
                            double* __restrict__ out_e, uint32_t* __restrict__ out_l, uint32_t* err) {
  const uint64_t s = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= num_slots) return;
  if (count[s] == 0) {
    out_e[s] = 0.0;
    out_l[s] = 0;
    return;
  }
  if (count[s] > kFoldLeaf) atomicOr(err, 2u);
  const unsigned long long f = first[s];
  const unsigned long long pick = isnan(en[f]) ? f : argfirst[s];
  out_e[s] = en[pick];
  out_l[s] = tl[pick];
}

// neighborhood_energy_sums, engine.cpp:147-152: one fold_range per run of
// equal adjacent keys (kernels.hpp:226-253).
__global__ void k_run_flags(const uint32_t* __restrict__ keys, uint64_t n, uint32_t* flags) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) flags[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
}

__global__ void k_run_starts(const uint32_t* __restrict__ flags, const uint32_t* __restrict__ pos,
                             uint64_t n, uint32_t* __restrict__ starts) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && flags[i]) starts[pos[i]] = static_cast<uint32_t>(i);
}

__global__ void k_run_fold(const double* __restrict__ x, uint64_t n,
                           const uint32_t* __restrict__ starts, const uint32_t* nruns_ptr,
                           double* __restrict__ out) {
  const uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t nruns = *nruns_ptr;
  if (r >= nruns) return;
  const uint64_t lo = starts[r], hi = r + 1 < nruns ? starts[r + 1] : n;
  if (hi - lo <= kFoldLeaf) {
    double acc = x[lo];
    for (uint64_t i = lo + 1; i < hi; ++i) acc = __dadd_rn(acc, x[i]);
    out[r] = acc;
  } else {
    TreeStack<double, AddOp> st;
    for (uint64_t b = lo; b < hi; b += kFoldLeaf) {
      const uint64_t e = b + kFoldLeaf < hi ? b + kFoldLeaf : hi;
      double acc = x[b];
      for (uint64_t i = b + 1; i < e; ++i) acc = __dadd_rn(acc, x[i]);
      st.push(acc, AddOp{});
    }
    out[r] = st.finish(AddOp{});
  }
}

// check_convergence, engine.cpp:154-169.
__global__ void k_window(const double* __restrict__ hist, uint64_t rows, uint64_t series,
                         int window, double tol, uint8_t* __restrict__ out) {
  const uint64_t c = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= series) return;
  const double last = hist[(rows - 1) * series + c];
  uint8_t ok = 1;
  for (int i = 1; i <= window; ++i) {
    const double prev = hist[(rows - 1 - uint64_t(i)) * series + c];
    if (!(fabs(__dsub_rn(last, prev)) < tol)) {
      ok = 0;
      break;
    }
  }
  out[c] = ok;
}

// update_labels, engine.cpp:171-191: first (lowest-hood) slot per vertex.
__global__ void k_first_slot(const uint32_t* __restrict__ members, uint64_t S, uint32_t R,
                             uint32_t* __restrict__ first, uint32_t* err) {
  const uint64_t s = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= S) return;
  const uint32_t v = members[s];
  if (v >= R) {
    atomicOr(err, 1u);
    return;
  }
  atomicMin(&first[v], static_cast<uint32_t>(s));
}

__global__ void k_apply_first(const uint32_t* __restrict__ first, const uint32_t* __restrict__ argmin,
                              const uint32_t* __restrict__ old_l, uint32_t R,
                              uint32_t* __restrict__ out) {
  const uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= R) return;
  const uint32_t f = first[v];
  out[v] = f == 0xFFFFFFFFu ? old_l[v] : argmin[f];
}

template <class T>
T* upload(dpmrf_b200::DevBuf<T>& b, const T* h, uint64_t n, cudaStream_t s) {
  T* d = b.ensure(n);
  if (n) CK(cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
  return d;
}

template <class T>
void download(T* h, const T* d, uint64_t n, cudaStream_t s) {
  if (n) CK(cudaMemcpyAsync(h, d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
}

uint32_t read_err(dpmrf_context* ctx, const uint32_t* d_err) {
  uint32_t e = 0;
  CK(cudaMemcpyAsync(&e, d_err, 4, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  return e;
}

void need(bool c, dpmrf_status s, const char* m) {
  if (!c) fail(s, m);
}

}  // namespace

// The C ABI translates internal errors exactly like capi.cu.
#define STEP_GUARD(...)                                               \
  try {                                                               \
    __VA_ARGS__;                                                          \
    return DPMRF_OK;                                                  \
  } catch (const Error& e) {                                          \
    dpmrf_b200_set_error(e.what());                                   \
    return e.status;                                                  \
  } catch (const std::exception& e) {                                 \
    dpmrf_b200_set_error(e.what());                                   \
    return DPMRF_INTERNAL_ERROR;                                      \
  }

void dpmrf_b200_set_error(const char* msg);

extern "C" dpmrf_status dpmrf_init_random(dpmrf_context* ctx, uint32_t M, uint32_t R,
                                          uint64_t seed, int allow_multilabel, double* mu,
                                          double* sigma, uint32_t* labels) {
  STEP_GUARD({
    ContextLock lock_(ctx);
    need(ctx != nullptr, DPMRF_INVALID_ARGUMENT, "null context");
    if (M != 2 && !(allow_multilabel && M >= 1)) fail(DPMRF_INPUT_ERROR, "only 2 labels are supported");
    ctx->bind();
    for (uint32_t l = 0; l < M; ++l)
      mu[l] = 255.0 * (static_cast<double>(splitmix_draw(seed, l) >> 11) * 0x1.0p-53);
    for (uint32_t l = 0; l < M; ++l) {
      const double s = 255.0 * (static_cast<double>(splitmix_draw(seed, M + l) >> 11) * 0x1.0p-53);
      sigma[l] = s < kSigmaFloor ? kSigmaFloor : s;
    }
    uint32_t* d = ctx->tmp_u32[0].ensure(R);
    if (R) {
      k_init_labels_u32<<<grid_for(R, 256), 256, 0, ctx->stream>>>(d, R, M, seed);
      CK_LAUNCH();
    }
    download(labels, d, R, ctx->stream);
    ctx->sync();
  })
}

extern "C" dpmrf_status dpmrf_replicate_by_label(dpmrf_context* ctx, uint32_t M, uint32_t* tl,
                                                 uint32_t* oi, uint32_t* hid) {
  STEP_GUARD({
    ContextLock lock_(ctx);
    need(ctx && ctx->has_hoods, DPMRF_INVALID_ARGUMENT, "no neighborhoods");
    ctx->bind();
    const uint64_t E = uint64_t(M) * ctx->S;
    uint32_t* a = ctx->tmp_u32[0].ensure(E);
    uint32_t* b = ctx->tmp_u32[1].ensure(E);
    uint32_t* c = ctx->tmp_u32[2].ensure(E);
    if (ctx->H) {
      k_replicate<<<grid_for(ctx->H, 256), 256, 0, ctx->stream>>>(ctx->h_off.get(), ctx->H, M, a,
                                                                  b, c, nullptr);
      CK_LAUNCH();
    }
    download(tl, a, E, ctx->stream);
    download(oi, b, E, ctx->stream);
    download(hid, c, E, ctx->stream);
    ctx->sync();
  })
}

extern "C" dpmrf_status dpmrf_slot_hood_map(dpmrf_context* ctx, uint32_t* slot_hood) {
  STEP_GUARD({
    ContextLock lock_(ctx);
    need(ctx && ctx->has_hoods, DPMRF_INVALID_ARGUMENT, "no neighborhoods");
    ctx->bind();
    uint32_t* a = ctx->tmp_u32[0].ensure(ctx->S);
    if (ctx->H) {
      k_replicate<<<grid_for(ctx->H, 256), 256, 0, ctx->stream>>>(ctx->h_off.get(), ctx->H, 0,
                                                                  nullptr, nullptr, nullptr, a);
      CK_LAUNCH();
    }
    download(slot_hood, a, ctx->S, ctx->stream);
    ctx->sync();
  })
}

extern "C" dpmrf_status dpmrf_discord_counts(dpmrf_context* ctx, const uint32_t* labels,
                                             uint32_t M, uint32_t* discord) {
  STEP_GUARD({
    ContextLock lock_(ctx);
    need(ctx && ctx->has_graph, DPMRF_INVALID_ARGUMENT, "no region graph");
    ctx->bind();
    const uint32_t R = ctx->R;
    const uint32_t* dl = upload(ctx->tmp_u32[0], labels, R, ctx->stream);
    uint32_t* out = ctx->tmp_u32[1].ensure(uint64_t(M) * R);
    if (uint64_t(M) * R) {
      k_discord<<<grid_for(uint64_t(M) * R, 256), 256, 0, ctx->stream>>>(
          ctx->g_off.get(), ctx->g_nbr.get(), dl, R, M, out);
      CK_LAUNCH();
    }
    download(discord, out, uint64_t(M) * R, ctx->stream);
    ctx->sync();
  })
}

extern "C" dpmrf_status dpmrf_compute_energies(dpmrf_context* ctx, uint64_t E,
                                               const uint32_t* tl, const uint32_t* oi,
                                               uint32_t M, const double* mu, const double* sigma,
                                               const uint32_t* labels, double beta,
                                               double* energies) {
  STEP_GUARD({
    ContextLock lock_(ctx);
    need(ctx && ctx->has_graph && ctx->has_hoods, DPMRF_INVALID_ARGUMENT,
         "graph and neighborhoods required");
    ctx->bind();
    cudaStream_t st = ctx->stream;
    std::vector<double> terms(3 * size_t(M));
    for (uint32_t l = 0; l < M; ++l) {  // make_label_terms, model.hpp:48-60
      terms[l] = mu[l];
      terms[M + l] = 2.0 * (sigma[l] * sigma[l]);
      terms[2 * M + l] = std::log(sigma[l]);
    }
    const double* dt = upload(ctx->tmp_f64[0], terms.data(), terms.size(), st);
    const uint32_t* dtl = upload(ctx->tmp_u32[0], tl, E, st);
    const uint32_t* doi = upload(ctx->tmp_u32[1], oi, E, st);
    const uint32_t* dl = upload(ctx->tmp_u32[2], labels, ctx->R, st);
    double* out = ctx->tmp_f64[1].ensure(E);
    uint32_t* err = ctx->prep_err.ensure(2);
    CK(cudaMemsetAsync(err, 0, 4, st));
    if (E) {
      k_energies<<<grid_for(E, 256), 256, 0, st>>>(ctx->g_off.get(), ctx->g_nbr.get(),
                                                    ctx->g_mean.get(), ctx->h_mem.get(), ctx->S,
                                                    ctx->R, dtl, doi, E, M, dt, dl, beta, out, err);
      CK_LAUNCH();
    }
    if (read_err(ctx, err)) fail(DPMRF_OUT_OF_RANGE, "gather: index out of range");
    download(energies, out, E, st);
    ctx->sync();
  })
}

extern "C" dpmrf_status dpmrf_min_label_energies(dpmrf_context* ctx, uint64_t E,
                                                 const uint32_t* tl, const uint32_t* oi,
                                                 const double* energies, uint64_t num_slots,
                                                 double* min_energy, uint32_t* min_label) {
  STEP_GUARD({
    ContextLock lock_(ctx);
    need(ctx != nullptr, DPMRF_INVALID_ARGUMENT, "null context");
    ctx->bind();
    cudaStream_t st = ctx->stream;
    const uint32_t* dtl = upload(ctx->tmp_u32[0], tl, E, st);
    const uint32_t* doi = upload(ctx->tmp_u32[1], oi, E, st);
    const double* den = upload(ctx->tmp_f64[0], energies, E, st);
    uint32_t* count = ctx->tmp_u32[2].ensure(num_slots);
    unsigned long long* first = ctx->tmp_u64[0].ensure(2 * num_slots);
    unsigned long long* minkey = ctx->tmp_u64[1].ensure(num_slots);
    unsigned long long* argfirst = first + num_slots;
    double* oe = ctx->tmp_f64[1].ensure(num_slots);
    uint32_t* ol = ctx->tmp_u32[3].ensure(num_slots);
    uint32_t* err = ctx->prep_err.ensure(2);
    CK(cudaMemsetAsync(err, 0, 4, st));
    CK(cudaMemsetAsync(count, 0, num_slots * 4, st));
    CK(cudaMemsetAsync(first, 0xFF, 2 * num_slots * 8, st));
    CK(cudaMemsetAsync(minkey, 0xFF, num_slots * 8, st));
    if (E) {
      k_min_pass1<<<grid_for(E, 256), 256, 0, st>>>(doi, den, E, num_slots, count, first, minkey,
                                                     err);
      CK_LAUNCH();
    }
    if (read_err(ctx, err)) fail(DPMRF_OUT_OF_RANGE, "scatter: index out of range");
    if (E) {
      k_min_pass2<<<grid_for(E, 256), 256, 0, st>>>(doi, den, E, minkey, argfirst);
      CK_LAUNCH();
    }
    if (num_slots) {
      k_min_pass3<<<grid_for(num_slots, 256), 256, 0, st>>>(dtl, den, num_slots, count, first,
                                                             argfirst, oe, ol, err);
      CK_LAUNCH();
    }
    if (read_err(ctx, err) & 2u)
      fail(DPMRF_INVALID_ARGUMENT, "min_label_energies: more than 1024 replicas of one slot");
    download(min_energy, oe, num_slots, st);
    download(min_label, ol, num_slots, st);
    ctx->sync();
  })
}

extern "C" dpmrf_status dpmrf_neighborhood_energy_sums(dpmrf_context* ctx, uint64_t S,
                                                       const uint32_t* slot_hood,
                                                       const double* mins, double* sums,
                                                       uint64_t* num_sums) {
  STEP_GUARD({
    ContextLock lock_(ctx);
    need(ctx != nullptr, DPMRF_INVALID_ARGUMENT, "null context");
    ctx->bind();
    cudaStream_t st = ctx->stream;
    if (S == 0) {
      if (num_sums) *num_sums = 0;
      return DPMRF_OK;
    }
    const uint32_t* dk = upload(ctx->tmp_u32[0], slot_hood, S, st);
    const double* dx = upload(ctx->tmp_f64[0], mins, S, st);
    uint32_t* flags = ctx->tmp_u32[1].ensure(S);
    uint32_t* pos = ctx->tmp_u32[2].ensure(S + 1);
    uint32_t* starts = ctx->tmp_u32[3].ensure(S);
    double* out = ctx->tmp_f64[1].ensure(S);
    k_run_flags<<<grid_for(S, 256), 256, 0, st>>>(dk, S, flags);
    CK_LAUNCH();
    exclusive_scan_u32(flags, pos, S, pos + S, ctx->scan, st);
    k_run_starts<<<grid_for(S, 256), 256, 0, st>>>(flags, pos, S, starts);
    CK_LAUNCH();
    k_run_fold<<<grid_for(S, 256), 256, 0, st>>>(dx, S, starts, pos + S, out);
    CK_LAUNCH();
    uint32_t nr = 0;
    CK(cudaMemcpyAsync(&nr, pos + S, 4, cudaMemcpyDeviceToHost, st));
    ctx->sync();
    download(sums, out, nr, st);
    ctx->sync();
    if (num_sums) *num_sums = nr;
  })
}

extern "C" dpmrf_status dpmrf_check_convergence(dpmrf_context* ctx, uint64_t rows,
                                                uint64_t series, const double* history,
                                                int32_t window, double tol, uint8_t* flags) {
  STEP_GUARD({
    ContextLock lock_(ctx);
    need(ctx != nullptr, DPMRF_INVALID_ARGUMENT, "null context");
    if (rows == 0 || series == 0) return DPMRF_OK;  // empty history -> {} (engine.cpp:160)
    if (rows < uint64_t(window) + 1) {
      std::memset(flags, 0, series);
      return DPMRF_OK;
    }
    ctx->bind();
    cudaStream_t st = ctx->stream;
    const double* dh = upload(ctx->tmp_f64[0], history, rows * series, st);
    uint8_t* out = ctx->tmp_u8[0].ensure(series);
    k_window<<<grid_for(series, 256), 256, 0, st>>>(dh, rows, series, window, tol, out);
    CK_LAUNCH();
    download(flags, out, series, st);
    ctx->sync();
  })
}

extern "C" dpmrf_status dpmrf_update_labels(dpmrf_context* ctx, const uint32_t* argmin,
                                            uint32_t R, const uint32_t* old_labels,
                                            uint32_t* labels) {
  STEP_GUARD({
    ContextLock lock_(ctx);
    need(ctx && ctx->has_hoods, DPMRF_INVALID_ARGUMENT, "no neighborhoods");
    ctx->bind();
    cudaStream_t st = ctx->stream;
    const uint64_t S = ctx->S;
    if (S == 0) {  // engine.cpp:177
      if (R) std::memcpy(labels, old_labels, uint64_t(R) * 4);
      return DPMRF_OK;
    }
    const uint32_t* da = upload(ctx->tmp_u32[0], argmin, S, st);
    const uint32_t* dold = upload(ctx->tmp_u32[1], old_labels, R, st);
    uint32_t* first = ctx->tmp_u32[2].ensure(R);
    uint32_t* out = ctx->tmp_u32[3].ensure(R);
    uint32_t* err = ctx->prep_err.ensure(2);
    CK(cudaMemsetAsync(err, 0, 4, st));
    CK(cudaMemsetAsync(first, 0xFF, uint64_t(R ? R : 1) * 4, st));
    k_first_slot<<<grid_for(S, 256), 256, 0, st>>>(ctx->h_mem.get(), S, R, first, err);
    CK_LAUNCH();
    if (read_err(ctx, err)) fail(DPMRF_OUT_OF_RANGE, "scatter: index out of range");
    if (R) {
      k_apply_first<<<grid_for(R, 256), 256, 0, st>>>(first, da, dold, R, out);
      CK_LAUNCH();
    }
    download(labels, out, R, st);
    ctx->sync();
  })
}

extern "C" dpmrf_status dpmrf_update_parameters(dpmrf_context* ctx, const uint32_t* labels,
                                                uint32_t M, const double* prev_mu,
                                                const double* prev_sigma, double* mu,
                                                double* sigma) {
  STEP_GUARD({
    ContextLock lock_(ctx);
    need(ctx && ctx->has_graph, DPMRF_INVALID_ARGUMENT, "no region graph");
    need(M >= 1 && M <= uint32_t(kMaxLabels), DPMRF_INVALID_ARGUMENT,
         "update_parameters: num_labels must be in [1, 255]");
    ctx->bind();
    cudaStream_t st = ctx->stream;
    const uint32_t R = ctx->R;
    double* params = ctx->tmp_f64[2].ensure(2 * M);
    CK(cudaMemcpyAsync(params, prev_mu, M * 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(params + M, prev_sigma, M * 8, cudaMemcpyHostToDevice, st));
    const uint32_t* dl = upload(ctx->tmp_u32[0], labels, R, st);
    launch_update_parameters_u32(ctx->g_mean.get(), R, M, dl, params, ctx->ms, ctx->tmp_u8[1], st);
    CK(cudaMemcpyAsync(mu, params, M * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(sigma, params + M, M * 8, cudaMemcpyDeviceToHost, st));
    ctx->sync();
  })
}
