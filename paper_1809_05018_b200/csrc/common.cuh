// common.cuh -- shared definitions of the sm_100a DPP-PMRF library.
//
// Arithmetic contract: every floating-point operation that the reference
// evaluates in a pinned order (proj/include/dpmrf/mrf/model.hpp:62-72 and
// the fold topology of proj/include/dpmrf/dpp/kernels.hpp:20-65) is written
// with explicit round-to-nearest intrinsics (__dadd_rn, __dsub_rn, __dmul_rn,
// __ddiv_rn, __dsqrt_rn) so no FMA contraction can change a bit; the library
// is additionally compiled with -fmad=false.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <map>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <tuple>
#include <utility>

#include "../../include/dpmrf_cuda.h"

namespace dpmrf_b200 {

// Internal exception; translated to dpmrf_status at the C ABI boundary.
struct Error : std::runtime_error {
  dpmrf_status status;
  Error(dpmrf_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(dpmrf_status s, const std::string& m) { throw Error(s, m); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    (void)cudaGetLastError();  // clear a non-sticky error so later launch checks stay clean
    char buf[512];
    std::snprintf(buf, sizeof buf, "%s failed at %s:%d: %s", what, file, line,
                  cudaGetErrorString(e));
    throw Error(DPMRF_CUDA_ERROR, buf);
  }
}
#define CK(x) ::dpmrf_b200::cuda_check((x), #x, __FILE__, __LINE__)
#define CK_LAUNCH() ::dpmrf_b200::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

constexpr uint32_t kFoldLeaf = 1024;       // kFoldLeafSize, kernels.hpp:27
constexpr double kSigmaFloor = 1e-3;       // kSigmaFloor, model.hpp:9
constexpr int kMaxLabels = 255;            // labels are stored as u8 in HBM
constexpr int kMaxMapIters = 4096;
constexpr int kNumSMs = 148;
// HBM budget of the full-trace stash of the device-resident EM loop (every
// EM's map_max x H rows of f64 energies + u8 flags); larger runs take the
// host-log loop.
constexpr double kTraceStashBytes = 24.0 * (1ull << 30);

// Growable device buffer (HBM). Contents are not preserved on growth.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  T* ensure(size_t n) {
    if (n == 0) n = 1;
    if (n > cap) {
      release();
      CK(cudaMalloc(&p, n * sizeof(T)));
      cap = n;
    }
    return p;
  }
  T* get() const { return p; }
};

// Growable pinned host buffer.
template <class T>
struct HostBuf {
  T* p = nullptr;
  size_t cap = 0;
  HostBuf() = default;
  HostBuf(const HostBuf&) = delete;
  HostBuf& operator=(const HostBuf&) = delete;
  ~HostBuf() { release(); }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
  T* ensure(size_t n) {
    if (n == 0) n = 1;
    if (n > cap) {
      release();
      CK(cudaMallocHost(&p, n * sizeof(T)));
      cap = n;
    }
    return p;
  }
};

// Opt a kernel into at least `bytes` of dynamic shared memory on the current
// device (the attribute only grows: a kernel launched with several sizes
// keeps the largest); thread-safe.
template <class F>
inline void ensure_dynamic_smem(F* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> set_to;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  const auto key = std::make_pair(reinterpret_cast<const void*>(kernel), dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = set_to.find(key);
  if (it != set_to.end() && it->second >= bytes) return;
  CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
  set_to[key] = bytes;
}

// Programmatic Dependent Launch: a kernel launched this way may be scheduled
// while its stream predecessor is still draining; it must execute pdl_wait()
// before touching anything the predecessor writes (griddepcontrol.wait
// returns once the predecessor has completed and its writes are visible).
inline bool& pdl_enabled() {
  static bool on = true;
  return on;
}

template <class... KArgs, class... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// launch_pdl with a thread-block cluster of `cluster` CTAs along x.
template <typename... KArgs, typename... Args>
inline void launch_pdl_cluster(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                               unsigned cluster, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = cluster;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  CK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// No kernel issues griddepcontrol.launch_dependents: releasing the next grid
// early (its blocks resident and parked in pdl_wait while this grid runs)
// measured 6% SLOWER at 2560^2 (11.9k vs 12.7k EM-it/s) and neutral at
// 16384^2 -- the parked blocks take slots from this grid's tail.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

inline unsigned grid_for(uint64_t n, unsigned block) {
  uint64_t g = (n + block - 1) / block;
  if (g == 0) g = 1;
  return static_cast<unsigned>(g);
}

// ---- device helpers ---------------------------------------------------------

// SplitMix64 finalizer (proj/src/mrf/engine.cpp:15-24); draw k (0-based) of
// the stream seeded with `seed` is mix64(seed + (k+1) * golden).
__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ inline uint64_t splitmix_draw(uint64_t seed, uint64_t k) {
  return mix64(seed + (k + 1) * 0x9E3779B97F4A7C15ull);
}

// label_energy, model.hpp:66-72: sub, mul, div, add, mul, add -- in that order.
__device__ __forceinline__ double label_energy(double x, double mu, double two_var,
                                               double log_sigma, double beta, uint32_t discord) {
  const double d = __dsub_rn(x, mu);
  const double q = __ddiv_rn(__dmul_rn(d, d), two_var);
  const double data_term = __dadd_rn(q, log_sigma);
  return __dadd_rn(data_term, __dmul_rn(beta, static_cast<double>(discord)));
}

// Pairwise tree of kernels.hpp:45-51 evaluated as a binary counter: push
// leaf partials in order; equal-sized blocks merge immediately; at the end
// the remaining blocks (sizes = binary digits of the count, decreasing)
// combine right to left.  Identical topology to splitting at bit_floor(n-1).
template <class T, class Op, int kDepth = 40>
struct TreeStack {
  T val[kDepth];
  uint64_t count = 0;
  int top = 0;
  __device__ __forceinline__ void push(T x, Op op) {
    ++count;
    val[top++] = x;
    // merge while the two top blocks have equal size: the lowest set bits
    for (uint64_t c = count; (c & 1u) == 0; c >>= 1) {
      val[top - 2] = op(val[top - 2], val[top - 1]);
      --top;
    }
  }
  __device__ __forceinline__ T finish(Op op) {
    T acc = val[top - 1];
    for (int i = top - 2; i >= 0; --i) acc = op(val[i], acc);
    return acc;
  }
};

struct AddOp {
  __device__ __forceinline__ double operator()(double a, double b) const { return __dadd_rn(a, b); }
};

// ---- correctly rounded natural log (double-double evaluation) ---------------
// make_label_terms takes log(sigma) from the host libm (model.hpp:57).  To run
// EM iterations back to back on the device, log(sigma) is evaluated here to
// ~2^-100 relative accuracy and rounded once, i.e. correctly rounded; glibc's
// log agrees with the correctly rounded value except in rare cases (measured
// ~5e-4 of random inputs), and the host verifies every value after the run
// and falls back to host-evaluated logs when one differs (capi.cu).
struct dd_t {
  double hi, lo;
};
__device__ __forceinline__ dd_t dd_two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  return {s, __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb))};
}
__device__ __forceinline__ dd_t dd_fast_two_sum(double a, double b) {  // |a| >= |b|
  const double s = __dadd_rn(a, b);
  return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd_t dd_add(dd_t a, dd_t b) {
  dd_t s = dd_two_sum(a.hi, b.hi);
  const dd_t t = dd_two_sum(a.lo, b.lo);
  s.lo = __dadd_rn(s.lo, t.hi);
  s = dd_fast_two_sum(s.hi, s.lo);
  s.lo = __dadd_rn(s.lo, t.lo);
  return dd_fast_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd_t dd_mul(dd_t a, dd_t b) {
  const double p = __dmul_rn(a.hi, b.hi);
  double e = __fma_rn(a.hi, b.hi, -p);
  e = __dadd_rn(e, __dadd_rn(__dmul_rn(a.hi, b.lo), __dmul_rn(a.lo, b.hi)));
  return dd_fast_two_sum(p, e);
}
__device__ __forceinline__ dd_t dd_div(dd_t a, dd_t b) {
  const double q1 = __ddiv_rn(a.hi, b.hi);
  dd_t r = dd_add(a, dd_mul({-q1, 0.0}, b));
  const double q2 = __ddiv_rn(r.hi, b.hi);
  r = dd_add(r, dd_mul({-q2, 0.0}, b));
  const double q3 = __ddiv_rn(r.hi, b.hi);
  return dd_add(dd_fast_two_sum(q1, q2), {q3, 0.0});
}
// log x = e ln2 + 2 atanh(f), f = (m-1)/(m+1), m in [1/sqrt2, sqrt2):
// |f| <= 0.1716, f^2 <= 0.0295, 23 series terms reach 2^-110.
// log x as a double-double for positive, finite, normal x.
__device__ inline dd_t log_dd(double x) {
  int e;
  double m = frexp(x, &e);
  if (m < 0.70710678118654752440) {
    m = __dmul_rn(m, 2.0);
    e -= 1;
  }
  const dd_t f = dd_div({__dsub_rn(m, 1.0), 0.0}, dd_two_sum(m, 1.0));
  const dd_t z = dd_mul(f, f);
  // 1/(2k+1) as double-doubles (hi = RN(1/n), lo = RN(1/n - hi))
  constexpr double C[23][2] = {
      {0x1.0000000000000p+0, 0x0.0p+0},
      {0x1.5555555555555p-2, 0x1.5555555555555p-56},
      {0x1.999999999999ap-3, -0x1.999999999999ap-57},
      {0x1.2492492492492p-3, 0x1.2492492492492p-57},
      {0x1.c71c71c71c71cp-4, 0x1.c71c71c71c71cp-58},
      {0x1.745d1745d1746p-4, -0x1.745d1745d1746p-59},
      {0x1.3b13b13b13b14p-4, -0x1.3b13b13b13b14p-58},
      {0x1.1111111111111p-4, 0x1.1111111111111p-60},
      {0x1.e1e1e1e1e1e1ep-5, 0x1.e1e1e1e1e1e1ep-61},
      {0x1.af286bca1af28p-5, 0x1.af286bca1af28p-59},
      {0x1.8618618618618p-5, 0x1.8618618618618p-59},
      {0x1.642c8590b2164p-5, 0x1.642c8590b2164p-60},
      {0x1.47ae147ae147bp-5, -0x1.eb851eb851eb8p-61},
      {0x1.2f684bda12f68p-5, 0x1.2f684bda12f68p-59},
      {0x1.1a7b9611a7b96p-5, 0x1.1a7b9611a7b96p-61},
      {0x1.0842108421084p-5, 0x1.0842108421084p-60},
      {0x1.f07c1f07c1f08p-6, -0x1.f07c1f07c1f08p-61},
      {0x1.d41d41d41d41dp-6, 0x1.0750750750750p-60},
      {0x1.bacf914c1bad0p-6, -0x1.bacf914c1bad0p-60},
      {0x1.a41a41a41a41ap-6, 0x1.0690690690690p-60},
      {0x1.8f9c18f9c18fap-6, -0x1.f3831f3831f38p-61},
      {0x1.7d05f417d05f4p-6, 0x1.7d05f417d05f4p-62},
      {0x1.6c16c16c16c17p-6, -0x1.f49f49f49f49fp-61},
  };
  // Estrin's scheme (all terms positive: no cancellation): depth 5 instead
  // of the 22 dependent steps of Horner's rule
  const dd_t z2 = dd_mul(z, z), z4 = dd_mul(z2, z2), z8 = dd_mul(z4, z4);
  const dd_t z16 = dd_mul(z8, z8);
  dd_t p[12];
#pragma unroll
  for (int i = 0; i < 11; ++i)
    p[i] = dd_add({C[2 * i][0], C[2 * i][1]}, dd_mul({C[2 * i + 1][0], C[2 * i + 1][1]}, z));
  p[11] = {C[22][0], C[22][1]};
  dd_t q[6];
#pragma unroll
  for (int j = 0; j < 6; ++j) q[j] = dd_add(p[2 * j], dd_mul(p[2 * j + 1], z2));
  const dd_t r0 = dd_add(q[0], dd_mul(q[1], z4)), r1 = dd_add(q[2], dd_mul(q[3], z4));
  const dd_t r2 = dd_add(q[4], dd_mul(q[5], z4));
  const dd_t s0 = dd_add(r0, dd_mul(r1, z8));
  const dd_t S = dd_add(s0, dd_mul(r2, z16));
  const dd_t lm = dd_mul({__dmul_rn(2.0, f.hi), __dmul_rn(2.0, f.lo)}, S);
  const dd_t ln2 = {0x1.62e42fefa39efp-1, 0x1.abc9e3b39803fp-56};
  return dd_add(dd_mul({static_cast<double>(e), 0.0}, ln2), lm);
}

__device__ inline double log_cr(double x) {
  if (!(x > 0.0) || isinf(x) || x < 2.2250738585072014e-308) return log(x);
  const dd_t r = log_dd(x);
  return __dadd_rn(r.hi, r.lo);
}

// ---- the EM loop's device log: the same value, table-driven -----------------
// m in [0.75, 1.5) is split at the nearest c_k = 0.75 + k/128 (k in [0, 96];
// c = 1 exactly around m = 1, so log x near 0 has no cancellation):
//   log x = e ln2 + log c_k + 2 atanh(f),  f = (m - c_k)/(m + c_k), |f| <= 1/512,
// z = f^2 < 2^-18 and the series 1 + z/3 + z^2/5 + ... + z^5/11 reaches 2^-108.
// log c_k comes from a per-device table of log_dd values (LogTable, built
// once); ~110 FP64 operations against log_dd's ~860.  Same contract as
// log_cr: the host compares every value with glibc after the run.
constexpr int kLogTable = 97;
struct LogTable {
  double hi[kLogTable];
  double lo[kLogTable];
};

__device__ inline double log_fast(double x, const double* thi, const double* tlo) {
  if (!(x > 0.0) || isinf(x) || x < 2.2250738585072014e-308) return log(x);
  int e;
  double m = frexp(x, &e);  // [0.5, 1)
  if (m < 0.75) {
    m = __dmul_rn(m, 2.0);
    e -= 1;
  }
  const int k = __double2int_rn(__dmul_rn(__dsub_rn(m, 0.75), 128.0));  // (both exact)
  const double c = __dadd_rn(0.75, __dmul_rn(static_cast<double>(k), 0.0078125));
  const double num = __dsub_rn(m, c);  // exact (Sterbenz)
  const dd_t den = dd_two_sum(m, c);   // exact
  const double q = __ddiv_rn(num, den.hi);
  const double rem = __dsub_rn(__fma_rn(-q, den.hi, num), __dmul_rn(q, den.lo));
  const dd_t f = dd_fast_two_sum(q, __ddiv_rn(rem, den.hi));
  const dd_t z = dd_mul(f, f);
  // S = 1 + z (1/3 + z (1/5 + z V)), V = 1/7 + z/9 + z^2/11 in double
  const double V = __fma_rn(z.hi, __fma_rn(z.hi, 0x1.745d1745d1746p-4, 0x1.c71c71c71c71cp-4),
                            0x1.2492492492492p-3);
  const dd_t U = dd_add({0x1.999999999999ap-3, -0x1.999999999999ap-57}, dd_mul(z, {V, 0.0}));
  const dd_t T = dd_add({0x1.5555555555555p-2, 0x1.5555555555555p-56}, dd_mul(z, U));
  const dd_t S = dd_add({1.0, 0.0}, dd_mul(z, T));
  const dd_t L = dd_mul({__dmul_rn(2.0, f.hi), __dmul_rn(2.0, f.lo)}, S);
  const dd_t ln2 = {0x1.62e42fefa39efp-1, 0x1.abc9e3b39803fp-56};
  const dd_t r = dd_add(dd_add(dd_mul({static_cast<double>(e), 0.0}, ln2), {thi[k], tlo[k]}), L);
  return __dadd_rn(r.hi, r.lo);
}

}  // namespace dpmrf_b200
