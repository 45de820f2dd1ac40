// dpmrf_b200/engine.hpp -- C++ drop-in for the reference's engine entry points.
//
// Same names, argument meaning and error behaviour as
//   /root/reference/proj/include/dpmrf/mrf/engine.hpp:15-116
//   /root/reference/proj/include/dpmrf/graph/neighborhoods.hpp:28-29
// with a CUDA backend selector.  Header-only: every call goes through the C
// ABI of dpmrf_cuda.h (libdpmrf_cuda.so) and rethrows the status as the
// reference's exception type:
//   DPMRF_INPUT_ERROR      -> dpmrf::InputError (error.hpp:11)
//   DPMRF_INVALID_ARGUMENT -> std::invalid_argument
//   DPMRF_OUT_OF_RANGE     -> std::out_of_range
//   anything else          -> std::runtime_error
// Value types mirror model.hpp / region_graph.hpp / cliques.hpp /
// neighborhoods.hpp member for member, so code written against the
// reference compiles after swapping the include and the namespace alias
// (see INTEGRATION.md).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../dpmrf_cuda.h"

namespace dpmrf_b200 {

class InputError : public std::runtime_error {
 public:
  explicit InputError(const std::string& what) : std::runtime_error(what) {}
};

inline void throw_status(dpmrf_status s, const char* where) {
  if (s == DPMRF_OK) return;
  const std::string msg = std::string(where) + ": " + dpmrf_last_error();
  switch (s) {
    case DPMRF_INPUT_ERROR: throw InputError(msg);
    case DPMRF_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case DPMRF_OUT_OF_RANGE: throw std::out_of_range(msg);
    default: throw std::runtime_error(msg);
  }
}

inline constexpr double kSigmaFloor = 1e-3;

struct LabelParams {
  std::vector<double> mu;
  std::vector<double> sigma;
  std::uint32_t num_labels() const { return static_cast<std::uint32_t>(mu.size()); }
};

struct OptimizerConfig {
  std::uint32_t num_labels = 2;
  int em_max_iters = 20;
  int map_max_iters = 10;
  int convergence_window = 3;
  double convergence_tol = 1e-4;
  double beta = 1.0;
  std::uint64_t rng_seed = 0;
};

struct ReplicatedIndex {
  std::vector<std::uint32_t> test_label, old_index, hood_id;
};

struct RegionGraph {
  std::uint32_t num_vertices = 0;
  std::vector<std::uint32_t> offsets, neighbors;
  std::vector<double> region_mean;
  std::vector<std::uint32_t> region_size;
  std::uint32_t degree(std::uint32_t v) const { return offsets[v + 1] - offsets[v]; }
};

struct CliqueSet {
  std::vector<std::uint32_t> offsets, members;
  std::size_t size() const { return offsets.empty() ? 0 : offsets.size() - 1; }
};

struct NeighborhoodSet {
  std::vector<std::uint32_t> offsets, members, source_clique;
  std::size_t size() const { return offsets.empty() ? 0 : offsets.size() - 1; }
  std::size_t total_slots() const { return members.size(); }
};

struct MinLabelEnergies {
  std::vector<double> energy;
  std::vector<std::uint32_t> label;
};

struct MapIterationLog {
  std::vector<double> hood_energy;
  std::vector<std::uint8_t> converged;
};

struct EmIterationLog {
  std::vector<MapIterationLog> map_iters;
  double total_energy = 0.0;
  bool converged = false;
  LabelParams params;
};

struct OptimizeResult {
  std::vector<std::uint32_t> labels;
  LabelParams params;
  std::vector<EmIterationLog> trace;
};

namespace dpp {
// dpp::Backend (backend.hpp:16-35) with the added Cuda kind; device_index
// selects the GPU.  Serial/Threaded remain the reference's CPU backends.
enum class BackendKind { Serial, Threaded, Cuda };
struct Backend {
  BackendKind kind = BackendKind::Cuda;
  int device_index = 0;
  static Backend cuda(int device = 0) { return Backend{BackendKind::Cuda, device}; }
};
}  // namespace dpp

namespace detail {

// One context per (thread, device).  The reference takes its inputs by const&
// on every call, so every call uploads them (an address-based cache would be
// fooled by a new object at a reused address); use the C ABI directly to keep
// a graph resident across calls.
struct Ctx {
  dpmrf_context* h = nullptr;
  explicit Ctx(int device) { throw_status(dpmrf_context_create(device, &h), "dpmrf_context_create"); }
  ~Ctx() { dpmrf_context_destroy(h); }
};

inline Ctx& ctx_for(const dpp::Backend& b) {
  if (b.kind != dpp::BackendKind::Cuda)
    throw InputError("dpmrf_b200: only the Cuda backend is provided by this library");
  thread_local std::map<int, std::unique_ptr<Ctx>> ctxs;
  auto& p = ctxs[b.device_index];
  if (!p) p = std::make_unique<Ctx>(b.device_index);
  return *p;
}

inline void graph(Ctx& c, const RegionGraph& g) {
  // a default-constructed (empty) graph has no offsets at all: the reference
  // accepts it, so pass the one-entry CSR {0}
  static const std::uint32_t zero = 0;
  if (g.offsets.empty() && g.num_vertices != 0)
    throw std::invalid_argument("region graph: offsets must hold num_vertices + 1 entries");
  throw_status(dpmrf_set_graph(c.h, g.num_vertices, g.offsets.empty() ? &zero : g.offsets.data(),
                               g.neighbors.data(), g.region_mean.data()),
               "set_graph");
}

inline void hoods(Ctx& c, const NeighborhoodSet& h) {
  std::vector<std::uint32_t> off = h.offsets.empty() ? std::vector<std::uint32_t>{0} : h.offsets;
  throw_status(dpmrf_set_hoods(c.h, off.size() - 1, off.data(), h.members.data()), "set_hoods");
}

}  // namespace detail

// ---- engine.hpp:20-21 ----
inline void init_random(std::uint32_t num_labels, std::uint32_t num_vertices, std::uint64_t seed,
                        LabelParams& params, std::vector<std::uint32_t>& labels,
                        const dpp::Backend& b = dpp::Backend::cuda()) {
  auto& c = detail::ctx_for(b);
  params.mu.assign(num_labels, 0.0);
  params.sigma.assign(num_labels, 0.0);
  labels.assign(num_vertices, 0);
  throw_status(dpmrf_init_random(c.h, num_labels, num_vertices, seed, 0, params.mu.data(),
                                 params.sigma.data(), labels.data()),
               "init_random");
}

// ---- engine.hpp:25-30 ----
inline ReplicatedIndex replicate_by_label(const dpp::Backend& b, const NeighborhoodSet& h,
                                          std::uint32_t num_labels) {
  auto& c = detail::ctx_for(b);
  detail::hoods(c, h);
  ReplicatedIndex r;
  const std::size_t E = std::size_t(num_labels) * h.total_slots();
  r.test_label.resize(E);
  r.old_index.resize(E);
  r.hood_id.resize(E);
  throw_status(dpmrf_replicate_by_label(c.h, num_labels, r.test_label.data(), r.old_index.data(),
                                        r.hood_id.data()),
               "replicate_by_label");
  return r;
}

inline std::vector<std::uint32_t> slot_hood_map(const dpp::Backend& b, const NeighborhoodSet& h) {
  auto& c = detail::ctx_for(b);
  detail::hoods(c, h);
  std::vector<std::uint32_t> out(h.total_slots());
  throw_status(dpmrf_slot_hood_map(c.h, out.data()), "slot_hood_map");
  return out;
}

// ---- engine.hpp:34-46 ----
inline std::vector<std::uint32_t> discord_counts(const dpp::Backend& b, const RegionGraph& g,
                                                 const std::vector<std::uint32_t>& labels,
                                                 std::uint32_t num_labels) {
  auto& c = detail::ctx_for(b);
  detail::graph(c, g);
  std::vector<std::uint32_t> out(std::size_t(num_labels) * g.num_vertices);
  throw_status(dpmrf_discord_counts(c.h, labels.data(), num_labels, out.data()), "discord_counts");
  return out;
}

inline std::vector<double> compute_energies(const dpp::Backend& b, const RegionGraph& g,
                                            const NeighborhoodSet& h, const ReplicatedIndex& rep,
                                            const LabelParams& params,
                                            const std::vector<std::uint32_t>& labels, double beta) {
  auto& c = detail::ctx_for(b);
  detail::graph(c, g);
  detail::hoods(c, h);
  std::vector<double> out(rep.old_index.size());
  throw_status(dpmrf_compute_energies(c.h, out.size(), rep.test_label.data(), rep.old_index.data(),
                                      params.num_labels(), params.mu.data(), params.sigma.data(),
                                      labels.data(), beta, out.data()),
               "compute_energies");
  return out;
}

// ---- engine.hpp:55-69 ----
inline MinLabelEnergies min_label_energies(const dpp::Backend& b, const ReplicatedIndex& rep,
                                           const std::vector<double>& energies,
                                           std::size_t num_slots) {
  if (rep.old_index.size() != energies.size() || rep.test_label.size() != energies.size())
    throw std::invalid_argument("min_label_energies: replicated index/energies mismatch");
  auto& c = detail::ctx_for(b);
  MinLabelEnergies m;
  m.energy.resize(num_slots);
  m.label.resize(num_slots);
  throw_status(dpmrf_min_label_energies(c.h, energies.size(), rep.test_label.data(),
                                        rep.old_index.data(), energies.data(), num_slots,
                                        m.energy.data(), m.label.data()),
               "min_label_energies");
  return m;
}

inline std::vector<double> neighborhood_energy_sums(const dpp::Backend& b,
                                                    const std::vector<std::uint32_t>& slot_hood,
                                                    const std::vector<double>& min_energy) {
  if (slot_hood.size() != min_energy.size())
    throw std::invalid_argument("reduce_by_key: keys/values length mismatch");
  auto& c = detail::ctx_for(b);
  std::vector<double> out(slot_hood.size());
  std::uint64_t n = 0;
  throw_status(dpmrf_neighborhood_energy_sums(c.h, slot_hood.size(), slot_hood.data(),
                                              min_energy.data(), out.data(), &n),
               "neighborhood_energy_sums");
  out.resize(n);
  return out;
}

inline std::vector<std::uint8_t> check_convergence(const dpp::Backend& b,
                                                   const std::vector<std::vector<double>>& history,
                                                   int window, double tol) {
  if (history.empty()) return {};
  auto& c = detail::ctx_for(b);
  const std::size_t series = history.back().size();
  std::vector<double> flat;
  flat.reserve(history.size() * series);
  for (const auto& row : history) flat.insert(flat.end(), row.begin(), row.end());
  std::vector<std::uint8_t> out(series);
  throw_status(dpmrf_check_convergence(c.h, history.size(), series, flat.data(), window, tol,
                                       out.data()),
               "check_convergence");
  return out;
}

// ---- engine.hpp:75-85 ----
inline std::vector<std::uint32_t> update_labels(const dpp::Backend& b, const NeighborhoodSet& h,
                                                const std::vector<std::uint32_t>& argmin_label,
                                                const std::vector<std::uint32_t>& old_labels) {
  if (argmin_label.size() != h.total_slots())
    throw std::invalid_argument("update_labels: one argmin per hood slot required");
  auto& c = detail::ctx_for(b);
  detail::hoods(c, h);
  std::vector<std::uint32_t> out(old_labels.size());
  throw_status(dpmrf_update_labels(c.h, argmin_label.data(),
                                   static_cast<std::uint32_t>(old_labels.size()),
                                   old_labels.data(), out.data()),
               "update_labels");
  return out;
}

inline LabelParams update_parameters(const dpp::Backend& b, const RegionGraph& g,
                                     const std::vector<std::uint32_t>& labels,
                                     const LabelParams& previous) {
  if (labels.size() != g.num_vertices)
    throw std::invalid_argument("update_parameters: one label per vertex required");
  auto& c = detail::ctx_for(b);
  detail::graph(c, g);
  LabelParams out = previous;
  throw_status(dpmrf_update_parameters(c.h, labels.data(), previous.num_labels(),
                                       previous.mu.data(), previous.sigma.data(), out.mu.data(),
                                       out.sigma.data()),
               "update_parameters");
  return out;
}

// ---- engine.hpp:99-100 ----
inline OptimizeResult optimize(const dpp::Backend& b, const RegionGraph& g,
                               const NeighborhoodSet& h, const OptimizerConfig& config,
                               int trace_level = DPMRF_TRACE_FULL, unsigned run_flags = 0) {
  auto& c = detail::ctx_for(b);
  dpmrf_optimizer_config cfg{config.num_labels, config.em_max_iters, config.map_max_iters,
                             config.convergence_window, config.convergence_tol, config.beta,
                             config.rng_seed};
  dpmrf_run_options opts{run_flags, trace_level};
  OptimizeResult r;
  r.labels.resize(g.num_vertices);
  r.params.mu.resize(config.num_labels);
  r.params.sigma.resize(config.num_labels);
  // graph + hoods upload and the run in one call (engine.hpp:99-100's shape)
  const std::vector<std::uint32_t> h_off =
      h.offsets.empty() ? std::vector<std::uint32_t>{0} : h.offsets;
  static const std::uint32_t zero = 0;
  throw_status(dpmrf_optimize_arrays(c.h, g.num_vertices, g.offsets.empty() ? &zero : g.offsets.data(),
                                     g.neighbors.data(),
                                     g.region_mean.data(), h_off.size() - 1, h_off.data(),
                                     h.members.data(), &cfg, &opts, r.labels.data(),
                                     r.params.mu.data(), r.params.sigma.data()),
               "optimize");
  std::int32_t em_n = 0;
  std::uint64_t series = 0;
  throw_status(dpmrf_trace_info(c.h, &em_n, &series), "trace_info");
  for (std::int32_t em = 0; em < em_n; ++em) {
    EmIterationLog log;
    std::int32_t it = 0;
    std::uint8_t conv = 0;
    log.params.mu.resize(config.num_labels);
    log.params.sigma.resize(config.num_labels);
    throw_status(dpmrf_trace_em(c.h, em, &it, &log.total_energy, &conv, log.params.mu.data(),
                                log.params.sigma.data()),
                 "trace_em");
    log.converged = conv != 0;
    if (trace_level >= DPMRF_TRACE_FULL) {
      for (std::int32_t t = 0; t < it; ++t) {
        MapIterationLog m;
        m.hood_energy.resize(series);
        m.converged.resize(series);
        throw_status(dpmrf_trace_map(c.h, em, t, m.hood_energy.data(), m.converged.data()),
                     "trace_map");
        log.map_iters.push_back(std::move(m));
      }
    }
    r.trace.push_back(std::move(log));
  }
  return r;
}

// ---- neighborhoods.hpp:28-29 (built on the device) ----
inline NeighborhoodSet build_neighborhoods(const dpp::Backend& b, const RegionGraph& g,
                                           const CliqueSet& cliques, std::uint32_t k = 1) {
  auto& c = detail::ctx_for(b);
  detail::graph(c, g);
  std::vector<std::uint32_t> off = cliques.offsets.empty() ? std::vector<std::uint32_t>{0}
                                                           : cliques.offsets;
  std::uint64_t S = 0;
  throw_status(dpmrf_build_neighborhoods(c.h, off.size() - 1, off.data(), cliques.members.data(), k,
                                         &S),
               "build_neighborhoods");
  NeighborhoodSet h;
  std::uint64_t H = 0;
  h.offsets.resize(off.size());
  h.members.resize(S);
  h.source_clique.resize(off.size() - 1);
  throw_status(dpmrf_get_hoods(c.h, &H, &S, h.offsets.data(), h.members.data(),
                               h.source_clique.data()),
               "get_hoods");
  return h;
}

// ---- graph/image.hpp, graph/label_map.hpp value types ----
struct GrayImage {
  std::uint32_t width = 0;
  std::uint32_t height = 0;
  std::vector<std::uint8_t> pixels;
  std::size_t size() const { return pixels.size(); }
};
struct BinaryImage {
  std::uint32_t width = 0;
  std::uint32_t height = 0;
  std::vector<std::uint8_t> pixels;
  std::size_t size() const { return pixels.size(); }
};
struct LabelMap {
  std::uint32_t width = 0;
  std::uint32_t height = 0;
  std::vector<std::uint32_t> region;
  std::uint32_t num_regions = 0;  // set by the reference's validate_label_map
};

// ---- label_map.hpp validate_label_map (label_map.cpp:38-78, on the device) ----
inline void validate_label_map(LabelMap& map, const dpp::Backend& b = dpp::Backend::cuda()) {
  if (map.region.size() != std::size_t(map.width) * map.height)
    throw InputError("label map: size does not match dimensions");
  auto& c = detail::ctx_for(b);
  std::uint32_t num = 0;
  throw_status(dpmrf_validate_label_map(c.h, map.width, map.height, map.region.data(), &num),
               "validate_label_map");
  map.num_regions = num;
}

// ---- region_graph.hpp:29-30 (built on the device) ----
inline RegionGraph build_region_graph(const dpp::Backend& b, const GrayImage& image,
                                      const LabelMap& labels) {
  if (image.width != labels.width || image.height != labels.height)
    throw InputError("region graph: image and label map dimensions differ");
  auto& c = detail::ctx_for(b);
  std::uint64_t A = 0;
  throw_status(dpmrf_build_region_graph(c.h, image.width, image.height, image.pixels.data(),
                                        labels.region.data(), labels.num_regions, &A),
               "build_region_graph");
  RegionGraph g;
  g.num_vertices = labels.num_regions;
  g.offsets.resize(std::size_t(g.num_vertices) + 1);
  g.neighbors.resize(A);
  g.region_mean.resize(g.num_vertices);
  g.region_size.resize(g.num_vertices);
  throw_status(dpmrf_get_graph(c.h, nullptr, nullptr, g.offsets.data(), g.neighbors.data(),
                               g.region_mean.data(), g.region_size.data()),
               "get_graph");
  return g;
}

// ---- cliques.hpp:26 (enumerated on the device) ----
inline CliqueSet enumerate_maximal_cliques(const dpp::Backend& b, const RegionGraph& g) {
  auto& c = detail::ctx_for(b);
  detail::graph(c, g);
  std::uint64_t C = 0, CS = 0;
  throw_status(dpmrf_enumerate_maximal_cliques(c.h, &C, &CS), "enumerate_maximal_cliques");
  CliqueSet out;
  out.offsets.resize(C + 1);
  out.members.resize(CS);
  throw_status(dpmrf_get_cliques(c.h, out.offsets.data(), out.members.data()), "get_cliques");
  return out;
}

// ---- eval/metrics.hpp (confusion counted on the device) ----
struct ConfusionCounts {
  std::uint64_t tp = 0;
  std::uint64_t tn = 0;
  std::uint64_t fp = 0;
  std::uint64_t fn = 0;
};
struct Metrics {
  double precision = 0.0;
  double recall = 0.0;
  double accuracy = 0.0;
  bool precision_defined = true;
  bool recall_defined = true;
};

inline ConfusionCounts confusion(const BinaryImage& pred, const BinaryImage& truth,
                                 const dpp::Backend& b = dpp::Backend::cuda()) {
  if (pred.width != truth.width || pred.height != truth.height)
    throw InputError("confusion: image dimensions differ");
  auto& c = detail::ctx_for(b);
  std::uint64_t k[4] = {0, 0, 0, 0};
  throw_status(dpmrf_confusion(c.h, pred.pixels.size(), pred.pixels.data(), truth.pixels.data(), k),
               "confusion");
  return {k[0], k[1], k[2], k[3]};
}

// metrics.cpp:16-35 (host arithmetic)
inline Metrics compute_metrics(const ConfusionCounts& c) {
  Metrics m;
  const double tp = static_cast<double>(c.tp), tn = static_cast<double>(c.tn);
  const double fp = static_cast<double>(c.fp), fn = static_cast<double>(c.fn);
  if (c.tp + c.fp == 0) m.precision_defined = false;
  else m.precision = tp / (tp + fp);
  if (c.tp + c.fn == 0) m.recall_defined = false;
  else m.recall = tp / (tp + fn);
  const double total = tp + tn + fp + fn;
  m.accuracy = total == 0.0 ? 0.0 : (tp + tn) / total;
  return m;
}

// metrics.cpp:37-42
inline double porosity(const BinaryImage& img) {
  if (img.pixels.empty()) return 0.0;
  std::uint64_t pore = 0;
  for (std::uint8_t p : img.pixels) pore += p;
  return static_cast<double>(pore) / static_cast<double>(img.pixels.size());
}

}  // namespace dpmrf_b200
