// The Cuda backend of the reference library: the functions
// integration/cuda_backend.patch dispatches to when backend.kind == Cuda.
// Every call marshals the caller's const& host vectors through the C ABI of
// include/dpmrf_cuda.h (inputs copied in, caller-owned outputs returned by
// value -- engine.hpp's ownership) and rethrows the status
// as the reference's exception type.
#include "dpmrf/cuda/engine_cuda.hpp"

#include <map>
#include <memory>
#include <stdexcept>
#include <string>

#include "dpmrf/error.hpp"
#include "dpmrf/mrf/engine.hpp"
#include "dpmrf_cuda.h"

namespace dpmrf::cuda {
namespace {

void check(dpmrf_status s, const char* where) {
  if (s == DPMRF_OK) return;
  const std::string msg = std::string(where) + ": " + dpmrf_last_error();
  switch (s) {
    case DPMRF_INPUT_ERROR: throw InputError(msg);
    case DPMRF_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case DPMRF_OUT_OF_RANGE: throw std::out_of_range(msg);
    default: throw std::runtime_error(msg);
  }
}

// One library context per (host thread, device): the reference's calls are
// externally synchronous and a context is not re-entrant.
struct Ctx {
  dpmrf_context* h = nullptr;
  explicit Ctx(unsigned device) {
    check(dpmrf_context_create(static_cast<int>(device), &h), "dpmrf_context_create");
  }
  ~Ctx() { dpmrf_context_destroy(h); }
  Ctx(const Ctx&) = delete;
  Ctx& operator=(const Ctx&) = delete;
};

dpmrf_context* ctx(const dpp::Backend& b) {
  thread_local std::map<unsigned, std::unique_ptr<Ctx>> ctxs;
  auto& p = ctxs[b.device];
  if (!p) p = std::make_unique<Ctx>(b.device);
  return p->h;
}

// Inputs arrive by const& on every call (and may have changed since the last
// one), so every call uploads them.
void upload_graph(dpmrf_context* c, const RegionGraph& g) {
  if (g.offsets.size() != std::size_t(g.num_vertices) + 1 && !(g.offsets.empty() && g.num_vertices == 0))
    throw std::invalid_argument("region graph: offsets must hold num_vertices + 1 entries");
  static const std::uint32_t zero = 0;
  check(dpmrf_set_graph(c, g.num_vertices, g.offsets.empty() ? &zero : g.offsets.data(),
                        g.neighbors.data(), g.region_mean.data()),
        "set_graph");
}

void upload_hoods(dpmrf_context* c, const NeighborhoodSet& h) {
  static const std::uint32_t zero = 0;
  check(dpmrf_set_hoods(c, h.size(), h.offsets.empty() ? &zero : h.offsets.data(),
                        h.members.data()),
        "set_hoods");
}

dpmrf_optimizer_config abi_config(const OptimizerConfig& c) {
  return {c.num_labels,        c.em_max_iters, c.map_max_iters, c.convergence_window,
          c.convergence_tol,   c.beta,         c.rng_seed};
}

}  // namespace

// engine.hpp:29-30 / engine.cpp:40-48
std::vector<std::uint32_t> slot_hood_map(const dpp::Backend& backend,
                                         const NeighborhoodSet& hoods) {
  auto* c = ctx(backend);
  upload_hoods(c, hoods);
  std::vector<std::uint32_t> out(hoods.total_slots());
  check(dpmrf_slot_hood_map(c, out.data()), "slot_hood_map");
  return out;
}

// engine.hpp:25-26 / engine.cpp:50-72
ReplicatedIndex replicate_by_label(const dpp::Backend& backend, const NeighborhoodSet& hoods,
                                   std::uint32_t num_labels) {
  auto* c = ctx(backend);
  upload_hoods(c, hoods);
  const std::size_t E = std::size_t(num_labels) * hoods.total_slots();
  ReplicatedIndex r;
  r.test_label.resize(E);
  r.old_index.resize(E);
  r.hood_id.resize(E);
  check(dpmrf_replicate_by_label(c, num_labels, r.test_label.data(), r.old_index.data(),
                                 r.hood_id.data()),
        "replicate_by_label");
  return r;
}

// engine.hpp:34-36 / engine.cpp:74-86
std::vector<std::uint32_t> discord_counts(const dpp::Backend& backend, const RegionGraph& graph,
                                          const std::vector<std::uint32_t>& labels,
                                          std::uint32_t num_labels) {
  auto* c = ctx(backend);
  upload_graph(c, graph);
  std::vector<std::uint32_t> out(std::size_t(num_labels) * graph.num_vertices);
  check(dpmrf_discord_counts(c, labels.data(), num_labels, out.data()), "discord_counts");
  return out;
}

// engine.hpp:43-46 / engine.cpp:88-113
std::vector<double> compute_energies(const dpp::Backend& backend, const RegionGraph& graph,
                                     const NeighborhoodSet& hoods, const ReplicatedIndex& rep,
                                     const LabelParams& params,
                                     const std::vector<std::uint32_t>& labels, double beta) {
  auto* c = ctx(backend);
  upload_graph(c, graph);
  upload_hoods(c, hoods);
  std::vector<double> out(rep.old_index.size());
  check(dpmrf_compute_energies(c, out.size(), rep.test_label.data(), rep.old_index.data(),
                               params.num_labels(), params.mu.data(), params.sigma.data(),
                               labels.data(), beta, out.data()),
        "compute_energies");
  return out;
}

// engine.hpp:53-54 / engine.cpp:115-145
MinLabelEnergies min_label_energies(const dpp::Backend& backend, const ReplicatedIndex& rep,
                                    const std::vector<double>& energies, std::size_t num_slots) {
  if (rep.old_index.size() != energies.size() || rep.test_label.size() != energies.size())
    throw std::invalid_argument("min_label_energies: replicated index/energies mismatch");
  auto* c = ctx(backend);
  MinLabelEnergies m;
  m.energy.resize(num_slots);
  m.label.resize(num_slots);
  check(dpmrf_min_label_energies(c, energies.size(), rep.test_label.data(), rep.old_index.data(),
                                 energies.data(), num_slots, m.energy.data(), m.label.data()),
        "min_label_energies");
  return m;
}

// engine.hpp:58-60 / engine.cpp:147-152
std::vector<double> neighborhood_energy_sums(const dpp::Backend& backend,
                                             const std::vector<std::uint32_t>& slot_hood,
                                             const std::vector<double>& min_energy) {
  if (slot_hood.size() != min_energy.size())
    throw std::invalid_argument("reduce_by_key: keys/values length mismatch");
  auto* c = ctx(backend);
  std::vector<double> out(slot_hood.size());
  std::uint64_t n = 0;
  check(dpmrf_neighborhood_energy_sums(c, slot_hood.size(), slot_hood.data(), min_energy.data(),
                                       out.data(), &n),
        "neighborhood_energy_sums");
  out.resize(n);
  return out;
}

// engine.hpp:65-67 / engine.cpp:154-169
std::vector<std::uint8_t> check_convergence(const dpp::Backend& backend,
                                            const std::vector<std::vector<double>>& history,
                                            int window, double tol) {
  if (history.empty()) return {};
  auto* c = ctx(backend);
  const std::size_t series = history.back().size();
  std::vector<double> flat;
  flat.reserve(history.size() * series);
  for (const auto& row : history) {
    if (row.size() != series)
      throw std::invalid_argument("check_convergence: history rows differ in length");
    flat.insert(flat.end(), row.begin(), row.end());
  }
  std::vector<std::uint8_t> out(series);
  check(dpmrf_check_convergence(c, history.size(), series, flat.data(), window, tol, out.data()),
        "check_convergence");
  return out;
}

// engine.hpp:73-76 / engine.cpp:171-191
std::vector<std::uint32_t> update_labels(const dpp::Backend& backend,
                                         const NeighborhoodSet& hoods,
                                         const std::vector<std::uint32_t>& argmin_label,
                                         const std::vector<std::uint32_t>& old_labels) {
  if (argmin_label.size() != hoods.total_slots())
    throw std::invalid_argument("update_labels: one argmin per hood slot required");
  auto* c = ctx(backend);
  upload_hoods(c, hoods);
  std::vector<std::uint32_t> out(old_labels.size());
  check(dpmrf_update_labels(c, argmin_label.data(), static_cast<std::uint32_t>(old_labels.size()),
                            old_labels.data(), out.data()),
        "update_labels");
  return out;
}

// engine.hpp:81-83 / engine.cpp:193-223
LabelParams update_parameters(const dpp::Backend& backend, const RegionGraph& graph,
                              const std::vector<std::uint32_t>& labels,
                              const LabelParams& previous) {
  if (labels.size() != graph.num_vertices)
    throw std::invalid_argument("update_parameters: one label per vertex required");
  auto* c = ctx(backend);
  upload_graph(c, graph);
  LabelParams out = previous;
  check(dpmrf_update_parameters(c, labels.data(), previous.num_labels(), previous.mu.data(),
                                previous.sigma.data(), out.mu.data(), out.sigma.data()),
        "update_parameters");
  return out;
}

// engine.hpp:107-108 / optimize.cpp:31-74: the device-resident EM loop with
// the reference's full trace (every MAP iteration's hood energies + flags).
OptimizeResult optimize(const dpp::Backend& backend, const RegionGraph& graph,
                        const NeighborhoodSet& hoods, const OptimizerConfig& config) {
  auto* c = ctx(backend);
  if (graph.offsets.size() != std::size_t(graph.num_vertices) + 1 &&
      !(graph.offsets.empty() && graph.num_vertices == 0))
    throw std::invalid_argument("region graph: offsets must hold num_vertices + 1 entries");
  const dpmrf_optimizer_config cfg = abi_config(config);
  const dpmrf_run_options opts{0u, DPMRF_TRACE_FULL};
  OptimizeResult r;
  r.labels.resize(graph.num_vertices);
  r.params.mu.resize(config.num_labels);
  r.params.sigma.resize(config.num_labels);
  static const std::uint32_t zero = 0;
  check(dpmrf_optimize_arrays(c, graph.num_vertices,
                              graph.offsets.empty() ? &zero : graph.offsets.data(),
                              graph.neighbors.data(), graph.region_mean.data(), hoods.size(),
                              hoods.offsets.empty() ? &zero : hoods.offsets.data(),
                              hoods.members.data(), &cfg, &opts, r.labels.data(),
                              r.params.mu.data(), r.params.sigma.data()),
        "optimize");
  std::int32_t em_n = 0;
  std::uint64_t series = 0;
  check(dpmrf_trace_info(c, &em_n, &series), "trace_info");
  r.trace.resize(static_cast<std::size_t>(em_n));
  for (std::int32_t em = 0; em < em_n; ++em) {
    EmIterationLog& log = r.trace[static_cast<std::size_t>(em)];
    std::int32_t it = 0;
    std::uint8_t conv = 0;
    log.params.mu.resize(config.num_labels);
    log.params.sigma.resize(config.num_labels);
    check(dpmrf_trace_em(c, em, &it, &log.total_energy, &conv, log.params.mu.data(),
                         log.params.sigma.data()),
          "trace_em");
    log.converged = conv != 0;
    log.map_iters.resize(static_cast<std::size_t>(it));
    for (std::int32_t t = 0; t < it; ++t) {
      MapIterationLog& m = log.map_iters[static_cast<std::size_t>(t)];
      m.hood_energy.resize(series);
      m.converged.resize(series);
      check(dpmrf_trace_map(c, em, t, m.hood_energy.data(), m.converged.data()), "trace_map");
    }
  }
  return r;
}

// neighborhoods.hpp:28-29 / neighborhoods.cpp:10-57, built on the device
NeighborhoodSet build_neighborhoods(const dpp::Backend& backend, const RegionGraph& graph,
                                    const CliqueSet& cliques, std::uint32_t k) {
  auto* c = ctx(backend);
  upload_graph(c, graph);
  static const std::uint32_t zero = 0;
  std::uint64_t S = 0;
  check(dpmrf_build_neighborhoods(c, cliques.size(),
                                  cliques.offsets.empty() ? &zero : cliques.offsets.data(),
                                  cliques.members.data(), k, &S),
        "build_neighborhoods");
  NeighborhoodSet h;
  std::uint64_t H = 0;
  h.offsets.resize(cliques.size() + 1);
  h.members.resize(S);
  h.source_clique.resize(cliques.size());
  check(dpmrf_get_hoods(c, &H, &S, h.offsets.data(), h.members.data(), h.source_clique.data()),
        "get_hoods");
  return h;
}

// region_graph.hpp:29-30 / region_graph.cpp:10-73, built on the device
RegionGraph build_region_graph(const dpp::Backend& backend, const GrayImage& image,
                               const LabelMap& labels) {
  if (image.width != labels.width || image.height != labels.height)
    throw InputError("region graph: image and label map dimensions differ");
  if (labels.num_regions == 0) throw InputError("region graph: label map not validated");
  auto* c = ctx(backend);
  std::uint64_t A = 0;
  check(dpmrf_build_region_graph(c, image.width, image.height, image.pixels.data(),
                                 labels.region.data(), labels.num_regions, &A),
        "build_region_graph");
  RegionGraph g;
  g.num_vertices = labels.num_regions;
  g.offsets.resize(std::size_t(g.num_vertices) + 1);
  g.neighbors.resize(A);
  g.region_mean.resize(g.num_vertices);
  g.region_size.resize(g.num_vertices);
  check(dpmrf_get_graph(c, nullptr, nullptr, g.offsets.data(), g.neighbors.data(),
                        g.region_mean.data(), g.region_size.data()),
        "get_graph");
  return g;
}

// cliques.hpp:26 / cliques.cpp:53-106, enumerated on the device
CliqueSet enumerate_maximal_cliques(const dpp::Backend& backend, const RegionGraph& graph) {
  auto* c = ctx(backend);
  upload_graph(c, graph);
  std::uint64_t C = 0, CS = 0;
  check(dpmrf_enumerate_maximal_cliques(c, &C, &CS), "enumerate_maximal_cliques");
  CliqueSet out;
  out.offsets.resize(C + 1);
  out.members.resize(CS);
  check(dpmrf_get_cliques(c, out.offsets.data(), out.members.data()), "get_cliques");
  return out;
}

}  // namespace dpmrf::cuda
