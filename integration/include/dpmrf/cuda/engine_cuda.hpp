// dpmrf/cuda/engine_cuda.hpp -- the Cuda backend of the reference library.
//
// integration/cuda_backend.patch adds BackendKind::Cuda to
// proj/include/dpmrf/dpp/backend.hpp:8 and one line at the top of each
// engine-level entry point,
//     if (backend.kind == dpp::BackendKind::Cuda) return cuda::<same call>;
// in proj/src/mrf/engine.cpp, optimize.cpp, graph/neighborhoods.cpp,
// region_graph.cpp and cliques.cpp.  These are the functions it lands in:
// same signatures as proj/include/dpmrf/mrf/engine.hpp:15-116,
// graph/neighborhoods.hpp:28-29, region_graph.hpp:29-30 and cliques.hpp:26,
// implemented over the C ABI of include/dpmrf_cuda.h (libdpmrf_cuda.so).
// Statuses come back as the reference's exception types:
//   DPMRF_INPUT_ERROR -> dpmrf::InputError (error.hpp:11),
//   DPMRF_INVALID_ARGUMENT -> std::invalid_argument,
//   DPMRF_OUT_OF_RANGE -> std::out_of_range, anything else -> std::runtime_error.
// Serial and Threaded never reach this file.
#pragma once

#include <cstdint>
#include <vector>

#include "dpmrf/dpp/backend.hpp"
#include "dpmrf/graph/cliques.hpp"
#include "dpmrf/graph/image.hpp"
#include "dpmrf/graph/label_map.hpp"
#include "dpmrf/graph/neighborhoods.hpp"
#include "dpmrf/graph/region_graph.hpp"
#include "dpmrf/mrf/model.hpp"

namespace dpmrf {

struct MinLabelEnergies;
struct OptimizeResult;

namespace cuda {

std::vector<std::uint32_t> slot_hood_map(const dpp::Backend& backend,
                                         const NeighborhoodSet& hoods);
ReplicatedIndex replicate_by_label(const dpp::Backend& backend, const NeighborhoodSet& hoods,
                                   std::uint32_t num_labels);
std::vector<std::uint32_t> discord_counts(const dpp::Backend& backend, const RegionGraph& graph,
                                          const std::vector<std::uint32_t>& labels,
                                          std::uint32_t num_labels);
std::vector<double> compute_energies(const dpp::Backend& backend, const RegionGraph& graph,
                                     const NeighborhoodSet& hoods, const ReplicatedIndex& rep,
                                     const LabelParams& params,
                                     const std::vector<std::uint32_t>& labels, double beta);
MinLabelEnergies min_label_energies(const dpp::Backend& backend, const ReplicatedIndex& rep,
                                    const std::vector<double>& energies, std::size_t num_slots);
std::vector<double> neighborhood_energy_sums(const dpp::Backend& backend,
                                             const std::vector<std::uint32_t>& slot_hood,
                                             const std::vector<double>& min_energy);
std::vector<std::uint8_t> check_convergence(const dpp::Backend& backend,
                                            const std::vector<std::vector<double>>& history,
                                            int window, double tol);
std::vector<std::uint32_t> update_labels(const dpp::Backend& backend,
                                         const NeighborhoodSet& hoods,
                                         const std::vector<std::uint32_t>& argmin_label,
                                         const std::vector<std::uint32_t>& old_labels);
LabelParams update_parameters(const dpp::Backend& backend, const RegionGraph& graph,
                              const std::vector<std::uint32_t>& labels,
                              const LabelParams& previous);
OptimizeResult optimize(const dpp::Backend& backend, const RegionGraph& graph,
                        const NeighborhoodSet& hoods, const OptimizerConfig& config);

NeighborhoodSet build_neighborhoods(const dpp::Backend& backend, const RegionGraph& graph,
                                    const CliqueSet& cliques, std::uint32_t k);
RegionGraph build_region_graph(const dpp::Backend& backend, const GrayImage& image,
                               const LabelMap& labels);
CliqueSet enumerate_maximal_cliques(const dpp::Backend& backend, const RegionGraph& graph);

}  // namespace cuda
}  // namespace dpmrf
