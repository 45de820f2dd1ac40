// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference library, compiled from its
// own sources under /root/reference/proj by oracle/Makefile into
// oracle/_ref/libdpmrf_ref.so.  Used to (a) pin the C restatement in
// oracle/dpmrf_oracle.c, (b) generate golden fixtures, and (c) time the
// reference CPU path for bench.py's cpu_baseline / --impl reference arm.
//
// Only the reference's PUBLIC entry points are called (proj/include/dpmrf/*).
// Two workloads need a recomposition because the reference hard-wires them:
//   * fixed work (no early exits): optimize() breaks at optimize.cpp:59/:71;
//     ref_optimize(mode=1) recomposes it from the public step functions, in
//     exactly optimize.cpp:43-72's order (bit-identical when exits are on).
//   * M != 2: init_random rejects it (engine.cpp:30); the recomposition uses
//     the same SplitMix64 stream for any M.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <map>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "dpmrf/dpp/kernels.hpp"
#include "dpmrf/error.hpp"
#include "dpmrf/eval/metrics.hpp"
#include "dpmrf/eval/phantom.hpp"
#include "dpmrf/graph/cliques.hpp"
#include "dpmrf/graph/label_map.hpp"
#include "dpmrf/graph/neighborhoods.hpp"
#include "dpmrf/graph/region_graph.hpp"
#include "dpmrf/mrf/engine.hpp"

using namespace dpmrf;

namespace {

int code_of(const std::exception_ptr& ep) {
  try {
    std::rethrow_exception(ep);
  } catch (const InputError&) {
    return 1;
  } catch (const std::invalid_argument&) {
    return 2;
  } catch (const std::out_of_range&) {
    return 3;
  } catch (...) {
    return 6;
  }
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

struct Pipe {
  GrayImage image;
  BinaryImage truth;
  LabelMap map;
  RegionGraph graph;
  CliqueSet cliques;
  NeighborhoodSet hoods;
  double t_graph = 0, t_cliques = 0, t_hoods = 0;
};

dpp::Backend backend_of(int threads) {
  return threads <= 1 ? dpp::Backend::serial() : dpp::Backend::threaded(unsigned(threads));
}

// Brick oversegmentation: block rows of height b, odd block rows shifted by
// b/2, ids assigned in first-seen row-major order.
LabelMap brick_oversegment(std::uint32_t w, std::uint32_t h, std::uint32_t b) {
  LabelMap map;
  map.width = w;
  map.height = h;
  map.region.resize(std::size_t(w) * h);
  std::map<std::pair<std::uint32_t, std::uint32_t>, std::uint32_t> ids;
  for (std::uint32_t y = 0; y < h; ++y) {
    const std::uint32_t r = y / b;
    const std::uint32_t shift = (r & 1u) ? b / 2 : 0;
    for (std::uint32_t x = 0; x < w; ++x) {
      const auto key = std::make_pair(r, (x + shift) / b);
      auto it = ids.find(key);
      if (it == ids.end()) it = ids.emplace(key, std::uint32_t(ids.size())).first;
      map.region[std::size_t(y) * w + x] = it->second;
    }
  }
  validate_label_map(map);
  return map;
}

double secs(std::chrono::steady_clock::time_point a) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
}

struct RefCfg {
  std::uint32_t num_labels;
  std::int32_t em_max_iters;
  std::int32_t map_max_iters;
  std::int32_t convergence_window;
  double convergence_tol;
  double beta;
  std::uint64_t rng_seed;
};

OptimizerConfig to_cfg(const RefCfg* c) {
  OptimizerConfig o;
  o.num_labels = c->num_labels;
  o.em_max_iters = c->em_max_iters;
  o.map_max_iters = c->map_max_iters;
  o.convergence_window = c->convergence_window;
  o.convergence_tol = c->convergence_tol;
  o.beta = c->beta;
  o.rng_seed = c->rng_seed;
  return o;
}

std::uint64_t next_u64(std::uint64_t& state) {
  std::uint64_t z = (state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// init_random's stream for any M (engine.cpp:28-38 draw order).
void init_any(std::uint32_t M, std::uint32_t R, std::uint64_t seed, LabelParams& p,
              std::vector<std::uint32_t>& labels) {
  if (M == 2) {
    init_random(M, R, seed, p, labels);
    return;
  }
  std::uint64_t st = seed;
  p.mu.resize(M);
  p.sigma.resize(M);
  for (auto& m : p.mu) m = 255.0 * (static_cast<double>(next_u64(st) >> 11) * 0x1.0p-53);
  for (auto& s : p.sigma)
    s = std::max(255.0 * (static_cast<double>(next_u64(st) >> 11) * 0x1.0p-53), kSigmaFloor);
  labels.resize(R);
  for (auto& l : labels) l = static_cast<std::uint32_t>(next_u64(st) % M);
}

void validate_any(const OptimizerConfig& c) {
  if (c.num_labels < 1) throw InputError("num_labels must be >= 1");
  if (c.em_max_iters < 0) throw InputError("em_max_iters must be >= 0");
  if (c.map_max_iters < 1) throw InputError("map_max_iters must be >= 1");
  if (c.convergence_window < 1) throw InputError("convergence_window must be >= 1");
  if (c.convergence_window >= c.map_max_iters) throw InputError("window");
  if (!(c.convergence_tol > 0.0)) throw InputError("tol");
  if (!(c.beta >= 0.0)) throw InputError("beta");
}

struct TraceOut {
  std::int32_t* em_map_iters;
  double* em_total;
  std::uint8_t* em_conv;
  double* em_mu;
  double* em_sigma;
  double* map_energy;  // (em*map_max + it)*H + h, may be null
  std::uint8_t* map_conv;
  std::int32_t em_iters;
  std::uint64_t series;
};

void emit(const OptimizeResult& r, const OptimizerConfig& c, std::size_t H, std::uint32_t* labels,
          double* mu, double* sigma, TraceOut* tr) {
  std::copy(r.labels.begin(), r.labels.end(), labels);
  std::copy(r.params.mu.begin(), r.params.mu.end(), mu);
  std::copy(r.params.sigma.begin(), r.params.sigma.end(), sigma);
  if (!tr) return;
  const std::size_t M = r.params.mu.size();
  tr->em_iters = static_cast<std::int32_t>(r.trace.size());
  tr->series = 0;
  for (std::size_t em = 0; em < r.trace.size(); ++em) {
    const auto& e = r.trace[em];
    tr->em_map_iters[em] = static_cast<std::int32_t>(e.map_iters.size());
    tr->em_total[em] = e.total_energy;
    tr->em_conv[em] = e.converged ? 1 : 0;
    std::copy(e.params.mu.begin(), e.params.mu.end(), tr->em_mu + em * M);
    std::copy(e.params.sigma.begin(), e.params.sigma.end(), tr->em_sigma + em * M);
    for (std::size_t it = 0; it < e.map_iters.size(); ++it) {
      const auto& m = e.map_iters[it];
      tr->series = m.hood_energy.size();
      if (!tr->map_energy) continue;
      const std::size_t base = (em * std::size_t(c.map_max_iters) + it) * H;
      std::copy(m.hood_energy.begin(), m.hood_energy.end(), tr->map_energy + base);
      std::copy(m.converged.begin(), m.converged.end(), tr->map_conv + base);
    }
  }
}

// optimize() recomposed from the public step functions, optimize.cpp:31-74
// order; fixed_work drops the two breaks.
OptimizeResult optimize_steps(const dpp::Backend& b, const RegionGraph& g,
                              const NeighborhoodSet& hoods, const OptimizerConfig& c,
                              bool fixed_work) {
  validate_any(c);
  OptimizeResult res;
  init_any(c.num_labels, g.num_vertices, c.rng_seed, res.params, res.labels);
  if (c.em_max_iters == 0) return res;
  const auto rep = replicate_by_label(b, hoods, c.num_labels);
  const auto slot_hood = slot_hood_map(b, hoods);
  const std::size_t num_slots = hoods.total_slots();
  std::vector<std::vector<double>> em_history;
  for (int em = 0; em < c.em_max_iters; ++em) {
    EmIterationLog em_log;
    std::vector<std::vector<double>> hood_history;
    for (int it = 0; it < c.map_max_iters; ++it) {
      const auto energies = compute_energies(b, g, hoods, rep, res.params, res.labels, c.beta);
      const auto mins = min_label_energies(b, rep, energies, num_slots);
      res.labels = update_labels(b, hoods, mins.label, res.labels);
      hood_history.push_back(neighborhood_energy_sums(b, slot_hood, mins.energy));
      MapIterationLog map_log;
      map_log.hood_energy = hood_history.back();
      map_log.converged =
          check_convergence(b, hood_history, c.convergence_window, c.convergence_tol);
      const bool done = std::all_of(map_log.converged.begin(), map_log.converged.end(),
                                    [](std::uint8_t f) { return f != 0; });
      em_log.map_iters.push_back(std::move(map_log));
      if (done && !fixed_work) break;
    }
    res.params = update_parameters(b, g, res.labels, res.params);
    em_log.params = res.params;
    em_log.total_energy =
        dpp::reduce(b, em_log.map_iters.back().hood_energy, std::plus<double>{}, 0.0);
    em_history.push_back({em_log.total_energy});
    const auto em_conv = check_convergence(b, em_history, c.convergence_window, c.convergence_tol);
    em_log.converged = !em_conv.empty() && em_conv[0] != 0;
    res.trace.push_back(std::move(em_log));
    if (res.trace.back().converged && !fixed_work) break;
  }
  return res;
}

// optimize_reference's body (optimize.cpp:76-144) for the fixed-work and
// M != 2 workloads; uses the reference's own label_energy / make_label_terms /
// update_parameters / check_convergence / dpp::reduce.
OptimizeResult sweep_steps(const RegionGraph& graph, const NeighborhoodSet& hoods,
                           const OptimizerConfig& config, bool fixed_work) {
  validate_any(config);
  const dpp::Backend serial = dpp::Backend::serial();
  OptimizeResult res;
  init_any(config.num_labels, graph.num_vertices, config.rng_seed, res.params, res.labels);
  if (config.em_max_iters == 0) return res;
  const std::size_t H = hoods.size();
  const std::uint32_t M = config.num_labels;
  std::vector<std::vector<double>> em_history;
  for (int em = 0; em < config.em_max_iters; ++em) {
    EmIterationLog em_log;
    const LabelTerms terms = make_label_terms(res.params);
    std::vector<std::vector<double>> hood_history;
    for (int it = 0; it < config.map_max_iters; ++it) {
      std::vector<double> hood_energy(H, 0.0);
      std::vector<std::uint32_t> winners;
      for (std::size_t h = 0; h < H; ++h) {
        const std::uint32_t lo = hoods.offsets[h];
        const std::uint32_t hi = hoods.offsets[h + 1];
        winners.assign(hi - lo, 0);
        double sum = 0.0;
        for (std::uint32_t s = lo; s < hi; ++s) {
          const std::uint32_t v = hoods.members[s];
          double best = 0.0;
          std::uint32_t best_label = 0;
          for (std::uint32_t l = 0; l < M; ++l) {
            std::uint32_t dc = 0;
            for (const std::uint32_t* u = graph.adj_begin(v); u != graph.adj_end(v); ++u)
              dc += res.labels[*u] != l;
            const double e = label_energy(graph.region_mean[v], terms.mu[l], terms.two_var[l],
                                          terms.log_sigma[l], config.beta, dc);
            if (l == 0 || e < best) {
              best = e;
              best_label = l;
            }
          }
          winners[s - lo] = best_label;
          sum = s == lo ? best : sum + best;
        }
        for (std::uint32_t s = lo; s < hi; ++s) res.labels[hoods.members[s]] = winners[s - lo];
        hood_energy[h] = sum;
      }
      hood_history.push_back(std::move(hood_energy));
      MapIterationLog map_log;
      map_log.hood_energy = hood_history.back();
      map_log.converged = check_convergence(serial, hood_history, config.convergence_window,
                                            config.convergence_tol);
      const bool done = std::all_of(map_log.converged.begin(), map_log.converged.end(),
                                    [](std::uint8_t f) { return f != 0; });
      em_log.map_iters.push_back(std::move(map_log));
      if (done && !fixed_work) break;
    }
    res.params = update_parameters(serial, graph, res.labels, res.params);
    em_log.params = res.params;
    em_log.total_energy =
        dpp::reduce(serial, em_log.map_iters.back().hood_energy, std::plus<double>{}, 0.0);
    em_history.push_back({em_log.total_energy});
    const auto em_conv =
        check_convergence(serial, em_history, config.convergence_window, config.convergence_tol);
    em_log.converged = !em_conv.empty() && em_conv[0] != 0;
    res.trace.push_back(std::move(em_log));
    if (res.trace.back().converged && !fixed_work) break;
  }
  return res;
}

}  // namespace

extern "C" {

// ---- pipelines -------------------------------------------------------------

// Phantom -> corrupt -> oversegment (grid, or brick when brick != 0) -> region
// graph -> maximal cliques -> neighborhoods, each with the reference's code.
void* ref_pipe_phantom(std::uint32_t w, std::uint32_t h, double pore, double sp, double gauss,
                       int ringing, std::uint64_t seed, std::uint32_t block, int brick,
                       int threads, int* status) {
  Pipe* p = new Pipe;
  *status = guarded([&] {
    PhantomSpec spec;
    spec.width = w;
    spec.height = h;
    spec.pore_fraction = pore;
    spec.sp_rate = sp;
    spec.gauss_sigma = gauss;
    spec.ringing = ringing != 0;
    spec.seed = seed;
    const auto ph = gen_phantom(spec);
    p->truth = ph.truth;
    p->image = corrupt(ph.clean, spec);
    if (brick) {
      p->map = brick_oversegment(w, h, block);
    } else {
      p->map = grid_oversegment(w, h, block);
      validate_label_map(p->map);
    }
    const auto b = backend_of(threads);
    auto t0 = std::chrono::steady_clock::now();
    p->graph = build_region_graph(b, p->image, p->map);
    p->t_graph = secs(t0);
    t0 = std::chrono::steady_clock::now();
    p->cliques = enumerate_maximal_cliques(b, p->graph);
    p->t_cliques = secs(t0);
    t0 = std::chrono::steady_clock::now();
    p->hoods = build_neighborhoods(b, p->graph, p->cliques);
    p->t_hoods = secs(t0);
  });
  if (*status) {
    delete p;
    return nullptr;
  }
  return p;
}

// Hand-made graph (CSR + means); cliques enumerated by the reference when
// c_off == nullptr, else taken as given; hoods built by the reference when
// h_off == nullptr, else taken as given (source_clique = identity).
void* ref_pipe_arrays(std::uint32_t R, const std::uint32_t* g_off, const std::uint32_t* g_nbr,
                      const double* mean, std::uint64_t C, const std::uint32_t* c_off,
                      const std::uint32_t* c_mem, std::uint64_t H, const std::uint32_t* h_off,
                      const std::uint32_t* h_mem, int* status) {
  Pipe* p = new Pipe;
  *status = guarded([&] {
    p->graph.num_vertices = R;
    p->graph.offsets.assign(g_off, g_off + R + 1);
    p->graph.neighbors.assign(g_nbr, g_nbr + g_off[R]);
    p->graph.region_mean.assign(mean, mean + R);
    p->graph.region_size.assign(R, 1);
    const auto b = dpp::Backend::serial();
    if (c_off) {
      p->cliques.offsets.assign(c_off, c_off + C + 1);
      p->cliques.members.assign(c_mem, c_mem + c_off[C]);
    } else {
      p->cliques = enumerate_maximal_cliques(b, p->graph);
    }
    if (h_off) {
      p->hoods.offsets.assign(h_off, h_off + H + 1);
      p->hoods.members.assign(h_mem, h_mem + h_off[H]);
      for (std::uint32_t i = 0; i < H; ++i) p->hoods.source_clique.push_back(i);
    } else {
      p->hoods = build_neighborhoods(b, p->graph, p->cliques);
    }
  });
  if (*status) {
    delete p;
    return nullptr;
  }
  return p;
}

// Caller's image + label map (num_regions = the validated map's region
// count): region graph, maximal cliques and neighborhoods by the reference.
void* ref_pipe_labelmap(std::uint32_t w, std::uint32_t h, const std::uint8_t* pixels,
                        const std::uint32_t* region, std::uint32_t num_regions, int threads,
                        int* status) {
  Pipe* p = new Pipe;
  *status = guarded([&] {
    const std::size_t n = std::size_t(w) * h;
    p->image.width = w;
    p->image.height = h;
    p->image.pixels.assign(pixels, pixels + n);
    p->map.width = w;
    p->map.height = h;
    p->map.region.assign(region, region + n);
    p->map.num_regions = num_regions;
    const auto b = backend_of(threads);
    auto t0 = std::chrono::steady_clock::now();
    p->graph = build_region_graph(b, p->image, p->map);
    p->t_graph = secs(t0);
    t0 = std::chrono::steady_clock::now();
    p->cliques = enumerate_maximal_cliques(b, p->graph);
    p->t_cliques = secs(t0);
    t0 = std::chrono::steady_clock::now();
    p->hoods = build_neighborhoods(b, p->graph, p->cliques);
    p->t_hoods = secs(t0);
  });
  if (*status) {
    delete p;
    return nullptr;
  }
  return p;
}

void ref_pipe_free(void* h) { delete static_cast<Pipe*>(h); }

// out: R, A, C, clique slots, H, S, width, height
void ref_pipe_sizes(void* h, std::uint64_t* out) {
  const Pipe* p = static_cast<Pipe*>(h);
  out[0] = p->graph.num_vertices;
  out[1] = p->graph.neighbors.size();
  out[2] = p->cliques.size();
  out[3] = p->cliques.members.size();
  out[4] = p->hoods.size();
  out[5] = p->hoods.total_slots();
  out[6] = p->image.width;
  out[7] = p->image.height;
}

void ref_pipe_times(void* h, double* out) {
  const Pipe* p = static_cast<Pipe*>(h);
  out[0] = p->t_graph;
  out[1] = p->t_cliques;
  out[2] = p->t_hoods;
}

void ref_pipe_graph(void* h, std::uint32_t* off, std::uint32_t* nbr, double* mean,
                    std::uint32_t* size) {
  const Pipe* p = static_cast<Pipe*>(h);
  std::copy(p->graph.offsets.begin(), p->graph.offsets.end(), off);
  std::copy(p->graph.neighbors.begin(), p->graph.neighbors.end(), nbr);
  std::copy(p->graph.region_mean.begin(), p->graph.region_mean.end(), mean);
  if (size) std::copy(p->graph.region_size.begin(), p->graph.region_size.end(), size);
}

void ref_pipe_cliques(void* h, std::uint32_t* off, std::uint32_t* mem) {
  const Pipe* p = static_cast<Pipe*>(h);
  std::copy(p->cliques.offsets.begin(), p->cliques.offsets.end(), off);
  std::copy(p->cliques.members.begin(), p->cliques.members.end(), mem);
}

void ref_pipe_hoods(void* h, std::uint32_t* off, std::uint32_t* mem, std::uint32_t* src) {
  const Pipe* p = static_cast<Pipe*>(h);
  std::copy(p->hoods.offsets.begin(), p->hoods.offsets.end(), off);
  std::copy(p->hoods.members.begin(), p->hoods.members.end(), mem);
  if (src) std::copy(p->hoods.source_clique.begin(), p->hoods.source_clique.end(), src);
}

void ref_pipe_image(void* h, std::uint8_t* pixels, std::uint8_t* truth, std::uint32_t* region) {
  const Pipe* p = static_cast<Pipe*>(h);
  std::copy(p->image.pixels.begin(), p->image.pixels.end(), pixels);
  if (truth) std::copy(p->truth.pixels.begin(), p->truth.pixels.end(), truth);
  if (region) std::copy(p->map.region.begin(), p->map.region.end(), region);
}

// ---- optimizers ------------------------------------------------------------

// mode 0: dpmrf::optimize itself (reference semantics; M must be 2).
// mode 1: the public-step recomposition (fixed_work and any M allowed).
int ref_optimize(void* h, const RefCfg* cfg, int threads, int mode, int fixed_work,
                 std::uint32_t* labels, double* mu, double* sigma, TraceOut* tr,
                 double* seconds) {
  const Pipe* p = static_cast<Pipe*>(h);
  return guarded([&] {
    const OptimizerConfig c = to_cfg(cfg);
    const auto b = backend_of(threads);
    const auto t0 = std::chrono::steady_clock::now();
    const OptimizeResult r = mode == 0 ? optimize(b, p->graph, p->hoods, c)
                                       : optimize_steps(b, p->graph, p->hoods, c, fixed_work != 0);
    if (seconds) *seconds = secs(t0);
    emit(r, c, p->hoods.size(), labels, mu, sigma, tr);
  });
}

// mode 0: dpmrf::optimize_reference itself; mode 1: its body with the exits
// optional and any M.
int ref_sweep(void* h, const RefCfg* cfg, int mode, int fixed_work, std::uint32_t* labels,
              double* mu, double* sigma, TraceOut* tr, double* seconds) {
  const Pipe* p = static_cast<Pipe*>(h);
  return guarded([&] {
    const OptimizerConfig c = to_cfg(cfg);
    const auto t0 = std::chrono::steady_clock::now();
    const OptimizeResult r = mode == 0 ? optimize_reference(p->graph, p->hoods, c)
                                       : sweep_steps(p->graph, p->hoods, c, fixed_work != 0);
    if (seconds) *seconds = secs(t0);
    emit(r, c, p->hoods.size(), labels, mu, sigma, tr);
  });
}

// ---- step functions (engine.hpp) over raw arrays ---------------------------

int ref_init_random(std::uint32_t M, std::uint32_t R, std::uint64_t seed, double* mu,
                    double* sigma, std::uint32_t* labels) {
  return guarded([&] {
    LabelParams p;
    std::vector<std::uint32_t> l;
    init_random(M, R, seed, p, l);
    std::copy(p.mu.begin(), p.mu.end(), mu);
    std::copy(p.sigma.begin(), p.sigma.end(), sigma);
    std::copy(l.begin(), l.end(), labels);
  });
}

static NeighborhoodSet hoods_of(std::uint64_t H, const std::uint32_t* off, const std::uint32_t* mem) {
  NeighborhoodSet hs;
  hs.offsets.assign(off, off + H + 1);
  hs.members.assign(mem, mem + off[H]);
  for (std::uint32_t i = 0; i < H; ++i) hs.source_clique.push_back(i);
  return hs;
}

int ref_replicate_by_label(std::uint64_t H, const std::uint32_t* off, const std::uint32_t* mem,
                           std::uint32_t M, std::uint32_t* tl, std::uint32_t* oi,
                           std::uint32_t* hid) {
  return guarded([&] {
    const auto rep = replicate_by_label(dpp::Backend::serial(), hoods_of(H, off, mem), M);
    std::copy(rep.test_label.begin(), rep.test_label.end(), tl);
    std::copy(rep.old_index.begin(), rep.old_index.end(), oi);
    std::copy(rep.hood_id.begin(), rep.hood_id.end(), hid);
  });
}

int ref_discord_counts(void* h, const std::uint32_t* labels, std::uint32_t M, std::uint32_t* out) {
  const Pipe* p = static_cast<Pipe*>(h);
  return guarded([&] {
    std::vector<std::uint32_t> l(labels, labels + p->graph.num_vertices);
    const auto d = discord_counts(dpp::Backend::serial(), p->graph, l, M);
    std::copy(d.begin(), d.end(), out);
  });
}

int ref_compute_energies(void* h, std::uint64_t E, const std::uint32_t* tl,
                         const std::uint32_t* oi, const std::uint32_t* hid, std::uint32_t M,
                         const double* mu, const double* sigma, const std::uint32_t* labels,
                         double beta, double* out) {
  const Pipe* p = static_cast<Pipe*>(h);
  return guarded([&] {
    ReplicatedIndex rep;
    rep.test_label.assign(tl, tl + E);
    rep.old_index.assign(oi, oi + E);
    rep.hood_id.assign(hid, hid + E);
    LabelParams prm;
    prm.mu.assign(mu, mu + M);
    prm.sigma.assign(sigma, sigma + M);
    std::vector<std::uint32_t> l(labels, labels + p->graph.num_vertices);
    const auto e = compute_energies(dpp::Backend::serial(), p->graph, p->hoods, rep, prm, l, beta);
    std::copy(e.begin(), e.end(), out);
  });
}

int ref_min_label_energies(std::uint64_t E, const std::uint32_t* tl, const std::uint32_t* oi,
                           const double* energies, std::uint64_t num_slots, double* out_e,
                           std::uint32_t* out_l) {
  return guarded([&] {
    ReplicatedIndex rep;
    rep.test_label.assign(tl, tl + E);
    rep.old_index.assign(oi, oi + E);
    rep.hood_id.assign(E, 0);
    const auto m = min_label_energies(dpp::Backend::serial(), rep,
                                      std::vector<double>(energies, energies + E), num_slots);
    std::copy(m.energy.begin(), m.energy.end(), out_e);
    std::copy(m.label.begin(), m.label.end(), out_l);
  });
}

int ref_neighborhood_energy_sums(std::uint64_t S, const std::uint32_t* slot_hood,
                                 const double* mins, double* out, std::uint64_t* n_out) {
  return guarded([&] {
    const auto s = neighborhood_energy_sums(dpp::Backend::serial(),
                                            std::vector<std::uint32_t>(slot_hood, slot_hood + S),
                                            std::vector<double>(mins, mins + S));
    std::copy(s.begin(), s.end(), out);
    *n_out = s.size();
  });
}

int ref_check_convergence(std::uint64_t rows, std::uint64_t series, const double* hist,
                          int window, double tol, std::uint8_t* out, std::uint64_t* n_out) {
  return guarded([&] {
    std::vector<std::vector<double>> h(rows);
    for (std::uint64_t r = 0; r < rows; ++r) h[r].assign(hist + r * series, hist + (r + 1) * series);
    const auto f = check_convergence(dpp::Backend::serial(), h, window, tol);
    std::copy(f.begin(), f.end(), out);
    *n_out = f.size();
  });
}

int ref_update_labels(std::uint64_t H, const std::uint32_t* off, const std::uint32_t* mem,
                      const std::uint32_t* argmin, std::uint32_t R, const std::uint32_t* old_l,
                      std::uint32_t* out) {
  return guarded([&] {
    const auto hs = hoods_of(H, off, mem);
    const auto r = update_labels(dpp::Backend::serial(), hs,
                                 std::vector<std::uint32_t>(argmin, argmin + hs.total_slots()),
                                 std::vector<std::uint32_t>(old_l, old_l + R));
    std::copy(r.begin(), r.end(), out);
  });
}

int ref_update_parameters(std::uint32_t R, const double* mean, const std::uint32_t* labels,
                          std::uint32_t M, const double* pmu, const double* psig, double* mu,
                          double* sigma) {
  return guarded([&] {
    RegionGraph g;
    g.num_vertices = R;
    g.offsets.assign(R + 1, 0);
    g.region_mean.assign(mean, mean + R);
    g.region_size.assign(R, 1);
    LabelParams prev;
    prev.mu.assign(pmu, pmu + M);
    prev.sigma.assign(psig, psig + M);
    const auto p = update_parameters(dpp::Backend::serial(), g,
                                     std::vector<std::uint32_t>(labels, labels + R), prev);
    std::copy(p.mu.begin(), p.mu.end(), mu);
    std::copy(p.sigma.begin(), p.sigma.end(), sigma);
  });
}

double ref_reduce_add(std::uint64_t n, const double* x) {
  return dpp::reduce(dpp::Backend::serial(), std::vector<double>(x, x + n), std::plus<double>{},
                     0.0);
}

std::uint32_t ref_hw_threads() { return std::max(1u, std::thread::hardware_concurrency()); }

// dpmrf::confusion (metrics.cpp:8-14) on two BinaryImages (w x h pixels each).
int ref_confusion(std::uint32_t w1, std::uint32_t h1, const std::uint8_t* pred, std::uint32_t w2,
                  std::uint32_t h2, const std::uint8_t* truth, std::uint64_t* counts) {
  return guarded([&] {
    BinaryImage a, b;
    a.width = w1;
    a.height = h1;
    a.pixels.assign(pred, pred + std::size_t(w1) * h1);
    b.width = w2;
    b.height = h2;
    b.pixels.assign(truth, truth + std::size_t(w2) * h2);
    const ConfusionCounts c = confusion(a, b);
    counts[0] = c.tp;
    counts[1] = c.tn;
    counts[2] = c.fp;
    counts[3] = c.fn;
  });
}

void ref_compute_metrics(const std::uint64_t* counts, double* out, int* defined) {
  ConfusionCounts c;
  c.tp = counts[0];
  c.tn = counts[1];
  c.fp = counts[2];
  c.fn = counts[3];
  const Metrics m = compute_metrics(c);
  out[0] = m.precision;
  out[1] = m.recall;
  out[2] = m.accuracy;
  defined[0] = m.precision_defined;
  defined[1] = m.recall_defined;
}

// dpmrf::validate_label_map (label_map.cpp:38-78); msg receives what() on failure.
int ref_validate_label_map(std::uint32_t w, std::uint32_t h, const std::uint32_t* region,
                           std::uint64_t n, std::uint32_t* num_regions, char* msg,
                           std::uint64_t msg_len) {
  std::string what;
  const int rc = guarded([&] {
    LabelMap m;
    m.width = w;
    m.height = h;
    m.region.assign(region, region + n);
    try {
      validate_label_map(m);
    } catch (const std::exception& e) {
      what = e.what();
      throw;
    }
    *num_regions = m.num_regions;
  });
  if (msg && msg_len) {
    std::strncpy(msg, what.c_str(), msg_len - 1);
    msg[msg_len - 1] = 0;
  }
  return rc;
}

double ref_porosity(std::uint32_t w, std::uint32_t h, const std::uint8_t* px) {
  BinaryImage a;
  a.width = w;
  a.height = h;
  a.pixels.assign(px, px + std::size_t(w) * h);
  return porosity(a);
}

}  // extern "C"
