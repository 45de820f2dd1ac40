// drop_in_test.cpp -- the reference's engine test cases, written against the
// C++ drop-in (include/dpmrf_b200/engine.hpp) and run on the B200.
// Mirrors proj/tests/mrf_engine_test.cpp and proj/tests/optimize_test.cpp
// (plain asserts: doctest is not vendored in the reference checkout).
#include <cstdio>
#include <cstdlib>
#include <set>
#include <utility>
#include <vector>

#include "dpmrf_b200/engine.hpp"

using namespace dpmrf_b200;

static int failures = 0;
#define CHECK(c)                                                      \
  do {                                                                \
    if (!(c)) {                                                       \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++failures;                                                     \
    }                                                                 \
  } while (0)
#define CHECK_THROWS_AS(expr, T)   \
  do {                             \
    bool thrown = false;           \
    try {                          \
      (void)(expr);                \
    } catch (const T&) {           \
      thrown = true;               \
    } catch (...) {                \
    }                              \
    CHECK(thrown);                 \
  } while (0)

static RegionGraph make_graph(std::uint32_t n,
                              const std::vector<std::pair<std::uint32_t, std::uint32_t>>& edges,
                              std::vector<double> means = {}) {
  std::vector<std::set<std::uint32_t>> adj(n);
  for (auto [a, b] : edges) {
    adj[a].insert(b);
    adj[b].insert(a);
  }
  RegionGraph g;
  g.num_vertices = n;
  g.offsets.push_back(0);
  for (std::uint32_t v = 0; v < n; ++v) {
    for (auto u : adj[v]) g.neighbors.push_back(u);
    g.offsets.push_back(static_cast<std::uint32_t>(g.neighbors.size()));
    g.region_mean.push_back(means.empty() ? 128.0 : means[v]);
    g.region_size.push_back(1);
  }
  return g;
}

static NeighborhoodSet make_hoods(std::vector<std::uint32_t> off, std::vector<std::uint32_t> mem) {
  NeighborhoodSet h;
  h.offsets = std::move(off);
  h.members = std::move(mem);
  for (std::uint32_t i = 0; i + 1 < h.offsets.size(); ++i) h.source_clique.push_back(i);
  return h;
}

int main() {
  const auto B = dpp::Backend::cuda(0);
  using V = std::vector<std::uint32_t>;

  // mrf_engine_test.cpp:132-145
  const auto worked = make_hoods({0, 4, 7}, {0, 1, 2, 5, 1, 3, 4});
  const auto rep = replicate_by_label(B, worked, 2);
  CHECK((rep.test_label == V{0, 0, 0, 0, 1, 1, 1, 1, 0, 0, 0, 1, 1, 1}));
  CHECK((rep.old_index == V{0, 1, 2, 3, 0, 1, 2, 3, 4, 5, 6, 4, 5, 6}));
  CHECK((rep.hood_id == V{0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 1}));
  CHECK((slot_hood_map(B, worked) == V{0, 0, 0, 0, 1, 1, 1}));

  // mrf_engine_test.cpp:186-190
  const auto g4 = make_graph(4, {{0, 1}, {0, 2}, {1, 2}, {2, 3}});
  CHECK((discord_counts(B, g4, {0, 1, 1, 0}, 2) == V{2, 1, 1, 1, 0, 1, 2, 0}));

  // mrf_engine_test.cpp:204-239
  {
    const auto g = make_graph(1, {}, {30.0});
    const auto h = make_hoods({0, 1}, {0});
    LabelParams p{{30.0, 100.0}, {1.0, 7.0}};
    CHECK(compute_energies(B, g, h, replicate_by_label(B, h, 2), p, {0}, 1.0)[0] == 0.0);
  }
  {
    const auto g = make_graph(1, {}, {40.0});
    const auto h = make_hoods({0, 1}, {0});
    LabelParams p{{30.0, 200.0}, {1.0, 1.0}};
    CHECK(compute_energies(B, g, h, replicate_by_label(B, h, 2), p, {0}, 0.0)[0] == 50.0);
  }
  {
    const auto g = make_graph(3, {{0, 1}, {0, 2}, {1, 2}}, {30.0, 30.0, 30.0});
    const auto h = make_hoods({0, 3}, {0, 1, 2});
    LabelParams p{{30.0, 99.0}, {1.0, 1.0}};
    CHECK(compute_energies(B, g, h, replicate_by_label(B, h, 2), p, {0, 1, 1}, 1.0)[0] == 2.0);
  }

  // mrf_engine_test.cpp:263-288
  {
    const auto h = make_hoods({0, 1}, {0});
    const auto r = replicate_by_label(B, h, 2);
    auto m = min_label_energies(B, r, {2.0, 5.0}, 1);
    CHECK(m.energy[0] == 2.0 && m.label[0] == 0);
    m = min_label_energies(B, r, {5.0, 2.0}, 1);
    CHECK(m.energy[0] == 2.0 && m.label[0] == 1);
    m = min_label_energies(B, r, {3.0, 3.0}, 1);
    CHECK(m.energy[0] == 3.0 && m.label[0] == 0);
    const auto mins = min_label_energies(B, rep, {1, 4, 2, 9, 0, 5, 3, 8, 6, 2, 7, 5, 1, 9}, 7);
    CHECK((mins.energy == std::vector<double>{0, 4, 2, 8, 5, 1, 7}));
    CHECK((mins.label == V{1, 0, 0, 1, 1, 1, 0}));
  }

  // mrf_engine_test.cpp:308-367
  CHECK((neighborhood_energy_sums(B, {0, 0, 0, 0, 1, 1, 1}, {0, 4, 2, 8, 1, 2, 7}) ==
         std::vector<double>{14.0, 10.0}));
  CHECK((check_convergence(B, {{5.0}, {5.0}, {5.0}, {5.0}}, 3, 1e-4) == std::vector<std::uint8_t>{1}));
  CHECK((check_convergence(B, {{5.0}, {5.1}, {5.0}, {5.0}}, 3, 1e-4) == std::vector<std::uint8_t>{0}));
  CHECK(check_convergence(B, {}, 3, 1e-4).empty());

  // mrf_engine_test.cpp:369-417
  CHECK((update_labels(B, worked, {0, 0, 1, 1, 1, 0, 0}, V(6, 1)) == V{0, 0, 1, 0, 0, 1}));
  CHECK((update_labels(B, make_hoods({0, 1}, {2}), {1}, {0, 0, 0, 0}) == V{0, 0, 1, 0}));
  {
    const auto g = make_graph(3, {}, {10.0, 20.0, 99.0});
    const auto p = update_parameters(B, g, {0, 0, 1}, LabelParams{{0.0, 0.0}, {1.0, 1.0}});
    CHECK((p.mu == std::vector<double>{15.0, 99.0}));
    CHECK((p.sigma == std::vector<double>{5.0, kSigmaFloor}));
    CHECK_THROWS_AS(update_parameters(B, g, {0, 2, 1}, LabelParams{{0.0, 0.0}, {1.0, 1.0}}),
                    std::invalid_argument);
  }

  // optimize_test.cpp:83-103 -- 4x4 blocks of a two-intensity image
  {
    std::vector<std::pair<std::uint32_t, std::uint32_t>> edges;
    std::vector<double> means;
    for (std::uint32_t r = 0; r < 4; ++r)
      for (std::uint32_t c = 0; c < 4; ++c) {
        if (c + 1 < 4) edges.push_back({r * 4 + c, r * 4 + c + 1});
        if (r + 1 < 4) edges.push_back({r * 4 + c, (r + 1) * 4 + c});
        means.push_back(c < 2 ? 50.0 : 200.0);
      }
    const auto g = make_graph(16, edges, means);
    CliqueSet cl;
    cl.offsets.push_back(0);
    std::set<std::pair<std::uint32_t, std::uint32_t>> sorted(edges.begin(), edges.end());
    for (auto [a, b] : sorted) {
      cl.members.push_back(a);
      cl.members.push_back(b);
      cl.offsets.push_back(static_cast<std::uint32_t>(cl.members.size()));
    }
    const auto hoods = build_neighborhoods(B, g, cl);
    OptimizerConfig cfg;
    cfg.rng_seed = 7;
    const auto res = optimize(B, g, hoods, cfg);
    const std::uint32_t lo = res.labels[0];
    for (std::uint32_t v = 0; v < 16; ++v) CHECK(res.labels[v] == (means[v] == 50.0 ? lo : 1 - lo));
    CHECK(res.params.mu[lo] == 50.0 && res.params.mu[1 - lo] == 200.0);
    CHECK(res.params.sigma[0] == kSigmaFloor && res.params.sigma[1] == kSigmaFloor);
    CHECK(!res.trace.empty() && res.trace.size() <= 20);
    // optimize_test.cpp:199-245 -- invalid configurations
    OptimizerConfig bad = cfg;
    bad.num_labels = 3;
    CHECK_THROWS_AS(optimize(B, g, hoods, bad), InputError);
    bad = cfg;
    bad.convergence_window = bad.map_max_iters;
    CHECK_THROWS_AS(optimize(B, g, hoods, bad), InputError);
    bad = cfg;
    bad.convergence_tol = 0.0;
    CHECK_THROWS_AS(optimize(B, g, hoods, bad), InputError);
    CHECK_THROWS_AS(build_neighborhoods(B, g, cl, 2), InputError);
  }
  {
    // graph_test.cpp:215-223 -- a 2x2 block grid is the 4-cycle
    GrayImage img;
    img.width = img.height = 4;
    for (std::uint32_t i = 0; i < 16; ++i) img.pixels.push_back(static_cast<std::uint8_t>(i * 13));
    LabelMap lm;
    lm.width = lm.height = 4;
    lm.num_regions = 4;
    for (std::uint32_t y = 0; y < 4; ++y)
      for (std::uint32_t x = 0; x < 4; ++x) lm.region.push_back((y / 2) * 2 + x / 2);
    // graph_test.cpp:160-190 -- validation
    LabelMap v = lm;
    v.num_regions = 0;
    validate_label_map(v, B);
    CHECK(v.num_regions == 4);
    auto lm_of = [](std::uint32_t w, std::uint32_t h, V r) {
      LabelMap m;
      m.width = w;
      m.height = h;
      m.region = std::move(r);
      return m;
    };
    LabelMap ok = lm_of(2, 2, {0, 0, 1, 1});
    validate_label_map(ok, B);
    CHECK(ok.num_regions == 2);
    LabelMap gap = lm_of(2, 1, {0, 2}), split = lm_of(3, 1, {0, 1, 0});
    LabelMap diag = lm_of(2, 2, {0, 1, 1, 0}), shortm = lm_of(2, 2, {0, 0, 0});
    CHECK_THROWS_AS(validate_label_map(gap, B), InputError);
    CHECK_THROWS_AS(validate_label_map(split, B), InputError);
    CHECK_THROWS_AS(validate_label_map(diag, B), InputError);
    CHECK_THROWS_AS(validate_label_map(shortm, B), InputError);
    const auto rg = build_region_graph(B, img, lm);
    CHECK(rg.num_vertices == 4);
    CHECK((rg.offsets == V{0, 2, 4, 6, 8}));
    CHECK((rg.neighbors == V{1, 2, 0, 3, 0, 3, 1, 2}));
    CHECK((rg.region_size == V{4, 4, 4, 4}));
    // graph_test.cpp:225-233 -- uniform image: exact means
    GrayImage flat = img;
    flat.pixels.assign(16, 77);
    for (double m : build_region_graph(B, flat, lm).region_mean) CHECK(m == 77.0);
    LabelMap bad = lm;
    bad.width = 2;
    CHECK_THROWS_AS(build_region_graph(B, img, bad), InputError);
    // the 4-cycle's maximal cliques are its edges, in lexicographic order
    const auto cq = enumerate_maximal_cliques(B, rg);
    CHECK((cq.offsets == V{0, 2, 4, 6, 8}));
    CHECK((cq.members == V{0, 1, 0, 2, 1, 3, 2, 3}));
    // K4 plus a pendant vertex: {0,1,2,3} and {3,4} (cliques_test.cpp style)
    const auto k4 = make_graph(5, {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}, {3, 4}});
    const auto ck = enumerate_maximal_cliques(B, k4);
    CHECK((ck.offsets == V{0, 4, 6}));
    CHECK((ck.members == V{0, 1, 2, 3, 3, 4}));
  }
  {
    // eval_test.cpp:149-210 -- confusion and metrics
    auto bin = [](std::uint32_t w, std::uint32_t h, std::vector<std::uint8_t> px) {
      BinaryImage b;
      b.width = w;
      b.height = h;
      b.pixels = std::move(px);
      return b;
    };
    const auto truth = bin(4, 1, {1, 1, 0, 0});
    const auto c = confusion(bin(4, 1, {1, 0, 0, 1}), truth, B);
    CHECK(c.tp == 1 && c.fn == 1 && c.tn == 1 && c.fp == 1);
    const auto perfect = confusion(truth, truth, B);
    CHECK(perfect.tp == 2 && perfect.tn == 2 && perfect.fp == 0 && perfect.fn == 0);
    const auto inv = confusion(bin(4, 1, {0, 0, 1, 1}), truth, B);
    CHECK(inv.tp == 0 && inv.tn == 0 && inv.fp == 2 && inv.fn == 2);
    CHECK_THROWS_AS(confusion(truth, bin(2, 2, {1, 1, 0, 0}), B), InputError);
    const auto m = compute_metrics(c);
    CHECK(m.precision == 0.5 && m.recall == 0.5 && m.accuracy == 0.5);
    ConfusionCounts none;
    none.tn = 3;
    const auto mn = compute_metrics(none);
    CHECK(!mn.precision_defined && !mn.recall_defined && mn.accuracy == 1.0);
    CHECK(porosity(truth) == 0.5);
  }
  if (failures) {
    std::fprintf(stderr, "%d check(s) failed\n", failures);
    return 1;
  }
  std::printf("drop-in C++ tests passed\n");
  return 0;
}
