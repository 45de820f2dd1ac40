// inputs.cpp -- synthetic inputs of the optimization phase (host, C++).
//
// Not part of the hot path: these build the region graph and maximal
// cliques the optimization consumes ("same region-adjacency graph and
// maximal-clique input", BASELINE.json north_star), with the reference's
// semantics so that the GPU path sees exactly the reference's inputs:
//   gen_phantom / corrupt   proj/src/eval/phantom.cpp:54-150
//   grid_oversegment        proj/src/graph/label_map.cpp:79-94
//   brick layout            SURVEY.md §8(d) config C (rows of height b,
//                           odd rows shifted by b/2, ids first-seen row-major)
//   build_region_graph      proj/src/graph/region_graph.cpp:10-73
//   maximal cliques         proj/src/graph/cliques.cpp:53-106 (same output:
//                           every maximal clique ascending, cliques in
//                           lexicographic order)
// Compiled with -ffp-contract=off so the phantom arithmetic matches.
// Multi-threaded with std::thread where the work is per pixel / per vertex.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <new>
#include <thread>
#include <unordered_map>
#include <vector>

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kRingAmplitude = 15.0;

uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t next_u64(uint64_t& s) { return mix64(s += 0x9E3779B97F4A7C15ull); }
double next_unit(uint64_t& s) { return static_cast<double>(next_u64(s) >> 11) * 0x1.0p-53; }
uint64_t pixel_draw(uint64_t seed, uint64_t px, uint64_t k) {
  return mix64(seed + 0x9E3779B97F4A7C15ull * (px * 8 + k + 1));
}

unsigned workers() {
  const unsigned n = std::thread::hardware_concurrency();
  return n ? std::min(n, 64u) : 1u;
}

void parallel_for(uint64_t n, const std::function<void(uint64_t, uint64_t)>& fn) {
  const unsigned T = workers();
  if (n < 4096 || T == 1) {
    fn(0, n);
    return;
  }
  std::vector<std::thread> th;
  const uint64_t chunk = (n + T - 1) / T;
  for (unsigned t = 0; t < T; ++t) {
    const uint64_t b = t * chunk, e = std::min(n, b + chunk);
    if (b >= e) break;
    th.emplace_back(fn, b, e);
  }
  for (auto& x : th) x.join();
}

struct Graph {
  std::vector<uint32_t> off, nbr, size;
  std::vector<double> mean;
};
struct Cliques {
  std::vector<uint32_t> off, mem;
};

}  // namespace

extern "C" {

// Returns 0, or 1 for an invalid spec (InputError in the reference).
int dpmrf_in_phantom(uint32_t w, uint32_t h, double pore_fraction, uint64_t seed,
                     uint8_t* truth, uint8_t* clean) {
  if (w == 0 || h == 0 || !(pore_fraction >= 0.0 && pore_fraction < 1.0)) return 1;
  const uint64_t n = uint64_t(w) * h;
  std::memset(truth, 0, n);
  const auto target = static_cast<uint64_t>(pore_fraction * static_cast<double>(n));
  const double r_max = std::max(2.0, std::min(w, h) / 3.0);
  uint64_t state = seed;
  uint64_t pore = 0;
  for (int guard = 0; pore < target && guard < 100000; ++guard) {
    const double deficit = static_cast<double>(target - pore);
    const double r = std::clamp(std::sqrt(deficit / kPi), 2.0, r_max);
    const double cx = next_unit(state) * w;
    const double cy = next_unit(state) * h;
    const auto y0 = static_cast<int64_t>(std::floor(cy - r));
    const auto y1 = static_cast<int64_t>(std::ceil(cy + r));
    const auto x0 = static_cast<int64_t>(std::floor(cx - r));
    const auto x1 = static_cast<int64_t>(std::ceil(cx + r));
    for (int64_t y = std::max<int64_t>(0, y0); y <= y1 && y < h; ++y)
      for (int64_t x = std::max<int64_t>(0, x0); x <= x1 && x < w; ++x) {
        const double dx = (x + 0.5) - cx;
        const double dy = (y + 0.5) - cy;
        if (dx * dx + dy * dy > r * r) continue;
        uint8_t& px = truth[uint64_t(y) * w + x];
        if (!px) {
          px = 1;
          ++pore;
        }
      }
  }
  for (uint64_t i = 0; i < n; ++i) clean[i] = truth[i] ? 50 : 200;
  return 0;
}

int dpmrf_in_corrupt(const uint8_t* clean, uint32_t w, uint32_t h, double sp_rate,
                     double gauss_sigma, int ringing, uint64_t seed, uint8_t* out) {
  if (w == 0 || h == 0 || !(sp_rate >= 0.0 && sp_rate <= 1.0) || !(gauss_sigma >= 0.0)) return 1;
  const uint64_t n = uint64_t(w) * h;
  const double half_sp = sp_rate / 2.0;
  const double wavelength = std::max(1.0, std::min(w, h) / 4.0);
  uint64_t phase_state = seed ^ 0xA5A5A5A5A5A5A5A5ull;
  const double phase = 2.0 * kPi * next_unit(phase_state);
  const double cx = w / 2.0, cy = h / 2.0;
  parallel_for(n, [&](uint64_t b, uint64_t e) {
    for (uint64_t i = b; i < e; ++i) {
      double val = clean[i];
      if (sp_rate > 0.0) {
        const double u = static_cast<double>(pixel_draw(seed, i, 0) >> 11) * 0x1.0p-53;
        if (u < half_sp)
          val = 0.0;
        else if (u < sp_rate)
          val = 255.0;
      }
      if (gauss_sigma > 0.0) {
        const double u1 = static_cast<double>((pixel_draw(seed, i, 1) >> 11) + 1) * 0x1.0p-53;
        const double u2 = static_cast<double>(pixel_draw(seed, i, 2) >> 11) * 0x1.0p-53;
        val += gauss_sigma * std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * kPi * u2);
      }
      if (ringing) {
        const double dx = (i % w + 0.5) - cx;
        const double dy = (i / w + 0.5) - cy;
        const double radius = std::sqrt(dx * dx + dy * dy);
        val += kRingAmplitude * std::sin(2.0 * kPi * radius / wavelength + phase);
      }
      val = std::clamp(val, 0.0, 255.0);
      out[i] = static_cast<uint8_t>(std::lround(val));
    }
  });
  return 0;
}

// Returns the region count (0 on invalid input).
uint32_t dpmrf_in_grid_oversegment(uint32_t w, uint32_t h, uint32_t b, uint32_t* region) {
  if (b == 0 || w == 0 || h == 0) return 0;
  const uint32_t bx = (w + b - 1) / b, by = (h + b - 1) / b;
  parallel_for(h, [&](uint64_t y0, uint64_t y1) {
    for (uint64_t y = y0; y < y1; ++y)
      for (uint32_t x = 0; x < w; ++x) region[y * w + x] = uint32_t(y / b) * bx + (x / b);
  });
  return bx * by;
}

uint32_t dpmrf_in_brick_oversegment(uint32_t w, uint32_t h, uint32_t b, uint32_t* region) {
  if (b == 0 || w == 0 || h == 0) return 0;
  // block row r covers rows [r*b, r*b+b); odd rows are shifted by b/2, so
  // column keys are (x + shift) / b; ids are assigned first-seen row-major,
  // i.e. block row by block row, left to right.
  uint32_t next = 0;
  std::vector<uint32_t> row_ids;
  for (uint32_t r = 0; uint64_t(r) * b < h; ++r) {
    const uint32_t shift = (r & 1u) ? b / 2 : 0;
    const uint32_t ncols = (w - 1 + shift) / b + 1;
    row_ids.assign(ncols, 0);
    for (uint32_t c = 0; c < ncols; ++c) row_ids[c] = next + c;
    next += ncols;
    for (uint32_t y = r * b; y < std::min<uint64_t>(h, uint64_t(r) * b + b); ++y)
      for (uint32_t x = 0; x < w; ++x) region[uint64_t(y) * w + x] = row_ids[(x + shift) / b];
  }
  return next;
}

// Region adjacency graph with the reference's CSR + means.  Returns an
// opaque handle (nullptr on invalid region ids).
void* dpmrf_in_region_graph(uint32_t w, uint32_t h, const uint8_t* pixels, const uint32_t* region,
                            uint32_t R, uint64_t* num_adj) {
  const uint64_t n = uint64_t(w) * h;
  auto* g = new (std::nothrow) Graph;
  if (!g) return nullptr;
  const unsigned T = workers();
  std::vector<std::vector<uint64_t>> parts(T);
  const uint64_t rows_per = (h + T - 1) / T;
  std::vector<std::thread> th;
  for (unsigned t = 0; t < T; ++t) {
    th.emplace_back([&, t] {
      auto& out = parts[t];
      const uint64_t y0 = t * rows_per, y1 = std::min<uint64_t>(h, y0 + rows_per);
      for (uint64_t y = y0; y < y1; ++y)
        for (uint32_t x = 0; x < w; ++x) {
          const uint64_t i = y * w + x;
          const uint32_t a = region[i];
          if (x + 1 < w) {
            const uint32_t b = region[i + 1];
            // skip repeats of the same pair along a vertical boundary run
            if (a != b && !(y > 0 && region[i - w] == a && region[i - w + 1] == b)) {
              out.push_back((uint64_t(a) << 32) | b);
              out.push_back((uint64_t(b) << 32) | a);
            }
          }
          if (y + 1 < h) {
            const uint32_t b = region[i + w];
            if (a != b && !(x > 0 && region[i - 1] == a && region[i - 1 + w] == b)) {
              out.push_back((uint64_t(a) << 32) | b);
              out.push_back((uint64_t(b) << 32) | a);
            }
          }
        }
      std::sort(out.begin(), out.end());
      out.erase(std::unique(out.begin(), out.end()), out.end());
    });
  }
  for (auto& x : th) x.join();
  std::vector<uint64_t> all;
  size_t tot = 0;
  for (auto& p : parts) tot += p.size();
  all.reserve(tot);
  for (auto& p : parts) {
    all.insert(all.end(), p.begin(), p.end());
    std::vector<uint64_t>().swap(p);
  }
  std::sort(all.begin(), all.end());
  all.erase(std::unique(all.begin(), all.end()), all.end());
  g->off.assign(uint64_t(R) + 1, 0);
  g->nbr.resize(all.size());
  for (size_t k = 0; k < all.size(); ++k) {
    const uint32_t a = uint32_t(all[k] >> 32);
    if (a >= R) {
      delete g;
      return nullptr;
    }
    g->off[a + 1]++;
    g->nbr[k] = static_cast<uint32_t>(all[k]);
  }
  for (uint32_t v = 0; v < R; ++v) g->off[v + 1] += g->off[v];
  // integer sums divided once (region_graph.cpp:58-71)
  std::vector<uint64_t> sums(R, 0);
  g->size.assign(R, 0);
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t r = region[i];
    if (r >= R) {
      delete g;
      return nullptr;
    }
    sums[r] += pixels[i];
    g->size[r]++;
  }
  g->mean.resize(R);
  for (uint32_t r = 0; r < R; ++r)
    g->mean[r] = static_cast<double>(sums[r]) / static_cast<double>(g->size[r]);
  *num_adj = g->nbr.size();
  return g;
}

void dpmrf_in_graph_arrays(void* hg, uint32_t* off, uint32_t* nbr, double* mean, uint32_t* size) {
  const Graph* g = static_cast<Graph*>(hg);
  std::copy(g->off.begin(), g->off.end(), off);
  std::copy(g->nbr.begin(), g->nbr.end(), nbr);
  std::copy(g->mean.begin(), g->mean.end(), mean);
  if (size) std::copy(g->size.begin(), g->size.end(), size);
}

void dpmrf_in_graph_free(void* hg) { delete static_cast<Graph*>(hg); }

// All maximal cliques by depth-first lexicographic extension from each
// vertex (the reference's breadth-first extension visited in DFS order):
// a clique is emitted when no vertex is adjacent to all its members;
// children extend by common neighbors above the last member, in ascending
// order, so per-vertex output is already lexicographic and vertex blocks
// concatenate in order.
void* dpmrf_in_maximal_cliques(uint32_t R, const uint32_t* off, const uint32_t* nbr,
                               uint64_t* num_cliques, uint64_t* num_members) {
  auto* out = new (std::nothrow) Cliques;
  if (!out) return nullptr;
  const unsigned T = workers();
  const uint64_t per = (uint64_t(R) + T - 1) / T;
  std::vector<Cliques> parts(T);
  std::vector<std::thread> th;
  for (unsigned t = 0; t < T; ++t) {
    th.emplace_back([&, t] {
      Cliques& p = parts[t];
      p.off.push_back(0);
      std::vector<uint32_t> clique;
      std::vector<std::vector<uint32_t>> common_stack;
      std::function<void(const std::vector<uint32_t>&)> rec = [&](const std::vector<uint32_t>& common) {
        if (common.empty()) {
          p.mem.insert(p.mem.end(), clique.begin(), clique.end());
          p.off.push_back(static_cast<uint32_t>(p.mem.size()));
          return;
        }
        const uint32_t last = clique.back();
        for (uint32_t u : common) {
          if (u <= last) continue;
          std::vector<uint32_t> next;
          std::set_intersection(common.begin(), common.end(), nbr + off[u], nbr + off[u + 1],
                                std::back_inserter(next));
          clique.push_back(u);
          rec(next);
          clique.pop_back();
        }
      };
      const uint64_t v0 = t * per, v1 = std::min<uint64_t>(R, v0 + per);
      for (uint64_t v = v0; v < v1; ++v) {
        clique.assign(1, static_cast<uint32_t>(v));
        rec(std::vector<uint32_t>(nbr + off[v], nbr + off[v + 1]));
      }
    });
  }
  for (auto& x : th) x.join();
  out->off.push_back(0);
  for (auto& p : parts) {
    const uint32_t base = static_cast<uint32_t>(out->mem.size());
    out->mem.insert(out->mem.end(), p.mem.begin(), p.mem.end());
    for (size_t i = 1; i < p.off.size(); ++i) out->off.push_back(base + p.off[i]);
  }
  *num_cliques = out->off.size() - 1;
  *num_members = out->mem.size();
  return out;
}

void dpmrf_in_clique_arrays(void* hc, uint32_t* off, uint32_t* mem) {
  const Cliques* c = static_cast<Cliques*>(hc);
  std::copy(c->off.begin(), c->off.end(), off);
  std::copy(c->mem.begin(), c->mem.end(), mem);
}

void dpmrf_in_cliques_free(void* hc) { delete static_cast<Cliques*>(hc); }

}  // extern "C"
