// dpmrf -- the reference's command-line tool (proj/tools/main.cpp) over the
// reference library with the Cuda backend patched in
// (integration/cuda_backend.patch).  Same subcommands, flags, output lines
// and exit codes (0 ok, 2 usage / InputError, 1 anything else,
// main.cpp:240-251), with one addition: `--backend cuda [--device N]` runs
// build_region_graph, enumerate_maximal_cliques, build_neighborhoods and
// optimize on the GPU (the `segment:` summary line is unchanged), and
// `bench --cuda` appends one `cuda` CSV row per repeat after the reference's
// own rows (harness.cpp:46-86 schema, wall_s = optimization phase only,
// speedup = the reference row's wall_s / this row's).
//
// The reference parses its flags with CLI11, which is absent here (its
// vendor/ copy is git-ignored upstream); this file has its own small parser.
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "dpmrf/bench/harness.hpp"
#include "dpmrf/dpp/backend.hpp"
#include "dpmrf/error.hpp"
#include "dpmrf/eval/metrics.hpp"
#include "dpmrf/eval/phantom.hpp"
#include "dpmrf/graph/cliques.hpp"
#include "dpmrf/graph/label_map.hpp"
#include "dpmrf/graph/neighborhoods.hpp"
#include "dpmrf/graph/region_graph.hpp"
#include "dpmrf/mrf/engine.hpp"
#include "dpmrf/simd/dispatch.hpp"

namespace {

using Clock = std::chrono::steady_clock;

double seconds(Clock::time_point from, Clock::time_point to) {
  return std::chrono::duration<double>(to - from).count();
}

// A usage error: the reference's CLI::ParseError (exit 2).
struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// --name value / --flag parser for one subcommand.
class Args {
 public:
  Args(int argc, char** argv, int first, const std::set<std::string>& options,
       const std::set<std::string>& flags) {
    for (int i = first; i < argc; ++i) {
      const std::string a = argv[i];
      if (flags.count(a)) {
        flags_.insert(a);
      } else if (options.count(a)) {
        if (i + 1 >= argc) throw UsageError(a + " requires an argument");
        values_[a] = argv[++i];
      } else {
        throw UsageError("unexpected argument " + a);
      }
    }
  }
  bool flag(const std::string& name) const { return flags_.count(name) != 0; }
  bool has(const std::string& name) const { return values_.count(name) != 0; }
  std::string str(const std::string& name, const std::string& dflt = "") const {
    auto it = values_.find(name);
    return it == values_.end() ? dflt : it->second;
  }
  std::string required(const std::string& name) const {
    if (!has(name)) throw UsageError(name + " is required");
    return str(name);
  }
  template <class T>
  T num(const std::string& name, T dflt) const {
    if (!has(name)) return dflt;
    std::istringstream in(str(name));
    T v{};
    in >> v;
    if (!in || !in.eof()) throw UsageError(name + ": invalid value " + str(name));
    return v;
  }

 private:
  std::map<std::string, std::string> values_;
  std::set<std::string> flags_;
};

const std::set<std::string> kExecOptions = {"--backend", "--threads", "--chunk", "--simd",
                                            "--device"};
const std::set<std::string> kConfigOptions = {"--seed", "--beta",   "--em-iters",
                                              "--map-iters", "--window", "--tol"};

std::set<std::string> join(std::set<std::string> a, const std::set<std::string>& b) {
  a.insert(b.begin(), b.end());
  return a;
}

// main.cpp:36-58, plus the Cuda kind.
dpmrf::dpp::Backend make_backend(const Args& a) {
  const std::string backend = a.str("--backend", "serial");
  const std::string simd = a.str("--simd", "auto");
  if (backend != "serial" && backend != "threaded" && backend != "cuda")
    throw UsageError("--backend: " + backend + " not in {serial,threaded,cuda}");
  if (simd != "auto" && simd != "scalar" && simd != "avx2")
    throw UsageError("--simd: " + simd + " not in {auto,scalar,avx2}");
  if (simd == "scalar") {
    dpmrf::simd::set_override(dpmrf::simd::Level::Scalar);
  } else if (simd == "avx2") {
    dpmrf::simd::set_override(dpmrf::simd::Level::Avx2);
  } else {
    dpmrf::simd::clear_override();
  }
  if (backend == "cuda") return dpmrf::dpp::Backend::cuda(a.num<unsigned>("--device", 0));
  if (backend == "threaded")
    return dpmrf::dpp::Backend::threaded(a.num<unsigned>("--threads", 1),
                                         a.num<std::size_t>("--chunk", 0));
  return dpmrf::dpp::Backend::serial();
}

// main.cpp:60-69
dpmrf::OptimizerConfig make_config(const Args& a) {
  dpmrf::OptimizerConfig c;
  c.rng_seed = a.num<std::uint64_t>("--seed", c.rng_seed);
  c.beta = a.num<double>("--beta", c.beta);
  c.em_max_iters = a.num<int>("--em-iters", c.em_max_iters);
  c.map_max_iters = a.num<int>("--map-iters", c.map_max_iters);
  c.convergence_window = a.num<int>("--window", c.convergence_window);
  c.convergence_tol = a.num<double>("--tol", c.convergence_tol);
  return c;
}

// main.cpp:71-82
dpmrf::LabelMap load_oversegmentation(const dpmrf::GrayImage& image, const std::string& overseg,
                                      std::uint32_t block) {
  if (!overseg.empty()) {
    dpmrf::LabelMap labels = dpmrf::read_rlm(overseg);
    if (labels.width != image.width || labels.height != image.height)
      throw dpmrf::InputError("oversegmentation dimensions do not match the image");
    return labels;
  }
  if (block > 0) return dpmrf::grid_oversegment(image.width, image.height, block);
  throw dpmrf::InputError("provide --overseg FILE or --block N");
}

std::string basename_of(const std::string& path) {
  const auto pos = path.find_last_of('/');
  return pos == std::string::npos ? path : path.substr(pos + 1);
}

// main.cpp:92-118
int gen_synth(int argc, char** argv) {
  const Args a(argc, argv, 2, {"--size", "--pore", "--sp", "--gauss", "--seed", "--out", "--truth"},
               {"--ringing"});
  dpmrf::PhantomSpec spec;
  const auto size = a.num<std::uint32_t>("--size", 128);
  spec.pore_fraction = a.num<double>("--pore", spec.pore_fraction);
  spec.sp_rate = a.num<double>("--sp", spec.sp_rate);
  spec.gauss_sigma = a.num<double>("--gauss", spec.gauss_sigma);
  spec.ringing = a.flag("--ringing");
  spec.seed = a.num<std::uint64_t>("--seed", spec.seed);
  const std::string out = a.required("--out");
  const std::string truth = a.required("--truth");
  spec.width = size;
  spec.height = size;
  const auto ph = dpmrf::gen_phantom(spec);
  const auto noisy = dpmrf::corrupt(ph.clean, spec);
  dpmrf::write_pgm(noisy, out);
  dpmrf::write_binary_pgm(ph.truth, truth);
  std::cout << "gen-synth: wrote " << out << " and " << truth << ", pore fraction " << std::fixed
            << std::setprecision(4) << dpmrf::porosity(ph.truth) << "\n";
  return 0;
}

// main.cpp:120-172
int segment(int argc, char** argv) {
  const Args a(argc, argv, 2,
               join(join({"--image", "--overseg", "--block", "--labels", "--out"}, kExecOptions),
                    kConfigOptions),
               {});
  const std::string image_path = a.required("--image");
  const std::string out_path = a.required("--out");
  const auto num_labels = a.num<std::uint32_t>("--labels", 2);
  const auto cfg = make_config(a);
  const auto backend = make_backend(a);
  if (num_labels != 2) throw dpmrf::InputError("only --labels 2 is supported");
  const auto image = dpmrf::read_pgm(image_path);
  const auto labels =
      load_oversegmentation(image, a.str("--overseg"), a.num<std::uint32_t>("--block", 0));

  const auto t0 = Clock::now();
  const auto graph = dpmrf::build_region_graph(backend, image, labels);
  const auto t1 = Clock::now();
  const auto cliques = dpmrf::enumerate_maximal_cliques(backend, graph);
  const auto t2 = Clock::now();
  const auto hoods = dpmrf::build_neighborhoods(backend, graph, cliques);
  const auto t3 = Clock::now();
  const auto res = dpmrf::optimize(backend, graph, hoods, cfg);
  const auto t4 = Clock::now();

  // The darker class (smaller mean) is the pore phase (main.cpp:156-157).
  const std::uint32_t pore_label = res.params.mu[0] <= res.params.mu[1] ? 0u : 1u;
  dpmrf::BinaryImage mask;
  mask.width = image.width;
  mask.height = image.height;
  mask.pixels.resize(image.size());
  for (std::size_t i = 0; i < mask.pixels.size(); ++i)
    mask.pixels[i] = res.labels[labels.region[i]] == pore_label ? 1 : 0;
  dpmrf::write_binary_pgm(mask, out_path);

  std::cout << "segment: regions=" << graph.num_vertices << " cliques=" << cliques.size()
            << " hoods=" << hoods.size() << " em_iters=" << res.trace.size() << std::fixed
            << std::setprecision(6) << " graph_s=" << seconds(t0, t1)
            << " cliques_s=" << seconds(t1, t2) << " hoods_s=" << seconds(t2, t3)
            << " optimize_s=" << seconds(t3, t4) << "\n";
  return 0;
}

// main.cpp:174-204
int verify(int argc, char** argv) {
  const Args a(argc, argv, 2, {"--pred", "--truth"}, {});
  const std::string pred_path = a.required("--pred");
  const std::string truth_path = a.required("--truth");
  const auto pred = dpmrf::read_binary_pgm(pred_path);
  const auto truth = dpmrf::read_binary_pgm(truth_path);
  const auto m = dpmrf::compute_metrics(dpmrf::confusion(pred, truth));
  std::ostringstream row;
  row << std::fixed << std::setprecision(6);
  if (m.precision_defined) {
    row << m.precision;
  } else {
    row << "undefined";
  }
  row << ',';
  if (m.recall_defined) {
    row << m.recall;
  } else {
    row << "undefined";
  }
  row << ',' << m.accuracy << ',' << dpmrf::porosity(pred) << ',' << dpmrf::porosity(truth);
  std::cout << "precision,recall,accuracy,porosity_pred,porosity_truth\n" << row.str() << "\n";
  return 0;
}

// harness.cpp:69-86's per-record loop on Backend::cuda(): structures and the
// optimization phase timed separately, wall_s = optimization phase.
std::vector<dpmrf::BenchRecord> cuda_records(const dpmrf::GrayImage& image,
                                             const dpmrf::LabelMap& labels,
                                             const dpmrf::BenchPlan& plan, unsigned device,
                                             double t_star) {
  std::vector<dpmrf::BenchRecord> out;
  const auto backend = dpmrf::dpp::Backend::cuda(device);
  for (unsigned rep = 0; rep < plan.repeats; ++rep) {
    dpmrf::BenchRecord rec;
    rec.dataset = plan.dataset;
    rec.backend = "cuda";
    rec.threads = 1;
    rec.rep = rep;
    const auto t0 = Clock::now();
    const auto graph = dpmrf::build_region_graph(backend, image, labels);
    const auto t1 = Clock::now();
    const auto cliques = dpmrf::enumerate_maximal_cliques(backend, graph);
    const auto t2 = Clock::now();
    const auto hoods = dpmrf::build_neighborhoods(backend, graph, cliques);
    const auto t3 = Clock::now();
    const auto res = dpmrf::optimize(backend, graph, hoods, plan.config);
    const auto t4 = Clock::now();
    (void)res;
    rec.graph_s = seconds(t0, t1);
    rec.cliques_s = seconds(t1, t2);
    rec.hoods_s = seconds(t2, t3);
    rec.optimize_s = seconds(t3, t4);
    rec.wall_s = rec.optimize_s;
    rec.speedup = rec.wall_s > 0.0 ? t_star / rec.wall_s : 0.0;
    out.push_back(rec);
  }
  return out;
}

std::vector<unsigned> parse_list(const std::string& s) {
  std::vector<unsigned> out;
  std::istringstream in(s);
  std::string item;
  while (std::getline(in, item, ',')) {
    std::istringstream v(item);
    unsigned x = 0;
    v >> x;
    if (!v || !v.eof()) throw UsageError("--threads: invalid list " + s);
    out.push_back(x);
  }
  return out;
}

// main.cpp:206-238
int bench(int argc, char** argv) {
  const Args a(argc, argv, 2,
               join({"--image", "--overseg", "--block", "--threads", "--repeat", "--csv",
                     "--device"},
                    kConfigOptions),
               {"--cuda"});
  const std::string image_path = a.required("--image");
  dpmrf::BenchPlan plan;
  if (a.has("--threads")) plan.threads = parse_list(a.str("--threads"));
  plan.repeats = a.num<unsigned>("--repeat", plan.repeats);
  plan.config = make_config(a);
  const auto image = dpmrf::read_pgm(image_path);
  const auto labels =
      load_oversegmentation(image, a.str("--overseg"), a.num<std::uint32_t>("--block", 0));
  plan.dataset = basename_of(image_path);
  auto records = dpmrf::run_bench(image, labels, plan);
  if (a.flag("--cuda")) {
    const auto more =
        cuda_records(image, labels, plan, a.num<unsigned>("--device", 0), records.front().wall_s);
    records.insert(records.end(), more.begin(), more.end());
  }
  const auto csv = dpmrf::bench_csv(records);
  const std::string csv_path = a.str("--csv");
  if (csv_path.empty()) {
    std::cout << csv;
  } else {
    std::ofstream out(csv_path);
    if (!out) throw dpmrf::InputError("cannot write " + csv_path);
    out << csv;
    std::cout << "bench: wrote " << records.size() << " records to " << csv_path << "\n";
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) throw UsageError("a subcommand is required: gen-synth, segment, verify, bench");
    const std::string cmd = argv[1];
    if (cmd == "gen-synth") return gen_synth(argc, argv);
    if (cmd == "segment") return segment(argc, argv);
    if (cmd == "verify") return verify(argc, argv);
    if (cmd == "bench") return bench(argc, argv);
    if (cmd == "--help" || cmd == "-h") {
      std::cout << "usage: dpmrf {gen-synth|segment|verify|bench} [options]\n";
      return 0;
    }
    throw UsageError("unknown subcommand " + cmd);
  } catch (const UsageError& e) {
    std::cerr << "usage error: " << e.what() << "\n";
    return 2;
  } catch (const dpmrf::InputError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "internal error: " << e.what() << "\n";
    return 1;
  }
}
