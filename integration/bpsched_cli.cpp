// bpsched-cuda: the reference CLI's run / bench / verify / generate
// subcommands (proj/tools/bpsched.cpp:128-374) with a --backend switch
// (SURVEY.md 8(f) N3).  Graph loading, trace CSV, generators and exact
// inference are the reference's own functions (linked from its core); the
// solver is bpsched_cuda::run (include/bpsched_cuda.hpp) for --backend cuda,
// bpsched::run for --backend cpu.  Outputs follow the reference CLI
// byte-for-byte: trace CSV (write_trace_csv), runs.csv / summary.csv /
// curve_<config>.csv, and the JSON summary line (sorted keys, shortest
// round-trip doubles, as nlohmann::json::dump prints them).
//
// Built by `make -C oracle cli` (it needs the reference core objects);
// the reference's third-party CLI/JSON headers are not used.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "bpsched/errors.hpp"
#include "bpsched/exact.hpp"
#include "bpsched/generators.hpp"
#include "bpsched/model_io.hpp"
#include "bpsched/schedulers.hpp"
#include "bpsched_cuda.hpp"

namespace fs = std::filesystem;

namespace {

constexpr int kOk = 0, kError = 1, kNotConverged = 2;  // bpsched.cpp:25-27

std::string shortest(double v) {  // std::to_chars shortest round trip (bpsched.cpp format_double)
  char buf[32];
  const auto r = std::to_chars(buf, buf + sizeof(buf), v);
  return std::string(buf, r.ptr);
}

// a JSON number as nlohmann::json::dump prints a double
std::string json_double(double v) {
  if (!std::isfinite(v)) return "null";
  std::string s = shortest(v);
  if (s.find_first_of(".e") == std::string::npos) s += ".0";
  return s;
}

// JSON object with sorted keys (nlohmann::json's std::map order)
struct JsonObj {
  std::map<std::string, std::string> kv;
  void b(const std::string& k, bool v) { kv[k] = v ? "true" : "false"; }
  void u(const std::string& k, uint64_t v) { kv[k] = std::to_string(v); }
  void d(const std::string& k, double v) { kv[k] = json_double(v); }
  void s(const std::string& k, const std::string& v) { kv[k] = "\"" + v + "\""; }
  std::string dump() const {
    std::string o = "{";
    for (const auto& [k, v] : kv) o += (o.size() > 1 ? "," : "") + ("\"" + k + "\":" + v);
    return o + "}";
  }
};

std::string slurp(const fs::path& p) {
  std::ifstream in(p, std::ios::binary);
  if (!in) throw bpsched::error("cannot open " + p.string());
  std::ostringstream b;
  b << in.rdbuf();
  return std::move(b).str();
}

void spit(const fs::path& p, const std::string& s) {
  std::ofstream out(p, std::ios::binary);
  if (!out) throw bpsched::error("cannot open " + p.string() + " for writing");
  out << s;
  if (!out) throw bpsched::error("write failure on " + p.string());
}

// --key value options; lists comma-separated or repeated
struct Args {
  std::map<std::string, std::vector<std::string>> opt;
  explicit Args(int argc, char** argv, int from) {
    for (int i = from; i < argc; ++i) {
      std::string k = argv[i];
      if (k.rfind("--", 0) != 0 || i + 1 >= argc) throw std::invalid_argument("expected --option value, got " + k);
      std::stringstream ss(argv[++i]);
      std::string item;
      while (std::getline(ss, item, ',')) opt[k.substr(2)].push_back(item);
    }
  }
  bool has(const std::string& k) const { return opt.count(k) != 0; }
  std::string str(const std::string& k, const std::string& def = "") const {
    auto it = opt.find(k);
    return it == opt.end() ? def : it->second.front();
  }
  std::string req(const std::string& k) const {
    if (!has(k)) throw std::invalid_argument("--" + k + " is required");
    return str(k);
  }
  double num(const std::string& k, double def) const { return has(k) ? std::stod(str(k)) : def; }
  uint64_t u64(const std::string& k, uint64_t def) const { return has(k) ? std::stoull(str(k)) : def; }
  std::vector<double> nums(const std::string& k) const {
    std::vector<double> v;
    if (has(k))
      for (const auto& s : opt.at(k)) v.push_back(std::stod(s));
    return v;
  }
};

// SchedulerFlags (bpsched.cpp:45-117): same defaults and validation
bpsched::SchedulerConfig config_from(const Args& a, const std::string& scheduler) {
  const auto kind = bpsched::scheduler_from_string(scheduler);
  if (!kind) throw bpsched::error("unknown scheduler '" + scheduler + "'");
  bpsched::SchedulerConfig c;
  c.kind = *kind;
  c.epsilon = a.num("epsilon", 1e-5);
  c.p = a.num("p", 1.0);
  c.low_p = a.num("low-p", 0.7);
  c.high_p = a.num("high-p", 1.0);
  c.edge_ratio_threshold = a.num("edge-ratio-threshold", 0.9);
  c.splash_depth = static_cast<uint32_t>(a.u64("splash-depth", 2));
  c.max_iterations = a.u64("max-iterations", 10000);
  c.time_limit = a.num("time-limit", 90.0);
  c.seed = a.u64("seed", 0);
  unsigned workers = 0;
  if (a.has("workers")) {
    workers = static_cast<unsigned>(std::stoul(a.str("workers")));
  } else if (const char* env = std::getenv("BP_SCHED_WORKERS")) {
    const long v = std::strtol(env, nullptr, 10);
    if (v > 0) workers = static_cast<unsigned>(v);
  }
  c.worker_count = workers;
  c.validate();
  return c;
}

bpsched::RunResult solve(const Args& a, const bpsched::PairwiseMRF& g, const bpsched::SchedulerConfig& c) {
  const std::string backend = a.str("backend", "cuda");
  if (backend == "cuda") return bpsched_cuda::run(g, c);
  if (backend == "cpu") return bpsched::run(g, c);
  throw std::invalid_argument("--backend must be cuda or cpu");
}

std::string label_of(const bpsched::SchedulerConfig& c) {  // bpsched.cpp:215-229
  using K = bpsched::SchedulerKind;
  switch (c.kind) {
    case K::lbp: return "lbp";
    case K::serial_rbp: return "srbp";
    case K::rbp: return "rbp_p" + shortest(c.p);
    case K::rs: return "rs_p" + shortest(c.p) + "_h" + std::to_string(c.splash_depth);
    case K::rnbp: return "rnbp_low" + shortest(c.low_p) + "_high" + shortest(c.high_p);
  }
  return "unknown";
}

double median_of(std::vector<double> v) {
  if (v.empty()) return std::nan("");
  std::sort(v.begin(), v.end());
  const size_t m = v.size() / 2;
  return v.size() % 2 ? v[m] : 0.5 * (v[m - 1] + v[m]);
}

int cmd_run(const Args& a) {
  const bpsched::PairwiseMRF g = bpsched::parse_model(slurp(a.req("model")));
  const bpsched::SchedulerConfig c = config_from(a, a.str("scheduler", "lbp"));
  const bpsched::RunResult r = solve(a, g, c);
  if (a.has("out")) {
    std::ofstream out(a.str("out"), std::ios::binary);
    if (!out) throw bpsched::error("cannot open " + a.str("out") + " for writing");
    bpsched::write_trace_csv(r, out);
  }
  JsonObj j;
  j.b("converged", r.converged);
  j.u("iterations", r.iterations);
  j.d("wall_time", r.wall_time);
  j.u("messages_updated_total", r.messages_updated_total);
  std::cout << j.dump() << "\n";
  return r.converged ? kOk : kNotConverged;
}

int cmd_bench(const Args& a) {
  const fs::path manifest(a.req("manifest")), out_dir(a.req("out"));
  if (!a.has("scheduler")) throw std::invalid_argument("--scheduler is required");
  // manifest: header, then path,kind,n,c,seed (bpsched.cpp:190-213)
  std::vector<std::pair<fs::path, uint64_t>> suite;
  {
    std::istringstream in(slurp(manifest));
    std::string line;
    bool header = true;
    while (std::getline(in, line)) {
      if (line.empty() || line[0] == '#') continue;
      if (header) {
        header = false;
        continue;
      }
      std::vector<std::string> f;
      std::stringstream ss(line);
      std::string x;
      while (std::getline(ss, x, ',')) f.push_back(x);
      if (f.size() < 5) throw bpsched::error("malformed manifest line: " + line);
      suite.emplace_back(manifest.parent_path() / f[0], std::stoull(f[4]));
    }
  }
  if (suite.empty()) throw bpsched::error("manifest lists no models");
  fs::create_directories(out_dir);
  std::vector<bpsched::SchedulerConfig> grid;
  for (const std::string& name : a.opt.at("scheduler")) {
    const bpsched::SchedulerConfig base = config_from(a, name);
    std::vector<double> ps = a.nums("p"), lows = a.nums("low-p");
    if (base.kind == bpsched::SchedulerKind::rbp || base.kind == bpsched::SchedulerKind::rs) {
      if (ps.empty()) ps.push_back(base.p);
      for (double p : ps) {
        bpsched::SchedulerConfig c = base;
        c.p = p;
        c.validate();
        grid.push_back(c);
      }
    } else if (base.kind == bpsched::SchedulerKind::rnbp) {
      if (lows.empty()) lows.push_back(base.low_p);
      for (double lo : lows) {
        bpsched::SchedulerConfig c = base;
        c.low_p = lo;
        c.validate();
        grid.push_back(c);
      }
    } else {
      grid.push_back(base);
    }
  }
  std::string runs = "config,model,seed,status,converged,iterations,wall_time_s,messages_updated\n";
  std::string summary = "config,runs,converged,median_time_s,median_iterations\n";
  for (const bpsched::SchedulerConfig& cfg : grid) {
    const std::string label = label_of(cfg);
    std::vector<double> times, iters;
    uint32_t conv = 0;
    for (size_t i = 0; i < suite.size(); ++i) {
      bpsched::SchedulerConfig c = cfg;
      c.seed = cfg.seed + i;
      std::string status = "ok";
      bpsched::RunResult r;
      try {
        r = solve(a, bpsched::parse_model(slurp(suite[i].first)), c);
      } catch (const std::exception& ex) {
        std::string m = ex.what();
        std::replace(m.begin(), m.end(), ',', ';');
        std::replace(m.begin(), m.end(), '\n', ' ');
        status = "error: " + m;
      }
      const bool ok = status == "ok";
      if (ok && r.converged) {
        ++conv;
        times.push_back(r.wall_time);
        iters.push_back(static_cast<double>(r.iterations));
      }
      runs += label + "," + suite[i].first.filename().string() + "," + std::to_string(c.seed) + "," + status + "," +
              (ok ? (r.converged ? "true" : "false") : "") + "," + (ok ? std::to_string(r.iterations) : "") + "," +
              (ok ? shortest(r.wall_time) : "") + "," + (ok ? std::to_string(r.messages_updated_total) : "") + "\n";
      std::cerr << label << " " << suite[i].first.filename().string() << ": "
                << (ok ? (r.converged ? "converged" : "not converged") : status) << " in " << shortest(r.wall_time)
                << "s\n";
    }
    std::sort(times.begin(), times.end());
    std::string curve = "time_s,fraction_converged\n";
    for (size_t i = 0; i < times.size(); ++i)
      curve += shortest(times[i]) + "," + shortest(static_cast<double>(i + 1) / static_cast<double>(suite.size())) +
               "\n";
    spit(out_dir / ("curve_" + label + ".csv"), curve);
    summary += label + "," + std::to_string(suite.size()) + "," + std::to_string(conv) + "," +
               shortest(median_of(times)) + "," + shortest(median_of(iters)) + "\n";
  }
  spit(out_dir / "runs.csv", runs);
  spit(out_dir / "summary.csv", summary);
  std::cout << summary;
  return kOk;
}

int cmd_verify(const Args& a) {
  const bpsched::PairwiseMRF g = bpsched::parse_model(slurp(a.req("model")));
  const bpsched::SchedulerConfig c = config_from(a, a.str("scheduler", "lbp"));
  const bpsched::RunResult r = solve(a, g, c);
  const std::vector<bpsched::vertex_id> order = bpsched::min_degree_order(g);
  const bpsched::BeliefTable exact = bpsched::variable_elimination(g, order);
  std::string rows = "vertex,kl\n";
  double sum = 0.0;
  for (bpsched::vertex_id v = 0; v < g.num_vertices(); ++v) {
    const double kl = bpsched::kl_divergence(exact.at(v), r.beliefs.at(v));
    sum += kl;
    rows += std::to_string(v) + "," + shortest(kl) + "\n";
  }
  std::cout << rows;
  JsonObj j;
  j.d("mean_kl", g.num_vertices() ? sum / static_cast<double>(g.num_vertices()) : 0.0);
  j.b("converged", r.converged);
  j.u("iterations", r.iterations);
  j.d("wall_time", r.wall_time);
  if (!r.converged) j.s("warning", "run did not converge; KL measured against non-converged beliefs");
  std::cout << j.dump() << "\n";
  return kOk;
}

int cmd_generate(const Args& a) {  // CPU generators (not on the device path), for suites
  const std::string kind = a.str("kind", "ising");
  if (kind != "ising" && kind != "chain") throw bpsched::error("unknown kind '" + kind + "' (expected ising or chain)");
  const uint32_t n = static_cast<uint32_t>(a.u64("n", 10)), count = static_cast<uint32_t>(a.u64("count", 25));
  const double cc = a.num("c", 2.0);
  const uint64_t seed0 = a.u64("seed", 0);
  const fs::path out(a.req("out"));
  fs::create_directories(out);
  std::string manifest = "path,kind,n,c,seed\n";
  for (uint32_t i = 0; i < count; ++i) {
    const uint64_t s = seed0 + i;
    const bpsched::PairwiseMRF g =
        kind == "ising" ? bpsched::generate_ising({n, cc, s}) : bpsched::generate_chain({n, cc, s});
    const std::string name = kind + "_n" + std::to_string(n) + "_c" + shortest(cc) + "_s" + std::to_string(s) + ".pgm";
    spit(out / name, bpsched::serialize_model(g));
    manifest += name + "," + kind + "," + std::to_string(n) + "," + shortest(cc) + "," + std::to_string(s) + "\n";
  }
  spit(out / "manifest.csv", manifest);
  std::cout << "wrote " << count << " models + manifest to " << out.string() << "\n";
  return kOk;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: bpsched-cuda {run|bench|verify|generate} [--option value ...] [--backend cuda|cpu]\n";
    return kError;
  }
  try {
    const std::string cmd = argv[1];
    const Args a(argc, argv, 2);
    if (cmd == "run") return cmd_run(a);
    if (cmd == "bench") return cmd_bench(a);
    if (cmd == "verify") return cmd_verify(a);
    if (cmd == "generate") return cmd_generate(a);
    std::cerr << "unknown subcommand " << cmd << "\n";
    return kError;
  } catch (const std::exception& ex) {
    std::cerr << "error: " << ex.what() << "\n";
    return kError;
  }
}
