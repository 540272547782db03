// C++ lockstep parity harness: the UNMODIFIED reference core (compiled from
// /root/reference by oracle/Makefile into oracle/_ref/obj) and the B200
// engine in one process, through the reference's own C++ API on one side and
// include/bpsched_cuda.hpp + include/bp_cuda.h on the other (SURVEY.md
// section 8(c), "lockstep oracle method").  Test infrastructure only: built by
// `make -C oracle harness` into oracle/_ref/parity_harness and driven by
// tests/test_gpu_cpp_harness.py.
//
// Checks (tolerances from the north star):
//   lbp_lockstep      frontier_lbp + apply_frontier vs bp_engine_step:
//                     every message within 1e-5 abs after every iteration
//   rnbp_injected     the reference's own rnbp_frontier (mt19937_64) applied
//                     to both engines: messages within 1e-5
//   rbp_injected      the reference's rbp_frontier applied to both
//   rs_injected       the reference's rs_frontier splashes applied to both
//                     (apply_splash_frontier vs bp_engine_apply_splashes)
//   run_<kind>        bpsched::run vs bpsched_cuda::run: same convergence
//                     verdict, converged beliefs within 1e-4
//   errors            std::invalid_argument / bpsched::model_error from both
#include <set>
#include <random>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "bpsched/errors.hpp"
#include "bpsched/generators.hpp"
#include "bpsched/messages.hpp"
#include "bpsched/mrf.hpp"
#include "bpsched/schedulers.hpp"
#include "bpsched_cuda.hpp"

namespace {

int g_fail = 0, g_pass = 0;

void report(const std::string& name, bool ok, const std::string& detail) {
  std::printf("%s %s %s\n", ok ? "[PASS]" : "[FAIL]", name.c_str(), detail.c_str());
  (ok ? g_pass : g_fail)++;
}

struct DevEngine {
  bp_engine* e = nullptr;
  DevEngine(const bpsched_cuda::DeviceGraph& g, const bpsched::SchedulerConfig& c) {
    const bp_sched_config cc = bpsched_cuda::to_c(c);
    bpsched_cuda::check(bp_engine_create(g.get(), &cc, &e));
  }
  ~DevEngine() { bp_engine_destroy(e); }
};

double max_msg_diff(const bpsched::EngineState& ref, const DevEngine& dev, uint64_t total) {
  std::vector<double> d(total);
  bpsched_cuda::check(bp_engine_messages(dev.e, d.data()));
  double worst = 0.0;
  size_t o = 0;
  for (bpsched::directed_edge_id k = 0; k < ref.graph().num_directed_edges(); ++k)
    for (double x : ref.messages().view(k)) worst = std::max(worst, std::fabs(x - d[o++]));
  return worst;
}

uint64_t total_message_len(const bpsched::PairwiseMRF& g) {
  uint64_t n = 0;
  for (bpsched::directed_edge_id d = 0; d < g.num_directed_edges(); ++d)
    n += g.cardinality(g.directed_edge(d).target);
  return n;
}

// mixed-cardinality random graph (test_helpers.hpp:90-132 shape)
bpsched::PairwiseMRF random_graph(uint64_t seed, uint32_t n, uint32_t max_card) {
  std::mt19937_64 rng(seed);
  auto unit = [&] { return bpsched::uniform_unit(rng); };
  std::vector<uint32_t> cards(n);
  for (auto& c : cards) c = 2 + static_cast<uint32_t>(unit() * (max_card - 1));
  std::vector<std::vector<double>> un(n);
  for (uint32_t v = 0; v < n; ++v)
    for (uint32_t x = 0; x < cards[v]; ++x) un[v].push_back(std::exp(2.0 * unit() - 1.0));
  std::vector<bpsched::PairwiseMRF::EdgeSpec> edges;
  std::vector<std::vector<bool>> has(n, std::vector<bool>(n, false));
  auto add = [&](uint32_t i, uint32_t j) {
    if (i > j) std::swap(i, j);
    if (has[i][j]) return;
    has[i][j] = true;
    std::vector<double> t(static_cast<size_t>(cards[i]) * cards[j]);
    for (auto& x : t) x = std::exp(2.0 * unit() - 1.0);
    edges.push_back({i, j, t});
  };
  for (uint32_t v = 1; v < n; ++v) add(static_cast<uint32_t>(unit() * v), v);
  for (uint32_t i = 0; i + 1 < n; ++i)
    for (uint32_t j = i + 1; j < n; ++j)
      if (unit() < 0.2) add(i, j);
  return bpsched::build_graph(cards, un, edges);
}

void lbp_lockstep(const std::string& name, const bpsched::PairwiseMRF& g, int iters) {
  bpsched::SchedulerConfig cfg;
  bpsched::EngineState ref(g, cfg);
  bpsched_cuda::DeviceGraph dg(g);
  DevEngine dev(dg, cfg);
  const uint64_t total = total_message_len(g);
  double worst = 0.0;
  int t = 0;
  for (; t < iters; ++t) {
    worst = std::max(worst, max_msg_diff(ref, dev, total));
    if (ref.tracker().unconverged_count() == 0) break;
    bpsched::apply_frontier(ref, bpsched::frontier_lbp(ref));
    uint64_t fs = 0;
    bpsched_cuda::check(bp_engine_step(dev.e, &fs));
  }
  report(name, worst <= 1e-5, "iterations " + std::to_string(t) + " max|dm| " + std::to_string(worst));
}

template <class Frontier>
void injected(const std::string& name, const bpsched::PairwiseMRF& g, const bpsched::SchedulerConfig& cfg,
              int iters, Frontier frontier) {
  bpsched::EngineState ref(g, cfg);
  bpsched_cuda::DeviceGraph dg(g);
  DevEngine dev(dg, cfg);
  const uint64_t total = total_message_len(g);
  double worst = 0.0;
  int t = 0;
  for (; t < iters && ref.tracker().unconverged_count() > 0; ++t) {
    frontier(ref, dev);
    worst = std::max(worst, max_msg_diff(ref, dev, total));
  }
  report(name, worst <= 1e-5, "iterations " + std::to_string(t) + " max|dm| " + std::to_string(worst));
}

void apply_both(bpsched::EngineState& ref, DevEngine& dev, const std::vector<bpsched::directed_edge_id>& f) {
  bpsched::apply_frontier(ref, f);
  bpsched_cuda::check(bp_engine_apply_frontier(dev.e, f.data(), f.size()));
}

void run_compare(const std::string& name, const bpsched::PairwiseMRF& g, bpsched::SchedulerConfig cfg) {
  cfg.time_limit = 600.0;
  const bpsched::RunResult a = bpsched::run(g, cfg);
  const bpsched::RunResult b = bpsched_cuda::run(g, cfg);
  double worst = 0.0;
  if (a.converged && b.converged)
    for (bpsched::vertex_id v = 0; v < g.num_vertices(); ++v) {
      const auto x = a.beliefs.at(v), y = b.beliefs.at(v);
      for (size_t k = 0; k < x.size(); ++k) worst = std::max(worst, std::fabs(x[k] - y[k]));
    }
  const bool trace_ok = b.trace.size() == b.iterations;
  const bool ok = a.converged == b.converged && worst <= 1e-4 && trace_ok;
  report(name, ok,
         std::string("converged ref/dev ") + (a.converged ? "1" : "0") + "/" + (b.converged ? "1" : "0") +
             " iterations " + std::to_string(a.iterations) + "/" + std::to_string(b.iterations) + " max|db| " +
             std::to_string(worst));
}

template <class E>
bool throws(const std::function<void()>& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

}  // namespace

int main() {
  using bpsched::SchedulerKind;
  // LBP lockstep: Ising grids (lattice fast path on the device), chains, mixed cardinalities
  lbp_lockstep("lbp_lockstep_ising10_c2.5", bpsched::generate_ising({10, 2.5, 11}), 40);
  lbp_lockstep("lbp_lockstep_ising16_c2.0", bpsched::generate_ising({16, 2.0, 3}), 40);
  lbp_lockstep("lbp_lockstep_chain50", bpsched::generate_chain({50, 2.0, 5}), 60);
  for (uint64_t s = 0; s < 4; ++s) lbp_lockstep("lbp_lockstep_random" + std::to_string(s), random_graph(100 + s, 12, 4), 30);

  // RnBP with the reference's own mt19937_64 frontier
  {
    bpsched::SchedulerConfig cfg;
    cfg.kind = SchedulerKind::rnbp;
    cfg.seed = 7;
    injected("rnbp_injected_ising12", bpsched::generate_ising({12, 2.5, 2}), cfg, 60,
             [&](bpsched::EngineState& ref, DevEngine& dev) {
               const uint32_t now = ref.tracker().unconverged_count();
               const double p = bpsched::select_parallelism(ref.prev_unconverged().value_or(0), now, cfg);
               ref.set_prev_unconverged(now);
               apply_both(ref, dev, bpsched::rnbp_frontier(ref, p, ref.rng()));
             });
  }
  // RBP top-k frontier from the reference
  {
    bpsched::SchedulerConfig cfg;
    cfg.kind = SchedulerKind::rbp;
    injected("rbp_injected_ising12", bpsched::generate_ising({12, 2.5, 4}), cfg, 60,
             [&](bpsched::EngineState& ref, DevEngine& dev) { apply_both(ref, dev, bpsched::rbp_frontier(ref, 1.0 / 16)); });
    injected("rbp_injected_random", random_graph(7, 14, 3), cfg, 40,
             [&](bpsched::EngineState& ref, DevEngine& dev) { apply_both(ref, dev, bpsched::rbp_frontier(ref, 0.2)); });
  }
  // Residual Splash: the reference's splashes, Gauss-Seidel inside each
  {
    bpsched::SchedulerConfig cfg;
    cfg.kind = SchedulerKind::rs;
    auto rs = [&](double p, uint32_t h) {
      return [p, h](bpsched::EngineState& ref, DevEngine& dev) {
        const auto splashes = bpsched::rs_frontier(ref, p, h);
        std::vector<uint32_t> roots;
        std::vector<uint64_t> off{0};
        std::vector<uint32_t> edges;
        for (const auto& s : splashes) {
          roots.push_back(s.root);
          edges.insert(edges.end(), s.edges.begin(), s.edges.end());
          off.push_back(edges.size());
        }
        bpsched::apply_splash_frontier(ref, splashes);
        bpsched_cuda::check(bp_engine_apply_splashes(dev.e, roots.size(), roots.data(), off.data(), edges.data()));
      };
    };
    injected("rs_injected_ising12_h2", bpsched::generate_ising({12, 2.5, 9}), cfg, 30, rs(1.0 / 16, 2));
    injected("rs_injected_random_h1", random_graph(9, 14, 3), cfg, 20, rs(0.2, 1));
  }
  // End-to-end: bpsched::run vs bpsched_cuda::run
  for (auto kind : {SchedulerKind::lbp, SchedulerKind::rbp, SchedulerKind::rs, SchedulerKind::rnbp}) {
    bpsched::SchedulerConfig cfg;
    cfg.kind = kind;
    cfg.p = kind == SchedulerKind::rs ? 1.0 / 32 : 1.0 / 16;
    cfg.low_p = 0.5;
    cfg.max_iterations = 100000;
    const std::string k = bpsched::to_string(kind);
    run_compare("run_" + k + "_ising20_c2.0", bpsched::generate_ising({20, 2.0, 2}), cfg);
    run_compare("run_" + k + "_random", random_graph(31, 16, 3), cfg);
  }
  // row-band partition driven by the engine (bp_band_run), all bands in this
  // process: LBP owned beliefs bitwise, RnBP within 1e-4 of the reference
  for (uint32_t parts : {2u, 3u}) {
    bpsched::SchedulerConfig cfg;
    cfg.kind = SchedulerKind::lbp;
    cfg.max_iterations = 100000;
    const auto g = bpsched::generate_ising({24, 1.5, 5});
    const bpsched::RunResult a = bpsched_cuda::run(g, cfg);
    const bpsched::RunResult b = bpsched_cuda::run_partitioned_local(g, cfg, parts);
    bool same = a.converged == b.converged && a.iterations == b.iterations;
    for (bpsched::vertex_id v = 0; v < g.num_vertices() && same; ++v)
      same = a.beliefs.at(v)[0] == b.beliefs.at(v)[0] && a.beliefs.at(v)[1] == b.beliefs.at(v)[1];
    report("bands_lbp_ising24_x" + std::to_string(parts), same, "bitwise equal to the one-band run");
    cfg.kind = SchedulerKind::rnbp;
    cfg.low_p = 0.5;
    const bpsched::RunResult c = bpsched_cuda::run_partitioned_local(g, cfg, parts);
    const bpsched::RunResult d = bpsched_cuda::run(g, cfg);
    const bpsched::RunResult ref = bpsched::run(g, cfg);
    double worst = 0.0;
    for (bpsched::vertex_id v = 0; v < g.num_vertices(); ++v)
      for (size_t k = 0; k < 2; ++k) worst = std::max(worst, std::fabs(ref.beliefs.at(v)[k] - c.beliefs.at(v)[k]));
    report("bands_rnbp_ising24_x" + std::to_string(parts),
           c.iterations == d.iterations && c.messages_updated_total == d.messages_updated_total && c.converged &&
               ref.converged && worst <= 1e-4,
           "iterations " + std::to_string(c.iterations) + " (one band " + std::to_string(d.iterations) +
               ", reference " + std::to_string(ref.iterations) + ") max|db| vs reference " + std::to_string(worst));
  }
  // vertex-range partition of a random binary model (bp_graph_create_part):
  // bitwise the one-GPU run, and the reference's converged marginals
  for (uint32_t parts : {2u, 3u}) {
    std::vector<uint32_t> cards(400, 2);
    std::vector<std::vector<double>> unary;
    std::vector<bpsched::PairwiseMRF::EdgeSpec> edges;
    std::mt19937_64 rng(77 + parts);
    std::uniform_real_distribution<double> u(0.5, 1.5);
    for (uint32_t v = 0; v < 400; ++v) unary.push_back({u(rng), u(rng)});
    std::set<std::pair<uint32_t, uint32_t>> seen;
    while (edges.size() < 700) {
      uint32_t i = static_cast<uint32_t>(rng() % 400), j = static_cast<uint32_t>(rng() % 400);
      if (i == j) continue;
      if (i > j) std::swap(i, j);
      if (!seen.insert({i, j}).second) continue;
      edges.push_back({i, j, {u(rng), u(rng) * 0.3, u(rng) * 0.3, u(rng)}});
    }
    std::sort(edges.begin(), edges.end(), [](const auto& x, const auto& y) { return std::make_pair(x.i, x.j) < std::make_pair(y.i, y.j); });
    const auto g = bpsched::build_graph(cards, unary, edges);
    for (auto kind : {SchedulerKind::lbp, SchedulerKind::rnbp}) {
      bpsched::SchedulerConfig cfg;
      cfg.kind = kind;
      cfg.low_p = 0.5;
      cfg.max_iterations = 5000;
      const bpsched::RunResult a = bpsched_cuda::run(g, cfg);
      const bpsched::RunResult b = bpsched_cuda::run_vertex_partitioned_local(g, cfg, parts);
      const bpsched::RunResult ref = bpsched::run(g, cfg);
      bool same = a.converged == b.converged && a.iterations == b.iterations;
      double worst = 0.0;
      for (bpsched::vertex_id v = 0; v < g.num_vertices(); ++v)
        for (size_t k = 0; k < 2; ++k) {
          same = same && a.beliefs.at(v)[k] == b.beliefs.at(v)[k];
          worst = std::max(worst, std::fabs(ref.beliefs.at(v)[k] - b.beliefs.at(v)[k]));
        }
      report(std::string("parts_") + (kind == SchedulerKind::lbp ? "lbp" : "rnbp") + "_random400_x" +
                 std::to_string(parts),
             same && b.converged && ref.converged && worst <= 1e-4,
             "bitwise the one-GPU run; iterations " + std::to_string(b.iterations) + " (reference " +
                 std::to_string(ref.iterations) + ") max|db| vs reference " + std::to_string(worst));
    }
  }
  // serial RBP goes through the reference's run_serial_rbp inside the facade
  {
    bpsched::SchedulerConfig cfg;
    cfg.kind = SchedulerKind::serial_rbp;
    cfg.max_iterations = 200000;
    run_compare("run_srbp_ising8", bpsched::generate_ising({8, 2.0, 1}), cfg);
  }
  // error behaviour (schedulers.cpp:78-90, errors.hpp)
  {
    const auto g = bpsched::generate_ising({4, 2.0, 0});
    bpsched::SchedulerConfig bad;
    bad.epsilon = -1.0;
    report("errors_invalid_config", throws<std::invalid_argument>([&] { bpsched_cuda::run(g, bad); }) &&
                                        throws<std::invalid_argument>([&] { bpsched::run(g, bad); }),
           "std::invalid_argument from both");
    bpsched_cuda::DeviceGraph dg(g);
    bp_engine* e = nullptr;
    bpsched::SchedulerConfig cfg;
    const bp_sched_config cc = bpsched_cuda::to_c(cfg);
    bpsched_cuda::check(bp_engine_create(dg.get(), &cc, &e));
    const uint32_t roots[2] = {0, 1};
    const uint64_t off[3] = {0, 2, 3};
    const uint32_t edges[3] = {1, 3, 1};
    const int rc = bp_engine_apply_splashes(e, 2, roots, off, edges);
    bp_engine_destroy(e);
    report("errors_overlapping_splashes", rc == BP_ERR_MODEL &&
                                              throws<bpsched::model_error>([&] { bpsched_cuda::check(rc); }),
           "model_error (schedulers.cpp:262-268)");
  }
  std::printf("summary: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
