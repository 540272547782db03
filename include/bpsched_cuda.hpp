/*
 * bpsched_cuda.hpp -- C++ drop-in for the reference's scheduler entry point.
 *
 *   bpsched::RunResult bpsched_cuda::run(const bpsched::PairwiseMRF&,
 *                                        const bpsched::SchedulerConfig&);
 *
 * has the signature, types, defaults and error behaviour of bpsched::run
 * (/root/reference/proj/core/include/bpsched/schedulers.hpp:156,
 * src/schedulers.cpp:293-353) and runs the scheduler loop on the B200 engine
 * through the C ABI in bp_cuda.h.  Header-only: a caller of the reference
 * (tools/bpsched.cpp:172,299,349) includes this next to the reference headers,
 * links libbp_b200.so, and switches `bpsched::run(` to `bpsched_cuda::run(`
 * (INTEGRATION.md).  Graph loading stays the reference's own
 * (build_graph / parse_model / generate_ising, mrf.hpp:94-96): the facade reads
 * only the public PairwiseMRF accessors (mrf.hpp:39-70).
 *
 * Errors are rethrown as the reference's exceptions (errors.hpp:10-38):
 * std::invalid_argument for a bad config, bpsched::model_error,
 * bpsched::numeric_error, bpsched::error for device failures.  Caps are not
 * errors (converged == false), exactly as in the reference.
 *
 * Serial RBP (SchedulerKind::serial_rbp) is strictly sequential by
 * definition and stays on the host: the facade forwards it to
 * the reference's bpsched::run_serial_rbp.
 */
#ifndef BPSCHED_CUDA_HPP
#define BPSCHED_CUDA_HPP

#include <algorithm>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "bp_cuda.h"
#include "bpsched/errors.hpp"
#include "bpsched/messages.hpp"
#include "bpsched/mrf.hpp"
#include "bpsched/schedulers.hpp"

namespace bpsched_cuda {

[[noreturn]] inline void throw_status(int rc) {
  const std::string msg = bp_last_error();
  switch (rc) {
    case BP_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case BP_ERR_MODEL: throw bpsched::model_error(msg);
    case BP_ERR_NUMERIC: throw bpsched::numeric_error(msg);
    default: throw bpsched::error("bp_cuda (status " + std::to_string(rc) + "): " + msg);
  }
}

inline void check(int rc) {
  if (rc != BP_OK) throw_status(rc);
}

/// SchedulerConfig (schedulers.hpp:26-41) -> bp_sched_config; same numbering
/// of SchedulerKind.
inline bp_sched_config to_c(const bpsched::SchedulerConfig& c) {
  bp_sched_config o{};
  o.kind = static_cast<int32_t>(c.kind);
  o.splash_depth = c.splash_depth;
  o.epsilon = c.epsilon;
  o.p = c.p;
  o.low_p = c.low_p;
  o.high_p = c.high_p;
  o.edge_ratio_threshold = c.edge_ratio_threshold;
  o.max_iterations = c.max_iterations;
  o.time_limit = c.time_limit;
  o.seed = c.seed;
  o.worker_count = c.worker_count;
  return o;
}

/// build_graph's input layout of a PairwiseMRF, read through its public
/// accessors (mrf.hpp:39-70) -- what the C ABI takes.
struct HostArrays {
  std::vector<uint32_t> cards, ep;
  std::vector<double> unary, tables;
  explicit HostArrays(const bpsched::PairwiseMRF& g) {
    const uint32_t V = g.num_vertices(), E = g.num_edges();
    cards.resize(V);
    for (bpsched::vertex_id v = 0; v < V; ++v) {
      cards[v] = g.cardinality(v);
      const auto u = g.unary(v);
      unary.insert(unary.end(), u.begin(), u.end());
    }
    ep.resize(2ull * E);
    for (bpsched::edge_id e = 0; e < E; ++e) {
      const auto [i, j] = g.edge_endpoints(e);
      ep[2ull * e] = i;
      ep[2ull * e + 1] = j;
      const auto t = g.pairwise(e);
      tables.insert(tables.end(), t.begin(), t.end());
    }
  }
  bp_graph_desc desc() const {
    return bp_graph_desc{static_cast<uint32_t>(cards.size()), static_cast<uint32_t>(ep.size() / 2), cards.data(),
                         unary.data(), ep.data(), tables.data()};
  }
};

/// A PairwiseMRF resident in HBM.  Upload once, run many times (the graph is
/// immutable and shareable across runs, mrf.hpp:24-25).
class DeviceGraph {
 public:
  explicit DeviceGraph(const bpsched::PairwiseMRF& g, int device = -1) {
    const HostArrays a(g);
    cards_ = a.cards;
    const bp_graph_desc d = a.desc();
    bp_device_opts o{device, BP_GRAPH_TRUSTED};  // build_graph already validated it
    check(bp_graph_create(&d, &o, &h_));
  }
  DeviceGraph(const DeviceGraph&) = delete;
  DeviceGraph& operator=(const DeviceGraph&) = delete;
  ~DeviceGraph() { bp_graph_destroy(h_); }

  const bp_graph* get() const { return h_; }
  const std::vector<uint32_t>& cardinalities() const { return cards_; }

 private:
  bp_graph* h_ = nullptr;
  std::vector<uint32_t> cards_;
};

/// bpsched::run on a device-resident graph.
inline bpsched::RunResult run(const DeviceGraph& g, const bpsched::SchedulerConfig& config) {
  config.validate();  // the reference's own validation (schedulers.cpp:78-90)
  const bp_sched_config c = to_c(config);
  size_t nb = 0;
  for (uint32_t q : g.cardinalities()) nb += q;
  std::vector<double> beliefs(nb);
  const uint64_t cap = config.max_iterations < (1ull << 22) ? config.max_iterations + 1 : (1ull << 22);
  std::vector<bp_iter_record> trace(cap);
  bp_run_result r{};
  check(bp_run(g.get(), &c, &r, beliefs.data(), trace.data(), cap));

  bpsched::RunResult out;
  out.converged = r.converged != 0;
  out.iterations = r.iterations;
  out.wall_time = r.wall_time;
  out.messages_updated_total = r.messages_updated_total;
  out.beliefs = bpsched::BeliefTable(g.cardinalities());
  size_t o = 0;
  for (bpsched::vertex_id v = 0; v < g.cardinalities().size(); ++v) {
    auto dst = out.beliefs.at(v);
    for (size_t x = 0; x < dst.size(); ++x) dst[x] = beliefs[o++];
  }
  const uint64_t n = r.trace_len < cap ? r.trace_len : cap;
  out.trace.reserve(n);
  for (uint64_t k = 0; k < n; ++k)
    out.trace.push_back({trace[k].iteration, trace[k].frontier_size, trace[k].unconverged, trace[k].elapsed_seconds});
  return out;
}

/// Drop-in for bpsched::run (schedulers.hpp:156).
inline bpsched::RunResult run(const bpsched::PairwiseMRF& graph, const bpsched::SchedulerConfig& config) {
  config.validate();
  if (config.kind == bpsched::SchedulerKind::serial_rbp) return bpsched::run_serial_rbp(graph, config);
  DeviceGraph g(graph);
  return run(g, config);
}

// ---------------------------------------------------------------------------
// Multi-GPU: row bands of a binary Ising lattice, the run()
// loop in the engine (bp_band_run), NCCL between the ranks.

/// The rank's share of a partitioned run: the global loop result with the
/// beliefs of the band's OWNED rows [row0, row1) (vertices row0*cols ..).
struct BandRunResult {
  bpsched::RunResult result;
  uint32_t row0 = 0, row1 = 0, cols = 0;
};

namespace detail {
struct BandHandles {
  bp_graph* g = nullptr;
  bp_engine* e = nullptr;
  bp_band_info info{};
  ~BandHandles() {
    if (e) bp_engine_destroy(e);
    if (g) bp_graph_destroy(g);
  }
};
inline void make_band(const HostArrays& a, const bp_sched_config& c, uint32_t part, uint32_t nparts, int device,
                      BandHandles& b) {
  const bp_graph_desc d = a.desc();
  bp_device_opts o{device, 0};
  check(bp_graph_create_band(&d, part, nparts, &o, &b.g, &b.info));
  check(bp_band_engine_create_owned(b.g, &c, &b.info, &b.e));
}
inline void owned_beliefs(BandHandles& b, bpsched::RunResult& out, std::vector<double>& all, size_t at) {
  const size_t nloc = 2ull * b.info.local_rows * b.info.cols;
  std::vector<double> bel(nloc);
  check(bp_engine_beliefs(b.e, bel.data()));
  const size_t first = 2ull * b.info.ghost_up * b.info.cols, n = 2ull * (b.info.row1 - b.info.row0) * b.info.cols;
  std::copy(bel.begin() + first, bel.begin() + first + n, all.begin() + at);
  (void)out;
}
inline void fill_result(const bp_run_result& r, bpsched::RunResult& out) {
  out.converged = r.converged != 0;
  out.iterations = r.iterations;
  out.wall_time = r.wall_time;
  out.messages_updated_total = r.messages_updated_total;
}
}  // namespace detail

/// This rank's band of `graph` (any binary Ising lattice in generate_ising's
/// numbering), run with the other ranks: every rank calls it with the same
/// graph, config and NCCL id (bp_nccl_unique_id on one rank, broadcast by the
/// caller's launcher).  Owned beliefs equal the one-GPU run's bit for bit
/// (LBP, RnBP); RBP / RS use per-partition local frontiers.
inline BandRunResult run_band(const bpsched::PairwiseMRF& graph, const bpsched::SchedulerConfig& config,
                              uint32_t rank, uint32_t nranks, const uint8_t nccl_id[128], int device = -1) {
  config.validate();
  const HostArrays a(graph);
  const bp_sched_config c = to_c(config);
  detail::BandHandles b;
  detail::make_band(a, c, rank, nranks, device, b);
  bp_band_comm* comm = nullptr;
  check(bp_band_comm_create_nccl(nccl_id, rank, nranks, device, &comm));
  bp_run_result r{};
  bp_engine* e = b.e;
  const int rc = bp_band_run(&e, 1, comm, &r);
  bp_band_comm_destroy(comm);
  check(rc);
  BandRunResult out;
  detail::fill_result(r, out.result);
  out.row0 = b.info.row0;
  out.row1 = b.info.row1;
  out.cols = b.info.cols;
  std::vector<uint32_t> cards(static_cast<size_t>(b.info.row1 - b.info.row0) * b.info.cols, 2);
  out.result.beliefs = bpsched::BeliefTable(cards);
  std::vector<double> all(2 * cards.size());
  detail::owned_beliefs(b, out.result, all, 0);
  for (bpsched::vertex_id v = 0; v < cards.size(); ++v) {
    auto dst = out.result.beliefs.at(v);
    dst[0] = all[2 * v];
    dst[1] = all[2 * v + 1];
  }
  return out;
}

/// Every band of an `nparts`-way partition inside this process (on `device`),
/// assembled into the whole graph's RunResult: the partitioned loop without
/// NCCL (the parity harness runs it against bpsched::run).
inline bpsched::RunResult run_partitioned_local(const bpsched::PairwiseMRF& graph,
                                                const bpsched::SchedulerConfig& config, uint32_t nparts,
                                                int device = -1) {
  config.validate();
  const HostArrays a(graph);
  const bp_sched_config c = to_c(config);
  std::vector<std::unique_ptr<detail::BandHandles>> bands;
  std::vector<bp_engine*> es;
  for (uint32_t p = 0; p < nparts; ++p) {
    bands.push_back(std::make_unique<detail::BandHandles>());
    detail::make_band(a, c, p, nparts, device, *bands.back());
    es.push_back(bands.back()->e);
  }
  bp_band_comm* comm = nullptr;
  check(bp_band_comm_create_local(&comm));
  bp_run_result r{};
  const int rc = bp_band_run(es.data(), nparts, comm, &r);
  bp_band_comm_destroy(comm);
  check(rc);
  bpsched::RunResult out;
  detail::fill_result(r, out);
  std::vector<double> all(a.unary.size());
  for (auto& b : bands) detail::owned_beliefs(*b, out, all, 2ull * b->info.row0 * b->info.cols);
  out.beliefs = bpsched::BeliefTable(a.cards);
  for (bpsched::vertex_id v = 0; v < a.cards.size(); ++v) {
    auto dst = out.beliefs.at(v);
    dst[0] = all[2 * v];
    dst[1] = all[2 * v + 1];
  }
  return out;
}

/// Vertex-range partition of ANY binary model (random graphs included):
/// every part of an `nparts`-way partition inside this process, assembled into
/// the whole graph's RunResult (LBP, RnBP; bitwise the one-GPU run).  Part p
/// owns vertices [V p / P, V (p + 1) / P) (bp_graph_create_part).
inline bpsched::RunResult run_vertex_partitioned_local(const bpsched::PairwiseMRF& graph,
                                                       const bpsched::SchedulerConfig& config, uint32_t nparts,
                                                       int device = -1) {
  config.validate();
  const HostArrays a(graph);
  const bp_sched_config c = to_c(config);
  const bp_graph_desc d = a.desc();
  bp_device_opts o{device, 0};
  std::vector<std::unique_ptr<detail::BandHandles>> parts;
  std::vector<bp_part_info> infos(nparts);
  std::vector<bp_engine*> es;
  for (uint32_t p = 0; p < nparts; ++p) {
    parts.push_back(std::make_unique<detail::BandHandles>());
    check(bp_graph_create_part(&d, p, nparts, &o, &parts.back()->g, &infos[p]));
    check(bp_part_engine_create(parts.back()->g, &c, &parts.back()->e));
    es.push_back(parts.back()->e);
  }
  bp_band_comm* comm = nullptr;
  check(bp_band_comm_create_local(&comm));
  bp_run_result r{};
  const int rc = bp_band_run(es.data(), nparts, comm, &r);
  bp_band_comm_destroy(comm);
  check(rc);
  bpsched::RunResult out;
  detail::fill_result(r, out);
  out.beliefs = bpsched::BeliefTable(a.cards);
  for (uint32_t p = 0; p < nparts; ++p) {
    bp_graph_info gi{};
    check(bp_graph_info_get(parts[p]->g, &gi));
    std::vector<double> bel(2ull * gi.num_vertices);
    check(bp_engine_beliefs(parts[p]->e, bel.data()));
    for (uint32_t v = infos[p].v0; v < infos[p].v1; ++v) {  // local ids [0, v1 - v0) are the owned vertices
      auto dst = out.beliefs.at(v);
      dst[0] = bel[2ull * (v - infos[p].v0)];
      dst[1] = bel[2ull * (v - infos[p].v0) + 1];
    }
  }
  return out;
}

}  // namespace bpsched_cuda

#endif  // BPSCHED_CUDA_HPP
