// TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrapper over the UNMODIFIED reference library, compiled from
// /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/libbpsched_ref.so.  It exposes the reference through the same
// signatures as oracle/bp_oracle.h (prefix ref_ instead of orc_) so the tests
// can drive the reference, the C restatement and the CUDA engine with one
// harness, and so bench.py --impl reference can time the reference's own
// bpsched::run on this host.  Nothing here is product code.
#include <bpsched/errors.hpp>
#include <bpsched/generators.hpp>
#include <bpsched/messages.hpp>
#include <bpsched/model_io.hpp>
#include <bpsched/mrf.hpp>
#include <bpsched/schedulers.hpp>

#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "bp_oracle.h"

using namespace bpsched;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return ORC_OK;
  } catch (const numeric_error& e) {
    g_err = e.what();
    return ORC_NUMERIC;
  } catch (const parse_error& e) {
    g_err = e.what();
    return 8;  // the engine's BP_ERR_PARSE
  } catch (const model_error& e) {
    g_err = e.what();
    return ORC_MODEL;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return ORC_INVALID_ARGUMENT;
  } catch (const std::bad_alloc& e) {
    g_err = e.what();
    return ORC_NOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ORC_INVALID_ARGUMENT;
  }
}

SchedulerConfig to_config(const orc_config* c) {
  SchedulerConfig cfg;
  switch (c->kind) {
    case ORC_LBP: cfg.kind = SchedulerKind::lbp; break;
    case ORC_SRBP: cfg.kind = SchedulerKind::serial_rbp; break;
    case ORC_RBP: cfg.kind = SchedulerKind::rbp; break;
    case ORC_RS: cfg.kind = SchedulerKind::rs; break;
    case ORC_RNBP: cfg.kind = SchedulerKind::rnbp; break;
    default: throw std::invalid_argument("unknown scheduler");
  }
  cfg.epsilon = c->epsilon;
  cfg.p = c->p;
  cfg.splash_depth = c->splash_depth;
  cfg.low_p = c->low_p;
  cfg.high_p = c->high_p;
  cfg.edge_ratio_threshold = c->edge_ratio_threshold;
  cfg.max_iterations = c->max_iterations;
  cfg.time_limit = c->time_limit;
  cfg.seed = c->seed;
  cfg.worker_count = c->worker_count;
  return cfg;
}

}  // namespace

struct ref_graph {
  PairwiseMRF g;
};
struct ref_engine {
  std::unique_ptr<EngineState> st;
  SchedulerConfig cfg;
};

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_graph_create(uint32_t V, const uint32_t* cards, const double* unary, uint32_t E,
                     const uint32_t* ep, const double* tables, ref_graph** out) {
  *out = nullptr;
  return guarded([&] {
    std::vector<uint32_t> c(cards, cards + V);
    std::vector<std::vector<double>> u(V);
    size_t off = 0;
    for (uint32_t v = 0; v < V; ++v) {
      u[v].assign(unary + off, unary + off + cards[v]);
      off += cards[v];
    }
    std::vector<PairwiseMRF::EdgeSpec> edges(E);
    size_t toff = 0;
    for (uint32_t e = 0; e < E; ++e) {
      const uint32_t i = ep[2 * e], j = ep[2 * e + 1];
      const size_t n = (i < V && j < V) ? static_cast<size_t>(cards[i]) * cards[j] : 0;
      edges[e] = {i, j, std::vector<double>(tables + toff, tables + toff + n)};
      toff += n;
    }
    *out = new ref_graph{build_graph(std::move(c), std::move(u), std::move(edges))};
  });
}

void ref_graph_destroy(ref_graph* g) { delete g; }

// parse_model / serialize_model (model_io.cpp:98-181), for the .pgm ingest tests
int ref_parse_model(const char* text, uint64_t len, ref_graph** out) {
  *out = nullptr;
  return guarded([&] { *out = new ref_graph{parse_model(std::string_view(text, len))}; });
}
uint64_t ref_serialize_model(const ref_graph* g, char* buf, uint64_t cap) {
  const std::string s = serialize_model(g->g);
  if (buf && cap >= s.size()) std::memcpy(buf, s.data(), s.size());
  return s.size();
}
uint32_t ref_graph_num_vertices(const ref_graph* g) { return g->g.num_vertices(); }
uint32_t ref_graph_num_edges(const ref_graph* g) { return g->g.num_edges(); }

uint64_t ref_graph_unary_size(const ref_graph* g) {
  uint64_t n = 0;
  for (vertex_id v = 0; v < g->g.num_vertices(); ++v) n += g->g.cardinality(v);
  return n;
}
uint64_t ref_graph_table_size(const ref_graph* g) {
  uint64_t n = 0;
  for (edge_id e = 0; e < g->g.num_edges(); ++e) n += g->g.pairwise(e).size();
  return n;
}

void ref_graph_export(const ref_graph* rg, uint32_t* cards, double* unary, uint32_t* ep,
                      double* tables) {
  const PairwiseMRF& g = rg->g;
  size_t uo = 0, to = 0;
  for (vertex_id v = 0; v < g.num_vertices(); ++v) {
    if (cards) cards[v] = g.cardinality(v);
    for (double x : g.unary(v)) {
      if (unary) unary[uo] = x;
      ++uo;
    }
  }
  for (edge_id e = 0; e < g.num_edges(); ++e) {
    const auto [i, j] = g.edge_endpoints(e);
    if (ep) {
      ep[2 * e] = i;
      ep[2 * e + 1] = j;
    }
    for (double x : g.pairwise(e)) {
      if (tables) tables[to] = x;
      ++to;
    }
  }
}

void ref_graph_incoming(const ref_graph* rg, uint64_t* offsets, uint32_t* adjacency) {
  const PairwiseMRF& g = rg->g;
  uint64_t o = 0;
  for (vertex_id v = 0; v < g.num_vertices(); ++v) {
    offsets[v] = o;
    for (directed_edge_id d : g.incoming(v)) adjacency[o++] = d;
  }
  offsets[g.num_vertices()] = o;
}

int ref_generate_ising(uint32_t n, double c, uint64_t seed, ref_graph** out) {
  return guarded([&] { *out = new ref_graph{generate_ising({n, c, seed})}; });
}
int ref_generate_chain(uint32_t length, double c, uint64_t seed, ref_graph** out) {
  return guarded([&] { *out = new ref_graph{generate_chain({length, c, seed})}; });
}

void ref_mt_draws(uint64_t seed, uint64_t count, uint64_t* out_raw, double* out_unit) {
  std::mt19937_64 rng(seed);
  for (uint64_t i = 0; i < count; ++i) {
    std::mt19937_64 copy = rng;
    const uint64_t x = rng();
    if (out_raw) out_raw[i] = x;
    if (out_unit) out_unit[i] = uniform_unit(copy);
  }
}

int ref_validate_config(const orc_config* c) {
  return guarded([&] { to_config(c).validate(); });
}

double ref_select_parallelism(uint32_t prev, uint32_t now, const orc_config* c) {
  return select_parallelism(prev, now, to_config(c));
}

int ref_run(const ref_graph* g, const orc_config* c, orc_result* res, double* beliefs,
            orc_record* trace, uint64_t trace_cap) {
  std::memset(res, 0, sizeof *res);
  return guarded([&] {
    const RunResult r = run(g->g, to_config(c));
    res->converged = r.converged ? 1 : 0;
    res->iterations = r.iterations;
    res->wall_time = r.wall_time;
    res->messages_updated_total = r.messages_updated_total;
    res->trace_len = r.trace.size();
    if (beliefs) {
      size_t o = 0;
      for (vertex_id v = 0; v < g->g.num_vertices(); ++v)
        for (double x : r.beliefs.at(v)) beliefs[o++] = x;
    }
    if (trace) {
      for (size_t k = 0; k < r.trace.size() && k < trace_cap; ++k) {
        trace[k].iteration = r.trace[k].iteration;
        trace[k].frontier_size = r.trace[k].frontier_size;
        trace[k].unconverged = r.trace[k].unconverged;
        trace[k].elapsed_seconds = r.trace[k].elapsed_seconds;
      }
    }
  });
}

int ref_engine_create(const ref_graph* g, const orc_config* c, ref_engine** out) {
  *out = nullptr;
  return guarded([&] {
    auto e = std::make_unique<ref_engine>();
    e->cfg = to_config(c);
    e->st = std::make_unique<EngineState>(g->g, e->cfg);
    *out = e.release();
  });
}
void ref_engine_destroy(ref_engine* e) { delete e; }
uint32_t ref_engine_unconverged(const ref_engine* e) { return e->st->tracker().unconverged_count(); }
uint64_t ref_engine_iteration(const ref_engine* e) { return e->st->iteration(); }
void ref_engine_advance(ref_engine* e) { e->st->advance_iteration(); }

void ref_engine_messages(const ref_engine* e, double* out) {
  size_t o = 0;
  for (directed_edge_id d = 0; d < e->st->graph().num_directed_edges(); ++d)
    for (double x : e->st->messages().view(d)) out[o++] = x;
}
void ref_engine_candidates(const ref_engine* e, double* out) {
  size_t o = 0;
  for (directed_edge_id d = 0; d < e->st->graph().num_directed_edges(); ++d)
    for (double x : e->st->tracker().candidate(d)) out[o++] = x;
}
void ref_engine_residuals(const ref_engine* e, double* out) {
  const auto r = e->st->tracker().residuals();
  std::memcpy(out, r.data(), sizeof(double) * r.size());
}

int ref_engine_apply_frontier(ref_engine* e, const uint32_t* f, uint64_t n) {
  return guarded([&] { apply_frontier(*e->st, std::span<const directed_edge_id>(f, n)); });
}
void ref_engine_frontier_lbp(const ref_engine* e, uint32_t* out, uint64_t* n) {
  const auto f = frontier_lbp(*e->st);
  std::memcpy(out, f.data(), sizeof(uint32_t) * f.size());
  *n = f.size();
}
void ref_engine_rbp_frontier(const ref_engine* e, double p, uint32_t* out, uint64_t* n) {
  const auto f = rbp_frontier(*e->st, p);
  std::memcpy(out, f.data(), sizeof(uint32_t) * f.size());
  *n = f.size();
}
void ref_engine_rnbp_frontier(ref_engine* e, double p, uint32_t* out, uint64_t* n) {
  const auto f = rnbp_frontier(*e->st, p, e->st->rng());
  std::memcpy(out, f.data(), sizeof(uint32_t) * f.size());
  *n = f.size();
}
int ref_engine_rs_frontier(ref_engine* e, double p, uint32_t h, uint32_t* roots, uint64_t* eoff,
                           uint32_t* edges, uint64_t* num) {
  return guarded([&] {
    const auto s = rs_frontier(*e->st, p, h);
    eoff[0] = 0;
    uint64_t o = 0;
    for (size_t k = 0; k < s.size(); ++k) {
      roots[k] = s[k].root;
      for (directed_edge_id d : s[k].edges) edges[o++] = d;
      eoff[k + 1] = o;
    }
    *num = s.size();
  });
}
int ref_engine_apply_splashes(ref_engine* e, uint64_t ns, const uint32_t* roots,
                              const uint64_t* eoff, const uint32_t* edges) {
  return guarded([&] {
    std::vector<Splash> s(ns);
    for (uint64_t k = 0; k < ns; ++k) {
      s[k].root = roots[k];
      s[k].edges.assign(edges + eoff[k], edges + eoff[k + 1]);
    }
    apply_splash_frontier(*e->st, s);
  });
}
int ref_engine_beliefs(const ref_engine* e, double* out) {
  return guarded([&] {
    const BeliefTable b = compute_beliefs(e->st->graph(), e->st->messages());
    size_t o = 0;
    for (vertex_id v = 0; v < b.num_vertices(); ++v)
      for (double x : b.at(v)) out[o++] = x;
  });
}
int ref_engine_update_message(const ref_engine* e, uint32_t d, double* out) {
  return guarded([&] {
    const auto m = update_message(e->st->graph(), e->st->messages(), d);
    std::memcpy(out, m.data(), sizeof(double) * m.size());
  });
}
int ref_engine_build_splash(const ref_engine* e, uint32_t root, uint32_t h, uint32_t* claimed,
                            uint32_t* edges, uint64_t* n) {
  return guarded([&] {
    std::vector<vertex_id> cl(claimed, claimed + e->st->graph().num_vertices());
    const Splash s = build_splash(*e->st, root, h, cl);
    std::memcpy(claimed, cl.data(), cl.size() * 4);
    std::memcpy(edges, s.edges.data(), s.edges.size() * 4);
    *n = s.edges.size();
  });
}

void ref_select_top_k(const double* r, uint64_t m, uint64_t k, uint32_t* out, uint64_t* n) {
  const auto f = select_top_k(std::span<const double>(r, m), k);
  std::memcpy(out, f.data(), sizeof(uint32_t) * f.size());
  *n = f.size();
}

}  // extern "C"
