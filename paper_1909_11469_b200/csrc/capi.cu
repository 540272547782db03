// extern "C" boundary (include/bp_cuda.h): exceptions -> bp_status codes,
// message kept per thread (errors.hpp:10-38 -> return codes).
#include <algorithm>
#include <cstring>
#include <string>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include "bp_device.cuh"
#include "engine.hpp"
#include "graph.hpp"
#include "partition.hpp"

struct bp_graph {
  std::unique_ptr<bpb::GraphImpl> impl;
};
struct bp_engine {
  std::unique_ptr<bpb::EngineBase> e;
  const bp_graph* g;
  bp_sched_config cfg;
  std::unique_ptr<bpb::Band> band;  // row-band engines: halo buffers, info, stream
};
struct bp_band_comm {
  std::unique_ptr<bpb::BandComm> c;
};

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return BP_OK;
  } catch (const bpb::Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_last_error = std::string("host allocation failed: ") + e.what();
    return BP_ERR_OOM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return BP_ERR_INVALID_ARGUMENT;
  }
}

// the device's Philox4x32-10 (bp_device.cuh), evaluated for known-answer tests
__global__ void k_philox_kat(uint64_t n, const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const uint4 r = bpb::philox4x32_10(make_uint4(ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]),
                                     make_uint2(key[2 * i], key[2 * i + 1]));
  out[4 * i] = r.x;
  out[4 * i + 1] = r.y;
  out[4 * i + 2] = r.z;
  out[4 * i + 3] = r.w;
}
__global__ void k_philox_u53(uint64_t seed, uint64_t iteration, uint32_t attempt, uint64_t n, const uint64_t* d,
                             uint64_t* out) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = bpb::philox_u53(seed, iteration, attempt, d[i]);
}

int wrap_graph(std::unique_ptr<bpb::GraphImpl> g, bp_graph** out) {
  *out = new bp_graph{std::move(g)};
  return BP_OK;
}

}  // namespace

extern "C" {

const char* bp_last_error(void) { return g_last_error.c_str(); }
int bp_abi_version(void) { return BP_CUDA_ABI_VERSION; }

int bp_graph_create(const bp_graph_desc* desc, const bp_device_opts* opts, bp_graph** out) {
  if (!out) return BP_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  return guarded([&] { wrap_graph(bpb::build_from_desc(desc, opts), out); });
}

int bp_graph_generate_ising(uint32_t n, double c, uint64_t seed, const bp_device_opts* opts, bp_graph** out) {
  if (!out) return BP_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  return guarded([&] { wrap_graph(bpb::build_lattice_binary(n, n, bpb::ising_streams(n, c, seed), opts), out); });
}

int bp_graph_generate_chain(uint32_t length, double c, uint64_t seed, const bp_device_opts* opts, bp_graph** out) {
  if (!out) return BP_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  return guarded([&] {
    wrap_graph(bpb::build_lattice_binary(length ? 1 : 0, length, bpb::chain_streams(length, c, seed), opts), out);
  });
}

int bp_graph_generate_potts(uint32_t n, uint32_t q, double c, uint64_t seed, const bp_device_opts* opts,
                            bp_graph** out) {
  if (!out) return BP_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  return guarded([&] { wrap_graph(bpb::build_potts(n, q, bpb::potts_streams(n, q, c, seed), opts), out); });
}

int bp_graph_generate_er(uint32_t n, uint32_t m, double c, uint64_t seed, const bp_device_opts* opts,
                         bp_graph** out) {
  if (!out) return BP_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  return guarded([&] { wrap_graph(bpb::build_er(n, bpb::er_instance(n, m, c, seed), opts), out); });
}

int bp_generate_ising_arrays(uint32_t n, double c, uint64_t seed, uint32_t* cards, double* unary, uint32_t* ep,
                             double* tables) {
  if (!cards || !unary || (n > 1 && (!ep || !tables))) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    std::vector<uint32_t> cv, ev;
    std::vector<double> uv, tv;
    bpb::ising_desc_arrays(n, n, c, seed, cv, uv, ev, tv);
    std::memcpy(cards, cv.data(), cv.size() * 4);
    std::memcpy(unary, uv.data(), uv.size() * 8);
    if (!ev.empty()) std::memcpy(ep, ev.data(), ev.size() * 4);
    if (!tv.empty()) std::memcpy(tables, tv.data(), tv.size() * 8);
  });
}

int bp_generate_er_arrays(uint32_t n, uint32_t m, double c, uint64_t seed, uint32_t* cards, double* unary,
                          uint32_t* ep, double* tables) {
  if ((n && (!cards || !unary)) || (m && (!ep || !tables))) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    std::vector<uint32_t> cv, ev;
    std::vector<double> uv, tv;
    bpb::er_desc_arrays(n, m, c, seed, cv, uv, ev, tv);
    if (!cv.empty()) std::memcpy(cards, cv.data(), cv.size() * 4);
    if (!uv.empty()) std::memcpy(unary, uv.data(), uv.size() * 8);
    if (!ev.empty()) std::memcpy(ep, ev.data(), ev.size() * 4);
    if (!tv.empty()) std::memcpy(tables, tv.data(), tv.size() * 8);
  });
}

struct bp_pgm {
  bpb::PgmArrays a;
};
int bp_pgm_parse(const char* text, uint64_t len, bp_pgm** out) {
  if (!out || (!text && len)) return BP_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  return guarded([&] {
    auto m = std::make_unique<bp_pgm>();
    bpb::parse_pgm(text ? text : "", len, m->a);
    *out = m.release();
  });
}
int bp_pgm_info(const bp_pgm* m, uint32_t* V, uint32_t* E, uint64_t* nu, uint64_t* nt) {
  if (!m) return BP_ERR_INVALID_ARGUMENT;
  if (V) *V = static_cast<uint32_t>(m->a.cards.size());
  if (E) *E = static_cast<uint32_t>(m->a.ep.size() / 2);
  if (nu) *nu = m->a.unary.size();
  if (nt) *nt = m->a.tables.size();
  return BP_OK;
}
int bp_pgm_arrays(const bp_pgm* m, uint32_t* cards, double* unary, uint32_t* ep, double* tables) {
  if (!m) return BP_ERR_INVALID_ARGUMENT;
  auto put = [](auto* dst, const auto& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
  };
  put(cards, m->a.cards);
  put(unary, m->a.unary);
  put(ep, m->a.ep);
  put(tables, m->a.tables);
  return BP_OK;
}
void bp_pgm_destroy(bp_pgm* m) { delete m; }
int bp_graph_create_pgm(const char* text, uint64_t len, const bp_device_opts* opts, bp_graph** out) {
  if (!out || (!text && len)) return BP_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  return guarded([&] {
    bpb::PgmArrays a;
    bpb::parse_pgm(text ? text : "", len, a);
    const bp_graph_desc d{static_cast<uint32_t>(a.cards.size()), static_cast<uint32_t>(a.ep.size() / 2),
                          a.cards.data(), a.unary.data(), a.ep.data(), a.tables.data()};
    *out = new bp_graph{bpb::build_from_desc(&d, opts)};
  });
}

void bp_graph_destroy(bp_graph* g) { delete g; }

int bp_graph_info_get(const bp_graph* g, bp_graph_info* info) {
  if (!g || !info) return BP_ERR_INVALID_ARGUMENT;
  const auto& G = *g->impl;
  info->num_vertices = G.V;
  info->num_edges = G.E;
  info->max_cardinality = G.maxq;
  info->state_stride = G.qs;
  info->device_bytes = G.device_bytes();
  info->device = G.device;
  info->layout = G.binary ? 0u : 1u;
  if (G.binary) {
    info->message_values = 4ull * G.E;
  } else {
    uint64_t n = 0;
    const auto& ep = G.host_ep();
    for (uint64_t d = 0; d < 2ull * G.E; ++d) n += G.card_of(ep[d ^ 1ull]);
    info->message_values = n;
  }
  return BP_OK;
}

int bp_validate_config(const bp_sched_config* cfg) {
  if (!cfg) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { bpb::validate_config(*cfg); });
}

double bp_select_parallelism(uint32_t prev, uint32_t now, const bp_sched_config* cfg) {
  return bpb::select_parallelism_host(prev, now, *cfg);
}

int bp_run_ex(const bp_graph* g, const bp_sched_config* cfg, const bp_run_opts* opts, bp_run_result* result,
              double* beliefs_out, bp_iter_record* trace_out, uint64_t trace_cap) {
  if (!g || !cfg || !result) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    bpb::validate_config(*cfg);
    if (cfg->kind == BP_SERIAL_RBP)
      throw bpb::Error(BP_ERR_UNSUPPORTED,
                       "serial RBP is strictly sequential and is not offloaded (use the reference run_serial_rbp)");
    static const bool dbg = std::getenv("BPB_DEBUG_BUILD") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    auto e = bpb::make_engine(*g->impl, *cfg);
    const auto t1 = std::chrono::steady_clock::now();
    e->run(opts, result, beliefs_out, trace_out, trace_cap);
    const auto t2 = std::chrono::steady_clock::now();
    e.reset();
    if (dbg) {
      const auto t3 = std::chrono::steady_clock::now();
      auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
      std::fprintf(stderr, "bp_run: engine %.2f ms, run %.2f ms (device %.2f), teardown %.2f ms\n", ms(t0, t1),
                   ms(t1, t2), result->device_ms, ms(t2, t3));
    }
  });
}

int bp_run(const bp_graph* g, const bp_sched_config* cfg, bp_run_result* result, double* beliefs_out,
           bp_iter_record* trace_out, uint64_t trace_cap) {
  return bp_run_ex(g, cfg, nullptr, result, beliefs_out, trace_out, trace_cap);
}

int bp_engine_create(const bp_graph* g, const bp_sched_config* cfg, bp_engine** out) {
  if (!g || !cfg || !out) return BP_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  return guarded([&] {
    bpb::validate_config(*cfg);
    auto e = bpb::make_engine(*g->impl, *cfg);
    e->lockstep_init();
    *out = new bp_engine{std::move(e), g, *cfg};
  });
}

void bp_engine_destroy(bp_engine* e) { delete e; }

int bp_engine_unconverged(const bp_engine* e, uint32_t* out) {
  if (!e || !out) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { *out = e->e->unconverged(); });
}
int bp_engine_advance_iteration(bp_engine* e) {
  if (!e) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { e->e->advance_iteration(); });
}
int bp_engine_iteration(const bp_engine* e, uint64_t* out) {
  if (!e || !out) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { *out = e->e->iteration(); });
}
int bp_engine_messages(const bp_engine* e, double* out) {
  if (!e || !out) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { e->e->messages(out, false); });
}
int bp_engine_candidates(const bp_engine* e, double* out) {
  if (!e || !out) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { e->e->messages(out, true); });
}
int bp_engine_residuals(const bp_engine* e, double* out) {
  if (!e || !out) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { e->e->residuals(out); });
}
int bp_engine_beliefs(const bp_engine* e, double* out) {
  if (!e || !out) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { e->e->beliefs(out); });
}
int bp_engine_apply_frontier(bp_engine* e, const uint32_t* frontier, uint64_t n) {
  if (!e || (n && !frontier)) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { e->e->apply_frontier(frontier, n); });
}
int bp_engine_apply_splashes(bp_engine* e, uint64_t ns, const uint32_t* roots, const uint64_t* eoff,
                             const uint32_t* edges) {
  if (!e) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { e->e->apply_splashes(ns, roots, eoff, edges); });
}
int bp_engine_rnbp_frontier(bp_engine* e, double p, uint32_t* out, uint64_t* n) {
  if (!e || !out || !n) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    std::vector<uint32_t> f;
    e->e->rnbp_frontier(p, f);
    std::memcpy(out, f.data(), f.size() * 4);
    *n = f.size();
  });
}
int bp_engine_rbp_frontier(bp_engine* e, double p, uint32_t* out, uint64_t* n) {
  if (!e || !out || !n) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    std::vector<uint32_t> f;
    e->e->rbp_frontier(p, f);
    std::memcpy(out, f.data(), f.size() * 4);
    *n = f.size();
  });
}
int bp_engine_rs_frontier(bp_engine* e, double p, uint32_t h, uint32_t* roots, uint64_t* eoff, uint32_t* edges,
                          uint64_t* ns) {
  if (!e || !roots || !eoff || !edges || !ns) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    std::vector<uint32_t> r, ed;
    std::vector<uint64_t> o;
    e->e->rs_frontier(p, h, r, o, ed);
    std::memcpy(roots, r.data(), r.size() * 4);
    std::memcpy(eoff, o.data(), o.size() * 8);
    std::memcpy(edges, ed.data(), ed.size() * 4);
    *ns = r.size();
  });
}
int bp_graph_generate_ising_band(uint32_t n, double c, uint64_t seed, uint32_t part, uint32_t nparts,
                                 const bp_device_opts* opts, bp_graph** out, bp_band_info* info) {
  if (!out || !info) return BP_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  return guarded([&] {
    if (nparts == 0 || part >= nparts || nparts > n) throw bpb::Error(BP_ERR_INVALID_ARGUMENT, "bad band partition");
    const uint32_t r0 = static_cast<uint32_t>(static_cast<uint64_t>(part) * n / nparts);
    const uint32_t r1 = static_cast<uint32_t>(static_cast<uint64_t>(part + 1) * n / nparts);
    const uint32_t gu = part > 0 ? 1u : 0u, gd = part + 1 < nparts ? 1u : 0u;
    auto g = bpb::build_lattice_binary(r1 + gd - (r0 - gu), n, bpb::ising_band_streams(n, c, seed, r0 - gu, r1 + gd),
                                       opts);
    g->cnt_row0 = gu;
    g->cnt_row1 = gu + (r1 - r0);
    uint64_t owned = 0;  // sum of degrees of the owned vertices in the full grid
    for (uint32_t r = r0; r < r1; ++r)
      owned += static_cast<uint64_t>(n) * ((r > 0) + (r + 1 < n)) + 2ull * (n - 1);
    g->owned_directed = owned;
    g->edge_offset = static_cast<uint64_t>(r0 - gu) * (2ull * n - 1ull);
    *info = bp_band_info{part, nparts, r0, r1, gu, gd, r1 + gd - (r0 - gu), n, owned};
    wrap_graph(std::move(g), out);
  });
}

int bp_band_engine_create(const bp_graph* g, const bp_sched_config* cfg, const bp_band_info* info,
                          const bp_halo_buffers* bufs, bp_engine** out) {
  if (!g || !cfg || !info || !bufs || !out) return BP_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  return guarded([&] {
    bpb::validate_config(*cfg);
    auto e = bpb::make_engine(*g->impl, *cfg);
    bpb::PartHalo h{};
    h.send_up = bufs->send_up;
    h.send_down = bufs->send_down;
    h.recv_up = bufs->recv_up;
    h.recv_down = bufs->recv_down;
    h.count = bufs->count;
    e->band_config(h, info->owned_directed);
    auto band = std::make_unique<bpb::Band>();
    band->engine = e.get();
    band->info = *info;
    band->cfg = *cfg;
    band->stream = e->stream();
    band->halo = h;
    band->lattice_peers();
    *out = new bp_engine{std::move(e), g, *cfg, std::move(band)};
  });
}

int bp_band_engine_create_owned(const bp_graph* g, const bp_sched_config* cfg, const bp_band_info* info,
                                bp_engine** out) {
  if (!g || !cfg || !info || !out) return BP_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  return guarded([&] {
    bpb::validate_config(*cfg);
    auto band = std::make_unique<bpb::Band>();
    for (int k = 0; k < 4; ++k) band->own[k].alloc(4ull * info->cols);  // zero-filled, completed
    band->own[4].alloc(8ull * 5);
    bpb::PartHalo h{};
    h.send_up = band->own[0].as<float>();
    h.send_down = band->own[1].as<float>();
    h.recv_up = band->own[2].as<float>();
    h.recv_down = band->own[3].as<float>();
    h.count = band->own[4].as<unsigned long long>();
    auto e = bpb::make_engine(*g->impl, *cfg);
    e->band_config(h, info->owned_directed);
    band->engine = e.get();
    band->info = *info;
    band->cfg = *cfg;
    band->stream = e->stream();
    band->halo = h;
    band->lattice_peers();
    *out = new bp_engine{std::move(e), g, *cfg, std::move(band)};
  });
}

int bp_graph_create_part(const bp_graph_desc* d, uint32_t part, uint32_t nparts, const bp_device_opts* opts,
                         bp_graph** out, bp_part_info* info) {
  if (!d || !out || !info) return BP_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  return guarded([&] {
    bpb::PartLayout L{};
    auto g = bpb::build_part(d, part, nparts, opts, L);
    *info = bp_part_info{L.part, L.nparts, L.v0, L.v1, L.ghost_vertices, L.local_edges, L.peers, 0,
                         L.send_messages, L.recv_messages, L.owned_directed};
    *out = new bp_graph{std::move(g)};
  });
}

int bp_part_engine_create(const bp_graph* g, const bp_sched_config* cfg, bp_engine** out) {
  if (!g || !cfg || !out) return BP_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  return guarded([&] {
    const bpb::GraphImpl& gi = *g->impl;
    if (!gi.nparts) throw bpb::Error(BP_ERR_INVALID_ARGUMENT, "not a partition graph (bp_graph_create_part)");
    bpb::validate_config(*cfg);
    uint64_t ns = 0, nr = 0;
    for (const auto& p : gi.peers) {
      ns += p.send_n;
      nr += p.recv_n;
    }
    auto band = std::make_unique<bpb::Band>();
    band->own[0].alloc(4 * std::max<uint64_t>(ns, 1));  // every peer's send run back to back
    band->own[2].alloc(4 * std::max<uint64_t>(nr, 1));  // every peer's recv run back to back
    band->own[4].alloc(8ull * 5);
    bpb::PartHalo h{};
    h.send_up = band->own[0].as<float>();
    h.recv_up = band->own[2].as<float>();
    h.count = band->own[4].as<unsigned long long>();
    auto e = bpb::make_engine(gi, *cfg);
    e->band_config(h, gi.owned_directed);
    band->engine = e.get();
    band->info = bp_band_info{gi.part, gi.nparts, 0, 0, 0, 0, 0, 0, gi.owned_directed};
    band->cfg = *cfg;
    band->stream = e->stream();
    band->halo = h;
    for (const auto& p : gi.peers)
      band->peers.push_back({p.part, h.send_up + p.send_off, p.send_n, const_cast<float*>(h.recv_up) + p.recv_off,
                             p.recv_n});
    *out = new bp_engine{std::move(e), g, *cfg, std::move(band)};
  });
}

int bp_graph_create_band(const bp_graph_desc* d, uint32_t part, uint32_t nparts, const bp_device_opts* opts,
                         bp_graph** out, bp_band_info* info) {
  if (!d || !out || !info) return BP_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  return guarded([&] {
    const uint32_t V = d->num_vertices, E = d->num_edges;
    const uint32_t C = E && d->edge_endpoints ? bpb::lattice_cols(V, E, d->edge_endpoints) : 0;
    if (!C || V % C) throw bpb::Error(BP_ERR_UNSUPPORTED, "row-band partition needs a lattice in generate_ising's numbering");
    const uint32_t R = V / C;
    if (nparts == 0 || part >= nparts || nparts > R) throw bpb::Error(BP_ERR_INVALID_ARGUMENT, "bad band partition");
    for (uint32_t v = 0; v < V; ++v)
      if (d->cardinalities[v] != 2) throw bpb::Error(BP_ERR_UNSUPPORTED, "row-band partition: binary lattices only");
    const uint32_t r0 = static_cast<uint32_t>(static_cast<uint64_t>(part) * R / nparts);
    const uint32_t r1 = static_cast<uint32_t>(static_cast<uint64_t>(part + 1) * R / nparts);
    const uint32_t gu = part > 0 ? 1u : 0u, gd = part + 1 < nparts ? 1u : 0u;
    const uint32_t lo = r0 - gu, hi = r1 + gd, L = hi - lo;
    // the local L x C lattice: full edge blocks of rows lo .. hi-2, the right
    // edges of row hi-1 (generators.cpp:37-43 numbering, relabelled)
    std::vector<uint32_t> cards(static_cast<size_t>(L) * C, 2), ep;
    std::vector<double> un(d->unary_values + 2ull * lo * C, d->unary_values + 2ull * hi * C), tb;
    const uint64_t row_edges = 2ull * C - 1ull;
    auto take = [&](uint64_t ge) {
      ep.push_back(d->edge_endpoints[2 * ge] - lo * C);
      ep.push_back(d->edge_endpoints[2 * ge + 1] - lo * C);
      tb.insert(tb.end(), d->pairwise_values + 4 * ge, d->pairwise_values + 4 * ge + 4);
    };
    for (uint32_t r = lo; r + 1 < hi; ++r)
      for (uint64_t k = 0; k < row_edges; ++k) take(static_cast<uint64_t>(r) * row_edges + k);
    const uint64_t last = static_cast<uint64_t>(hi - 1) * row_edges;
    for (uint32_t c = 0; c + 1 < C; ++c) take(hi == R ? last + c : last + 2ull * c);
    bp_graph_desc ld{L * C, static_cast<uint32_t>(ep.size() / 2), cards.data(), un.data(), ep.data(), tb.data()};
    auto g = bpb::build_from_desc(&ld, opts);
    if (g->lat_cols != C || !g->binary || g->par_mode != 1)
      throw bpb::Error(BP_ERR_UNSUPPORTED, "row-band partition needs Ising tables {a, d, d, a}");
    g->cnt_row0 = gu;
    g->cnt_row1 = gu + (r1 - r0);
    uint64_t owned = 0;  // sum of the owned vertices' degrees in the full lattice
    for (uint32_t r = r0; r < r1; ++r) owned += static_cast<uint64_t>(C) * ((r > 0) + (r + 1 < R)) + 2ull * (C - 1);
    g->owned_directed = owned;
    g->edge_offset = static_cast<uint64_t>(lo) * row_edges;
    *info = bp_band_info{part, nparts, r0, r1, gu, gd, L, C, owned};
    wrap_graph(std::move(g), out);
  });
}

int bp_nccl_unique_id(uint8_t* id) {
  if (!id) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { bpb::nccl_unique_id(id); });
}

int bp_band_comm_create_nccl(const uint8_t* id, uint32_t rank, uint32_t nranks, int32_t device, bp_band_comm** out) {
  if (!id || !out || rank >= nranks) return BP_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  return guarded([&] {
    int dev = device;
    if (dev < 0) bpb::cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    *out = new bp_band_comm{std::unique_ptr<bpb::BandComm>(bpb::make_nccl_comm(id, static_cast<int>(rank),
                                                                                   static_cast<int>(nranks), dev))};
  });
}

int bp_band_comm_create_local(bp_band_comm** out) {
  if (!out) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { *out = new bp_band_comm{std::unique_ptr<bpb::BandComm>(bpb::make_local_comm())}; });
}

void bp_band_comm_destroy(bp_band_comm* c) { delete c; }

int bp_band_run(bp_engine* const* bands, uint32_t nbands, bp_band_comm* comm, bp_run_result* result) {
  if (!bands || !nbands || !comm || !result) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    std::vector<bpb::Band*> b;
    for (uint32_t i = 0; i < nbands; ++i) {
      if (!bands[i] || !bands[i]->band) throw bpb::Error(BP_ERR_INVALID_ARGUMENT, "not a band engine");
      b.push_back(bands[i]->band.get());
    }
    bpb::run_bands(b, *comm->c, result);
  });
}

int bp_band_stream(const bp_engine* e, uint64_t* stream) {
  if (!e || !stream) return BP_ERR_INVALID_ARGUMENT;
  *stream = reinterpret_cast<uint64_t>(e->e->stream());
  return BP_OK;
}
int bp_band_lbp_sweep(bp_engine* e) {
  if (!e) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { e->e->band_sweep(); });
}
int bp_band_lbp_finish(bp_engine* e) {
  if (!e) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { e->e->band_finish(); });
}
int bp_band_status(bp_engine* e, bp_run_result* r) {
  if (!e || !r) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { e->e->band_status(r); });
}

int bp_band_rnbp_begin(bp_engine* e) {
  if (!e) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { e->e->band_rnbp_begin(); });
}
int bp_band_rnbp_finish_init(bp_engine* e) {
  if (!e) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { e->e->band_rnbp_finish_init(); });
}
int bp_band_rnbp_select(bp_engine* e, uint32_t attempt) {
  if (!e || attempt > 1) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { e->e->band_rnbp_select(attempt); });
}
int bp_band_rbp_select(bp_engine* e) {
  if (!e) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { e->e->band_rbp_select(); });
}
int bp_band_rs_select(bp_engine* e) {
  if (!e) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { e->e->band_rs_select(); });
}
int bp_band_rnbp_refresh(bp_engine* e) {
  if (!e) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { e->e->band_rnbp_refresh(); });
}
int bp_band_rnbp_finish(bp_engine* e) {
  if (!e) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] { e->e->band_rnbp_finish(); });
}
int bp_band_survivors(bp_engine* e, uint64_t* ids, uint64_t cap, uint64_t* n) {
  if (!e || !n || (cap && !ids)) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    std::vector<uint64_t> v;
    e->e->band_survivors(v);
    *n = v.size();
    std::memcpy(ids, v.data(), std::min<uint64_t>(cap, v.size()) * 8);
  });
}
int bp_band_rnbp_fallback(bp_engine* e, uint64_t gd) {
  if (!e) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    e->e->band_commit_global(gd);
    e->e->band_rnbp_pack();
  });
}

// Philox4x32-10 draw of the device (bp_device.cuh philox_u53), for host-side
// decisions that must match the device stream (the band fallback).
uint64_t bp_philox_u53(uint64_t seed, uint64_t iteration, uint32_t attempt, uint64_t d) {
  return bpb::philox_u53_host(seed, iteration, attempt, d);
}

}  // extern "C"

namespace bpb {
uint64_t philox_u53_host(uint64_t seed, uint64_t iteration, uint32_t attempt, uint64_t d) {
  const uint64_t e = d >> 1;
  uint32_t c0 = static_cast<uint32_t>(e), c1 = static_cast<uint32_t>(e >> 32), c2 = static_cast<uint32_t>(iteration),
           c3 = (static_cast<uint32_t>(iteration >> 32) & 0x3FFFFFFFu) | (attempt << 30);
  uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c0, p1 = static_cast<uint64_t>(0xCD9E8D57u) * c2;
    const uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
    const uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
    if (r < 9) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
  }
  const uint64_t hi = (d & 1ull) ? c2 : c0, lo = (d & 1ull) ? c3 : c1;
  return ((hi << 32) | lo) >> 11;
}
}  // namespace bpb

extern "C" {

int bp_philox4x32_10_device(int32_t device, uint64_t n, const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
  if (n && (!ctr || !key || !out)) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    if (device >= 0) bpb::cuda_check(cudaSetDevice(device), "cudaSetDevice");
    if (!n) return;
    bpb::DevBuf dc, dk, dout;
    dc.upload(ctr, n * 16);
    dk.upload(key, n * 8);
    dout.alloc(n * 16);
    k_philox_kat<<<static_cast<unsigned>((n + 127) / 128), 128>>>(n, dc.as<uint32_t>(), dk.as<uint32_t>(),
                                                                  dout.as<uint32_t>());
    bpb::cuda_check(cudaGetLastError(), "philox launch");
    bpb::cuda_check(cudaMemcpy(out, dout.p, n * 16, cudaMemcpyDeviceToHost), "d2h");
  });
}

int bp_philox_u53_device(int32_t device, uint64_t seed, uint64_t iteration, uint32_t attempt, uint64_t n,
                         const uint64_t* d, uint64_t* out) {
  if (n && (!d || !out)) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    if (device >= 0) bpb::cuda_check(cudaSetDevice(device), "cudaSetDevice");
    if (!n) return;
    bpb::DevBuf dd, dout;
    dd.upload(d, n * 8);
    dout.alloc(n * 8);
    k_philox_u53<<<static_cast<unsigned>((n + 127) / 128), 128>>>(seed, iteration, attempt, n, dd.as<uint64_t>(),
                                                                  dout.as<uint64_t>());
    bpb::cuda_check(cudaGetLastError(), "philox launch");
    bpb::cuda_check(cudaMemcpy(out, dout.p, n * 8, cudaMemcpyDeviceToHost), "d2h");
  });
}

int bp_engine_lbp_sweep(bp_engine* e, uint32_t flags, uint32_t* kernel_out) {
  if (!e) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    const uint32_t k = e->e->lbp_sweep(flags);
    if (kernel_out) *kernel_out = k;
  });
}

int bp_engine_step(bp_engine* e, uint64_t* frontier_size) {
  if (!e) return BP_ERR_INVALID_ARGUMENT;
  return guarded([&] {
    const uint64_t f = e->e->step();
    if (frontier_size) *frontier_size = f;
  });
}

}  // extern "C"
