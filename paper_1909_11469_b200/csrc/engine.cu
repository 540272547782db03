// Engine entry points: config validation (schedulers.cpp:78-90),
// select_parallelism (schedulers.cpp:218-224) and the per-stride dispatch.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>

#include "engine.hpp"

namespace bpb {

namespace {
struct PinnedPool {
  std::mutex mu;
  std::multimap<size_t, void*> free;
};
PinnedPool& pinned_pool() {
  static PinnedPool* p = new PinnedPool;  // process lifetime
  return *p;
}
}  // namespace

void* pinned_acquire(size_t bytes) {
  {
    PinnedPool& pp = pinned_pool();
    std::lock_guard<std::mutex> lk(pp.mu);
    auto it = pp.free.find(bytes);
    if (it != pp.free.end()) {
      void* p = it->second;
      pp.free.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  cuda_check(cudaMallocHost(&p, bytes), "cudaMallocHost");
  return p;
}

void pinned_release(void* p, size_t bytes) {
  PinnedPool& pp = pinned_pool();
  std::lock_guard<std::mutex> lk(pp.mu);
  pp.free.emplace(bytes, p);
}


void validate_config(const bp_sched_config& c) {  // schedulers.cpp:78-90
  if (!(c.epsilon > 0.0) || !std::isfinite(c.epsilon)) throw_invalid("epsilon must be positive");
  if (!(c.p > 0.0) || c.p > 1.0) throw_invalid("p must be in (0, 1]");
  if (!(c.low_p > 0.0) || c.low_p > c.high_p || c.high_p > 1.0)
    throw_invalid("parallelism settings must satisfy 0 < low_p <= high_p <= 1");
  if (!(c.edge_ratio_threshold > 0.0) || c.edge_ratio_threshold > 1.0)
    throw_invalid("edge_ratio_threshold must be in (0, 1]");
  if (!(c.time_limit > 0.0)) throw_invalid("time_limit must be positive");
  if (c.kind < BP_LBP || c.kind > BP_RNBP) throw_invalid("unknown scheduler kind");
}

double select_parallelism_host(uint32_t prev, uint32_t now, const bp_sched_config& c) {
  if (prev == 0) return c.high_p;
  const double ratio = static_cast<double>(now) / static_cast<double>(prev);
  return ratio > c.edge_ratio_threshold ? c.low_p : c.high_p;
}


std::unique_ptr<EngineBase> make_engine_q1(const GraphImpl& g, const bp_sched_config& cfg);
std::unique_ptr<EngineBase> make_engine_q4(const GraphImpl& g, const bp_sched_config& cfg);
std::unique_ptr<EngineBase> make_engine_q8(const GraphImpl& g, const bp_sched_config& cfg);
std::unique_ptr<EngineBase> make_engine_q16(const GraphImpl& g, const bp_sched_config& cfg);
std::unique_ptr<EngineBase> make_engine_q32(const GraphImpl& g, const bp_sched_config& cfg);
std::unique_ptr<EngineBase> make_engine_q64(const GraphImpl& g, const bp_sched_config& cfg);
std::unique_ptr<EngineBase> make_engine_q128(const GraphImpl& g, const bp_sched_config& cfg);

std::unique_ptr<EngineBase> make_engine(const GraphImpl& g, const bp_sched_config& cfg) {
  switch (g.qs) {
    case 1: return make_engine_q1(g, cfg);
    case 4: return make_engine_q4(g, cfg);
    case 8: return make_engine_q8(g, cfg);
    case 16: return make_engine_q16(g, cfg);
    case 64: return make_engine_q64(g, cfg);
    case 128: return make_engine_q128(g, cfg);
    case 32: return make_engine_q32(g, cfg);
    default: throw Error(BP_ERR_UNSUPPORTED, "unsupported message stride");
  }
}

}  // namespace bpb
