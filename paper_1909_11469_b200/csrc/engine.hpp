// Host-side engine: owns the per-run device state and drives the kernels.
// Restates EngineState (schedulers.hpp:61-90) and run() (schedulers.cpp:293-353).
#pragma once

#include <memory>
#include <vector>

#include "graph.hpp"

namespace bpb {

// Process-wide pool of pinned host blocks (one size class per size):
// cudaMallocHost / cudaFreeHost cost milliseconds to hundreds of ms per call.
void* pinned_acquire(size_t bytes);
void pinned_release(void* p, size_t bytes);

class EngineBase {
 public:
  virtual ~EngineBase() = default;
  // full run (bp_run_ex)
  virtual void run(const bp_run_opts* opts, bp_run_result* res, double* beliefs_host,
                   bp_iter_record* trace, uint64_t trace_cap) = 0;
  // lockstep API
  virtual void lockstep_init() = 0;
  virtual uint32_t unconverged() = 0;
  virtual uint64_t iteration() = 0;
  virtual void messages(double* out, bool candidates) = 0;
  virtual void residuals(double* out) = 0;
  virtual void beliefs(double* out) = 0;
  virtual void apply_frontier(const uint32_t* f, uint64_t n) = 0;
  virtual void rnbp_frontier(double p, std::vector<uint32_t>& out) = 0;
  virtual void rbp_frontier(double p, std::vector<uint32_t>& out) = 0;
  virtual void rs_frontier(double p, uint32_t h, std::vector<uint32_t>& roots,
                           std::vector<uint64_t>& eoff, std::vector<uint32_t>& edges) = 0;
  virtual void apply_splashes(uint64_t ns, const uint32_t* roots, const uint64_t* eoff,
                              const uint32_t* edges) = 0;
  virtual uint64_t step() = 0;
  virtual uint32_t lbp_sweep(uint32_t flags) = 0;  // fused LBP sweep (lockstep of the production kernel)
  virtual void advance_iteration() = 0;  // EngineState::advance_iteration (schedulers.hpp:75)
  // row-band partition (bp_band_*): LBP on a lattice band with ghost rows
  virtual void band_config(const PartHalo& h, uint64_t owned_directed) = 0;
  // RnBP on a band: begin = init + first refresh; select (attempt 0/1) =
  // rnbp_frontier + commit + pack; refresh = unpack (+ flags) + touched refresh
  // + sums; finish = loop control on the all-reduced sums
  virtual void band_rnbp_begin() = 0;
  virtual void band_rnbp_finish_init() = 0;
  virtual void band_rnbp_select(unsigned attempt) = 0;
  virtual void band_rnbp_refresh() = 0;
  virtual void band_rnbp_finish() = 0;
  virtual void band_survivors(std::vector<uint64_t>& global_ids) = 0;
  virtual void band_commit_global(uint64_t global_d) = 0;  // UINT64_MAX: nothing to commit here
  virtual void band_rnbp_pack() = 0;
  virtual void band_rbp_select() = 0;
  virtual void band_rs_select() = 0;
  virtual void band_sweep() = 0;
  virtual void band_finish() = 0;
  virtual void band_status(bp_run_result* r) = 0;
  // polling host (partition.cu): RnBP iterations run back to back on the
  // device; one whose attempt-0 frontier is empty parks the band (band_wait)
  virtual void band_set_poll(bool on) = 0;
  virtual bool band_waiting() = 0;  // after band_status (reads the fetched header)
  virtual void band_clear_wait() = 0;
  virtual cudaStream_t stream() const = 0;
};

std::unique_ptr<EngineBase> make_engine(const GraphImpl& g, const bp_sched_config& cfg);

void validate_config(const bp_sched_config& c);
double select_parallelism_host(uint32_t prev, uint32_t now, const bp_sched_config& c);

}  // namespace bpb
