// Link-time drop-in for the reference's scheduler entry point
// (proj/core/include/bpsched/schedulers.hpp:156):
//
//   bpsched::RunResult bpsched::run(const PairwiseMRF&, const SchedulerConfig&);
//
// defined here on top of the B200 engine (include/bpsched_cuda.hpp), so an
// UNMODIFIED caller of the reference -- its CLI (tools/bpsched.cpp:172, 299,
// 349), tests, or the reference core itself when built as a shared library --
// runs the device scheduler without a source change: link this object ahead of
// the reference library, or preload the shared build
//
//   LD_PRELOAD=oracle/_ref/libbpsched_cuda_shim.so  <reference caller>
//
// (ELF symbol interposition: the first definition of bpsched::run wins).
// Serial RBP stays on the host: bpsched_cuda::run forwards it to the
// reference's run_serial_rbp.  bpsched_cuda_shim_calls() counts the runs that
// went through the shim (tests check it).
#include <atomic>
#include <cstdint>

#include "bpsched_cuda.hpp"

namespace {
std::atomic<uint64_t> g_calls{0};
}

namespace bpsched {

RunResult run(const PairwiseMRF& graph, const SchedulerConfig& config) {
  g_calls.fetch_add(1, std::memory_order_relaxed);
  return bpsched_cuda::run(graph, config);
}

}  // namespace bpsched

extern "C" __attribute__((visibility("default"))) uint64_t bpsched_cuda_shim_calls(void) {
  return g_calls.load(std::memory_order_relaxed);
}
