// EngineT<128> instantiation (see engine_impl.cuh).
#include "engine_impl.cuh"

namespace bpb {
std::unique_ptr<EngineBase> make_engine_q128(const GraphImpl& g, const bp_sched_config& cfg) {
  return std::make_unique<EngineT<128>>(g, cfg);
}
}  // namespace bpb
