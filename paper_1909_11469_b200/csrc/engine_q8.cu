// EngineT<8> instantiation (see engine_impl.cuh).
#include "engine_impl.cuh"

namespace bpb {
std::unique_ptr<EngineBase> make_engine_q8(const GraphImpl& g, const bp_sched_config& cfg) {
  return std::make_unique<EngineT<8>>(g, cfg);
}
}  // namespace bpb
