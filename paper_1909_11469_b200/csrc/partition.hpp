// Row-band partition driver (partition.cu): bands, transports, the loop.
#pragma once

#include <cstdint>
#include <vector>

#include "engine.hpp"

namespace bpb {

// One band of a row partition: its engine, halo buffers (device) and stream.
struct Band {
  EngineBase* engine = nullptr;
  bp_band_info info{};
  bp_sched_config cfg{};
  cudaStream_t stream = nullptr;
  PartHalo halo{};
  DevBuf own[5];  // halo buffers owned by the band (bp_band_engine_create_owned)
  // the parts this band exchanges cut messages with: per peer, the run of the
  // send buffer it receives and the run of the recv buffer it fills (row
  // bands: the band above / below, cols floats each way; vertex-range parts:
  // any peer, the graph's list lengths)
  struct Peer {
    uint32_t part;
    float* send;
    uint32_t ns;
    float* recv;
    uint32_t nr;
  };
  std::vector<Peer> peers;
  void lattice_peers() {  // row bands: the band above and the band below
    peers.clear();
    if (info.ghost_up) peers.push_back({info.part - 1, halo.send_up, info.cols, recv_up(), info.cols});
    if (info.ghost_down) peers.push_back({info.part + 1, halo.send_down, info.cols, recv_down(), info.cols});
  }
  float* send_up() const { return halo.send_up; }
  float* send_down() const { return halo.send_down; }
  float* recv_up() const { return const_cast<float*>(halo.recv_up); }
  float* recv_down() const { return const_cast<float*>(halo.recv_down); }
  unsigned long long* count() const { return halo.count; }
};

// The exchange steps of an iteration, enqueued on the bands' streams.
struct BandComm {
  virtual ~BandComm() = default;
  // send_up -> band above's recv_down, send_down -> band below's recv_up
  virtual void halo(const std::vector<Band*>& bands) = 0;
  // count[0 .. n) <- sum over all bands
  virtual void all_reduce(const std::vector<Band*>& bands, uint32_t n) = 0;
  // every band's survivor ids (global), merged in ascending order
  virtual std::vector<uint64_t> gather(const std::vector<Band*>& bands,
                                       const std::vector<std::vector<uint64_t>>& local) = 0;
};

BandComm* make_nccl_comm(const uint8_t id[128], int rank, int nranks, int device);
BandComm* make_local_comm();
void nccl_unique_id(uint8_t out[128]);
void run_bands(std::vector<Band*>& bands, BandComm& comm, bp_run_result* res);
uint64_t philox_u53_host(uint64_t seed, uint64_t iteration, uint32_t attempt, uint64_t d);

}  // namespace bpb
