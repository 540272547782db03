// Device-resident graph (host handle).  See bp_device.cuh for the layout.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "bp_device.cuh"
#include "bp_internal.hpp"

namespace bpb {

void cuda_check(cudaError_t e, const char* what);

// Device buffer.  Freed blocks go back to a process-wide cache (keyed by
// size) instead of cudaFree: a run allocates ~10 arrays of O(D) and graph
// construction as many again, and cudaMalloc/cudaFree of such blocks costs
// milliseconds each (and stalls the device) on the end-to-end path.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  size_t cap = 0;  // allocated bytes (>= bytes + 64)
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf();
  void alloc(size_t n);
  // no zero-fill and no device synchronisation: the caller overwrites [0, n)
  // on stream st (only the 64-byte slack is zeroed there)
  void alloc_async(size_t n, cudaStream_t st);
  void upload(const void* src, size_t n);
  void reset();
  static void trim_cache();  // cudaFree every cached block
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Vertices within distance h of every vertex (the balls the splash builder
// reserves), CSR layout; built on the device on first use per h.
struct BallLists {
  DevBuf off;   // u64[V+1]
  DevBuf list;  // u32[off[V]]
};

struct GraphImpl {
  int device = 0;
  uint32_t V = 0, E = 0, D = 0, maxq = 0, qs = 1;
  uint32_t uniform_q = 0;  // all cardinalities equal to this (0 = mixed)
  bool binary = true;
  DevBuf in_off, in_adj, ep, unary_lo, epar, card, unary_log, table, bel_off, ising_a, pw;
  // numeric_error parity on models whose messages can collapse (graph.cu):
  // log-domain tables and the reference's mass computed on the device
  bool check_collapse = false;
  uint32_t lat_rows = 0, lat_cols = 0;  // lattice topology detected / generated (0 = CSR only)
  uint32_t par_mode = 0;                // 1: Ising couplings (binary) / Potts weights (generic)
  // row-band partition (bp_graph_generate_ising_band): owned local rows
  // [cnt_row0, cnt_row1); other rows are ghosts of the neighbouring bands
  uint32_t cnt_row0 = 0, cnt_row1 = 0xFFFFFFFFu;
  uint64_t owned_directed = 0;          // directed edges whose source is owned
  uint64_t edge_offset = 0;             // global id of local edge 0
  // vertex-range partition (bp_graph_create_part): owned local vertices
  // [0, own_v), local -> global edge ids, and the cut-message lists per peer
  uint32_t own_v = 0xFFFFFFFFu;
  DevBuf egid;                           // u32[E]
  std::vector<uint32_t> egid_host;
  struct PartPeer {
    uint32_t part;
    uint32_t send_off, send_n;  // into send_idx: owned-source messages whose target the peer owns
    uint32_t recv_off, recv_n;  // into recv_idx: messages from the peer's vertices into owned ones
  };
  std::vector<PartPeer> peers;
  DevBuf send_idx, recv_idx;             // local directed ids, each peer's run in global directed-id order
  uint32_t part = 0, nparts = 0, v0 = 0, v1 = 0;
  std::vector<uint32_t> cards_host;  // mixed cardinalities only

  DevGraph dev() const;
  uint64_t device_bytes() const;
  uint64_t unary_size() const {
    if (uniform_q) return static_cast<uint64_t>(V) * uniform_q;
    uint64_t n = 0;
    for (uint32_t c : cards_host) n += c;
    return n;
  }
  uint32_t card_of(uint32_t v) const;
  const std::vector<uint32_t>& host_ep() const;
  const std::vector<uint32_t>& host_in_off() const;
  const std::vector<uint32_t>& host_in_adj() const;

  // nullptr when the lists would be too large (the kernels then walk the CSR)
  const BallLists* balls(uint32_t h) const;

  mutable std::mutex host_mu;
  mutable std::map<uint32_t, std::unique_ptr<BallLists>> balls_;
  mutable std::map<uint32_t, bool> balls_too_big_;
  mutable std::vector<uint32_t> ep_host, in_off_host, in_adj_host;
};

// internal bp_device_opts flag: keep the given edge orientation (i > j allowed)
constexpr uint32_t kBuildAnyOrder = 1u << 31;
std::unique_ptr<GraphImpl> build_from_desc(const bp_graph_desc* d, const bp_device_opts* opts);
struct PartLayout {
  uint32_t part, nparts, v0, v1, ghost_vertices, local_edges, peers;
  uint64_t send_messages, recv_messages, owned_directed;
};
std::unique_ptr<GraphImpl> build_part(const bp_graph_desc* d, uint32_t part, uint32_t nparts,
                                      const bp_device_opts* opts, PartLayout& out);
// columns of the generate_ising lattice numbering of this edge list (0: not a lattice)
uint32_t lattice_cols(uint32_t V, uint32_t E, const uint32_t* ep);
std::unique_ptr<GraphImpl> build_lattice_binary(uint32_t rows, uint32_t cols, const BinaryStreams& s,
                                                const bp_device_opts* opts);
std::unique_ptr<GraphImpl> build_potts(uint32_t n, uint32_t q, const PottsStreams& s,
                                       const bp_device_opts* opts);
std::unique_ptr<GraphImpl> build_er(uint32_t n, const ErInstance& inst, const bp_device_opts* opts);

}  // namespace bpb
