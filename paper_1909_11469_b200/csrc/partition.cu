// Row-band partition driver in C++ (SURVEY.md 8(e)): the run() loop of one
// lattice band per GPU (schedulers.cpp:301-347), with the halo exchange and the
// all-reduce of the loop counters enqueued on the band's CUDA stream through
// NCCL -- no Python and no host round trip inside an LBP iteration.
//
//   LBP   per iteration: sweep (+ boundary pack + local count) | halo send /
//         recv of 2 x cols floats per cut + all-reduce {count, time vote} |
//         unpack + loop control on the GLOBAL count.  The host polls the stop
//         flag every kPollEvery iterations (later iterations are no-ops).
//   RnBP  per iteration: select attempt 0 (Philox keyed by GLOBAL edge ids) +
//   RBP   commit + pack | halo | ghost unpack + flagged refresh | all-reduce
//   RS    {delta, frontier, survivors, time vote, count}; the loop control
//         runs on the device from the all-reduced sums and the host polls
//         every kPollEvery iterations.  RnBP's retry and single-survivor
//         fallback (schedulers.cpp:204-214) need the host: an iteration with
//         an empty attempt-0 frontier parks the bands (Ctl::band_wait) until
//         the next poll runs them.
//
// Transports: NcclTransport (one band per rank, ncclSend/ncclRecv/ncclAllReduce
// on the band stream; libnccl is loaded at first use, so single-GPU users need
// no NCCL) and LocalTransport (every band of the partition inside this
// process, e.g. on one GPU: host-staged copies, the parity tests' vehicle).
// Both drive the same loop, so the loop logic tested on one GPU is the one
// that runs across GPUs.
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <nccl.h>

#include "engine.hpp"
#include "partition.hpp"

namespace bpb {

// ---------------------------------------------------------------- libnccl
namespace {
struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl() {
  static std::once_flag once;
  static NcclApi api;
  static std::string err;
  std::call_once(once, [] {
    // whichever libnccl the process already has (torch's), else the system one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    auto sym = [&](auto& f, const char* n) { f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, n)); };
    sym(api.get_unique_id, "ncclGetUniqueId");
    sym(api.init_rank, "ncclCommInitRank");
    sym(api.destroy, "ncclCommDestroy");
    sym(api.send, "ncclSend");
    sym(api.recv, "ncclRecv");
    sym(api.all_reduce, "ncclAllReduce");
    sym(api.all_gather, "ncclAllGather");
    sym(api.group_start, "ncclGroupStart");
    sym(api.group_end, "ncclGroupEnd");
    sym(api.error_string, "ncclGetErrorString");
  });
  if (!api.get_unique_id || !api.init_rank || !api.send || !api.recv || !api.all_reduce || !api.all_gather ||
      !api.group_start || !api.group_end)
    throw Error(BP_ERR_NCCL, err.empty() ? "libnccl: missing symbols" : err);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  const char* s = nccl().error_string ? nccl().error_string(r) : "?";
  throw Error(BP_ERR_NCCL, std::string(what) + ": " + s);
}
}  // namespace

void nccl_unique_id(uint8_t out[128]) {
  ncclUniqueId id;
  nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out, &id, 128);
}

// ---------------------------------------------------------------- NCCL
struct NcclComm final : BandComm {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  NcclComm(const uint8_t id[128], int r, int n, int device) : rank(r), nranks(n) {
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    nccl_check(nccl().init_rank(&comm, n, uid, r), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm && nccl().destroy) nccl().destroy(comm);
  }
  void check_bands(const std::vector<Band*>& b) const {
    if (b.size() != 1) throw Error(BP_ERR_INVALID_ARGUMENT, "NCCL partition: one band per rank");
    if (b[0]->info.part != static_cast<uint32_t>(rank) || b[0]->info.nparts != static_cast<uint32_t>(nranks))
      throw Error(BP_ERR_INVALID_ARGUMENT, "band part / nparts do not match the communicator's rank / size");
  }
  void halo(const std::vector<Band*>& bands) override {
    check_bands(bands);
    Band& b = *bands[0];
    const auto& a = nccl();
    nccl_check(a.group_start(), "ncclGroupStart");
    for (const Band::Peer& p : b.peers) {
      if (p.ns) nccl_check(a.send(p.send, p.ns, ncclFloat32, static_cast<int>(p.part), comm, b.stream), "ncclSend");
      if (p.nr) nccl_check(a.recv(p.recv, p.nr, ncclFloat32, static_cast<int>(p.part), comm, b.stream), "ncclRecv");
    }
    nccl_check(a.group_end(), "ncclGroupEnd");
  }
  void all_reduce(const std::vector<Band*>& bands, uint32_t n) override {
    check_bands(bands);
    Band& b = *bands[0];
    nccl_check(nccl().all_reduce(b.count(), b.count(), n, ncclUint64, ncclSum, comm, b.stream), "ncclAllReduce");
  }
  // survivors of every rank in ascending global id (the fallback's order,
  // schedulers.cpp:212-214): sizes, then a padded all-gather of the ids
  std::vector<uint64_t> gather(const std::vector<Band*>& bands, const std::vector<std::vector<uint64_t>>& local) override {
    check_bands(bands);
    Band& b = *bands[0];
    DevBuf sz, all_sz;
    sz.alloc(8);
    all_sz.alloc(8ull * nranks);
    const uint64_t mine = local[0].size();
    cuda_check(cudaMemcpyAsync(sz.p, &mine, 8, cudaMemcpyHostToDevice, b.stream), "h2d");
    nccl_check(nccl().all_gather(sz.p, all_sz.p, 1, ncclUint64, comm, b.stream), "ncclAllGather");
    std::vector<uint64_t> sizes(nranks);
    cuda_check(cudaMemcpyAsync(sizes.data(), all_sz.p, 8ull * nranks, cudaMemcpyDeviceToHost, b.stream), "d2h");
    cuda_check(cudaStreamSynchronize(b.stream), "sync");
    const uint64_t mx = std::max<uint64_t>(1, *std::max_element(sizes.begin(), sizes.end()));
    std::vector<uint64_t> pad(mx, ~0ull);
    std::copy(local[0].begin(), local[0].end(), pad.begin());
    DevBuf ids, all_ids;
    ids.upload(pad.data(), mx * 8);
    all_ids.alloc(mx * 8 * nranks);
    nccl_check(nccl().all_gather(ids.p, all_ids.p, mx, ncclUint64, comm, b.stream), "ncclAllGather");
    std::vector<uint64_t> all(mx * nranks);
    cuda_check(cudaMemcpyAsync(all.data(), all_ids.p, all.size() * 8, cudaMemcpyDeviceToHost, b.stream), "d2h");
    cuda_check(cudaStreamSynchronize(b.stream), "sync");
    std::vector<uint64_t> out;
    for (uint64_t x : all)
      if (x != ~0ull) out.push_back(x);
    std::sort(out.begin(), out.end());
    return out;
  }
};

BandComm* make_nccl_comm(const uint8_t id[128], int rank, int nranks, int device) {
  return new NcclComm(id, rank, nranks, device);
}

// ---------------------------------------------------------------- local
// Every band of the partition in this process: host-staged copies between the
// bands' buffers (a test vehicle: one GPU holds all bands).
struct LocalComm final : BandComm {
  static void sync_all(const std::vector<Band*>& bands) {
    for (Band* b : bands) cuda_check(cudaStreamSynchronize(b->stream), "band sync");
  }
  void halo(const std::vector<Band*>& bands) override {
    sync_all(bands);
    for (Band* b : bands)
      for (const Band::Peer& p : b->peers) {
        if (p.part >= bands.size()) throw Error(BP_ERR_INVALID_ARGUMENT, "local partition: missing part");
        const Band& o = *bands[p.part];  // bands are parts 0 .. P-1 in order
        auto q = std::find_if(o.peers.begin(), o.peers.end(), [&](const Band::Peer& x) { return x.part == b->info.part; });
        if (q == o.peers.end() || q->ns != p.nr) throw Error(BP_ERR_INVALID_ARGUMENT, "local partition: halo sizes disagree");
        if (p.nr) cuda_check(cudaMemcpy(p.recv, q->send, 4ull * p.nr, cudaMemcpyDefault), "halo copy");
      }
    cuda_check(cudaDeviceSynchronize(), "halo");
  }
  void all_reduce(const std::vector<Band*>& bands, uint32_t n) override {
    sync_all(bands);
    std::vector<uint64_t> tot(n, 0), x(n);
    for (Band* b : bands) {
      cuda_check(cudaMemcpy(x.data(), b->count(), 8ull * n, cudaMemcpyDeviceToHost), "d2h");
      for (uint32_t k = 0; k < n; ++k) tot[k] += x[k];
    }
    for (Band* b : bands) cuda_check(cudaMemcpy(b->count(), tot.data(), 8ull * n, cudaMemcpyHostToDevice), "h2d");
    cuda_check(cudaDeviceSynchronize(), "all-reduce");
  }
  std::vector<uint64_t> gather(const std::vector<Band*>&, const std::vector<std::vector<uint64_t>>& local) override {
    std::vector<uint64_t> out;
    for (const auto& l : local) out.insert(out.end(), l.begin(), l.end());
    std::sort(out.begin(), out.end());
    return out;
  }
};

// ---------------------------------------------------------------- loops
namespace {
constexpr int kPollEvery = 16;  // LBP: host polls the stop flag every 16 iterations

void lbp_loop(std::vector<Band*>& bands, BandComm& comm, uint64_t max_iterations) {
  for (uint64_t it = 0; it <= max_iterations; ++it) {  // sweep 0 computes r(m_0) (ResidualTracker ctor)
    for (Band* b : bands) b->engine->band_sweep();
    comm.halo(bands);
    comm.all_reduce(bands, 2);
    for (Band* b : bands) b->engine->band_finish();
    if (it % kPollEvery == kPollEvery - 1) {
      bp_run_result st;
      bands[0]->engine->band_status(&st);
      if (st.stopped) return;
    }
  }
}

void frontier_loop(std::vector<Band*>& bands, BandComm& comm, int kind, uint64_t max_iterations, uint64_t seed) {
  auto phase = [&](unsigned attempt) {
    for (Band* b : bands) {
      if (kind == BP_RNBP) b->engine->band_rnbp_select(attempt);
      else if (kind == BP_RBP) b->engine->band_rbp_select();
      else b->engine->band_rs_select();
    }
    comm.halo(bands);
    for (Band* b : bands) b->engine->band_rnbp_refresh();
    comm.all_reduce(bands, 5);
  };
  auto read_counts = [&](uint64_t* c) {
    Band& b = *bands[0];
    cuda_check(cudaMemcpyAsync(c, b.count(), 40, cudaMemcpyDeviceToHost, b.stream), "d2h");
    cuda_check(cudaStreamSynchronize(b.stream), "sync");
  };
  for (Band* b : bands) b->engine->band_rnbp_begin();
  comm.all_reduce(bands, 5);
  for (Band* b : bands) b->engine->band_rnbp_finish_init();
  // RnBP: an iteration whose attempt-0 frontier is empty parks every band on
  // the device (the finalize sees the all-reduced sums, so all ranks park at
  // the same iteration); the iterations enqueued behind it are no-ops -- their
  // collectives still run, on zeroed sums -- until the next poll runs the retry
  if (kind == BP_RNBP)
    for (Band* b : bands) b->engine->band_set_poll(true);
  const uint64_t max_polls = max_iterations / kPollEvery + 2;
  for (uint64_t poll = 0; poll <= max_polls + 2 * (max_iterations + 1); ++poll) {
    bp_run_result st;
    bands[0]->engine->band_status(&st);  // one D2H + sync per kPollEvery iterations
    if (st.stopped) break;
    if (kind == BP_RNBP && bands[0]->engine->band_waiting()) {
      for (Band* b : bands) b->engine->band_clear_wait();
      phase(1);  // retry once, then one survivor (schedulers.cpp:204-214)
      uint64_t c[5];
      read_counts(c);
      if (c[1] == 0) {
        std::vector<std::vector<uint64_t>> local(bands.size());
        for (size_t i = 0; i < bands.size(); ++i) bands[i]->engine->band_survivors(local[i]);
        const std::vector<uint64_t> ids = comm.gather(bands, local);
        if (!ids.empty()) {
          const double u = static_cast<double>(philox_u53_host(seed, st.iterations, 2u, 0ull)) * 0x1.0p-53;
          const uint64_t pick = ids[std::min<uint64_t>(ids.size() - 1, static_cast<uint64_t>(u * ids.size()))];
          for (size_t i = 0; i < bands.size(); ++i) {
            const bool owned = std::binary_search(local[i].begin(), local[i].end(), pick);
            bands[i]->engine->band_commit_global(owned ? pick : ~0ull);
            bands[i]->engine->band_rnbp_pack();
          }
          comm.halo(bands);
          for (Band* b : bands) b->engine->band_rnbp_refresh();
          comm.all_reduce(bands, 5);
        }
      }
      for (Band* b : bands) b->engine->band_rnbp_finish();
      continue;  // poll again: the retried iteration may have been the last
    }
    for (int j = 0; j < kPollEvery; ++j) {
      phase(0);
      for (Band* b : bands) b->engine->band_rnbp_finish();
    }
  }
  if (kind == BP_RNBP)
    for (Band* b : bands) b->engine->band_set_poll(false);
}
}  // namespace

void run_bands(std::vector<Band*>& bands, BandComm& comm, bp_run_result* res) {
  if (bands.empty()) throw Error(BP_ERR_INVALID_ARGUMENT, "no bands");
  const bp_sched_config& cfg = bands[0]->cfg;
  for (size_t i = 0; i < bands.size(); ++i) {
    if (bands[i]->cfg.kind != cfg.kind) throw Error(BP_ERR_INVALID_ARGUMENT, "bands run different schedulers");
    if (i && bands[i]->info.part != bands[i - 1]->info.part + 1)
      throw Error(BP_ERR_INVALID_ARGUMENT, "local partition: bands must be parts 0..P-1 in order");
  }
  if (cfg.kind == BP_LBP) lbp_loop(bands, comm, cfg.max_iterations);
  else if (cfg.kind == BP_RNBP || cfg.kind == BP_RBP || cfg.kind == BP_RS)
    frontier_loop(bands, comm, cfg.kind, cfg.max_iterations, cfg.seed);
  else
    throw Error(BP_ERR_UNSUPPORTED, "row-band partition: scheduler not partitioned");
  bands[0]->engine->band_status(res);
}

BandComm* make_local_comm() { return new LocalComm(); }

}  // namespace bpb
