// Graph construction and upload: the device counterpart of build_graph
// (mrf.cpp:25-106) and of the generators (generators.cpp:24-71).
#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <limits>
#include <thread>
#include <unordered_set>

#include "bp_device.cuh"
#include "engine.hpp"
#include "graph.hpp"
#include "host_pool.hpp"

namespace bpb {

void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation) throw Error(BP_ERR_OOM, std::string(what) + ": " + cudaGetErrorString(e));
  throw Error(BP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

namespace {
struct BlockCache {
  std::mutex mu;
  std::multimap<std::pair<int, size_t>, void*> free;  // (device, capacity) -> block
  size_t held = 0;
};
BlockCache& block_cache() {
  static BlockCache* c = new BlockCache;  // process lifetime (no teardown-order issues)
  return *c;
}
constexpr size_t kCacheMaxBlock = size_t{1} << 31;  // larger blocks are freed, not cached
constexpr size_t kCacheMaxHeld = size_t{16} << 30;
}  // namespace

void DevBuf::trim_cache() {
  BlockCache& c = block_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  int dev = 0;
  cudaGetDevice(&dev);
  for (auto& kv : c.free) {
    cudaSetDevice(kv.first.first);
    cudaFree(kv.second);
  }
  cudaSetDevice(dev);
  c.free.clear();
  c.held = 0;
}

DevBuf::~DevBuf() { reset(); }
void DevBuf::reset() {
  if (p) {
    BlockCache& c = block_cache();
    // the block may still be read by queued work: settle the device first
    // (cudaFree would synchronise too)
    cudaDeviceSynchronize();
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(c.mu);
    if (cap <= kCacheMaxBlock && c.held + cap <= kCacheMaxHeld) {
      c.free.emplace(std::make_pair(dev, cap), p);
      c.held += cap;
    } else {
      cudaFree(p);
    }
  }
  p = nullptr;
  bytes = 0;
  cap = 0;
}
void DevBuf::alloc_async(size_t n, cudaStream_t st) {
  reset();
  if (n == 0) n = 16;
  const size_t want = n + 64;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    BlockCache& c = block_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.free.lower_bound(std::make_pair(dev, want));
    if (it != c.free.end() && it->first.first == dev && it->first.second <= want + want / 4) {
      p = it->second;
      cap = it->first.second;
      c.held -= cap;
      c.free.erase(it);
    }
  }
  if (!p) {
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      trim_cache();
      e = cudaMalloc(&p, want);
    }
    cuda_check(e, "cudaMalloc");
    cap = want;
  }
  bytes = n;
  cuda_check(cudaMemsetAsync(static_cast<char*>(p) + n, 0, cap - n, st), "memset (slack)");
}
void DevBuf::alloc(size_t n) {
  reset();
  if (n == 0) n = 16;
  // 64 bytes of slack: 16-byte-granular bulk copies (kernels_lbp.cuh) may read
  // up to one granule past the end of an array
  const size_t want = n + 64;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    BlockCache& c = block_cache();
    std::unique_lock<std::mutex> lk(c.mu);
    auto it = c.free.lower_bound(std::make_pair(dev, want));
    if (it != c.free.end() && it->first.first == dev && it->first.second <= want + want / 4) {  // close fit only
      p = it->second;
      cap = it->first.second;
      c.held -= cap;
      c.free.erase(it);
      lk.unlock();
      bytes = n;
      // zero-filled like a fresh allocation in practice is; completed before
      // returning (the engines' streams are non-blocking: a legacy-stream
      // memset is not ordered before their kernels)
      cuda_check(cudaMemset(p, 0, cap), "memset (cached block)");
      cuda_check(cudaDeviceSynchronize(), "memset (cached block)");
      return;
    }
  }
  cudaError_t e = cudaMalloc(&p, want);
  if (e == cudaErrorMemoryAllocation) {  // cached blocks first
    cudaGetLastError();
    trim_cache();
    e = cudaMalloc(&p, want);
  }
  cuda_check(e, "cudaMalloc");
  // zero-filled like the recycled blocks (memory freed earlier in this
  // process comes back from cudaMalloc with its old contents), completed
  // before returning
  cuda_check(cudaMemset(p, 0, want), "memset (new block)");
  cuda_check(cudaDeviceSynchronize(), "memset (new block)");
  bytes = n;
  cap = want;
}
void DevBuf::upload(const void* src, size_t n) {
  alloc(n);
  if (src && n) {
    cuda_check(cudaMemcpy(p, src, n, cudaMemcpyHostToDevice), "upload");
    // a pageable-source cudaMemcpy may return before the DMA has landed, and
    // the engines' non-blocking streams are not ordered after the legacy
    // stream: complete it before any kernel can read the buffer
    cuda_check(cudaDeviceSynchronize(), "upload");
  }
}

DevGraph GraphImpl::dev() const {
  DevGraph g{};
  g.V = V;
  g.E = E;
  g.D = D;
  g.qs = qs;
  g.in_off = in_off.as<uint32_t>();
  g.in_adj = in_adj.as<uint32_t>();
  g.ep = ep.as<uint32_t>();
  g.unary_lo = unary_lo.as<float>();
  g.epar = epar.as<float4>();
  g.card = card.as<uint32_t>();
  g.unary_log = unary_log.as<float>();
  g.table = table.as<float>();
  g.bel_off = bel_off.as<uint32_t>();
  g.lat_rows = lat_rows;
  g.lat_cols = lat_cols;
  g.par_mode = par_mode;
  g.uniform_q = uniform_q;
  g.cnt_row0 = cnt_row0;
  g.cnt_row1 = cnt_row1;
  g.edge_offset = edge_offset;
  g.ising_a = ising_a.as<float>();
  g.pw = pw.as<float>();
  g.log_tables = check_collapse ? 1u : 0u;
  g.own_v = own_v;
  g.egid = egid.p ? egid.as<uint32_t>() : nullptr;
  return g;
}

uint64_t GraphImpl::device_bytes() const {
  return in_off.bytes + in_adj.bytes + ep.bytes + unary_lo.bytes + epar.bytes + card.bytes +
         unary_log.bytes + table.bytes + bel_off.bytes + ising_a.bytes + pw.bytes + egid.bytes + send_idx.bytes +
         recv_idx.bytes;
}

namespace {

int select_device(const bp_device_opts* opts) {
  int dev = 0;
  if (opts && opts->device >= 0) {
    cuda_check(cudaSetDevice(opts->device), "cudaSetDevice");
    dev = opts->device;
  } else {
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  }
  return dev;
}

uint32_t stride_for(uint32_t maxq) {
  if (maxq <= 4) return 4;
  if (maxq <= 8) return 8;
  if (maxq <= 16) return 16;
  if (maxq <= 32) return 32;
  if (maxq <= 64) return 64;  // q >= 33: q-vectors in local memory (correct, not tuned)
  if (maxq <= 128) return 128;
  throw Error(BP_ERR_UNSUPPORTED, "cardinalities above 128 are not supported by the device kernels (max " +
                                      std::to_string(maxq) + ")");
}

// CSR of incoming directed edges in edge-id order (mrf.cpp:93-104)
void build_csr(uint32_t V, uint32_t E, const uint32_t* ep, std::vector<uint32_t>& off,
               std::vector<uint32_t>& adj) {
  const uint64_t D = 2ull * E;
  off.assign(static_cast<size_t>(V) + 1, 0);
  for (uint64_t d = 0; d < D; ++d) off[ep[d ^ 1ull] + 1]++;  // tgt(d) = ep[d ^ 1]
  for (uint32_t v = 0; v < V; ++v) off[v + 1] += off[v];
  adj.resize(D);
  std::vector<uint32_t> cur(off.begin(), off.end() - 1);
  for (uint64_t d = 0; d < D; ++d) adj[cur[ep[d ^ 1ull]]++] = static_cast<uint32_t>(d);
}

// Lattice topology (rows x cols, row-major vertices; per vertex the right edge
// then the down edge -- generators.cpp:37-43), written straight into HBM.
__global__ void k_lattice_topology(uint32_t R, uint32_t C, uint32_t* in_off, uint32_t* in_adj,
                                   uint32_t* ep) {
  const uint64_t V = static_cast<uint64_t>(R) * C;
  for (uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; v < V;
       v += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = v / C, c = v % C;
    auto ebase = [&](uint64_t rr, uint64_t cc) -> uint64_t {
      return rr + 1 < R ? rr * (2ull * C - 1) + 2 * cc : rr * (2ull * C - 1) + cc;
    };
    const uint64_t vert = (r > 0) + (r + 1 < R);
    const uint64_t before_rows = 2ull * (C - 1) * r + static_cast<uint64_t>(C) *
                                                          ((r > 0 ? r - 1 : 0) + (r < R - 1 ? r : R - 1));
    const uint64_t within = c * vert + (c > 0 ? c - 1 : 0) + (c < C - 1 ? c : C - 1);
    uint64_t o = before_rows + within;
    in_off[v] = static_cast<uint32_t>(o);
    if (v + 1 == V) in_off[V] = static_cast<uint32_t>(2ull * ((R - 1) * C + (C - 1) * R));
    if (r > 0) in_adj[o++] = static_cast<uint32_t>(2 * (ebase(r - 1, c) + (c + 1 < C)));  // up: v is hi
    if (c > 0) in_adj[o++] = static_cast<uint32_t>(2 * ebase(r, c - 1));                 // left: v is hi
    if (c + 1 < C) {                                                                      // right: v is lo
      const uint64_t e = ebase(r, c);
      in_adj[o++] = static_cast<uint32_t>(2 * e + 1);
      ep[2 * e] = static_cast<uint32_t>(v);
      ep[2 * e + 1] = static_cast<uint32_t>(v + 1);
    }
    if (r + 1 < R) {  // down: v is lo
      const uint64_t e = ebase(r, c) + (c + 1 < C);
      in_adj[o++] = static_cast<uint32_t>(2 * e + 1);
      ep[2 * e] = static_cast<uint32_t>(v);
      ep[2 * e + 1] = static_cast<uint32_t>(v + C);
    }
  }
}

__global__ void k_fill_u32(uint32_t* p, size_t n, uint32_t v) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    p[i] = v;
}

__global__ void k_iota_mul(uint32_t* p, size_t n, uint32_t mul) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    p[i] = static_cast<uint32_t>(i * mul);
}

// smallest index in [0, n) with bad(i), or n (host pool, host_pool.hpp);
// `heavy`: every index is a long scan (rows), so split even small n
template <class F>
uint64_t first_bad(uint64_t n, F&& bad, bool heavy = false) {
  std::atomic<uint64_t> first{n};
  const unsigned chunks = heavy ? static_cast<unsigned>(std::min<uint64_t>(n, HostPool::get().size() * 2))
                                : pool_chunks(n);
  auto body = [&](uint64_t a, uint64_t b, unsigned) {
    for (uint64_t i = a; i < b && i < first.load(std::memory_order_relaxed); ++i)
      if (bad(i)) {
        uint64_t cur = first.load();
        while (i < cur && !first.compare_exchange_weak(cur, i)) {
        }
        return;
      }
  };
  if (chunks <= 1) body(0, n, 0);
  else HostPool::get().run(chunks, [&](unsigned t) { body(n * t / chunks, n * (t + 1) / chunks, t); });
  return first.load();
}

unsigned grid_for(size_t n) {
  return static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 148ull * 32));
}

// Does the edge list equal generate_ising's lattice numbering for some
// rows x cols (generators.cpp:37-43)?  Then the device derives incoming
// edges arithmetically.  Returns cols (0 = not a lattice).
uint32_t detect_lattice(uint32_t V, uint32_t E, const uint32_t* ep) {
  if (V < 2 || E == 0) return 0;
  uint32_t C = V;  // a single row (also covers a single column)
  if (E >= 2 && ep[0] == 0 && ep[1] == 1 && ep[2] == 0 && ep[3] > 1) C = ep[3];
  if (V % C) return 0;
  const uint64_t R = V / C;
  if (static_cast<uint64_t>(E) != R * (C - 1) + (R - 1) * C) return 0;
  uint64_t e = 0;
  for (uint64_t r = 0; r < R; ++r)
    for (uint64_t c = 0; c < C; ++c) {
      const uint64_t v = r * C + c;
      if (c + 1 < C && (ep[2 * e] != v || ep[2 * e + 1] != v + 1)) return 0;
      if (c + 1 < C) ++e;
      if (r + 1 < R && (ep[2 * e] != v || ep[2 * e + 1] != v + C)) return 0;
      if (r + 1 < R) ++e;
    }
  return C;
}

// a = e^J (a / d of the table), clamped so the device arithmetic stays finite
const double kIsingAMax = std::exp(69.0), kIsingAMin = std::exp(-69.0);
float ising_weight(double J) {
  const double j = std::min(69.0, std::max(-69.0, J));
  return static_cast<float>(std::exp(j));
}

void upload_ising_weights(GraphImpl& g, const std::vector<float>& J) {
  std::vector<float> a(J.size());
  for (size_t e = 0; e < J.size(); ++e) a[e] = ising_weight(static_cast<double>(J[e]));
  g.ising_a.upload(a.data(), a.size() * 4);
}

}  // namespace

namespace {

bool bad_entry(double u) { return !(u > 0.0) || !std::isfinite(u); }

// build_graph's validation restated sequentially in the reference's order
// (mrf.cpp:37-85: per vertex cardinality then entries; per edge range,
// self-loop, order, duplicate, entries).  Runs only after the parallel passes
// found a violation, so the error raised is the reference's first one.
void validate_sequential(const bp_graph_desc* d, bool check_duplicates) {
  const uint32_t V = d->num_vertices, E = d->num_edges;
  size_t o = 0;
  for (uint32_t v = 0; v < V; ++v) {
    const uint32_t q = d->cardinalities[v];
    if (q == 0) throw_model("vertex " + std::to_string(v) + " has cardinality 0");
    for (uint32_t x = 0; x < q; ++x)
      if (bad_entry(d->unary_values[o + x]))
        throw_model("unary(" + std::to_string(v) + ") entries must be strictly positive and finite");
    o += q;
  }
  std::unordered_set<uint64_t> seen;
  seen.reserve(static_cast<size_t>(E) * 2);
  size_t t = 0;
  for (uint32_t e = 0; e < E; ++e) {
    const uint32_t i = d->edge_endpoints[2ull * e], j = d->edge_endpoints[2ull * e + 1];
    if (i >= V || j >= V) throw_model("edge " + std::to_string(e) + " references a vertex out of range");
    if (i == j) throw_model("edge " + std::to_string(e) + " is a self-loop on vertex " + std::to_string(i));
    if (i > j) throw_model("edge " + std::to_string(e) + " endpoints must satisfy i < j");
    if (check_duplicates && !seen.insert((static_cast<uint64_t>(i) << 32) | j).second)
      throw_model("duplicate edge (" + std::to_string(i) + ", " + std::to_string(j) + ")");
    const size_t sz = static_cast<size_t>(d->cardinalities[i]) * d->cardinalities[j];
    for (size_t k = 0; k < sz; ++k)
      if (bad_entry(d->pairwise_values[t + k]))
        throw_model("pairwise(" + std::to_string(i) + "," + std::to_string(j) +
                    ") entries must be strictly positive and finite");
    t += sz;
  }
}
[[noreturn]] void throw_first_model_error(const bp_graph_desc* d) {
  validate_sequential(d, true);
  throw Error(BP_ERR_CUDA, "internal: graph validation passes disagree");
}

// Pinned host blocks (the process-wide pool, engine.cu) the conversion passes
// write the device layout into; their H2D copies run on the build stream.
struct Staging {
  cudaStream_t st = nullptr;
  std::vector<std::pair<void*, size_t>> blocks;  // size 0: plain heap block (no device present yet)
  ~Staging() {
    if (st) cudaStreamSynchronize(st);
    for (auto& b : blocks)
      if (b.second) pinned_release(b.first, b.second);
      else std::free(b.first);
    if (st) cudaStreamDestroy(st);
  }
  cudaStream_t stream() {
    if (!st) cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    return st;
  }
  template <class T>
  T* get(size_t n) {
    const size_t bytes = ((std::max<size_t>(n * sizeof(T), 1) + (1u << 20) - 1) >> 20) << 20;  // 1 MiB classes
    try {
      void* p = pinned_acquire(bytes);
      blocks.emplace_back(p, bytes);
      return static_cast<T*>(p);
    } catch (const Error&) {  // no usable device: validation still runs (and raises) on the host
      cudaGetLastError();
      void* p = std::malloc(bytes);
      if (!p) throw Error(BP_ERR_OOM, "host staging");
      blocks.emplace_back(p, 0);
      return static_cast<T*>(p);
    }
  }
  // buf <- host[0, n) (host: a staged block, or pageable memory)
  void put(DevBuf& buf, const void* host, size_t n) {
    buf.alloc_async(n, stream());
    if (n) cuda_check(cudaMemcpyAsync(buf.p, host, n, cudaMemcpyHostToDevice, st), "h2d");
  }
  // pageable source: copied into a staged block by the pool first
  void put_copy(DevBuf& buf, const void* host, size_t n) {
    char* h = get<char>(n);
    parallel_for(n, [&](uint64_t a, uint64_t b) { std::memcpy(h + a, static_cast<const char*>(host) + a, b - a); });
    put(buf, h, n);
  }
};

// generate_ising's lattice numbering, checked row by row on the pool
uint32_t detect_lattice_parallel(uint32_t V, uint32_t E, const uint32_t* ep) {
  if (V < 2 || E == 0) return 0;
  uint32_t C = V;
  if (E >= 2 && ep[0] == 0 && ep[1] == 1 && ep[2] == 0 && ep[3] > 1) C = ep[3];
  if (V % C) return 0;
  const uint64_t R = V / C;
  if (static_cast<uint64_t>(E) != R * (C - 1) + (R - 1) * C) return 0;
  const uint64_t bad = first_bad(R, [&](uint64_t r) {
    uint64_t e = r * (2ull * C - 1);  // every earlier row holds C - 1 right + C down edges
    for (uint64_t c = 0; c < C; ++c) {
      const uint64_t v = r * C + c;
      if (c + 1 < C) {
        if (ep[2 * e] != v || ep[2 * e + 1] != v + 1) return true;
        ++e;
      }
      if (r + 1 < R) {
        if (ep[2 * e] != v || ep[2 * e + 1] != v + C) return true;
        ++e;
      }
    }
    return false;
  }, C >= 64);
  return bad == R ? C : 0;
}

struct VAcc {
  uint32_t maxq = 0, minq = std::numeric_limits<uint32_t>::max();
  uint64_t usz = 0;
  bool zero = false, bad = false;
  double min_mu = std::numeric_limits<double>::infinity();
  double min_u = std::numeric_limits<double>::infinity();  // smallest unary entry
};
struct EAcc {
  bool bad = false, ising = true;
  double min_rho = 1.0, min_m = std::numeric_limits<double>::infinity();
  // binary tables: the smallest entry and the extreme row / column sums
  double tmin = std::numeric_limits<double>::infinity(), smin = std::numeric_limits<double>::infinity(), smax = 0.0;
};

// collapse-bound minima of one table t (ci x cj, row-major) of edge (i, j):
// rho = min t(y,x) / row sum, m = max_x psi(x) * row sum, both orientations
inline void table_minima(const double* t, uint32_t ci, uint32_t cj, const double* ui, const double* uj,
                         double& rho, double& m) {
  double mf = 0.0, mb = 0.0;
  for (uint32_t x = 0; x < ci; ++x) {
    double r = 0.0;
    for (uint32_t y = 0; y < cj; ++y) r += t[static_cast<size_t>(x) * cj + y];
    for (uint32_t y = 0; y < cj; ++y) rho = std::min(rho, t[static_cast<size_t>(x) * cj + y] / r);
    mf = std::max(mf, ui[x] * r);
  }
  for (uint32_t y = 0; y < cj; ++y) {
    double r = 0.0;
    for (uint32_t x = 0; x < ci; ++x) r += t[static_cast<size_t>(x) * cj + y];
    for (uint32_t x = 0; x < ci; ++x) rho = std::min(rho, t[static_cast<size_t>(x) * cj + y] / r);
    mb = std::max(mb, uj[y] * r);
  }
  m = std::min(m, std::min(mf, mb));
}

}  // namespace

std::unique_ptr<GraphImpl> build_from_desc(const bp_graph_desc* d, const bp_device_opts* opts) {
  // BPB_DEBUG_BUILD: stage times on stderr (tuning aid)
  static const bool dbg = std::getenv("BPB_DEBUG_BUILD") != nullptr;
  auto tprev = std::chrono::steady_clock::now();
  auto stage = [&](const char* what) {
    if (!dbg) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "build %-12s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(t - tprev).count());
    tprev = t;
  };
  if (!d) throw_invalid("null graph descriptor");
  const uint32_t V = d->num_vertices, E = d->num_edges;
  if (E > (1u << 31) - 1) throw_model("too many edges for 32-bit directed edge ids");
  if (V && !d->cardinalities) throw_invalid("null cardinalities");
  const uint32_t* cards = d->cardinalities;
  // a partition's local graph keeps the global edge orientation (local ids
  // need not satisfy i < j); its input was validated globally
  const bool any_order = opts && (opts->flags & kBuildAnyOrder);
  // --- validation (mrf.cpp:28-91) and layout conversion: O(V + E) passes on
  // the host pool; any violation re-runs the reference's sequential order
  // (throw_first_model_error) so the first error and its message match ---
  VAcc va;
  {
    const unsigned nch = pool_chunks(V);
    std::vector<VAcc> acc(nch);
    parallel_chunks(V, nch, [&](uint64_t lo, uint64_t hi, unsigned t) {
      VAcc a;
      for (uint64_t v = lo; v < hi; ++v) {
        const uint32_t q = cards[v];
        a.zero |= q == 0;
        a.maxq = std::max(a.maxq, q);
        a.minq = std::min(a.minq, q);
        a.usz += q;
      }
      acc[t] = a;
    });
    for (const VAcc& a : acc) {
      va.zero |= a.zero;
      va.maxq = std::max(va.maxq, a.maxq);
      va.minq = std::min(va.minq, a.minq);
      va.usz += a.usz;
    }
  }
  if (va.zero) throw_first_model_error(d);
  const uint32_t maxq = va.maxq;
  const uint64_t usz = va.usz;
  if (usz && !d->unary_values) throw_invalid("null unary values");
  const bool uniform_cards = V == 0 || va.minq == va.maxq;
  const bool bin_cards = V > 0 && uniform_cards && maxq == 2;
  stage("cards");
  Staging stg;
  float* ulo = bin_cards ? stg.get<float>(V) : nullptr;
  std::vector<size_t> uoff;  // mixed cardinalities: unary offsets
  if (!uniform_cards) {
    uoff.assign(static_cast<size_t>(V) + 1, 0);
    for (uint32_t v = 0; v < V; ++v) uoff[v + 1] = uoff[v] + cards[v];
  }
  auto unary_at = [&](uint64_t v) -> size_t { return uniform_cards ? v * maxq : uoff[v]; };
  {
    const unsigned nch = pool_chunks(V);
    std::vector<VAcc> acc(nch);
    parallel_chunks(V, nch, [&](uint64_t lo, uint64_t hi, unsigned t) {
      VAcc a;  // in registers; written back once
      for (uint64_t v = lo; v < hi; ++v) {
        const double* u = d->unary_values + unary_at(v);
        double mu = 0.0, mn = std::numeric_limits<double>::infinity();
        for (uint32_t x = 0; x < cards[v]; ++x) {
          a.bad |= bad_entry(u[x]);
          mu = std::max(mu, u[x]);
          mn = std::min(mn, u[x]);
        }
        a.min_mu = std::min(a.min_mu, mu);
        a.min_u = std::min(a.min_u, mn);
        if (bin_cards) {
          // base-2 log-odds, kept in fp32: the ratio's log in single precision
          // when the ratio is a normal float (error below 1e-7 absolute), else
          // the difference of double logs
          const double r = u[1] / u[0];
          ulo[v] = r >= 1e-30 && r <= 1e30 ? log2f(static_cast<float>(r))
                                           : static_cast<float>(std::log2(u[1]) - std::log2(u[0]));
        }
      }
      acc[t] = a;
    });
    for (const VAcc& a : acc) {
      va.bad |= a.bad;
      va.min_mu = std::min(va.min_mu, a.min_mu);
      va.min_u = std::min(va.min_u, a.min_u);
    }
  }
  if (va.bad) throw_first_model_error(d);
  stage("unary");
  if (E && (!d->edge_endpoints || !d->pairwise_values)) throw_invalid("null edge arrays");
  const uint32_t* ep = d->edge_endpoints;
  // table offsets: e q^2 for a uniform cardinality q, else a prefix sum (after
  // the endpoints are known to be in range)
  std::vector<size_t> poff;
  if (!uniform_cards) {
    if (first_bad(E, [&](uint64_t e) {
          const uint32_t i = ep[2 * e], j = ep[2 * e + 1];
          return i >= V || j >= V || (any_order ? i == j : i >= j);
        }) < E)
      throw_first_model_error(d);
    poff.assign(static_cast<size_t>(E) + 1, 0);
    for (uint32_t e = 0; e < E; ++e)
      poff[e + 1] = poff[e] + static_cast<size_t>(cards[ep[2 * e]]) * cards[ep[2 * e + 1]];
  }
  auto table_at = [&](uint64_t e) -> size_t { return uniform_cards ? e * maxq * maxq : poff[e]; };
  // one pass over the edges: endpoints, table entries, collapse-bound minima,
  // and on binary graphs the Ising couplings a = e^J of tables {a, d, d, a}
  float* isa = bin_cards ? stg.get<float>(E) : nullptr;
  EAcc ea;
  {
    const unsigned nch = pool_chunks(E);
    std::vector<EAcc> acc(nch);
    parallel_chunks(E, nch, [&](uint64_t lo, uint64_t hi, unsigned t) {
      EAcc a;  // in registers; written back once (the per-chunk slots share cache lines)
      for (uint64_t e = lo; e < hi; ++e) {
        const uint32_t i = ep[2 * e], j = ep[2 * e + 1];
        if (i >= V || j >= V || (any_order ? i == j : i >= j)) {
          a.bad = true;
          continue;
        }
        const double* tb = d->pairwise_values + table_at(e);
        const uint32_t ci = cards[i], cj = cards[j];
        if (bin_cards) {
          const double t0 = tb[0], t1 = tb[1], t2 = tb[2], t3 = tb[3];
          a.bad |= bad_entry(t0) || bad_entry(t1) || bad_entry(t2) || bad_entry(t3);
          // collapse-bound inputs without per-edge divisions: rho >= tmin / smax
          // and m >= (smallest unary entry) x smin over the whole model
          const double r0 = t0 + t1, r1 = t2 + t3, c0 = t0 + t2, c1 = t1 + t3;
          a.tmin = std::min(a.tmin, std::min(std::min(t0, t1), std::min(t2, t3)));
          a.smin = std::min(a.smin, std::min(std::min(r0, r1), std::min(c0, c1)));
          a.smax = std::max(a.smax, std::max(std::max(r0, r1), std::max(c0, c1)));
          const bool is = t0 == t3 && t1 == t2;
          a.ising &= is;
          // a = e^J = t0 / t1, clamped to e^{+-69} as ising_weight
          if (is) isa[e] = static_cast<float>(std::min(kIsingAMax, std::max(kIsingAMin, t0 / t1)));
        } else {
          const size_t sz = static_cast<size_t>(ci) * cj;
          for (size_t k = 0; k < sz; ++k) a.bad |= bad_entry(tb[k]);
          table_minima(tb, ci, cj, d->unary_values + unary_at(i), d->unary_values + unary_at(j), a.min_rho,
                       a.min_m);
        }
      }
      acc[t] = a;
    });
    for (const EAcc& a : acc) {
      ea.bad |= a.bad;
      ea.ising &= a.ising;
      ea.min_rho = std::min(ea.min_rho, a.min_rho);
      ea.min_m = std::min(ea.min_m, a.min_m);
      ea.tmin = std::min(ea.tmin, a.tmin);
      ea.smin = std::min(ea.smin, a.smin);
      ea.smax = std::max(ea.smax, a.smax);
    }
    if (bin_cards && E) {  // lower bounds of the per-edge minima (the exact bound runs if these do not clear)
      ea.min_rho = std::min(1.0, ea.tmin / ea.smax);
      ea.min_m = va.min_u * ea.smin;
    }
  }
  if (ea.bad) throw_first_model_error(d);
  stage("edges");
  const uint32_t lat_cols = detect_lattice_parallel(V, E, ep);
  stage("lattice");
  std::vector<uint32_t> off, adj;
  uint32_t maxdeg = lat_cols ? 4 : 0;
  if (!lat_cols) {
    build_csr(V, E, ep, off, adj);
    for (uint32_t v = 0; v < V; ++v) maxdeg = std::max(maxdeg, off[v + 1] - off[v]);
    if (!(opts && (opts->flags & BP_GRAPH_TRUSTED))) {
      // duplicate edges: two incoming edges of one vertex from the same source
      std::vector<uint32_t> mark(V, std::numeric_limits<uint32_t>::max());
      for (uint32_t v = 0; v < V; ++v)
        for (uint32_t a = off[v]; a < off[v + 1]; ++a) {
          const uint32_t src = ep[adj[a]];
          if (mark[src] == v) throw_first_model_error(d);
          mark[src] = v;
        }
    }
  }
  stage("csr");
  // Can the reference's numeric_error (normalize_in_place: total mass below
  // 1e-300, messages.cpp:41-49) ever fire on this model?  A lower bound of
  // every message's unnormalised mass: a message m_k out of a table t_k has
  // m_k(x) >= rho_k = min_{y,x} t_k(y,x) / sum_x' t_k(y,x') (any non-negative
  // mixture of the rows; also the uniform initial messages), so the mass of
  // d = (i -> j) is >= max_x psi_i(x) R_d(x) prod_{k in in(i), k != d^1} rho_k
  // (R_d = row sums of t oriented i -> j), and a belief's is >= max_x psi_v(x)
  // prod_{k in in(v)} rho_k.  Models where every bound clears 1e-290 (all
  // generated instances, any sane input) never collapse in the reference; the
  // others are built with the q-state layout and log-domain tables, and the
  // device computes the reference's mass exactly (generic_logmatvec) to raise
  // the same error.  First the bound from the global minima (rho, R psi, psi)
  // and the maximum degree, with a margin of e; the per-message bound only
  // when that one does not clear.
  const double floor = std::log(1e-290);
  bool collapse_free;
  {
    const double lr = std::log(ea.min_rho), lm = std::log(ea.min_m), lmu = std::log(va.min_mu);
    collapse_free = lmu + maxdeg * lr >= floor + 1.0 && (E == 0 || lm + (maxdeg - 1.0) * lr >= floor + 1.0);
  }
  if (!collapse_free) {
    collapse_free = true;
    std::vector<double> lrho(2ull * E), lrmax(2ull * E), LI(V, 0.0);
    for (uint32_t e = 0; e < E; ++e) {
      const uint32_t i = ep[2 * e], j = ep[2 * e + 1];
      const uint32_t ci = cards[i], cj = cards[j];
      const double* t = d->pairwise_values + table_at(e);
      double rho_f = 1.0, rho_b = 1.0, mf = 0.0, mb = 0.0;
      for (uint32_t x = 0; x < ci; ++x) {  // d = 2e: rows x_i
        double r = 0.0;
        for (uint32_t y = 0; y < cj; ++y) r += t[static_cast<size_t>(x) * cj + y];
        for (uint32_t y = 0; y < cj; ++y) rho_f = std::min(rho_f, t[static_cast<size_t>(x) * cj + y] / r);
        mf = std::max(mf, d->unary_values[unary_at(i) + x] * r);
      }
      for (uint32_t y = 0; y < cj; ++y) {  // d = 2e + 1: rows x_j
        double r = 0.0;
        for (uint32_t x = 0; x < ci; ++x) r += t[static_cast<size_t>(x) * cj + y];
        for (uint32_t x = 0; x < ci; ++x) rho_b = std::min(rho_b, t[static_cast<size_t>(x) * cj + y] / r);
        mb = std::max(mb, d->unary_values[unary_at(j) + y] * r);
      }
      lrho[2ull * e] = std::log(rho_f);      // message into j
      lrho[2ull * e + 1] = std::log(rho_b);  // message into i
      lrmax[2ull * e] = std::log(mf);
      lrmax[2ull * e + 1] = std::log(mb);
      LI[j] += lrho[2ull * e];
      LI[i] += lrho[2ull * e + 1];
    }
    for (uint64_t dd = 0; dd < 2ull * E && collapse_free; ++dd) {
      const uint32_t src = ep[dd];  // ep[d] = source of d
      collapse_free = lrmax[dd] + LI[src] - lrho[dd ^ 1ull] >= floor;
    }
    for (uint32_t v = 0; v < V && collapse_free; ++v) {
      double mu = 0.0;
      for (uint32_t x = 0; x < cards[v]; ++x) mu = std::max(mu, d->unary_values[unary_at(v) + x]);
      collapse_free = std::log(mu) + LI[v] >= floor;
    }
  }
  stage("collapse bound");
  auto g = std::make_unique<GraphImpl>();
  g->device = select_device(opts);
  g->V = V;
  g->E = E;
  g->D = 2 * E;
  g->maxq = maxq;
  g->binary = bin_cards && collapse_free;
  if (uniform_cards && V) g->uniform_q = cards[0];
  else g->cards_host.assign(cards, cards + V);
  if (lat_cols) {
    g->in_off.alloc_async((static_cast<size_t>(V) + 1) * 4, stg.stream());
    g->in_adj.alloc_async(static_cast<size_t>(E) * 8, stg.st);
    g->ep.alloc_async(static_cast<size_t>(E) * 8, stg.st);
    k_lattice_topology<<<grid_for(V), 256, 0, stg.st>>>(V / lat_cols, lat_cols, g->in_off.as<uint32_t>(),
                                                        g->in_adj.as<uint32_t>(), g->ep.as<uint32_t>());
    cuda_check(cudaGetLastError(), "lattice topology");
  } else {
    stg.put_copy(g->in_off, off.data(), off.size() * 4);
    stg.put_copy(g->in_adj, adj.data(), adj.size() * 4);
    stg.put_copy(g->ep, ep, static_cast<size_t>(E) * 8);
  }
  stage("topology");
  if (g->binary || V == 0) {
    g->binary = true;
    g->qs = 1;
    stg.put(g->unary_lo, ulo, ulo ? static_cast<size_t>(V) * 4 : 0);
    if (E > 0 && ea.ising) {  // Ising tables {a, d, d, a} (generators.cpp:18-22): one coupling per edge
      stg.put(g->ising_a, isa, static_cast<size_t>(E) * 4);
      g->par_mode = 1;
    } else {
      float4* par = stg.get<float4>(E);
      parallel_for(E, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t e = lo; e < hi; ++e) {
          const double* t = d->pairwise_values + 4ull * e;
          const double l00 = std::log2(t[0]), l01 = std::log2(t[1]), l10 = std::log2(t[2]), l11 = std::log2(t[3]);
          const double alpha = l01 - l00, beta = l10 - l00, gg = l11 - l00;
          par[e] = make_float4(static_cast<float>(alpha), static_cast<float>(beta), static_cast<float>(gg - alpha),
                               static_cast<float>(gg - beta));
        }
      });
      stg.put(g->epar, par, static_cast<size_t>(E) * 16);
    }
  } else {
    const uint32_t qs = stride_for(maxq);
    g->qs = qs;
    std::vector<float> ul(static_cast<size_t>(V) * qs, 0.f);
    std::vector<uint32_t> bo(static_cast<size_t>(V) + 1, 0);
    for (uint32_t v = 0, o = 0; v < V; o += d->cardinalities[v], ++v) {
      bo[v + 1] = bo[v] + d->cardinalities[v];
      for (uint32_t x = 0; x < d->cardinalities[v]; ++x)
        ul[static_cast<size_t>(v) * qs + x] = static_cast<float>(std::log2(d->unary_values[o + x]));  // base 2
    }
    // Potts tables (a on the diagonal, d off it, square): one weight per edge
    // (not on collapse-checked models: their mass check uses the dense tables' scales)
    bool potts = E > 0 && collapse_free;
    std::vector<float> w1(potts ? E : 0);
    for (uint32_t e = 0; e < E && potts; ++e) {
      const uint32_t i = d->edge_endpoints[2 * e], j = d->edge_endpoints[2 * e + 1];
      const uint32_t ci = d->cardinalities[i], cj = d->cardinalities[j];
      const double* t = d->pairwise_values + table_at(e);
      if (ci != cj || ci < 2) {
        potts = false;
        break;
      }
      const double a = t[0], dd = t[1];
      for (uint32_t x = 0; x < ci && potts; ++x)
        for (uint32_t y = 0; y < cj && potts; ++y) potts = t[static_cast<size_t>(x) * cj + y] == (x == y ? a : dd);
      if (potts) w1[e] = static_cast<float>(a / dd - 1.0);
    }
    std::vector<float> tb(potts ? 0 : static_cast<size_t>(E) * qs * qs, 0.f);
    if (potts) {
      g->pw.upload(w1.data(), w1.size() * 4);
      g->par_mode = 1;
    }
    for (uint32_t e = 0; e < E && !potts; ++e) {
      const uint32_t i = d->edge_endpoints[2 * e], j = d->edge_endpoints[2 * e + 1];
      const uint32_t ci = d->cardinalities[i], cj = d->cardinalities[j];
      const double* t = d->pairwise_values + table_at(e);
      double mx = 0.0;
      for (size_t k = 0; k < static_cast<size_t>(ci) * cj; ++k) mx = std::max(mx, t[k]);
      if (!collapse_free) {  // log-domain tables: log2 t, unscaled (generic_logmatvec)
        for (uint32_t a = 0; a < ci; ++a)
          for (uint32_t b = 0; b < cj; ++b)
            tb[static_cast<size_t>(e) * qs * qs + static_cast<size_t>(a) * qs + b] =
                static_cast<float>(std::log2(t[static_cast<size_t>(a) * cj + b]));
        continue;
      }
      for (uint32_t a = 0; a < ci; ++a)
        for (uint32_t b = 0; b < cj; ++b) {
          // max-scaled linear fp32; clamped so no entry underflows to 0
          const double s = t[static_cast<size_t>(a) * cj + b] / mx;
          tb[static_cast<size_t>(e) * qs * qs + static_cast<size_t>(a) * qs + b] =
              static_cast<float>(std::max(s, 1e-30));
        }
    }
    g->card.upload(d->cardinalities, static_cast<size_t>(V) * 4);
    g->unary_log.upload(ul.data(), ul.size() * 4);
    if (!potts) g->table.upload(tb.data(), tb.size() * 4);
    g->check_collapse = !collapse_free;
    g->bel_off.upload(bo.data(), bo.size() * 4);
  }
  g->lat_cols = lat_cols;
  g->lat_rows = lat_cols ? V / lat_cols : 0;
  cuda_check(cudaStreamSynchronize(stg.stream()), "graph upload");
  cuda_check(cudaDeviceSynchronize(), "graph upload");
  stage("potentials");
  return g;
}

// Vertex-range partition of any binary model (north_star: LBP / RnBP on large
// grids AND random graphs partitioned across GPUs).  Part g of P owns global
// vertices [V g / P, V (g + 1) / P) and every message whose source it owns.
// Its local graph: the global edges with an owned endpoint, in global order
// and orientation; local vertices = owned ones (in order) then one ghost per
// outside endpoint (ascending global id).  Ghosts are never updated: their
// messages into owned vertices arrive from their owners every iteration
// (recv lists), and the owned-source messages into ghosts leave for their
// owners (send lists); both sides order a peer's run by global directed id.
std::unique_ptr<GraphImpl> build_part(const bp_graph_desc* d, uint32_t part, uint32_t nparts,
                                      const bp_device_opts* opts, PartLayout& out) {
  if (!d) throw_invalid("null graph descriptor");
  const uint32_t V = d->num_vertices, E = d->num_edges;
  if (nparts == 0 || part >= nparts || (V && nparts > V)) throw_invalid("bad vertex-range partition");
  if (V && !d->cardinalities) throw_invalid("null cardinalities");
  if (E && (!d->edge_endpoints || !d->pairwise_values)) throw_invalid("null edge arrays");
  validate_sequential(d, !(opts && (opts->flags & BP_GRAPH_TRUSTED)));  // build_graph's checks, globally
  for (uint32_t v = 0; v < V; ++v)
    if (d->cardinalities[v] != 2) throw Error(BP_ERR_UNSUPPORTED, "vertex-range partition: binary models only");
  const uint32_t v0 = static_cast<uint32_t>(uint64_t{V} * part / nparts);
  const uint32_t v1 = static_cast<uint32_t>(uint64_t{V} * (part + 1) / nparts);
  const uint32_t nown = v1 - v0;
  auto owner = [&](uint32_t v) {
    uint32_t h = static_cast<uint32_t>(uint64_t{v} * nparts / V);
    while (h + 1 < nparts && uint64_t{V} * (h + 1) / nparts <= v) ++h;
    while (h > 0 && uint64_t{V} * h / nparts > v) --h;
    return h;
  };
  const uint32_t* ep = d->edge_endpoints;
  auto own = [&](uint32_t v) { return v >= v0 && v < v1; };
  std::vector<uint32_t> gid, ghosts;
  for (uint32_t e = 0; e < E; ++e) {
    const uint32_t i = ep[2ull * e], j = ep[2ull * e + 1];
    if (!own(i) && !own(j)) continue;
    gid.push_back(e);
    if (!own(i)) ghosts.push_back(i);
    if (!own(j)) ghosts.push_back(j);
  }
  std::sort(ghosts.begin(), ghosts.end());
  ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
  auto loc = [&](uint32_t v) -> uint32_t {
    return own(v) ? v - v0 : nown + static_cast<uint32_t>(std::lower_bound(ghosts.begin(), ghosts.end(), v) - ghosts.begin());
  };
  const uint32_t VL = nown + static_cast<uint32_t>(ghosts.size()), EL = static_cast<uint32_t>(gid.size());
  std::vector<uint32_t> lcards(VL, 2), lep(2ull * EL);
  std::vector<double> lun(2ull * VL), ltb(4ull * EL);
  for (uint32_t v = 0; v < VL; ++v) {
    const uint32_t gv = v < nown ? v0 + v : ghosts[v - nown];
    lun[2ull * v] = d->unary_values[2ull * gv];
    lun[2ull * v + 1] = d->unary_values[2ull * gv + 1];
  }
  for (uint32_t e = 0; e < EL; ++e) {
    const uint64_t ge = gid[e];
    lep[2ull * e] = loc(ep[2 * ge]);
    lep[2ull * e + 1] = loc(ep[2 * ge + 1]);
    for (int k = 0; k < 4; ++k) ltb[4ull * e + k] = d->pairwise_values[4 * ge + k];
  }
  const bp_graph_desc ld{VL, EL, lcards.data(), lun.data(), lep.data(), ltb.data()};
  bp_device_opts lo{opts ? opts->device : -1, BP_GRAPH_TRUSTED | kBuildAnyOrder};
  auto g = build_from_desc(&ld, &lo);
  g->lat_cols = g->lat_rows = 0;  // the CSR is complete either way; ownership is by vertex id
  g->own_v = nown;
  g->part = part;
  g->nparts = nparts;
  g->v0 = v0;
  g->v1 = v1;
  g->egid_host = gid;
  if (EL) g->egid.upload(gid.data(), 4ull * EL);
  // cut-message lists per peer, each run sorted by global directed id
  std::vector<std::vector<std::pair<uint64_t, uint32_t>>> snd(nparts), rcv(nparts);
  uint64_t owned_directed = 0;
  for (uint32_t e = 0; e < EL; ++e)
    for (uint32_t b = 0; b < 2; ++b) {
      const uint32_t dl = 2 * e + b;
      const uint32_t src = lep[dl], tgt = lep[dl ^ 1u];
      const uint64_t key = 2ull * gid[e] + b;
      if (src < nown) {
        ++owned_directed;
        if (tgt >= nown) snd[owner(ghosts[tgt - nown])].emplace_back(key, dl);
      } else if (tgt < nown) {
        rcv[owner(ghosts[src - nown])].emplace_back(key, dl);
      }
    }
  std::vector<uint32_t> sidx, ridx;
  for (uint32_t h = 0; h < nparts; ++h) {
    if (snd[h].empty() && rcv[h].empty()) continue;
    std::sort(snd[h].begin(), snd[h].end());
    std::sort(rcv[h].begin(), rcv[h].end());
    GraphImpl::PartPeer p{h, static_cast<uint32_t>(sidx.size()), static_cast<uint32_t>(snd[h].size()),
                          static_cast<uint32_t>(ridx.size()), static_cast<uint32_t>(rcv[h].size())};
    for (auto& x : snd[h]) sidx.push_back(x.second);
    for (auto& x : rcv[h]) ridx.push_back(x.second);
    g->peers.push_back(p);
  }
  g->send_idx.upload(sidx.data(), 4ull * sidx.size());
  g->recv_idx.upload(ridx.data(), 4ull * ridx.size());
  g->owned_directed = owned_directed;
  out = PartLayout{part, nparts, v0, v1, static_cast<uint32_t>(ghosts.size()), EL,
                   static_cast<uint32_t>(g->peers.size()), sidx.size(), ridx.size(), owned_directed};
  return g;
}

uint32_t lattice_cols(uint32_t V, uint32_t E, const uint32_t* ep) { return detect_lattice(V, E, ep); }

std::unique_ptr<GraphImpl> build_lattice_binary(uint32_t rows, uint32_t cols, const BinaryStreams& s,
                                                const bp_device_opts* opts) {
  auto g = std::make_unique<GraphImpl>();
  g->device = select_device(opts);
  const uint64_t V = static_cast<uint64_t>(rows) * cols;
  const uint64_t E = s.coupling.size();
  if (2 * E >= (1ull << 32)) throw_model("too many edges for 32-bit directed edge ids");
  g->V = static_cast<uint32_t>(V);
  g->E = static_cast<uint32_t>(E);
  g->D = static_cast<uint32_t>(2 * E);
  g->maxq = V ? 2 : 0;
  g->binary = true;
  g->qs = 1;
  g->uniform_q = 2;
  g->in_off.alloc((V + 1) * 4);
  g->in_adj.alloc(2 * E * 4);
  g->ep.alloc(2 * E * 4);
  if (V) {
    k_lattice_topology<<<grid_for(V), 256>>>(rows, cols, g->in_off.as<uint32_t>(), g->in_adj.as<uint32_t>(),
                                             g->ep.as<uint32_t>());
    cuda_check(cudaGetLastError(), "lattice topology");
  } else {
    cuda_check(cudaMemset(g->in_off.p, 0, 4), "memset");
  }
  g->unary_lo.upload(s.unary_lo.data(), V * 4);
  upload_ising_weights(*g, s.coupling);  // J = 2 lambda c: table {e^lc, e^-lc, e^-lc, e^lc}
  g->par_mode = 1;
  if (V > 1) {
    g->lat_rows = rows;
    g->lat_cols = cols;
  }
  cuda_check(cudaDeviceSynchronize(), "lattice build");
  return g;
}

std::unique_ptr<GraphImpl> build_potts(uint32_t n, uint32_t q, const PottsStreams& s,
                                       const bp_device_opts* opts) {
  if (q < 2) throw_invalid("potts: q must be >= 2");
  auto g = std::make_unique<GraphImpl>();
  g->device = select_device(opts);
  const uint64_t V = static_cast<uint64_t>(n) * n;
  const uint64_t E = s.lambda_c.size();
  if (2 * E >= (1ull << 32)) throw_model("too many edges for 32-bit directed edge ids");
  g->V = static_cast<uint32_t>(V);
  g->E = static_cast<uint32_t>(E);
  g->D = static_cast<uint32_t>(2 * E);
  g->maxq = q;
  g->uniform_q = q;
  g->binary = false;
  const uint32_t qs = stride_for(q);
  g->qs = qs;
  g->in_off.alloc((V + 1) * 4);
  g->in_adj.alloc(2 * E * 4);
  g->ep.alloc(2 * E * 4);
  if (V) {
    k_lattice_topology<<<grid_for(V), 256>>>(n, n, g->in_off.as<uint32_t>(), g->in_adj.as<uint32_t>(),
                                             g->ep.as<uint32_t>());
    cuda_check(cudaGetLastError(), "lattice topology");
  }
  std::vector<float> ul(V * qs, 0.f);
  for (uint64_t v = 0; v < V; ++v)
    for (uint32_t x = 0; x < q; ++x) ul[v * qs + x] = s.unary_log[v * q + x];
  g->unary_log.upload(ul.data(), ul.size() * 4);
  g->card.alloc(V * 4);
  if (V) k_fill_u32<<<grid_for(V), 256>>>(g->card.as<uint32_t>(), V, q);
  g->bel_off.alloc((V + 1) * 4);
  k_iota_mul<<<grid_for(V + 1), 256>>>(g->bel_off.as<uint32_t>(), V + 1, q);
  // table: exp(lc) on the diagonal, exp(-lc) off it -> w1 = exp(2 lc) - 1
  std::vector<float> w1(E);
  for (uint64_t e = 0; e < E; ++e) w1[e] = static_cast<float>(std::expm1(2.0 * static_cast<double>(s.lambda_c[e])));
  g->pw.upload(w1.data(), E * 4);
  g->par_mode = 1;
  if (V > 1) {
    g->lat_rows = n;
    g->lat_cols = n;
  }
  cuda_check(cudaDeviceSynchronize(), "potts build");
  return g;
}

std::unique_ptr<GraphImpl> build_er(uint32_t n, const ErInstance& inst, const bp_device_opts* opts) {
  auto g = std::make_unique<GraphImpl>();
  g->device = select_device(opts);
  const uint32_t E = static_cast<uint32_t>(inst.coupling.size());
  g->V = n;
  g->E = E;
  g->D = 2 * E;
  g->maxq = n ? 2 : 0;
  g->uniform_q = 2;
  g->binary = true;
  g->qs = 1;
  std::vector<uint32_t> off, adj;
  build_csr(n, E, inst.endpoints.data(), off, adj);
  g->in_off.upload(off.data(), off.size() * 4);
  g->in_adj.upload(adj.data(), adj.size() * 4);
  g->ep.upload(inst.endpoints.data(), static_cast<size_t>(E) * 8);
  g->unary_lo.upload(inst.unary_lo.data(), static_cast<size_t>(n) * 4);
  upload_ising_weights(*g, inst.coupling);
  g->par_mode = 1;
  cuda_check(cudaDeviceSynchronize(), "er build");
  return g;
}

// ---------------------------------------------------------------------------
// ball lists (kernels_rs.cuh): distinct vertices within distance h, walk order

constexpr int kBallCap = 256;

template <class F>
__device__ __forceinline__ int distinct_ball(const DevGraph& g, uint32_t v, uint32_t h, uint32_t* buf, bool& of,
                                             F&& emit) {
  int n = 0;
  of = false;
  ball_walk(g, v, h, [&](uint32_t w) {
    for (int i = 0; i < n; ++i)
      if (buf[i] == w) return true;
    if (n == kBallCap) {
      of = true;
      return false;
    }
    buf[n++] = w;
    emit(w);
    return true;
  });
  return n;
}

__global__ void k_ball_count(DevGraph g, uint32_t h, unsigned* cnt, unsigned* overflow) {
  uint32_t buf[kBallCap];
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < g.V; v += gridDim.x * blockDim.x) {
    bool of;
    cnt[v] = distinct_ball(g, v, h, buf, of, [](uint32_t) {});
    if (of) *overflow = 1u;
  }
}

__global__ void k_ball_fill(DevGraph g, uint32_t h, const unsigned long long* off, uint32_t* out) {
  uint32_t buf[kBallCap];
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < g.V; v += gridDim.x * blockDim.x) {
    bool of;
    unsigned long long o = off[v];
    distinct_ball(g, v, h, buf, of, [&](uint32_t w) { out[o++] = w; });
  }
}

const BallLists* GraphImpl::balls(uint32_t h) const {
  std::lock_guard<std::mutex> lk(host_mu);
  auto it = balls_.find(h);
  if (it != balls_.end()) return it->second.get();
  if (balls_too_big_.count(h) || V == 0) return nullptr;
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  const DevGraph dg = dev();
  DevBuf cnt, of;
  cnt.alloc(static_cast<size_t>(V) * 4);
  of.alloc(4);
  cuda_check(cudaMemset(of.p, 0, 4), "memset");
  const unsigned grid = static_cast<unsigned>(std::min<size_t>((V + 127) / 128, 148ull * 16));
  k_ball_count<<<grid, 128>>>(dg, h, cnt.as<unsigned>(), of.as<unsigned>());
  cuda_check(cudaGetLastError(), "ball count");
  unsigned overflow = 0;
  std::vector<unsigned> c(V);
  cuda_check(cudaMemcpy(&overflow, of.p, 4, cudaMemcpyDeviceToHost), "d2h");
  cuda_check(cudaMemcpy(c.data(), cnt.p, 4ull * V, cudaMemcpyDeviceToHost), "d2h");
  std::vector<unsigned long long> off(static_cast<size_t>(V) + 1, 0);
  for (uint32_t v = 0; v < V; ++v) off[v + 1] = off[v] + c[v];
  // budget: 32 entries per vertex on average (grid h=2: 13, ER deg 4 h=2: ~21)
  if (overflow || off[V] > 32ull * V + (1ull << 20)) {
    balls_too_big_[h] = true;
    return nullptr;
  }
  auto b = std::make_unique<BallLists>();
  b->off.upload(off.data(), off.size() * 8);
  b->list.alloc(std::max<size_t>(off[V] * 4, 16));
  k_ball_fill<<<grid, 128>>>(dg, h, b->off.as<unsigned long long>(), b->list.as<uint32_t>());
  cuda_check(cudaDeviceSynchronize(), "ball fill");
  const BallLists* out = b.get();
  balls_[h] = std::move(b);
  return out;
}

// Host copies needed only by the lockstep API (message conversion).
const std::vector<uint32_t>& GraphImpl::host_ep() const {
  std::lock_guard<std::mutex> lk(host_mu);
  if (ep_host.size() != 2ull * E) {
    ep_host.resize(2ull * E);
    if (E) cuda_check(cudaMemcpy(ep_host.data(), ep.p, 8ull * E, cudaMemcpyDeviceToHost), "ep download");
  }
  return ep_host;
}

const std::vector<uint32_t>& GraphImpl::host_in_off() const {
  std::lock_guard<std::mutex> lk(host_mu);
  if (in_off_host.size() != static_cast<size_t>(V) + 1) {
    in_off_host.resize(static_cast<size_t>(V) + 1);
    cuda_check(cudaMemcpy(in_off_host.data(), in_off.p, 4ull * (V + 1), cudaMemcpyDeviceToHost), "csr download");
  }
  return in_off_host;
}

const std::vector<uint32_t>& GraphImpl::host_in_adj() const {
  std::lock_guard<std::mutex> lk(host_mu);
  if (in_adj_host.size() != static_cast<size_t>(D)) {
    in_adj_host.resize(D);
    if (D) cuda_check(cudaMemcpy(in_adj_host.data(), in_adj.p, 4ull * D, cudaMemcpyDeviceToHost), "csr download");
  }
  return in_adj_host;
}

uint32_t GraphImpl::card_of(uint32_t v) const {
  if (uniform_q) return uniform_q;
  return cards_host[v];
}

}  // namespace bpb
