// Host-side instance generators.  The Ising / chain streams restate
// generators.cpp:24-71 of the reference (all unaries in vertex order via
// unit_open, then one lambda = uniform_unit - 0.5 per edge in edge order), so
// the generated instance equals generate_ising / generate_chain bit for bit;
// only the derived fp32 device parameters are produced here, which is what
// lets 16384^2 grids be generated without a PairwiseMRF on the host.
#include <algorithm>
#include <cmath>
#include <thread>
#include <unordered_set>

#include "bp_internal.hpp"

namespace bpb {

Mt64::Mt64(uint64_t seed) {
  mt_[0] = seed;
  for (int i = 1; i < 312; ++i) mt_[i] = 6364136223846793005ULL * (mt_[i - 1] ^ (mt_[i - 1] >> 62)) + i;
  idx_ = 312;
}

uint64_t Mt64::next() {
  constexpr uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
  if (idx_ >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (mt_[i] & UM) | (mt_[(i + 1) % 312] & LM);
      mt_[i] = mt_[(i + 156) % 312] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
    }
    idx_ = 0;
  }
  uint64_t x = mt_[idx_++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

namespace {

// Parallel map over [0, n) on the host (log transforms of the drawn values).
template <class F>
void parallel_for(size_t n, F&& f) {
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (n < (1u << 20) || hw == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> ts;
  for (unsigned t = 0; t < hw; ++t)
    ts.emplace_back([&, t] { f(n * t / hw, n * (t + 1) / hw); });
  for (auto& t : ts) t.join();
}

BinaryStreams lattice_streams(uint32_t rows, uint32_t cols, double c, uint64_t seed) {
  Mt64 rng(seed);
  const size_t V = static_cast<size_t>(rows) * cols;
  std::vector<double> u(2 * V);
  for (size_t k = 0; k < 2 * V; ++k) u[k] = rng.unit_open();
  const size_t E = (rows ? static_cast<size_t>(rows) * (cols - (cols ? 1 : 0)) : 0) +
                   (cols && rows ? static_cast<size_t>(rows - 1) * cols : 0);
  BinaryStreams s;
  s.coupling.resize(E);
  for (size_t e = 0; e < E; ++e) {
    const double lambda = rng.unit() - 0.5;
    // table {e^{lc}, e^{-lc}, e^{-lc}, e^{lc}} (generators.cpp:18-22): the
    // log-table differences are alpha = beta = -2 lc, g = 0.
    s.coupling[e] = static_cast<float>(2.0 * (lambda * c));
  }
  s.unary_lo.resize(V);
  parallel_for(V, [&](size_t b, size_t e) {
    for (size_t v = b; v < e; ++v) s.unary_lo[v] = static_cast<float>(std::log2(u[2 * v + 1]) - std::log2(u[2 * v]));
  });
  return s;
}

}  // namespace

BinaryStreams ising_streams(uint32_t n, double c, uint64_t seed) { return lattice_streams(n, n, c, seed); }

// Rows [a, b) of generate_ising's n x n instance as a stand-alone
// (b - a) x n lattice: same unaries and couplings; the band's last row keeps
// only its right edges (its down edges lead out of the band).
BinaryStreams ising_band_streams(uint32_t n, double c, uint64_t seed, uint32_t a, uint32_t b) {
  if (a >= b || b > n) throw_invalid("ising band: need 0 <= a < b <= n");
  const BinaryStreams full = lattice_streams(n, n, c, seed);
  const size_t C = n, L = b - a, row = 2 * C - 1;
  BinaryStreams s;
  s.unary_lo.assign(full.unary_lo.begin() + a * C, full.unary_lo.begin() + b * C);
  s.coupling.resize((L - 1) * row + (C - 1));
  for (size_t lr = 0; lr + 1 < L; ++lr)
    std::copy(full.coupling.begin() + (a + lr) * row, full.coupling.begin() + (a + lr + 1) * row,
              s.coupling.begin() + lr * row);
  const size_t r = b - 1;
  for (size_t col = 0; col + 1 < C; ++col)
    s.coupling[(L - 1) * row + col] = full.coupling[r * row + (r + 1 == n ? col : 2 * col)];
  return s;
}
BinaryStreams chain_streams(uint32_t length, double c, uint64_t seed) {
  return lattice_streams(length ? 1 : 0, length, c, seed);
}

PottsStreams potts_streams(uint32_t n, uint32_t q, double c, uint64_t seed) {
  Mt64 rng(seed);
  const size_t V = static_cast<size_t>(n) * n;
  PottsStreams s;
  std::vector<double> u(V * q);
  for (size_t k = 0; k < V * q; ++k) u[k] = rng.unit_open();
  const size_t E = n ? 2ull * n * (n - 1) : 0;
  s.lambda_c.resize(E);
  for (size_t e = 0; e < E; ++e) s.lambda_c[e] = static_cast<float>((rng.unit() - 0.5) * c);
  s.unary_log.resize(V * q);
  parallel_for(V * q, [&](size_t b, size_t e) {
    for (size_t k = b; k < e; ++k) s.unary_log[k] = static_cast<float>(std::log2(u[k]));  // base-2 (device layout)
  });
  return s;
}

// G(n, m) stream: unaries 2 x unit_open per vertex, then
// (floor(u n), floor(u n)) pairs redrawn on self-loops / duplicates until m
// distinct edges, sorted by (i, j), then one lambda per edge
namespace {
struct ErStream {
  std::vector<double> u;         // 2n unaries
  std::vector<uint64_t> keys;    // (i << 32) | j, sorted
  std::vector<double> lambda;    // per edge
};
ErStream er_stream(uint32_t n, uint32_t m, uint64_t seed) {
  if (m > 0 && n < 2) throw_invalid("er: need n >= 2");
  if (static_cast<uint64_t>(m) > static_cast<uint64_t>(n) * (n - 1) / 2) throw_invalid("er: too many edges");
  Mt64 rng(seed);
  ErStream st;
  st.u.resize(2 * static_cast<size_t>(n));
  for (auto& x : st.u) x = rng.unit_open();
  st.keys.reserve(m);
  std::unordered_set<uint64_t> seen;
  seen.reserve(static_cast<size_t>(m) * 2);
  while (st.keys.size() < m) {
    uint32_t a = static_cast<uint32_t>(rng.unit() * static_cast<double>(n));
    uint32_t b = static_cast<uint32_t>(rng.unit() * static_cast<double>(n));
    if (a == b) continue;
    if (a > b) std::swap(a, b);
    const uint64_t key = (static_cast<uint64_t>(a) << 32) | b;
    if (!seen.insert(key).second) continue;
    st.keys.push_back(key);
  }
  std::sort(st.keys.begin(), st.keys.end());
  st.lambda.resize(m);
  for (auto& l : st.lambda) l = rng.unit() - 0.5;
  return st;
}
}  // namespace

ErInstance er_instance(uint32_t n, uint32_t m, double c, uint64_t seed) {
  const ErStream st = er_stream(n, m, seed);
  ErInstance inst;
  inst.endpoints.resize(2 * static_cast<size_t>(m));
  inst.coupling.resize(m);
  for (uint32_t k = 0; k < m; ++k) {
    inst.endpoints[2 * k] = static_cast<uint32_t>(st.keys[k] >> 32);
    inst.endpoints[2 * k + 1] = static_cast<uint32_t>(st.keys[k]);
    inst.coupling[k] = static_cast<float>(2.0 * (st.lambda[k] * c));
  }
  inst.unary_lo.resize(n);
  for (uint32_t v = 0; v < n; ++v)
    inst.unary_lo[v] = static_cast<float>(std::log2(st.u[2 * v + 1]) - std::log2(st.u[2 * v]));
  return inst;
}

void er_desc_arrays(uint32_t n, uint32_t m, double c, uint64_t seed, std::vector<uint32_t>& cards,
                    std::vector<double>& unary, std::vector<uint32_t>& ep, std::vector<double>& tables) {
  const ErStream st = er_stream(n, m, seed);
  cards.assign(n, 2);
  unary = st.u;
  ep.resize(2 * static_cast<size_t>(m));
  tables.resize(4 * static_cast<size_t>(m));
  for (uint32_t k = 0; k < m; ++k) {
    ep[2 * k] = static_cast<uint32_t>(st.keys[k] >> 32);
    ep[2 * k + 1] = static_cast<uint32_t>(st.keys[k]);
    const double agree = std::exp(st.lambda[k] * c), disagree = std::exp(-st.lambda[k] * c);
    tables[4 * k] = agree;
    tables[4 * k + 1] = disagree;
    tables[4 * k + 2] = disagree;
    tables[4 * k + 3] = agree;
  }
}

void ising_desc_arrays(uint32_t rows, uint32_t cols, double c, uint64_t seed,
                       std::vector<uint32_t>& cards, std::vector<double>& unary,
                       std::vector<uint32_t>& ep, std::vector<double>& tables) {
  Mt64 rng(seed);
  const size_t V = static_cast<size_t>(rows) * cols;
  cards.assign(V, 2);
  unary.resize(2 * V);
  for (auto& x : unary) x = rng.unit_open();
  ep.clear();
  for (uint32_t r = 0; r < rows; ++r)
    for (uint32_t col = 0; col < cols; ++col) {
      const uint32_t v = r * cols + col;
      if (col + 1 < cols) {
        ep.push_back(v);
        ep.push_back(v + 1);
      }
      if (r + 1 < rows) {
        ep.push_back(v);
        ep.push_back(v + cols);
      }
    }
  const size_t E = ep.size() / 2;
  tables.resize(4 * E);
  for (size_t e = 0; e < E; ++e) {
    const double lambda = rng.unit() - 0.5;
    const double agree = std::exp(lambda * c), disagree = std::exp(-lambda * c);
    tables[4 * e] = agree;
    tables[4 * e + 1] = disagree;
    tables[4 * e + 2] = disagree;
    tables[4 * e + 3] = agree;
  }
}

}  // namespace bpb
