// Device-side data layout, numerics and RNG of the B200 BP engine.
//
// Layout in HBM:
//   * directed edge d of undirected edge e = d >> 1: 2e = lo->hi, 2e+1 = hi->lo
//     (mrf.cpp:89-90); src(d) = ep[d], tgt(d) = ep[d ^ 1] with ep = (lo, hi)
//     pairs, so the reference's DirectedEdge table (mrf.hpp:14-18) is implicit.
//   * incoming CSR in edge-id order (mrf.cpp:93-104): in_off[V+1], in_adj[D].
//   * messages are stored per directed edge in id order, so the two directions
//     of one undirected edge are adjacent ("edge pair"): a vertex update loads
//     one pair and gets both the incoming message and the old outgoing message
//     it needs for the residual.
//   * binary graphs (all cardinalities 2): one fp32 BASE-2 log-odds per
//     message, log2(m(1)/m(0)); unary log2-odds per vertex; per edge either
//     a = e^J (Ising tables) or a float4 of log2-table differences.  Base 2
//     makes every transcendental one SFU instruction (ex2/lg2.approx).  Generic graphs: qs fp32 log-probabilities per message
//     (qs = padded max cardinality), qs x qs max-scaled linear tables.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace bpb {

constexpr int kBlock = 256;

struct DevGraph {
  uint32_t V, E, D;
  uint32_t qs;                            // floats per message (1 = binary log-odds)
  const uint32_t* __restrict__ in_off;    // V+1
  const uint32_t* __restrict__ in_adj;    // D
  const uint32_t* __restrict__ ep;        // 2E (lo, hi)
  // binary
  const float* __restrict__ unary_lo;     // V: log psi(1) - log psi(0)
  const float4* __restrict__ epar;        // E: (alpha, beta, g-alpha, g-beta), see graph.cu
  // generic
  const uint32_t* __restrict__ card;      // V
  const float* __restrict__ unary_log;    // V*qs
  const float* __restrict__ table;        // E*qs*qs, row = lo state, max-scaled linear
  const uint32_t* __restrict__ bel_off;   // V+1 belief offsets (generic)
  // Structured fast paths (uniform-branch flags, no extra template axes):
  //   lattice topology: rows x cols row-major grid with the generator's edge
  //   order (generators.cpp:37-43) -> incoming edges by arithmetic, no CSR reads;
  //   par_mode 1: binary Ising tables {a, d, d, a} -> one weight a/d per edge
  //   (ising_a), generic Potts tables (a on the diagonal, d off it) -> one
  //   w1 = a/d - 1 per edge (pw).  0: float4 epar / dense q x q tables.
  uint32_t lat_rows, lat_cols;
  uint32_t par_mode;
  uint32_t uniform_q;                     // all cardinalities equal (0 = mixed)
  uint32_t cnt_row0, cnt_row1;            // lattice rows whose messages are owned (row-band partition)
  unsigned long long edge_offset;         // global id of local edge 0 (band: RnBP draws use global ids)
  const float* __restrict__ ising_a;      // E  (binary, par_mode 1): a = e^J of the table {a, 1/a, 1/a, a}
  const float* __restrict__ pw;           // E  (generic, par_mode 1)
  // 1: `table` holds log2 t (unscaled) and messages are contracted in the log
  // domain (models whose messages can collapse in the reference, graph.cu)
  uint32_t log_tables;
  // vertex-range partition (bp_graph_create_part): local vertices [0, own_v)
  // are owned (the rest are ghosts, never updated); egid maps a local edge to
  // its global id (RnBP draws use global ids).  own_v = UINT32_MAX, egid =
  // nullptr: no such partition.
  uint32_t own_v;
  const uint32_t* __restrict__ egid;
};

// global id of local edge e (partitions draw with global ids)
__device__ __forceinline__ unsigned long long global_edge(const DevGraph& g, uint32_t e) {
  return g.egid ? static_cast<unsigned long long>(g.egid[e]) : e + g.edge_offset;
}
__device__ __forceinline__ unsigned long long global_directed(const DevGraph& g, uint32_t d) {
  return 2ull * global_edge(g, d >> 1) + (d & 1u);
}

// numeric_error parity (normalize_in_place, messages.cpp:41-49): the reference
// throws when a message's unnormalised mass falls below 1e-300.
constexpr float kLog2MinMass = -996.578428f;  // log2(1e-300)

constexpr uint32_t kUncl = 0xFFFFFFFFu;
constexpr uint32_t kRsMaxDepth = 8;

// Non-backtracking walks of length <= h from r (covers every vertex within
// distance h, some more than once).  f(w) returning false stops the walk.
template <class F>
__device__ __forceinline__ bool ball_walk(const DevGraph& g, uint32_t r, uint32_t h, F&& f) {
  if (!f(r)) return false;
  if (h == 0) return true;
  uint32_t vs[kRsMaxDepth], par[kRsMaxDepth], pos[kRsMaxDepth], end[kRsMaxDepth];
  int d = 0;
  vs[0] = r;
  par[0] = kUncl;
  pos[0] = g.in_off[r];
  end[0] = g.in_off[r + 1];
  while (d >= 0) {
    if (pos[d] < end[d]) {
      const uint32_t w = g.ep[g.in_adj[pos[d]++]];  // source of an incoming edge = neighbour
      if (w == par[d]) continue;
      if (!f(w)) return false;
      if (d + 1 < static_cast<int>(h)) {
        ++d;
        vs[d] = w;
        par[d] = vs[d - 1];
        pos[d] = g.in_off[w];
        end[d] = g.in_off[w + 1];
      }
    } else {
      --d;
    }
  }
  return true;
}

// Row-band partition: does the band own directed edge d (its source row)?
__device__ __forceinline__ bool band_graph(const DevGraph& g) {
  return g.lat_cols != 0u && (g.cnt_row0 > 0u || g.cnt_row1 < g.lat_rows);
}
__device__ __forceinline__ bool edge_owned(const DevGraph& g, uint32_t d) {
  const uint32_t r = g.ep[d] / g.lat_cols;
  return r >= g.cnt_row0 && r < g.cnt_row1;
}

// Incoming directed edges of v in CSR order (mrf.cpp:93-104).  Lattice: up,
// left, right, down, from the edge numbering of generate_ising
// (generators.cpp:37-43): per row the right edge then the down edge of each
// vertex; the last row has right edges only.
// target vertex of directed edge d in generate_ising's lattice numbering
// (generators.cpp:37-43): rows r < R-1 hold (right, down) per column and a
// last down edge, the last row only right edges; d = 2e runs lo -> hi.
__device__ __forceinline__ uint32_t lattice_edge_target(const DevGraph& g, uint32_t d) {
  const uint32_t C = g.lat_cols, R = g.lat_rows, W = 2u * C - 1u, e = d >> 1;
  uint32_t r, c, down;
  if (e < (R - 1u) * W) {
    r = e / W;
    const uint32_t o = e - r * W;
    c = o < 2u * (C - 1u) ? o >> 1 : C - 1u;
    down = o < 2u * (C - 1u) ? (o & 1u) : 1u;
  } else {
    r = R - 1u;
    c = e - (R - 1u) * W;
    down = 0u;
  }
  const uint32_t lo = r * C + c, hi = down ? lo + C : lo + 1u;
  return (d & 1u) ? lo : hi;
}

template <class F>
__device__ __forceinline__ void for_each_in(const DevGraph& g, uint32_t v, F&& f) {
  if (g.lat_cols) {
    const uint32_t C = g.lat_cols, R = g.lat_rows;
    const uint32_t r = v / C, c = v - r * C;
    const uint32_t row = r * (2u * C - 1u);
    const bool last = r + 1u == R;
    if (r > 0u) f(2u * ((r - 1u) * (2u * C - 1u) + 2u * c + (c + 1u < C ? 1u : 0u)));
    if (c > 0u) f(2u * (last ? row + c - 1u : row + 2u * (c - 1u)));
    if (c + 1u < C) f(2u * (last ? row + c : row + 2u * c) + 1u);
    if (!last) f(2u * (row + 2u * c + (c + 1u < C ? 1u : 0u)) + 1u);
  } else {
    const uint32_t b = g.in_off[v], e = g.in_off[v + 1];
    for (uint32_t a = b; a < e; ++a) f(g.in_adj[a]);
  }
}

// Per-run control block in device memory.  Written only by single threads
// (finalizers) or by atomics; read by every kernel at entry.
struct TraceRec {
  unsigned long long iteration;
  unsigned long long frontier_size;
  unsigned int unconverged;
  unsigned int pad;
  double elapsed_seconds;
};

constexpr unsigned kTraceRing = 16384;  // 512 KB: a 10^4-iteration run drains twice

enum StopReason : unsigned { kStopNone = 0, kStopConverged = 1, kStopMaxIter = 2, kStopTime = 3, kStopNumeric = 4 };

// Per-block contributions are accumulated into kSlots cache-line-separated
// slots (block b adds into slot b % kSlots) so no single address sees more
// than gridDim/kSlots atomics; a one-block finalize kernel reduces them.
constexpr int kSlots = 128;
struct alignas(128) Accum {
  long long delta;                // unconverged-count change
  unsigned long long count;       // r >= eps count (LBP sweep / init)
  unsigned long long frontier;    // committed edges
  unsigned long long survivors;   // r >= eps seen by the RnBP filter
  unsigned long long evals;       // messages recomputed
  unsigned long long visits;      // vertices updated
};

struct Ctl {
  unsigned int done;
  unsigned int converged;
  unsigned int numeric_error;
  unsigned int has_prev;
  unsigned int unconverged;
  unsigned int prev_unconverged;
  unsigned int nflag;         // vertices queued in vlist this iteration (sparse mode)
  unsigned int dense;         // this iteration flags vertices without a list
  unsigned long long iteration;
  unsigned long long sweeps;  // LBP sweeps completed
  unsigned long long max_iterations;
  unsigned long long msgs_total;
  unsigned long long evals_total;
  unsigned long long vertex_visits;
  unsigned long long t0_ns;
  unsigned long long time_limit_ns;
  unsigned long long frontier;    // reduced by the retry kernel (RnBP)
  unsigned long long survivors;
  // radix select (RBP top-k): prefix of the k-th key found so far, and how
  // many keys are strictly above it
  unsigned int rx_prefix;
  unsigned int rx_need;
  unsigned long long rx_above;
  unsigned long long rx_ties;
  unsigned int stamp;         // vflag generation
  unsigned int splashes;
  unsigned long long splash_edges;
  unsigned int rs_rounds;     // splash claiming rounds (all iterations)
  unsigned int rs_passes;     // candidate-prefix passes (all iterations)
  unsigned long long trace_len;
  unsigned long long cond_handle;  // cudaGraphConditionalHandle of the WHILE loop (0 = none)
  unsigned int stop_reason;
  unsigned int cl_cur;        // candidate list (RnBP): current buffer
  unsigned int cl_n[2];       // candidate list sizes
  unsigned int use_clist;
  unsigned int cl_state;      // 0 scan residuals, 1 build the list this iteration, 2 walk the list
  unsigned int persist_ok;    // RnBP: hand list mode over to the persistent kernel (graph loop exits)
  unsigned int rx_n;          // RBP top-k: entries of the compacted candidate list (k_rx_compact)
  // persistent kernel: per-iteration sums (delta, count, frontier, survivors,
  // evals, visits), triple-buffered by iteration; the time-limit verdict of
  // the bookkeeping thread
  unsigned long long pacc3[3][6];
  unsigned long long handover_it;  // iteration at which the graph loop handed over to the persistent kernel
  unsigned int time_stop;
  unsigned int blocks_done;  // last-block-done counter of the kernel-fused finalize / retry (reset by the last block)
  unsigned int fused_par;    // fused RnBP sweep (kernels_fused.cuh): the state lives in the scratch set when odd
  unsigned int fused_abort;  // fused RnBP sweep: an empty attempt-0 frontier, the per-kernel loop redoes the iteration
  unsigned int band_poll;    // band RnBP driven by a polling host (partition.cu): an empty attempt-0 frontier waits
  unsigned int band_wait;    // ... for the host's retry: every kernel is a no-op until the host clears it
  unsigned long long persist_bytes;  // algorithmic bytes moved by the persistent kernel
  unsigned long long vote_limit_ns;  // row-band partition: time limit, decided by an all-reduced vote
  unsigned long long phase_ns[8];    // persistent kernel phase clock (CTA 0)
  Accum acc[kSlots];
  TraceRec trace[kTraceRing];
};

// Halo buffers of a row-band partition (device pointers owned by the caller;
// kernels.cuh: k_part_pack / k_part_count / k_part_unpack).
struct PartHalo {
  float* send_up;             // C: up messages of the first owned row (to the band above)
  float* send_down;           // C: down messages of the last owned row (to the band below)
  const float* recv_up;       // C: the band above's send_down
  const float* recv_down;     // C: the band below's send_up
  unsigned long long* count;  // LBP: [0] unconverged count, [1] time vote.  RnBP: [0] delta, [1] frontier,
                              // [2] survivors, [3] time vote, [4] init count.  All-reduced (sum) in place
  uint32_t ghost_up, ghost_down;
};

// ---------------------------------------------------------------------------
// numerics.  Raw SFU instructions (one SASS op each; __expf/__logf/__fdividef
// add denormal guards that cost 4-6 extra instructions per call).  ftz: the
// operands here never need denormals (2^-126 is far below any message scale).

__device__ __forceinline__ float fex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float flg2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float frcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// log2(1 + 2^x) = max(x, 0) + log2(1 + 2^-|x|)
__device__ __forceinline__ float softplus2(float x) { return fmaxf(x, 0.f) + flg2(1.f + fex2(-fabsf(x))); }

// probability of state 1 of a base-2 log-odds message
__device__ __forceinline__ float sigmoid2(float x) { return frcp(1.f + fex2(-x)); }

// Binary sum-product update (Eq. 2, messages.hpp:114-151) in log2-odds form:
// with cavity log2-odds h of the source and the 2x2 table A oriented source x
// target, out = log2(A01 + A11 2^h) - log2(A00 + A10 2^h)
//             = c + softplus2(h + a) - softplus2(h + b).
// par = (alpha, beta, g - alpha, g - beta) with alpha = lT01 - lT00,
// beta = lT10 - lT00, g = lT11 - lT00 (log2 of the table, row = lo state).
// Even d (lo -> hi): c = alpha, a = g - alpha, b = beta.  Odd d: c = beta,
// a = g - beta, b = alpha.
__device__ __forceinline__ float binary_update(float h, float4 par, bool odd) {
  const float c = odd ? par.y : par.x;
  const float a = odd ? par.w : par.z;
  const float b = odd ? par.x : par.y;
  return c + softplus2(h + a) - softplus2(h + b);
}

// L-inf residual in linear probability space (messages.cpp:56-65): for binary
// messages |m'(1) - m(1)| = |m'(0) - m(0)|.
__device__ __forceinline__ float binary_residual(float lnew, float lold) {
  return fabsf(sigmoid2(lnew) - sigmoid2(lold));
}

// Ising message (table {a, 1, 1, a} up to scale, a = e^J): with u = 2^h the
// outgoing odds are X = (1 + u a) / (a + u); evaluated through
// v = 2^-|h| <= 1 so nothing overflows.
struct IsingOut {
  float l;  // log2-odds log2 X
};
__device__ __forceinline__ IsingOut ising_msg(float h, float a) {
  const float v = fex2(-fabsf(h));
  float num, den;
  if (h >= 0.f) {
    num = v + a;
    den = fmaf(a, v, 1.f);
  } else {
    num = fmaf(v, a, 1.f);
    den = a + v;
  }
  IsingOut o;
  o.l = flg2(num * frcp(den));
  return o;
}

// Ising message + its L-inf residual in one pass (5 SFU ops: ex2, rcp, lg2 for
// the message, ex2, rcp for the residual).  With X = num/den the new odds and
// Y = 2^{l_old} the old ones, |sigma(l_new) - sigma(l_old)| =
// |num - Y den| / ((num + den)(1 + Y)); for l_old >= 0 the mirrored form
// (sigma(-x) = 1 - sigma(x)) keeps Y = 2^-|l_old| <= 1 so nothing overflows.
// A bitwise fixed point (l_new == l_old) reports exactly 0, so tree exactness
// at epsilon 1e-8 holds (test_schedulers.cpp:418-434).
__device__ __forceinline__ float ising_update(float h, float a, float l_old, float& l_new) {
  const float v = fex2(-fabsf(h));
  const bool pos = h >= 0.f;
  const float num = pos ? v + a : fmaf(v, a, 1.f);
  const float den = pos ? fmaf(a, v, 1.f) : a + v;
  l_new = flg2(num * frcp(den));
  const bool po = l_old >= 0.f;
  const float Y = fex2(-fabsf(l_old));
  const float nn = po ? den : num, dd = po ? num : den;
  const float r = fabsf(fmaf(-Y, dd, nn)) * frcp((num + den) * (1.f + Y));
  return l_new == l_old ? 0.f : r;
}

// Outgoing binary message on directed edge `out` from the cavity log-odds h.
__device__ __forceinline__ float binary_msg(const DevGraph& g, float h, uint32_t out) {
  if (g.par_mode) return ising_msg(h, __ldg(&g.ising_a[out >> 1])).l;
  return binary_update(h, __ldg(&g.epar[out >> 1]), (out & 1u) != 0u);
}

// Unnormalised outgoing q-vector on `out` from the source distribution p
// (p[x] = 0 for x >= |A_src|): the contraction of messages.hpp:134-149, row
// orientation by out & 1.  Potts tables contract in O(q): o = S + w1 p.
template <int QS>
__device__ __forceinline__ void generic_matvec(const DevGraph& g, uint32_t out, const float* p, float* o) {
  if (g.par_mode) {
    const float w1 = __ldg(&g.pw[out >> 1]);
    float S = 0.f;
#pragma unroll (QS <= 8 ? QS : 2)
    for (int x = 0; x < QS; ++x) S += p[x];
#pragma unroll (QS <= 8 ? QS : 2)
    for (int x = 0; x < QS; ++x) o[x] = fmaf(w1, p[x], S);
    return;
  }
  const float* tab = g.table + static_cast<size_t>(out >> 1) * QS * QS;
  if ((out & 1u) == 0u) {  // source is lo: A(xs, xt) = T[xs][xt]
#pragma unroll (QS <= 8 ? QS : 2)
    for (int xt = 0; xt < QS; ++xt) o[xt] = 0.f;
#pragma unroll (QS <= 8 ? QS : 2)
    for (int xs = 0; xs < QS; ++xs) {
#pragma unroll (QS <= 8 ? QS : 2)
      for (int xt = 0; xt < QS; ++xt) o[xt] = fmaf(__ldg(&tab[xs * QS + xt]), p[xs], o[xt]);
    }
  } else {  // source is hi: A(xs, xt) = T[xt][xs]
#pragma unroll (QS <= 8 ? QS : 2)
    for (int xt = 0; xt < QS; ++xt) {
      float acc = 0.f;
#pragma unroll (QS <= 8 ? QS : 2)
      for (int xs = 0; xs < QS; ++xs) acc = fmaf(__ldg(&tab[xt * QS + xs]), p[xs], acc);
      o[xt] = acc;
    }
  }
}

// Log-domain update for collapse-checked models (log_tables): p = log2 of the
// product psi_i * prod m (unshifted, messages.hpp:123-131), the contraction
// with the table is a log-sum-exp per target state, lo = the normalised log2
// message; returns log2 of the reference's unnormalised mass, so the caller
// can raise numeric_error exactly where normalize_in_place would.  No value
// is formed in linear fp32, so nothing under- or overflows.
template <int QS>
__device__ __forceinline__ float generic_logmatvec(const DevGraph& g, uint32_t out, const float* p, uint32_t ci,
                                                   uint32_t cj, float* lo) {
  const float* lt = g.table + static_cast<size_t>(out >> 1) * QS * QS;
  float Mt = -INFINITY;
  for (int xt = 0; xt < QS; ++xt) {
    if (xt >= static_cast<int>(cj)) {
      lo[xt] = -INFINITY;
      continue;
    }
    float m = -INFINITY;
    for (int xs = 0; xs < static_cast<int>(ci); ++xs)
      m = fmaxf(m, p[xs] + __ldg(&lt[(out & 1u) ? xt * QS + xs : xs * QS + xt]));
    float s = 0.f;
    for (int xs = 0; xs < static_cast<int>(ci); ++xs)
      s += fex2(p[xs] + __ldg(&lt[(out & 1u) ? xt * QS + xs : xs * QS + xt]) - m);
    lo[xt] = m + flg2(s);
    Mt = fmaxf(Mt, lo[xt]);
  }
  float S = 0.f;
  for (int xt = 0; xt < static_cast<int>(cj); ++xt) S += fex2(lo[xt] - Mt);
  const float tot = Mt + flg2(S);
  for (int xt = 0; xt < static_cast<int>(cj); ++xt) lo[xt] -= tot;
  return tot;
}

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11), counter-based: the RnBP Bernoulli draw
// for edge d in (iteration, attempt) is a pure function of (seed, iteration,
// attempt, d), independent of launch shape and GPU count.

__device__ __forceinline__ uint4 philox4x32_10(uint4 ctr, uint2 key) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(M0, ctr.x), lo0 = M0 * ctr.x;
    const uint32_t hi1 = __umulhi(M1, ctr.z), lo1 = M1 * ctr.z;
    ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
    if (r < 9) {  // key schedule between rounds (Random123 philox4x32_R)
      key.x += W0;
      key.y += W1;
    }
  }
  return ctr;
}

// One Philox block serves the two directions of undirected edge e = d >> 1:
// 64 bits each, the top 53 give u = value * 2^-53 in [0, 1) like
// uniform_unit (rng.hpp:11-13).  Counter = (e, iteration, attempt), key = seed.
__device__ __forceinline__ uint4 philox_edge(unsigned long long seed, unsigned long long iteration,
                                             unsigned attempt, unsigned long long e) {
  const uint4 ctr = make_uint4(static_cast<uint32_t>(e), static_cast<uint32_t>(e >> 32),
                               static_cast<uint32_t>(iteration),
                               (static_cast<uint32_t>(iteration >> 32) & 0x3FFFFFFFu) | (attempt << 30));
  const uint2 key = make_uint2(static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
  return philox4x32_10(ctr, key);
}
__device__ __forceinline__ unsigned long long u53_of(const uint4& r, unsigned long long d) {
  return (d & 1ull) ? (((static_cast<unsigned long long>(r.z) << 32) | r.w) >> 11)
                    : (((static_cast<unsigned long long>(r.x) << 32) | r.y) >> 11);
}
__device__ __forceinline__ unsigned long long philox_u53(unsigned long long seed,
                                                         unsigned long long iteration,
                                                         unsigned attempt, unsigned long long d) {
  return u53_of(philox_edge(seed, iteration, attempt, d >> 1), d);
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// warp-aggregated append of x (pred) to list[*counter]
__device__ __forceinline__ void warp_append(bool pred, uint32_t x, uint32_t* list, unsigned* counter) {
  const unsigned lane = threadIdx.x & 31u;
  const unsigned mask = __ballot_sync(0xffffffffu, pred);
  if (!mask) return;
  const unsigned leader = __ffs(mask) - 1;
  unsigned base = 0;
  if (lane == leader) base = atomicAdd(counter, __popc(mask));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (pred) list[base + __popc(mask & ((1u << lane) - 1u))] = x;
}

// ---------------------------------------------------------------------------
// block reductions

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum over the block; valid in thread 0.  `sh` must hold blockDim/32 entries.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  T r = 0;
  if (wid == 0) {
    r = lane < static_cast<int>(blockDim.x >> 5) ? sh[lane] : T(0);
    r = warp_sum(r);
  }
  return r;
}

}  // namespace bpb
