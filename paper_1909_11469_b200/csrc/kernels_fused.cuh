// RnBP dense iteration on binary Ising lattices as ONE sweep: rnbp_frontier's
// attempt 0 (filter r >= eps, Bernoulli(p_now) with the Philox draw keyed by
// (seed, iteration, 0, edge)), apply_frontier's commit and the refresh of the
// touched vertices (schedulers.cpp:194-216, 226-251; residuals.cpp:26-59),
// fused.
//
// Every decision an iteration makes about a directed edge d is a function of
// d's own state (r, candidate, Philox draw), so the thread of vertex v can
// restate, for each of its four edge pairs, whether the incoming edge and the
// outgoing edge are committed this iteration without waiting for anybody:
//   m_in'  = committed(in)  ? cand(in)  : live(in)     (v is touched iff any)
//   live'(out) = committed(out) ? cand(out) : live(out),  r(out) -> 0 if committed
// and then, when v is touched, recompute every outgoing candidate from the
// post-commit messages (the cavity sum in the refresh's order), exactly as
// k_rnbp_select + k_vertex_update<Delta> do in two launches with a touched-set
// round trip in between.  Candidates and unconverged predicates are read from
// one buffer set and written to the other (ping-pong: a neighbour's refresh
// never races with this vertex's reads); live messages are updated in place --
// a live message changes only when its edge is committed, and then its target
// reads the candidate instead, so every other write stores the value already
// there.  ctl->fused_par says which set holds the candidates / predicates;
// k_fused_exit copies them back to the canonical set when the fused phase
// ends on an odd count.
//
// Used while the run scans residuals (cl_state == 0, i.e. at least 1/16 of
// the edges unconverged: the touched set covers most vertices).  An empty
// attempt-0 frontier (survivors but no draw below p) changes nothing here;
// the finalize then raises fused_abort and the per-kernel loop redoes the
// iteration with the retry / single-survivor fallback (:204-214).
#pragma once

#include <cooperative_groups.h>

#include "kernels.cuh"

namespace bpb {

namespace cgp_fused = cooperative_groups;

// The per-edge state the sweep carries: live and candidate messages (float2
// per edge pair, both directions) and the unconverged predicate r >= eps as
// one byte per directed edge (uchar2 per pair).  The RnBP schedule reads a
// residual only through that predicate (filter 1 and the unconverged count,
// schedulers.cpp:196-203, 304, 326), so the predicate is an exact state of
// the run; the residual VALUES are rematerialised as 1 / 0 when the phase
// ends (k_fused_exit) -- the later kernels compare them with eps only.
struct FusedPair {
  float2 l, c;   // live, candidate of directions (2e, 2e + 1)
  uint32_t u;    // bit 0: r(2e) >= eps, bit 1: r(2e + 1) >= eps
  float a;       // Ising coupling a = e^J
  uint32_t sel;  // bit 0 / 1: direction committed this iteration
};

// Philox4x32-10 (philox4x32_10, bp_device.cuh) with the round keys of the
// (uniform) seed computed once per launch instead of once per draw.
struct PhiloxKeys {
  uint32_t k0[10], k1[10];
  __device__ __forceinline__ explicit PhiloxKeys(unsigned long long seed) {
    uint32_t x = static_cast<uint32_t>(seed), y = static_cast<uint32_t>(seed >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      k0[r] = x;
      k1[r] = y;
      x += 0x9E3779B9u;
      y += 0xBB67AE85u;
    }
  }
  __device__ __forceinline__ uint4 edge(unsigned long long it, unsigned long long e) const {  // = philox_edge(.., 0, e)
    uint4 ctr = make_uint4(static_cast<uint32_t>(e), static_cast<uint32_t>(e >> 32), static_cast<uint32_t>(it),
                           static_cast<uint32_t>(it >> 32) & 0x3FFFFFFFu);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      const uint32_t hi0 = __umulhi(0xD2511F53u, ctr.x), lo0 = 0xD2511F53u * ctr.x;
      const uint32_t hi1 = __umulhi(0xCD9E8D57u, ctr.z), lo1 = 0xCD9E8D57u * ctr.z;
      ctr = make_uint4(hi1 ^ ctr.y ^ k0[r], lo1, hi0 ^ ctr.w ^ k1[r], lo0);
    }
    return ctr;
  }
};

// the draws of one edge pair (one Philox block serves both directions):
// committed = unconverged && u53 < thresh (attempt 0, global edge id), with
// u53 = X >> 11 of the 64-bit word X: u53 < thresh <=> X < thresh << 11
// (thresh < 2^53 whenever draw is set, so the shifted bound fits), one
// 64-bit compare per direction instead of a 64-bit shift and compare
__device__ __forceinline__ uint32_t pair_select(uint32_t u, unsigned long long e, bool draw, const PhiloxKeys& pk,
                                                unsigned long long it, unsigned long long thresh) {
  if (!draw) return u;
  const uint4 ph = pk.edge(it, e);
  const unsigned long long bound = thresh << 11;
  uint32_t s = 0u;
  if ((u & 1u) && ((static_cast<unsigned long long>(ph.x) << 32) | ph.y) < bound) s |= 1u;
  if ((u & 2u) && ((static_cast<unsigned long long>(ph.z) << 32) | ph.w) < bound) s |= 2u;
  return s;
}

// NC: candidates / predicates through the read-only path (one launch per
// sweep); the persistent variant rereads buffers other CTAs rewrote, so it
// loads them coherently (behind the barrier's L1 invalidation)
template <bool NC = true>
__device__ __forceinline__ FusedPair load_pair(const float2* L, const float2* __restrict__ Cn,
                                               const uint16_t* __restrict__ U, const float* __restrict__ ea,
                                               uint32_t e) {
  FusedPair p;
  p.l = L[e];  // coherent: the live set is updated in place
  p.c = NC ? __ldg(&Cn[e]) : Cn[e];
  const uint32_t u = NC ? __ldg(&U[e]) : U[e];  // bytes are 0 / 1
  p.u = (u & 1u) | ((u >> 7) & 2u);
  p.a = __ldg(&ea[e]);
  p.sel = 0u;
  return p;
}

__device__ __forceinline__ FusedPair shfl_up_pair(const FusedPair& p) {
  FusedPair q;
  q.l.x = __shfl_up_sync(0xffffffffu, p.l.x, 1);
  q.l.y = __shfl_up_sync(0xffffffffu, p.l.y, 1);
  q.c.x = __shfl_up_sync(0xffffffffu, p.c.x, 1);
  q.c.y = __shfl_up_sync(0xffffffffu, p.c.y, 1);
  const uint32_t us = __shfl_up_sync(0xffffffffu, p.u | (p.sel << 2), 1);  // both 2-bit fields in one shuffle
  q.u = us & 3u;
  q.sel = us >> 2;
  q.a = __shfl_up_sync(0xffffffffu, p.a, 1);
  return q;
}

// columns per warp strip: lane 0 of every warp is a halo lane that only
// loads and draws the right pair of the column left of the warp's first one
// (so every lane's left pair arrives by shuffle and the draw costs no extra
// warp instruction)
constexpr uint32_t kFusedWarpCols = 31;
constexpr uint32_t kFusedStrip = (kBlock / 32) * kFusedWarpCols;  // block-wide strip

// Tiles per warp (31-column strips) instead of per block (248-column strips)
// when the block strips would leave a ragged end: a block walking the last
// strip with most warps past the edge holds an SM slot for little work (20%
// of the grid at 1000^2).  Block strips where they divide the lattice
// evenly: their 8 warps read adjacent columns of one row, which keeps the
// DRAM pages and partially used sectors shared (16384^2: 13% faster).
__host__ __device__ inline bool fused_warp_tiles(uint32_t C) {
  const uint32_t nb = (C + kFusedStrip - 1) / kFusedStrip;
  return 20u * (nb * kFusedStrip - C) > nb * kFusedStrip;  // > 5% of the block strips' lanes idle
}

// dir: the parity this launch serves (0: canonical -> scratch, 1: back); a
// launch of the wrong parity is a no-op (the loop body holds both).
//
// Lanes = columns, block (or warp, fused_warp_tiles) = a contiguous run of
// (strip, row) tiles walked down the strip.  Every edge pair is loaded and drawn once: a vertex owns its
// right and down pairs; its left pair comes from lane - 1 (shuffle), its up
// pair is the down pair the same thread held one row ago (carried in
// registers; loaded at the start of the block's run).  A pair leaves as one
// float2 / uchar2 store holding both directions: right pairs with the
// neighbour lane's outgoing value (shuffle), vertical pairs one row later
// with the lower vertex's.  Pairs split between warps / blocks leave as two
// single-direction stores.
// Per-thread sums of one sweep.
struct FusedSums {
  int n_delta = 0;
  uint32_t n_surv = 0, n_front = 0, n_evals = 0, n_visits = 0;
  bool bad = false;
};

// One fused sweep over this unit's tiles (unit = warp when WT, else block;
// units = the grid's warps / blocks): the body of k_rnbp_fused and of its
// persistent variant.
template <bool WT, bool NC>
__device__ __forceinline__ void fused_sweep(const DevGraph& g, const float* L0, const float* __restrict__ C0,
                                            const uint8_t* __restrict__ U0, float* L1, float* __restrict__ C1,
                                            uint8_t* __restrict__ U1, float eps, bool draw,
                                            unsigned long long thresh, unsigned long long it,
                                            const PhiloxKeys& pk, FusedSums& sums) {
  const unsigned long long eoff = g.edge_offset;
  const uint32_t C = g.lat_cols, R = g.lat_rows;
  constexpr bool wt = WT;
  constexpr uint32_t SW = wt ? kFusedWarpCols : kFusedStrip;  // strip width
  const uint32_t nstrips = (C + SW - 1) / SW;
  const uint64_t ntiles = static_cast<uint64_t>(R) * nstrips;
  // live messages IN PLACE (L0 == L1): a directed edge's live message changes
  // only when it is committed, and then its target reads the candidate
  // instead; every other write stores the value already there
  const float2* La = reinterpret_cast<const float2*>(L0);
  const float2* __restrict__ Ca = reinterpret_cast<const float2*>(C0);
  const uint16_t* __restrict__ Ua = reinterpret_cast<const uint16_t*>(U0);
  float2* Lb = reinterpret_cast<float2*>(L1);
  float2* __restrict__ Cb = reinterpret_cast<float2*>(C1);
  uint16_t* __restrict__ Ub = reinterpret_cast<uint16_t*>(U1);
  const float* __restrict__ ea = g.ising_a;
  const uint32_t lane = threadIdx.x & 31u;
  const bool halo = lane == 0u;
  // column of this lane within a strip (the halo lane: the column before the warp's first)
  const uint32_t col_in_strip = (wt ? 0u : (threadIdx.x >> 5) * kFusedWarpCols) + lane - 1u;  // wraps for halo of warp 0
  // per-thread counts in 32 bits (a thread sees at most a few thousand tiles)
  int& n_delta = sums.n_delta;
  uint32_t &n_surv = sums.n_surv, &n_front = sums.n_front, &n_evals = sums.n_evals, &n_visits = sums.n_visits;
  bool& bad = sums.bad;
  // carried from the row above (same column): its down pair (old state +
  // draws) and the upper vertex's new outgoing message on it
  FusedPair dprev{};
  float dl_new = 0.f, dc_new = 0.f;
  uint32_t du_new = 0u;
  // (warp tiles: any block size; block strips: kBlock threads)
  const uint64_t gw = wt ? static_cast<uint64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5) : blockIdx.x;
  const uint64_t nw = wt ? static_cast<uint64_t>(gridDim.x) * (blockDim.x / 32) : gridDim.x;
  const uint64_t t_begin = ntiles * gw / nw, t_end = ntiles * (gw + 1) / nw;
  uint32_t strip = static_cast<uint32_t>(t_begin / R), r = static_cast<uint32_t>(t_begin - static_cast<uint64_t>(strip) * R);
  for (uint64_t t = t_begin; t < t_end; ++t) {
    const uint32_t c = strip * SW + col_in_strip;  // halo of the first warp of strip 0: 0xffffffff
    const bool inb = c < C;                                  // a real column (the halo lane's included)
    if (__all_sync(0xffffffffu, !inb || (halo && c + 1u >= C))) {  // a warp past the ragged end: no vertex
      if (++r == R) {
        r = 0u;
        ++strip;
      }
      continue;
    }
    const bool act = inb && !halo;                           // this lane updates vertex (r, c)
    const bool first = r == 0u, last = r + 1u == R;
    const bool carry = t > t_begin && !first;  // the previous tile of this block was row r - 1 of this strip
    const bool more = t + 1 < t_end && !last;  // the next one is row r + 1 of this strip
    const uint32_t row = r * (2u * C - 1u);
    const uint32_t dn = c + 1u < C ? 1u : 0u;
    const bool hasR = inb && dn, hasU = act && !first, hasL = act && c > 0u, hasD = act && !last;
    const uint32_t eR = last ? row + c : row + 2u * c, eD = row + 2u * c + dn;
    FusedPair pr{}, pd{}, pu{};
    if (hasR) pr = load_pair<NC>(La, Ca, Ua, ea, eR);
    if (hasD) pd = load_pair<NC>(La, Ca, Ua, ea, eD);
    const uint32_t eU = first ? 0u : (r - 1u) * (2u * C - 1u) + 2u * c + dn;
    if (hasU) pu = carry ? dprev : load_pair<NC>(La, Ca, Ua, ea, eU);
    const float un = act ? __ldg(&g.unary_lo[r * C + c]) : 0.f;
    if (hasR) pr.sel = pair_select(pr.u, eR + eoff, draw, pk, it, thresh);
    if (hasD) pd.sel = pair_select(pd.u, eD + eoff, draw, pk, it, thresh);
    if (hasU && !carry) pu.sel = pair_select(pu.u, eU + eoff, draw, pk, it, thresh);
    const FusedPair pl = shfl_up_pair(pr);  // lane - 1's right pair is this vertex's left pair
    const uint32_t eL = last ? row + c - 1u : row + 2u * c - 2u;
    // per pair k (up, left, right, down): incoming direction is 2e for up /
    // left (v is hi), 2e + 1 for right / down (v is lo).  Branch-free: the
    // refresh is evaluated for every vertex and kept where v is touched.
    const FusedPair* P[4] = {&pu, &pl, &pr, &pd};
    const bool has[4] = {hasU, hasL, act && dn, hasD};
    float m_in[4], l_out[4], c_out[4];
    uint32_t u_new[4], was[4], s_out[4];
    uint32_t s_any = 0u;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const FusedPair& q = *P[k];
      const bool in_hi = k >= 2;
      const uint32_t bin = in_hi ? 2u : 1u, bout = in_hi ? 1u : 2u;
      const uint32_t hk = has[k] ? 1u : 0u;
      const uint32_t s_in = (q.sel & bin) ? hk : 0u;
      s_out[k] = (q.sel & bout) ? hk : 0u;
      was[k] = (q.u & bout) ? hk : 0u;
      const float l_in = in_hi ? q.l.y : q.l.x, c_in = in_hi ? q.c.y : q.c.x;
      m_in[k] = hk ? (s_in ? c_in : l_in) : 0.f;
      l_out[k] = in_hi ? q.l.x : q.l.y;
      c_out[k] = in_hi ? q.c.x : q.c.y;
      if (s_out[k]) l_out[k] = c_out[k];  // commit: live <- candidate
      s_any |= s_in;
      n_surv += was[k];
      n_front += s_out[k];
    }
    const bool touched = s_any != 0u;
    // refresh of v: the cavity sum in the refresh kernels' order
    const float T = un + m_in[0] + m_in[1] + m_in[2] + m_in[3];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float cn;
      const float rn = ising_update(T - m_in[k], P[k]->a, l_out[k], cn);
      if (touched) {
        bad |= has[k] && !(fabsf(cn) < INFINITY);
        c_out[k] = cn;
        u_new[k] = has[k] && rn >= eps ? 1u : 0u;
      } else {
        u_new[k] = was[k] & (s_out[k] ^ 1u);
      }
      n_delta += static_cast<int>(u_new[k]) - static_cast<int>(was[k]);
      n_evals += touched && has[k] ? 1u : 0u;
    }
    n_visits += touched ? 1u : 0u;
    // ---- stores: the left-out value travels to lane - 1, which holds the pair
    const float nl = __shfl_down_sync(0xffffffffu, l_out[1], 1);
    const float nc = __shfl_down_sync(0xffffffffu, c_out[1], 1);
    const uint32_t nu = __shfl_down_sync(0xffffffffu, u_new[1], 1);
    if (act && dn) {
      if (lane < 31u) {  // (my right-out, neighbour's left-out)
        Lb[eR] = make_float2(l_out[2], nl);
        Cb[eR] = make_float2(c_out[2], nc);
        Ub[eR] = static_cast<uint16_t>(u_new[2] | (nu << 8));
      } else {  // the neighbour is the next warp's first vertex
        L1[2ull * eR] = l_out[2];
        C1[2ull * eR] = c_out[2];
        U1[2ull * eR] = static_cast<uint8_t>(u_new[2]);
      }
    }
    if (hasL && lane == 1u) {  // the pair's other half comes from the previous warp / block
      L1[2ull * eL + 1] = l_out[1];
      C1[2ull * eL + 1] = c_out[1];
      U1[2ull * eL + 1] = static_cast<uint8_t>(u_new[1]);
    }
    if (hasU) {
      if (carry) {  // (upper vertex's down-out, my up-out)
        Lb[eU] = make_float2(dl_new, l_out[0]);
        Cb[eU] = make_float2(dc_new, c_out[0]);
        Ub[eU] = static_cast<uint16_t>(du_new | (u_new[0] << 8));
      } else {
        L1[2ull * eU + 1] = l_out[0];
        C1[2ull * eU + 1] = c_out[0];
        U1[2ull * eU + 1] = static_cast<uint8_t>(u_new[0]);
      }
    }
    if (hasD) {
      if (more) {  // the row below completes the pair
        dprev = pd;
        dl_new = l_out[3];
        dc_new = c_out[3];
        du_new = u_new[3];
      } else {
        L1[2ull * eD] = l_out[3];
        C1[2ull * eD] = c_out[3];
        U1[2ull * eD] = static_cast<uint8_t>(u_new[3]);
      }
    }
    if (++r == R) {
      r = 0u;
      ++strip;
    }
  }
}

__device__ __forceinline__ void fused_accumulate(Ctl* ctl, const FusedSums& s) {
  if (s.bad) ctl->numeric_error = 1u;
  Contrib acc;
  acc.delta = s.n_delta;
  acc.survivors = s.n_surv;
  acc.frontier = s.n_front;
  acc.evals = s.n_evals;
  acc.visits = s.n_visits;
  block_accumulate(ctl, acc);
}

// p_now -> Bernoulli threshold of the iteration (uniform_unit < p <=> u53 < ceil(p 2^53))
__device__ __forceinline__ unsigned long long fused_thresh(const Ctl* ctl, const RnbpParams& prm) {
  const double p = device_p_now(ctl, prm.low_p, prm.high_p, prm.thr);
  return static_cast<unsigned long long>(ceil(ldexp(p, 53)));
}

// dir: the parity this launch serves (0: canonical -> scratch, 1: back); a
// launch of the wrong parity is a no-op (the loop body holds both).  The last
// block to finish runs the loop control (finalize kFinFused).
template <bool WT>  // fused_warp_tiles(lat_cols)
static __global__ void __launch_bounds__(kBlock) k_rnbp_fused(DevGraph g, const float* L0,
                                                              const float* __restrict__ C0,
                                                              const uint8_t* __restrict__ U0, float* L1,
                                                              float* __restrict__ C1, uint8_t* __restrict__ U1,
                                                              Ctl* ctl, float eps, RnbpParams prm, unsigned dir) {
  if (run_done(ctl)) return;
  if (ctl->cl_state != 0u || ctl->fused_abort) {  // the fused phase is over: leave the loop
    if (ctl->cond_handle && blockIdx.x == 0 && threadIdx.x == 0)
      cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(ctl->cond_handle), 0u);
    return;
  }
  if (ctl->fused_par != dir) return;
  const unsigned long long thresh = fused_thresh(ctl, prm);
  const PhiloxKeys pk(prm.seed);
  FusedSums sums;
  fused_sweep<WT, true>(g, L0, C0, U0, L1, C1, U1, eps, thresh < (1ull << 53), thresh, ctl->iteration, pk, sums);
  fused_accumulate(ctl, sums);
  if (last_block_done(ctl)) finalize_block(ctl, kFinFused, g.D);
}

// The dense phase of a SMALL lattice inside one launch: sweeps back to back,
// each followed by a barrier, the loop control in CTA 0 (finalize kFinFused)
// and a second barrier -- a 16-CTA cluster (hardware barrier) or a
// cooperative grid.  One launch per 100x100 dense phase instead of one per
// sweep, whose launch gap and last-block finalize chain (~13 us at 100^2)
// were most of the iteration.  Same sweeps, same finalize: the same run.
constexpr int kFusedPersistBlock = 512;  // warp tiles, 16 warps per CTA

template <bool CLUSTER>
static __global__ void __launch_bounds__(kFusedPersistBlock) k_rnbp_fused_persist(DevGraph g, float* L, float* CA,
                                                                                  uint8_t* UA,
                                                                      float* CB, uint8_t* UB, Ctl* ctl, float eps,
                                                                      RnbpParams prm) {
  auto sync_all = [] {
    if constexpr (CLUSTER)
      cgp_fused::this_cluster().sync();
    else
      cgp_fused::this_grid().sync();
  };
  const PhiloxKeys pk(prm.seed);
  for (;;) {
    // loop state: written by CTA 0's finalize before the last barrier (whose
    // acquire invalidated L1: plain loads see it)
    if (ctl->done || ctl->cl_state != 0u || ctl->fused_abort) break;
    const bool odd = ctl->fused_par & 1u;
    const unsigned long long thresh = fused_thresh(ctl, prm);
    FusedSums sums;
    fused_sweep<true, false>(g, L, odd ? CB : CA, odd ? UB : UA, L, odd ? CA : CB, odd ? UA : UB, eps,
                           thresh < (1ull << 53), thresh, ctl->iteration, pk, sums);
    fused_accumulate(ctl, sums);
    sync_all();
    if (blockIdx.x == 0) finalize_block(ctl, kFinFused, g.D);
    sync_all();
  }
}


// Start of the fused phase: the unconverged predicate of every directed edge.
static __global__ void __launch_bounds__(kBlock) k_fused_enter(const float* __restrict__ res, uint8_t* __restrict__ U,
                                                               uint32_t D, float eps) {
  for (uint32_t d = blockIdx.x * blockDim.x + threadIdx.x; d < D; d += gridDim.x * blockDim.x)
    U[d] = res[d] >= eps ? 1u : 0u;
}

// End of the fused phase: the state back in the canonical set when the last
// sweep left it in the scratch set (odd count), and the residual array
// rematerialised from the predicate (1 = unconverged, 0 = converged) -- for
// the phases that follow; a finished run keeps only the live messages.
static __global__ void __launch_bounds__(kBlock) k_fused_exit(const Ctl* ctl, const float* __restrict__ C1,
                                                              const uint8_t* __restrict__ Ucur,
                                                              const uint8_t* __restrict__ Ualt, float* __restrict__ C0,
                                                              float* __restrict__ res, uint32_t D) {
  const bool odd = ctl->fused_par & 1u;
  if (ctl->done != 0u) return;  // a finished run needs only the live messages (always in place)
  const uint8_t* __restrict__ U = odd ? Ualt : Ucur;
  for (uint32_t d = blockIdx.x * blockDim.x + threadIdx.x; d < D; d += gridDim.x * blockDim.x) {
    if (odd) C0[d] = C1[d];
    res[d] = U[d] ? 1.f : 0.f;
  }
}

}  // namespace bpb
