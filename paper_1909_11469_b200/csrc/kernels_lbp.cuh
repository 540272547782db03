// The LBP sweep of a binary Ising lattice, TMA-staged (sm_100a): the
// HBM-bound kernel of the path (refresh_residuals over every edge,
// residuals.cpp:26-59, fused with the Jacobi commit of apply_frontier,
// schedulers.cpp:243-245).
//
// A block walks a contiguous run of (strip, row) tiles down a kSW-column
// strip.  Row data (edge pairs = both message directions, couplings a = e^J,
// unaries) arrive in SMEM through 1-D bulk copies (cp.async.bulk, completion
// on an mbarrier) into a 3-slot ring: the row above, the tile row, and the
// prefetch of the next row -- so the upper neighbours cost no DRAM re-read
// and the next row's latency hides behind this row's arithmetic.  New
// messages are assembled in SMEM; once row r is done, row r-1's edges are
// complete (row r supplied their up messages) and leave with one bulk store.
// No thread moves data through registers except the arithmetic operands, and
// every DRAM sector is read and written once: 44 B per vertex.
#pragma once

#include "kernels.cuh"

namespace bpb {

constexpr int kSVPT = 2;                  // vertices per thread per tile
constexpr uint32_t kSW = kBlock * kSVPT;  // strip width (columns)
constexpr int kSEdges = 2 * kSW;          // edges of a strip row

// ring of row slots: the row above, the tile row, and kLbpAhead rows in flight
constexpr int kLbpAhead = 2;
constexpr int kRing = 2 + kLbpAhead;

struct LbpSmem {
  float2 A[kRing][kSEdges + 6];  // ring: message pairs (+ left neighbour pair + alignment slack)
  float E[kRing][kSEdges + 12];  // ring: couplings (+ left neighbour + alignment slack)
  float U[kRing][kSW + 8];       // ring: unaries
  float2 B[2][kSEdges + 2];  // new message pairs being assembled (row above / tile row)
  unsigned long long bar[kRing];  // mbarriers of the ring slots
  uint32_t aoff[kRing], eoff[kRing], uoff[kRing];  // alignment offsets of the ring slots
  // S.B[b] holds the pair of global edge e0 + k at index k + boff[b]: same
  // 16-byte phase as global memory, so completed rows leave by bulk store
};

// edge offsets inside a strip row (local column j, global column c)
__device__ __forceinline__ uint32_t ko_r(uint32_t j, bool lastrow) { return lastrow ? j : 2u * j; }
__device__ __forceinline__ uint32_t ko_d(uint32_t j, uint32_t c, uint32_t C) { return c + 1u < C ? 2u * j + 1u : 2u * j; }
__device__ __forceinline__ uint32_t strip_e0(uint32_t r, uint32_t c0, uint32_t C, bool lastrow) {
  return r * (2u * C - 1u) + (lastrow ? c0 : 2u * c0);
}
__device__ __forceinline__ uint32_t strip_ne(uint32_t c0, uint32_t w, uint32_t C, bool lastrow) {
  const bool lastcol = c0 + w == C;
  return lastrow ? (lastcol ? w - 1u : w) : (lastcol ? 2u * w - 1u : 2u * w);
}

// ---- PTX: mbarrier + 1-D bulk copies
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

static __global__ void __launch_bounds__(kBlock) k_lbp_lattice(DevGraph g, const float* A0, float* B0, Ctl* ctl,
                                                               float eps) {
  if (run_done(ctl)) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  LbpSmem& S = *reinterpret_cast<LbpSmem*>(smem_raw);
  const float* A = A0;
  float* B = B0;
  if (ctl->sweeps & 1ull) {  // ping-pong (run()'s fused LBP shift)
    A = B0;
    B = const_cast<float*>(A0);
  }
  const float2* __restrict__ A2 = reinterpret_cast<const float2*>(A);
  float2* B2 = reinterpret_cast<float2*>(B);
  const float* __restrict__ ea = g.ising_a;
  const uint32_t C = g.lat_cols, R = g.lat_rows;
  const uint32_t nstrip = (C + kSW - 1) / kSW;
  const uint64_t ntiles = static_cast<uint64_t>(R) * nstrip;
  const uint64_t t_begin = ntiles * blockIdx.x / gridDim.x, t_end = ntiles * (blockIdx.x + 1) / gridDim.x;
  if (t_begin >= t_end) return;
  // the bulk-copy issuer sits in the last warp: warp 0 already carries the
  // strip's first column (general path), so the two costs land on different warps
  const bool leader = threadIdx.x == kBlock - 32;
  if (leader) {
    for (int k = 0; k < kRing; ++k) mbar_init(&S.bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phase = 0;  // bit s: parity of ring slot s

  // bulk-load row r of `strip` (and its edge pairs, couplings, unaries) into ring slot s
  auto issue_row = [&](int s, uint32_t strip, uint32_t r) {
    const uint32_t c0 = strip * kSW, w = min(kSW, C - c0);
    const bool lastrow = r + 1u == R;
    const uint32_t e0 = strip_e0(r, c0, C, lastrow), ne = strip_ne(c0, w, C, lastrow);
    // one more edge on the left: the strip-boundary left edge of column c0
    // (it belongs to the previous strip), so column 0 reads it from SMEM too
    const uint32_t ext = c0 > 0u ? (lastrow ? 1u : 2u) : 0u;
    const uint32_t a0 = (e0 - ext) & ~1u, a1 = (e0 + ne + 1u) & ~1u;  // pairs, 16-byte granules
    const uint32_t f0 = (e0 - ext) & ~3u, f1 = (e0 + ne + 3u) & ~3u;  // floats
    const uint32_t v0 = r * C + c0, u0 = v0 & ~3u, u1 = (v0 + w + 3u) & ~3u;
    S.aoff[s] = e0 - a0;
    S.eoff[s] = e0 - f0;
    S.uoff[s] = v0 - u0;
    const uint32_t bytes = 8u * (a1 - a0) + 4u * (f1 - f0) + 4u * (u1 - u0);
    mbar_expect_tx(&S.bar[s], bytes);
    bulk_g2s(&S.A[s][0], A2 + a0, 8u * (a1 - a0), &S.bar[s]);
    bulk_g2s(&S.E[s][0], ea + f0, 4u * (f1 - f0), &S.bar[s]);
    bulk_g2s(&S.U[s][0], g.unary_lo + u0, 4u * (u1 - u0), &S.bar[s]);
  };
  auto wait_slot = [&](int s) {
    mbar_wait(&S.bar[s], (phase >> s) & 1u);
    phase ^= 1u << s;
  };

  // write the completed strip region of (non-last) row rr from S.B[bb]:
  // the interior with one bulk store, the ragged ends and the excluded slots
  // (R.y of the strip's last column when a next strip exists -- that strip
  // writes it; D.y when the row below belongs to another block) with scalar stores
  auto write_row = [&](int bb, uint32_t strip, uint32_t rr, bool with_dy) {
    const uint32_t c0 = strip * kSW, w = min(kSW, C - c0);
    const bool lastrow = rr + 1u == R;
    const uint32_t e0 = strip_e0(rr, c0, C, lastrow), ne = strip_ne(c0, w, C, lastrow);
    const float2* SB = S.B[bb] + (e0 & 1u);
    const bool has_next = c0 + w < C;
    const uint32_t k_skip = has_next ? ko_r(w - 1u, lastrow) : 0xFFFFFFFFu;
    if (with_dy) {
      // bulk part: pairs [kb0, kb1) with 16-byte aligned global addresses, below k_skip
      const uint32_t kend = has_next ? k_skip : ne;
      const uint32_t kb0 = (e0 & 1u) ? 1u : 0u;
      uint32_t kb1 = kend >= kb0 ? kb0 + ((kend - kb0) & ~1u) : kb0;
      if (kb1 > kb0) {
        if (leader) {
          fence_proxy_async();
          bulk_s2g(B2 + e0 + kb0, SB + kb0, 8u * (kb1 - kb0));
          bulk_commit();
        }
      } else {
        kb1 = kb0;
      }
      // ragged ends only: [0, kb0) and [kb1, ne) -- a handful of pairs
      const uint32_t nt = ne - kb1;
      for (uint32_t i = threadIdx.x; i < kb0 + nt; i += kBlock) {
        const uint32_t k = i < kb0 ? i : kb1 + (i - kb0);
        const float2 v = SB[k];
        if (k == k_skip)
          B[2u * (e0 + k)] = v.x;
        else
          B2[e0 + k] = v;
      }
    } else {
      for (uint32_t k = threadIdx.x; k < ne; k += kBlock) {
        const float2 v = SB[k];
        const bool is_d = !lastrow && ((k & 1u) == 1u || (c0 + (k >> 1) == C - 1u));
        if (k == k_skip || is_d)
          B[2u * (e0 + k)] = v.x;
        else
          B2[e0 + k] = v;
      }
    }
  };

  int cnt = 0;
  unsigned long long evals = 0, visits = 0;
  bool bad = false;
  // Ring bookkeeping is modular: rows enter the ring in consumption order, so
  // tile i of this block (i = t - t_begin) holds slot (base + i) % kRing, its
  // row above (the previous tile's row, or the prologue's row) the slot
  // before, and the row kLbpAhead + 1 tiles ahead goes into that slot once
  // the tile is done.  (A strip change restarts at row 0: no row above.)
  static_assert((kRing & (kRing - 1)) == 0, "power-of-two ring");
  int b_cur = 0;           // S.B[b_cur] receives the tile row; S.B[b_cur ^ 1] the row above
  bool prev_b = false;     // S.B[b_cur ^ 1] holds the row above's messages (to write out)
  uint32_t prev_strip = 0xFFFFFFFFu, prev_row = 0;
  auto step = [&](uint32_t& st, uint32_t& rr) {  // (strip, row) of the next tile
    if (++rr == R) {
      rr = 0;
      ++st;
    }
  };
  uint32_t strip = static_cast<uint32_t>(t_begin / R), r = static_cast<uint32_t>(t_begin % R);
  const int base = r > 0u ? 1 : 0;
  // (strip, row) of the tile whose row is issued next (leader only)
  uint32_t st_i = strip, r_i = r;
  if (leader) {  // prologue: the first tile's row above, its row and kLbpAhead more rows
    if (r > 0u) issue_row(0, strip, r - 1u);
    for (int k = 0; k <= kLbpAhead && t_begin + k < t_end; ++k) {
      issue_row((base + k) & (kRing - 1), st_i, r_i);
      step(st_i, r_i);
    }
  }
  if (r > 0u) wait_slot(0);
  int s_cur = base;
  for (uint64_t t = t_begin; t < t_end; ++t, s_cur = (s_cur + 1) & (kRing - 1)) {
    const int s_up = r > 0u ? (s_cur + kRing - 1) & (kRing - 1) : -1;
    const uint32_t c0 = strip * kSW, w = min(kSW, C - c0);
    const bool lastrow = r + 1u == R, first = r == 0u;
    const bool cont = prev_b && prev_strip == strip && prev_row + 1u == r;
    wait_slot(s_cur);
    if (!cont && prev_b) {  // strip changed: flush the previous row without its D.y
      write_row(b_cur ^ 1, prev_strip, prev_row, false);
      prev_b = false;
    }
    // ---- the sweep of the tile row
    const bool owned = r >= g.cnt_row0 && r < g.cnt_row1;
    const uint32_t e0 = strip_e0(r, c0, C, lastrow);
    const float2* Ac = S.A[s_cur] + S.aoff[s_cur];
    const float* Ec = S.E[s_cur] + S.eoff[s_cur];
    const float* Uc = S.U[s_cur] + S.uoff[s_cur];
    const float2* Au = s_up >= 0 ? S.A[s_up] + S.aoff[s_up] : nullptr;
    const float* Eu = s_up >= 0 ? S.E[s_up] + S.eoff[s_up] : nullptr;
    float2* Bc = S.B[b_cur] + (e0 & 1u);
    float2* Bu = S.B[b_cur ^ 1] + (first ? 0u : (strip_e0(r - 1u, c0, C, false) & 1u));
    // interior tiles (row above staged and its messages in SMEM, row below
    // present): the hot path reads every operand from SMEM without predicates
    const bool fast_tile = cont && !first && !lastrow;
#pragma unroll
    for (int q = 0; q < kSVPT; ++q) {
      const uint32_t j = threadIdx.x + q * kBlock;
      if (j >= w) continue;
      const uint32_t c = c0 + j;
      // (column 0 of a strip takes this path too: its left pair is staged with
      // the row; only its left message goes to the previous strip's pair in HBM)
      if (fast_tile && c > 0u && c + 1u < C) {
        const int jl = 2 * static_cast<int>(j) - 2;  // left pair: index -2 (staged) for column 0
        const float2 pR = Ac[2u * j], pD = Ac[2u * j + 1u], pL = Ac[jl], pU = Au[2u * j + 1u];
        const float aR = Ec[2u * j], aD = Ec[2u * j + 1u], aL = Ec[jl], aU = Eu[2u * j + 1u];
        const float T = Uc[j] + pU.x + pL.x + pR.y + pD.y;
        float lu, ll, lr, ld;
        const float ru = ising_update(T - pU.x, aU, pU.y, lu);
        const float rl = ising_update(T - pL.x, aL, pL.y, ll);
        const float rr = ising_update(T - pR.y, aR, pR.x, lr);
        const float rd = ising_update(T - pD.y, aD, pD.x, ld);
        Bc[2u * j].x = lr;
        Bc[2u * j + 1u].x = ld;
        if (j > 0u)
          Bc[2u * j - 2u].y = ll;
        else
          B[2u * (e0 - 2u) + 1u] = ll;
        Bu[2u * j + 1u].y = lu;
        bad |= !(fabsf(lu + ll + lr + ld) < INFINITY);
        if (owned) {
          cnt += (ru >= eps) + (rl >= eps) + (rr >= eps) + (rd >= eps);
          evals += 4u;
          ++visits;
        }
        continue;
      }
      const bool hu = !first, hl = c > 0u, hr = c + 1u < C, hd = !lastrow;
      const float2 z = make_float2(0.f, 0.f);
      const uint32_t kr = ko_r(j, lastrow), kd = ko_d(j, c, C), kup = ko_d(j, c, C);
      const float2 pR = hr ? Ac[kr] : z;
      const float aR = hr ? Ec[kr] : 1.f;
      const float2 pD = hd ? Ac[kd] : z;
      const float aD = hd ? Ec[kd] : 1.f;
      const float2 pU = hu ? Au[kup] : z;
      const float aU = hu ? Eu[kup] : 1.f;
      float2 pL = z;
      float aL = 1.f;
      if (hl) {
        if (j > 0u) {
          pL = Ac[ko_r(j - 1u, lastrow)];
          aL = Ec[ko_r(j - 1u, lastrow)];
        } else {  // strip boundary: the left edge belongs to the previous strip
          pL = Ac[-static_cast<int>(lastrow ? 1u : 2u)];  // staged with the row
          aL = Ec[-static_cast<int>(lastrow ? 1u : 2u)];
        }
      }
      const float T = Uc[j] + pU.x + pL.x + pR.y + pD.y;
      float lu, ll, lr, ld;
      const float ru = ising_update(T - pU.x, aU, pU.y, lu);
      const float rl = ising_update(T - pL.x, aL, pL.y, ll);
      const float rr = ising_update(T - pR.y, aR, pR.x, lr);
      const float rd = ising_update(T - pD.y, aD, pD.x, ld);
      if (hr) Bc[kr].x = lr;  // (r, c) -> (r, c+1): even slot of its right edge
      if (hd) Bc[kd].x = ld;  // (r, c) -> (r+1, c)
      if (hl) {               // (r, c) -> (r, c-1): odd slot of the left edge
        if (j > 0u)
          Bc[ko_r(j - 1u, lastrow)].y = ll;
        else
          B[2u * (e0 - (lastrow ? 1u : 2u)) + 1u] = ll;
      }
      if (hu) {  // (r, c) -> (r-1, c): odd slot of the upper row's down edge
        if (cont)
          Bu[kup].y = lu;
        else
          B[2u * (strip_e0(r - 1u, c0, C, false) + kup) + 1u] = lu;
      }
      bad |= (hu && !(fabsf(lu) < INFINITY)) || (hl && !(fabsf(ll) < INFINITY)) ||
             (hr && !(fabsf(lr) < INFINITY)) || (hd && !(fabsf(ld) < INFINITY));
      if (owned) {
        cnt += (hu && ru >= eps) + (hl && rl >= eps) + (hr && rr >= eps) + (hd && rd >= eps);
        evals += static_cast<unsigned>(hu) + hl + hr + hd;
        ++visits;
      }
    }
    __syncthreads();
    // ---- row r-1 is complete: write its strip region
    if (cont) write_row(b_cur ^ 1, strip, r - 1u, true);
    // the bulk store must have read S.B[b_cur ^ 1] before the next tile refills it
    if (leader) bulk_wait_read();
    __syncthreads();
    prev_b = true;
    prev_strip = strip;
    prev_row = r;
    b_cur ^= 1;
    // the row above's slot is free now: it takes the row kLbpAhead + 1 tiles ahead
    if (leader && t + 1 + kLbpAhead < t_end) {
      issue_row((s_cur + kRing - 1) & (kRing - 1), st_i, r_i);
      step(st_i, r_i);
    }
    step(strip, r);
  }
  if (prev_b) write_row(b_cur ^ 1, prev_strip, prev_row, false);  // its D.y: the next block
  if (leader) bulk_wait_all();
  if (bad) ctl->numeric_error = 1u;
  Contrib ct;
  ct.count = static_cast<unsigned long long>(cnt);
  ct.evals = evals;
  ct.visits = visits;
  block_accumulate(ctl, ct);
}

}  // namespace bpb
