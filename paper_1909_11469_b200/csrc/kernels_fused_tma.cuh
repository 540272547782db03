// The fused dense RnBP sweep (kernels_fused.cuh) with the rows staged in SMEM
// by bulk copies, as the TMA LBP sweep stages them (kernels_lbp.cuh): for
// grids far beyond L2, where the register version waits on its loads.
//
// A block walks a contiguous run of (strip, row) tiles down a kBlock-column
// strip (one column per thread).  Row r's edge pairs -- live, candidate,
// unconverged predicates, couplings -- and unaries arrive through 1-D bulk
// copies (cp.async.bulk + mbarrier complete_tx) into a 4-slot ring: the row
// above, the tile row, two rows in flight.  Per tile:
//   phase A  each thread draws its own right and down pairs (one Philox block
//            per pair, selection bits into SMEM; thread 0 also the staged
//            left pair of the strip, and the row above's down pairs when that
//            row was not processed by this block);
//   phase B  the vertex update of fused_vertex semantics (bitwise the same
//            arithmetic and summation order as k_rnbp_fused), reading the
//            four pairs and their bits from SMEM, writing the new state
//            (live, candidate, predicate of every outgoing direction) into
//            SMEM assembly rows;
//   then row r-1 is complete (row r wrote its up-outs) and leaves with bulk
//   stores; the strip-boundary halves and the rows whose other half belongs
//   to another block leave as single-direction stores.
// Every pair is read once from DRAM and written once: 40 B per edge pair +
// 4 B per vertex, as the register version.
#pragma once

#include "kernels_fused.cuh"
#include "kernels_lbp.cuh"

namespace bpb {

constexpr uint32_t kFW = kBlock;   // strip width: one column per thread
constexpr int kFE = 2 * kFW;       // edge pairs of a strip row
constexpr int kFAhead = 2;
constexpr int kFRing = 2 + kFAhead;

struct FusedSmem {
  alignas(16) float2 L[kFRing][kFE + 8];    // live pairs (+ staged left pairs + alignment slack)
  alignas(16) float2 C[kFRing][kFE + 8];    // candidate pairs
  alignas(16) uint16_t U[kFRing][kFE + 24]; // predicate pairs (byte 0: 2e, byte 1: 2e + 1)
  alignas(16) float E[kFRing][kFE + 12];    // couplings a = e^J
  alignas(16) float V[kFRing][kFW + 8];     // unaries
  alignas(16) uint8_t S[kFRing][kFE + 8];   // selection bits of the pairs (phase A)
  alignas(16) float2 BL[2][kFE + 8];        // new live pairs being assembled (row above / tile row)
  alignas(16) float2 BC[2][kFE + 8];        // new candidate pairs
  alignas(16) uint16_t BU[2][kFE + 24];     // new predicate pairs
  unsigned long long bar[kFRing];
  int aoff[kFRing], uoff[kFRing], eoff[kFRing], voff[kFRing];  // slot index of the row's first pair / vertex
};

// k of a strip row's pair e0 + k in slot arrays: L / C / S at k + aoff,
// U at k + uoff, E at k + eoff; BL / BC at k + (e0 & 1), BU at k + (e0 & 7)
static __global__ void __launch_bounds__(kBlock) k_rnbp_fused_tma(DevGraph g, const float* L0,
                                                                  const float* __restrict__ C0,
                                                                  const uint8_t* __restrict__ U0, float* L1, float* C1,
                                                                  uint8_t* U1, Ctl* ctl, float eps, RnbpParams prm,
                                                                  unsigned dir) {
  if (run_done(ctl)) return;
  if (ctl->cl_state != 0u || ctl->fused_abort) {  // the fused phase is over: leave the loop
    if (ctl->cond_handle && blockIdx.x == 0 && threadIdx.x == 0)
      cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(ctl->cond_handle), 0u);
    return;
  }
  if (ctl->fused_par != dir) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  FusedSmem& S = *reinterpret_cast<FusedSmem*>(smem_raw);
  const double p = device_p_now(ctl, prm.low_p, prm.high_p, prm.thr);
  const unsigned long long thresh = static_cast<unsigned long long>(ceil(ldexp(p, 53)));
  const bool draw = thresh < (1ull << 53);
  const unsigned long long it = ctl->iteration, eoffs = g.edge_offset;
  const PhiloxKeys pk(prm.seed);
  const float2* La = reinterpret_cast<const float2*>(L0);  // == L1: live messages in place (k_rnbp_fused)
  const float2* __restrict__ Ca = reinterpret_cast<const float2*>(C0);
  const uint16_t* __restrict__ Ua = reinterpret_cast<const uint16_t*>(U0);
  float2* Lb = reinterpret_cast<float2*>(L1);
  float2* Cb = reinterpret_cast<float2*>(C1);
  uint16_t* Ub = reinterpret_cast<uint16_t*>(U1);
  const float* __restrict__ ea = g.ising_a;
  const uint32_t C = g.lat_cols, R = g.lat_rows;
  const uint32_t nstrip = (C + kFW - 1) / kFW;
  const uint64_t ntiles = static_cast<uint64_t>(R) * nstrip;
  const uint64_t t_begin = ntiles * blockIdx.x / gridDim.x, t_end = ntiles * (blockIdx.x + 1) / gridDim.x;
  int n_delta = 0;
  uint32_t n_surv = 0, n_front = 0, n_evals = 0, n_visits = 0;
  bool bad = false;
  if (t_begin < t_end) {
    const bool leader = threadIdx.x == kBlock - 32;
    if (leader) {
      for (int k = 0; k < kFRing; ++k) mbar_init(&S.bar[k], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t phase = 0;
    // bulk-load row r of `strip` into ring slot s
    auto issue_row = [&](int s, uint32_t strip, uint32_t r) {
      const uint32_t c0 = strip * kFW, w = min(kFW, C - c0);
      const bool lastrow = r + 1u == R;
      const uint32_t e0 = strip_e0(r, c0, C, lastrow), ne = strip_ne(c0, w, C, lastrow);
      const uint32_t ext = c0 > 0u ? (lastrow ? 1u : 2u) : 0u;
      const uint32_t a0 = (e0 - ext) & ~1u, a1 = (e0 + ne + 1u) & ~1u;  // pairs, 16-byte granules
      const uint32_t u0 = (e0 - ext) & ~7u, u1 = (e0 + ne + 7u) & ~7u;  // predicate pairs
      const uint32_t f0 = (e0 - ext) & ~3u, f1 = (e0 + ne + 3u) & ~3u;  // couplings
      const uint32_t v0 = r * C + c0, w0 = v0 & ~3u, w1 = (v0 + w + 3u) & ~3u;
      S.aoff[s] = static_cast<int>(e0 - a0);
      S.uoff[s] = static_cast<int>(e0 - u0);
      S.eoff[s] = static_cast<int>(e0 - f0);
      S.voff[s] = static_cast<int>(v0 - w0);
      const uint32_t bytes = 16u * (a1 - a0) + 2u * (u1 - u0) + 4u * (f1 - f0) + 4u * (w1 - w0);
      mbar_expect_tx(&S.bar[s], bytes);
      bulk_g2s(&S.L[s][0], La + a0, 8u * (a1 - a0), &S.bar[s]);
      bulk_g2s(&S.C[s][0], Ca + a0, 8u * (a1 - a0), &S.bar[s]);
      bulk_g2s(&S.U[s][0], Ua + u0, 2u * (u1 - u0), &S.bar[s]);
      bulk_g2s(&S.E[s][0], ea + f0, 4u * (f1 - f0), &S.bar[s]);
      bulk_g2s(&S.V[s][0], g.unary_lo + w0, 4u * (w1 - w0), &S.bar[s]);
    };
    auto wait_slot = [&](int s) {
      mbar_wait(&S.bar[s], (phase >> s) & 1u);
      phase ^= 1u << s;
    };
    auto sel_of = [&](int s, int k, uint32_t e0) -> uint32_t {  // draws of pair e0 + k of slot s
      const uint32_t u = S.U[s][k + S.uoff[s]];
      const uint32_t bits = (u & 1u) | ((u >> 7) & 2u);
      return pair_select(bits, static_cast<unsigned long long>(e0) + k + eoffs, draw, pk, it, thresh);
    };
    // write the completed strip region of row rr from the assembly rows bb:
    // 16-byte-aligned runs by bulk store, ragged ends and single-direction
    // halves (the strip's last right pair when a next strip exists: its .y
    // is that strip's; the down pairs when the row below is another block's)
    // by scalar stores
    auto write_row = [&](int bb, uint32_t strip, uint32_t rr, bool with_dy) {
      const uint32_t c0 = strip * kFW, w = min(kFW, C - c0);
      const bool lastrow = rr + 1u == R;
      const uint32_t e0 = strip_e0(rr, c0, C, lastrow), ne = strip_ne(c0, w, C, lastrow);
      const float2* SL = S.BL[bb] + (e0 & 1u);
      const float2* SC = S.BC[bb] + (e0 & 1u);
      const uint16_t* SU = S.BU[bb] + (e0 & 7u);
      const bool has_next = c0 + w < C;
      const uint32_t k_skip = has_next ? ko_r(w - 1u, lastrow) : 0xFFFFFFFFu;
      auto half = [&](uint32_t k) {  // only the .x direction of pair e0 + k is this block's
        L1[2ull * (e0 + k)] = SL[k].x;
        C1[2ull * (e0 + k)] = SC[k].x;
        U1[2ull * (e0 + k)] = static_cast<uint8_t>(SU[k] & 0xffu);
      };
      auto whole = [&](uint32_t k) {
        Lb[e0 + k] = SL[k];
        Cb[e0 + k] = SC[k];
        Ub[e0 + k] = SU[k];
      };
      if (with_dy) {
        const uint32_t kend = has_next ? k_skip : ne;
        // float2 arrays: 16-byte runs of 2 pairs; the predicate pairs: of 8
        const uint32_t kb0 = (e0 & 1u) ? 1u : 0u;
        uint32_t kb1 = kend >= kb0 ? kb0 + ((kend - kb0) & ~1u) : kb0;
        const uint32_t ku0 = (8u - (e0 & 7u)) & 7u;
        uint32_t ku1 = kend >= ku0 ? ku0 + ((kend - ku0) & ~7u) : ku0;
        if (kb1 <= kb0) kb1 = kb0;
        if (ku1 <= ku0) ku1 = ku0;
        if (leader) {
          fence_proxy_async();
          if (kb1 > kb0) {
            bulk_s2g(Lb + e0 + kb0, SL + kb0, 8u * (kb1 - kb0));
            bulk_s2g(Cb + e0 + kb0, SC + kb0, 8u * (kb1 - kb0));
          }
          if (ku1 > ku0) bulk_s2g(Ub + e0 + ku0, SU + ku0, 2u * (ku1 - ku0));
          bulk_commit();
        }
        // ragged ends: pairs outside [kb0, kb1) for L / C, outside [ku0, ku1) for U
        for (uint32_t k = threadIdx.x; k < ne; k += kBlock) {
          const bool in_b = k >= kb0 && k < kb1, in_u = k >= ku0 && k < ku1;
          if (in_b && in_u) continue;
          if (k == k_skip) {
            half(k);
            continue;
          }
          if (!in_b) {
            Lb[e0 + k] = SL[k];
            Cb[e0 + k] = SC[k];
          }
          if (!in_u) Ub[e0 + k] = SU[k];
        }
      } else {
        for (uint32_t k = threadIdx.x; k < ne; k += kBlock) {
          const bool is_d = !lastrow && ((k & 1u) == 1u || (c0 + (k >> 1) == C - 1u));
          if (k == k_skip || is_d)
            half(k);
          else
            whole(k);
        }
      }
    };

    static_assert((kFRing & (kFRing - 1)) == 0, "power-of-two ring");
    int b_cur = 0;
    bool prev_b = false;
    uint32_t prev_strip = 0xFFFFFFFFu, prev_row = 0;
    auto step = [&](uint32_t& st, uint32_t& rr) {
      if (++rr == R) {
        rr = 0;
        ++st;
      }
    };
    uint32_t strip = static_cast<uint32_t>(t_begin / R), r = static_cast<uint32_t>(t_begin % R);
    const int base = r > 0u ? 1 : 0;
    uint32_t st_i = strip, r_i = r;
    if (leader) {  // prologue: the first tile's row above, its row and kFAhead more rows
      if (r > 0u) issue_row(0, strip, r - 1u);
      for (int k = 0; k <= kFAhead && t_begin + k < t_end; ++k) {
        issue_row((base + k) & (kFRing - 1), st_i, r_i);
        step(st_i, r_i);
      }
    }
    if (r > 0u) wait_slot(0);
    int s_cur = base;
    for (uint64_t t = t_begin; t < t_end; ++t, s_cur = (s_cur + 1) & (kFRing - 1)) {
      const int s_up = r > 0u ? (s_cur + kFRing - 1) & (kFRing - 1) : -1;
      const uint32_t c0 = strip * kFW, w = min(kFW, C - c0);
      const bool lastrow = r + 1u == R, first = r == 0u;
      const bool cont = prev_b && prev_strip == strip && prev_row + 1u == r;
      wait_slot(s_cur);
      if (!cont && prev_b) {  // strip changed: flush the previous row without its D.y
        write_row(b_cur ^ 1, prev_strip, prev_row, false);
        prev_b = false;
      }
      const uint32_t e0 = strip_e0(r, c0, C, lastrow);
      const uint32_t ext = c0 > 0u ? (lastrow ? 1u : 2u) : 0u;
      const uint32_t eu0 = first ? 0u : strip_e0(r - 1u, c0, C, false);
      const uint32_t j = threadIdx.x, c = c0 + j;
      const bool act = j < w;
      const uint32_t kr = ko_r(j, lastrow), kd = ko_d(j, c, C), kup = ko_d(j, c, C);
      const bool hu = act && !first, hl = act && c > 0u, hr = act && c + 1u < C, hd = act && !lastrow;
      // ---- phase A: selection bits of the pairs this thread owns
      if (hr) S.S[s_cur][kr + S.aoff[s_cur]] = static_cast<uint8_t>(sel_of(s_cur, static_cast<int>(kr), e0));
      if (hd) S.S[s_cur][kd + S.aoff[s_cur]] = static_cast<uint8_t>(sel_of(s_cur, static_cast<int>(kd), e0));
      if (j == 0u && ext)  // the staged left pair of the strip (the previous strip's right pair)
        S.S[s_cur][S.aoff[s_cur] - static_cast<int>(ext)] =
            static_cast<uint8_t>(sel_of(s_cur, -static_cast<int>(ext), e0));
      if (hu && !cont)  // the row above was not this block's: draw its down pairs here
        S.S[s_up][kup + S.aoff[s_up]] = static_cast<uint8_t>(sel_of(s_up, static_cast<int>(kup), eu0));
      __syncthreads();
      // ---- phase B: the vertex update (k_rnbp_fused's arithmetic and order)
      if (act) {
        const int kl = j > 0u ? static_cast<int>(ko_r(j - 1u, lastrow)) : -static_cast<int>(ext);
        const int sp[4] = {s_up, s_cur, s_cur, s_cur};
        const int kk[4] = {static_cast<int>(kup), kl, static_cast<int>(kr), static_cast<int>(kd)};
        const bool has[4] = {hu, hl, hr, hd};
        FusedPair P[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          P[k] = FusedPair{};
          if (!has[k]) continue;
          const int s = sp[k];
          P[k].l = S.L[s][kk[k] + S.aoff[s]];
          P[k].c = S.C[s][kk[k] + S.aoff[s]];
          const uint32_t u = S.U[s][kk[k] + S.uoff[s]];
          P[k].u = (u & 1u) | ((u >> 7) & 2u);
          P[k].a = S.E[s][kk[k] + S.eoff[s]];
          P[k].sel = S.S[s][kk[k] + S.aoff[s]];
        }
        const float un = S.V[s_cur][j + S.voff[s_cur]];
        float m_in[4], l_out[4], c_out[4];
        uint32_t u_new[4], was[4], s_out[4];
        uint32_t s_any = 0u;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const FusedPair& q = P[k];
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
        const float T = un + m_in[0] + m_in[1] + m_in[2] + m_in[3];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float cn;
          const float rn = ising_update(T - m_in[k], P[k].a, l_out[k], cn);
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
        // ---- outgoing state into the assembly rows (bytes of the predicate pairs)
        float2* BLc = S.BL[b_cur] + (e0 & 1u);
        float2* BCc = S.BC[b_cur] + (e0 & 1u);
        uint8_t* BUc = reinterpret_cast<uint8_t*>(S.BU[b_cur] + (e0 & 7u));
        if (hr) {  // right-out: .x of the right pair
          BLc[kr].x = l_out[2];
          BCc[kr].x = c_out[2];
          BUc[2u * kr] = static_cast<uint8_t>(u_new[2]);
        }
        if (hd) {  // down-out: .x of the down pair
          BLc[kd].x = l_out[3];
          BCc[kd].x = c_out[3];
          BUc[2u * kd] = static_cast<uint8_t>(u_new[3]);
        }
        if (hl) {  // left-out: .y of the left pair
          if (j > 0u) {
            BLc[kl].y = l_out[1];
            BCc[kl].y = c_out[1];
            BUc[2u * kl + 1u] = static_cast<uint8_t>(u_new[1]);
          } else {  // the previous strip's pair
            const uint64_t e = e0 - ext;
            L1[2ull * e + 1] = l_out[1];
            C1[2ull * e + 1] = c_out[1];
            U1[2ull * e + 1] = static_cast<uint8_t>(u_new[1]);
          }
        }
        if (hu) {  // up-out: .y of the row above's down pair
          if (cont) {
            float2* BLu = S.BL[b_cur ^ 1] + (eu0 & 1u);
            float2* BCu = S.BC[b_cur ^ 1] + (eu0 & 1u);
            uint8_t* BUu = reinterpret_cast<uint8_t*>(S.BU[b_cur ^ 1] + (eu0 & 7u));
            BLu[kup].y = l_out[0];
            BCu[kup].y = c_out[0];
            BUu[2u * kup + 1u] = static_cast<uint8_t>(u_new[0]);
          } else {
            const uint64_t e = eu0 + kup;
            L1[2ull * e + 1] = l_out[0];
            C1[2ull * e + 1] = c_out[0];
            U1[2ull * e + 1] = static_cast<uint8_t>(u_new[0]);
          }
        }
      }
      __syncthreads();
      // ---- row r-1 is complete: write its strip region
      if (cont) write_row(b_cur ^ 1, strip, r - 1u, true);
      if (leader) bulk_wait_read();
      __syncthreads();
      prev_b = true;
      prev_strip = strip;
      prev_row = r;
      b_cur ^= 1;
      if (leader && t + 1 + kFAhead < t_end) {
        issue_row((s_cur + kFRing - 1) & (kFRing - 1), st_i, r_i);
        step(st_i, r_i);
      }
      step(strip, r);
    }
    if (prev_b) write_row(b_cur ^ 1, prev_strip, prev_row, false);  // its D.y: the next block
    if (leader) bulk_wait_all();
  }
  if (bad) ctl->numeric_error = 1u;
  Contrib acc;
  acc.delta = n_delta;
  acc.survivors = n_surv;
  acc.frontier = n_front;
  acc.evals = n_evals;
  acc.visits = n_visits;
  block_accumulate(ctl, acc);
  if (last_block_done(ctl)) finalize_block(ctl, kFinFused, g.D);
}

}  // namespace bpb
