// Residual Splash on the device (sm_100a).
//
// Reference (paths relative to /root/reference/proj/core/src):
//   vertex_residual        schedulers.cpp:128-134
//   build_splash           schedulers.cpp:136-167
//   rs_frontier            schedulers.cpp:169-192
//   apply_splash_frontier  schedulers.cpp:253-291 (+ SplashOverlayView :47-54)
//
// The reference walks all vertices in (vertex residual desc, id asc) order and
// greedily claims BFS balls of depth h around unclaimed roots until k splashes
// exist.  The device restates that sequential greedy EXACTLY, in parallel:
//
//   * only a prefix of the priority order can matter: the top-M vertices
//     (radix select, ties to the lower id) are the candidates; if they yield
//     fewer than k splashes the prefix is extended (M *= 4);
//   * a candidate r is "ready" once no unresolved candidate of higher priority
//     has a depth-h ball intersecting r's ball (ballmax: every candidate
//     atomicMax-es its 64-bit priority key over its ball, r is ready iff it
//     holds the max on its whole ball).  Deep splashes (h above the walk
//     stack, no ball lists) use the equivalent distance test instead: balls
//     intersect iff the roots are within 2h, so 2h max-propagation sweeps over
//     the vertex graph give each root the highest key within 2h -- any depth,
//     at O(h (V + E)) per round.  Ready roots have pairwise disjoint
//     balls, so their BFS claims run concurrently without conflicts and give
//     the claims of the sequential walk; candidates found claimed are the
//     skipped roots of the walk (their claimer always has higher priority);
//   * after all candidates resolve, the k built splashes of highest priority
//     are kept (a second radix select).  Built-but-dropped splashes have lower
//     priority than every kept one, so they never influenced a kept splash.
//
// The BFS visit order of each splash is a linked list through qnext[] (each
// vertex is claimed at most once, so no allocation is needed); spos[] holds the
// position in the visit order, which is all the Gauss-Seidel overlay needs: an
// incoming message k -> v reads the splash's own write iff k belongs to the
// same splash and was visited before v (SplashOverlayView::view).
//
// Everything from the vertex residuals to the commit of the splash messages is
// one cooperative persistent kernel with grid-wide barriers between phases;
// the touched-set refresh reuses k_vertex_update.
#pragma once

#include <cooperative_groups.h>

#include "kernels.cuh"

namespace bpb {

namespace cg = cooperative_groups;

constexpr int kRsBlock = 512;

enum RsState : uint32_t { kRsNone = 0, kRsCand = 1, kRsBuilt = 2, kRsSkip = 3, kRsKept = 4 };

struct RsCtl {
  unsigned long long k;       // splashes wanted: max(1, llround(p V))  (schedulers.cpp:172-173)
  unsigned M;                 // candidate prefix size
  unsigned ncand, nbuilt, nready, nkept, unres, rounds, passes;
  unsigned prefix, ties, need, total, all;
  unsigned long long above;
  unsigned long long edges;   // splash edges (frontier_size, schedulers.cpp:335)
  unsigned dense;
  unsigned pad_;
};

struct RsBufs {
  float* vres;
  uint32_t* state;
  uint32_t* claimed;
  uint32_t* qnext;
  uint32_t* spos;
  uint32_t* depth;
  unsigned long long* ballmax;
  unsigned long long* ballmax2;    // V more: the propagation ping-pong (deep splashes)
  uint32_t* clist;
  uint32_t* blist;
  uint32_t* rlist;
  uint32_t* klist;
  unsigned* hist;   // 4096
  unsigned* blk;    // gridDim
  RsCtl* rc;
  float* shadow;    // D * QS
  const unsigned long long* boff;  // ball lists (GraphImpl::balls): V+1 offsets, or null
  const uint32_t* bl;
};

// every vertex within distance h of r (precomputed list, else a walk)
template <class F>
__device__ __forceinline__ bool ball_each(const DevGraph& g, const RsBufs& b, uint32_t r, uint32_t h, F&& f) {
  if (b.boff) {
    const unsigned long long e = b.boff[r + 1];
    for (unsigned long long i = b.boff[r]; i < e; ++i)
      if (!f(__ldg(&b.bl[i]))) return false;
    return true;
  }
  return ball_walk(g, r, h, f);
}

__device__ __forceinline__ unsigned long long rs_key64(float vres, uint32_t v) {
  return (static_cast<unsigned long long>(__float_as_uint(vres)) << 32) | static_cast<unsigned long long>(~v);
}

// ---------------------------------------------------------------------------
// block helpers (kRsBlock threads)

// exclusive scan of x over the block; returns the prefix, *total the sum
__device__ __forceinline__ unsigned block_excl_scan(unsigned x, unsigned* total) {
  __shared__ unsigned ws[kRsBlock / 32];
  const unsigned lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  unsigned v = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= static_cast<unsigned>(o)) v += n;
  }
  __syncthreads();
  if (lane == 31) ws[wid] = v;
  __syncthreads();
  unsigned before = 0, tot = 0;
  for (unsigned w = 0; w < blockDim.x / 32; ++w) {
    if (w < wid) before += ws[w];
    tot += ws[w];
  }
  *total = tot;
  return before + v - x;
}

// ---------------------------------------------------------------------------
// Grid-wide exact top-k of 32-bit keys, ties to the lower index
// (select_top_k semantics, schedulers.cpp:105-116).  keyof(i, key) -> valid.
// mark(i) is called once for each selected i.  Loops over i are grid-stride
// and warp-uniform (every lane of a warp runs the same trip count).

template <class KeyOf, class Mark>
__device__ void coop_topk(cg::grid_group& grid, uint32_t n, unsigned long long k, KeyOf keyof, Mark mark,
                          const RsBufs& b) {
  __shared__ unsigned sh[4096];
  __shared__ unsigned s_find[4];
  RsCtl* rc = b.rc;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (int pass = 0; pass < 3; ++pass) {
    const int nb = pass == 2 ? 256 : 4096;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const uint32_t prefix = pass == 0 ? 0u : __ldcg(&rc->prefix);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      uint32_t key;
      if (!keyof(i, key)) continue;
      if (pass == 0)
        atomicAdd(&sh[key >> 20], 1u);
      else if (pass == 1) {
        if ((key >> 20) == prefix) atomicAdd(&sh[(key >> 8) & 0xfffu], 1u);
      } else if ((key >> 8) == prefix) {
        atomicAdd(&sh[key & 0xffu], 1u);
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nb; i += blockDim.x)
      if (sh[i]) atomicAdd(&b.hist[i], sh[i]);
    grid.sync();
    if (blockIdx.x == 0) {
      // copy + clear the histogram, then find the bin of the need-th key from the top
      for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        sh[i] = __ldcg(&b.hist[i]);
        b.hist[i] = 0;
      }
      __syncthreads();
      const int per = nb / blockDim.x > 0 ? nb / blockDim.x : 1;
      unsigned mine = 0;
      if (static_cast<int>(threadIdx.x) * per < nb)
        for (int j = 0; j < per; ++j) mine += sh[nb - 1 - (threadIdx.x * per + j)];
      unsigned total;
      const unsigned excl = block_excl_scan(mine, &total);
      if (pass == 0 && threadIdx.x == 0) {
        rc->total = total;
        rc->above = 0;
        rc->all = total <= k ? 1u : 0u;
      }
      __syncthreads();
      const unsigned long long above0 = pass == 0 ? 0ull : __ldcg(&rc->above);
      const bool all = pass == 0 ? (total <= k) : __ldcg(&rc->all) != 0u;
      if (!all) {
        const unsigned long long need = k - above0;
        if (static_cast<int>(threadIdx.x) * per < nb && excl < need && need <= static_cast<unsigned long long>(excl) + mine) {
          unsigned long long acc = excl;
          for (int j = 0; j < per; ++j) {
            const int bin = nb - 1 - (threadIdx.x * per + j);
            const unsigned c = sh[bin];
            if (acc < need && need <= acc + c) {
              s_find[0] = static_cast<unsigned>(bin);
              s_find[1] = static_cast<unsigned>(acc);
              s_find[2] = c;
              s_find[3] = static_cast<unsigned>(need - acc);
              break;
            }
            acc += c;
          }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          const int bits = pass == 2 ? 8 : 12;
          rc->prefix = (pass == 0 ? 0u : (__ldcg(&rc->prefix) << bits)) | s_find[0];
          rc->above = above0 + s_find[1];
          rc->ties = s_find[2];
          rc->need = s_find[3];
        }
      }
    }
    grid.sync();
    if (__ldcg(&rc->all)) break;
  }
  const bool all = __ldcg(&rc->all) != 0u;
  const uint32_t T = __ldcg(&rc->prefix);
  const unsigned need = __ldcg(&rc->need), ties = __ldcg(&rc->ties);
  if (all || need == ties) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      uint32_t key;
      if (keyof(i, key) && (all || key >= T)) mark(i);
    }
    grid.sync();
    return;
  }
  // rank the ties at T by ascending index: contiguous chunk per block
  const uint32_t cs = (n + gridDim.x - 1) / gridDim.x;
  const uint32_t c0 = blockIdx.x * cs, c1 = min(n, c0 + cs);
  unsigned cnt = 0;
  for (uint32_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
    uint32_t key;
    cnt += (keyof(i, key) && key == T) ? 1u : 0u;
  }
  unsigned tot;
  block_excl_scan(cnt, &tot);
  if (threadIdx.x == 0) b.blk[blockIdx.x] = tot;
  grid.sync();
  unsigned before = 0;
  for (uint32_t j = threadIdx.x; j < blockIdx.x; j += blockDim.x) before += __ldcg(&b.blk[j]);
  {
    // block sum of `before`
    __shared__ unsigned red[kRsBlock / 32];
    unsigned v = warp_sum(before);
    if ((threadIdx.x & 31u) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    before = 0;
    for (unsigned w = 0; w < blockDim.x / 32; ++w) before += red[w];
    __syncthreads();
  }
  unsigned running = before;
  for (uint32_t base = c0; base < c1; base += blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    uint32_t key = 0;
    const bool valid = i < c1 && keyof(i, key);
    const bool tie = valid && key == T;
    unsigned tt;
    const unsigned rank = block_excl_scan(tie ? 1u : 0u, &tt);
    if (valid && (key > T || (tie && running + rank < need))) mark(i);
    running += tt;
  }
  grid.sync();
}

// ---------------------------------------------------------------------------
// overlay update of every outgoing message of v inside splash `root`
// (update_message_into through SplashOverlayView, schedulers.cpp:270-279)

template <int QS>
__device__ __forceinline__ void splash_vertex_update(const DevGraph& g, uint32_t v, uint32_t root,
                                                     const float* __restrict__ live, float* shadow,
                                                     const uint32_t* claimed, const uint32_t* spos,
                                                     unsigned* nf) {
  const uint32_t b0 = g.in_off[v], e0 = g.in_off[v + 1];
  const uint32_t pv = __ldcg(&spos[v]);
  auto src_of = [&](uint32_t in) -> const float* {
    const uint32_t k = g.ep[in];
    const bool ov = __ldcg(&claimed[k]) == root && __ldcg(&spos[k]) < pv;
    return ov ? shadow + static_cast<size_t>(in) * QS : live + static_cast<size_t>(in) * QS;
  };
  if constexpr (QS == 1) {
    float T = g.unary_lo[v];
    for (uint32_t a = b0; a < e0; ++a) T += *src_of(g.in_adj[a]);
    for (uint32_t a = b0; a < e0; ++a) {
      const uint32_t in = g.in_adj[a], out = in ^ 1u;
      const float lnew = binary_msg(g, T - *src_of(in), out);
      if (!(fabsf(lnew) < INFINITY)) *nf = 1u;
      shadow[out] = lnew;
    }
  } else {
    const uint32_t ci = g.card[v];
    float T[QS];
#pragma unroll (QS <= 8 ? QS : 2)
    for (int x = 0; x < QS; ++x) T[x] = g.unary_log[static_cast<size_t>(v) * QS + x];
    for (uint32_t a = b0; a < e0; ++a) {
      const float* m = src_of(g.in_adj[a]);
#pragma unroll (QS <= 8 ? QS : 2)
      for (int x = 0; x < QS; ++x) T[x] += m[x];
    }
    for (uint32_t a = b0; a < e0; ++a) {
      const uint32_t in = g.in_adj[a], out = in ^ 1u;
      const uint32_t cj = g.card[g.ep[in]];
      const float* m_in = src_of(in);
      float p[QS], M = -INFINITY;
#pragma unroll (QS <= 8 ? QS : 2)
      for (int x = 0; x < QS; ++x) {
        p[x] = T[x] - m_in[x];
        if (x < static_cast<int>(ci)) M = fmaxf(M, p[x]);
      }
      float* dst = shadow + static_cast<size_t>(out) * QS;
      if (g.log_tables) {  // collapse-checked model (generic_logmatvec)
        float lo[QS];
        if (!(generic_logmatvec<QS>(g, out, p, ci, cj, lo) >= kLog2MinMass)) *nf = 1u;
        for (int xt = 0; xt < static_cast<int>(cj); ++xt) dst[xt] = lo[xt];
        continue;
      }
#pragma unroll (QS <= 8 ? QS : 2)
      for (int x = 0; x < QS; ++x) p[x] = x < static_cast<int>(ci) ? fex2(p[x] - M) : 0.f;
      float o[QS], s = 0.f;
      generic_matvec<QS>(g, out, p, o);
#pragma unroll (QS <= 8 ? QS : 2)
      for (int xt = 0; xt < QS; ++xt) s += xt < static_cast<int>(cj) ? o[xt] : 0.f;
      if (!(s > 0.f) || !(s < INFINITY)) *nf = 1u;
      const float inv = frcp(s);
#pragma unroll (QS <= 8 ? QS : 2)
      for (int xt = 0; xt < QS; ++xt)
        if (xt < static_cast<int>(cj)) dst[xt] = flg2(o[xt] * inv);
    }
  }
}

// flag x for the touched-set refresh (collect_touched, schedulers.cpp:31-42)
__device__ __forceinline__ void rs_flag(uint32_t x, uint32_t* vflag, uint32_t* vlist, unsigned* nflag,
                                        uint32_t stamp, bool dense) {
  if (dense) {
    vflag[x] = stamp;
  } else if (atomicMax(&vflag[x], stamp) < stamp) {
    vlist[atomicAdd(nflag, 1u)] = x;
  }
}

struct RsParams {
  unsigned long long k;
  uint32_t h;
  int apply;  // 0: frontier query only (lockstep rs_frontier)
};

// One Residual-Splash iteration up to the commit (cooperative launch).
template <int QS>
__global__ void __launch_bounds__(kRsBlock) k_rs_iteration(DevGraph g, float* live, const float* res,
                                                           uint32_t* vflag, uint32_t* vlist, Ctl* ctl,
                                                           RsBufs b, RsParams prm) {
  cg::grid_group grid = cg::this_grid();
  if (__ldcg(&ctl->done)) {
    if (ctl->cond_handle && blockIdx.x == 0 && threadIdx.x == 0)
      cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(ctl->cond_handle), 0u);
    return;
  }
  RsCtl* rc = b.rc;
  const uint32_t V = g.V;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  const unsigned long long k = prm.k;
  const uint32_t h = prm.h;
  const uint32_t stamp = __ldcg(&ctl->stamp);
  // row-band partition: splashes are local to the band (roots and claims on
  // owned vertices only; SURVEY 8(e) per-partition local frontiers)
  const bool band = band_graph(g);
  auto vown = [&](uint32_t v) {
    if (!band) return true;
    const uint32_t row = v / g.lat_cols;
    return row >= g.cnt_row0 && row < g.cnt_row1;
  };
  const uint32_t Vown = band ? (min(g.cnt_row1, g.lat_rows) - g.cnt_row0) * g.lat_cols : V;

  // P0: vertex residuals (vertex_residual, schedulers.cpp:128-134) + reset
  for (uint32_t v = tid; v < V; v += stride) {
    float m = 0.f;
    for (uint32_t a = g.in_off[v]; a < g.in_off[v + 1]; ++a) m = fmaxf(m, res[g.in_adj[a]]);
    b.vres[v] = m;
    b.state[v] = kRsNone;
    b.claimed[v] = kUncl;
    b.ballmax[v] = 0ull;
  }
  if (tid == 0) {
    const unsigned long long m0 = k * 4ull < 1024ull ? 1024ull : k * 4ull;
    rc->k = k;
    rc->M = static_cast<unsigned>(m0 < Vown ? m0 : Vown);
    rc->ncand = rc->nbuilt = rc->nready = rc->nkept = rc->unres = 0;
    rc->rounds = rc->passes = 0;
    rc->edges = 0;
    // touched vertices <= 2 (1 + d) per splash vertex; sparse lists below V/16
    rc->dense = (k * 64ull > V / 16) ? 1u : 0u;
    ctl->dense = rc->dense;
  }
  grid.sync();

  for (;;) {
    // P1: candidates = top-M vertices (ties to the lower id)
    const unsigned M = __ldcg(&rc->M);
    coop_topk(
        grid, V, M,
        [&](uint32_t v, uint32_t& key) {
          key = __float_as_uint(__ldcg(&b.vres[v]));
          return vown(v);
        },
        [&](uint32_t v) {
          if (__ldcg(&b.state[v]) == kRsNone) {
            const bool skip = __ldcg(&b.claimed[v]) != kUncl;
            b.state[v] = skip ? kRsSkip : kRsCand;
            if (!skip) b.clist[atomicAdd(&rc->ncand, 1u)] = v;
          }
        },
        b);
    if (tid == 0) rc->passes += 1;
    // rounds of ready-root resolution
    for (;;) {
      const uint32_t nc = __ldcg(&rc->ncand);
      // A1: skip claimed candidates, publish priorities over the balls.
      // With ball lists a warp takes a candidate and its lanes split the
      // ball (hubs of random graphs have balls of hundreds of vertices; one
      // thread per candidate would serialise a load per ball vertex).
      unsigned unres = 0;
      const bool wl = b.boff != nullptr;
      const bool prop = !wl && h > kRsMaxDepth;  // distance test by propagation
      const uint32_t lane = threadIdx.x & 31u, gw = tid >> 5, nw = stride >> 5;
      auto warp_ball = [&](uint32_t r, auto&& f) -> bool {  // all lanes; AND of f over the ball
        const unsigned long long e0 = b.boff[r], e1 = b.boff[r + 1];
        for (unsigned long long base = e0; base < e1; base += 32) {
          const unsigned long long i = base + lane;
          const bool v = i < e1 ? f(__ldg(&b.bl[i])) : true;
          if (!__all_sync(0xffffffffu, v)) return false;
        }
        return true;
      };
      for (uint32_t i = wl ? gw : tid; i < nc; i += wl ? nw : stride) {
        const uint32_t r = __ldcg(&b.clist[i]);
        if (__ldcg(&b.state[r]) != kRsCand) continue;
        if (__ldcg(&b.claimed[r]) != kUncl) {
          if (!wl || lane == 0) b.state[r] = kRsSkip;
          continue;
        }
        if (!wl || lane == 0) ++unres;
        const unsigned long long key = rs_key64(__ldcg(&b.vres[r]), r);
        if (prop)
          b.ballmax[r] = key;
        else if (wl)
          warp_ball(r, [&](uint32_t w) {
            atomicMax(&b.ballmax[w], key);
            return true;
          });
        else
          ball_each(g, b, r, h, [&](uint32_t w) {
            atomicMax(&b.ballmax[w], key);
            return true;
          });
      }
      unres = warp_sum(unres);
      if ((threadIdx.x & 31u) == 0 && unres) atomicAdd(&rc->unres, unres);
      if (tid == 0) rc->nready = 0;
      grid.sync();
      if (__ldcg(&rc->unres) == 0) break;
      if (prop) {  // ballmax[v] = max key of the unresolved candidates within 2h of v
        for (uint32_t t = 0; t < 2u * h; ++t) {
          const unsigned long long* src = (t & 1u) ? b.ballmax2 : b.ballmax;
          unsigned long long* dst = (t & 1u) ? b.ballmax : b.ballmax2;
          for (uint32_t v = tid; v < V; v += stride) {
            unsigned long long m = __ldcg(&src[v]);
            for (uint32_t a = g.in_off[v]; a < g.in_off[v + 1]; ++a) {
              const unsigned long long x = __ldcg(&src[g.ep[g.in_adj[a]]]);
              m = x > m ? x : m;
            }
            dst[v] = m;
          }
          grid.sync();
        }
      }
      // A2: ready = maximum priority over the whole ball
      for (uint32_t i = wl ? gw : tid; i < nc; i += wl ? nw : stride) {
        const uint32_t r = __ldcg(&b.clist[i]);
        if (__ldcg(&b.state[r]) != kRsCand) continue;
        const unsigned long long key = rs_key64(__ldcg(&b.vres[r]), r);
        const bool ready = prop ? __ldcg(&b.ballmax[r]) <= key
                           : wl ? warp_ball(r, [&](uint32_t w) { return __ldcg(&b.ballmax[w]) <= key; })
                                : ball_each(g, b, r, h, [&](uint32_t w) { return __ldcg(&b.ballmax[w]) <= key; });
        if (ready && (!wl || lane == 0)) b.rlist[atomicAdd(&rc->nready, 1u)] = r;
      }
      grid.sync();
      // B: build the ready splashes (build_splash, schedulers.cpp:136-167); clear the balls
      const uint32_t nr = __ldcg(&rc->nready);
      if (wl) {
        // one warp per ready root, level by level: the lanes flatten the
        // (frontier vertex, CSR neighbour) pairs of a BFS level in queue x CSR
        // order and claim the first occurrence of every unclaimed neighbour in
        // that order -- build_splash's visit order, with a handful of dependent
        // round trips per LEVEL instead of per queued vertex (the walk one
        // vertex at a time was the round's critical path: ~5 round trips per
        // ball vertex).  A level wider than the warp's SMEM frontier finishes
        // with the vertex-by-vertex walk from the level's first vertex.
        constexpr uint32_t kFront = 64;
        __shared__ uint32_t s_front[kRsBlock / 32][2][kFront];
        const uint32_t wib = threadIdx.x >> 5;
        const unsigned lt_mask = (1u << lane) - 1u;
        for (uint32_t i = gw; i < nr; i += nw) {
          const uint32_t r = __ldcg(&b.rlist[i]);
          if (lane == 0) {
            b.claimed[r] = r;
            b.spos[r] = 0;
            b.depth[r] = 0;
            b.qnext[r] = kUncl;
            s_front[wib][0][0] = r;
          }
          __syncwarp();
          uint32_t tail = r, n = 1, nf = 1, cur = 0, dlev = 0, seq_from = kUncl;
          while (nf && dlev < h) {
            uint32_t nn = 0, head = kUncl;
            for (uint32_t f0 = 0; f0 < nf; f0 += 32) {
              const uint32_t fi = f0 + lane;
              uint32_t a0 = 0, deg = 0;
              if (fi < nf) {
                const uint32_t v = s_front[wib][cur][fi];
                a0 = g.in_off[v];
                deg = g.in_off[v + 1] - a0;
              }
              uint32_t incl = deg;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (static_cast<int>(lane) >= o) incl += t;
              }
              const uint32_t total = __shfl_sync(0xffffffffu, incl, 31), excl = incl - deg;
              for (uint32_t p0 = 0; p0 < total; p0 += 32) {
                const uint32_t p = p0 + lane;
                // owner = the last lane whose exclusive prefix is <= p
                uint32_t lo = 0;
#pragma unroll
                for (uint32_t step = 16; step > 0; step >>= 1) {
                  const uint32_t ex = __shfl_sync(0xffffffffu, excl, lo + step);
                  if (ex <= p) lo += step;
                }
                const uint32_t a0o = __shfl_sync(0xffffffffu, a0, lo), exo = __shfl_sync(0xffffffffu, excl, lo);
                uint32_t w = kUncl;
                bool cand = false;
                if (p < total) {
                  w = g.ep[g.in_adj[a0o + (p - exo)]];
                  cand = __ldcg(&b.claimed[w]) == kUncl && vown(w);
                }
                // two frontier vertices can share a neighbour: the first pair wins
                const unsigned cm = __ballot_sync(0xffffffffu, cand);
                const unsigned same = __match_any_sync(0xffffffffu, w) & cm;
                const bool win = cand && lane == static_cast<uint32_t>(__ffs(same) - 1);
                const unsigned m = __ballot_sync(0xffffffffu, win);
                if (m) {
                  const unsigned below = m & lt_mask;
                  const int prev_lane = below ? 31 - __clz(below) : 0;
                  const uint32_t wp = __shfl_sync(0xffffffffu, w, prev_lane);
                  if (win) {
                    b.claimed[w] = r;
                    b.depth[w] = dlev + 1;
                    b.spos[w] = n + __popc(below);
                    b.qnext[w] = kUncl;
                    b.qnext[below ? wp : tail] = w;
                    const uint32_t pos = nn + __popc(below);
                    if (pos < kFront) s_front[wib][cur ^ 1u][pos] = w;
                  }
                  if (head == kUncl) head = __shfl_sync(0xffffffffu, w, __ffs(m) - 1);
                  tail = __shfl_sync(0xffffffffu, w, 31 - __clz(m));
                  n += __popc(m);
                  nn += __popc(m);
                }
                __syncwarp();
              }
            }
            ++dlev;
            cur ^= 1u;
            nf = nn;
            if (nn > kFront) {  // too wide for the SMEM frontier: walk on from the level's first vertex
              seq_from = head;
              break;
            }
          }
          for (uint32_t v = seq_from; v != kUncl;) {
            const uint32_t dv = b.depth[v];
            if (dv < h) {
              const uint32_t a0 = g.in_off[v], a1 = g.in_off[v + 1];
              for (uint32_t base = a0; base < a1; base += 32) {
                const uint32_t a = base + lane;
                uint32_t w = kUncl;
                bool cand = false;
                if (a < a1) {
                  w = g.ep[g.in_adj[a]];
                  cand = __ldcg(&b.claimed[w]) == kUncl && vown(w);
                }
                const unsigned m = __ballot_sync(0xffffffffu, cand);
                if (m) {
                  const unsigned below = m & ((1u << lane) - 1u);
                  const int prev_lane = below ? 31 - __clz(below) : 0;
                  const uint32_t wp = __shfl_sync(0xffffffffu, w, prev_lane);
                  if (cand) {
                    b.claimed[w] = r;
                    b.depth[w] = dv + 1;
                    b.spos[w] = n + __popc(below);
                    b.qnext[w] = kUncl;
                    b.qnext[below ? wp : tail] = w;
                  }
                  tail = __shfl_sync(0xffffffffu, w, 31 - __clz(m));
                  n += __popc(m);
                }
                __syncwarp();
              }
            }
            __syncwarp();
            v = b.qnext[v];
          }
          if (lane == 0) {
            b.state[r] = kRsBuilt;
            b.blist[atomicAdd(&rc->nbuilt, 1u)] = r;
          }
          warp_ball(r, [&](uint32_t w) {
            b.ballmax[w] = 0ull;
            return true;
          });
        }
      }
      for (uint32_t i = tid; i < (wl ? 0u : nr); i += stride) {
        const uint32_t r = __ldcg(&b.rlist[i]);
        b.claimed[r] = r;
        b.spos[r] = 0;
        b.depth[r] = 0;
        b.qnext[r] = kUncl;
        uint32_t tail = r, n = 1;
        for (uint32_t v = r; v != kUncl; v = b.qnext[v]) {
          const uint32_t dv = b.depth[v];
          if (dv < h) {
            for (uint32_t a = g.in_off[v]; a < g.in_off[v + 1]; ++a) {
              const uint32_t w = g.ep[g.in_adj[a]];
              if (__ldcg(&b.claimed[w]) == kUncl && vown(w)) {
                b.claimed[w] = r;
                b.depth[w] = dv + 1;
                b.spos[w] = n++;
                b.qnext[w] = kUncl;
                b.qnext[tail] = w;
                tail = w;
              }
            }
          }
        }
        b.state[r] = kRsBuilt;
        b.blist[atomicAdd(&rc->nbuilt, 1u)] = r;
        if (!prop)
          ball_each(g, b, r, h, [&](uint32_t w) {
            b.ballmax[w] = 0ull;
            return true;
          });
      }
      // unresolved candidates clear their balls (a ready root racing to
      // kRsBuilt may be cleared twice: idempotent)
      if (prop)  // the propagation filled every vertex: clear them all
        for (uint32_t v = tid; v < V; v += stride) b.ballmax[v] = 0ull;
      for (uint32_t i = wl ? gw : (prop ? nc : tid); i < nc; i += wl ? nw : stride) {
        const uint32_t r = __ldcg(&b.clist[i]);
        uint32_t st = __ldcg(&b.state[r]);
        // builders flip states concurrently in this phase: one read per warp
        if (wl) st = __shfl_sync(0xffffffffu, st, 0);
        if (st != kRsCand) continue;
        if (wl)
          warp_ball(r, [&](uint32_t w) {
            b.ballmax[w] = 0ull;
            return true;
          });
        else
          ball_each(g, b, r, h, [&](uint32_t w) {
            b.ballmax[w] = 0ull;
            return true;
          });
      }
      if (tid == 0) {
        rc->unres = 0;
        rc->rounds += 1;
      }
      grid.sync();
    }
    const unsigned nbuilt = __ldcg(&rc->nbuilt), Mc = __ldcg(&rc->M);
    if (nbuilt >= k || Mc >= Vown) break;
    grid.sync();
    if (tid == 0) rc->M = static_cast<unsigned>(min(static_cast<unsigned long long>(Vown), 4ull * Mc));
    grid.sync();
  }

  // P4: keep the k built splashes of highest priority
  const unsigned nbuilt = __ldcg(&rc->nbuilt);
  if (nbuilt > k) {
    coop_topk(
        grid, V, k,
        [&](uint32_t v, uint32_t& key) {
          key = __float_as_uint(__ldcg(&b.vres[v]));
          return __ldcg(&b.state[v]) == kRsBuilt;
        },
        [&](uint32_t v) {
          b.state[v] = kRsKept;
          b.klist[atomicAdd(&rc->nkept, 1u)] = v;
        },
        b);
  } else {
    for (uint32_t i = tid; i < nbuilt; i += stride) b.klist[i] = __ldcg(&b.blist[i]);
    if (tid == 0) rc->nkept = nbuilt;
    grid.sync();
  }
  if (!prm.apply) return;

  // P5: Gauss-Seidel updates inside each splash into the shadow buffer; the
  // live buffer stays the pre-step snapshot for every other splash.
  const unsigned nk = __ldcg(&rc->nkept);
  unsigned long long edges = 0;
  // binary graphs: a warp per splash, lanes over the incoming edges of each
  // visited vertex (cavity sums by warp reduction); otherwise a thread per splash
  const bool wsplash = QS == 1;
  const uint32_t wlane = threadIdx.x & 31u, wgw = tid >> 5, wnw = stride >> 5;
  if (wsplash) {
    for (uint32_t i = wgw; i < nk; i += wnw) {
      const uint32_t r = __ldcg(&b.klist[i]);
      for (uint32_t v = r; v != kUncl; v = __ldcg(&b.qnext[v])) {
        const uint32_t a0 = g.in_off[v], a1 = g.in_off[v + 1];
        const uint32_t pv = __ldcg(&b.spos[v]);
        auto msg_in = [&](uint32_t in) {
          const uint32_t k = g.ep[in];
          const bool ov = __ldcg(&b.claimed[k]) == r && __ldcg(&b.spos[k]) < pv;
          return ov ? b.shadow[in] : live[in];
        };
        // cavity total in CSR order (unary first), exactly as the refresh
        // kernels sum it, so a fixed point stays bitwise stable: the lanes load
        // in parallel, the accumulation walks the lanes in order
        float T = g.unary_lo[v];
        for (uint32_t base = a0; base < a1; base += 32) {
          const float m = base + wlane < a1 ? msg_in(g.in_adj[base + wlane]) : 0.f;
          const uint32_t cnt = min(32u, a1 - base);
          for (uint32_t j = 0; j < cnt; ++j) T += __shfl_sync(0xffffffffu, m, j);
        }
        bool bad = false;
        for (uint32_t base = a0; base < a1; base += 32) {
          if (base + wlane < a1) {
            const uint32_t in = g.in_adj[base + wlane], out = in ^ 1u;
            const float lnew = binary_msg(g, T - msg_in(in), out);
            bad |= !(fabsf(lnew) < INFINITY);
            b.shadow[out] = lnew;
          }
        }
        if (bad) ctl->numeric_error = 1u;
        if (wlane == 0) edges += a1 - a0;
        __syncwarp();
      }
    }
  } else {
    for (uint32_t i = tid; i < nk; i += stride) {
      const uint32_t r = __ldcg(&b.klist[i]);
      for (uint32_t v = r; v != kUncl; v = __ldcg(&b.qnext[v])) {
        splash_vertex_update<QS>(g, v, r, live, b.shadow, b.claimed, b.spos, &ctl->numeric_error);
        edges += g.in_off[v + 1] - g.in_off[v];
      }
    }
  }
  edges = warp_sum(edges);
  if ((threadIdx.x & 31u) == 0 && edges) {
    atomicAdd(&rc->edges, edges);
    atomicAdd(&ctl->frontier, edges);
  }
  grid.sync();
  // P6: commit_shadow + touched flags (every vertex of a splash and its neighbours)
  const bool dense = __ldcg(&rc->dense) != 0u;
  if (wsplash) {  // same splash -> warp mapping as P5: the shadow writes are this warp's own
    for (uint32_t i = wgw; i < nk; i += wnw) {
      const uint32_t r = __ldcg(&b.klist[i]);
      for (uint32_t v = r; v != kUncl; v = __ldcg(&b.qnext[v])) {
        if (wlane == 0) rs_flag(v, vflag, vlist, &ctl->nflag, stamp, dense);
        const uint32_t a0 = g.in_off[v], a1 = g.in_off[v + 1];
        for (uint32_t a = a0 + wlane; a < a1; a += 32) {
          const uint32_t in = g.in_adj[a], out = in ^ 1u;
          live[out] = b.shadow[out];
          rs_flag(g.ep[in], vflag, vlist, &ctl->nflag, stamp, dense);
        }
      }
    }
  }
  for (uint32_t i = tid; i < (wsplash ? 0u : nk); i += stride) {
    const uint32_t r = __ldcg(&b.klist[i]);
    for (uint32_t v = r; v != kUncl; v = __ldcg(&b.qnext[v])) {
      rs_flag(v, vflag, vlist, &ctl->nflag, stamp, dense);
      for (uint32_t a = g.in_off[v]; a < g.in_off[v + 1]; ++a) {
        const uint32_t in = g.in_adj[a], out = in ^ 1u;
#pragma unroll (QS <= 8 ? QS : 2)
        for (int x = 0; x < QS; ++x)
          live[static_cast<size_t>(out) * QS + x] = b.shadow[static_cast<size_t>(out) * QS + x];
        rs_flag(g.ep[in], vflag, vlist, &ctl->nflag, stamp, dense);
      }
    }
  }
  if (tid == 0) {
    ctl->splashes += nk;
    ctl->rs_rounds += rc->rounds;
    ctl->rs_passes += rc->passes;
  }
}

// ---------------------------------------------------------------------------
// Lockstep apply of host-supplied splashes (apply_splash_frontier with an
// arbitrary edge order): one thread per splash, one message at a time; the
// overlay is "written by this splash already" = written[d] == own stamp.

template <int QS>
__global__ void __launch_bounds__(kBlock) k_splash_apply_edges(DevGraph g, const float* __restrict__ live,
                                                               float* shadow, uint32_t* written,
                                                               const unsigned long long* eoff,
                                                               const uint32_t* edges, uint32_t ns,
                                                               uint32_t stamp0, unsigned* nf) {
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= ns) return;
  const uint32_t me = stamp0 + s;
  for (unsigned long long j = eoff[s]; j < eoff[s + 1]; ++j) {
    const uint32_t d = edges[j];
    const uint32_t v = g.ep[d];       // source of d
    const uint32_t back = d ^ 1u;     // the incoming edge excluded from the product
    auto src_of = [&](uint32_t in) -> const float* {
      return written[in] == me ? shadow + static_cast<size_t>(in) * QS : live + static_cast<size_t>(in) * QS;
    };
    if constexpr (QS == 1) {
      float T = g.unary_lo[v];
      for (uint32_t a = g.in_off[v]; a < g.in_off[v + 1]; ++a) {
        const uint32_t in = g.in_adj[a];
        if (in != back) T += *src_of(in);
      }
      const float lnew = binary_msg(g, T, d);
      if (!(fabsf(lnew) < INFINITY)) *nf = 1u;
      shadow[d] = lnew;
    } else {
      const uint32_t ci = g.card[v], cj = g.card[g.ep[back]];
      float p[QS], M = -INFINITY;
#pragma unroll (QS <= 8 ? QS : 2)
      for (int x = 0; x < QS; ++x) p[x] = g.unary_log[static_cast<size_t>(v) * QS + x];
      for (uint32_t a = g.in_off[v]; a < g.in_off[v + 1]; ++a) {
        const uint32_t in = g.in_adj[a];
        if (in == back) continue;
        const float* m = src_of(in);
#pragma unroll (QS <= 8 ? QS : 2)
        for (int x = 0; x < QS; ++x) p[x] += m[x];
      }
#pragma unroll (QS <= 8 ? QS : 2)
      for (int x = 0; x < QS; ++x)
        if (x < static_cast<int>(ci)) M = fmaxf(M, p[x]);
      if (g.log_tables) {  // collapse-checked model (generic_logmatvec)
        float lo[QS];
        if (!(generic_logmatvec<QS>(g, d, p, ci, cj, lo) >= kLog2MinMass)) *nf = 1u;
        for (int xt = 0; xt < static_cast<int>(cj); ++xt) shadow[static_cast<size_t>(d) * QS + xt] = lo[xt];
      } else {
#pragma unroll (QS <= 8 ? QS : 2)
        for (int x = 0; x < QS; ++x) p[x] = x < static_cast<int>(ci) ? fex2(p[x] - M) : 0.f;
        float o[QS], s2 = 0.f;
        generic_matvec<QS>(g, d, p, o);
#pragma unroll (QS <= 8 ? QS : 2)
        for (int xt = 0; xt < QS; ++xt) s2 += xt < static_cast<int>(cj) ? o[xt] : 0.f;
        if (!(s2 > 0.f) || !(s2 < INFINITY)) *nf = 1u;
        const float inv = frcp(s2);
#pragma unroll (QS <= 8 ? QS : 2)
        for (int xt = 0; xt < QS; ++xt)
          if (xt < static_cast<int>(cj)) shadow[static_cast<size_t>(d) * QS + xt] = flg2(o[xt] * inv);
      }
    }
    written[d] = me;
  }
}

// commit_shadow + touched flags for host-supplied splash edges (thread per edge)
template <int QS>
__global__ void __launch_bounds__(kBlock) k_splash_commit_edges(DevGraph g, float* live, const float* shadow,
                                                                const uint32_t* edges, uint32_t n, uint32_t* vflag,
                                                                uint32_t* vlist, Ctl* ctl) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (blockIdx.x == 0 && threadIdx.x == 0) ctl->dense = 0;
  if (i >= n) return;
  const uint32_t d = edges[i];
#pragma unroll (QS <= 8 ? QS : 2)
  for (int x = 0; x < QS; ++x) live[static_cast<size_t>(d) * QS + x] = shadow[static_cast<size_t>(d) * QS + x];
  const uint32_t stamp = ctl->stamp;
  rs_flag(g.ep[d], vflag, vlist, &ctl->nflag, stamp, false);
  rs_flag(g.ep[d ^ 1u], vflag, vlist, &ctl->nflag, stamp, false);
}

}  // namespace bpb
