// CUDA kernels of the B200 BP engine (sm_100a).  See DESIGN.md section 5 for
// the roofline of each kernel and its algorithmic bytes.
//
// Reference correspondence (paths relative to /root/reference/proj/core):
//   vertex_update  <- refresh_residuals (src/residuals.cpp:26-59) calling
//                     update_message_into (include/bpsched/messages.hpp:114-151)
//                     + residual (src/messages.cpp:56-65), and one LBP sweep
//                     (apply_frontier fast path, src/schedulers.cpp:243-245)
//   rnbp_select    <- rnbp_frontier (src/schedulers.cpp:194-216) fused with the
//                     commit loop of apply_frontier (src/schedulers.cpp:231-241)
//                     and collect_touched (src/schedulers.cpp:31-42)
//   radix_*        <- select_top_k (src/schedulers.cpp:105-116)
//   finalize       <- the loop control of run() (src/schedulers.cpp:301-347)
//   beliefs        <- compute_beliefs (src/messages.cpp:82-105)
#pragma once

#include "bp_device.cuh"

namespace bpb {

enum UpdateMode : int {
  kModeCount = 0,  // LBP sweep: write next messages, count r >= eps
  kModeInit = 1,   // first refresh: write candidates + residuals, count r >= eps
  kModeDelta = 2,  // refresh: write candidates + residuals, count (now - was)
};

enum FinMode : int { kFinNone = 0, kFinLbp = 1, kFinInit = 2, kFinIter = 3, kFinApply = 4,
                     kFinInitExt = 5, kFinIterExt = 6, kFinFused = 7 };  // *Ext: RnBP band, all-reduced sums

constexpr int kSinkCap = 4096;

// Block-level staging of list appends: pushes go to shared memory (spilling
// straight to the global list when full), flushes reserve the block's range
// with one global atomic.
struct Stager {
  uint32_t* sbuf;     // shared, cap entries
  unsigned* scount;   // shared
  unsigned* sbase;    // shared
  unsigned cap;
  uint32_t* gdst;     // global list
  unsigned* gcount;   // global counter

  __device__ __forceinline__ void init() {
    if (threadIdx.x == 0) *scount = 0;
    __syncthreads();
  }
  // any thread, any time: one shared atomic per group of converged lanes
  __device__ __forceinline__ void push(uint32_t x) {
    const unsigned m = __activemask();
    const unsigned lane = threadIdx.x & 31u;
    const unsigned leader = __ffs(m) - 1;
    unsigned base = 0;
    if (lane == leader) base = atomicAdd(scount, __popc(m));
    base = __shfl_sync(m, base, leader);
    const unsigned i = base + __popc(m & ((1u << lane) - 1u));
    if (i < cap)
      sbuf[i] = x;
    else
      gdst[atomicAdd(gcount, 1u)] = x;
  }
  // warp-aggregated push; all lanes of the warp must call it
  __device__ __forceinline__ void push_warp(bool pred, uint32_t x) {
    const unsigned lane = threadIdx.x & 31u;
    const unsigned mask = __ballot_sync(0xffffffffu, pred);
    if (mask == 0) return;
    const unsigned leader = __ffs(mask) - 1;
    unsigned base = 0;
    if (lane == leader) base = atomicAdd(scount, __popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (pred) {
      const unsigned i = base + __popc(mask & ((1u << lane) - 1u));
      if (i < cap)
        sbuf[i] = x;
      else
        gdst[atomicAdd(gcount, 1u)] = x;
    }
  }
  // block-uniform: flush when fewer than `room` slots remain (room == 0: always)
  __device__ __forceinline__ void flush(unsigned room) {
    __syncthreads();
    const unsigned n0 = *scount;
    const unsigned n = n0 < cap ? n0 : cap;
    if (n == 0 || (room && n0 + room <= cap)) return;
    __syncthreads();
    if (threadIdx.x == 0) *sbase = atomicAdd(gcount, n);
    __syncthreads();
    const unsigned gb = *sbase;
    for (unsigned i = threadIdx.x; i < n; i += blockDim.x) gdst[gb + i] = sbuf[i];
    __syncthreads();
    if (threadIdx.x == 0) *scount = 0;
    __syncthreads();
  }
};

// Last flush of a phase: one barrier before the reservation, one after; the
// buffer is not reset (the next phase's init() does that behind its barrier).
__device__ __forceinline__ void flush_final(Stager& st) {
  __syncthreads();
  const unsigned n = min(*st.scount, st.cap);
  if (n == 0) return;
  if (threadIdx.x == 0) *st.sbase = atomicAdd(st.gcount, n);
  __syncthreads();
  const unsigned gb = *st.sbase;
  for (unsigned i = threadIdx.x; i < n; i += blockDim.x) st.gdst[gb + i] = st.sbuf[i];
}

// Flush two stagers with their global reservations issued concurrently
// (threads 0 and 32), one round trip instead of two.
__device__ __forceinline__ void flush2(Stager& a, Stager& b) {
  __syncthreads();
  const unsigned na = min(*a.scount, a.cap), nb = min(*b.scount, b.cap);
  if (na == 0 && nb == 0) return;
  if (threadIdx.x == 0 && na) *a.sbase = atomicAdd(a.gcount, na);
  if (threadIdx.x == 32 && nb) *b.sbase = atomicAdd(b.gcount, nb);
  __syncthreads();
  for (unsigned i = threadIdx.x; i < na; i += blockDim.x) a.gdst[*a.sbase + i] = a.sbuf[i];
  for (unsigned i = threadIdx.x; i < nb; i += blockDim.x) b.gdst[*b.sbase + i] = b.sbuf[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    *a.scount = 0;
    *b.scount = 0;
  }
  __syncthreads();
}

#define BPB_STAGER(name, capacity, dst, counter)          \
  __shared__ uint32_t name##_buf[capacity];               \
  __shared__ unsigned name##_cnt, name##_base;            \
  Stager name{name##_buf, &name##_cnt, &name##_base, capacity, dst, counter}


// ---------------------------------------------------------------------------
// accumulation: block reduction, then <= 6 atomics into slot blockIdx % kSlots

struct Contrib {
  long long delta = 0;
  unsigned long long count = 0, frontier = 0, survivors = 0, evals = 0, visits = 0;
};

__device__ __forceinline__ void block_accumulate(Ctl* ctl, const Contrib& c) {
  __shared__ unsigned long long sh[6][32];
  const unsigned lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  unsigned long long v[6] = {static_cast<unsigned long long>(c.delta), c.count, c.frontier, c.survivors,
                             c.evals, c.visits};
#pragma unroll
  for (int k = 0; k < 6; ++k) v[k] = warp_sum(v[k]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < 6; ++k) sh[k][wid] = v[k];
  __syncthreads();
  if (wid == 0) {
    const unsigned nw = blockDim.x >> 5;
    unsigned long long mine = 0;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      unsigned long long x = lane < nw ? sh[k][lane] : 0ull;
      x = warp_sum(x);
      if (static_cast<int>(lane) == k) mine = x;
    }
    if (lane < 6 && mine) {
      Accum& a = ctl->acc[blockIdx.x % kSlots];
      unsigned long long* f = lane == 0 ? reinterpret_cast<unsigned long long*>(&a.delta)
                              : lane == 1 ? &a.count
                              : lane == 2 ? &a.frontier
                              : lane == 3 ? &a.survivors
                              : lane == 4 ? &a.evals
                                          : &a.visits;
      atomicAdd(f, mine);
    }
  }
}

// Stream-ordered scalar stores into the control block (the value travels as a
// kernel argument: no pinned staging, no host synchronisation)
static __global__ void k_set_u64(unsigned long long* p, unsigned long long v) { *p = v; }
static __global__ void k_set_u32(unsigned* p, unsigned v) { *p = v; }

// Early exit of every loop kernel once the run is over; inside the device-side
// WHILE loop it also clears the loop condition.
__device__ __forceinline__ bool run_done(Ctl* c) {
  if (!c->done && !c->band_wait) return false;
  if (c->cond_handle && blockIdx.x == 0 && threadIdx.x == 0)
    cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(c->cond_handle), 0u);
  return true;
}

// ---------------------------------------------------------------------------
// finalize: one block reduces the slots and restates the loop control of
// run() (schedulers.cpp:301-347).

// (t0_ns: the run's start, Ctl::t0_ns, passed in by callers that hold it in a register)
__device__ __forceinline__ void fin_record(Ctl* c, unsigned long long it, unsigned long long fs,
                                           unsigned un, unsigned long long t0_ns) {
  TraceRec& r = c->trace[it % kTraceRing];
  r.iteration = it;
  r.frontier_size = fs;
  r.unconverged = un;
  r.elapsed_seconds = 1e-9 * static_cast<double>(globaltimer_ns() - t0_ns);
  c->trace_len = it + 1;
}
__device__ __forceinline__ void fin_record(Ctl* c, unsigned long long it, unsigned long long fs,
                                           unsigned un) {
  fin_record(c, it, fs, un, c->t0_ns);
}

// The loop-control fields of Ctl the finalize touches, loaded into registers
// as one batch of independent loads and stored back as one batch: the
// finalize is the serial tail of every iteration, and a chain of dependent
// control-block round trips would cost microseconds.
struct FinRegs {
  unsigned done, converged, numeric_error, has_prev, unconverged, prev_unconverged, nflag, dense;
  unsigned stamp, stop_reason, cl_cur, use_clist, cl_state, persist_ok, rx_prefix, fused_par, fused_abort;
  unsigned cl_n[2];
  unsigned long long iteration, sweeps, max_iterations, msgs_total, evals_total, vertex_visits, t0_ns,
      time_limit_ns, frontier, survivors, rx_above, trace_len, cond_handle, handover_it;

  __device__ __forceinline__ void load(const Ctl* c) {
    done = c->done;
    converged = c->converged;
    numeric_error = c->numeric_error;
    has_prev = c->has_prev;
    unconverged = c->unconverged;
    prev_unconverged = c->prev_unconverged;
    nflag = c->nflag;
    dense = c->dense;
    stamp = c->stamp;
    stop_reason = c->stop_reason;
    cl_cur = c->cl_cur;
    use_clist = c->use_clist;
    cl_state = c->cl_state;
    persist_ok = c->persist_ok;
    rx_prefix = c->rx_prefix;
    fused_par = c->fused_par;
    fused_abort = c->fused_abort;
    cl_n[0] = c->cl_n[0];
    cl_n[1] = c->cl_n[1];
    iteration = c->iteration;
    sweeps = c->sweeps;
    max_iterations = c->max_iterations;
    msgs_total = c->msgs_total;
    evals_total = c->evals_total;
    vertex_visits = c->vertex_visits;
    t0_ns = c->t0_ns;
    time_limit_ns = c->time_limit_ns;
    frontier = c->frontier;
    survivors = c->survivors;
    rx_above = c->rx_above;
    trace_len = c->trace_len;
    cond_handle = c->cond_handle;
    handover_it = c->handover_it;
  }
  // numeric_error is never stored back: any thread may raise it concurrently
  __device__ __forceinline__ void store(Ctl* c) const {
    c->done = done;
    c->converged = converged;
    c->has_prev = has_prev;
    c->unconverged = unconverged;
    c->prev_unconverged = prev_unconverged;
    c->nflag = nflag;
    c->dense = dense;
    c->stamp = stamp;
    c->stop_reason = stop_reason;
    c->cl_cur = cl_cur;
    c->cl_state = cl_state;
    c->rx_prefix = rx_prefix;
    c->fused_par = fused_par;
    c->fused_abort = fused_abort;
    c->cl_n[0] = cl_n[0];
    c->cl_n[1] = cl_n[1];
    c->iteration = iteration;
    c->sweeps = sweeps;
    c->msgs_total = msgs_total;
    c->evals_total = evals_total;
    c->vertex_visits = vertex_visits;
    c->time_limit_ns = time_limit_ns;
    c->frontier = frontier;
    c->survivors = survivors;
    c->rx_above = rx_above;
    c->trace_len = trace_len;
    c->handover_it = handover_it;
  }
};

__device__ __forceinline__ void fin_record(FinRegs& f, TraceRec* trace, unsigned long long it, unsigned long long fs,
                                           unsigned un) {
  TraceRec& r = trace[it % kTraceRing];
  r.iteration = it;
  r.frontier_size = fs;
  r.unconverged = un;
  r.elapsed_seconds = 1e-9 * static_cast<double>(globaltimer_ns() - f.t0_ns);
  f.trace_len = it + 1;
}

// top of the loop: converged check BEFORE the cap check (schedulers.cpp:302-309)
__device__ __forceinline__ void fin_check_top(FinRegs& c) {
  if (c.numeric_error) {
    c.done = 1;
    c.stop_reason = kStopNumeric;
    return;
  }
  if (c.unconverged == 0) {
    c.converged = 1;
    c.done = 1;
    c.stop_reason = kStopConverged;
    return;
  }
  if (c.iteration >= c.max_iterations) {
    c.done = 1;
    c.stop_reason = kStopMaxIter;
  } else if (globaltimer_ns() - c.t0_ns >= c.time_limit_ns) {
    c.done = 1;
    c.stop_reason = kStopTime;
  }
}

__device__ __forceinline__ void fin_reset_scratch(FinRegs& c) {
  c.frontier = 0;
  c.survivors = 0;
  c.nflag = 0;
  c.dense = 0;
  c.stamp += 1;
  c.rx_prefix = 0;
  c.rx_above = 0;
}

// end of one iteration of the run loop (schedulers.cpp:326-346)
__device__ __forceinline__ void fin_iter(FinRegs& c, TraceRec* trace, long long delta, unsigned long long frontier,
                                         uint32_t D) {
  const unsigned start = c.unconverged;
  c.unconverged = static_cast<unsigned>(static_cast<long long>(start) + delta);
  fin_record(c, trace, c.iteration, frontier, c.unconverged);
  c.msgs_total += frontier;
  c.prev_unconverged = start;  // set_prev_unconverged (schedulers.cpp:327)
  c.has_prev = 1;
  c.iteration += 1;
  if (c.use_clist) {
    // RnBP candidate list: scan residuals while most edges are unconverged;
    // once fewer than 1/16 are, the next select builds the list (state 1) and
    // from then on iterations walk it (state 2)
    if (c.cl_state >= 1u) {
      c.cl_cur ^= 1u;
      c.cl_n[c.cl_cur ^ 1u] = 0;
      c.cl_state = 2u;
    } else if (16ull * c.unconverged < D) {
      c.cl_state = 1u;
    }
  }
  fin_reset_scratch(c);
  fin_check_top(c);
}

// ---------------------------------------------------------------------------
// row-band partition: halo rows of a lattice band.  The band
// holds its owned rows plus one ghost row per neighbouring band.  After a
// sweep writes the new messages into B, the band's boundary messages go to
// the neighbours (send) and the neighbours' messages overwrite the ghost-row
// messages that flow into owned rows (recv), so every owned vertex sees
// exactly the messages of the unpartitioned sweep.

__device__ __forceinline__ uint32_t lat_edge_down(uint32_t lr, uint32_t c, uint32_t C) {
  return lr * (2u * C - 1u) + 2u * c + (c + 1u < C ? 1u : 0u);
}

// pack after the sweep: B = the buffer the sweep just wrote (ping-pong parity)
static __global__ void k_part_pack(DevGraph g, const float* buf0, const float* buf1, Ctl* ctl, PartHalo h) {
  const float* B = (ctl->sweeps & 1ull) ? buf0 : buf1;
  const uint32_t C = g.lat_cols, L = g.lat_rows;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    if (h.ghost_up) h.send_up[c] = B[2u * lat_edge_down(0u, c, C) + 1u];     // (1, c) -> (0, c)
    if (h.ghost_down) h.send_down[c] = B[2u * lat_edge_down(L - 2u, c, C)];  // (L-2, c) -> (L-1, c)
  }
}

// local count of the sweep (slots) -> h.count[0]; time-limit vote -> h.count[1]
static __global__ void __launch_bounds__(kSlots) k_part_count(Ctl* c, PartHalo h) {
  unsigned long long v = c->acc[threadIdx.x].count;
  __shared__ unsigned long long sh[kSlots / 32];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < kSlots / 32; ++w) t += sh[w];
    h.count[0] = t;
    h.count[1] = (globaltimer_ns() - c->t0_ns >= c->vote_limit_ns) ? 1ull : 0ull;
  }
}

static __global__ void k_part_unpack(DevGraph g, float* buf0, float* buf1, const Ctl* ctl, PartHalo h) {
  float* B = (ctl->sweeps & 1ull) ? buf0 : buf1;
  const uint32_t C = g.lat_cols, L = g.lat_rows;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    if (h.ghost_up) B[2u * lat_edge_down(0u, c, C)] = h.recv_up[c];               // (0, c) -> (1, c)
    if (h.ghost_down) B[2u * lat_edge_down(L - 2u, c, C) + 1u] = h.recv_down[c];  // (L-1, c) -> (L-2, c)
  }
}

// RnBP on a band: halos of the LIVE messages after the commit; a ghost
// message that changed flags the owned vertex it flows into, whose outgoing
// messages the refresh then recomputes (collect_touched, schedulers.cpp:31-42)
static __global__ void k_part_pack_live(DevGraph g, const float* M, PartHalo h) {
  const uint32_t C = g.lat_cols, L = g.lat_rows;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    if (h.ghost_up) h.send_up[c] = M[2u * lat_edge_down(0u, c, C) + 1u];
    if (h.ghost_down) h.send_down[c] = M[2u * lat_edge_down(L - 2u, c, C)];
  }
}

static __global__ void k_part_unpack_flag(DevGraph g, float* M, Ctl* ctl, uint32_t* vflag, uint32_t* vlist,
                                          PartHalo h) {
  if (run_done(ctl)) return;
  const uint32_t C = g.lat_cols, L = g.lat_rows;
  const uint32_t stamp = ctl->stamp;
  const bool dense = ctl->dense != 0u;
  auto flag = [&](uint32_t v) {
    if (dense) {
      vflag[v] = stamp;
    } else if (atomicMax(&vflag[v], stamp) < stamp) {
      vlist[atomicAdd(&ctl->nflag, 1u)] = v;
    }
  };
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < C; c += gridDim.x * blockDim.x) {
    if (h.ghost_up) {
      float* m = &M[2u * lat_edge_down(0u, c, C)];
      if (*m != h.recv_up[c]) {
        *m = h.recv_up[c];
        flag(C + c);  // (1, c)
      }
    }
    if (h.ghost_down) {
      float* m = &M[2u * lat_edge_down(L - 2u, c, C) + 1u];
      if (*m != h.recv_down[c]) {
        *m = h.recv_down[c];
        flag((L - 2u) * C + c);  // (L-2, c)
      }
    }
  }
}

// vertex-range partition (bp_graph_create_part): the cut messages of any
// graph move through index lists -- send: owned-source messages whose target
// a peer owns, recv: messages from a peer's vertices into owned ones, each
// peer's run in global directed-id order on both sides.
// pingpong: M = the buffer the LBP sweep just wrote (ctl->sweeps parity).
static __global__ void k_plist_pack(const float* buf0, const float* buf1, const Ctl* ctl, int pingpong,
                                    const uint32_t* __restrict__ idx, uint32_t n, float* __restrict__ out) {
  const float* M = pingpong && !(ctl->sweeps & 1ull) ? buf1 : buf0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = M[idx[i]];
}

static __global__ void k_plist_unpack(float* buf0, float* buf1, const Ctl* ctl, int pingpong,
                                      const uint32_t* __restrict__ idx, uint32_t n, const float* __restrict__ in) {
  float* M = pingpong && !(ctl->sweeps & 1ull) ? buf1 : buf0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) M[idx[i]] = in[i];
}

// RnBP: a changed message from a peer flags the owned vertex it flows into
// (collect_touched across the cut, schedulers.cpp:31-42)
static __global__ void k_plist_unpack_flag(DevGraph g, float* M, Ctl* ctl, uint32_t* vflag, uint32_t* vlist,
                                           const uint32_t* __restrict__ idx, uint32_t n, const float* __restrict__ in) {
  if (run_done(ctl)) return;
  const uint32_t stamp = ctl->stamp;
  const bool dense = ctl->dense != 0u;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t d = idx[i];
    if (M[d] != in[i]) {
      M[d] = in[i];
      const uint32_t v = g.ep[d ^ 1u];  // target
      if (dense) {
        vflag[v] = stamp;
      } else if (atomicMax(&vflag[v], stamp) < stamp) {
        vlist[atomicAdd(&ctl->nflag, 1u)] = v;
      }
    }
  }
}

// the band's contributions of the iteration -> h.count = {delta, frontier,
// survivors, time vote, count (init)}; slots are left for the finalize
static __global__ void __launch_bounds__(kSlots) k_part_count_rnbp(Ctl* c, PartHalo h) {
  if (c->band_wait) {  // waiting for the host's retry: zeros keep the in-place all-reduce bounded
    if (threadIdx.x < 5) h.count[threadIdx.x] = 0ull;
    return;
  }
  __shared__ unsigned long long sh[5][kSlots / 32];
  const Accum a = c->acc[threadIdx.x];
  unsigned long long v[4] = {static_cast<unsigned long long>(a.delta), a.frontier, a.survivors, a.count};
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = warp_sum(v[k]);
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int k = 0; k < 4; ++k) sh[k][threadIdx.x >> 5] = v[k];
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t[4] = {0, 0, 0, 0};
    for (int k = 0; k < 4; ++k)
      for (int w = 0; w < kSlots / 32; ++w) t[k] += sh[k][w];
    h.count[0] = t[0];
    h.count[1] = t[1] + c->frontier;
    h.count[2] = t[2];
    h.count[3] = (globaltimer_ns() - c->t0_ns >= c->vote_limit_ns) ? 1ull : 0ull;
    h.count[4] = t[3];
  }
}

// <<<1, kSlots>>>
// ext (row-band partition): {global unconverged count, time-limit votes},
// all-reduced over the ranks, replaces the local count and the local clock so
// every rank takes the same stop decision.
// finalize_block: the same by one whole block of any size >= kSlots (a
// multiple of 32), inside the persistent loop kernels.
__device__ __forceinline__ void finalize_block(Ctl* c, int mode, uint32_t D, const unsigned long long* ext = nullptr) {
  if (run_done(c)) return;
  const int t = threadIdx.x;
  // band RnBP under a polling host: an empty attempt-0 frontier with survivors
  // (the GLOBAL sums) leaves the iteration open -- slots and state untouched --
  // until the host runs the retry / single-survivor fallback (schedulers.cpp:204-214)
  if (mode == kFinIterExt && ext && c->band_poll && ext[1] == 0ull && ext[2] > 0ull) {
    if (t == 0) c->band_wait = 1u;
    return;
  }
  // thread 0's control-block loads are issued with the slot loads
  FinRegs f;
  if (t == 0) f.load(c);
  const Accum a = t < kSlots ? c->acc[t] : Accum{};
  if (t < kSlots) c->acc[t] = Accum{};
  __shared__ unsigned long long sh[6][32];
  unsigned long long v[6] = {static_cast<unsigned long long>(a.delta), a.count, a.frontier, a.survivors,
                             a.evals, a.visits};
#pragma unroll
  for (int k = 0; k < 6; ++k) v[k] = warp_sum(v[k]);
  if ((t & 31) == 0)
#pragma unroll
    for (int k = 0; k < 6; ++k) sh[k][t >> 5] = v[k];
  __syncthreads();
  if (t != 0) return;
  for (int k = 0; k < 6; ++k) {
    v[k] = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) v[k] += sh[k][w];
  }
  const bool rnbp_ext = mode == kFinInitExt || mode == kFinIterExt;
  const long long delta = static_cast<long long>(rnbp_ext ? ext[0] : v[0]);
  const unsigned long long count = ext ? (rnbp_ext ? ext[4] : ext[0]) : v[1];
  const unsigned long long frontier = rnbp_ext ? ext[1] : v[2] + f.frontier;
  if (ext && ext[rnbp_ext ? 3 : 1]) f.time_limit_ns = 0;  // some rank hit the time limit: stop everywhere
  f.evals_total += v[4];
  f.vertex_visits += v[5];
  switch (mode) {
    case kFinLbp: {  // sweep s computed r(m_s): it closes iteration s-1
      const unsigned long long s = f.sweeps;
      if (s > 0) {
        fin_record(f, c->trace, s - 1, D, static_cast<unsigned>(count));
        f.msgs_total += D;
      }
      f.iteration = s;
      f.unconverged = static_cast<unsigned>(count);
      f.sweeps = s + 1;
      fin_reset_scratch(f);
      fin_check_top(f);
      break;
    }
    case kFinInit:
    case kFinInitExt:
      f.unconverged = static_cast<unsigned>(count);
      f.iteration = 0;
      if (f.use_clist && 16ull * f.unconverged < D) f.cl_state = 1u;
      fin_reset_scratch(f);
      fin_check_top(f);
      break;
    case kFinIter:
    case kFinIterExt:
      fin_iter(f, c->trace, delta, frontier, D);
      break;
    case kFinApply:
      f.unconverged = static_cast<unsigned>(static_cast<long long>(f.unconverged) + delta);
      fin_reset_scratch(f);
      break;
    case kFinFused:  // one fused RnBP sweep wrote the other buffer set
      f.fused_par ^= 1u;
      if (frontier == 0 && v[3] > 0)
        f.fused_abort = 1u;  // empty attempt-0 frontier: nothing changed, the retry path redoes the iteration
      else
        fin_iter(f, c->trace, delta, frontier, D);
      break;
    default:
      break;
  }
  // the graph loop also hands RnBP list mode over to the persistent kernel
  const bool handover = f.persist_ok && f.cl_state == 2u;
  if (handover && !f.handover_it) f.handover_it = f.iteration;
  f.store(c);
  const bool stop = f.done || handover || (mode == kFinFused && (f.fused_abort || f.cl_state != 0u));
  if (f.cond_handle && mode != kFinApply)
    cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(f.cond_handle), stop ? 0u : 1u);
}

static __global__ void __launch_bounds__(kSlots) k_finalize(Ctl* c, int mode, uint32_t D,
                                                          const unsigned long long* ext = nullptr) {
  finalize_block(c, mode, D, ext);
}

// Kernel-fused loop control: the LAST block of a launch to finish runs the
// finalize (or the RnBP retry) itself, so an iteration needs no extra
// one-block launch.  threadFenceReduction pattern: the warp that issued the
// block's slot atomics fences them before the block counts itself done, and
// the block that takes the last count fences again before reading the slots.
__device__ __forceinline__ bool last_block_done(Ctl* c) {
  __shared__ unsigned s_last;
  // the slot atomics of block_accumulate are issued by warp 0
  if (threadIdx.x < 32) __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&c->blocks_done, 1u) == gridDim.x - 1u ? 1u : 0u;
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  if (threadIdx.x == 0) c->blocks_done = 0u;  // for the next launch (stream-ordered)
  return true;
}

struct FinArgs {
  int mode;    // kFinNone: no fused finalize
  uint32_t D;  // directed edges counted by the finalize
  int gate;    // 1: the launch refreshes only in RnBP list mode (k_lattice_qsweep refreshes the other iterations)
};

__device__ __forceinline__ void fused_finalize(Ctl* c, const FinArgs& f) {
  if (f.mode != kFinNone && last_block_done(c)) finalize_block(c, f.mode, f.D);
}

// ---------------------------------------------------------------------------
// vertex-centric sum-product update.  One thread owns vertex v: it reads every
// incoming message of v once (edge pair loads), forms the vertex total in log
// space, and for each incoming edge `in` produces the outgoing message
// out = in ^ 1 from the cavity (total minus the message on `in`).  This is
// refresh_residuals over the outgoing edges of v: each message is read once
// per vertex and written once, instead of deg times as in the edge-parallel
// reference loop.

// CL: candidate-list maintenance (RnBP): an outgoing edge whose residual is
// >= eps and that is not in the list yet is pushed to `cl`.
// ldm<NC>: read-only-path load (__ldg) inside normal kernels; a plain
// coherent load inside persistent kernels, where the data changes between
// grid barriers of the same launch.
template <bool NC, class T>
__device__ __forceinline__ T ldm(const T* p) {
  if constexpr (NC) return __ldg(p);
  else return *p;
}

template <int MODE, bool CL, bool NC = true>
__device__ __forceinline__ int vertex_update_binary(const DevGraph& g, uint32_t v,
                                                    const float* __restrict__ A,
                                                    float* __restrict__ B, float* __restrict__ res,
                                                    float eps, unsigned* numeric_flag,
                                                    unsigned long long& evals, uint8_t* inlist,
                                                    Stager* cl, bool cl_on, const uint32_t* cstamp = nullptr,
                                                    uint32_t stamp = 0u, uint32_t via = 0u,
                                                    bool* skipped = nullptr) {
  // cstamp (persistent tail, lattice): v was reached through committed edge
  // `via`; the vertex is refreshed by the thread of its LOWEST committed
  // incoming edge (cstamp == stamp) only, so duplicate targets need no
  // atomic dedupe -- the stamps are loaded with the messages
  float T = g.unary_lo[v];
  const float2* __restrict__ A2 = reinterpret_cast<const float2*>(A);
  // incoming messages and (same edge pair) the old outgoing ones, kept in
  // registers between the two passes (lattice: exactly 4; CSR: re-read in
  // groups of 4)
  int cnt = 0;
  uint32_t deg = 0;
  // emit with prefetched residual / in-list flag
  auto emit_pre = [&](uint32_t in, float2 pr, float r_was, bool in_list, float a) {
    const uint32_t out = in ^ 1u;
    const float m_in = (in & 1u) ? pr.y : pr.x;
    const float m_old = (in & 1u) ? pr.x : pr.y;
    float lnew, r;
    if (g.par_mode) {
      r = ising_update(T - m_in, a, m_old, lnew);
    } else {
      lnew = binary_msg(g, T - m_in, out);
      r = binary_residual(lnew, m_old);
    }
    if (!(fabsf(lnew) < INFINITY)) *numeric_flag = 1u;
    B[out] = lnew;
    const int now = r >= eps;
    if (MODE == kModeDelta) {
      cnt += now - (r_was >= eps);
      res[out] = r;
    } else {
      if (MODE == kModeInit) res[out] = r;
      cnt += now;
    }
    if (CL && cl_on && now && !in_list) {
      inlist[out] = 1;
      cl->push(out);
    }
  };
  if (g.lat_cols) {
    // fixed neighbour slots (up, left, right, down): statically indexed, so
    // everything stays in registers (a compacted list would live in local memory)
    const uint32_t C = g.lat_cols, R = g.lat_rows;
    const uint32_t r = v / C, c = v - r * C;
    const uint32_t row = r * (2u * C - 1u);
    const bool last = r + 1u == R;
    const bool has[4] = {r > 0u, c > 0u, c + 1u < C, !last};
    const uint32_t ins[4] = {
        has[0] ? 2u * ((r - 1u) * (2u * C - 1u) + 2u * c + (c + 1u < C ? 1u : 0u)) : 0u,
        has[1] ? 2u * (last ? row + c - 1u : row + 2u * (c - 1u)) : 0u,
        has[2] ? 2u * (last ? row + c : row + 2u * c) + 1u : 0u,
        has[3] ? 2u * (row + 2u * c + (c + 1u < C ? 1u : 0u)) + 1u : 0u};
    float2 prs[4];
    float rw[4], ia[4];
    bool il[4];
    uint32_t cs[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      cs[k] = (cstamp && has[k]) ? cstamp[ins[k]] : 0u;
      prs[k] = has[k] ? ldm<NC>(&A2[ins[k] >> 1]) : make_float2(0.f, 0.f);
      ia[k] = (g.par_mode && has[k]) ? __ldg(&g.ising_a[ins[k] >> 1]) : 0.f;  // with the pair loads
      // prefetch the per-message state so the four updates do not serialise
      // on (possibly aliasing) loads between their stores
      rw[k] = (MODE == kModeDelta && has[k]) ? res[ins[k] ^ 1u] : 0.f;
      il[k] = (CL && cl_on && has[k]) ? inlist[ins[k] ^ 1u] != 0 : true;
    }
    if (cstamp) {
      uint32_t owner = 0xffffffffu;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (has[k] && cs[k] == stamp) owner = min(owner, ins[k]);
      if (owner != via) {
        *skipped = true;
        return 0;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) T += has[k] ? ((ins[k] & 1u) ? prs[k].y : prs[k].x) : 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (has[k]) {
        emit_pre(ins[k], prs[k], rw[k], il[k], ia[k]);
        ++deg;
      }
  } else {
    const uint32_t b = g.in_off[v], e = g.in_off[v + 1];
    for (uint32_t a = b; a < e; ++a) {
      const uint32_t in = g.in_adj[a];
      const float2 pr = ldm<NC>(&A2[in >> 1]);
      T += (in & 1u) ? pr.y : pr.x;
    }
    deg = e - b;
    // emit in groups of 4 with the per-message state prefetched, so the
    // updates do not serialise on loads behind the previous group's stores
    for (uint32_t a0 = b; a0 < e; a0 += 4) {
      uint32_t ins[4];
      float2 prs[4];
      float rw[4], ia[4];
      bool il[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool has = a0 + k < e;
        ins[k] = has ? g.in_adj[a0 + k] : 0u;
        prs[k] = has ? ldm<NC>(&A2[ins[k] >> 1]) : make_float2(0.f, 0.f);
        rw[k] = (MODE == kModeDelta && has) ? res[ins[k] ^ 1u] : 0.f;
        il[k] = (CL && cl_on && has) ? inlist[ins[k] ^ 1u] != 0 : true;
        ia[k] = (g.par_mode && has) ? __ldg(&g.ising_a[ins[k] >> 1]) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (a0 + k < e) emit_pre(ins[k], prs[k], rw[k], il[k], ia[k]);
    }
  }
  evals += deg;
  return cnt;
}

template <int QS, int MODE, bool CL, bool NC = true>
__device__ __forceinline__ int vertex_update_generic(const DevGraph& g, uint32_t v,
                                                     const float* __restrict__ A,
                                                     float* __restrict__ B, float* __restrict__ res,
                                                     float eps, unsigned* numeric_flag,
                                                     unsigned long long& evals, uint8_t* inlist,
                                                     Stager* cl, bool cl_on) {
  const uint32_t ci = g.card[v];
  float T[QS];
#pragma unroll (QS <= 8 ? QS : 2)
  for (int x = 0; x < QS; ++x) T[x] = g.unary_log[static_cast<size_t>(v) * QS + x];
  auto load_q = [&](uint32_t d, float* m) {  // a q-vector with 16-byte loads (QS % 4 == 0)
    const float4* m4 = reinterpret_cast<const float4*>(A + static_cast<size_t>(d) * QS);
#pragma unroll (QS <= 8 ? QS / 4 : 1)
    for (int x4 = 0; x4 < QS / 4; ++x4) {
      const float4 q4 = ldm<NC>(&m4[x4]);
      m[4 * x4] = q4.x;
      m[4 * x4 + 1] = q4.y;
      m[4 * x4 + 2] = q4.z;
      m[4 * x4 + 3] = q4.w;
    }
  };
  int cnt = 0;
  // one outgoing message from the incoming q-vector mi (same edge pair) and
  // the old outgoing one mo
  auto emit = [&](uint32_t in, const float* mi, const float* mo, float r_was) {
    const uint32_t out = in ^ 1u;
    const uint32_t cj = g.uniform_q ? g.uniform_q : g.card[g.ep[in]];  // target of `out` = source of `in`
    float p[QS];
    float M = -INFINITY;
#pragma unroll (QS <= 8 ? QS : 2)
    for (int x = 0; x < QS; ++x) {
      p[x] = T[x] - mi[x];
      if (x < static_cast<int>(ci)) M = fmaxf(M, p[x]);
    }
    float o[QS], s, inv;
    if (g.log_tables) {  // collapse-checked model: log-domain contraction (o = log2 message), exact mass
      const float lm = generic_logmatvec<QS>(g, out, p, ci, cj, o);
      if (!(lm >= kLog2MinMass)) *numeric_flag = 1u;
      s = 1.f;
      inv = 1.f;
    } else {
#pragma unroll (QS <= 8 ? QS : 2)
      for (int x = 0; x < QS; ++x) p[x] = x < static_cast<int>(ci) ? fex2(p[x] - M) : 0.f;
      generic_matvec<QS>(g, out, p, o);
      s = 0.f;
#pragma unroll (QS <= 8 ? QS : 2)
      for (int xt = 0; xt < QS; ++xt) s += xt < static_cast<int>(cj) ? o[xt] : 0.f;
      inv = frcp(s);
    }
    float r = 0.f;
    // the residual compares 2^(stored log) on both sides, so a bitwise fixed
    // point reports exactly 0 (as for the binary layout); states >= cj keep
    // their stored value, so the q-vector leaves with 16-byte stores
#pragma unroll (QS <= 8 ? QS : 2)
    for (int xt = 0; xt < QS; ++xt) {
      if (xt < static_cast<int>(cj)) {
        const float ln = g.log_tables ? o[xt] : flg2(o[xt] * inv);
        r = fmaxf(r, fabsf(fex2(ln) - fex2(mo[xt])));
        o[xt] = ln;
      } else {
        o[xt] = mo[xt];
      }
    }
    float4* dst4 = reinterpret_cast<float4*>(B + static_cast<size_t>(out) * QS);
#pragma unroll (QS <= 8 ? QS / 4 : 1)
    for (int x4 = 0; x4 < QS / 4; ++x4)
      dst4[x4] = make_float4(o[4 * x4], o[4 * x4 + 1], o[4 * x4 + 2], o[4 * x4 + 3]);
    if (!(s > 0.f) || !(s < INFINITY)) *numeric_flag = 1u;
    const int now = r >= eps;
    if (MODE == kModeDelta) {
      cnt += now - (r_was >= eps);
      res[out] = r;
    } else {
      if (MODE == kModeInit) res[out] = r;
      cnt += now;
    }
    if (CL && cl_on && now && !inlist[out]) {
      inlist[out] = 1;
      cl->push(out);
    }
  };
  uint32_t deg = 0;
  if (MODE == kModeCount && QS <= 8 && g.lat_cols) {
    // LBP sweep on a lattice, q <= 8: the (at most 4) incoming and old outgoing
    // q-vectors are loaded at once and kept in registers for both passes
    const uint32_t C = g.lat_cols, R = g.lat_rows;
    const uint32_t r = v / C, c = v - r * C;
    const uint32_t row = r * (2u * C - 1u);
    const bool last = r + 1u == R;
    const bool has[4] = {r > 0u, c > 0u, c + 1u < C, !last};
    const uint32_t ins[4] = {
        has[0] ? 2u * ((r - 1u) * (2u * C - 1u) + 2u * c + (c + 1u < C ? 1u : 0u)) : 0u,
        has[1] ? 2u * (last ? row + c - 1u : row + 2u * (c - 1u)) : 0u,
        has[2] ? 2u * (last ? row + c : row + 2u * c) + 1u : 0u,
        has[3] ? 2u * (row + 2u * c + (c + 1u < C ? 1u : 0u)) + 1u : 0u};
    float mi[4][QS], mo[4][QS];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (has[k]) {
        load_q(ins[k], mi[k]);
        load_q(ins[k] ^ 1u, mo[k]);
      }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (has[k]) {
#pragma unroll
        for (int x = 0; x < QS; ++x) T[x] += mi[k][x];
        ++deg;
      }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (has[k]) emit(ins[k], mi[k], mo[k], 0.f);
  } else {
    for_each_in(g, v, [&](uint32_t in) {
      float mi[QS];
      load_q(in, mi);
#pragma unroll (QS <= 8 ? QS : 2)
      for (int x = 0; x < QS; ++x) T[x] += mi[x];
      ++deg;
    });
    for_each_in(g, v, [&](uint32_t in) {
      const float r_was = MODE == kModeDelta ? res[in ^ 1u] : 0.f;
      float mi[QS], mo[QS];
      load_q(in, mi);
      load_q(in ^ 1u, mo);
      emit(in, mi, mo, r_was);
    });
  }
  evals += deg;
  return cnt;
}

// Dense sweep over a binary Ising lattice (par_mode 1, lat_cols > 0): the
// HBM-bound LBP kernel.  A tile is kLatVPT * kBlock consecutive vertices of
// one row; thread t owns columns t, t + kBlock, ... so every load instruction
// of a warp touches one contiguous span.  Each vertex needs its own (right,
// down) edge pairs, the left neighbour's right pair and the upper neighbour's
// down pair (L1 / L2 hits), the four a = e^J and its unary: all kLatVPT x 9
// loads are issued before any arithmetic.  check_flag: dense touched-set
// refresh (only vertices with vflag == stamp).
constexpr int kLatVPT = 1;  // measured at 1000^2: 4 -> 2 -> 1 vertices per thread, 23.0 -> 22.5 -> 22.4 us per LBP iteration
constexpr uint32_t kLatTile = kBlock * kLatVPT;

template <int MODE, bool CL, int VPT = kLatVPT, bool NC = true>
__device__ __forceinline__ void lattice_binary_tiles(const DevGraph& g, const float* __restrict__ A,
                                                     float* __restrict__ B, float* __restrict__ res,
                                                     const uint32_t* __restrict__ vflag, uint32_t stamp,
                                                     bool check_flag, float eps, unsigned* nf, int& cnt,
                                                     unsigned long long& evals, unsigned long long& visits,
                                                     uint8_t* inlist, Stager* cl, bool cl_on) {
  const uint32_t C = g.lat_cols, R = g.lat_rows;
  const uint32_t tpr = (C + (kBlock * VPT) - 1) / (kBlock * VPT);
  const uint64_t ntiles = static_cast<uint64_t>(R) * tpr;
  const float2* __restrict__ A2 = reinterpret_cast<const float2*>(A);
  const float* __restrict__ ea = g.ising_a;
  bool bad = false;
  // Each block walks a contiguous run of tiles in (column strip, row) order:
  // down the rows of one (kBlock * VPT)-wide strip, so the upper neighbour's edge
  // pairs were read by this block one tile ago and the message sectors it
  // half-writes are completed by its next tile -- the live working set is
  // ~2 rows x strip x blocks (L2-resident even at 16384^2).
  const uint64_t t_begin = ntiles * blockIdx.x / gridDim.x, t_end = ntiles * (blockIdx.x + 1) / gridDim.x;
  for (uint64_t t = t_begin; t < t_end; ++t) {
    const uint32_t strip = static_cast<uint32_t>(t / R);
    const uint32_t r = static_cast<uint32_t>(t - static_cast<uint64_t>(strip) * R);
    const uint32_t c0 = strip * (kBlock * VPT) + threadIdx.x;
    const bool last = r + 1u == R, first = r == 0u;
    const uint32_t row = r * (2u * C - 1u), prow = first ? 0u : (r - 1u) * (2u * C - 1u);
    bool act[VPT];
    float2 pU[VPT], pL[VPT], pR[VPT], pD[VPT];
    float aU[VPT], aL[VPT], aR[VPT], aD[VPT], un[VPT];
    // per vertex, prefetched with the messages: bit j = old residual of out
    // message j (up, left, right, down) >= eps, bit 4 + j = it is in the
    // candidate list; the bookkeeping below then needs no dependent loads
    uint32_t pre[VPT];
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const uint32_t c = c0 + k * kBlock;
      act[k] = c < C;
      if (check_flag && act[k]) act[k] = vflag[r * C + c] == stamp;
    }
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const uint32_t c = c0 + k * kBlock;
      pU[k] = pL[k] = pR[k] = pD[k] = make_float2(0.f, 0.f);
      aU[k] = aL[k] = aR[k] = aD[k] = 1.f;
      un[k] = 0.f;
      if (!act[k]) continue;
      const uint32_t dn = c + 1u < C ? 1u : 0u;
      if (!first) {
        const uint32_t e = prow + 2u * c + dn;
        pU[k] = ldm<NC>(&A2[e]);
        aU[k] = __ldg(&ea[e]);
      }
      if (c > 0u) {
        const uint32_t e = last ? row + c - 1u : row + 2u * c - 2u;
        pL[k] = ldm<NC>(&A2[e]);
        aL[k] = __ldg(&ea[e]);
      }
      if (dn) {
        const uint32_t e = last ? row + c : row + 2u * c;
        pR[k] = ldm<NC>(&A2[e]);
        aR[k] = __ldg(&ea[e]);
      }
      if (!last) {
        const uint32_t e = row + 2u * c + dn;
        pD[k] = ldm<NC>(&A2[e]);
        aD[k] = __ldg(&ea[e]);
      }
      un[k] = __ldg(&g.unary_lo[r * C + c]);
    }
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      pre[k] = 0u;
      if (MODE != kModeDelta && !(CL && cl_on)) continue;
      const uint32_t c = c0 + k * kBlock;
      const uint32_t dn = c + 1u < C ? 1u : 0u;
      const bool has[4] = {act[k] && !first, act[k] && c > 0u, act[k] && dn, act[k] && !last};
      const uint32_t outs[4] = {2u * (prow + 2u * c + dn) + 1u, 2u * (last ? row + c - 1u : row + 2u * c - 2u) + 1u,
                                2u * (last ? row + c : row + 2u * c), 2u * (row + 2u * c + dn)};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (!has[j]) continue;
        if (MODE == kModeDelta && res[outs[j]] >= eps) pre[k] |= 1u << j;
        if (CL && cl_on && inlist[outs[j]]) pre[k] |= 16u << j;
      }
    }
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      if (CL) cl->flush(1024);  // <= 4 kBlock pushes per k
      const uint32_t c = c0 + k * kBlock;
      const uint32_t dn = c + 1u < C ? 1u : 0u;
      const bool hu = act[k] && !first, hl = act[k] && c > 0u, hr = act[k] && dn, hd = act[k] && !last;
      const bool owned = r >= g.cnt_row0 && r < g.cnt_row1;  // ghost rows of a band: computed, not counted
      // incoming: up (2eU, .x), left (2eL, .x), right (2eR+1, .y), down (2eD+1, .y); absent ones hold 0
      const float T = un[k] + pU[k].x + pL[k].x + pR[k].y + pD[k].y;
      // all four messages are computed (predicated stores, no divergence at the borders)
      float lu, ll, lr, ld;
      const float ru = ising_update(T - pU[k].x, aU[k], pU[k].y, lu);
      const float rl = ising_update(T - pL[k].x, aL[k], pL[k].y, ll);
      const float rr = ising_update(T - pR[k].y, aR[k], pR[k].x, lr);
      const float rd = ising_update(T - pD[k].y, aD[k], pD[k].x, ld);
      const uint32_t ou = 2u * (prow + 2u * c + dn) + 1u;
      const uint32_t ol = 2u * (last ? row + c - 1u : row + 2u * c - 2u) + 1u;
      const uint32_t orr = 2u * (last ? row + c : row + 2u * c);
      const uint32_t od = 2u * (row + 2u * c + dn);
      bad |= (hu && !(fabsf(lu) < INFINITY)) || (hl && !(fabsf(ll) < INFINITY)) ||
             (hr && !(fabsf(lr) < INFINITY)) || (hd && !(fabsf(ld) < INFINITY));
      if (hu) B[ou] = lu;
      if (hl) B[ol] = ll;
      if (hr) B[orr] = lr;
      if (hd) B[od] = ld;
      auto track = [&](int j, bool has, uint32_t out, float r_msg) {
        // messages of a band's ghost rows belong to the neighbour band: their
        // residuals stay 0 here, so they are never counted or selected
        const int now = has && owned && r_msg >= eps;
        if (MODE == kModeDelta) {
          if (has && owned) {
            cnt += now - static_cast<int>((pre[k] >> j) & 1u);
            res[out] = r_msg;
          }
        } else {
          if (MODE == kModeInit && has && owned) res[out] = r_msg;
          cnt += now;
        }
        if (CL && cl_on && now && !((pre[k] >> (4 + j)) & 1u)) {
          inlist[out] = 1;
          cl->push(out);
        }
      };
      track(0, hu, ou, ru);
      track(1, hl, ol, rl);
      track(2, hr, orr, rr);
      track(3, hd, od, rd);
      const uint32_t deg = (hu ? 1u : 0u) + (hl ? 1u : 0u) + (hr ? 1u : 0u) + (hd ? 1u : 0u);
      evals += owned ? deg : 0u;
      visits += act[k] && owned ? 1u : 0u;
    }
  }
  if (bad) *nf = 1u;
}

// QS == 1 selects the binary layout.
template <int QS, int MODE, bool CL, bool NC = true>
__device__ __forceinline__ int vertex_update(const DevGraph& g, uint32_t v, const float* A, float* B,
                                             float* res, float eps, unsigned* nf,
                                             unsigned long long& evals, uint8_t* inlist, Stager* cl,
                                             bool cl_on, const uint32_t* cstamp = nullptr, uint32_t stamp = 0u,
                                             uint32_t via = 0u, bool* skipped = nullptr) {
  if constexpr (QS == 1)
    return vertex_update_binary<MODE, CL, NC>(g, v, A, B, res, eps, nf, evals, inlist, cl, cl_on, cstamp, stamp, via,
                                              skipped);
  else
    return vertex_update_generic<QS, MODE, CL, NC>(g, v, A, B, res, eps, nf, evals, inlist, cl, cl_on);
}

// Sweep over all vertices (LIST = false) or over the vertices flagged this
// iteration (collect_touched): sparse iterations walk vlist, dense ones scan
// vflag in vertex order so the accesses stay coalesced.
// For the LBP sweep the source/destination buffers alternate with the sweep
// index held on the device (A = buf[s & 1], B = buf[(s + 1) & 1]).
// CL: maintain the RnBP candidate list (init appends to list cl_cur, the
// refresh to list cl_cur ^ 1, which the select of this iteration is filling).
constexpr uint32_t kSlotEmpty = 0xffffffffu;  // hole of a slot list (persistent tail)

struct CandList {
  uint32_t* list[2];
  uint8_t* inlist;
};

// One pass of the vertex update over the grid (every block of the launch
// calls it): the body of k_vertex_update, also run inside the persistent loop
// kernels (NC = false: messages change inside the launch, so they are read
// with coherent loads).
template <int QS, int MODE, bool LIST, bool PINGPONG, bool CL, bool NC = true>
__device__ __forceinline__ void vertex_update_pass(const DevGraph& g, const float* A0, float* B0, float* res,
                                                   const uint32_t* vlist, const uint32_t* vflag, Ctl* ctl,
                                                   float eps, const CandList& cand_list) {
  const float* A = A0;
  float* B = B0;
  if (PINGPONG) {
    if (ctl->sweeps & 1ull) {
      A = B0;
      B = const_cast<float*>(A0);
    }
  }
  const bool dense = !LIST || ctl->dense;
  const uint32_t n = dense ? g.V : ctl->nflag;
  const uint32_t stamp = LIST ? ctl->stamp : 0u;
  const unsigned tgt_list = CL ? (MODE == kModeInit ? ctl->cl_cur : ctl->cl_cur ^ 1u) : 0u;
  BPB_STAGER(cl, CL ? 2048 : 1, CL ? (tgt_list ? cand_list.list[1] : cand_list.list[0]) : nullptr, &ctl->cl_n[tgt_list]);
  if (CL) cl.init();
  int cnt = 0;
  unsigned long long evals = 0, visits = 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  // candidate list maintained once the RnBP run is in list mode (cl_state >= 1)
  const bool cl_on = CL && ctl->cl_state >= 1u;
  const bool lattice = QS == 1 && g.lat_cols != 0u && g.par_mode != 0u && dense;
  if (lattice)
    // one vertex per thread: more warps in flight (the delta-mode refresh
    // measured 63 -> 56 us per early RnBP iteration going from 2 to 1)
    lattice_binary_tiles<MODE, CL, kLatVPT, NC>(g, A, B, res, vflag, stamp, LIST, eps, &ctl->numeric_error, cnt, evals,
                                               visits, cand_list.inlist, &cl, cl_on);
  for (uint32_t base = lattice ? n : blockIdx.x * blockDim.x; base < n; base += stride) {
    const uint32_t i = base + threadIdx.x;
    if (i < n) {
      uint32_t v = i;
      bool go = true;
      if (LIST) {
        if (dense)
          go = vflag[i] == stamp;
        else
          v = vlist[i];
      }
      if (go && g.lat_cols && (g.cnt_row0 > 0u || g.cnt_row1 < g.lat_rows)) {  // band: owned rows only
        const uint32_t row = v / g.lat_cols;
        go = row >= g.cnt_row0 && row < g.cnt_row1;
      }
      go = go && v < g.own_v;  // vertex-range partition: ghosts' messages come from their owners
      if (go) {
        cnt += vertex_update<QS, MODE, CL, NC>(g, v, A, B, res, eps, &ctl->numeric_error, evals, cand_list.inlist,
                                               &cl, cl_on);
        ++visits;
      }
    }
    if (CL) cl.flush(1024);
  }
  if (CL) cl.flush(0);
  Contrib c;
  if (MODE == kModeDelta)
    c.delta = cnt;
  else
    c.count = static_cast<unsigned long long>(cnt);
  c.evals = evals;
  c.visits = visits;
  block_accumulate(ctl, c);
}

// fin: the loop control of the iteration, run by the last block (FinArgs)
template <int QS, int MODE, bool LIST, bool PINGPONG, bool CL>
__global__ void __launch_bounds__(kBlock) k_vertex_update(DevGraph g, const float* A0, float* B0,
                                                          float* res, const uint32_t* vlist,
                                                          const uint32_t* vflag, Ctl* ctl, float eps,
                                                          CandList cand_list, FinArgs fin) {
  if (run_done(ctl)) return;
  // gated (after k_lattice_qsweep's refresh): outside list mode the lanes
  // kernel refreshed this iteration, so only the loop control runs here --
  // the iteration's ONE finalize, after both launches (a finalize in the lanes
  // kernel could enter list mode mid-iteration and make this launch refresh
  // and finalize the same iteration a second time)
  if (!(fin.gate && ctl->cl_state < 1u))
    vertex_update_pass<QS, MODE, LIST, PINGPONG, CL>(g, A0, B0, res, vlist, vflag, ctl, eps, cand_list);
  fused_finalize(ctl, fin);
}

// ---------------------------------------------------------------------------
// LBP sweep over a q-state lattice, FOUR STATES PER LANE: a group of QS / 4
// lanes owns one vertex (q = 8: a lane pair), lane l holds states
// [4l, 4l + 4) of every q-vector, so each q-vector moves as one 16-byte access
// per lane (a 32-byte sector per pair) and a reduction over the states is
// three in-register steps plus log2(QS / 4) xor-shuffles (one lane per state
// needed three shuffles per reduction, ~12 per message: the sweep was
// instruction-bound at 1.96G warp instructions per 4096^2 sweep; a thread per
// vertex holding 8 in + 8 out vectors needs ~128 registers: latency-bound).
// Same arithmetic as vertex_update_generic (kModeCount): m_{t+1} = f(m_t) into
// B, count r(m_t) >= eps; the finalize of the iteration runs in the last block.
// POTTS: Potts tables (par_mode 1, the O(q) contraction); else dense tables.
// MODE kModeCount: the LBP sweep (ping-pong buffers, count r >= eps).
// MODE kModeDelta: refresh_residuals of the touched vertices (flagged in
// vflag, or listed in vlist on sparse iterations) outside RnBP list mode:
// candidates into B, residuals r / res[out] and the unconverged delta, as
// vertex_update_generic<kModeDelta> (list mode runs that kernel, gated).
template <int QS, bool POTTS, int MODE>
__global__ void __launch_bounds__(kBlock) k_lattice_qsweep(DevGraph g, const float* A0, float* B0, float* res,
                                                           const uint32_t* vlist, const uint32_t* vflag, Ctl* ctl,
                                                           float eps, FinArgs fin) {
  static_assert(QS == 4 || QS == 8, "four states per lane: QS = 4 or 8");
  static_assert(MODE == kModeCount || MODE == kModeDelta || MODE == kModeInit, "sweep, touched refresh or init");
  constexpr int SPL = 4, LPV = QS / SPL;  // states per lane, lanes per vertex
  if (run_done(ctl)) return;
  if (MODE == kModeDelta && ctl->cl_state >= 1u) return;  // list mode: the gated vertex kernel
  const float* A = A0;
  float* B = B0;
  if (MODE == kModeCount && (ctl->sweeps & 1ull)) {
    A = B0;
    B = const_cast<float*>(A0);
  }
  const bool dense_items = MODE != kModeDelta || ctl->dense != 0u;
  const uint32_t stamp = ctl->stamp;
  const uint32_t C = g.lat_cols, R = g.lat_rows, q = g.uniform_q;
  const int l = static_cast<int>(threadIdx.x % LPV);
  const int x0 = l * SPL;
  bool live_state[SPL];
#pragma unroll
  for (int j = 0; j < SPL; ++j) live_state[j] = x0 + j < static_cast<int>(q);
  auto gmax = [](float v) {
#pragma unroll
    for (int o = LPV / 2; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
  };
  auto gsum = [](float v) {
#pragma unroll
    for (int o = LPV / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
  };
  auto ld4 = [](const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); };
  int cnt = 0;
  unsigned long long evals = 0, visits = 0;
  bool bad = false;
  const uint64_t groups = static_cast<uint64_t>(gridDim.x) * (blockDim.x / LPV);
  const uint64_t V = dense_items ? g.V : ctl->nflag;  // items: vertices, or the touched list
  // every lane of the warp runs every trip (the shuffles need all of them)
  const uint64_t trips = (V + groups - 1) / groups;
  const uint64_t item0 = static_cast<uint64_t>(blockIdx.x) * (blockDim.x / LPV) + threadIdx.x / LPV;
  // refresh: the touched flag (dense) or list entry (sparse) of the NEXT
  // trip is loaded one trip ahead, so a trip's message loads do not wait
  // behind a flag round trip (k_rnbp_select wrote both in the previous launch)
  auto item_word = [&](uint64_t vv) -> uint32_t {
    if (MODE != kModeDelta || vv >= V) return 0u;
    return dense_items ? __ldg(&vflag[vv]) : __ldg(&vlist[vv]);
  };
  uint32_t next_word = item_word(item0);
  for (uint64_t t = 0; t < trips; ++t) {
    const uint64_t vv = t * groups + item0;
    bool act = vv < V;
    uint32_t v = act ? static_cast<uint32_t>(vv) : 0u;
    const uint32_t word = next_word;
    if (MODE == kModeDelta) next_word = item_word(vv + groups);
    if (MODE == kModeDelta && act) {
      if (dense_items)
        act = word == stamp;
      else
        v = word;
    }
    if (!act) v = 0u;
    const uint32_t r = v / C, c = v - r * C;
    const uint32_t row = r * (2u * C - 1u);
    const bool last = r + 1u == R;
    const bool has[4] = {act && r > 0u, act && c > 0u, act && c + 1u < C, act && !last};
    const uint32_t ins[4] = {
        has[0] ? 2u * ((r - 1u) * (2u * C - 1u) + 2u * c + (c + 1u < C ? 1u : 0u)) : 0u,
        has[1] ? 2u * (last ? row + c - 1u : row + 2u * (c - 1u)) : 0u,
        has[2] ? 2u * (last ? row + c : row + 2u * c) + 1u : 0u,
        has[3] ? 2u * (row + 2u * c + (c + 1u < C ? 1u : 0u)) + 1u : 0u};
    float4 mi[4], mo[4];
    float w[4];
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 T4 = act ? ld4(&g.unary_log[static_cast<size_t>(v) * QS + x0]) : z4;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      mi[k] = has[k] ? ld4(&A[static_cast<size_t>(ins[k]) * QS + x0]) : z4;
      mo[k] = has[k] ? ld4(&A[static_cast<size_t>(ins[k] ^ 1u) * QS + x0]) : z4;
      w[k] = has[k] && POTTS ? __ldg(&g.pw[ins[k] >> 1]) : 0.f;
    }
    // old residuals of the outgoing messages (refresh), issued with the
    // message loads: a load after this thread's stores would wait in line
    bool was[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) was[k] = MODE == kModeDelta && l == 0 && has[k] && res[ins[k] ^ 1u] >= eps;
    float T[SPL] = {T4.x, T4.y, T4.z, T4.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      T[0] += mi[k].x;
      T[1] += mi[k].y;
      T[2] += mi[k].z;
      T[3] += mi[k].w;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t out = ins[k] ^ 1u;
      const float mik[SPL] = {mi[k].x, mi[k].y, mi[k].z, mi[k].w};
      const float mok[SPL] = {mo[k].x, mo[k].y, mo[k].z, mo[k].w};
      float pl[SPL], e[SPL], o[SPL];
      float M = -INFINITY;
#pragma unroll
      for (int j = 0; j < SPL; ++j) {
        pl[j] = live_state[j] ? T[j] - mik[j] : -INFINITY;
        M = fmaxf(M, pl[j]);
      }
      M = gmax(M);
      float S = 0.f;
#pragma unroll
      for (int j = 0; j < SPL; ++j) {
        e[j] = live_state[j] ? fex2(pl[j] - M) : 0.f;
        S += e[j];
      }
      if constexpr (POTTS) {  // Potts: o(x) = sum_y e(y) t(y, x) / d = (a/d - 1) e(x) + sum_y e(y)
        S = gsum(S);
#pragma unroll
        for (int j = 0; j < SPL; ++j) o[j] = fmaf(w[k], e[j], S);
      } else {  // dense max-scaled table, oriented by the direction of `out`
        const float* tab = g.table + static_cast<size_t>(out >> 1) * QS * QS;
#pragma unroll
        for (int j = 0; j < SPL; ++j) o[j] = 0.f;
#pragma unroll
        for (int y = 0; y < QS; ++y) {
          // e(y) lives in lane y / SPL of the group, slot y % SPL
          const float ey = __shfl_sync(0xffffffffu, e[y % SPL], (threadIdx.x & 31u & ~(LPV - 1u)) + y / SPL);
#pragma unroll
          for (int j = 0; j < SPL; ++j) {
            const int x = x0 + j;
            const float tv = has[k] ? __ldg(&tab[(out & 1u) ? x * QS + y : y * QS + x]) : 0.f;
            o[j] = fmaf(tv, ey, o[j]);
          }
        }
      }
      float sm = 0.f;
#pragma unroll
      for (int j = 0; j < SPL; ++j) {
        o[j] = live_state[j] ? o[j] : 0.f;
        sm += o[j];
      }
      sm = gsum(sm);
      const float inv = frcp(sm);
      float ln[SPL], rr = 0.f;
#pragma unroll
      for (int j = 0; j < SPL; ++j) {
        ln[j] = flg2(o[j] * inv);
        rr = fmaxf(rr, live_state[j] ? fabsf(fex2(ln[j]) - fex2(mok[j])) : 0.f);
      }
      rr = gmax(rr);
      if (has[k]) {
        float4 st;
        st.x = live_state[0] ? ln[0] : mok[0];
        st.y = live_state[1] ? ln[1] : mok[1];
        st.z = live_state[2] ? ln[2] : mok[2];
        st.w = live_state[3] ? ln[3] : mok[3];
        *reinterpret_cast<float4*>(&B[static_cast<size_t>(out) * QS + x0]) = st;
        if (l == 0) {
          if (MODE == kModeDelta) {
            cnt += (rr >= eps ? 1 : 0) - (was[k] ? 1 : 0);
            res[out] = rr;
          } else {
            if (MODE == kModeInit) res[out] = rr;
            cnt += rr >= eps;
          }
          ++evals;
          bad |= !(sm > 0.f) || !(sm < INFINITY);
        }
      }
    }
    if (act && l == 0) ++visits;
  }
  if (bad) ctl->numeric_error = 1u;
  Contrib cb;
  if (MODE == kModeDelta)
    cb.delta = cnt;
  else
    cb.count = static_cast<unsigned long long>(cnt);
  cb.evals = evals;
  cb.visits = visits;
  block_accumulate(ctl, cb);
  fused_finalize(ctl, fin);
}

// ---------------------------------------------------------------------------
// initial messages (init_messages, messages.cpp:23-39): uniform over the
// target's states; binary log-odds 0.

template <int QS>
__global__ void k_init_messages(DevGraph g, float* M, Ctl* ctl, int set_t0) {
  if (set_t0 && blockIdx.x == 0 && threadIdx.x == 0) ctl->t0_ns = globaltimer_ns();
  const size_t n = static_cast<size_t>(g.D) * QS;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    if (QS == 1) {
      M[i] = 0.f;
    } else {
      const uint32_t x = static_cast<uint32_t>(i % QS);
      // uniform cardinality: no per-message lookup of the target's q
      const uint32_t q = g.uniform_q ? g.uniform_q : g.card[g.ep[static_cast<uint32_t>(i / QS) ^ 1u]];
      M[i] = x < q ? -log2f(static_cast<float>(q)) : 0.f;  // base-2 log-probabilities
    }
  }
}

// ---------------------------------------------------------------------------
// Frontier commit and touched-vertex flagging.
//
// commit: live <- candidate (MessageStore::write, messages.cpp:11-13) and
// r <- 0 (the candidate of d is unchanged unless its source is touched, in
// which case the refresh recomputes it); its target joins the touched set
// (collect_touched: every outgoing edge of tgt(d)).  Dense iterations mark
// vflag with plain stores; sparse ones dedupe with atomicMax and stage new
// vertices in shared memory, one global append per block flush.

template <int QS>
__device__ __forceinline__ void commit_edge(const DevGraph& g, uint32_t d, float r, float* live,
                                            const float* cand, float* res, float eps,
                                            uint32_t* vflag, uint32_t stamp, bool dense, Contrib& c,
                                            bool& new_flag, uint32_t& tgt) {
  c.delta -= (r >= eps) ? 1 : 0;
  c.frontier += 1;
  res[d] = 0.f;
  if constexpr (QS % 4 == 0) {  // q-vectors move as 16-byte loads / stores
    float4* dst = reinterpret_cast<float4*>(live + static_cast<size_t>(d) * QS);
    const float4* src = reinterpret_cast<const float4*>(cand + static_cast<size_t>(d) * QS);
#pragma unroll (QS <= 16 ? QS / 4 : 2)
    for (int x4 = 0; x4 < QS / 4; ++x4) dst[x4] = src[x4];
  } else {
#pragma unroll (QS <= 8 ? QS : 2)
    for (int x = 0; x < QS; ++x) live[static_cast<size_t>(d) * QS + x] = cand[static_cast<size_t>(d) * QS + x];
  }
  tgt = g.ep[d ^ 1u];
  if (dense) {
    vflag[tgt] = stamp;
    new_flag = false;
  } else {
    new_flag = atomicMax(&vflag[tgt], stamp) < stamp;
  }
}

// commit_edge for the committed edges of one quad of directed edges
// 4q .. 4q + 3 (all < D) with q-vectors of QS = 4 / 8 floats: every load
// (candidate q-vectors, the quad's endpoint ids) is issued before the first
// store -- commit_edge one edge after another serialised a candidate round
// trip and a target round trip per commit behind the previous commit's
// stores.  Same stores, same values, same counts.
template <int QS>
__device__ __forceinline__ void commit_quad_qvec(const DevGraph& g, uint32_t q, const bool (&com)[4],
                                                 const float (&r)[4], float* __restrict__ live,
                                                 const float* __restrict__ cand, float* __restrict__ res, float eps,
                                                 uint32_t* __restrict__ vflag, uint32_t stamp, bool dense,
                                                 Contrib& c, bool (&new_flag)[4], uint32_t (&tgt)[4]) {
  static_assert(QS % 4 == 0 && QS <= 8, "two 16-byte halves at most per q-vector");
  constexpr int H = QS / 4;
  const uint4 ep4 = __ldg(reinterpret_cast<const uint4*>(g.ep) + q);
  const uint32_t tgs[4] = {ep4.y, ep4.x, ep4.w, ep4.z};  // target of d = ep[d ^ 1]
  float4 v[4][H];
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (com[k]) {
      const float4* src = reinterpret_cast<const float4*>(cand + static_cast<size_t>(4 * q + k) * QS);
#pragma unroll
      for (int h = 0; h < H; ++h) v[k][h] = src[h];
    }
  float rv[4] = {r[0], r[1], r[2], r[3]};
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (com[k]) {
      c.delta -= (r[k] >= eps) ? 1 : 0;
      c.frontier += 1;
      rv[k] = 0.f;
      float4* dst = reinterpret_cast<float4*>(live + static_cast<size_t>(4 * q + k) * QS);
#pragma unroll
      for (int h = 0; h < H; ++h) dst[h] = v[k][h];
      tgt[k] = tgs[k];
      if (dense) {
        vflag[tgt[k]] = stamp;
        new_flag[k] = false;
      } else {
        new_flag[k] = atomicMax(&vflag[tgt[k]], stamp) < stamp;
      }
    }
  // res is padded to a multiple of four floats: the quad leaves as one store
  reinterpret_cast<float4*>(res)[q] = make_float4(rv[0], rv[1], rv[2], rv[3]);
}

// select_parallelism (schedulers.cpp:218-224)
__device__ __forceinline__ double device_p_now(const Ctl* c, double low_p, double high_p,
                                               double thr) {
  if (!c->has_prev || c->prev_unconverged == 0) return high_p;
  const double ratio = static_cast<double>(c->unconverged) / static_cast<double>(c->prev_unconverged);
  return ratio > thr ? low_p : high_p;
}

struct RnbpParams {
  unsigned long long seed;
  double low_p, high_p, thr;
  double fixed_p;  // >= 0: lockstep override of p_now
  int commit;      // 0: only mark `sel` (lockstep frontier query)
  unsigned attempt;  // Philox attempt of the select kernel (band retries use 1)
};

// rnbp_frontier (schedulers.cpp:194-216) attempt 0, fused with the commit of
// apply_frontier: filter 1 (r >= eps), filter 2 Bernoulli(p_now) with Philox.
//
// CL = false: scan every residual (4 per thread per trip, one 16-byte load;
// res is padded to a multiple of 4 with zeros).
// CL = true: scan the candidate list (a superset of the edges with r >= eps,
// maintained by the refresh): converged entries and committed edges leave the
// list, surviving unselected ones are kept in the next list, so the cost of an
// iteration follows the unconverged count instead of 2|E|.  The Bernoulli draw
// is keyed by the edge id, so list order does not matter.
template <int QS, bool CL>
__device__ __forceinline__ void rnbp_select_pass(const DevGraph& g, float* live, const float* cand, float* res,
                                                 uint32_t* vflag, uint32_t* vlist, uint8_t* sel, Ctl* ctl,
                                                 float eps, const RnbpParams& prm, const CandList& cl) {
  const double p = prm.fixed_p >= 0.0 ? prm.fixed_p : device_p_now(ctl, prm.low_p, prm.high_p, prm.thr);
  const unsigned long long thresh = static_cast<unsigned long long>(ceil(ldexp(p, 53)));
  const unsigned long long it = ctl->iteration;
  const uint32_t stamp = ctl->stamp;
  // dense iterations (expected frontier > V/16) flag without a list
  const bool dense =
      prm.commit && static_cast<double>(ctl->unconverged) * p > static_cast<double>(g.V) / 16.0;
  if (blockIdx.x == 0 && threadIdx.x == 0) ctl->dense = dense ? 1u : 0u;
  BPB_STAGER(fl, 2048, vlist, &ctl->nflag);
  const unsigned cur = CL ? ctl->cl_cur : 0u;
  const unsigned st = CL && prm.commit ? ctl->cl_state : 0u;  // 1: build the list, 2: walk it
  BPB_STAGER(keep, CL ? 2048 : 1, CL ? (cur ? cl.list[0] : cl.list[1]) : nullptr, &ctl->cl_n[cur ^ 1u]);
  fl.init();
  if (CL) keep.init();
  Contrib c;
  const uint32_t stride = gridDim.x * blockDim.x;
  if (st != 2u) {
    const uint32_t D4 = (g.D + 3) / 4;
    const float4* res4 = reinterpret_cast<const float4*>(res);
    for (uint32_t base = blockIdx.x * blockDim.x; base < D4; base += stride) {
      const uint32_t q = base + threadIdx.x;
      bool nf[4] = {false, false, false, false}, kp[4] = {false, false, false, false};
      uint32_t tg[4] = {0, 0, 0, 0};
      if (q < D4) {
        const float4 r4 = res4[q];
        const float rr[4] = {r4.x, r4.y, r4.z, r4.w};
        // one Philox block per edge pair, only when a survivor needs a draw
        const bool draw = thresh < (1ull << 53);
        uint4 ph[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
        if (draw) {
          // keyed by the GLOBAL edge id (edge_offset != 0 for a band of a partition)
          if (rr[0] >= eps || rr[1] >= eps) ph[0] = philox_edge(prm.seed, it, prm.attempt, global_edge(g, 2u * q));
          if (rr[2] >= eps || rr[3] >= eps)
            ph[1] = philox_edge(prm.seed, it, prm.attempt, global_edge(g, 2u * q + 1u));
        }
        // binary: the four commits' operands (candidates, targets) in two
        // 16-byte loads, one round trip instead of one per commit
        float4 cv4 = make_float4(0.f, 0.f, 0.f, 0.f), lv4 = cv4;
        uint4 ep4 = make_uint4(0u, 0u, 0u, 0u);
        const bool quad = QS == 1 && prm.commit && 4 * q + 3 < g.D &&
                          (rr[0] >= eps || rr[1] >= eps || rr[2] >= eps || rr[3] >= eps);
        if (quad) {
          cv4 = reinterpret_cast<const float4*>(cand)[q];
          lv4 = reinterpret_cast<const float4*>(live)[q];
          ep4 = __ldg(reinterpret_cast<const uint4*>(g.ep) + q);
        }
        // q-vectors (QS = 4 / 8): the quad's commits are decided first and
        // committed together (commit_quad_qvec), so their candidate loads are
        // one round trip instead of one per commit
        constexpr bool kQBatch = QS == 4 || QS == 8;
        const bool qbatch = kQBatch && prm.commit && 4 * q + 3 < g.D;
        bool com[4] = {false, false, false, false};
        float cvs[4] = {cv4.x, cv4.y, cv4.z, cv4.w};
        float lvs[4] = {lv4.x, lv4.y, lv4.z, lv4.w};
        float rvs[4] = {rr[0], rr[1], rr[2], rr[3]};
        bool any = false;
        const uint32_t tgs[4] = {ep4.y, ep4.x, ep4.w, ep4.z};  // target of d = ep[d ^ 1]
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t d = 4 * q + k;
          if (rr[k] >= eps) {  // padding entries are 0
            c.survivors += 1;
            if (!draw || u53_of(ph[k >> 1], d) < thresh) {
              if (quad) {  // commit_edge with the prefetched operands; the quad is stored whole below
                c.delta -= 1;
                c.frontier += 1;
                rvs[k] = 0.f;
                lvs[k] = cvs[k];
                any = true;
                tg[k] = tgs[k];
                if (dense) {
                  vflag[tg[k]] = stamp;
                } else {
                  nf[k] = atomicMax(&vflag[tg[k]], stamp) < stamp;
                }
              } else if (qbatch) {  // committed below, the quad's loads first
                com[k] = true;
              } else if (prm.commit) {
                commit_edge<QS>(g, d, rr[k], live, cand, res, eps, vflag, stamp, dense, c, nf[k], tg[k]);
              } else {
                sel[d] = 1;
                c.frontier += 1;
              }
            } else if (CL && st == 1u) {
              cl.inlist[d] = 1;
              kp[k] = true;
            }
          }
        }
        if (any) {  // one 16-byte store per array instead of one 4-byte store per commit
          reinterpret_cast<float4*>(live)[q] = make_float4(lvs[0], lvs[1], lvs[2], lvs[3]);
          reinterpret_cast<float4*>(res)[q] = make_float4(rvs[0], rvs[1], rvs[2], rvs[3]);
        }
        if constexpr (kQBatch) {
          if (com[0] || com[1] || com[2] || com[3])
            commit_quad_qvec<QS>(g, q, com, rr, live, cand, res, eps, vflag, stamp, dense, c, nf, tg);
        }
      }
      if (prm.commit && !dense) {
#pragma unroll
        for (int k = 0; k < 4; ++k) fl.push_warp(nf[k], tg[k]);
        fl.flush(4 * kBlock);
      }
      if (CL && st == 1u) {
#pragma unroll
        for (int k = 0; k < 4; ++k) keep.push_warp(kp[k], 4 * q + k);
        keep.flush(4 * kBlock);
      }
    }
    if (CL && st == 1u) keep.flush(0);
  } else {
    const uint32_t n = ctl->cl_n[cur];
    const uint32_t* list = cur ? cl.list[1] : cl.list[0];
    for (uint32_t base = blockIdx.x * blockDim.x; base < n; base += stride) {
      const uint32_t i = base + threadIdx.x;
      bool nf = false, kept = false;
      uint32_t tg = 0, d = 0;
      if (i < n) {
        d = list[i];
        const float r = res[d];
        if (r >= eps) {
          c.survivors += 1;
          if ((thresh >= (1ull << 53) || philox_u53(prm.seed, it, 0u, global_directed(g, d)) < thresh)) {
            cl.inlist[d] = 0;
            commit_edge<QS>(g, d, r, live, cand, res, eps, vflag, stamp, dense, c, nf, tg);
          } else {
            kept = true;
          }
        } else {
          cl.inlist[d] = 0;
        }
      }
      keep.push_warp(kept, d);
      keep.flush(kBlock);
      if (!dense) {
        fl.push_warp(nf, tg);
        fl.flush(kBlock);
      }
    }
    keep.flush(0);
  }
  if (prm.commit && !dense) fl.flush(0);
  block_accumulate(ctl, c);
}


// Retry + fallback of rnbp_frontier (schedulers.cpp:204-214), single block:
// reduces the attempt-0 frontier and survivor counts; when the frontier came
// back empty it redraws every survivor once (attempt 1) and, if still empty,
// commits survivors[min(S-1, floor(u*S))] in ascending id order.  The redraw
// runs only on that rare path, so one block suffices.  With the candidate
// list the survivors are exactly the kept list.
// Attempt 1 + fallback of rnbp_frontier (schedulers.cpp:204-214) by one
// block, called only when attempt 0 selected nothing and survivors exist.
// The commits' count change goes to *delta_out (atomic).
template <int QS, bool CL>
__device__ __forceinline__ void rnbp_retry_block(const DevGraph& g, float* live, const float* cand, float* res,
                                                 uint32_t* vflag, uint32_t* vlist, uint8_t* sel, Ctl* ctl,
                                                 float eps, const RnbpParams& prm, const CandList& cl,
                                                 unsigned long long surv, long long* delta_out,
                                                 const uint32_t* slots = nullptr, uint32_t slot_n = 0,
                                                 uint32_t* vslot = nullptr, uint32_t* cstamp = nullptr) {
  // cstamp != nullptr (persistent tail, lattice): a committed edge is stamped
  // and its slot names the EDGE (the refresh's owner test dedupes targets)
  // slots != nullptr (persistent tail): the survivors are the kept entries of
  // the slot list (kSlotEmpty holes), and a committed edge's target goes to
  // the refresh slot of the same index (the fallback's to slot 0, which is
  // empty whenever the fallback runs)
  __shared__ unsigned long long s_front, s_surv;
  __shared__ unsigned warp_tot[32];
  __shared__ unsigned long long running_s;
  __shared__ int found;
  if (threadIdx.x == 0) s_surv = surv;
  const double p = prm.fixed_p >= 0.0 ? prm.fixed_p : device_p_now(ctl, prm.low_p, prm.high_p, prm.thr);
  const unsigned long long thresh = static_cast<unsigned long long>(ceil(ldexp(p, 53)));
  const unsigned long long it = ctl->iteration;
  const uint32_t stamp = ctl->stamp;
  if (threadIdx.x == 0) {
    ctl->dense = 0;
    found = 0;
    running_s = 0;
  }
  __syncthreads();
  // attempt 1: every survivor redrawn
  unsigned long long fr = 0;
  long long delta = 0;
  const bool use_list = CL && ctl->cl_state == 2u;  // survivors = the kept list
  const uint32_t n = slots ? slot_n : use_list ? ctl->cl_n[ctl->cl_cur ^ 1u] : g.D;
  const uint32_t* list = slots ? slots : use_list ? (ctl->cl_cur ? cl.list[0] : cl.list[1]) : nullptr;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    const uint32_t d = (use_list || slots) ? list[i] : i;
    if (d == kSlotEmpty) continue;
    const float r = res[d];
    if (r >= eps && philox_u53(prm.seed, it, 1u, global_directed(g, d)) < thresh) {
      ++fr;
      if (prm.commit) {
        Contrib c;
        bool nf = false;
        uint32_t tg = 0;
        commit_edge<QS>(g, d, r, live, cand, res, eps, vflag, stamp, false, c, nf, tg);
        delta += c.delta;
        if (cstamp) {
          cstamp[d] = stamp;
          vslot[i] = d;
        } else if (vslot)
          vslot[i] = nf ? tg : kSlotEmpty;
        else if (nf)
          vlist[atomicAdd(&ctl->nflag, 1u)] = tg;
      } else {
        sel[d] = 1;
      }
    }
  }
  __shared__ unsigned long long sh_f[32];
  __shared__ long long sh_d[32];
  fr = block_sum(fr, sh_f);
  delta = block_sum(delta, sh_d);
  if (threadIdx.x == 0) {
    ctl->frontier = fr;  // counted here; the attempt-0 slots hold 0
    if (delta) atomicAdd(reinterpret_cast<unsigned long long*>(delta_out), static_cast<unsigned long long>(delta));
    s_front = fr;
  }
  __syncthreads();
  if (s_front > 0) return;
  // fallback: one uniformly chosen survivor, ascending id order
  const unsigned long long S = s_surv;
  const double u = static_cast<double>(philox_u53(prm.seed, it, 2u, 0ull)) * 0x1.0p-53;
  unsigned long long pick = static_cast<unsigned long long>(u * static_cast<double>(S));
  if (pick > S - 1) pick = S - 1;
  const unsigned lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  for (size_t base = 0; base < g.D; base += blockDim.x) {
    const size_t di = base + threadIdx.x;
    const bool f = di < g.D && res[di] >= eps;
    const unsigned m = __ballot_sync(0xffffffffu, f);
    if (lane == 0) warp_tot[wid] = __popc(m);
    __syncthreads();
    unsigned before = 0, total = 0;
    for (unsigned w = 0; w < (blockDim.x >> 5); ++w) {
      if (w < wid) before += warp_tot[w];
      total += warp_tot[w];
    }
    const unsigned long long rank = running_s + before + __popc(m & ((1u << lane) - 1u));
    if (f && rank == pick) {
      const uint32_t d = static_cast<uint32_t>(di);
      if (prm.commit) {
        Contrib c;
        bool nf = false;
        uint32_t tg = 0;
        commit_edge<QS>(g, d, res[d], live, cand, res, eps, vflag, stamp, false, c, nf, tg);
        if (cstamp) {
          cstamp[d] = stamp;
          vslot[0] = d;
        } else if (vslot)
          vslot[0] = nf ? tg : kSlotEmpty;
        else if (nf)
          vlist[atomicAdd(&ctl->nflag, 1u)] = tg;
        atomicAdd(reinterpret_cast<unsigned long long*>(delta_out), static_cast<unsigned long long>(c.delta));
      } else {
        sel[d] = 1;
      }
      ctl->frontier = 1;
      found = 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) running_s += total;
    __syncthreads();
    if (found) break;
  }
}

// the retry decision + retry of one iteration, by ONE block (any size, a
// multiple of 32): reduces the attempt-0 frontier / survivor slots
template <int QS, bool CL>
__device__ __forceinline__ void rnbp_retry_pass(const DevGraph& g, float* live, const float* cand, float* res,
                                                uint32_t* vflag, uint32_t* vlist, uint8_t* sel, Ctl* ctl,
                                                float eps, const RnbpParams& prm, const CandList& cl) {
  __shared__ unsigned long long s_f, s_s;
  if (threadIdx.x < 32) {
    unsigned long long f = 0, s = 0;
    for (int k = threadIdx.x; k < kSlots; k += 32) {
      f += ctl->acc[k].frontier;
      s += ctl->acc[k].survivors;
    }
    f = warp_sum(f);
    s = warp_sum(s);
    if (threadIdx.x == 0) {
      s_f = f;
      s_s = s;
      ctl->survivors = s;
    }
  }
  __syncthreads();
  if (s_f > 0 || s_s == 0) return;
  rnbp_retry_block<QS, CL>(g, live, cand, res, vflag, vlist, sel, ctl, eps, prm, cl, s_s, &ctl->acc[0].delta);
}

// retry != 0: the last block runs the retry + fallback of the iteration
// (rnbp_retry_pass; the lockstep frontier query); the run loop launches
// k_rnbp_retry instead
template <int QS, bool CL>
__global__ void __launch_bounds__(kBlock) k_rnbp_select(DevGraph g, float* live, const float* cand,
                                                        float* res, uint32_t* vflag, uint32_t* vlist,
                                                        uint8_t* sel, Ctl* ctl, float eps,
                                                        RnbpParams prm, CandList cl, int retry) {
  if (run_done(ctl)) return;
  rnbp_select_pass<QS, CL>(g, live, cand, res, vflag, vlist, sel, ctl, eps, prm, cl);
  if (retry && last_block_done(ctl)) rnbp_retry_pass<QS, CL>(g, live, cand, res, vflag, vlist, sel, ctl, eps, prm, cl);
}

template <int QS, bool CL>
__global__ void __launch_bounds__(1024) k_rnbp_retry(DevGraph g, float* live, const float* cand,
                                                     float* res, uint32_t* vflag, uint32_t* vlist,
                                                     uint8_t* sel, Ctl* ctl, float eps, RnbpParams prm,
                                                     CandList cl) {
  if (run_done(ctl)) return;
  rnbp_retry_pass<QS, CL>(g, live, cand, res, vflag, vlist, sel, ctl, eps, prm, cl);
}

// Commit of a host-supplied frontier (lockstep apply_frontier).
template <int QS>
__global__ void __launch_bounds__(kBlock) k_commit_list(DevGraph g, const uint32_t* list, uint32_t n,
                                                        float* live, const float* cand, float* res,
                                                        uint32_t* vflag, uint32_t* vlist, Ctl* ctl,
                                                        float eps, int dense) {
  BPB_STAGER(fl, 2048, vlist, &ctl->nflag);
  if (blockIdx.x == 0 && threadIdx.x == 0) ctl->dense = dense;
  fl.init();
  const uint32_t stamp = ctl->stamp;
  Contrib c;
  for (uint32_t base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    bool nf = false;
    uint32_t tgt = 0;
    if (i < n) {
      const uint32_t d = list[i];
      commit_edge<QS>(g, d, res[d], live, cand, res, eps, vflag, stamp, dense != 0, c, nf, tgt);
    }
    if (!dense) {
      fl.push_warp(nf, tgt);
      fl.flush(kBlock);
    }
  }
  if (!dense) fl.flush(0);
  block_accumulate(ctl, c);
}

// ---------------------------------------------------------------------------
// RBP top-k (select_top_k, schedulers.cpp:105-116): exact radix select of the
// k-th largest residual over the 32-bit float pattern (residuals are >= +0,
// so the unsigned order equals the float order), three passes of 12/12/8
// bits (k_rx_* below), then a commit pass; ties at the threshold go to the
// lowest ids via per-chunk tie counts.  k_rbp_commit is the select-all commit
// (k >= the directed edges).

constexpr int kRadixBins = 4096;

__device__ __forceinline__ uint32_t float_key(float r) { return __float_as_uint(r); }

constexpr uint32_t kTieChunk = 8192;

// Commit the top-k: key > K*, or key == K* with tie rank < need.
// One block per tie chunk so tie ranks follow ascending edge id.
template <int QS>
__global__ void __launch_bounds__(kBlock) k_rbp_commit(DevGraph g, float* live, const float* cand,
                                                       float* res, uint32_t* vflag, uint32_t* vlist,
                                                       uint8_t* sel, const unsigned* chunk_off,
                                                       Ctl* ctl, float eps, int select_all,
                                                       int commit, int dense) {
  if (run_done(ctl)) return;
  BPB_STAGER(fl, 2048, vlist, &ctl->nflag);
  if (blockIdx.x == 0 && threadIdx.x == 0 && commit) ctl->dense = dense;
  fl.init();
  const uint32_t key = ctl->rx_prefix;
  const bool band = band_graph(g);
  const bool rank_ties = !select_all && ctl->rx_need != ctl->rx_ties;
  const unsigned need = ctl->rx_need;
  const uint32_t stamp = ctl->stamp;
  __shared__ unsigned wt[kBlock / 32];
  __shared__ unsigned running;
  if (threadIdx.x == 0) running = rank_ties ? chunk_off[blockIdx.x] : 0u;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  Contrib c;
  const size_t c0 = static_cast<size_t>(blockIdx.x) * kTieChunk;
  for (size_t base = c0; base < c0 + kTieChunk && base < g.D; base += blockDim.x) {
    const size_t di = base + threadIdx.x;
    const bool valid = di < g.D && di < c0 + kTieChunk && (!band || edge_owned(g, static_cast<uint32_t>(di)));
    const float r = valid ? res[di] : 0.f;
    const uint32_t k = float_key(r);
    bool take = valid && (select_all || k > key);
    const bool tie = valid && !select_all && k == key;
    if (rank_ties) {
      const unsigned m = __ballot_sync(0xffffffffu, tie);
      if (lane == 0) wt[wid] = __popc(m);
      __syncthreads();
      unsigned before = 0, total = 0;
      for (unsigned w = 0; w < (blockDim.x >> 5); ++w) {
        if (w < wid) before += wt[w];
        total += wt[w];
      }
      const unsigned rank = running + before + __popc(m & ((1u << lane) - 1u));
      if (tie && rank < need) take = true;
      __syncthreads();
      if (threadIdx.x == 0) running += total;
    } else if (tie) {
      take = true;
    }
    bool nf = false;
    uint32_t tgt = 0;
    if (take) {
      if (commit) {
        commit_edge<QS>(g, static_cast<uint32_t>(di), r, live, cand, res, eps, vflag, stamp, dense != 0, c, nf,
                        tgt);
      } else {
        sel[di] = 1;
        c.frontier += 1;
      }
    }
    if (commit && !dense) {
      fl.push_warp(nf, tgt);
      fl.flush(kBlock);
    }
  }
  if (commit && !dense) fl.flush(0);
  block_accumulate(ctl, c);
}

// ---------------------------------------------------------------------------
// RBP top-k over a compacted candidate list: the same exact radix select in
// five launches and two full passes over the residuals (instead of eight
// launches and five passes):
//   k_rx_hist0    pass-0 histogram (top 12 bits) of every residual; the last
//                 block scans it (bin of the k-th key)
//   k_rx_compact  edges whose top 12 bits reach that bin join a list; the
//                 bin's own members feed the pass-1 histogram; last block: scan 1
//   k_rx_hist2    pass-2 histogram over the list; last block: scan 2 = K*
//   k_rx_ties     only when K* is shared and not every tie is taken: per-chunk
//                 tie counts over all edges, prefix summed by the last block
//   k_rbp_commit_list  the list's keys >= K* -- or, when ties are ranked,
//                 every chunk of edges with k_rbp_commit's ascending-id rank
// Outcome (frontier, commits, touched vertices) is identical to the
// eight-launch path; only the order of the touched list differs.

// k_radix_scan for one block of any size (a multiple of 32, <= 1024): the bin
// holding the k-th largest key counted from the top, the prefix extended,
// the count strictly above it accumulated, the histogram cleared.
static __device__ void radix_scan_block(unsigned* hist, int pass, unsigned long long k, Ctl* ctl) {
  __shared__ unsigned long long wsum[32];
  const int nb = pass == 2 ? 256 : kRadixBins;
  const int nt = static_cast<int>(blockDim.x);
  const int per = (nb + nt - 1) / nt;
  const int t = threadIdx.x;
  unsigned long long mine = 0;
  for (int j = 0; j < per; ++j)
    if (t * per + j < nb) mine += __ldcg(&hist[nb - 1 - (t * per + j)]);
  unsigned long long v = mine;
  const unsigned lane = t & 31, wid = t >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= static_cast<unsigned>(o)) v += n;
  }
  if (lane == 31) wsum[wid] = v;
  __syncthreads();
  if (wid == 0) {
    unsigned long long w = lane < static_cast<unsigned>(nt >> 5) ? wsum[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long n = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= static_cast<unsigned>(o)) w += n;
    }
    wsum[lane] = w;  // inclusive
  }
  __syncthreads();
  const unsigned long long excl = v - mine + (wid ? wsum[wid - 1] : 0ull);
  const unsigned long long above0 = pass == 0 ? 0ull : ctl->rx_above;
  const unsigned long long need = k - above0;  // >= 1
  if (excl < need && need <= excl + mine) {
    unsigned long long acc = excl;
    for (int j = 0; j < per && t * per + j < nb; ++j) {
      const int bin = nb - 1 - (t * per + j);
      const unsigned c = __ldcg(&hist[bin]);
      if (acc < need && need <= acc + c) {
        const int bits = pass == 2 ? 8 : 12;
        ctl->rx_prefix = (pass == 0 ? 0u : (ctl->rx_prefix << bits)) | static_cast<unsigned>(bin);
        ctl->rx_above = above0 + acc;
        ctl->rx_ties = c;
        ctl->rx_need = static_cast<unsigned>(need - acc);
        break;
      }
      acc += c;
    }
  }
  __syncthreads();
  for (int i = t; i < nb; i += nt) hist[i] = 0;
}

// block histogram -> global (every thread fences its own atomics), then the
// last block to finish scans
// (a release fence only in the threads that issued bin atomics: a full
// __threadfence in every thread was a fifth of the pass-0 kernel's stalls)
__device__ __forceinline__ void rx_flush_and_scan(const unsigned* sh, int nb, unsigned* hist, int pass,
                                                  unsigned long long k, Ctl* ctl) {
  __syncthreads();
  bool any = false;
  for (int i = threadIdx.x; i < nb; i += blockDim.x)
    if (sh[i]) {
      atomicAdd(&hist[i], sh[i]);
      any = true;
    }
  if (any) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  if (last_block_done(ctl)) radix_scan_block(hist, pass, k, ctl);
}

constexpr int kRxUnroll = 2;

// exclusive scan over the block (kBlock threads); *total the sum; ends behind a barrier
__device__ __forceinline__ unsigned block_excl_scan_u32(unsigned x, unsigned* total) {
  __shared__ unsigned ws[kBlock / 32];
  const unsigned lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  unsigned v = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= static_cast<unsigned>(o)) v += n;
  }
  __syncthreads();  // ws is reused across calls
  if (lane == 31) ws[wid] = v;
  __syncthreads();
  unsigned before = 0, tot = 0;
#pragma unroll
  for (unsigned w = 0; w < kBlock / 32; ++w) {
    const unsigned c = ws[w];
    before += w < wid ? c : 0u;
    tot += c;
  }
  *total = tot;
  return before + v - x;
}

static __global__ void __launch_bounds__(kBlock) k_rx_hist0(DevGraph g, const float* res, uint32_t D,
                                                     unsigned* hist, Ctl* ctl, unsigned long long k) {
  if (run_done(ctl)) return;
  const bool band = band_graph(g);
  __shared__ unsigned sh[kRadixBins];
  for (int i = threadIdx.x; i < kRadixBins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint32_t D4 = (D + 3) / 4;
  const float4* res4 = reinterpret_cast<const float4*>(res);
  // kRxUnroll float4 loads in flight per thread (the pass is latency-bound)
  for (uint32_t q0 = blockIdx.x * blockDim.x * kRxUnroll + threadIdx.x; q0 < D4;
       q0 += gridDim.x * blockDim.x * kRxUnroll) {
    float4 r4[kRxUnroll];
#pragma unroll
    for (int u = 0; u < kRxUnroll; ++u) {
      const uint32_t q = q0 + u * blockDim.x;
      r4[u] = q < D4 ? res4[q] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < kRxUnroll; ++u) {
      const uint32_t q = q0 + u * blockDim.x;
      const float rr[4] = {r4[u].x, r4[u].y, r4[u].z, r4[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (q >= D4 || 4 * q + j >= D) continue;
        if (band && !edge_owned(g, 4 * q + j)) continue;
        atomicAdd(&sh[float_key(rr[j]) >> 20], 1u);
      }
    }
  }
  rx_flush_and_scan(sh, kRadixBins, hist, 0, k, ctl);
  if (threadIdx.x == 0 && blockIdx.x == 0) ctl->rx_n = 0u;  // read by k_rx_compact only (next launch)
}

static __global__ void __launch_bounds__(kBlock) k_rx_compact(DevGraph g, const float* res, uint32_t D,
                                                       unsigned* hist, uint32_t* list, Ctl* ctl,
                                                       unsigned long long k) {
  if (run_done(ctl)) return;
  const bool band = band_graph(g);
  __shared__ unsigned sh[kRadixBins];
  __shared__ unsigned s_base;
  for (int i = threadIdx.x; i < kRadixBins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint32_t p0 = ctl->rx_prefix;
  const uint32_t D4 = (D + 3) / 4;
  const float4* res4 = reinterpret_cast<const float4*>(res);
  for (uint32_t base = blockIdx.x * blockDim.x * kRxUnroll; base < D4; base += gridDim.x * blockDim.x * kRxUnroll) {
    float4 r4[kRxUnroll];
#pragma unroll
    for (int u = 0; u < kRxUnroll; ++u) {
      const uint32_t q = base + u * blockDim.x + threadIdx.x;
      r4[u] = q < D4 ? res4[q] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    // this thread's candidates as a bit mask, one block scan, one global
    // reservation per block and step
    uint32_t m = 0u;
#pragma unroll
    for (int u = 0; u < kRxUnroll; ++u) {
      const uint32_t q = base + u * blockDim.x + threadIdx.x;
      const float rr[4] = {r4[u].x, r4[u].y, r4[u].z, r4[u].w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t d = 4 * q + j;
        const bool ok = q < D4 && d < D && (!band || edge_owned(g, d));
        const uint32_t key = float_key(rr[j]);
        if (ok && (key >> 20) == p0) atomicAdd(&sh[(key >> 8) & 0xfffu], 1u);
        if (ok && (key >> 20) >= p0) m |= 1u << (4 * u + j);
      }
    }
    unsigned tot;
    const unsigned pre = block_excl_scan_u32(__popc(m), &tot);
    if (tot == 0u) continue;  // block-uniform
    if (threadIdx.x == 0) s_base = atomicAdd(&ctl->rx_n, tot);
    __syncthreads();
    unsigned o = s_base + pre;
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1u;
      list[o++] = 4 * (base + (b >> 2) * blockDim.x + threadIdx.x) + (b & 3);
    }
    __syncthreads();  // s_base is rewritten by the next step
  }
  rx_flush_and_scan(sh, kRadixBins, hist, 1, k, ctl);
}

static __global__ void __launch_bounds__(kBlock) k_rx_hist2(const float* res, const uint32_t* list, unsigned* hist,
                                                     Ctl* ctl, unsigned long long k) {
  if (run_done(ctl)) return;
  __shared__ unsigned sh[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const uint32_t n = __ldcg(&ctl->rx_n), p01 = ctl->rx_prefix;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t key = float_key(res[__ldcg(&list[i])]);
    if ((key >> 8) == p01) atomicAdd(&sh[key & 0xffu], 1u);
  }
  rx_flush_and_scan(sh, 256, hist, 2, k, ctl);
}

// k_tie_count + k_tie_scan in one launch (the last block prefix-sums the chunk counts)
static __global__ void __launch_bounds__(kBlock) k_rx_ties(DevGraph g, const float* res, uint32_t D,
                                                    unsigned* chunk_cnt, uint32_t nchunks, Ctl* ctl) {
  const bool band = band_graph(g);
  if (run_done(ctl) || ctl->rx_need == ctl->rx_ties) return;
  const uint32_t key = ctl->rx_prefix;
  __shared__ unsigned sh[kBlock / 32];
  for (uint32_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {  // grid-stride: a no-op launch stays small
    const size_t c0 = static_cast<size_t>(ch) * kTieChunk;
    unsigned n = 0;
    for (size_t d = c0 + threadIdx.x; d < c0 + kTieChunk && d < D; d += blockDim.x)
      n += float_key(res[d]) == key && (!band || edge_owned(g, static_cast<uint32_t>(d)));
    const unsigned tot = block_sum(n, sh);
    if (threadIdx.x == 0) chunk_cnt[ch] = tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) __threadfence();
  if (!last_block_done(ctl)) return;
  __shared__ unsigned wsum[kBlock / 32];
  __shared__ unsigned carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint32_t base = 0; base < nchunks; base += blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    const unsigned c = i < nchunks ? __ldcg(&chunk_cnt[i]) : 0u;
    unsigned v = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned x = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= static_cast<unsigned>(o)) v += x;
    }
    if (lane == 31) wsum[wid] = v;
    __syncthreads();
    unsigned before = 0, total = 0;
    for (unsigned w = 0; w < (blockDim.x >> 5); ++w) {
      if (w < wid) before += wsum[w];
      total += wsum[w];
    }
    if (i < nchunks) chunk_cnt[i] = carry + before + v - c;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
}

// Commit (or mark, commit == 0) the top-k: the list's keys >= K* when every
// tie is taken; otherwise k_rbp_commit's chunk walk (key > K*, or a tie whose
// ascending-id rank is below need) over every chunk -- grid-stride over the
// chunks, since the list pass would change residuals a tie walk reads.
template <int QS>
__global__ void __launch_bounds__(kBlock) k_rbp_commit_list(DevGraph g, float* live, const float* cand, float* res,
                                                            uint32_t* vflag, uint32_t* vlist, uint8_t* sel,
                                                            const uint32_t* list, const unsigned* chunk_off,
                                                            uint32_t nchunks, Ctl* ctl, float eps, int commit,
                                                            int dense) {
  if (run_done(ctl)) return;
  BPB_STAGER(fl, 2048, vlist, &ctl->nflag);
  if (blockIdx.x == 0 && threadIdx.x == 0 && commit) ctl->dense = dense;
  fl.init();
  const uint32_t key = ctl->rx_prefix;
  const bool band = band_graph(g);
  const bool rank_ties = ctl->rx_need != ctl->rx_ties;
  const unsigned need = ctl->rx_need;
  const uint32_t stamp = ctl->stamp;
  Contrib c;
  auto take_edge = [&](uint32_t d, float r, bool take) {
    bool nf = false;
    uint32_t tgt = 0;
    if (take) {
      if (commit) {
        commit_edge<QS>(g, d, r, live, cand, res, eps, vflag, stamp, dense != 0, c, nf, tgt);
      } else {
        sel[d] = 1;
        c.frontier += 1;
      }
    }
    if (commit && !dense) {
      fl.push_warp(nf, tgt);
      fl.flush(kBlock);
    }
  };
  if (!rank_ties) {
    const uint32_t n = __ldcg(&ctl->rx_n);
    for (uint32_t base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
      const uint32_t i = base + threadIdx.x;
      uint32_t d = 0;
      float r = 0.f;
      if (i < n) {
        d = __ldcg(&list[i]);
        r = res[d];
      }
      take_edge(d, r, i < n && float_key(r) >= key);
    }
  } else {
    __shared__ unsigned wt[kBlock / 32];
    __shared__ unsigned running;
    const unsigned lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    for (uint32_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
      __syncthreads();
      if (threadIdx.x == 0) running = __ldcg(&chunk_off[ch]);
      __syncthreads();
      const size_t c0 = static_cast<size_t>(ch) * kTieChunk;
      for (size_t base = c0; base < c0 + kTieChunk && base < g.D; base += blockDim.x) {
        const size_t di = base + threadIdx.x;
        const bool valid = di < g.D && di < c0 + kTieChunk && (!band || edge_owned(g, static_cast<uint32_t>(di)));
        const float r = valid ? res[di] : 0.f;
        const uint32_t kk = float_key(r);
        const bool tie = valid && kk == key;
        const unsigned m = __ballot_sync(0xffffffffu, tie);
        if (lane == 0) wt[wid] = __popc(m);
        __syncthreads();
        unsigned before = 0, total = 0;
        for (unsigned w = 0; w < (blockDim.x >> 5); ++w) {
          if (w < wid) before += wt[w];
          total += wt[w];
        }
        const unsigned rank = running + before + __popc(m & ((1u << lane) - 1u));
        __syncthreads();
        if (threadIdx.x == 0) running += total;
        take_edge(static_cast<uint32_t>(di), r, (valid && kk > key) || (tie && rank < need));
      }
    }
  }
  if (commit && !dense) fl.flush(0);
  block_accumulate(ctl, c);
}

// ---------------------------------------------------------------------------
// beliefs (compute_beliefs, messages.cpp:82-105): normalize(psi_v * prod m_in)

template <int QS>
__global__ void k_beliefs(DevGraph g, const float* A0, const float* A1, int pingpong, Ctl* ctl,
                          double* out) {
  const float* A = (pingpong && (ctl->iteration & 1ull)) ? A1 : A0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < g.V; v += gridDim.x * blockDim.x) {
    if (QS == 1) {
      float T = g.unary_lo[v];
      for_each_in(g, v, [&](uint32_t in) { T += A[in]; });
      const double t = static_cast<double>(T);
      out[2 * static_cast<size_t>(v)] = 1.0 / (1.0 + exp2(t));  // base-2 log-odds
      out[2 * static_cast<size_t>(v) + 1] = 1.0 / (1.0 + exp2(-t));
    } else {
      const uint32_t q = g.card[v];
      float T[QS];
#pragma unroll (QS <= 8 ? QS : 2)
      for (int x = 0; x < QS; ++x) T[x] = g.unary_log[static_cast<size_t>(v) * QS + x];
      for_each_in(g, v, [&](uint32_t in) {
        const float* m = A + static_cast<size_t>(in) * QS;
#pragma unroll (QS <= 8 ? QS : 2)
        for (int x = 0; x < QS; ++x) T[x] += m[x];
      });
      float M = -INFINITY;
#pragma unroll (QS <= 8 ? QS : 2)
      for (int x = 0; x < QS; ++x)
        if (x < static_cast<int>(q)) M = fmaxf(M, T[x]);
      double p[QS];
      double s = 0.0;
#pragma unroll (QS <= 8 ? QS : 2)
      for (int x = 0; x < QS; ++x) {
        p[x] = x < static_cast<int>(q) ? exp2(static_cast<double>(T[x] - M)) : 0.0;
        s += p[x];
      }
      // compute_belief normalises too (messages.cpp:75-105): same mass check
      if (g.log_tables && static_cast<double>(M) + log2(s) < static_cast<double>(kLog2MinMass)) ctl->numeric_error = 1u;
      double* o = out + g.bel_off[v];
#pragma unroll (QS <= 8 ? QS : 2)
      for (int x = 0; x < QS; ++x)
        if (x < static_cast<int>(q)) o[x] = p[x] / s;
    }
  }
}

}  // namespace bpb
