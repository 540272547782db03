// Persistent RnBP tail (sm_100a; cooperative grid of one CTA per SM, or one
// 16-CTA thread-block cluster for short lists).
//
// Once the RnBP run walks its candidate list (cl_state 2: fewer than 1/16 of
// the directed edges unconverged) an iteration is a few thousand message
// updates, and four kernel launches per iteration would cost more than the
// work.  k_rnbp_persist runs the iterations of run() (schedulers.cpp:301-347)
// back to back inside one launch, with two grid-wide barriers per iteration:
//
//   select   rnbp_frontier attempt 0 over the candidate list + the Jacobi
//            commit of apply_frontier (schedulers.cpp:194-216, 231-241), in
//            slot form (outcomes stay at the entry's index)
//   --- barrier
//   retry    CTA 0, when nothing was drawn: attempt 1 + single-survivor
//            fallback (:204-214)
//   refresh  refresh_residuals over the touched vertices (residuals.cpp:26-59)
//            + compaction of the next candidate list
//   --- barrier
//   finalize replicated in every CTA: the loop control of run() (fin_iter);
//            the bookkeeping thread writes the trace record
//
// It stops when the run is done (converged / max_iterations / time limit /
// the host's trace-ring budget).  All data written inside the launch is read
// with coherent loads (ldm<false>); __ldg only touches the immutable graph.
#pragma once

#include <cooperative_groups.h>

#include "kernels.cuh"

namespace bpb {

namespace cgp = cooperative_groups;

constexpr int kPersistBlock = 512;
// candidate-list length below which the tail runs on one 16-CTA cluster (above it: a grid of one CTA per SM)
// (cluster barrier ~0.35 us vs grid barrier ~1.3 us, but 16 SMs instead of
// 148 share the list: measured at 115 entries cluster 8.9 vs grid 11.5
// us/iteration, at 6443 entries 12.0 vs 10.8)
constexpr uint32_t kPersistClusterList = 2048;

// Per-iteration contributions: one redux.sync per value and warp, summed in
// shared memory (s_pacc), pushed to acc[0..5] by threads 0..5 after the next
// block barrier (pacc_push).  The warp sums fit 32 bits (a warp touches at
// most a few thousand entries per iteration, a CTA a few hundred thousand).
__device__ __forceinline__ void warp_contrib(unsigned* s_pacc, const Contrib& c) {
  const int d = __reduce_add_sync(0xffffffffu, static_cast<int>(c.delta));
  const unsigned v[5] = {__reduce_add_sync(0xffffffffu, static_cast<unsigned>(c.count)),
                         __reduce_add_sync(0xffffffffu, static_cast<unsigned>(c.frontier)),
                         __reduce_add_sync(0xffffffffu, static_cast<unsigned>(c.survivors)),
                         __reduce_add_sync(0xffffffffu, static_cast<unsigned>(c.evals)),
                         __reduce_add_sync(0xffffffffu, static_cast<unsigned>(c.visits))};
  if ((threadIdx.x & 31u) == 0) {
    if (d) atomicAdd(reinterpret_cast<int*>(&s_pacc[0]), d);
#pragma unroll
    for (int k = 0; k < 5; ++k)
      if (v[k]) atomicAdd(&s_pacc[k + 1], v[k]);
  }
}
// after a block barrier that follows every warp_contrib of the phase
__device__ __forceinline__ void pacc_push(unsigned* s_pacc, unsigned long long* accum) {
  if (threadIdx.x < 6) {
    const unsigned x = s_pacc[threadIdx.x];
    if (x) {  // slot 0 (unconverged delta) is signed: sign-extend
      const unsigned long long w = threadIdx.x == 0 ? static_cast<unsigned long long>(static_cast<long long>(
                                                          static_cast<int>(x)))
                                                    : static_cast<unsigned long long>(x);
      atomicAdd(&accum[threadIdx.x], w);
      s_pacc[threadIdx.x] = 0u;
    }
  }
}

// CLUSTER: the whole grid is one thread-block cluster (<= 16 CTAs) and the
// phases are separated by the hardware cluster barrier; otherwise a
// cooperative grid barrier.
//
// The loop state of run() (iteration, unconverged count, previous count,
// vflag stamp, current list) is REPLICATED in every CTA: after the refresh
// barrier each CTA applies the finalize step itself from the reduced sums,
// so an iteration needs two barriers and no global read-modify-write of the
// control block.  Reductions and list counters are multi-buffered by
// iteration so no CTA resets a value another CTA may still read.  The bookkeeping thread (last CTA)
// mirrors the state into Ctl and writes the trace record for the host.
template <int QS, bool CLUSTER>
__global__ void __launch_bounds__(kPersistBlock) k_rnbp_persist(DevGraph g, float* live, float* cand, float* res,
                                                                uint32_t* vflag, uint32_t* vslot, uint32_t* cstamp,
                                                                Ctl* ctl,
                                                                float eps, RnbpParams prm, CandList cl) {
  auto sync_all = [] {
    if constexpr (CLUSTER)
      cgp::this_cluster().sync();
    else
      cgp::this_grid().sync();
  };
  const uint32_t stride = gridDim.x * blockDim.x;
  // binary lattice: refresh targets are deduplicated by the owner test on
  // per-edge commit stamps instead of an atomic on the target's flag
  const bool own = QS == 1 && g.lat_cols != 0u;
  // Entry slot of this thread within a stride: consecutive 32-entry chunks go
  // to the same warp slot of consecutive CTAs, so a short list spreads over
  // every SM (latency, not one SM's L1/L2 request rate, bounds the phase)
  // while each warp still reads a contiguous chunk.  The trip count stays
  // block-uniform (the stagers flush at block barriers).
  const uint32_t spread = (((threadIdx.x >> 5) * gridDim.x + blockIdx.x) << 5) + (threadIdx.x & 31u);
  // the bookkeeping thread lives in the LAST CTA, which rarely holds list work
  // (lists are short and start at CTA 0), so its global writes stay off the
  // critical path of the iteration
  const bool lead = blockIdx.x == gridDim.x - 1 && threadIdx.x == 0;
  // replicated loop state (identical in every thread of every CTA)
  if (ctl->done || ctl->cl_state != 2u) return;
  __shared__ unsigned s_pacc[6];  // per-CTA sums of one phase (32 bits suffice)
  if (threadIdx.x < 6) s_pacc[threadIdx.x] = 0u;
  unsigned long long it = ctl->iteration;
  unsigned unc = ctl->unconverged, prev = ctl->prev_unconverged, has_prev = ctl->has_prev;
  uint32_t stamp = ctl->stamp;
  unsigned cur = ctl->cl_cur;
  const unsigned long long max_it = ctl->max_iterations;
  // Bernoulli thresholds of both parallelism levels (uniform_unit < p <=> u53 < ceil(p 2^53))
  const unsigned long long th_low = static_cast<unsigned long long>(ceil(ldexp(prm.low_p, 53)));
  const unsigned long long th_high = static_cast<unsigned long long>(ceil(ldexp(prm.high_p, 53)));
  unsigned long long msgs = ctl->msgs_total;
  // the bookkeeping thread's per-launch constants and running sums, kept in
  // registers (written back when the launch returns): no Ctl round trip on
  // its path between the barriers
  const unsigned long long t0_ns = lead ? ctl->t0_ns : 0ull, tlim_ns = lead ? ctl->time_limit_ns : 0ull;
  unsigned long long evals_sum = 0ull, visits_sum = 0ull, bytes_sum = 0ull;
  // reduction buffers indexed by iteration: pacc3[it % 3]
  unsigned long long* pacc3 = ctl->pacc3[0];
  if (lead) {
    for (int b = 0; b < 3; ++b)
      for (int k = 0; k < 6; ++k) ctl->pacc3[b][k] = 0ull;
    ctl->time_stop = 0u;
  }
  sync_all();
  uint32_t list_n = ctl->cl_n[cur];
  // first-pass list entry of this thread, loaded ahead (with the loads after
  // the previous barrier) so the select does not start with a round trip
  uint32_t pre_d = spread < g.D ? (cur ? cl.list[1] : cl.list[0])[spread] : 0u;
  // phase clock of CTA 0, the CTA that holds the most list work (profiling
  // aid, one timer read per phase)
  const bool clk = blockIdx.x == 0 && threadIdx.x == 0;
  // (accumulated in registers and written once when the launch returns: a
  // read-modify-write of Ctl per phase put a dependent global round trip on
  // CTA 0's critical path eight times per iteration)
  unsigned long long tclk = clk ? globaltimer_ns() : 0ull;
  unsigned long long ph[8] = {0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
  auto mark = [&](int k) {
    if (clk) {
      const unsigned long long t = globaltimer_ns();
      ph[k] += t - tclk;
      tclk = t;
    }
  };
  for (;;) {
    const unsigned pb = static_cast<unsigned>(it % 3ull);
    unsigned long long* acc = pacc3 + 6 * pb;
    // ---- select + commit over the candidate list (rnbp_frontier attempt 0).
    // Slot form: entry i's outcome stays at index i -- list[i] keeps the edge
    // if it stays a candidate (else kSlotEmpty), vslot[i] names the target to
    // refresh if this commit flagged it first (else kSlotEmpty) -- so the
    // phase needs no compaction; the refresh compacts both in one flush.
    uint32_t* list = cur ? cl.list[1] : cl.list[0];
    const uint32_t n = list_n;
    {
      unsigned long long thresh = th_high;  // select_parallelism (schedulers.cpp:218-224)
      if (has_prev && prev != 0u) {
        const double ratio = static_cast<double>(unc) / static_cast<double>(prev);
        thresh = ratio > prm.thr ? th_low : th_high;
      }
      if (lead) {  // buffers of the NEXT iteration: last read two barriers ago
        unsigned long long* nx = pacc3 + 6 * static_cast<unsigned>((it + 1) % 3ull);
        for (int k = 0; k < 6; ++k) nx[k] = 0ull;
      }
      Contrib c;
      for (uint32_t base = 0; base < n; base += stride) {
        const uint32_t i = base + spread;
        if (i < n) {
          bool nf = false, kept = false;
          uint32_t tg = 0;
          const uint32_t d = base == 0 ? pre_d : list[i];
          const float r = res[d];
          // binary: the commit's loads (candidate, target) are issued with the
          // residual's, speculatively, saving a dependent round trip
          const float cv = QS == 1 ? cand[d] : 0.f;
          const uint32_t tgp = (QS == 1 && !own) ? __ldg(&g.ep[d ^ 1u]) : 0u;
          c.count += 16;  // algorithmic bytes: list entry + residual, both slots written
          if (r >= eps) {
            c.survivors += 1;
            if ((thresh >= (1ull << 53) || philox_u53(prm.seed, it, 0u, d) < thresh)) {
              cl.inlist[d] = 0;
              if (QS == 1) {  // commit_edge with the prefetched operands
                c.delta -= 1;
                c.frontier += 1;
                res[d] = 0.f;
                live[d] = cv;
                if (own) {  // the slot names the edge; the refresh's owner test dedupes targets
                  cstamp[d] = stamp;
                  tg = d;
                  nf = true;
                } else {
                  tg = tgp;
                  nf = atomicMax(&vflag[tg], stamp) < stamp;
                }
              } else {
                commit_edge<QS>(g, d, r, live, cand, res, eps, vflag, stamp, false, c, nf, tg);
              }
              c.count += 8 * QS + 12;  // candidate -> live, residual, target id, flag
            } else {
              kept = true;
            }
          } else {
            cl.inlist[d] = 0;
          }
          if (!kept) list[i] = kSlotEmpty;
          vslot[i] = nf ? tg : kSlotEmpty;
        }
      }
      mark(7);
      warp_contrib(s_pacc, c);
      __syncthreads();
      pacc_push(s_pacc, acc);
    }
    mark(0);
    sync_all();
    // ---- retry / fallback (schedulers.cpp:204-214): uniform decision, one block
    unsigned long long retry_front = 0;
    // the refresh's first-pass slots, loaded with the retry test's sums
    const uint32_t pre_k = spread < n ? list[spread] : kSlotEmpty;
    uint32_t pre_v = spread < n ? vslot[spread] : kSlotEmpty;
    if (acc[2] == 0ull && acc[3] > 0ull) {
      if (blockIdx.x == 0) {
        // rnbp_retry_block reads the loop state from Ctl: mirror it first
        if (threadIdx.x == 0) {
          ctl->iteration = it;
          ctl->unconverged = unc;
          ctl->prev_unconverged = prev;
          ctl->has_prev = has_prev;
          ctl->stamp = stamp;
          ctl->cl_cur = cur;
          ctl->nflag = 0;
          ctl->frontier = 0;
        }
        __syncthreads();
        rnbp_retry_block<QS, true>(g, live, cand, res, vflag, nullptr, nullptr, ctl, eps, prm, cl, acc[3],
                                   reinterpret_cast<long long*>(&acc[0]), list, n, vslot, own ? cstamp : nullptr);
      }
      sync_all();
      retry_front = ctl->frontier;
      pre_v = spread < n ? vslot[spread] : kSlotEmpty;  // the retry wrote refresh targets
    }
    mark(1);
    // ---- refresh: per slot, carry the kept entry over and refresh the
    // flagged target; new unconverged edges join the list
    {
      if (lead) ctl->cl_n[cur] = 0u;  // the list just read is refilled next iteration
      BPB_STAGER(st, 2048, cur ? cl.list[0] : cl.list[1], &ctl->cl_n[cur ^ 1u]);
      st.init();
      int cnt = 0;
      unsigned long long evals = 0, visits = 0, kept = 0, slots = 0;
      for (uint32_t base = 0; base < n; base += stride) {
        const uint32_t i = base + spread;
        if (i < n) {
          ++slots;
          const uint32_t d = base == 0 ? pre_k : list[i], v = base == 0 ? pre_v : vslot[i];
          if (d != kSlotEmpty) {
            st.push(d);
            ++kept;
          }
          if (v != kSlotEmpty && own) {  // v = the committed edge
            bool skipped = false;
            cnt += vertex_update<QS, kModeDelta, true, false>(g, lattice_edge_target(g, v), live, cand, res, eps,
                                                              &ctl->numeric_error, evals, cl.inlist, &st, true,
                                                              cstamp, stamp, v, &skipped);
            visits += skipped ? 0u : 1u;
          } else if (v != kSlotEmpty) {
            cnt += vertex_update<QS, kModeDelta, true, false>(g, v, live, cand, res, eps, &ctl->numeric_error,
                                                              evals, cl.inlist, &st, true);
            ++visits;
          }
        }
        st.flush(1024);
      }
      mark(4);
      Contrib c;
      c.delta = cnt;
      c.evals = evals;
      c.visits = visits;
      // per slot: two slot words; per kept entry: list write; per vertex:
      // unary; per message: edge pair (in + old out), coupling, candidate
      // write, residual read + write
      c.count = 8ull * slots + 4ull * kept + 4ull * visits +
                static_cast<unsigned long long>(8 * QS + 4 + 4 * QS + 8) * evals;
      warp_contrib(s_pacc, c);
      flush_final(st);  // its first barrier orders the warp sums
      mark(5);
      pacc_push(s_pacc, acc);
      mark(6);
      if (lead && globaltimer_ns() - t0_ns >= tlim_ns) ctl->time_stop = 1u;
    }
    mark(2);
    sync_all();
    // ---- finalize (fin_iter), replicated: converged check before the caps
    const long long delta = static_cast<long long>(acc[0]);
    const unsigned long long frontier = acc[2] + retry_front;
    const unsigned start = unc;
    unc = static_cast<unsigned>(static_cast<long long>(start) + delta);
    prev = start;  // set_prev_unconverged (schedulers.cpp:327)
    has_prev = 1u;
    msgs += frontier;
    // the list refilled this iteration: loaded with the other finalize reads,
    // reused by the next select
    const uint32_t next_n = ctl->cl_n[cur ^ 1u];
    pre_d = spread < g.D ? (cur ? cl.list[0] : cl.list[1])[spread] : 0u;  // the next iteration's list
    const bool numeric = ctl->numeric_error != 0u;
    const bool tstop = ctl->time_stop != 0u;
    if (lead) {
      fin_record(ctl, it, frontier, unc, t0_ns);
      evals_sum += acc[4];
      visits_sum += acc[5];
      bytes_sum += acc[1];
      ctl->survivors = acc[3];
    }
    it += 1;
    stamp += 1u;
    cur ^= 1u;
    bool done = false;
    unsigned reason = kStopNone;
    if (numeric) {
      done = true;
      reason = kStopNumeric;
    } else if (unc == 0u) {
      done = true;
      reason = kStopConverged;
    } else if (it >= max_it) {
      done = true;
      reason = kStopMaxIter;
    } else if (tstop) {
      done = true;
      reason = kStopTime;
    }
    mark(3);
    // barrier flavour no longer fits the list length: hand back to the host,
    // which relaunches with the other one (hysteresis around the host's
    // kPersistClusterList choice)
    list_n = next_n;
    const bool switch_mode = CLUSTER ? next_n > 2u * kPersistClusterList : next_n < kPersistClusterList / 2u;
    if (done || switch_mode) {
      if (clk)
#pragma unroll
        for (int k = 0; k < 8; ++k) ctl->phase_ns[k] += ph[k];
      if (lead) {  // mirror the loop state for the host
        ctl->evals_total += evals_sum;
        ctl->vertex_visits += visits_sum;
        ctl->persist_bytes += bytes_sum;
        ctl->iteration = it;
        ctl->unconverged = unc;
        ctl->prev_unconverged = prev;
        ctl->has_prev = has_prev;
        ctl->stamp = stamp;
        ctl->cl_cur = cur;
        ctl->msgs_total = msgs;
        ctl->frontier = 0;
        ctl->nflag = 0;
        if (done) {
          ctl->done = 1u;
          ctl->converged = reason == kStopConverged ? 1u : 0u;
          ctl->stop_reason = reason;
        }
      }
      return;
    }
  }
}

}  // namespace bpb
