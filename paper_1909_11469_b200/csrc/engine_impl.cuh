// EngineT<QS>: per-run device state + the scheduler loop of run()
// (schedulers.cpp:293-353), executed as a device-side CUDA-graph WHILE loop so
// no host round trip happens per iteration.  Instantiated once per message
// stride in engine_q*.cu (parallel builds).
#pragma once
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>

#include "engine.hpp"
#include "host_pool.hpp"
#include "kernels.cuh"
#include "kernels_rs.cuh"
#include "kernels_persist.cuh"
#include "kernels_lbp.cuh"
#include "kernels_fused.cuh"
#include "kernels_fused_tma.cuh"

namespace bpb {
namespace {

using Clock = std::chrono::steady_clock;

// smallest float >= eps: r (fp32) >= eps (fp64) <=> r >= eps_ceil
float eps_ceil(double eps) {
  float f = static_cast<float>(eps);
  if (static_cast<double>(f) < eps) f = std::nextafter(f, std::numeric_limits<float>::infinity());
  return f;
}

// SM count of the current device (cached per ordinal)
int sm_count() {
  static std::mutex mu;
  static std::map<int, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int c = 148;
  cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
  return cache[dev] = c > 0 ? c : 148;
}

unsigned grid_cap(size_t n, int per_sm = 8) {
  const size_t want = (n + kBlock - 1) / kBlock;
  const size_t cap = static_cast<size_t>(sm_count()) * per_sm;
  return static_cast<unsigned>(std::max<size_t>(1, std::min(want, cap)));
}

enum KClass { kKUpdate = 0, kKSelect = 1, kKTopk = 2, kKSplash = 3, kKInit = 4, kKBeliefs = 5, kKOther = 6,
              kKPersist = 7, kKFused = 8 };

template <int QS>
class EngineT final : public EngineBase {
 public:
  // engine buffers: zero-filled on the engine stream (a cached block's
  // synchronous memset + device sync per buffer was ~0.3 ms of every run)
  void zalloc(DevBuf& b, size_t n) {
    b.alloc_async(n, s_);
    cuda_check(cudaMemsetAsync(b.p, 0, b.bytes, s_), "memset");
  }
  EngineT(const GraphImpl& g, const bp_sched_config& cfg) : g_(g), cfg_(cfg) {
    cuda_check(cudaSetDevice(g.device), "cudaSetDevice");
    cuda_check(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking), "stream");
    dg_ = g.dev();
    eps_ = eps_ceil(cfg.epsilon);
    const size_t msz = static_cast<size_t>(g.D) * QS * sizeof(float);
    zalloc(bufA_, msz);
    zalloc(bufB_, msz);
    zalloc(res_, (static_cast<size_t>(g.D) + 3) / 4 * 16);  // padded to float4, tail stays 0
    zalloc(vflag_, static_cast<size_t>(g.V) * 4);
    if (cfg.kind == BP_RNBP) {  // candidate list (run mode)
      zalloc(clist_[0], static_cast<size_t>(g.D) * 4);
      zalloc(clist_[1], static_cast<size_t>(g.D) * 4);
      zalloc(inlist_, g.D ? g.D : 1);
      zalloc(vslot_, static_cast<size_t>(g.D ? g.D : 1) * 4);  // here, not mid-run: cudaMalloc can stall the device
      zalloc(cstamp_, static_cast<size_t>(g.D ? g.D : 1) * 4);
    }
    zalloc(vlist_, static_cast<size_t>(g.V) * 4);
    if (fused_capable()) {  // scratch buffer set of the fused dense RnBP sweep (here, not mid-run)
      zalloc(fc_, msz);
      zalloc(fu_[0], g.D);
      zalloc(fu_[1], g.D);
    }
    zalloc(ctl_, sizeof(Ctl));
    hctl_ = static_cast<Ctl*>(pinned_acquire(sizeof(Ctl)));
    std::memset(hctl_, 0, sizeof(Ctl));
    if (cfg.kind == BP_RBP) {
      zalloc(hist_, kRadixBins * 4);
      nchunks_ = std::max<uint32_t>(1, (g.D + kTieChunk - 1) / kTieChunk);
      zalloc(chunk_, static_cast<size_t>(nchunks_) * 4);
      zalloc(rx_list_, std::max<size_t>(g.D, 1) * 4);
      const long long kr = std::llround(cfg.p * static_cast<double>(g.D));  // schedulers.cpp:124
      k_ = kr < 1 ? 1 : static_cast<uint64_t>(kr);
    }
    if (cfg.kind == BP_RS) ensure_rs(cfg.splash_depth);
    prm_.seed = cfg.seed;
    prm_.low_p = cfg.low_p;
    prm_.high_p = cfg.high_p;
    prm_.thr = cfg.edge_ratio_threshold;
    prm_.fixed_p = -1.0;
    prm_.commit = 1;
    prm_.attempt = 0;
    // the set-up memsets above ran on the legacy stream, which the engine's
    // non-blocking stream does not wait for
    cuda_check(cudaDeviceSynchronize(), "engine set-up");
  }

  ~EngineT() override {
    if (gexec_) cudaGraphExecDestroy(gexec_);
    if (graph_) cudaGraphDestroy(graph_);
    if (fgexec_) cudaGraphExecDestroy(fgexec_);
    if (fgraph_) cudaGraphDestroy(fgraph_);
    for (auto& ev : evs_) cudaEventDestroy(ev);
    // back to the process-wide pool: cudaFreeHost was measured at 75-750 ms
    // on some calls (page unpinning), on the end-to-end path of every run
    if (s_) cudaStreamSynchronize(s_);  // no copy into / out of the mirror may be in flight
    if (hctl_) pinned_release(hctl_, sizeof(Ctl));
    if (s_) cudaStreamDestroy(s_);
  }

  // ------------------------------------------------------------------ run
  void run(const bp_run_opts* opts, bp_run_result* res, double* beliefs_host, bp_iter_record* trace,
           uint64_t trace_cap) override {
    const uint32_t flags = opts ? opts->flags : 0u;
    timing_ = (flags & BP_RUN_KERNEL_TIMING) != 0;
    fused_iters_ = fused_sweeps_ = 0;
    stats_ = opts ? opts->stats : nullptr;
    if (stats_) std::memset(stats_, 0, sizeof(*stats_));
    launches_ = 0;
    const bool use_graph = !(flags & BP_RUN_NO_GRAPHS) && !timing_;
    persist_ = cfg_.kind == BP_RNBP && !(flags & BP_RUN_NO_PERSIST);
    lbp_force_ = flags & (BP_RUN_LBP_TMA | BP_RUN_LBP_TILES | BP_RUN_LBP_VERTEX);
    if (gexec_ && lbp_force_ != graph_force_) {  // the captured loop body embeds the sweep choice
      cudaGraphExecDestroy(gexec_);
      cudaGraphDestroy(graph_);
      gexec_ = nullptr;
      graph_ = nullptr;
    }
    graph_force_ = lbp_force_;
    const Clock::time_point t0 = Clock::now();  // schedulers.cpp:297

    cudaEvent_t e0, e1;
    cuda_check(cudaEventCreate(&e0), "event");
    cuda_check(cudaEventCreate(&e1), "event");
    cuda_check(cudaEventRecord(e0, s_), "event record");
    reset_ctl(cfg_.max_iterations, cfg_.time_limit, cfg_.kind == BP_RNBP, persist_);
    enqueue_init(cfg_.kind == BP_LBP);

    uint64_t copied = 0;
    // first look: did the initial sweep already converge / hit a cap?  (The
    // device loop checks that itself, so the graph path skips the round trip.)
    if (!use_graph) {
      fetch_ctl_header();
      drain_trace(trace, trace_cap, copied);
    }
    // RnBP on binary Ising lattices: the dense iterations as fused sweeps
    if (fused_capable() && !(flags & BP_RUN_NO_FUSED) && prm_.fixed_p < 0.0 && !hctl_->done) {
      const uint32_t ff = flags & (BP_RUN_FUSED_TMA | BP_RUN_FUSED_REGS);
      if (fgexec_ && ff != fused_force_) {  // the captured body embeds the kernel choice
        cudaGraphExecDestroy(fgexec_);
        cudaGraphDestroy(fgraph_);
        fgexec_ = nullptr;
        fgraph_ = nullptr;
      }
      fused_force_ = ff;
      run_fused_phase(use_graph, opts, trace, trace_cap, copied);
    }
    if (!hctl_->done) {
      if (use_graph) {
        run_graph_loop(trace, trace_cap, copied);
      } else {
        uint32_t batch = opts && opts->batch ? opts->batch : 16;
        while (!hctl_->done && !handover()) {
          for (uint32_t b = 0; b < batch; ++b) enqueue_iteration();
          fetch_ctl_header();
          drain_trace(trace, trace_cap, copied);
          if (!(opts && opts->batch)) batch = std::min<uint32_t>(batch * 2, 256);
        }
      }
      if (!hctl_->done && handover()) run_persist_loop(trace, trace_cap, copied);
    }
    fetch_ctl_header();
    drain_trace(trace, trace_cap, copied);
    if (hctl_->numeric_error) throw Error(BP_ERR_NUMERIC, "probability vector collapsed (total mass below 1e-300 or non-finite)");

    if (opts && opts->messages_host)  // LBP reports m_t, which lives in buf[t & 1]
      read_messages(opts->messages_host, cfg_.kind == BP_LBP && (hctl_->iteration & 1ull));
    const size_t nb = g_.unary_size();
    if (!(flags & BP_RUN_NO_BELIEFS) && (beliefs_host || (opts && opts->beliefs_device))) {
      double* dst = opts && opts->beliefs_device ? opts->beliefs_device : nullptr;
      if (!dst) {
        ensure_beliefs_buf(nb);
        dst = bel_.as<double>();
      }
      enqueue_beliefs(dst, cfg_.kind == BP_LBP);
      if (beliefs_host) {
        // large tables through a pinned block (full-rate DMA), then copied out
        // on the host pool; small ones straight into the caller's memory
        if (nb * 8 >= kPinnedBeliefs) {
          bel_pinned_bytes_ = ((nb * 8 + (1u << 20) - 1) >> 20) << 20;
          bel_pinned_ = pinned_acquire(bel_pinned_bytes_);
          cuda_check(cudaMemcpyAsync(bel_pinned_, dst, nb * 8, cudaMemcpyDeviceToHost, s_), "beliefs d2h");
        } else {
          cuda_check(cudaMemcpyAsync(beliefs_host, dst, nb * 8, cudaMemcpyDeviceToHost, s_), "beliefs d2h");
        }
      }
    }
    cuda_check(cudaEventRecord(e1, s_), "event record");
    cuda_check(cudaStreamSynchronize(s_), "run");
    if (bel_pinned_) {
      const char* src = static_cast<const char*>(bel_pinned_);
      char* out = reinterpret_cast<char*>(beliefs_host);
      parallel_for(nb * 8, [&](uint64_t a, uint64_t b) { std::memcpy(out + a, src + a, b - a); });
      pinned_release(bel_pinned_, bel_pinned_bytes_);
      bel_pinned_ = nullptr;
    }
    if (g_.check_collapse) {  // compute_belief's mass check (k_beliefs) on collapse-checked models
      fetch_ctl_header();
      if (hctl_->numeric_error) throw Error(BP_ERR_NUMERIC, "probability vector collapsed (total mass below 1e-300)");
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    collect_timing();
    if (stats_) {
      stats_->bytes[kKPersist] = hctl_->persist_bytes;
      // fused sweep (kernels_fused.cuh): per edge pair live + candidate read and
      // written (2 x 16 B), predicates (2 x 2 B), coupling 4 B; unary 4 B per vertex
      stats_->bytes[kKFused] = fused_sweeps_ * (40ull * g_.E + 4ull * g_.V);
    }

    std::memset(res, 0, sizeof(*res));
    res->converged = hctl_->converged ? 1 : 0;
    res->iterations = hctl_->iteration;
    res->messages_updated_total = hctl_->msgs_total;
    res->trace_len = hctl_->trace_len;
    res->device_ms = ms;
    res->message_evaluations = hctl_->evals_total;
    res->vertex_visits = hctl_->vertex_visits;
    res->splashes = hctl_->splashes;
    res->splash_rounds = hctl_->rs_rounds;
    res->persist_iterations =
        persist_ && hctl_->handover_it && hctl_->iteration > hctl_->handover_it ? hctl_->iteration - hctl_->handover_it : 0;
    res->fused_iterations = fused_iters_;
    res->gpu_launches = launches_;
    res->wall_time = std::chrono::duration<double>(Clock::now() - t0).count();
  }

  // ------------------------------------------------------------- lockstep
  void lockstep_init() override {
    reset_ctl(std::numeric_limits<uint64_t>::max(), 1e300);
    enqueue_init(false);
    sync();
  }
  uint32_t unconverged() override {
    fetch_ctl_header();
    return hctl_->unconverged;
  }
  uint64_t iteration() override {
    fetch_ctl_header();
    return hctl_->iteration;
  }
  // the iteration keys the Philox draws of rnbp_frontier (the reference's
  // draws advance with its mt19937_64 instead)
  void advance_iteration() override {
    fetch_ctl_header();
    k_set_u64<<<1, 1, 0, s_>>>(&ctl()->iteration, hctl_->iteration + 1);
    launch_check();
    sync();
  }
  void messages(double* out, bool candidates) override {
    // fused LBP sweeps (lockstep, bands) ping-pong like run()'s LBP: m_t lives in buf[t & 1]
    bool flip = false;
    if (pingpong_ && cfg_.kind == BP_LBP) {
      fetch_ctl_header();
      flip = (hctl_->iteration & 1ull) != 0;
    }
    read_messages(out, candidates != flip);
  }
  // the messages of one buffer (A = live, B = candidates / the other ping-pong
  // buffer) as fp64 probabilities in MessageStore order
  void read_messages(double* out, bool buf_b) {
    std::vector<float> raw(static_cast<size_t>(g_.D) * QS);
    const DevBuf& src = buf_b ? bufB_ : bufA_;
    if (!raw.empty()) cuda_check(cudaMemcpyAsync(raw.data(), src.p, raw.size() * 4, cudaMemcpyDeviceToHost, s_), "d2h");
    sync();
    const auto& ep = g_.host_ep();
    size_t o = 0;
    for (uint32_t d = 0; d < g_.D; ++d) {
      if (QS == 1) {
        const double l = raw[d];
        out[o++] = 1.0 / (1.0 + std::exp2(l));  // base-2 log-odds
        out[o++] = 1.0 / (1.0 + std::exp2(-l));
      } else {
        const uint32_t q = g_.card_of(ep[d ^ 1u]);
        for (uint32_t x = 0; x < q; ++x) out[o++] = std::exp2(static_cast<double>(raw[static_cast<size_t>(d) * QS + x]));
      }
    }
  }
  void residuals(double* out) override {
    std::vector<float> raw(g_.D);
    if (g_.D) cuda_check(cudaMemcpyAsync(raw.data(), res_.p, raw.size() * 4, cudaMemcpyDeviceToHost, s_), "d2h");
    sync();
    for (uint32_t d = 0; d < g_.D; ++d) out[d] = raw[d];
  }
  void beliefs(double* out) override {
    const size_t nb = g_.unary_size();
    ensure_beliefs_buf(nb);
    enqueue_beliefs(bel_.as<double>(), pingpong_ && cfg_.kind == BP_LBP);
    cuda_check(cudaMemcpyAsync(out, bel_.p, nb * 8, cudaMemcpyDeviceToHost, s_), "d2h");
    sync();
  }
  void apply_frontier(const uint32_t* f, uint64_t n) override {
    if (n == 0) return;  // schedulers.cpp:230
    std::vector<uint32_t> u(f, f + n);
    for (uint32_t d : u)
      if (d >= g_.D) throw_invalid("frontier edge out of range");
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end()), u.end());
    DevBuf list;
    list.upload(u.data(), u.size() * 4);
    force_not_done();
    const int dense = u.size() > g_.V / 16 ? 1 : 0;
    k_commit_list<QS><<<grid_cap(u.size()), kBlock, 0, s_>>>(dg_, list.as<uint32_t>(), static_cast<uint32_t>(u.size()),
                                                            live(), cand(), res_.as<float>(), vflag_.as<uint32_t>(),
                                                            vlist_.as<uint32_t>(), ctl(), eps_, dense);
    launch_check();
    enqueue_refresh(kFinApply);
    sync();
  }
  void rnbp_frontier(double p, std::vector<uint32_t>& out) override {
    ensure_sel();
    force_not_done();
    RnbpParams q = prm_;
    q.fixed_p = p;
    q.commit = 0;
    k_rnbp_select<QS, false><<<grid_cap(g_.D / 4 + 1), kBlock, 0, s_>>>(
        dg_, live(), cand(), res_.as<float>(), vflag_.as<uint32_t>(), vlist_.as<uint32_t>(), sel_.as<uint8_t>(),
        ctl(), eps_, q, cand_list(), 1);
    launch_check();
    collect_sel(out);
  }
  void rbp_frontier(double p, std::vector<uint32_t>& out) override {
    ensure_sel();
    force_not_done();
    const long long kr = std::llround(p * static_cast<double>(g_.D));
    const uint64_t k = kr < 1 ? 1 : static_cast<uint64_t>(kr);
    ensure_rbp_scratch();
    enqueue_topk(k, /*commit=*/0);
    collect_sel(out);
  }
  // rs_frontier (schedulers.cpp:169-192): the device builds the splashes;
  // the host only serialises them in the reference's layout (roots in
  // priority order, edges in BFS visit order, schedulers.cpp:160-165).
  void rs_frontier(double p, uint32_t h, std::vector<uint32_t>& roots, std::vector<uint64_t>& eoff,
                   std::vector<uint32_t>& edges) override {
    roots.clear();
    edges.clear();
    eoff.assign(1, 0);
    if (g_.V == 0) return;
    ensure_rs(h);
    force_not_done();
    launch_rs(rs_k(p), h, /*apply=*/0);
    sync();
    RsCtl rc{};
    cuda_check(cudaMemcpy(&rc, rs_ctl_.p, sizeof(RsCtl), cudaMemcpyDeviceToHost), "d2h");
    std::vector<uint32_t> kept(rc.nkept), qnext(g_.V);
    std::vector<float> vres(g_.V);
    if (rc.nkept) cuda_check(cudaMemcpy(kept.data(), rs_klist_.p, 4ull * rc.nkept, cudaMemcpyDeviceToHost), "d2h");
    cuda_check(cudaMemcpy(qnext.data(), rs_qnext_.p, 4ull * g_.V, cudaMemcpyDeviceToHost), "d2h");
    cuda_check(cudaMemcpy(vres.data(), rs_vres_.p, 4ull * g_.V, cudaMemcpyDeviceToHost), "d2h");
    std::sort(kept.begin(), kept.end(), [&](uint32_t a, uint32_t b) {
      if (vres[a] != vres[b]) return vres[a] > vres[b];
      return a < b;
    });
    const auto& off = g_.host_in_off();
    const auto& adj = g_.host_in_adj();
    for (uint32_t r : kept) {
      roots.push_back(r);
      for (uint32_t v = r; v != kUncl; v = qnext[v])
        for (uint32_t a = off[v]; a < off[v + 1]; ++a) edges.push_back(adj[a] ^ 1u);
      eoff.push_back(edges.size());
    }
  }
  // apply_splash_frontier (schedulers.cpp:253-291) for host-supplied splashes
  void apply_splashes(uint64_t ns, const uint32_t* roots, const uint64_t* eoff, const uint32_t* edges) override {
    (void)roots;
    if (ns == 0 || eoff[ns] == eoff[0]) return;
    const uint64_t n = eoff[ns] - eoff[0];
    std::vector<uint32_t> all(edges + eoff[0], edges + eoff[ns]);
    for (uint32_t d : all)
      if (d >= g_.D) throw_invalid("splash edge out of range");
    {
      std::vector<uint32_t> check(all);
      std::sort(check.begin(), check.end());
      if (std::adjacent_find(check.begin(), check.end()) != check.end())
        throw_model("overlapping splashes: an edge is updated by two splashes");  // schedulers.cpp:262-268
    }
    ensure_rs(0);
    if (!rs_written_.p) {
      rs_written_.alloc(static_cast<size_t>(g_.D) * 4);
      cuda_check(cudaMemset(rs_written_.p, 0, rs_written_.bytes), "memset");
      cuda_check(cudaDeviceSynchronize(), "memset");  // legacy stream: not ordered before s_
    }
    std::vector<unsigned long long> off(ns + 1);
    for (uint64_t i = 0; i <= ns; ++i) off[i] = eoff[i] - eoff[0];
    DevBuf doff, dedges;
    doff.upload(off.data(), off.size() * 8);
    dedges.upload(all.data(), all.size() * 4);
    force_not_done();
    k_splash_apply_edges<QS><<<static_cast<unsigned>((ns + kBlock - 1) / kBlock), kBlock, 0, s_>>>(
        dg_, live(), rs_shadow_.as<float>(), rs_written_.as<uint32_t>(), doff.as<unsigned long long>(),
        dedges.as<uint32_t>(), static_cast<uint32_t>(ns), rs_stamp_ + 1, &ctl()->numeric_error);
    rs_stamp_ += static_cast<uint32_t>(ns);
    launch_check();
    k_splash_commit_edges<QS><<<static_cast<unsigned>((n + kBlock - 1) / kBlock), kBlock, 0, s_>>>(
        dg_, live(), rs_shadow_.as<float>(), dedges.as<uint32_t>(), static_cast<uint32_t>(n),
        vflag_.as<uint32_t>(), vlist_.as<uint32_t>(), ctl());
    launch_check();
    enqueue_refresh(kFinApply);
    sync();
    fetch_ctl_header();
    if (hctl_->numeric_error) throw Error(BP_ERR_NUMERIC, "probability vector collapsed (total mass below 1e-300 or non-finite)");
  }
  // One fused LBP sweep exactly as run() executes it (the production kernel
  // for this graph, or the one the flags force): sweep t reads m_t, writes
  // m_{t+1} = f(m_t) and counts r(m_t) >= eps.  Afterwards messages() = m_t,
  // candidates() = m_{t+1}, unconverged() = #{r(m_t) >= eps}, iteration() = t
  // -- the reference's EngineState after t apply_frontier(frontier_lbp())
  // calls (schedulers.cpp:99-103, 226-251).
  uint32_t lbp_sweep(uint32_t flags) override {
    if (cfg_.kind != BP_LBP) throw_invalid("lbp_sweep on a non-LBP engine");
    if (band_owned_) throw_invalid("lbp_sweep on a band engine (use bp_band_lbp_sweep)");
    lbp_force_ = flags & (BP_RUN_LBP_TMA | BP_RUN_LBP_TILES | BP_RUN_LBP_VERTEX);
    if (!pingpong_) {
      reset_ctl(std::numeric_limits<uint64_t>::max(), 1e300);
      const unsigned gi = grid_cap(static_cast<size_t>(g_.D) * QS);
      k_init_messages<QS><<<gi, kBlock, 0, s_>>>(dg_, live(), ctl(), 1);
      launch_check();
      pingpong_ = true;
    }
    enqueue_lbp_sweep(kFinLbp);
    sync();
    fetch_ctl_header();
    if (hctl_->numeric_error) throw Error(BP_ERR_NUMERIC, "probability vector collapsed (total mass below 1e-300 or non-finite)");
    return lbp_kernel_;
  }

  uint64_t step() override {
    force_not_done();
    fetch_ctl_header();
    const uint64_t before = hctl_->msgs_total;
    if (cfg_.kind == BP_LBP) {
      // lockstep LBP = frontier_lbp + apply_frontier (commit all + refresh all)
      ensure_rbp_scratch();
      enqueue_topk_all();
      enqueue_refresh(kFinIter);
      sync();
    } else {
      enqueue_iteration();
    }
    fetch_ctl_header();
    return hctl_->msgs_total - before;
  }

 private:
  float* live() { return bufA_.as<float>(); }
  float* cand() { return bufB_.as<float>(); }
  Ctl* ctl() { return ctl_.as<Ctl>(); }

  void sync() { cuda_check(cudaStreamSynchronize(s_), "stream sync"); }
  void launch_check() { cuda_check(cudaGetLastError(), "kernel launch"); }

  CandList cand_list() {
    CandList c{};
    c.list[0] = clist_[0].as<uint32_t>();
    c.list[1] = clist_[1].as<uint32_t>();
    c.inlist = inlist_.as<uint8_t>();
    return c;
  }

  void reset_ctl(uint64_t max_iter, double time_limit, bool use_clist = false, bool persist = false) {
    use_clist_ = use_clist && clist_[0].p != nullptr;
    std::memset(hctl_, 0, offsetof(Ctl, trace));
    hctl_->use_clist = use_clist_ ? 1u : 0u;
    hctl_->persist_ok = use_clist_ && persist ? 1u : 0u;
    if (use_clist_) cuda_check(cudaMemsetAsync(inlist_.p, 0, inlist_.bytes, s_), "memset inlist");
    if (use_clist_ && persist) cuda_check(cudaMemsetAsync(cstamp_.p, 0, cstamp_.bytes, s_), "memset cstamp");
    hctl_->max_iterations = max_iter;
    const double ns = time_limit * 1e9;
    hctl_->time_limit_ns = ns >= 1.8e19 ? std::numeric_limits<unsigned long long>::max()
                                        : static_cast<unsigned long long>(ns);
    hctl_->stamp = 1;
    cuda_check(cudaMemcpyAsync(ctl_.p, hctl_, offsetof(Ctl, trace), cudaMemcpyHostToDevice, s_), "ctl h2d");
    cuda_check(cudaMemsetAsync(vflag_.p, 0, static_cast<size_t>(g_.V) * 4, s_), "memset vflag");
  }

  void fetch_ctl_header() {
    cuda_check(cudaMemcpyAsync(hctl_, ctl_.p, offsetof(Ctl, trace), cudaMemcpyDeviceToHost, s_), "ctl d2h");
    sync();
  }

  void force_not_done() {
    const unsigned zero = 0;
    cuda_check(cudaMemcpyAsync(reinterpret_cast<char*>(ctl_.p) + offsetof(Ctl, done), &zero, 4,
                               cudaMemcpyHostToDevice, s_),
               "ctl h2d");
    sync();
  }

  // copy trace records [copied, trace_len) from the device ring
  void drain_trace(bp_iter_record* trace, uint64_t cap, uint64_t& copied) {
    const uint64_t n = hctl_->trace_len;
    if (n <= copied) return;
    if (!trace || copied >= cap) {
      copied = n;
      return;
    }
    if (n - copied > kTraceRing) throw Error(BP_ERR_CUDA, "trace ring overrun");
    // only the new records: at most two contiguous pieces of the ring
    std::vector<TraceRec> tmp(kTraceRing);
    const uint64_t last = std::min(n, cap);
    for (uint64_t it = copied; it < last;) {
      const uint64_t slot = it % kTraceRing, len = std::min<uint64_t>(last - it, kTraceRing - slot);
      cuda_check(cudaMemcpy(tmp.data() + slot,
                            reinterpret_cast<char*>(ctl_.p) + offsetof(Ctl, trace) + sizeof(TraceRec) * slot,
                            sizeof(TraceRec) * len, cudaMemcpyDeviceToHost),
                 "trace d2h");
      it += len;
    }
    for (uint64_t it = copied; it < n && it < cap; ++it) {
      const TraceRec& r = tmp[it % kTraceRing];
      trace[it].iteration = r.iteration;
      trace[it].frontier_size = r.frontier_size;
      trace[it].unconverged = r.unconverged;
      trace[it]._pad = 0;
      trace[it].elapsed_seconds = r.elapsed_seconds;
    }
    copied = n;
  }

  // ---- kernel timing (BP_RUN_KERNEL_TIMING): an event pair per launch
  struct Timed {
    int cls;
    cudaEvent_t a, b;
    uint64_t bytes;
  };
  std::vector<Timed> pending_;
  std::vector<cudaEvent_t> evs_;
  size_t ev_next_ = 0;
  cudaEvent_t next_event() {
    if (ev_next_ == evs_.size()) {
      cudaEvent_t ev;
      cuda_check(cudaEventCreate(&ev), "event");
      evs_.push_back(ev);
    }
    return evs_[ev_next_++];
  }
  template <class F>
  void timed(int cls, F&& launch) {
    ++launches_;
    if (!timing_) {
      launch();
      return;
    }
    Timed t{cls, next_event(), next_event(), 0};
    cudaEventRecord(t.a, s_);
    launch();
    cudaEventRecord(t.b, s_);
    pending_.push_back(t);
    if (ev_next_ > 4096) collect_timing();
  }
  void collect_timing() {
    if (pending_.empty()) return;
    sync();
    for (auto& t : pending_) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, t.a, t.b);
      if (stats_) {
        stats_->ms[t.cls] += ms;
        stats_->launches[t.cls] += 1;
      }
    }
    pending_.clear();
    ev_next_ = 0;
  }

  // resident grid for a grid-stride kernel: blocks/SM from the occupancy
  // calculator x SMs (one wave, no tail), capped by the work
  std::map<const void*, int> occ_;
  template <class K>
  unsigned vgrid(K kern, size_t items) {
    auto it = occ_.find(reinterpret_cast<const void*>(kern));
    int per = 0;
    if (it == occ_.end()) {
      cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kBlock, 0), "occupancy");
      occ_[reinterpret_cast<const void*>(kern)] = per;
    } else {
      per = it->second;
    }
    const size_t want = (items + kBlock - 1) / kBlock;
    return static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>(want, static_cast<size_t>(std::max(per, 1)) * sm_count())));
  }

  // one LBP sweep (ping-pong): the SMEM-staged lattice kernel for binary Ising
  // lattices, the vertex-centric kernel otherwise
  unsigned lbp_grid_ = 0;
  static constexpr uint64_t kLbpTmaMinVertices = uint64_t{1} << 21;  // TMA = tiles at 1000^2, 7% faster at 2048^2, 22% at 8192^2
  uint32_t lbp_force_ = 0;   // BP_RUN_LBP_TMA / BP_RUN_LBP_TILES of the current call
  uint32_t lbp_kernel_ = 0;  // BP_LBP_KERNEL_* of the last sweep
  // TMA-staged rows pay off once the grid is far beyond L2; below that the
  // register-tiled lattice kernel (k_vertex_update) is faster.  The per-call
  // flags BP_RUN_LBP_TMA / BP_RUN_LBP_TILES override the size rule.
  bool lbp_uses_tma() const {
    const bool tma_ok = QS == 1 && g_.lat_cols && g_.par_mode == 1 && g_.lat_rows >= 2;
    const bool big = static_cast<uint64_t>(g_.V) >= kLbpTmaMinVertices;
    return tma_ok && ((lbp_force_ & BP_RUN_LBP_TMA) || (!(lbp_force_ & BP_RUN_LBP_TILES) && big));
  }
  // fin: the loop control fused into the sweep's last block (kFinNone: none)
  void enqueue_lbp_sweep(int fin) {
    const FinArgs fa{fin, g_.D};
    if (lbp_uses_tma()) {
      lbp_kernel_ = BP_LBP_KERNEL_TMA;
      if (!lbp_grid_) {
        cuda_check(cudaFuncSetAttribute(k_lbp_lattice, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(sizeof(LbpSmem))),
                   "smem attribute");
        int per = 0;
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_lbp_lattice, kBlock, sizeof(LbpSmem)),
                   "occupancy");
        lbp_grid_ = static_cast<unsigned>(std::max(1, per) * sm_count());
      }
      timed(kKUpdate, [&] {
        k_lbp_lattice<<<lbp_grid_, kBlock, sizeof(LbpSmem), s_>>>(dg_, live(), cand(), ctl(), eps_);
      });
      // separate finalize: the fused one's static shared memory would cost the
      // TMA sweep its third resident block per SM (2.66 -> 3.10 ms at 16384^2)
      if (fin != kFinNone) enqueue_finalize(fin);
    } else if constexpr (QS == 4 || QS == 8) {
      if (g_.lat_cols && g_.uniform_q && !g_.check_collapse && !(lbp_force_ & BP_RUN_LBP_VERTEX)) {
        // q-state lattice: four states per lane (k_lattice_qsweep)
        lbp_kernel_ = BP_LBP_KERNEL_QLANES;
        if (g_.par_mode) {
          const unsigned grid = vgrid(k_lattice_qsweep<QS, true, kModeCount>, static_cast<size_t>(g_.V) * (QS / 4));
          timed(kKUpdate, [&] {
            k_lattice_qsweep<QS, true, kModeCount><<<grid, kBlock, 0, s_>>>(dg_, live(), cand(), nullptr, nullptr,
                                                                          nullptr, ctl(), eps_, fa);
          });
        } else {
          const unsigned grid = vgrid(k_lattice_qsweep<QS, false, kModeCount>, static_cast<size_t>(g_.V) * (QS / 4));
          timed(kKUpdate, [&] {
            k_lattice_qsweep<QS, false, kModeCount><<<grid, kBlock, 0, s_>>>(dg_, live(), cand(), nullptr, nullptr,
                                                                           nullptr, ctl(), eps_, fa);
          });
        }
      } else {
        lbp_kernel_ = BP_LBP_KERNEL_VERTEX;
        timed(kKUpdate, [&] {
          k_vertex_update<QS, kModeCount, false, true, false>
              <<<vgrid(k_vertex_update<QS, kModeCount, false, true, false>, g_.V), kBlock, 0, s_>>>(
                  dg_, live(), cand(), nullptr, nullptr, nullptr, ctl(), eps_, cand_list(), fa);
        });
      }
    } else {
      lbp_kernel_ = (QS == 1 && g_.lat_cols && g_.par_mode) ? BP_LBP_KERNEL_TILES : BP_LBP_KERNEL_VERTEX;
      timed(kKUpdate, [&] {
        k_vertex_update<QS, kModeCount, false, true, false>
            <<<vgrid(k_vertex_update<QS, kModeCount, false, true, false>, g_.V), kBlock, 0, s_>>>(
                dg_, live(), cand(), nullptr, nullptr, nullptr, ctl(), eps_, cand_list(), fa);
      });
    }
    launch_check();
  }

  // ---- launch sequences
  void enqueue_finalize(int mode, uint32_t D = 0xFFFFFFFFu, const unsigned long long* ext = nullptr) {
    const uint32_t d = D == 0xFFFFFFFFu ? g_.D : D;
    timed(kKOther, [&] { k_finalize<<<1, kSlots, 0, s_>>>(ctl(), mode, d, ext); });
    launch_check();
  }

  // ---- row-band partition: sweep -> pack halos + local count -> [caller's
  // collectives on stream()] -> unpack ghosts -> finalize with the global count
  PartHalo halo_{};
  uint64_t band_owned_ = 0;
  bool pingpong_ = false;
  cudaStream_t stream() const override { return s_; }
  // vertex-range partition of any binary graph (bp_graph_create_part): cut
  // messages through the graph's index lists; halo_.send_up / recv_up hold
  // every peer's run back to back
  bool part_mode_ = false;
  uint32_t part_ns_ = 0, part_nr_ = 0;
  void band_config(const PartHalo& h, uint64_t owned_directed) override {
    part_mode_ = g_.nparts != 0;
    if (part_mode_) {
      if (QS != 1) throw Error(BP_ERR_UNSUPPORTED, "vertex-range partition: binary graphs only");
      if (cfg_.kind != BP_LBP && cfg_.kind != BP_RNBP)
        throw Error(BP_ERR_UNSUPPORTED, "vertex-range partition: LBP and RnBP (RBP / RS: row bands of lattices)");
      part_ns_ = part_nr_ = 0;
      for (const auto& p : g_.peers) {
        part_ns_ += p.send_n;
        part_nr_ += p.recv_n;
      }
    } else if (QS != 1 || !g_.lat_cols || g_.par_mode != 1) {
      throw Error(BP_ERR_UNSUPPORTED, "row-band partition needs a binary Ising lattice band");
    }
    if (cfg_.kind == BP_SERIAL_RBP) throw Error(BP_ERR_UNSUPPORTED, "row-band partition: not for serial RBP");
    halo_ = h;
    halo_.ghost_up = g_.cnt_row0 > 0 ? 1u : 0u;
    halo_.ghost_down = g_.cnt_row1 < g_.lat_rows ? 1u : 0u;
    band_owned_ = owned_directed;
    pingpong_ = false;
  }
  unsigned list_grid(uint32_t n) const { return grid_cap(std::max<uint32_t>(n, 1u), 4); }
  void part_pack(bool pingpong) {
    k_plist_pack<<<list_grid(part_ns_), kBlock, 0, s_>>>(live(), cand(), ctl(), pingpong ? 1 : 0,
                                                         g_.send_idx.as<uint32_t>(), part_ns_, halo_.send_up);
  }
  void band_sweep() override {
    if (cfg_.kind != BP_LBP) throw_invalid("band_lbp_* on a non-LBP engine");
    if (!pingpong_) {
      band_start_common();
      pingpong_ = true;
    }
    enqueue_lbp_sweep(kFinNone);
    const unsigned gc = static_cast<unsigned>((g_.lat_cols + kBlock - 1) / kBlock);
    if (part_mode_) part_pack(true);
    else k_part_pack<<<gc, kBlock, 0, s_>>>(dg_, live(), cand(), ctl(), halo_);
    k_part_count<<<1, kSlots, 0, s_>>>(ctl(), halo_);
    launch_check();
    launches_ += 2;
  }
  void band_finish() override {
    const unsigned gc = static_cast<unsigned>((g_.lat_cols + kBlock - 1) / kBlock);
    if (part_mode_)
      k_plist_unpack<<<list_grid(part_nr_), kBlock, 0, s_>>>(live(), cand(), ctl(), 1, g_.recv_idx.as<uint32_t>(),
                                                             part_nr_, halo_.recv_up);
    else
      k_part_unpack<<<gc, kBlock, 0, s_>>>(dg_, live(), cand(), ctl(), halo_);
    launch_check();
    ++launches_;
    enqueue_finalize(kFinLbp, static_cast<uint32_t>(band_owned_), halo_.count);
  }
  void band_start_common() {
    reset_ctl(cfg_.max_iterations, 1e300);  // the local clock never stops a band alone
    const double ns = cfg_.time_limit * 1e9;
    const unsigned long long lim = ns >= 1.8e19 ? ~0ull : static_cast<unsigned long long>(ns);
    cuda_check(cudaMemcpyAsync(reinterpret_cast<char*>(ctl_.p) + offsetof(Ctl, vote_limit_ns), &lim, 8,
                               cudaMemcpyHostToDevice, s_), "ctl h2d");
    const unsigned gi = grid_cap(static_cast<size_t>(g_.D) * QS);
    k_init_messages<QS><<<gi, kBlock, 0, s_>>>(dg_, live(), ctl(), 1);
    launch_check();
    ++launches_;
  }
  unsigned band_cols_grid() const { return static_cast<unsigned>((g_.lat_cols + kBlock - 1) / kBlock); }
  void band_rnbp_begin() override {
    if (cfg_.kind == BP_LBP) throw_invalid("band frontier API on an LBP engine");
    band_start_common();
    k_vertex_update<QS, kModeInit, false, false, false>
        <<<vgrid(k_vertex_update<QS, kModeInit, false, false, false>, g_.V), kBlock, 0, s_>>>(
            dg_, live(), cand(), res_.as<float>(), nullptr, nullptr, ctl(), eps_, cand_list(), FinArgs{kFinNone, 0});
    k_part_count_rnbp<<<1, kSlots, 0, s_>>>(ctl(), halo_);
    launch_check();
    launches_ += 2;
  }
  void band_rnbp_finish_init() override { enqueue_finalize(kFinInitExt, g_.D, halo_.count); }
  void band_rnbp_select(unsigned attempt) override {
    RnbpParams q = prm_;
    q.attempt = attempt;
    k_rnbp_select<QS, false><<<grid_cap(g_.D / 4 + 1), kBlock, 0, s_>>>(
        dg_, live(), cand(), res_.as<float>(), vflag_.as<uint32_t>(), vlist_.as<uint32_t>(), nullptr, ctl(), eps_, q,
        cand_list(), 0);
    if (part_mode_) part_pack(false);
    else k_part_pack_live<<<band_cols_grid(), kBlock, 0, s_>>>(dg_, live(), halo_);
    launch_check();
    launches_ += 2;
  }
  // RBP on a band: local top-k over the band's own edges, k = max(1, llround(p owned))
  // (per-partition local frontier, a deviation from the global select_top_k by design)
  void band_rbp_select() override {
    ensure_rbp_scratch();
    const long long kr = std::llround(cfg_.p * static_cast<double>(band_owned_));
    enqueue_topk(kr < 1 ? 1ull : static_cast<uint64_t>(kr), 1);
    k_part_pack_live<<<band_cols_grid(), kBlock, 0, s_>>>(dg_, live(), halo_);
    launch_check();
    ++launches_;
  }
  // RS on a band: local splashes, k = max(1, llround(p owned vertices))
  void band_rs_select() override {
    const uint64_t vown = static_cast<uint64_t>(g_.cnt_row1 - g_.cnt_row0) * g_.lat_cols;
    const long long kr = std::llround(cfg_.p * static_cast<double>(vown));
    ensure_rs(cfg_.splash_depth);
    launch_rs(kr < 1 ? 1ull : static_cast<unsigned long long>(kr), cfg_.splash_depth, 1);
    k_part_pack_live<<<band_cols_grid(), kBlock, 0, s_>>>(dg_, live(), halo_);
    launch_check();
    launches_ += 2;
  }
  void band_rnbp_refresh() override {
    if (part_mode_)
      k_plist_unpack_flag<<<list_grid(part_nr_), kBlock, 0, s_>>>(dg_, live(), ctl(), vflag_.as<uint32_t>(),
                                                                  vlist_.as<uint32_t>(), g_.recv_idx.as<uint32_t>(),
                                                                  part_nr_, halo_.recv_up);
    else
      k_part_unpack_flag<<<band_cols_grid(), kBlock, 0, s_>>>(dg_, live(), ctl(), vflag_.as<uint32_t>(),
                                                             vlist_.as<uint32_t>(), halo_);
    k_vertex_update<QS, kModeDelta, true, false, false>
        <<<vgrid(k_vertex_update<QS, kModeDelta, true, false, false>, g_.V), kBlock, 0, s_>>>(
            dg_, live(), cand(), res_.as<float>(), vlist_.as<uint32_t>(), vflag_.as<uint32_t>(), ctl(), eps_,
            cand_list(), FinArgs{kFinNone, 0});
    k_part_count_rnbp<<<1, kSlots, 0, s_>>>(ctl(), halo_);
    launch_check();
    launches_ += 3;
  }
  void band_rnbp_finish() override { enqueue_finalize(kFinIterExt, g_.D, halo_.count); }
  // owned survivors (r >= eps) as GLOBAL directed ids, for the fallback of
  // rnbp_frontier (schedulers.cpp:212-214) across bands
  void band_survivors(std::vector<uint64_t>& out) override {
    std::vector<float> r(g_.D);
    sync();
    if (g_.D) cuda_check(cudaMemcpy(r.data(), res_.p, 4ull * g_.D, cudaMemcpyDeviceToHost), "d2h");
    out.clear();
    for (uint32_t d = 0; d < g_.D; ++d)
      if (r[d] >= eps_)
        out.push_back(part_mode_ ? 2ull * g_.egid_host[d >> 1] + (d & 1u) : d + 2ull * g_.edge_offset);
  }
  void band_rnbp_pack() override {
    if (part_mode_) part_pack(false);
    else k_part_pack_live<<<band_cols_grid(), kBlock, 0, s_>>>(dg_, live(), halo_);
    launch_check();
    ++launches_;
  }
  void band_commit_global(uint64_t gd) override {
    if (gd == ~0ull) return;
    uint64_t d = gd - 2ull * g_.edge_offset;
    if (part_mode_) {  // the local copy of global edge gd >> 1 (its source is owned here)
      d = g_.D;
      for (uint32_t e = 0; e < g_.E && d == g_.D; ++e)
        if (g_.egid_host[e] == (gd >> 1)) d = 2ull * e + (gd & 1u);
      if (d == g_.D) throw_invalid("edge not in this part");
    } else if (gd < 2ull * g_.edge_offset || d >= g_.D) {
      throw_invalid("edge not in this band");
    }
    const uint32_t d32 = static_cast<uint32_t>(d);
    DevBuf list;
    list.upload(&d32, 4);
    k_commit_list<QS><<<1, kBlock, 0, s_>>>(dg_, list.as<uint32_t>(), 1, live(), cand(), res_.as<float>(),
                                           vflag_.as<uint32_t>(), vlist_.as<uint32_t>(), ctl(), eps_, 0);
    launch_check();
    ++launches_;
    sync();
  }

  void ctl_put_u32(size_t off, unsigned v) {
    cuda_check(cudaMemcpyAsync(reinterpret_cast<char*>(ctl_.p) + off, &v, 4, cudaMemcpyHostToDevice, s_), "ctl h2d");
    sync();  // v lives on this stack frame
  }
  void band_set_poll(bool on) override { ctl_put_u32(offsetof(Ctl, band_poll), on ? 1u : 0u); }
  bool band_waiting() override { return hctl_->band_wait != 0u; }
  void band_clear_wait() override { ctl_put_u32(offsetof(Ctl, band_wait), 0u); }

  void band_status(bp_run_result* r) override {
    fetch_ctl_header();
    std::memset(r, 0, sizeof(*r));
    r->converged = hctl_->converged ? 1 : 0;
    r->stopped = hctl_->done ? 1 : 0;
    r->iterations = hctl_->iteration;
    r->messages_updated_total = hctl_->msgs_total;
    r->trace_len = hctl_->trace_len;
    r->message_evaluations = hctl_->evals_total;
    r->vertex_visits = hctl_->vertex_visits;
    r->gpu_launches = launches_;
    if (hctl_->numeric_error) throw Error(BP_ERR_NUMERIC, "probability vector collapsed (total mass below 1e-300 or non-finite)");
  }

  void enqueue_init(bool lbp) {
    const unsigned gi = grid_cap(static_cast<size_t>(g_.D) * QS);
    timed(kKInit, [&] { k_init_messages<QS><<<gi, kBlock, 0, s_>>>(dg_, live(), ctl(), 1); });
    launch_check();
    if (lbp) {  // sweep 0 (ResidualTracker ctor, residuals.cpp:9-24)
      enqueue_lbp_sweep(kFinLbp);
    } else {
      const FinArgs fa{kFinInit, g_.D};
      if constexpr (QS == 4 || QS == 8) {
        // q-state lattices: the initial candidates / residuals with four
        // states per lane (the candidate list starts empty: cl_state is 0
        // until this launch's finalize)
        if (qlanes_refresh()) {
          const unsigned grid = vgrid(k_lattice_qsweep<QS, true, kModeInit>, static_cast<size_t>(g_.V) * (QS / 4));
          timed(kKUpdate, [&] {
            if (g_.par_mode)
              k_lattice_qsweep<QS, true, kModeInit><<<grid, kBlock, 0, s_>>>(
                  dg_, live(), cand(), res_.as<float>(), nullptr, nullptr, ctl(), eps_, fa);
            else
              k_lattice_qsweep<QS, false, kModeInit><<<grid, kBlock, 0, s_>>>(
                  dg_, live(), cand(), res_.as<float>(), nullptr, nullptr, ctl(), eps_, fa);
          });
          launch_check();
          return;
        }
      }
      timed(kKUpdate, [&] {
        if (use_clist_)
          k_vertex_update<QS, kModeInit, false, false, true><<<vgrid(k_vertex_update<QS, kModeInit, false, false, true>, g_.V), kBlock, 0, s_>>>(
              dg_, live(), cand(), res_.as<float>(), nullptr, nullptr, ctl(), eps_, cand_list(), fa);
        else
          k_vertex_update<QS, kModeInit, false, false, false><<<vgrid(k_vertex_update<QS, kModeInit, false, false, false>, g_.V), kBlock, 0, s_>>>(
              dg_, live(), cand(), res_.as<float>(), nullptr, nullptr, ctl(), eps_, cand_list(), fa);
      });
      launch_check();
    }
  }

  // touched refresh; the iteration's loop control (fin) runs in its last block
  // q-state lattices (q <= 8): the touched refresh with four states per lane
  // outside RnBP list mode (k_lattice_qsweep<kModeDelta>); the vertex kernel
  // after it is gated to list mode
  bool qlanes_refresh() const {
    static const bool off = std::getenv("BPB_NO_QLANES_REFRESH") != nullptr;  // tuning aid
    return !off && (QS == 4 || QS == 8) && g_.lat_cols && g_.uniform_q && !g_.check_collapse && !band_owned_;
  }
  void enqueue_refresh(int fin) {
    FinArgs fa{fin, g_.D, 0};
    if constexpr (QS == 4 || QS == 8) {
      if (qlanes_refresh()) {
        // with a candidate list the gated vertex kernel below runs the
        // iteration's finalize (its refresh only in list mode)
        const FinArgs fq{use_clist_ ? static_cast<int>(kFinNone) : fin, g_.D, 0};
        const unsigned grid = vgrid(k_lattice_qsweep<QS, true, kModeDelta>, static_cast<size_t>(g_.V) * (QS / 4));
        timed(kKUpdate, [&] {
          if (g_.par_mode)
            k_lattice_qsweep<QS, true, kModeDelta><<<grid, kBlock, 0, s_>>>(
                dg_, live(), cand(), res_.as<float>(), vlist_.as<uint32_t>(), vflag_.as<uint32_t>(), ctl(), eps_, fq);
          else
            k_lattice_qsweep<QS, false, kModeDelta><<<grid, kBlock, 0, s_>>>(
                dg_, live(), cand(), res_.as<float>(), vlist_.as<uint32_t>(), vflag_.as<uint32_t>(), ctl(), eps_, fq);
        });
        launch_check();
        if (!use_clist_) return;  // no list mode: the lanes kernel refreshes every iteration
        fa.gate = 1;
      }
    }
    timed(kKUpdate, [&] {
      if (use_clist_)
        k_vertex_update<QS, kModeDelta, true, false, true><<<vgrid(k_vertex_update<QS, kModeDelta, true, false, true>, g_.V), kBlock, 0, s_>>>(
            dg_, live(), cand(), res_.as<float>(), vlist_.as<uint32_t>(), vflag_.as<uint32_t>(), ctl(), eps_,
            cand_list(), fa);
      else
        k_vertex_update<QS, kModeDelta, true, false, false><<<vgrid(k_vertex_update<QS, kModeDelta, true, false, false>, g_.V), kBlock, 0, s_>>>(
            dg_, live(), cand(), res_.as<float>(), vlist_.as<uint32_t>(), vflag_.as<uint32_t>(), ctl(), eps_,
            cand_list(), fa);
    });
    launch_check();
  }

  void ensure_rbp_scratch() {
    if (!hist_.p) {
      hist_.alloc(kRadixBins * 4);
      cuda_check(cudaMemset(hist_.p, 0, kRadixBins * 4), "memset");
      cuda_check(cudaDeviceSynchronize(), "memset");  // legacy stream: not ordered before s_
    }
    if (!chunk_.p) {
      nchunks_ = std::max<uint32_t>(1, (g_.D + kTieChunk - 1) / kTieChunk);
      chunk_.alloc(static_cast<size_t>(nchunks_) * 4);
    }
    if (!rx_list_.p) rx_list_.alloc(std::max<size_t>(g_.D, 1) * 4);
  }

  // select_all commit (|F| = 2|E|)
  void enqueue_topk_all() {
    timed(kKSelect, [&] {
      k_rbp_commit<QS><<<nchunks_, kBlock, 0, s_>>>(dg_, live(), cand(), res_.as<float>(), vflag_.as<uint32_t>(),
                                                    vlist_.as<uint32_t>(), sel_.as<uint8_t>(), chunk_.as<unsigned>(),
                                                    ctl(), eps_, 1, 1, 1);
    });
    launch_check();
  }

  void enqueue_topk(uint64_t k, int commit) {
    const int dense = k > g_.V / 16 ? 1 : 0;
    if (k >= (band_owned_ ? band_owned_ : g_.D)) {
      timed(kKSelect, [&] {
        k_rbp_commit<QS><<<nchunks_, kBlock, 0, s_>>>(dg_, live(), cand(), res_.as<float>(), vflag_.as<uint32_t>(),
                                                      vlist_.as<uint32_t>(), sel_.as<uint8_t>(), chunk_.as<unsigned>(),
                                                      ctl(), eps_, 1, commit, dense);
      });
      launch_check();
      return;
    }
    // radix select over a compacted candidate list (kernels.cuh k_rx_*):
    // five launches, two full passes over the residuals
    const unsigned gh = grid_cap(g_.D / 4 + 1, 4);
    float* res = res_.as<float>();
    unsigned* hist = hist_.as<unsigned>();
    uint32_t* list = rx_list_.as<uint32_t>();
    timed(kKTopk, [&] { k_rx_hist0<<<gh, kBlock, 0, s_>>>(dg_, res, g_.D, hist, ctl(), k); });
    timed(kKTopk, [&] { k_rx_compact<<<gh, kBlock, 0, s_>>>(dg_, res, g_.D, hist, list, ctl(), k); });
    // the list (k .. a few k entries; its length lives on the device): one
    // resident wave, so each thread's dependent list -> residual -> commit
    // round trips happen once, not once per grid-stride step
    const unsigned gl = grid_cap(std::min<uint64_t>(4 * k, g_.D), 2);
    timed(kKTopk, [&] { k_rx_hist2<<<gl, kBlock, 0, s_>>>(res, list, hist, ctl(), k); });
    timed(kKTopk, [&] {
      k_rx_ties<<<std::min<unsigned>(nchunks_, 2 * sm_count()), kBlock, 0, s_>>>(dg_, res, g_.D,
                                                                                 chunk_.as<unsigned>(), nchunks_, ctl());
    });
    timed(kKSelect, [&] {
      k_rbp_commit_list<QS><<<gl, kBlock, 0, s_>>>(
          dg_, live(), cand(), res, vflag_.as<uint32_t>(), vlist_.as<uint32_t>(), sel_.as<uint8_t>(), list,
          chunk_.as<unsigned>(), nchunks_, ctl(), eps_, commit, dense);
    });
    launch_check();
  }

  // one iteration of the loop body (schedulers.cpp:311-346) for the configured scheduler
  void enqueue_iteration() {
    switch (cfg_.kind) {
      case BP_LBP:
        enqueue_lbp_sweep(kFinLbp);
        break;
      case BP_RNBP: {
        // select + commit; its last block runs the retry / fallback
        // select + commit, then the retry / fallback as its own one-block
        // launch (a last-block-done retry in the select measured 5% slower:
        // ~1000 blocks serialise on the done counter)
        timed(kKSelect, [&] {
          if (use_clist_)
            k_rnbp_select<QS, true><<<grid_cap(g_.D), kBlock, 0, s_>>>(
                dg_, live(), cand(), res_.as<float>(), vflag_.as<uint32_t>(), vlist_.as<uint32_t>(), nullptr, ctl(),
                eps_, prm_, cand_list(), 0);
          else
            k_rnbp_select<QS, false><<<grid_cap(g_.D / 4 + 1), kBlock, 0, s_>>>(
                dg_, live(), cand(), res_.as<float>(), vflag_.as<uint32_t>(), vlist_.as<uint32_t>(), nullptr, ctl(),
                eps_, prm_, cand_list(), 0);
        });
        timed(kKSelect, [&] {
          if (use_clist_)
            k_rnbp_retry<QS, true><<<1, 1024, 0, s_>>>(dg_, live(), cand(), res_.as<float>(), vflag_.as<uint32_t>(),
                                                       vlist_.as<uint32_t>(), nullptr, ctl(), eps_, prm_, cand_list());
          else
            k_rnbp_retry<QS, false><<<1, 1024, 0, s_>>>(dg_, live(), cand(), res_.as<float>(), vflag_.as<uint32_t>(),
                                                        vlist_.as<uint32_t>(), nullptr, ctl(), eps_, prm_,
                                                        cand_list());
        });
        launch_check();
        enqueue_refresh(kFinIter);
        break;
      }
      case BP_RBP:
        ensure_rbp_scratch();
        enqueue_topk(k_, 1);
        enqueue_refresh(kFinIter);
        break;
      case BP_RS:
        timed(kKSplash, [&] { launch_rs(rs_k(cfg_.p), cfg_.splash_depth, 1); });
        enqueue_refresh(kFinIter);
        break;
      default:
        throw Error(BP_ERR_UNSUPPORTED, "scheduler not available on the device");
    }
  }

  // Device-side loop: WHILE(cond) { iteration } as one CUDA graph launch; the
  // last block of each iteration sets cond = !done.
  void run_graph_loop(bp_iter_record* trace, uint64_t cap, uint64_t& copied) {
    if (!gexec_) {
      cuda_check(cudaGraphCreate(&graph_, 0), "graph create");
      cuda_check(cudaGraphConditionalHandleCreate(&cond_, graph_, 1, cudaGraphCondAssignDefault), "cond handle");
      cudaGraphNodeParams p{};
      p.type = cudaGraphNodeTypeConditional;
      p.conditional.handle = cond_;
      p.conditional.type = cudaGraphCondTypeWhile;
      p.conditional.size = 1;
      cudaGraphNode_t node;
      cuda_check(cudaGraphAddNode(&node, graph_, nullptr, 0, &p), "graph add conditional");
      cudaGraph_t body = p.conditional.phGraph_out[0];
      cuda_check(cudaStreamBeginCaptureToGraph(s_, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed),
                 "begin capture");
      const uint64_t l0 = launches_;
      enqueue_iteration();
      body_launches_ = launches_ - l0;
      launches_ = l0;
      cudaGraph_t out_body;
      cuda_check(cudaStreamEndCapture(s_, &out_body), "end capture");
      cuda_check(cudaGraphInstantiate(&gexec_, graph_, 0), "graph instantiate");
    }
    set_cond_handle(static_cast<unsigned long long>(cond_));
    const uint64_t it0 = hctl_->iteration;
    // The device loop stops itself (converged / max_iterations / time_limit
    // via %globaltimer).  The trace ring holds kTraceRing records, so long
    // runs are split into chunks that the host drains in between.
    for (;;) {
      const uint64_t start_it = hctl_->iteration;
      set_iteration_budget(start_it + kTraceRing / 2);
      cuda_check(cudaGraphLaunch(gexec_, s_), "graph launch");
      // RnBP: the persistent tail is enqueued right behind the graph (it
      // returns at once unless the graph handed list mode over), so the
      // handover costs no host round trip
      if (persist_) launch_persist(false);
      fetch_ctl_header();
      drain_trace(trace, cap, copied);
      if (!hctl_->done && handover()) break;  // RnBP list mode -> persistent kernel
      if (hctl_->done) {
        if (hctl_->stop_reason == kStopMaxIter && hctl_->iteration < cfg_.max_iterations && budget_stop_) {
          // stopped by the chunk budget, not by the run: continue
          clear_budget_stop();
          if (handover()) break;
          continue;
        }
        break;
      }
    }
    // iterations run by the graph body (the chained persistent kernel counts its own launches)
    const uint64_t graph_end = hctl_->handover_it >= it0 && hctl_->handover_it ? std::min(hctl_->iteration, hctl_->handover_it)
                                                                               : hctl_->iteration;
    launches_ += (graph_end - it0) * body_launches_;
    set_cond_handle(0);
  }

  // Chunking of the device loop: temporarily lower max_iterations so the ring
  // never overruns; a stop caused by it is undone before continuing.
  bool budget_stop_ = false;
  // (stream-ordered: no host synchronisation, so the device never idles on
  // these between a loop launch and the next)
  void set_iteration_budget(uint64_t limit) {
    const uint64_t eff = std::min<uint64_t>(limit, cfg_.max_iterations);
    budget_stop_ = eff < cfg_.max_iterations;
    k_set_u64<<<1, 1, 0, s_>>>(&ctl()->max_iterations, eff);
    launch_check();
  }
  void clear_budget_stop() {
    k_set_u32<<<1, 1, 0, s_>>>(&ctl()->done, 0u);
    launch_check();
    hctl_->done = 0u;  // host mirror
  }
  void set_cond_handle(unsigned long long h) {
    k_set_u64<<<1, 1, 0, s_>>>(&ctl()->cond_handle, h);
    launch_check();
  }

  static constexpr size_t kPinnedBeliefs = size_t{1} << 20;
  void* bel_pinned_ = nullptr;
  size_t bel_pinned_bytes_ = 0;

  // ---- fused dense RnBP sweeps (kernels_fused.cuh)
  DevBuf fc_;  // scratch candidate set (live messages are updated in place)
  DevBuf fu_[2];    // unconverged predicates (r >= eps) of the canonical / scratch set
  uint64_t fused_iters_ = 0, fused_sweeps_ = 0;  // iterations run fused; sweeps (an aborted one included)
  cudaGraph_t fgraph_ = nullptr;
  cudaGraphExec_t fgexec_ = nullptr;
  cudaGraphConditionalHandle fcond_{};
  bool fused_capable() const {
    return cfg_.kind == BP_RNBP && QS == 1 && g_.lat_cols && g_.par_mode == 1 && !g_.check_collapse &&
           g_.cnt_row0 == 0 && g_.cnt_row1 >= g_.lat_rows && g_.edge_offset == 0;
  }
  unsigned fused_grid() {
    // one resident wave; BPB_FUSED_TPB = n: ~n tiles per block instead (tuning)
    static const char* e = std::getenv("BPB_FUSED_TPB");
    const uint64_t ntiles = static_cast<uint64_t>(g_.lat_rows) * ((g_.lat_cols + kFusedStrip - 1) / kFusedStrip);
    if (e && std::atoi(e) > 0)  // ~n block-strip tiles per block
      return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(ntiles / std::atoi(e), 1u << 30)));
    return fused_warp_tiles(g_.lat_cols) ? vgrid(k_rnbp_fused<true>, g_.V) : vgrid(k_rnbp_fused<false>, g_.V);
  }
  // the SMEM-staged version only on request (BP_RUN_FUSED_TMA): it moves
  // exactly the algorithmic bytes (23.4 GB per 16384^2 sweep against 26.6 GB)
  // but measured slower (8.8 vs 7.0 ms): both versions are instruction-bound
  // (~600 / ~780 instructions per vertex), and the staged one adds three
  // block barriers per row tile
  uint32_t fused_force_ = 0;
  unsigned fused_tma_grid_ = 0;
  bool fused_uses_tma() const { return (fused_force_ & BP_RUN_FUSED_TMA) != 0; }
  // small lattices run the dense phase as ONE persistent launch
  // (k_rnbp_fused_persist): 0 = per-sweep launches, 1 = 16-CTA cluster,
  // 2 = cooperative grid (BPB_FUSED_PERSIST: tuning override)
  // (measured, whole 10k-cap runs: 100^2 4.71 -> 4.48 ms with the cluster,
  // 128^2 5.93 -> 5.58; 200^2 12.51 -> 11.94 with the grid, where the cluster
  // was slower: 16 SMs for 1300 warp tiles)
  static constexpr uint32_t kFusedPersistClusterV = 16384, kFusedPersistGridV = 48000;
  unsigned fused_persist_mode() const {
    static const char* e = std::getenv("BPB_FUSED_PERSIST");
    if (fused_uses_tma()) return 0;
    if (e) return static_cast<unsigned>(std::atoi(e));
    return g_.V <= kFusedPersistClusterV ? 1u : g_.V <= kFusedPersistGridV ? 2u : 0u;
  }
  void launch_fused_persist(bool cluster) {
    static std::map<int, bool> attr_set;  // per device
    if (!attr_set[g_.device]) {
      cuda_check(cudaFuncSetAttribute(k_rnbp_fused_persist<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                 "cluster attribute");
      attr_set[g_.device] = true;
    }
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(cluster ? 16u : static_cast<unsigned>(sm_count()));
    lc.blockDim = dim3(kFusedPersistBlock);
    lc.stream = s_;
    cudaLaunchAttribute at[1];
    if (cluster) {
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 16;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
    } else {
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
    }
    lc.attrs = at;
    lc.numAttrs = 1;
    float* L = live();
    float* CA = cand();
    float* CB = fc_.as<float>();
    uint8_t* UA = fu_[0].as<uint8_t>();
    uint8_t* UB = fu_[1].as<uint8_t>();
    timed(kKFused, [&] {
      auto k = cluster ? k_rnbp_fused_persist<true> : k_rnbp_fused_persist<false>;
      cuda_check(cudaLaunchKernelEx(&lc, k, dg_, L, CA, UA, CB, UB, ctl(), eps_, prm_), "fused persistent launch");
    });
    ++launches_;
  }
  void enqueue_fused(unsigned dir) {
    if (fused_uses_tma()) {
      if (!fused_tma_grid_) {
        cuda_check(cudaFuncSetAttribute(k_rnbp_fused_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(sizeof(FusedSmem))),
                   "smem attribute");
        int per = 0;
        cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_rnbp_fused_tma, kBlock, sizeof(FusedSmem)),
                   "occupancy");
        fused_tma_grid_ = static_cast<unsigned>(std::max(1, per) * sm_count());
      }
      timed(kKFused, [&] {
        if (dir == 0)
          k_rnbp_fused_tma<<<fused_tma_grid_, kBlock, sizeof(FusedSmem), s_>>>(
              dg_, live(), cand(), fu_[0].as<uint8_t>(), live(), fc_.as<float>(), fu_[1].as<uint8_t>(), ctl(), eps_,
              prm_, 0u);
        else
          k_rnbp_fused_tma<<<fused_tma_grid_, kBlock, sizeof(FusedSmem), s_>>>(
              dg_, live(), fc_.as<float>(), fu_[1].as<uint8_t>(), live(), cand(), fu_[0].as<uint8_t>(), ctl(), eps_,
              prm_, 1u);
      });
      launch_check();
      return;
    }
    const unsigned grid = fused_grid();
    const auto kern = fused_warp_tiles(g_.lat_cols) ? k_rnbp_fused<true> : k_rnbp_fused<false>;
    timed(kKFused, [&] {
      if (dir == 0)
        kern<<<grid, kBlock, 0, s_>>>(dg_, live(), cand(), fu_[0].as<uint8_t>(), live(), fc_.as<float>(),
                                      fu_[1].as<uint8_t>(), ctl(), eps_, prm_, 0u);
      else
        kern<<<grid, kBlock, 0, s_>>>(dg_, live(), fc_.as<float>(), fu_[1].as<uint8_t>(), live(), cand(),
                                      fu_[0].as<uint8_t>(), ctl(), eps_, prm_, 1u);
    });
    launch_check();
  }
  // The dense phase: WHILE(cond) { fused sweep A -> S, fused sweep S -> A } as
  // one CUDA graph (the finalize of each sweep sets cond), chunked like
  // run_graph_loop for the trace ring; then the state back in the canonical
  // set.  Without graphs (kernel timing): batches of sweep pairs.
  void run_fused_phase(bool use_graph, const bp_run_opts* opts, bp_iter_record* trace, uint64_t cap,
                       uint64_t& copied) {
    const uint64_t it_in = hctl_->iteration;
    timed(kKOther, [&] {
      k_fused_enter<<<grid_cap(g_.D), kBlock, 0, s_>>>(res_.as<float>(), fu_[0].as<uint8_t>(), g_.D, eps_);
    });
    launch_check();
    if (const unsigned pm = fused_persist_mode()) {
      for (;;) {
        set_iteration_budget(hctl_->iteration + kTraceRing / 2);
        launch_fused_persist(pm == 1);
        fetch_ctl_header();
        drain_trace(trace, cap, copied);
        if (hctl_->done && hctl_->stop_reason == kStopMaxIter && hctl_->iteration < cfg_.max_iterations &&
            budget_stop_) {
          clear_budget_stop();
          if (hctl_->cl_state == 0u && !hctl_->fused_abort) continue;
        }
        break;
      }
    } else if (use_graph) {
      if (!fgexec_) {
        cuda_check(cudaGraphCreate(&fgraph_, 0), "graph create");
        cuda_check(cudaGraphConditionalHandleCreate(&fcond_, fgraph_, 1, cudaGraphCondAssignDefault), "cond handle");
        cudaGraphNodeParams p{};
        p.type = cudaGraphNodeTypeConditional;
        p.conditional.handle = fcond_;
        p.conditional.type = cudaGraphCondTypeWhile;
        p.conditional.size = 1;
        cudaGraphNode_t node;
        cuda_check(cudaGraphAddNode(&node, fgraph_, nullptr, 0, &p), "graph add conditional");
        cuda_check(cudaStreamBeginCaptureToGraph(s_, p.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                                 cudaStreamCaptureModeRelaxed),
                   "begin capture");
        const uint64_t l0 = launches_;
        enqueue_fused(0);
        enqueue_fused(1);
        launches_ = l0;
        cudaGraph_t out_body;
        cuda_check(cudaStreamEndCapture(s_, &out_body), "end capture");
        cuda_check(cudaGraphInstantiate(&fgexec_, fgraph_, 0), "graph instantiate");
      }
      set_cond_handle(static_cast<unsigned long long>(fcond_));
      uint64_t bodies = 0;
      for (;;) {
        const uint64_t start_it = hctl_->iteration, par0 = hctl_->fused_par;
        set_iteration_budget(start_it + kTraceRing / 2);
        cuda_check(cudaGraphLaunch(fgexec_, s_), "graph launch");
        fetch_ctl_header();
        drain_trace(trace, cap, copied);
        // each body launches both sweeps; an aborted sweep ran without advancing the iteration
        const uint64_t sweeps = hctl_->iteration - start_it + hctl_->fused_abort;
        bodies += std::max<uint64_t>(1, (sweeps + par0 + 1) / 2);
        if (hctl_->done && hctl_->stop_reason == kStopMaxIter && hctl_->iteration < cfg_.max_iterations &&
            budget_stop_) {
          clear_budget_stop();
          if (hctl_->cl_state == 0u && !hctl_->fused_abort) continue;
        }
        break;
      }
      launches_ += 2 * bodies;
      set_cond_handle(0);
    } else {
      uint32_t batch = opts && opts->batch ? opts->batch : 16;
      while (!hctl_->done && hctl_->cl_state == 0u && !hctl_->fused_abort) {
        for (uint32_t b = 0; b < (batch + 1) / 2; ++b) {
          enqueue_fused(0);
          enqueue_fused(1);
        }
        fetch_ctl_header();
        drain_trace(trace, cap, copied);
        if (!(opts && opts->batch)) batch = std::min<uint32_t>(batch * 2, 256);
      }
    }
    fused_iters_ = hctl_->iteration - it_in;
    fused_sweeps_ = fused_iters_ + hctl_->fused_abort;
    timed(kKOther, [&] {
      k_fused_exit<<<grid_cap(g_.D), kBlock, 0, s_>>>(ctl(), fc_.as<float>(), fu_[0].as<uint8_t>(),
                                                      fu_[1].as<uint8_t>(), cand(), res_.as<float>(), g_.D);
    });
    launch_check();
  }

  // ---- persistent RnBP tail (kernels_persist.cuh)
  bool persist_ = false;
  unsigned persist_grid_ = 0;
  bool handover() const { return hctl_->persist_ok && hctl_->cl_state == 2u; }
  // The tail runs on one 16-CTA cluster (hardware cluster barrier, ~sub-us)
  // while the candidate list is short, else on a cooperative grid of one CTA
  // per SM.
  // BPB_PERSIST_GRID / BPB_PERSIST_CLUSTER override the choice (tuning).
  DevBuf vslot_;   // refresh slots of the persistent tail (one per candidate-list entry)
  DevBuf cstamp_;  // per-edge commit stamps of the persistent tail (owner test, lattices)
  void ensure_persist_setup() {
    if (persist_grid_) return;
    // once per process: one CTA per SM (the tail is latency-bound, a second
    // CTA per SM only adds barrier participants: 296 CTAs measured 3% slower
    // than 148)
    // function attributes are per device: set them once per device ordinal
    static std::mutex mu;
    static std::map<int, unsigned> grids;
    std::lock_guard<std::mutex> lk(mu);
    auto it = grids.find(g_.device);
    if (it == grids.end()) {
      int per_sm = 0;
      cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rnbp_persist<QS, false>, kPersistBlock, 0),
                 "occupancy");
      if (per_sm < 1) throw Error(BP_ERR_CUDA, "persistent RnBP kernel does not fit on an SM");
      cuda_check(cudaFuncSetAttribute(k_rnbp_persist<QS, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                 "cluster attribute");
      it = grids.emplace(g_.device, static_cast<unsigned>(sm_count())).first;
    }
    persist_grid_ = it->second;
  }

  // one launch of the persistent tail: a 16-CTA cluster or a cooperative grid
  // of one CTA per SM (BPB_PERSIST_GRID / BPB_PERSIST_CLUSTER: tuning overrides)
  void launch_persist(bool cluster) {
    ensure_persist_setup();
    static const char* eg = std::getenv("BPB_PERSIST_GRID");
    static const char* ec = std::getenv("BPB_PERSIST_CLUSTER");
    if (ec) cluster = std::atoi(ec) != 0;
    unsigned grid = cluster ? 16u : persist_grid_;
    if (eg && !cluster) grid = std::min<unsigned>(persist_grid_, std::max(1, std::atoi(eg)));
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(kPersistBlock);
    lc.stream = s_;
    cudaLaunchAttribute at[1];
    if (cluster) {
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = grid;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
    } else {
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
    }
    lc.attrs = at;
    lc.numAttrs = 1;
    timed(kKPersist, [&] {
      if (cluster)
        cuda_check(cudaLaunchKernelEx(&lc, k_rnbp_persist<QS, true>, dg_, live(), cand(), res_.as<float>(),
                                      vflag_.as<uint32_t>(), vslot_.as<uint32_t>(), cstamp_.as<uint32_t>(), ctl(),
                                      eps_, prm_, cand_list()),
                   "persistent cluster launch");
      else
        cuda_check(cudaLaunchKernelEx(&lc, k_rnbp_persist<QS, false>, dg_, live(), cand(), res_.as<float>(),
                                      vflag_.as<uint32_t>(), vslot_.as<uint32_t>(), cstamp_.as<uint32_t>(), ctl(),
                                      eps_, prm_, cand_list()),
                   "persistent launch");
    });
  }

  void run_persist_loop(bp_iter_record* trace, uint64_t cap, uint64_t& copied) {
    for (;;) {
      set_iteration_budget(hctl_->iteration + kTraceRing / 2);
      launch_persist(hctl_->cl_n[hctl_->cl_cur] < kPersistClusterList);
      fetch_ctl_header();
      drain_trace(trace, cap, copied);
      if (hctl_->done) {
        if (hctl_->stop_reason == kStopMaxIter && hctl_->iteration < cfg_.max_iterations && budget_stop_) {
          clear_budget_stop();
          continue;
        }
        break;
      }
      if (!handover()) break;  // not reached: list mode is final
    }
    if (std::getenv("BPB_DEBUG_PHASES")) {
      unsigned long long ph[8];
      cuda_check(cudaMemcpy(ph, reinterpret_cast<char*>(ctl_.p) + offsetof(Ctl, phase_ns), sizeof(ph),
                            cudaMemcpyDeviceToHost), "d2h");
      std::fprintf(stderr, "persist phases of CTA 0 (ms): select-loop %.2f select-flush+pacc %.2f  sync+retry %.2f  "
                   "refresh-loop %.2f flush %.2f pacc %.2f tail %.2f  sync+finalize %.2f\n",
                   ph[7] * 1e-6, ph[0] * 1e-6, ph[1] * 1e-6, ph[4] * 1e-6, ph[5] * 1e-6, ph[6] * 1e-6, ph[2] * 1e-6,
                   ph[3] * 1e-6);
    }
  }

  // ---- Residual Splash state (kernels_rs.cuh)
  static unsigned long long rs_k_of(double p, uint32_t V) {  // schedulers.cpp:172-173
    const long long kr = std::llround(p * static_cast<double>(V));
    return kr < 1 ? 1ull : static_cast<unsigned long long>(kr);
  }
  unsigned long long rs_k(double p) const { return rs_k_of(p, g_.V); }
  void ensure_rs(uint32_t h) {
    // any depth: above the walk stack the builder tests ball intersection by
    // distance propagation instead of ball lists / walks (kernels_rs.cuh)
    if (h <= kRsMaxDepth) (void)g_.balls(h);  // built here, never inside a graph capture
    if (rs_vres_.p) return;
    const size_t V = std::max<size_t>(g_.V, 1);
    for (DevBuf* b : {&rs_vres_, &rs_state_, &rs_claimed_, &rs_qnext_, &rs_spos_, &rs_depth_, &rs_clist_,
                      &rs_blist_, &rs_rlist_, &rs_klist_})
      b->alloc(V * 4);
    rs_ballmax_.alloc(V * 16);
    rs_hist_.alloc(4096 * 4);
    cuda_check(cudaMemset(rs_hist_.p, 0, 4096 * 4), "memset");
    int per_sm = 0;
    cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rs_iteration<QS>, kRsBlock, 0),
               "occupancy");
    rs_grid_ = static_cast<unsigned>(std::max(1, per_sm) * sm_count());
    rs_blk_.alloc(static_cast<size_t>(rs_grid_) * 4);
    rs_ctl_.alloc(sizeof(RsCtl));
    cuda_check(cudaMemset(rs_ctl_.p, 0, sizeof(RsCtl)), "memset");
      cuda_check(cudaDeviceSynchronize(), "memset");  // legacy stream: not ordered before s_
    rs_shadow_.alloc(std::max<size_t>(static_cast<size_t>(g_.D) * QS * 4, 16));
  }
  RsBufs rs_bufs() {
    RsBufs b{};
    b.vres = rs_vres_.as<float>();
    b.state = rs_state_.as<uint32_t>();
    b.claimed = rs_claimed_.as<uint32_t>();
    b.qnext = rs_qnext_.as<uint32_t>();
    b.spos = rs_spos_.as<uint32_t>();
    b.depth = rs_depth_.as<uint32_t>();
    b.ballmax = rs_ballmax_.as<unsigned long long>();
    b.ballmax2 = b.ballmax + std::max<size_t>(g_.V, 1);
    b.clist = rs_clist_.as<uint32_t>();
    b.blist = rs_blist_.as<uint32_t>();
    b.rlist = rs_rlist_.as<uint32_t>();
    b.klist = rs_klist_.as<uint32_t>();
    b.hist = rs_hist_.as<unsigned>();
    b.blk = rs_blk_.as<unsigned>();
    b.rc = rs_ctl_.as<RsCtl>();
    b.shadow = rs_shadow_.as<float>();
    return b;
  }
  void launch_rs(unsigned long long k, uint32_t h, int apply) {
    RsParams prm{k, h, apply};
    RsBufs bufs = rs_bufs();
    if (const BallLists* bl = h <= kRsMaxDepth ? g_.balls(h) : nullptr) {
      bufs.boff = bl->off.as<unsigned long long>();
      bufs.bl = bl->list.as<uint32_t>();
    }
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(rs_grid_);
    lc.blockDim = dim3(kRsBlock);
    lc.stream = s_;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    cuda_check(cudaLaunchKernelEx(&lc, k_rs_iteration<QS>, dg_, live(), static_cast<const float*>(res_.as<float>()),
                                  vflag_.as<uint32_t>(), vlist_.as<uint32_t>(), ctl(), bufs, prm),
               "cooperative splash launch");
  }

  void ensure_beliefs_buf(size_t nb) {
    if (bel_.bytes < nb * 8) bel_.alloc(nb * 8);
  }
  void enqueue_beliefs(double* dst, bool pingpong) {
    timed(kKBeliefs, [&] {
      k_beliefs<QS><<<grid_cap(g_.V), kBlock, 0, s_>>>(dg_, live(), cand(), pingpong ? 1 : 0, ctl(), dst);
    });
    launch_check();
  }

  void ensure_sel() {
    if (!sel_.p) sel_.alloc(g_.D ? g_.D : 1);
    cuda_check(cudaMemsetAsync(sel_.p, 0, g_.D ? g_.D : 1, s_), "memset sel");
  }
  void collect_sel(std::vector<uint32_t>& out) {
    std::vector<uint8_t> h(g_.D);
    if (g_.D) cuda_check(cudaMemcpyAsync(h.data(), sel_.p, g_.D, cudaMemcpyDeviceToHost, s_), "d2h");
    sync();
    out.clear();
    for (uint32_t d = 0; d < g_.D; ++d)
      if (h[d]) out.push_back(d);
    // the queries do not change the state: clear the per-iteration counters
    fetch_ctl_header();
    hctl_->frontier = 0;
    hctl_->survivors = 0;
    hctl_->rx_prefix = 0;
    hctl_->rx_above = 0;
    std::memset(hctl_->acc, 0, sizeof(hctl_->acc));
    cuda_check(cudaMemcpyAsync(ctl_.p, hctl_, offsetof(Ctl, trace), cudaMemcpyHostToDevice, s_), "ctl h2d");
    sync();
  }

  const GraphImpl& g_;
  bp_sched_config cfg_;
  DevGraph dg_{};
  float eps_ = 0.f;
  cudaStream_t s_ = nullptr;
  DevBuf bufA_, bufB_, res_, vflag_, vlist_, ctl_, hist_, chunk_, sel_, bel_, inlist_;
  DevBuf clist_[2];
  DevBuf rx_list_;  // RBP top-k candidate list (k_rx_compact)
  DevBuf rs_vres_, rs_state_, rs_claimed_, rs_qnext_, rs_spos_, rs_depth_, rs_clist_, rs_blist_, rs_rlist_,
      rs_klist_, rs_ballmax_, rs_hist_, rs_blk_, rs_ctl_, rs_shadow_, rs_written_;
  unsigned rs_grid_ = 1;
  uint32_t rs_stamp_ = 0;
  bool use_clist_ = false;
  Ctl* hctl_ = nullptr;
  uint32_t nchunks_ = 1;
  uint64_t k_ = 1;
  RnbpParams prm_{};
  bool timing_ = false;
  bp_kernel_stats* stats_ = nullptr;
  uint64_t launches_ = 0;
  uint64_t body_launches_ = 0;
  cudaGraph_t graph_ = nullptr;
  cudaGraphExec_t gexec_ = nullptr;
  uint32_t graph_force_ = 0;
  cudaGraphConditionalHandle cond_{};
};

}  // namespace
}  // namespace bpb
