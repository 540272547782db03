// Host-side worker pool for the O(V + E) passes of graph construction from
// host arrays (build_graph's validation and the layout conversion are on the
// end-to-end path).  Workers are created once per process: spawning threads
// per pass cost ~1 ms per pass on the 16-core GPU hosts.
#pragma once

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace bpb {

class HostPool {
 public:
  static HostPool& get() {
    static HostPool* p = new HostPool;  // process lifetime (no teardown-order issues)
    return *p;
  }
  unsigned size() const { return nworkers_ + 1; }

  // f(t) for t in [0, n): the caller runs tasks too; returns when all are done.
  // Nested calls (from inside a task) and concurrent callers are serialised
  // onto the calling thread / the job mutex.
  void run(unsigned n, const std::function<void(unsigned)>& f) {
    if (n <= 1 || nworkers_ == 0 || in_task_) {
      for (unsigned t = 0; t < n; ++t) f(t);
      return;
    }
    std::lock_guard<std::mutex> job(job_mu_);
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &f;
      ntasks_ = n;
      next_.store(0);
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    const unsigned mine = work(&f, n);
    std::unique_lock<std::mutex> lk(mu_);
    done_ += mine;
    // every task finished and no worker still inside this job (a worker joins
    // a job under mu_ only while fn_ is set, so none can outlive it)
    done_cv_.wait(lk, [&] { return done_ == ntasks_ && active_ == 0; });
    fn_ = nullptr;
  }

 private:
  HostPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    unsigned n = std::min(32u, hw);
    if (const char* e = std::getenv("BPB_HOST_THREADS")) n = std::max(1, std::min(64, std::atoi(e)));
    nworkers_ = n - 1;
    for (unsigned i = 0; i < nworkers_; ++i)
      std::thread([this] { loop(); }).detach();
  }
  unsigned work(const std::function<void(unsigned)>* f, unsigned n) {
    in_task_ = true;
    unsigned finished = 0;
    for (unsigned t = next_.fetch_add(1); t < n; t = next_.fetch_add(1)) {
      (*f)(t);
      ++finished;
    }
    in_task_ = false;
    return finished;
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(unsigned)>* f;
      unsigned n;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen && fn_ != nullptr; });
        seen = gen_;
        f = fn_;
        n = ntasks_;
        ++active_;
      }
      const unsigned finished = work(f, n);
      std::lock_guard<std::mutex> lk(mu_);
      done_ += finished;
      --active_;
      if (done_ == ntasks_ && active_ == 0) done_cv_.notify_all();
    }
  }
  unsigned nworkers_ = 0;
  std::mutex job_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(unsigned)>* fn_ = nullptr;
  unsigned ntasks_ = 0, done_ = 0, active_ = 0;
  std::atomic<unsigned> next_{0};
  uint64_t gen_ = 0;
  static inline thread_local bool in_task_ = false;
};

// Loop [0, n) split into contiguous chunks over the pool; f(lo, hi, chunk).
template <class F>
void parallel_chunks(uint64_t n, unsigned chunks, F&& f) {
  if (chunks <= 1 || n < (1u << 15)) {
    f(uint64_t{0}, n, 0u);
    return;
  }
  HostPool::get().run(chunks, [&](unsigned t) { f(n * t / chunks, n * (t + 1) / chunks, t); });
}
inline unsigned pool_chunks(uint64_t n) {
  return n < (1u << 15) ? 1u : HostPool::get().size() * 2;
}
template <class F>
void parallel_for(uint64_t n, F&& f) {
  parallel_chunks(n, pool_chunks(n), [&](uint64_t a, uint64_t b, unsigned) { f(a, b); });
}

}  // namespace bpb
