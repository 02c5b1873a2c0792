// Fork-join helper for the host side of observe(): the GP fit (kernel matrix, blocked Cholesky,
// L^-1) and the per-path operand tables run on up to 16 host threads.  Every element is computed by
// exactly one task with the same operations in the same order as a sequential loop, so the results
// do not depend on the thread count.  Threads are created once (lazily) and sleep between calls.
#pragma once
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace as {

class HostPool {
 public:
  static HostPool& get() {
    static HostPool pool;
    return pool;
  }
  int threads() const { return static_cast<int>(workers_.size()) + 1; }
  // fn(task) for every task in [0, n); the caller takes part and returns when all tasks are done
  // parallel = false: inline on the caller (small fits, where waking the pool costs more than it saves)
  void run(int n, const std::function<void(int)>& fn, bool parallel = true) {
    if (n <= 0) return;
    if (!parallel) {
      for (int i = 0; i < n; ++i) fn(i);
      return;
    }
    std::lock_guard<std::mutex> caller(run_mu_);   // one fork-join at a time (e.g. two spaces' fits)
    if (n == 1 || workers_.empty()) {
      for (int i = 0; i < n; ++i) fn(i);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      n_ = n;
      next_.store(0);
      done_.store(0);
      ++gen_;
      gen_a_.store(gen_, std::memory_order_release);
    }
    cv_.notify_all();
    work();
    // return only when every task is done AND no worker is still inside work() for this
    // generation (a straggler must not see the counters of the next run)
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return done_.load() == n_ && active_ == 0; });
    fn_ = nullptr;
  }

 private:
  HostPool() {
    unsigned hw = std::thread::hardware_concurrency();
    if (const char* e = std::getenv("AS_HOST_THREADS")) hw = static_cast<unsigned>(std::max(1, std::atoi(e)));
    const int n = static_cast<int>(std::min(16u, hw == 0 ? 1u : hw)) - 1;
    for (int i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  void work() {
    for (;;) {
      const int i = next_.fetch_add(1);
      if (i >= n_) return;
      (*fn_)(i);
      done_.fetch_add(1);
    }
  }
  void loop() {
    unsigned long long seen = 0;
    for (;;) {
      // spin briefly before sleeping: the fit issues ~20 short parallel regions back to back, and a
      // condition-variable wake-up per region (tens of microseconds) would dominate them
      for (int k = 0; k < 200000 && gen_a_.load(std::memory_order_acquire) == seen; ++k) std::this_thread::yield();
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        ++active_;
      }
      work();
      {
        std::lock_guard<std::mutex> lk(mu_);
        --active_;
      }
      done_cv_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, run_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int n_ = 0;
  int active_ = 0;                 // workers inside work() for the current generation
  std::atomic<int> next_{0}, done_{0};
  unsigned long long gen_ = 0;
  std::atomic<unsigned long long> gen_a_{0};   // gen_ for the lock-free spin
  bool stop_ = false;
};

}  // namespace as
