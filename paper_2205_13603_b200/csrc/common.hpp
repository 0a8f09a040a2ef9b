// Error plumbing shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <string>

namespace lsb {

void set_error(const std::string& msg);
const char* last_error();

#define LSB_CUDA(expr)                                                                      \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      ::lsb::set_error(std::string(#expr) + ": " + cudaGetErrorString(e_));                 \
      return LS_ERR_CUDA;                                                                   \
    }                                                                                       \
  } while (0)

// Parse + encode work is spread over host threads (the GPU kernels need the
// descriptors of a whole batch at once).
template <class F>
void parallel_for(int n, F&& f);

}  // namespace lsb

#include <atomic>
#include <cstdint>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace lsb {

// A persistent pool of host threads for the per-candidate parse / plan /
// encode work (spawning a fresh set of std::threads on every call cost more
// than the work for a 1024-program batch).  One job at a time; a call made
// from inside a job runs inline.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool pool;
    return pool;
  }
  int size() const { return static_cast<int>(workers_.size()) + 1; }
  void run(int n, const std::function<void(int)>& f) {
    if (in_job_) {
      for (int i = 0; i < n; ++i) f(i);
      return;
    }
    std::lock_guard<std::mutex> one_job(job_mu_);
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &f;
      n_ = n;
      next_.store(0);
      busy_ = static_cast<int>(workers_.size());
      ++gen_;
    }
    cv_.notify_all();
    work();  // the caller takes part
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return busy_ == 0; });
    fn_ = nullptr;
  }

 private:
  HostPool() {
    unsigned hw = std::thread::hardware_concurrency();
    int nt = static_cast<int>(hw ? hw : 4);
    if (nt > 16) nt = 16;
    for (int t = 1; t < nt; ++t) workers_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  void work() {
    in_job_ = true;
    for (int i = next_.fetch_add(1); i < n_; i = next_.fetch_add(1)) (*fn_)(i);
    in_job_ = false;
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      work();
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (--busy_ == 0) done_cv_.notify_one();
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, job_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int n_ = 0, busy_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
  std::atomic<int> next_{0};
  static inline thread_local bool in_job_ = false;
};

template <class F>
void parallel_for(int n, F&& f) {
  if (n < 64) {
    for (int i = 0; i < n; ++i) f(i);
    return;
  }
  std::function<void(int)> fn = [&](int i) { f(i); };
  HostPool::get().run(n, fn);
}
}  // namespace lsb
