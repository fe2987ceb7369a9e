// hostpool.hpp -- a small persistent host thread pool for the engine's
// pageable-memory staging: the copies between caller (pageable) buffers and
// the pinned bounce ring are the host side of the pipeline, and one core's
// memcpy bandwidth is far below PCIe.
#pragma once
#include <algorithm>
#include <condition_variable>
#include <cstddef>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "numa.hpp"

namespace pc {

class HostPool {
 public:
  // Threads run on the GPU-local CPUs of `where` (see numa.hpp).
  explicit HostPool(unsigned n, const DevicePlacement &where = DevicePlacement()) {
    for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this, where] {
      bind_thread(where);
      loop();
    });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto &t : workers_) t.join();
  }
  unsigned size() const { return static_cast<unsigned>(workers_.size()); }

  // Run fn(i) for i in [0, n) on the pool plus the calling thread; returns
  // when all parts are done.  One parallel_for at a time per pool.
  void parallel_for(unsigned n, const std::function<void(unsigned)> &fn) {
    if (n == 0) return;
    if (n == 1 || workers_.empty()) {
      for (unsigned i = 0; i < n; ++i) fn(i);
      return;
    }
    std::unique_lock<std::mutex> call(call_mu_);
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      n_ = n;
      next_ = 0;
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    for (;;) { // the caller works too
      unsigned i;
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (next_ >= n_) break;
        i = next_++;
      }
      fn(i);
      std::lock_guard<std::mutex> lk(mu_);
      ++done_;
    }
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return done_ == n_; });
    fn_ = nullptr;
  }

  // memcpy split into parts of >= 1 MiB.
  void memcpy(void *dst, const void *src, size_t bytes) {
    const size_t min_part = size_t(1) << 20;
    const unsigned parts = static_cast<unsigned>(std::min<size_t>(size() + 1, std::max<size_t>(1, bytes / min_part)));
    if (parts <= 1) {
      std::memcpy(dst, src, bytes);
      return;
    }
    parallel_for(parts, [&](unsigned i) {
      const size_t lo = bytes * i / parts, hi = bytes * (i + 1) / parts;
      std::memcpy(static_cast<char *>(dst) + lo, static_cast<const char *>(src) + lo, hi - lo);
    });
  }

 private:
  void loop() {
    unsigned seen = 0;
    for (;;) {
      unsigned i;
      const std::function<void(unsigned)> *fn;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || (gen_ != seen && next_ < n_); });
        if (stop_) return;
        if (next_ >= n_) {
          seen = gen_;
          continue;
        }
        i = next_++;
        fn = fn_;
      }
      (*fn)(i);
      std::lock_guard<std::mutex> lk(mu_);
      if (++done_ == n_) done_cv_.notify_all();
    }
  }

  std::vector<std::thread> workers_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(unsigned)> *fn_ = nullptr;
  unsigned n_ = 0, next_ = 0, done_ = 0, gen_ = 0;
  bool stop_ = false;
};

// One persistent thread that runs submitted jobs in order.  Engines own one
// so multi-device calls never pay a fresh thread's first-CUDA-call setup
// (measured at ~40 ms per new thread on the B200 host).
class Runner {
 public:
  explicit Runner(const DevicePlacement &where = DevicePlacement()) : t_([this, where] {
    bind_thread(where);
    loop();
  }) {}
  ~Runner() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    t_.join();
  }
  // Run fn on the runner thread; the returned waiter blocks until it is done.
  std::function<void()> submit(std::function<void()> fn) {
    auto done = std::make_shared<std::pair<std::mutex, std::condition_variable>>();
    auto flag = std::make_shared<bool>(false);
    {
      std::lock_guard<std::mutex> lk(mu_);
      jobs_.push_back([fn, done, flag] {
        fn();
        std::lock_guard<std::mutex> l(done->first);
        *flag = true;
        done->second.notify_all();
      });
    }
    cv_.notify_all();
    return [done, flag] {
      std::unique_lock<std::mutex> l(done->first);
      done->second.wait(l, [&] { return *flag; });
    };
  }

 private:
  void loop() {
    for (;;) {
      std::function<void()> job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || !jobs_.empty(); });
        if (stop_ && jobs_.empty()) return;
        job = std::move(jobs_.front());
        jobs_.erase(jobs_.begin());
      }
      job();
    }
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::vector<std::function<void()>> jobs_;
  bool stop_ = false;
  std::thread t_;
};

} // namespace pc
