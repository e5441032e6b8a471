// thread_pool.h — minimal persistent worker pool for host-side planning (block hashing is
// embarrassingly parallel across fragments).
#pragma once
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

namespace spq {

class ThreadPool {
 public:
  explicit ThreadPool(int n_workers);
  ~ThreadPool();
  // Run fn(i) for i in [0, n); the caller participates. Blocks until all are done.
  void parallel_for(int64_t n, const std::function<void(int64_t)>& fn);
  int size() const { return static_cast<int>(workers_.size()) + 1; }

 private:
  struct Job {
    const std::function<void(int64_t)>* fn;
    int64_t n;
    std::atomic<int64_t> next{0};
    std::atomic<int64_t> done{0};
  };
  void worker();
  static void drain(Job& j);
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::shared_ptr<Job> job_;
  uint64_t generation_ = 0;
  bool stop_ = false;
};

}  // namespace spq
