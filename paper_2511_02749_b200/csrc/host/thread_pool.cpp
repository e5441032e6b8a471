// thread_pool.cpp — see thread_pool.h. Each parallel_for owns a Job (shared_ptr): a worker that
// wakes late only ever claims indices of the job it picked up, so it cannot run a stale fn.
#include "thread_pool.h"

namespace spq {

ThreadPool::ThreadPool(int n_workers) {
  for (int i = 0; i < n_workers; ++i) workers_.emplace_back([this] { worker(); });
}

ThreadPool::~ThreadPool() {
  {
    std::lock_guard<std::mutex> g(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& t : workers_) t.join();
}

void ThreadPool::drain(Job& j) {
  for (int64_t i = j.next.fetch_add(1); i < j.n; i = j.next.fetch_add(1)) {
    (*j.fn)(i);
    j.done.fetch_add(1);
  }
}

void ThreadPool::worker() {
  uint64_t seen = 0;
  for (;;) {
    std::shared_ptr<Job> j;
    {
      std::unique_lock<std::mutex> l(mu_);
      cv_.wait(l, [&] { return stop_ || generation_ != seen; });
      if (stop_) return;
      seen = generation_;
      j = job_;
    }
    if (!j) continue;
    drain(*j);
    if (j->done.load() == j->n) {
      std::lock_guard<std::mutex> g(mu_);
      done_cv_.notify_all();
    }
  }
}

void ThreadPool::parallel_for(int64_t n, const std::function<void(int64_t)>& fn) {
  if (n <= 0) return;
  if (workers_.empty() || n == 1) {
    for (int64_t i = 0; i < n; ++i) fn(i);
    return;
  }
  auto j = std::make_shared<Job>();
  j->fn = &fn;
  j->n = n;
  {
    std::lock_guard<std::mutex> g(mu_);
    job_ = j;
    generation_++;
  }
  cv_.notify_all();
  drain(*j);
  std::unique_lock<std::mutex> l(mu_);
  done_cv_.wait(l, [&] { return j->done.load() == j->n; });
  job_.reset();
}

}  // namespace spq
