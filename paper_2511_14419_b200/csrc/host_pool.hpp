// host_pool.hpp — a small fixed thread pool for the host side of the ingest / egress pipeline
// (runtime.cu): converting frames into pinned staging buffers before their H2D copy and
// unpacking returned PBM masks into the caller's RoiMask bytes, both overlapped with the GPU.
//
// It plays the role of the reference's parallel_for (parallel.hpp:20-49) for host work only:
// a static block partition, every index processed exactly once, the first exception rethrown.
#pragma once

#include <condition_variable>
#include <deque>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

namespace froi {

class HostPool {
   public:
    // Completion handle of a submitted task.
    struct Task {
        std::mutex m;
        std::condition_variable cv;
        bool done = false;
        std::exception_ptr err;
        void wait() {
            std::unique_lock<std::mutex> lk(m);
            cv.wait(lk, [&] { return done; });
            if (err) std::rethrow_exception(err);
        }
    };
    using TaskPtr = std::shared_ptr<Task>;

    // `init` runs once in every worker before it takes work (e.g. cudaSetDevice).
    explicit HostPool(int threads, std::function<void()> init = {}) {
        for (int i = 0; i < threads; ++i)
            workers_.emplace_back([this, init] {
                if (init) init();
                loop();
            });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    HostPool(const HostPool&) = delete;
    HostPool& operator=(const HostPool&) = delete;

    int threads() const { return (int)workers_.size(); }

    TaskPtr submit(std::function<void()> fn) {
        auto t = std::make_shared<Task>();
        {
            std::lock_guard<std::mutex> lk(m_);
            q_.emplace_back([t, fn = std::move(fn)] {
                try {
                    fn();
                } catch (...) {
                    t->err = std::current_exception();
                }
                {
                    std::lock_guard<std::mutex> g(t->m);
                    t->done = true;
                }
                t->cv.notify_all();
            });
        }
        cv_.notify_one();
        return t;
    }

    // fn(i) for i in [0, n): static blocks over the workers and the calling thread; blocks until
    // every index ran, then rethrows the first exception.
    void parallel_for(size_t n, const std::function<void(size_t)>& fn) {
        if (n == 0) return;
        const size_t parts = std::min(n, (size_t)workers_.size() + 1);
        const size_t chunk = (n + parts - 1) / parts;
        std::vector<TaskPtr> tasks;
        for (size_t p = 1; p < parts; ++p) {
            const size_t lo = p * chunk, hi = std::min(n, lo + chunk);
            if (lo >= hi) break;
            tasks.push_back(submit([&fn, lo, hi] {
                for (size_t i = lo; i < hi; ++i) fn(i);
            }));
        }
        std::exception_ptr first;
        try {
            for (size_t i = 0; i < std::min(n, chunk); ++i) fn(i);
        } catch (...) {
            first = std::current_exception();
        }
        for (auto& t : tasks) {
            try {
                t->wait();
            } catch (...) {
                if (!first) first = std::current_exception();
            }
        }
        if (first) std::rethrow_exception(first);
    }

   private:
    void loop() {
        for (;;) {
            std::function<void()> job;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return stop_ || !q_.empty(); });
                if (stop_ && q_.empty()) return;
                job = std::move(q_.front());
                q_.pop_front();
            }
            job();
        }
    }

    std::vector<std::thread> workers_;
    std::deque<std::function<void()>> q_;
    std::mutex m_;
    std::condition_variable cv_;
    bool stop_ = false;
};

}  // namespace froi
