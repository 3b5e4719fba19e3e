// Persistent host worker pool behind detail::parallel_for (run_internal.hpp).
//
// The host side of a run (frame staging, partial files, map widening, CSV writers) fans out
// over up to 16 threads several times per call; creating those threads per call cost
// 0.1-0.3 ms each time, which is visible next to sub-millisecond device runs (the release
// gate's crossover sweep times whole ddm::run calls at 64x64). Workers are created once
// and sleep on a condition variable between jobs. One job runs at a time; a parallel_for
// issued from inside a job (or while another thread's job is running) runs inline on the
// caller, so nesting never deadlocks.
#include "run_internal.hpp"

#include <condition_variable>

#include <pthread.h>

namespace ddm::detail {

namespace {

thread_local bool tls_in_pool = false;
// a forked child inherits the pool object but none of its threads: it runs jobs inline
std::atomic<bool> g_forked{false};

class Pool {
public:
    Pool() : size_(std::max(1u, std::min(16u, std::thread::hardware_concurrency()))) {
        for (unsigned t = 1; t < size_; ++t) workers_.emplace_back([this] { loop(); });
        pthread_atfork(nullptr, nullptr, [] { g_forked.store(true); });
    }
    ~Pool() {
        if (g_forked.load()) {
            for (auto& w : workers_) w.detach();
            return;
        }
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& w : workers_) w.join();
    }

    void run(std::size_t n, void (*call)(void*, std::size_t), void* ctx) {
        std::unique_lock<std::mutex> busy(job_mu_, std::try_to_lock);
        if (!busy.owns_lock() || size_ < 2 || g_forked.load()) {
            for (std::size_t i = 0; i < n; ++i) call(ctx, i);
            return;
        }
        err_ = nullptr;
        next_.store(0);
        {
            std::lock_guard<std::mutex> lk(mu_);
            n_ = n;
            call_ = call;
            ctx_ = ctx;
            want_ = unsigned(std::min<std::size_t>(n, size_)) - 1;  // workers that join
            joined_ = finished_ = 0;
            ++gen_;
        }
        cv_.notify_all();
        tls_in_pool = true;
        drain();
        tls_in_pool = false;
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return finished_ == want_; });
        if (err_) std::rethrow_exception(err_);
    }

private:
    void drain() {
        for (std::size_t i; (i = next_.fetch_add(1)) < n_;) {
            try {
                call_(ctx_, i);
            } catch (...) {
                std::lock_guard<std::mutex> lk(err_mu_);
                if (!err_) err_ = std::current_exception();
                next_.store(n_);
            }
        }
    }

    void loop() {
        tls_in_pool = true;
        std::uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                if (joined_ >= want_) continue;  // the job has all the workers it asked for
                ++joined_;
            }
            drain();
            std::lock_guard<std::mutex> lk(mu_);
            if (++finished_ == want_) done_cv_.notify_all();
        }
    }

    const unsigned size_;
    std::vector<std::thread> workers_;
    std::mutex job_mu_;  // one job at a time
    std::mutex mu_, err_mu_;
    std::condition_variable cv_, done_cv_;
    std::uint64_t gen_ = 0;
    unsigned want_ = 0, joined_ = 0, finished_ = 0;
    bool stop_ = false;
    std::size_t n_ = 0;
    void (*call_)(void*, std::size_t) = nullptr;
    void* ctx_ = nullptr;
    std::atomic<std::size_t> next_{0};
    std::exception_ptr err_;
};

Pool& pool() {
    static Pool p;
    return p;
}

}  // namespace

void parallel_for_impl(std::size_t n, void (*call)(void*, std::size_t), void* ctx) {
    if (tls_in_pool || n < 2) {
        for (std::size_t i = 0; i < n; ++i) call(ctx, i);
        return;
    }
    pool().run(n, call, ctx);
}

}  // namespace ddm::detail
