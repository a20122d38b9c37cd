// Host thread pool for the automaton build (parallel.hpp).
#include "parallel.hpp"

#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <mutex>
#include <thread>

namespace acg {

namespace {

class Pool {
public:
    explicit Pool(unsigned threads) {
        for (unsigned i = 1; i < threads; ++i) workers_.emplace_back([this] { loop(); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    unsigned size() const { return static_cast<unsigned>(workers_.size()) + 1; }

    // false when another caller holds the pool (the caller then runs inline)
    bool run(std::size_t n, std::size_t grain, const std::function<void(std::size_t, std::size_t)>& f) {
        std::unique_lock<std::mutex> owner(busy_, std::try_to_lock);
        if (!owner.owns_lock()) return false;
        {
            std::lock_guard<std::mutex> g(mu_);
            f_ = &f;
            n_ = n;
            grain_ = grain;
            next_.store(0, std::memory_order_relaxed);
            active_ = static_cast<unsigned>(workers_.size());
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> g(mu_);
        done_cv_.wait(g, [this] { return active_ == 0; });
        f_ = nullptr;
        return true;
    }

private:
    void work() {
        for (;;) {
            const std::size_t lo = next_.fetch_add(grain_, std::memory_order_relaxed);
            if (lo >= n_) return;
            (*f_)(lo, std::min(n_, lo + grain_));
        }
    }
    void loop() {
        std::uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> g(mu_);
                cv_.wait(g, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
            }
            work();
            std::lock_guard<std::mutex> g(mu_);
            if (--active_ == 0) done_cv_.notify_one();
        }
    }

    std::vector<std::thread> workers_;
    std::mutex busy_, mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(std::size_t, std::size_t)>* f_ = nullptr;
    std::size_t n_ = 0, grain_ = 1;
    std::atomic<std::size_t> next_{0};
    unsigned active_ = 0;
    std::uint64_t gen_ = 0;
    bool stop_ = false;
};

unsigned want_threads() {
    unsigned t = std::thread::hardware_concurrency();
    if (const char* e = std::getenv("ACG_BUILD_THREADS")) {
        const long v = std::strtol(e, nullptr, 10);
        if (v >= 1) t = static_cast<unsigned>(v);
    }
    return std::max(1u, std::min(t, 64u));
}

Pool& pool() {
    static Pool p(want_threads());
    return p;
}

}  // namespace

unsigned build_threads() { return pool().size(); }

void parallel_for(std::size_t n, std::size_t grain, const std::function<void(std::size_t, std::size_t)>& f) {
    if (n == 0) return;
    grain = std::max<std::size_t>(grain, 1);
    if (n <= grain || build_threads() == 1 || !pool().run(n, grain, f)) f(0, n);
}

}  // namespace acg
