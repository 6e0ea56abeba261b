// host_pool.cpp -- see host_pool.h.  Plain C++ threads; no device code.
#include "host_pool.h"

#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <mutex>
#include <thread>
#include <vector>

namespace pdm {
namespace host {
namespace {

inline int64_t now_us() {
    return std::chrono::duration_cast<std::chrono::microseconds>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

struct Job {
    std::atomic<int64_t> next{0};
    std::atomic<int64_t> done{0};
    int64_t n = 0;
    const std::function<void(int64_t)> *fn = nullptr;
};

// Take units until none is left; publish them (stores fenced) with one add.
inline void run(Job *j) {
    int64_t mine = 0;
    for (;;) {
        const int64_t i = j->next.fetch_add(1, std::memory_order_relaxed);
        if (i >= j->n) break;
        (*j->fn)(i);
        ++mine;
    }
    if (mine) {
        _mm_sfence();  // non-temporal stores of the units reach memory first
        j->done.fetch_add(mine, std::memory_order_release);
    }
}

// A helper keeps spinning this long after a job before it sleeps, so the next
// piece of a D' expansion and the next TF change's alpha gather find it
// awake (a futex wake-up costs ~50 us, longer than a whole 2 MB gather):
// the same trade as OpenMP runtimes' spin-before-sleep (GOMP_SPINCOUNT,
// KMP_BLOCKTIME).  PDM_HOST_LINGER_US overrides (0: sleep at once).
int64_t linger_us() {
    static const int64_t v = [] {
        const char *e = getenv("PDM_HOST_LINGER_US");
        return e ? (int64_t)atoll(e) : (int64_t)1000;
    }();
    return v;
}

class Pool {
  public:
    Pool() {
        int hw = (int)std::thread::hardware_concurrency();
        if (const char *e = getenv("PDM_HOST_THREADS")) hw = atoi(e);
        helpers_ = std::max(0, hw - 1);
        for (int i = 0; i < helpers_; ++i) std::thread([this] { loop(); }).detach();
    }

    int threads() const { return helpers_ + 1; }

    void parallel_for(int64_t n, const std::function<void(int64_t)> &fn) {
        if (n <= 0) return;
        std::lock_guard<std::mutex> serial(call_mu_);  // one job at a time
        if (n == 1 || helpers_ == 0) {
            for (int64_t i = 0; i < n; ++i) fn(i);
            _mm_sfence();
            return;
        }
        Job j;
        j.n = n;
        j.fn = &fn;
        {
            std::lock_guard<std::mutex> lk(mu_);
            job_ = &j;
            gen_.fetch_add(1, std::memory_order_release);
        }
        cv_.notify_all();
        run(&j);  // the caller never waits for a helper to start
        while (j.done.load(std::memory_order_acquire) < n) _mm_pause();
        {
            std::lock_guard<std::mutex> lk(mu_);
            job_ = nullptr;  // no helper can take `j` any more ...
        }
        // ... and the ones holding it find its counter exhausted
        while (holders_.load(std::memory_order_acquire) > 0) _mm_pause();
    }

    void prewake(int us) {
        const int64_t until = now_us() + us;
        int64_t cur = spin_until_.load(std::memory_order_relaxed);
        while (cur < until && !spin_until_.compare_exchange_weak(cur, until)) {
        }
        {
            std::lock_guard<std::mutex> lk(mu_);
            wake_.fetch_add(1, std::memory_order_release);
        }
        cv_.notify_all();
    }

  private:
    Job *take(uint64_t &seen) {  // under the lock: the current job, if new
        std::lock_guard<std::mutex> lk(mu_);
        const uint64_t g = gen_.load(std::memory_order_acquire);
        if (g == seen) return nullptr;
        seen = g;
        if (job_) holders_.fetch_add(1, std::memory_order_acq_rel);
        return job_;
    }

    void loop() {
        uint64_t seen = gen_.load(), seen_wake = wake_.load();
        int64_t linger = 0;
        for (;;) {
            Job *j = nullptr;
            // spin phase: after a job (linger) or while a prewake lasts
            for (;;) {
                if (gen_.load(std::memory_order_acquire) != seen) {
                    j = take(seen);
                    break;
                }
                const int64_t t = now_us();
                if (t >= linger && t >= spin_until_.load(std::memory_order_relaxed)) break;
                _mm_pause();
            }
            if (!j) {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] {
                    return gen_.load() != seen || wake_.load() != seen_wake;
                });
                seen_wake = wake_.load();
                const uint64_t g = gen_.load();
                if (g != seen) {
                    seen = g;
                    j = job_;
                    if (j) holders_.fetch_add(1, std::memory_order_acq_rel);
                }
                if (!j) continue;  // a prewake: back to the spin phase
            }
            if (j) {
                run(j);
                holders_.fetch_sub(1, std::memory_order_acq_rel);
                linger = now_us() + linger_us();
            }
        }
    }

    int helpers_ = 0;
    std::mutex call_mu_, mu_;
    std::condition_variable cv_;
    std::atomic<uint64_t> gen_{0}, wake_{0};
    std::atomic<int64_t> spin_until_{0};
    std::atomic<int> holders_{0};
    Job *job_ = nullptr;
};

Pool &pool() {
    static Pool *p = new Pool();  // never destroyed: detached helpers outlive main
    return *p;
}

}  // namespace

void parallel_for(int64_t n, const std::function<void(int64_t)> &fn) {
    pool().parallel_for(n, fn);
}

void prewake(int us) { pool().prewake(us); }

int threads() { return pool().threads(); }

}  // namespace host
}  // namespace pdm
