// Host-side scenario setup: new_environment (src/state.cpp:17-75).
//
// The keyed Fisher-Yates is a sequential swap chain (each swap depends on the
// previous ones), so it stays on the host. Its draws are pure functions of
// (seed, side, i), so they are generated in parallel first; only the swaps
// run in order, over 32-bit cell indices.
#include "pf_setup.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <deque>
#include <exception>
#include <future>
#include <list>
#include <map>
#include <mutex>
#include <thread>
#include <tuple>
#include <vector>

namespace pfhost {

uint64_t philox_bits(uint64_t seed, uint32_t step, uint32_t phase, uint64_t entity, uint32_t counter) {
    uint32_t c0 = uint32_t(entity), c1 = uint32_t(entity >> 32), c2 = step;
    uint32_t c3 = (phase << 28) | (counter & 0x0FFFFFFFu);
    uint32_t k0 = uint32_t(seed), k1 = uint32_t(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = uint64_t(0xD2511F53u) * c0;
        const uint64_t p1 = uint64_t(0xCD9E8D57u) * c2;
        const uint32_t n0 = uint32_t(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n2 = uint32_t(p0 >> 32) ^ c3 ^ k1;
        c1 = uint32_t(p1);
        c3 = uint32_t(p0);
        c0 = n0;
        c2 = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return (uint64_t(c0) << 32) | c1;
}

double uniform(uint64_t seed, uint32_t step, uint32_t phase, uint64_t entity, uint32_t counter) {
    return double(philox_bits(seed, step, phase, entity, counter) >> 11) * 0x1.0p-53;
}

int32_t band_height(int32_t agents_per_side, int32_t width) {
    if (width <= 0) return 0;
    return int32_t((int64_t(agents_per_side) + width - 1) / width);
}

namespace {

// Persistent host worker pool (pool_for): jobs are queued FIFO; workers and
// the submitting thread take ranges of the front job until it is exhausted.
struct PoolJob {
    const std::function<void(size_t, size_t)>* fn;
    size_t n, parts;
    std::atomic<size_t> next{0}, done{0};
    std::mutex m;
    std::condition_variable cv;
};

class Pool {
  public:
    Pool() {
        const size_t hw = std::max<unsigned>(2u, std::thread::hardware_concurrency());
        for (size_t i = 0; i + 1 < std::min<size_t>(hw, 64); ++i) ths_.emplace_back([this] { work(); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : ths_) t.join();
    }
    size_t threads() const { return ths_.size(); }
    void run(size_t n, size_t parts, const std::function<void(size_t, size_t)>& fn) {
        auto job = std::make_shared<PoolJob>();
        job->fn = &fn;
        job->n = n;
        job->parts = parts;
        {
            std::lock_guard<std::mutex> g(mu_);
            q_.push_back(job);
        }
        cv_.notify_all();
        help(*job);
        std::unique_lock<std::mutex> lk(job->m);
        job->cv.wait(lk, [&] { return job->done.load() == job->parts; });
        std::lock_guard<std::mutex> g(mu_);
        for (auto it = q_.begin(); it != q_.end(); ++it)
            if (it->get() == job.get()) {
                q_.erase(it);
                break;
            }
    }

  private:
    static void help(PoolJob& j) {
        for (size_t i; (i = j.next.fetch_add(1)) < j.parts;) {
            (*j.fn)(j.n * i / j.parts, j.n * (i + 1) / j.parts);
            if (j.done.fetch_add(1) + 1 == j.parts) {
                std::lock_guard<std::mutex> g(j.m);
                j.cv.notify_all();
            }
        }
    }
    void work() {
        for (;;) {
            std::shared_ptr<PoolJob> j;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] {
                    if (stop_) return true;
                    for (auto& x : q_)
                        if (x->next.load() < x->parts) return true;
                    return false;
                });
                if (stop_) return;
                for (auto& x : q_)
                    if (x->next.load() < x->parts) {
                        j = x;
                        break;
                    }
            }
            if (j) help(*j);
        }
    }
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::shared_ptr<PoolJob>> q_;
    std::vector<std::thread> ths_;
    bool stop_ = false;
};

Pool& pool() {
    static Pool p;
    return p;
}

}  // namespace

void pool_for(size_t n, size_t parts, const std::function<void(size_t, size_t)>& fn) {
    if (n == 0) return;
    parts = std::max<size_t>(1, std::min(parts, n));
    if (parts == 1) {
        fn(0, n);
        return;
    }
    pool().run(n, parts, fn);
}

size_t pool_threads() { return pool().threads(); }

void parallel_for(size_t n, const std::function<void(size_t, size_t)>& fn) {
    const size_t hw = std::max<size_t>(1, std::thread::hardware_concurrency());
    pool_for(n, std::min<size_t>(hw, std::max<size_t>(1, n / (1u << 16))), fn);
}

void place_side(int32_t width, uint32_t group, int32_t row_begin, int32_t row_end, int32_t n, uint32_t first_id,
                uint64_t seed, const std::function<void(uint32_t cell, uint32_t id)>& put) {
    const uint64_t m = uint64_t(row_end - row_begin) * uint64_t(width);
    if (m == 0 || n == 0) return;
    // Draws: j_i = i + min(floor(u_i * (m - i)), m - i - 1) with
    // u_i = uniform({seed, 0, Placement, side = group, i}) (src/state.cpp:24-30).
    std::vector<uint32_t> jump(m - 1);
    parallel_for(m - 1, [&](size_t b, size_t e) {
        for (size_t i = b; i < e; ++i) {
            const double u = uniform(seed, 0, 0 /*Placement*/, group, uint32_t(i));
            const uint64_t left = m - i;
            const uint64_t off = std::min<uint64_t>(uint64_t(u * double(left)), left - 1);
            jump[i] = uint32_t(off);
        }
    });
    std::vector<uint32_t> cells(m);
    const uint32_t first = uint32_t(uint64_t(row_begin) * uint64_t(width));
    for (uint64_t i = 0; i < m; ++i) cells[i] = first + uint32_t(i);
    for (uint64_t i = 0; i + 1 < m; ++i) std::swap(cells[i], cells[i + jump[i]]);
    for (int32_t k = 0; k < n; ++k) put(cells[size_t(k)], first_id + uint32_t(k));
}

namespace {

using Key = std::tuple<int32_t, int32_t, int32_t, uint64_t>;
using Pending = std::shared_future<std::shared_ptr<const Placement>>;

struct Cache {
    std::mutex mu;
    std::map<Key, Pending> entries;
    std::list<Key> lru;  // front = most recent
    size_t bytes = 0;
    static constexpr size_t kCapacity = size_t(3) << 29;  // 1.5 GB of cell lists
};

Cache& cache() {
    static Cache c;
    return c;
}

std::shared_ptr<const Placement> compute(int32_t width, int32_t height, int32_t n, uint64_t seed) {
    auto pl = std::make_shared<Placement>();
    pl->band = band_height(n, width);
    const int32_t band = pl->band;
    std::exception_ptr err[2];
    auto side = [&](int s) {
        try {
            std::vector<uint32_t>& out = pl->cells[s];
            out.resize(size_t(std::max(0, n)));
            place_side(width, uint32_t(s + 1), s == 0 ? 0 : height - band, s == 0 ? band : height, n, 0, seed,
                       [&](uint32_t cell, uint32_t k) { out[k] = cell; });
        } catch (...) {
            err[s] = std::current_exception();
        }
    };
    std::thread bottom(side, 1);  // the two sides are independent swap chains
    side(0);
    bottom.join();
    for (const auto& e : err)
        if (e) std::rethrow_exception(e);
    return pl;
}

Pending request(int32_t width, int32_t height, int32_t n, uint64_t seed, bool async) {
    Cache& c = cache();
    const Key key{width, height, n, seed};
    std::unique_lock<std::mutex> lk(c.mu);
    auto it = c.entries.find(key);
    if (it != c.entries.end()) {
        c.lru.remove(key);
        c.lru.push_front(key);
        return it->second;
    }
    std::promise<std::shared_ptr<const Placement>> prom;
    Pending fut = prom.get_future().share();
    c.entries.emplace(key, fut);
    c.lru.push_front(key);
    lk.unlock();
    auto work = [width, height, n, seed, key, p = std::move(prom)]() mutable {
        std::shared_ptr<const Placement> pl;
        try {
            pl = compute(width, height, n, seed);
        } catch (...) {  // out of host memory: forget the entry, report to every waiter
            Cache& cc = cache();
            {
                std::lock_guard<std::mutex> g(cc.mu);
                cc.entries.erase(key);
                cc.lru.remove(key);
            }
            p.set_exception(std::current_exception());
            return;
        }
        Cache& cc = cache();
        {
            std::lock_guard<std::mutex> g(cc.mu);
            cc.bytes += pl->bytes();
            // Evict least recently used finished entries beyond the capacity.
            const std::vector<Key> order(cc.lru.rbegin(), cc.lru.rend());
            for (const Key& k : order) {
                if (cc.bytes <= Cache::kCapacity) break;
                auto e = cc.entries.find(k);
                if (k == key || e == cc.entries.end() ||
                    e->second.wait_for(std::chrono::seconds(0)) != std::future_status::ready)
                    continue;
                cc.bytes -= e->second.get()->bytes();
                cc.entries.erase(e);
                cc.lru.remove(k);
            }
        }
        p.set_value(std::move(pl));
    };
    if (async) std::thread(std::move(work)).detach();
    else work();
    return fut;
}

}  // namespace

std::shared_ptr<const Placement> placement(int32_t width, int32_t height, int32_t n, uint64_t seed) {
    return request(width, height, n, seed, false).get();
}

void prefetch_placement(int32_t width, int32_t height, int32_t n, uint64_t seed) {
    request(width, height, n, seed, true);
}

void place_all(int32_t width, int32_t height, int32_t n, uint64_t seed,
               const std::function<void(uint32_t cell, uint32_t id, uint32_t group)>& put) {
    if (n <= 0) return;
    const std::shared_ptr<const Placement> pl = placement(width, height, n, seed);
    parallel_for(size_t(n), [&](size_t b, size_t e) {
        for (size_t k = b; k < e; ++k) {
            put(pl->cells[0][k], uint32_t(k) + 1, 1);
            put(pl->cells[1][k], uint32_t(n) + uint32_t(k) + 1, 2);
        }
    });
}

}  // namespace pfhost
