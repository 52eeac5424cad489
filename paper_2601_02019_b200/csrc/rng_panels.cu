// Host-owned random projection panels (rng_panels.hpp).
#include <algorithm>
#include <cmath>
#include <string>

#include "aero_common.cuh"
#include "rng_panels.hpp"

namespace aero_b200 {

// ---------------------------------------------------------------- pool
HostPool& HostPool::get() {
    static HostPool pool;
    return pool;
}

HostPool::HostPool() {
    const char* env = getenv("AERO_RNG_THREADS");
    int n = env ? atoi(env) : (int)std::thread::hardware_concurrency();
    n = std::max(0, std::min(n, 32) - 1);  // the caller is one of the workers
    for (int i = 0; i < n; ++i) th_.emplace_back([this] { work(); });
}

HostPool::~HostPool() {
    {
        std::lock_guard<std::mutex> lk(mu_);
        stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
}

void HostPool::work() {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> lk(mu_);
    while (true) {
        cv_.wait(lk, [&] { return stop_ || (gen_ != seen && next_ < n_); });
        if (stop_) return;
        seen = gen_;
        while (next_ < n_) {
            const int i = next_++;
            const auto* fn = fn_;
            lk.unlock();
            (*fn)(i);
            lk.lock();
            if (--pending_ == 0) done_cv_.notify_all();
        }
    }
}

void HostPool::parallel_for(int n, const std::function<void(int)>& fn) {
    if (n <= 0) return;
    std::unique_lock<std::mutex> cl(call_mu_, std::try_to_lock);
    if (th_.empty() || n == 1 || !cl.owns_lock()) {
        for (int i = 0; i < n; ++i) fn(i);
        return;
    }
    std::unique_lock<std::mutex> lk(mu_);
    fn_ = &fn;
    n_ = n;
    next_ = 0;
    pending_ = n;
    ++gen_;
    cv_.notify_all();
    while (next_ < n_) {  // the caller works too
        const int i = next_++;
        lk.unlock();
        fn(i);
        lk.lock();
        --pending_;
    }
    done_cv_.wait(lk, [&] { return pending_ == 0; });
    fn_ = nullptr;
    n_ = 0;
}

// ---------------------------------------------------------------- draws
// rng.hpp:60-78: uniform = (splitmix >> 11) + 1 scaled by 2^-53; a Gaussian
// pair from one Box-Muller step (cos first, the sin value is the cached spare)
double host_gaussian_at(uint64_t state0, uint64_t i) {
    const uint64_t p = i >> 1;
    const double u1 = rng_uniform_at(state0, 2 * p + 1);
    const double u2 = rng_uniform_at(state0, 2 * p + 2);
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    return (i & 1) ? r * std::sin(a) : r * std::cos(a);
}

// ---------------------------------------------------------------- panels
RngPanels::~RngPanels() {
    if (free_) {
        cudaEventSynchronize(free_);
        cudaEventDestroy(free_);
    }
    if (host_) cudaFreeHost(host_);
    if (dev_) cudaFree(dev_);
}

const double* RngPanels::prepare(cudaStream_t st, IterJob* jobs, int n) {
    if (mode_ == DEVICE) {
        for (int j = 0; j < n; ++j) jobs[j].panel = -1;
        return nullptr;
    }
    size_t total = 0;
    for (int j = 0; j < n; ++j) {
        jobs[j].panel = (int)total;
        total += (size_t)jobs[j].r * jobs[j].k;
        total += total & 1;  // 16-byte aligned panels
    }
    if (total > (size_t)INT32_MAX) throw InvalidInput("rng panel exceeds 2^31 values");
    if (!free_) AERO_CUDA(cudaEventCreateWithFlags(&free_, cudaEventDisableTiming));
    // the previous upload must have read host_ before it is overwritten
    AERO_CUDA(cudaEventSynchronize(free_));
    if (total > cap_) {
        if (host_) cudaFreeHost(host_);
        if (dev_) {
            AERO_CUDA(cudaStreamSynchronize(st));
            cudaFree(dev_);
        }
        cap_ = std::max(total, cap_ * 2);
        AERO_CUDA(cudaMallocHost(&host_, sizeof(double) * cap_));
        AERO_CUDA(cudaMalloc(&dev_, sizeof(double) * cap_));
    }
    // work items: (job, chunk) so that one large simul panel still spreads
    // over the pool; callbacks take whole jobs (they return a fork's prefix)
    constexpr int64_t kChunk = 16384;
    struct Item {
        int job;
        int64_t lo, hi;
    };
    std::vector<Item> items;
    for (int j = 0; j < n; ++j) {
        const int64_t cnt = (int64_t)jobs[j].r * jobs[j].k;
        if (mode_ == CALLBACK || cnt <= kChunk) {
            items.push_back({j, 0, cnt});
        } else {
            for (int64_t lo = 0; lo < cnt; lo += kChunk) items.push_back({j, lo, std::min(cnt, lo + kChunk)});
        }
    }
    std::vector<int> rc(items.size(), 0);
    HostPool::get().parallel_for((int)items.size(), [&](int i) {
        const Item& it = items[i];
        const IterJob& jb = jobs[it.job];
        double* out = host_ + jb.panel + it.lo;
        if (mode_ == CALLBACK) {
            rc[i] = fn_(ctx_, jb.fork, out, it.hi - it.lo);
        } else {
            int64_t e = it.lo;
            if (e & 1) {
                out[0] = host_gaussian_at(jb.rng0, (uint64_t)e);
                ++e;
            }
            for (; e + 1 < it.hi; e += 2) {  // one Box-Muller step per pair
                const uint64_t p = (uint64_t)e >> 1;
                const double u1 = rng_uniform_at(jb.rng0, 2 * p + 1);
                const double u2 = rng_uniform_at(jb.rng0, 2 * p + 2);
                const double r = std::sqrt(-2.0 * std::log(u1));
                const double a = 6.283185307179586476925286766559 * u2;
                out[e - it.lo] = r * std::cos(a);
                out[e + 1 - it.lo] = r * std::sin(a);
            }
            if (e < it.hi) out[e - it.lo] = host_gaussian_at(jb.rng0, (uint64_t)e);
        }
    });
    for (size_t i = 0; i < items.size(); ++i)
        if (rc[i] != 0)
            throw InvalidInput("aero_rng_fill callback failed for fork " + std::to_string(jobs[items[i].job].fork));
    AERO_CUDA(cudaMemcpyAsync(dev_, host_, sizeof(double) * total, cudaMemcpyHostToDevice, st));
    AERO_CUDA(cudaEventRecord(free_, st));
    filled_ += (int64_t)total;
    return dev_;
}

}  // namespace aero_b200
