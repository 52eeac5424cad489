// Host-owned random projection panels (SURVEY.md 8(b) aero_rng_fill): the
// start vectors of power_iteration (linalg.cpp:106-108) and the Pi of
// simul_iter (linalg.cpp:141) are the first r*k Gaussians of one RngState
// fork (rng.hpp:54-78). By default the engine draws them on the device
// (aero_common.cuh rng_gaussian_at: same splitmix stream, device libm, so a
// draw can differ from the host's in the last bit). In panel mode the host
// supplies them instead -- either this library's host restatement of
// rng.hpp (host libm, bit-identical to the reference built on the same host)
// or a caller callback registered through the C-ABI -- and the device reads
// them from an uploaded panel.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/aero_b200.h"
#include "kernels.cuh"

namespace aero_b200 {

// fixed worker pool for the host-side panel fills
class HostPool {
  public:
    static HostPool& get();
    // run fn(i) for i in [0, n) on the pool (and the calling thread); blocks
    void parallel_for(int n, const std::function<void(int)>& fn);
    int workers() const { return (int)th_.size(); }
    ~HostPool();

  private:
    HostPool();
    std::vector<std::thread> th_;
    std::mutex call_mu_;  // one parallel_for at a time; concurrent callers run inline
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int)>* fn_ = nullptr;
    int n_ = 0, next_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
    void work();
};

// i-th Gaussian (0-based) of a fresh RngState with splitmix state0, on the
// host (rng.hpp:60-78 with the host's std::log / std::sin / std::cos)
double host_gaussian_at(uint64_t state0, uint64_t i);

class RngPanels {
  public:
    enum Mode { DEVICE = 0, HOST = 1, CALLBACK = 2 };
    ~RngPanels();
    void set_host() { mode_ = HOST; }
    void set_callback(aero_rng_fill fn, void* ctx) {
        fn_ = fn;
        ctx_ = ctx;
        mode_ = fn ? CALLBACK : DEVICE;
    }
    void set_device() { mode_ = DEVICE; }
    Mode mode() const { return mode_; }
    bool active() const { return mode_ != DEVICE; }
    // assign panel offsets to jobs[0..n) (or -1 in DEVICE mode), fill the
    // panels on the host and enqueue their upload on `st`; returns the device
    // panel base (nullptr in DEVICE mode)
    const double* prepare(cudaStream_t st, IterJob* jobs, int n);
    int64_t values_filled() const { return filled_; }

  private:
    Mode mode_ = DEVICE;
    aero_rng_fill fn_ = nullptr;
    void* ctx_ = nullptr;
    double* host_ = nullptr;  // pinned
    double* dev_ = nullptr;
    size_t cap_ = 0;
    cudaEvent_t free_ = nullptr;  // the previous upload has left host_
    int64_t filled_ = 0;
};

}  // namespace aero_b200
