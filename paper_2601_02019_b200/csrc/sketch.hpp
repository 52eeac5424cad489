// Host-side engine of one AeroState on a B200: device-resident buffer C'
// (d x 2ell, column-major == reference row-major rows), its Gram G = C'C'^T
// (2ell x 2ell), snapshot arena; host-side control mirrors
// /root/reference/proj/src/sketch.cpp:82-141 with speculative row batching.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <deque>
#include <string>
#include <vector>

#include "../../include/aero_b200.h"
#include "kernels.cuh"
#include "rng_panels.hpp"

namespace aero_b200 {

struct Chunk {
    double* z = nullptr;   // d x cap (column-major): snapshot directions
    double* mt = nullptr;  // d x cap: m^T of each snapshot (m = (C'z)^T C')
    int cap = 0, used = 0, live = 0;
};
struct SnapRec {
    int xi;
    int64_t s, t;
    double theta;
    Chunk* chunk;
    int col;
};

struct DeviceBuf {  // RAII device allocation
    double* p = nullptr;
    size_t n = 0;
    void alloc(size_t count);
    void release();
    ~DeviceBuf() { release(); }
};

class Sketch {
  public:
    explicit Sketch(const aero_cfg& cfg);
    ~Sketch();
    Sketch(const Sketch&) = delete;
    Sketch& operator=(const Sketch&) = delete;

    void set_theta(double th);
    // sketches sharing one GPU concurrently (MlState levels, co-hosted sites):
    // cooperative iterate launches use at most 1/share of the resident CTAs so
    // that the sharers' persistent kernels co-run instead of serializing
    void set_grid_share(int share) { grid_share_ = share < 1 ? 1 : share; }
    // rows: host or device pointer (row-major, ld); n sequential updates
    // amplified: n sequential update_amplified calls (sketch.cpp:45-48); an
    // AttpState built with delta always amplifies (attp.hpp:24)
    void update_block(const double* rows, bool device, int64_t n, int64_t ld, const int64_t* t,
                      const double* theta_per_row, aero_event* log, bool amplified = false);
    double delta() const { return delta_; }
    // restored Gram (sketch.cpp:146-159) into device d x d buffer; returns ptr
    const double* query_gram_device(int64_t lb, int64_t ub);
    void query(int64_t lb, int64_t ub, double* out_host);       // ell x d
    void query_gram(int64_t lb, int64_t ub, double* out_host);  // d x d
    void residual(double* out, int64_t max_rows);
    int64_t snap_count() const { return (int64_t)snaps_.size(); }
    const SnapRec& snap(int64_t i) const;
    void snap_get(int64_t i, double* z, double* m);
    void snap_pop_front();
    void info(aero_info* out) const;
    const aero_event& last_event() const { return last_ev_; }
    void synchronize();
    // start-vector / Pi panels from the host (rng_panels.hpp): fn == nullptr
    // with host == true uses the library's host restatement of rng.hpp
    void set_rng_source(bool host, aero_rng_fill fn, void* ctx);
    RngPanels::Mode rng_mode() const { return rng_.mode(); }
    bool host_rng_default() const { return host_rng_default_; }

    int d() const { return d_; }
    int ell() const { return ell_; }
    int rows() const { return r_; }
    int64_t clock() const { return clock_; }
    double theta() const { return theta_; }
    double eps() const { return eps_; }
    int device() const { return dev_; }
    cudaStream_t stream() const { return st_; }
    const double* buffer() const { return C_.p; }  // d x rows column-major
    // snapshot device views for the coordinator / queries
    const std::deque<SnapRec>& snaps() const { return snaps_; }
    // add restore contributions of snaps [first, last) into device B (d x d)
    void accumulate_restore(double* B, int64_t first, int64_t last);
    // B += C C^T of the live residual
    void accumulate_residual(double* B, double beta_first);

    // counters
    int64_t rows_processed = 0, batches = 0, mispredicts = 0;
    int64_t end_nofire = 0, end_fired = 0, end_doubling = 0, end_dump = 0;
    aero_profile prof{};
    bool profiling = false;

  private:
    enum Pattern { NOFIRE = 0, FIRE1 = 1 };
    void process_rows(const double* dev_rows, int64_t n, const int64_t* t, const double* thetas,
                      aero_event* log);
    int64_t run_batch(const double* dev_rows, int64_t B, const int64_t* t, const double* thetas,
                      aero_event* log);
    void single_row(const double* dev_row, int64_t t, double theta, aero_event* ev);
    void append_rows(const double* dev_rows, int64_t B);
    void reduce();
    // finish a row whose gate fired: doubling from k (forks already consumed up
    // to the gate / previous steps); uses device X/H columns of a job if given
    void doubling(int k, int64_t t, double theta, aero_event* ev);
    void dump_from_job(int col, int k, int xi, int64_t t, double theta, bool zero_buffer);
    // run jobs already written to jobs_h_ (njobs); results in sig_h_/status_h_/clamp_h_
    void run_iterate(int njobs, int R, int max_k);
    void run_simul_large(int k, uint64_t fork, int r, int q);
    // sketch.cpp:55-79: r candidates at eps_si = 0.2 scored by s power
    // iterations on the residual; leaves the winner in H col 0 / vr / sig_h_
    // and returns whether its buffer was exactly zero
    bool amplified_factorize(int k, aero_event* ev);
    uint64_t fork_state0(uint64_t n) const;
    Chunk* arena_alloc(int xi, int* col);
    void arena_release(const SnapRec& s);
    void ensure_query_buffers();

    // config
    int d_, ell_, cap_, kp_, q_, mode_, max_batch_, cur_batch_ = 64;
    bool exact_;
    std::vector<cudaEvent_t> ev_pool_;
    cudaEvent_t evA_ = nullptr, evB_ = nullptr;
    cudaEvent_t ev_at(size_t i);
    double eps_, eps_si_;
    double delta_ = 0.0;  // amplification failure bound (sketch.hpp:44-46), 0 = none
    bool amp_ = false;    // the current update_block call is amplified
    DeviceBuf Gres_, Hc_, Hb_, vrc_, vrb_;  // amplification: residual Gram, candidate / best factors
    uint64_t seed_, stream_;
    int dev_;
    cudaStream_t st_ = nullptr;
    // host state
    double theta_, fro_mass_ = 0.0;
    bool host_prof_ = getenv("AERO_HOST_PROF") != nullptr;  // dev instrumentation
    double prof_append_ms_ = 0.0, prof_iter_ms_ = 0.0;
    int cfg_max_batch_ = 0;  // caller-set batch cap (0 = engine default)
    int grid_share_ = 1;
    int64_t clock_ = 0, last_dump_t_ = 0;
    uint64_t forks_ = 0;
    int r_ = 0;
    Pattern pattern_ = FIRE1;
    double fire_ema_ = 1.0;   // moving average of gate fires (batch prediction)
    double end_rate_ = 0.01;  // moving average of batch-ending rows per row (batch size)
    std::deque<SnapRec> snaps_;
    std::deque<Chunk*> chunks_;
    aero_event last_ev_{};
    // device buffers
    DeviceBuf C_, C2_, G_, E_, ew_, fw_, stage_[2], nrm_, X_, Y_, H_, sig_, vr_, small_, Bq_, Wq_,
        qw_, qy_, ws_;
    static constexpr int kMaxPhases = 256;
    int* phase_d_ = nullptr;   // per-phase active columns | split-K factors (persistent iterate)
    int* phase_h_ = nullptr;
    unsigned* bar_d_ = nullptr;  // grid-barrier counter of the persistent iterate
    bool persistent_ = getenv("AERO_NO_PERSISTENT") == nullptr;  // dev A/B switch
    // iteration products of large buffers on the int8 tensor cores (ozaki.cu);
    // AERO_PRODUCT_I8=0 keeps them on fp64 DMMA (dev A/B switch)
    bool i8_ = !(getenv("AERO_PRODUCT_I8") && getenv("AERO_PRODUCT_I8")[0] == '0');
    // buffer rows from which it is used (tools/product_i8_bench.py: at r = 1500,
    // n = 128..192 it beats DMMA); AERO_I8_MIN_ROWS overrides (tests force it on)
    int i8_min_rows_ = getenv("AERO_I8_MIN_ROWS") ? atoi(getenv("AERO_I8_MIN_ROWS")) : 1024;
    // int8 iterate: slices used by the steering phases / full-precision tail phases per job
    int oz_se_ = getenv("AERO_OZ_SE") ? std::min(ozaki_slices(), std::max(ozaki_slices() - 1, atoi(getenv("AERO_OZ_SE"))))
                                      : ozaki_slices();
    int oz_tail_ = getenv("AERO_OZ_TAIL") ? std::max(1, atoi(getenv("AERO_OZ_TAIL"))) : 3;
    OzakiGram oz_;
    RngPanels rng_;
    bool host_rng_default_ = false;  // AERO_FLAG_HOST_RNG
    const double* panel_d_ = nullptr;  // this launch's host-supplied panels (or nullptr)
    // assign panels to jobs_h_[0..njobs) and upload them (before the jobs H2D)
    void prepare_rng(int njobs) { panel_d_ = rng_.prepare(st_, jobs_h_, njobs); }
    double host_wall_s_ = 0.0, host_sync_s_ = 0.0;  // dev instrumentation (AERO_HOST_PROF)
    int64_t host_syncs_ = 0;
    int* status_d_ = nullptr;
    int* clamp_d_ = nullptr;
    int* colmask_d_ = nullptr;
    int* bad_d_ = nullptr;  // 2 x stage_rows_ (one half per staging buffer)
    cudaStream_t cs_ = nullptr;  // staging stream: H2D + K1 of chunk k+1 overlap chunk k
    cudaEvent_t ev_ready_[2] = {nullptr, nullptr}, ev_free_[2] = {nullptr, nullptr};
    IterJob* jobs_d_ = nullptr;
    int ldx_ = 0, ncols_ = 0, kv_ = 64, stage_rows_ = 0;
    // pinned host mirrors
    IterJob* jobs_h_ = nullptr;
    int* colmask_h_ = nullptr;
    double* sig_h_ = nullptr;
    int* status_h_ = nullptr;
    int* clamp_h_ = nullptr;
    double* nrm_h_ = nullptr;
    int* bad_h_ = nullptr;
};

}  // namespace aero_b200
