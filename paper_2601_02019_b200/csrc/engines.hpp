// Wrappers above the single-level Sketch: MlState (sliding window), the
// distributed coordinator merge, the AMM CodState, and the stream generator.
#pragma once

#include <cstdint>
#include <deque>
#include <memory>
#include <vector>

#include "../../include/aero_b200.h"
#include "sketch.hpp"

namespace aero_b200 {

// ---- MlState (sliding_window.hpp:39-81, sliding_window.cpp:15-156) --------
struct HeavyRow {
    std::vector<double> row;
    int64_t s, t;
};
class MlEngine {
  public:
    MlEngine(int d, int64_t n, double r_max, double eps, uint64_t seed, uint64_t stream, int device,
             double delta = 0.0);
    ~MlEngine();
    MlEngine(const MlEngine&) = delete;
    MlEngine& operator=(const MlEngine&) = delete;
    void update_block(const double* rows, bool device, int64_t n, int64_t ld, const int64_t* t);
    void query(double* out_host, aero_ml_query_result* res);
    void info(aero_ml_info* out) const;
    int levels() const { return (int)levels_.size(); }
    Sketch& level(int j) { return *levels_[j]; }
    int64_t heavy_count(int j) const;
    void heavy_get(int j, int64_t idx, double* row, int64_t* s, int64_t* t) const;

  private:
    struct LevelQueue {  // replay view of the combined per-level queue
        int64_t avail = 0;  // snapshots at the front of the sketch deque created so far
    };
    int64_t combined_len(int j) const;
    int64_t front_t(int j) const;
    int64_t front_s(int j) const;
    int64_t tail_t(int j) const;
    void pop_front(int j);
    int d_, ell_, dev_;
    int64_t n_, cap_, clock_ = 0, norm_warnings_ = 0;
    double r_max_, eps_, window_mass_ = 0.0;
    bool amplified_ = false;  // levels update_amplified (sliding_window.cpp:90-91)
    std::vector<std::unique_ptr<Sketch>> levels_;
    std::vector<std::deque<HeavyRow>> heavy_;
    std::vector<LevelQueue> lq_;
    std::deque<double> ring_;
    DeviceBuf stage_, gather_, nrm_, out_, qa_, qb_;
    int* bad_d_ = nullptr;                     // K1 finiteness flags (stage rows)
    std::vector<DeviceBuf> gath_;              // per-level gathered rows
    std::vector<int64_t*> gidx_d_;             // per-level gather indices (device)
    std::vector<size_t> gidx_n_;
    cudaStream_t st_ = nullptr;
};

// ---- distributed (distributed.cpp:31-173) ---------------------------------
void dist_theta_schedule(int m, int64_t T, double eps, int64_t latency, const double* sq_norms,
                         double* theta_out, int64_t* mass_bytes, int64_t* broadcasts);
// streaming form of the replay (state persists across advance() calls)
class DistProtocol {
  public:
    // window > 0: sliding-window protocol (distributed.cpp:33-55: exact
    // window mass per site, signed FroMass deltas, theta = eps * own window
    // mass; the broadcast replaces the estimate, distributed.cpp:27-30)
    DistProtocol(int m, double eps, int64_t latency, int64_t window = 0);
    void advance(int64_t T, const double* sq_norms, double* theta_out);
    int64_t ticks = 0, bytes = 0, broadcasts = 0;
    double f_hat = 0.0;

  private:
    int m_;
    double eps_;
    int64_t latency_, window_;
    std::vector<double> f_local_, f_self_, f_known_, w_local_, w_sent_;
    std::vector<std::deque<double>> ring_;
    int msg_count_ = 0;
    std::deque<std::pair<int64_t, double>> to_coord_, to_sites_;
};
// The coordinator's share on one rank. Whole-stream mode: shipped snapshots
// are folded into one fp64 d x d accumulator (CoordinatorState::receive,
// distributed.cpp:124-136). Sliding-window mode: a contribution lives from its
// delivery (t + latency) until its Expire message is delivered
// (t + window + latency, distributed.cpp:87-97,137-144); the live snapshots
// stay factored in the site's own queue (the coordinator's cache) and a probe
// restores them, so an expiry is a queue pop, not a d x d subtraction.
class Coordinator {
  public:
    Coordinator(int d, int m, int device, void* nccl_comm, int64_t window = 0, int64_t latency = 0);
    ~Coordinator();
    // ship the site's snapshots up to its clock; returns the protocol bytes of
    // the SnapshotUpdate (and, window mode, Expire) messages sent since the last call
    int64_t absorb(Sketch& site);
    void probe(const std::vector<Sketch*>& sites, int root, int ell, double* out_host, double* gram_host);
    // shrink_to_sketch of a merged Gram supplied by the host (a merge done
    // over a non-NCCL process group)
    void shrink(const double* gram_host, int ell, double* out_host);

  private:
    int d_, m_, dev_;
    void* comm_;
    int64_t window_, latency_;
    struct SiteBook {
        int64_t shipped_t = 0;  // snapshots with t <= shipped_t were counted as sent
        std::deque<int64_t> unexpired;  // shipped snapshot times whose Expire is not sent yet
    };
    std::vector<std::pair<const Sketch*, SiteBook>> books_;
    SiteBook& book(const Sketch* s);
    DeviceBuf B_, P_, W_, out_;
    cudaStream_t st_ = nullptr;
};
void nccl_unique_id(char* id128);
void* nccl_comm_init(const char* id128, int nranks, int rank, int device);
void nccl_comm_destroy(void* comm);

// ---- CodState (amm.hpp:35-69, amm.cpp:27-122) --------------------------------
class CodEngine {
  public:
    CodEngine(int dx, int dy, double eps, double theta, int64_t n, uint64_t seed, uint64_t stream,
              int device);
    ~CodEngine();
    void update_block(const double* xs, const double* ys, int64_t n, const int64_t* t,
                      aero_event* log);
    void query(double* astar, double* bstar);
    void query_product(double* p);
    void info(int32_t* ell, int64_t* cols, int64_t* snaps, int64_t* clock) const;
    double theta() const;
    void set_theta(double theta);  // amm.cpp:38-41
    int64_t window() const;
    int64_t snap_count() const;
    int64_t snap_t(int64_t idx) const;  // queue order (oldest first)

  private:
    struct Impl;
    Impl* im_;
};

// ---- AdaptiveState (amm.hpp:71-93, amm.cpp:131-161) ------------------------
// main/auxiliary CodEngine pair; the threshold doubles / halves with the main
// queue length. Rows run through both engines in chunks that provably contain
// no adaptation point except possibly their last row (the queue grows by at
// most one snapshot per row, and expiry is known from the snapshot times), so
// each engine keeps its speculative row batches.
class AdaptiveEngine {
  public:
    AdaptiveEngine(int dx, int dy, double eps, double theta0, int64_t n, uint64_t seed,
                   uint64_t stream, int device);
    void update_block(const double* xs, const double* ys, int64_t n, const int64_t* t,
                      aero_event* log, int32_t* level_out);
    CodEngine& main() { return *main_; }
    CodEngine& aux() { return *aux_; }
    int level() const { return level_; }

  private:
    int dx_, dy_, dev_;
    double eps_;
    int64_t n_;
    int level_ = 1;
    uint64_t seed_, stream_, forks_ = 0;  // rng_ of amm.hpp:92 (parent stream)
    std::unique_ptr<CodEngine> main_, aux_;
};

// ---- generator ---------------------------------------------------------------
void gen_rows_device(const aero_gen_params& p, int64_t t0, int64_t n, double* out, int device);

// shrink_to_sketch on device: B (d x d, device, destroyed) -> out (ell x d
// row-major, device)
void shrink_device(cudaStream_t st, int d, int ell, double* B, double* w, double* out);

}  // namespace aero_b200
