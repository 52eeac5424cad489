// MlState, distributed coordinator (NCCL), generator; see engines.hpp.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <exception>
#include <limits>
#include <mutex>
#include <thread>

#include "aero_common.cuh"
#include "engines.hpp"

namespace aero_b200 {

void shrink_device(cudaStream_t st, int d, int ell, double* B, double* w, double* out) {
    eigh(st, d, B, d, w, 1, 0, std::min(ell, d));
    shrink_rows(st, w, B, d, d, ell, out);
}

// ============================================================================
// MlState
// ============================================================================
// sliding_window.cpp:15-30
MlEngine::MlEngine(int d, int64_t n, double r_max, double eps, uint64_t seed, uint64_t stream,
                   int device, double delta)
    : d_(d), dev_(device), n_(n), r_max_(r_max), eps_(eps), amplified_(delta != 0.0) {
    if (n < 1) throw InvalidInput("MlState: window size must be >= 1");
    if (r_max < 1.0) throw InvalidInput("MlState: r_max must be >= 1 (squared norms in [1, R])");
    if (!(eps > 0.0 && eps <= 1.0)) throw InvalidInput("MlState: eps out of (0,1]");
    if (d < 1) throw InvalidInput("AeroState: d must be >= 1");
    ell_ = static_cast<int>(std::ceil(2.0 / eps));
    cap_ = static_cast<int64_t>(std::ceil(8.0 / eps));
    const int big_l = static_cast<int>(std::ceil(std::log2(std::max(r_max, 2.0))));
    AERO_CUDA(cudaSetDevice(dev_));
    AERO_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    for (int j = 0; j < std::max(big_l, 1); ++j) {
        aero_cfg c{};
        c.d = d;
        c.eps = eps;
        c.theta = std::pow(2.0, j) * eps * static_cast<double>(n);
        c.seed = seed;
        c.stream = fork_stream(stream, (uint64_t)(j + 1));  // levels_[j] gets rng.fork()
        c.device = device;
        c.theta_mode = AERO_THETA_FIXED;
        c.delta = delta;
        levels_.emplace_back(new Sketch(c));
        heavy_.emplace_back();
        lq_.emplace_back();
    }
    // the levels ingest concurrently: their cooperative iterate launches must
    // co-reside instead of serializing on the whole GPU
    for (auto& l : levels_) l->set_grid_share(levels());
}

int64_t MlEngine::combined_len(int j) const {
    return lq_[j].avail + (int64_t)heavy_[j].size();
}
int64_t MlEngine::front_t(int j) const {
    int64_t t = std::numeric_limits<int64_t>::max();
    if (lq_[j].avail > 0) t = std::min(t, levels_[j]->snaps().front().t);
    if (!heavy_[j].empty()) t = std::min(t, heavy_[j].front().t);
    return t;
}
int64_t MlEngine::front_s(int j) const {
    const bool se = lq_[j].avail == 0, he = heavy_[j].empty();
    if (se && he) return std::numeric_limits<int64_t>::max();
    if (se) return heavy_[j].front().s;
    if (he) return levels_[j]->snaps().front().s;
    const auto& sf = levels_[j]->snaps().front();
    return (sf.t <= heavy_[j].front().t) ? sf.s : heavy_[j].front().s;
}
int64_t MlEngine::tail_t(int j) const {
    int64_t t = 0;
    if (lq_[j].avail > 0) t = std::max(t, levels_[j]->snaps()[lq_[j].avail - 1].t);
    if (!heavy_[j].empty()) t = std::max(t, heavy_[j].back().t);
    return t;
}
void MlEngine::pop_front(int j) {
    const bool se = lq_[j].avail == 0, he = heavy_[j].empty();
    if (se && he) return;
    if (he || (!se && levels_[j]->snaps().front().t <= heavy_[j].front().t)) {
        levels_[j]->snap_pop_front();
        lq_[j].avail--;
    } else {
        heavy_[j].pop_front();
    }
}

MlEngine::~MlEngine() {
    cudaSetDevice(dev_);
    for (auto& l : levels_) l->synchronize();
    if (bad_d_) cudaFree(bad_d_);
    for (int64_t* p : gidx_d_)
        if (p) cudaFree(p);
}

// sliding_window.cpp:67-100. Level sketches ingest their (non-heavy) rows of
// a block concurrently (one host thread + CUDA stream per level); the
// combined-queue bookkeeping (expiry, heavy routing, cap) is then replayed
// row by row exactly in the reference order, bit-exact on int64 indices.
void MlEngine::update_block(const double* rows, bool device, int64_t n, int64_t ld,
                            const int64_t* t) {
    if (n <= 0) return;
    if (ld < d_) throw InvalidInput("MlState: row dimension mismatch");
    AERO_CUDA(cudaSetDevice(dev_));
    const int64_t S = 4096;
    stage_.alloc((size_t)S * d_);
    nrm_.alloc(S);
    std::vector<double> nrm_h(S);
    if (!bad_d_) AERO_CUDA(cudaMalloc(&bad_d_, sizeof(int) * S));
    int* bad_d = bad_d_;
    std::vector<int> bad_h(S);
    const int L = levels();
    if ((int)gath_.size() < L) {
        gath_.resize(L);
        gidx_d_.resize(L, nullptr);
        gidx_n_.resize(L, 0);
    }
    for (int64_t off = 0; off < n; off += S) {
        const int64_t cnt = std::min(S, n - off);
        AERO_CUDA(cudaMemcpy2DAsync(stage_.p, sizeof(double) * d_, rows + off * ld,
                                    sizeof(double) * ld, sizeof(double) * d_, cnt,
                                    device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st_));
        ingest_rows(st_, stage_.p, cnt, d_, d_, nrm_.p, bad_d);
        AERO_CUDA(cudaMemcpyAsync(nrm_h.data(), nrm_.p, sizeof(double) * cnt, cudaMemcpyDeviceToHost, st_));
        AERO_CUDA(cudaMemcpyAsync(bad_h.data(), bad_d, sizeof(int) * cnt, cudaMemcpyDeviceToHost, st_));
        AERO_CUDA(cudaStreamSynchronize(st_));
        int64_t good = cnt;
        std::string err;
        int64_t prev = (off == 0) ? clock_ : t[off - 1];
        for (int64_t j = 0; j < cnt; ++j) {
            if (bad_h[j]) { good = j; err = "MlState: non-finite row"; break; }
            if (t[off + j] <= prev) { good = j; err = "MlState: timestamp regression"; break; }
            prev = t[off + j];
        }
        // heavy routing per level (nsq >= theta_j bypasses the level sketch)
        std::vector<std::vector<int64_t>> sub(L);
        for (int lv = 0; lv < L; ++lv)
            for (int64_t j = 0; j < good; ++j)
                if (!(nrm_h[j] >= levels_[lv]->theta())) sub[lv].push_back(j);
        // level sketches in parallel
        std::vector<std::exception_ptr> errs(L);
        std::vector<std::thread> th;
        for (int lv = 0; lv < L; ++lv) {
            th.emplace_back([&, lv] {
                try {
                    AERO_CUDA(cudaSetDevice(dev_));
                    const auto& idx = sub[lv];
                    if (idx.empty()) return;
                    std::vector<int64_t> ts(idx.size());
                    for (size_t q = 0; q < idx.size(); ++q) ts[q] = t[off + idx[q]];
                    const double* src = stage_.p;
                    if ((int64_t)idx.size() != good) {  // gather the level's rows (one kernel)
                        gath_[lv].alloc(idx.size() * (size_t)d_);
                        if (gidx_n_[lv] < idx.size()) {
                            if (gidx_d_[lv]) cudaFree(gidx_d_[lv]);
                            AERO_CUDA(cudaMalloc(&gidx_d_[lv], sizeof(int64_t) * S));
                            gidx_n_[lv] = S;
                        }
                        cudaStream_t ls = levels_[lv]->stream();
                        AERO_CUDA(cudaMemcpyAsync(gidx_d_[lv], idx.data(), sizeof(int64_t) * idx.size(),
                                                  cudaMemcpyHostToDevice, ls));
                        gather_rows(ls, stage_.p, d_, gidx_d_[lv], (int64_t)idx.size(), d_, gath_[lv].p);
                        src = gath_[lv].p;
                    }
                    levels_[lv]->update_block(src, true, (int64_t)idx.size(), d_, ts.data(), nullptr,
                                              nullptr, amplified_);
                    levels_[lv]->synchronize();
                } catch (...) {
                    errs[lv] = std::current_exception();
                }
            });
        }
        for (auto& x : th) x.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
        // bookkeeping replay (sliding_window.cpp:72-98)
        std::vector<double> rowbuf;
        for (int64_t j = 0; j < good; ++j) {
            const int64_t i = t[off + j];
            const double nsq = nrm_h[j];
            if (nsq < 1.0 || nsq > r_max_) ++norm_warnings_;
            ring_.push_back(nsq);
            window_mass_ += nsq;
            while ((int64_t)ring_.size() > n_) {
                window_mass_ -= ring_.front();
                ring_.pop_front();
            }
            for (int lv = 0; lv < L; ++lv) {
                while (combined_len(lv) > 0 && front_t(lv) <= i - n_) pop_front(lv);
                if (nsq >= levels_[lv]->theta()) {
                    if (rowbuf.empty()) {
                        rowbuf.resize(d_);
                        if (device)
                            AERO_CUDA(cudaMemcpy(rowbuf.data(), rows + (off + j) * ld,
                                                 sizeof(double) * d_, cudaMemcpyDeviceToHost));
                        else
                            std::memcpy(rowbuf.data(), rows + (off + j) * ld, sizeof(double) * d_);
                    }
                    heavy_[lv].push_back(HeavyRow{rowbuf, tail_t(lv) + 1, i});
                } else {
                    const auto& sn = levels_[lv]->snaps();
                    while (lq_[lv].avail < (int64_t)sn.size() && sn[lq_[lv].avail].t <= i)
                        lq_[lv].avail++;
                }
                while (combined_len(lv) > cap_) pop_front(lv);
            }
            rowbuf.clear();
            clock_ = i;
        }
        if (good < cnt) throw InvalidInput(err);
    }
}

// sliding_window.cpp:102-146
void MlEngine::query(double* out_host, aero_ml_query_result* res) {
    if (clock_ == 0) throw InvalidInput("MlState: query before any update");
    AERO_CUDA(cudaSetDevice(dev_));
    const int64_t t_now = clock_;
    const int64_t wstart = t_now - n_;
    const int64_t head = std::max<int64_t>(wstart + 1, 1);
    aero_ml_query_result r{};
    int pick = -1;
    for (int j = 0; j < levels(); ++j) {
        if (combined_len(j) == 0) continue;
        const int64_t s0 = front_s(j);
        if (s0 >= 1 && s0 <= head) {
            pick = j;
            break;
        }
    }
    if (pick < 0) {
        r.fallback = 1;
        double guess = 0.0;
        if (window_mass_ > 0.0) guess = std::floor(std::log2(window_mass_ / (double)n_));
        pick = (int)std::clamp(guess, 0.0, (double)(levels() - 1));
    }
    r.level = pick;
    Sketch& lv = *levels_[pick];
    cudaStream_t st = lv.stream();
    const int64_t lb = std::max<int64_t>(wstart, 0);
    qa_.alloc((size_t)ell_ * d_ + d_);
    double* base = qa_.p;  // ell x d row-major == d x ell column-major
    if (lv.clock() > lb) {
        double* B = const_cast<double*>(lv.query_gram_device(lb, lv.clock()));
        shrink_device(st, d_, ell_, B, base + (size_t)ell_ * d_, base);
    } else {
        fill_zero(st, base, (int64_t)ell_ * d_);
    }
    for (const SnapRec& s : lv.snaps())
        if (s.t > wstart && s.t <= t_now) r.xi_sum += s.xi;
    std::vector<const HeavyRow*> hv;
    for (const HeavyRow& h : heavy_[pick])
        if (h.t > wstart && h.t <= t_now) hv.push_back(&h);
    r.heavy_used = (int)hv.size();
    // stack [base; heavy rows] and shrink again (sliding_window.cpp:135-144)
    qb_.alloc((size_t)d_ * d_ + (size_t)d_ * std::max<size_t>(hv.size(), 1) + d_);
    double* Gm = qb_.p;
    double* Hm = Gm + (size_t)d_ * d_;
    double* w = Hm + (size_t)d_ * std::max<size_t>(hv.size(), 1);
    dgemm(st, false, true, d_, d_, ell_, 1.0, base, d_, base, d_, 0.0, Gm, d_);
    if (!hv.empty()) {
        std::vector<double> hh((size_t)d_ * hv.size());
        for (size_t q = 0; q < hv.size(); ++q)
            std::memcpy(hh.data() + q * d_, hv[q]->row.data(), sizeof(double) * d_);
        AERO_CUDA(cudaMemcpyAsync(Hm, hh.data(), sizeof(double) * hh.size(), cudaMemcpyHostToDevice, st));
        dgemm(st, false, true, d_, d_, (int)hv.size(), 1.0, Hm, d_, Hm, d_, 1.0, Gm, d_);
        AERO_CUDA(cudaStreamSynchronize(st));
    }
    out_.alloc((size_t)ell_ * d_);
    shrink_device(st, d_, ell_, Gm, w, out_.p);
    AERO_CUDA(cudaMemcpyAsync(out_host, out_.p, sizeof(double) * ell_ * d_, cudaMemcpyDeviceToHost, st));
    AERO_CUDA(cudaStreamSynchronize(st));
    if (res) *res = r;
}

void MlEngine::info(aero_ml_info* o) const {
    o->d = d_;
    o->ell = ell_;
    o->levels = levels();
    o->n = n_;
    o->cap = cap_;
    o->clock = clock_;
    o->norm_warnings = norm_warnings_;
    int64_t total = (int64_t)ring_.size();  // sliding_window.cpp:148-156
    for (int j = 0; j < levels(); ++j) {
        total += (int64_t)levels_[j]->rows() * d_;
        for (const SnapRec& s : levels_[j]->snaps()) total += 2 * (int64_t)s.xi * d_;
        total += (int64_t)heavy_[j].size() * d_;
    }
    o->stored_floats = total;
    o->window_mass = window_mass_;
}
int64_t MlEngine::heavy_count(int j) const {
    if (j < 0 || j >= levels()) throw InvalidInput("MlState: level out of range");
    return (int64_t)heavy_[j].size();
}
void MlEngine::heavy_get(int j, int64_t idx, double* row, int64_t* s, int64_t* t) const {
    if (j < 0 || j >= levels() || idx < 0 || idx >= (int64_t)heavy_[j].size())
        throw InvalidInput("MlState: heavy index out of range");
    const HeavyRow& h = heavy_[j][idx];
    if (row) std::memcpy(row, h.row.data(), sizeof(double) * d_);
    if (s) *s = h.s;
    if (t) *t = h.t;
}

// ============================================================================
// distributed
// ============================================================================
// Norm-only replay of the whole-stream mass protocol (distributed.cpp:31-69
// for the site side, :107-123 for the coordinator, :201-239 for the tick loop
// and FIFO latencies). Snapshot messages ride the same FIFO but never change
// the mass estimate, so every site's threshold is a function of norms alone.
DistProtocol::DistProtocol(int m, double eps, int64_t latency, int64_t window)
    : m_(m), eps_(eps), latency_(latency), window_(window), f_local_(m > 0 ? m : 0, 0.0),
      f_self_(m > 0 ? m : 0, 0.0), f_known_(m > 0 ? m : 0, 0.0), w_local_(m > 0 ? m : 0, 0.0),
      w_sent_(m > 0 ? m : 0, 0.0), ring_(window > 0 && m > 0 ? m : 0) {
    if (m < 1) throw InvalidInput("run_simulation: m must be >= 1");
    if (!(eps > 0.0 && eps <= 1.0)) throw InvalidInput("run_simulation: eps out of (0,1]");
    if (latency < 0) throw InvalidInput("run_simulation: latency must be >= 0");
    if (window < 0) throw InvalidInput("run_simulation: window must be >= 0");
}

// ticks ticks+1 .. ticks+T; site j's norms at sq_norms[j * T + q]
void DistProtocol::advance(int64_t T, const double* sq_norms, double* theta_out) {
    const int m = m_;
    const double eps = eps_;
    const bool win = window_ > 0;
    for (int64_t q = 0; q < T; ++q) {
        const int64_t i = ticks + q + 1;
        while (!to_sites_.empty() && to_sites_.front().first <= i) {  // distributed.cpp:211-215
            const double fb = to_sites_.front().second;
            for (int j = 0; j < m; ++j) f_known_[j] = win ? fb : std::max(f_known_[j], fb);  // :27-30
            to_sites_.pop_front();
        }
        for (int j = 0; j < m; ++j) {
            const double nsq = sq_norms[(int64_t)j * T + q];
            if (win) {  // SiteState::update, distributed.cpp:33-55
                std::deque<double>& ring = ring_[j];
                ring.push_back(nsq);
                w_local_[j] += nsq;
                while ((int64_t)ring.size() > window_) {
                    w_local_[j] -= ring.front();
                    ring.pop_front();
                }
                const double delta = w_local_[j] - w_sent_[j];
                if (std::abs(delta) >= (eps / m) * f_known_[j]) {
                    to_coord_.emplace_back(i + latency_, delta);
                    bytes += 8 + 16;
                    w_sent_[j] = w_local_[j];
                }
                theta_out[(int64_t)j * T + q] = eps * w_local_[j];
            } else {  // SiteState::update, distributed.cpp:57-69
                f_local_[j] += nsq;
                if (f_local_[j] >= (eps / m) * f_known_[j]) {
                    to_coord_.emplace_back(i + latency_, f_local_[j]);
                    bytes += 8 + 16;
                    f_self_[j] += f_local_[j];
                    f_local_[j] = 0.0;
                }
                theta_out[(int64_t)j * T + q] = eps * std::max(f_known_[j], f_self_[j] + f_local_[j]);
            }
        }
        while (!to_coord_.empty() && to_coord_.front().first <= i) {  // distributed.cpp:231-239
            const double f = to_coord_.front().second;
            to_coord_.pop_front();
            if (!win && !(f >= 0.0)) throw ProtocolError("FroMass: negative mass");
            f_hat = std::max(f_hat + f, 0.0);  // CoordinatorState::receive, :109-123
            if (++msg_count_ >= m) {
                msg_count_ = 0;
                ++broadcasts;
                bytes += (int64_t)m * (8 + 16);
                to_sites_.emplace_back(i + 1 + latency_, f_hat);
            }
        }
    }
    ticks += T;
}

void dist_theta_schedule(int m, int64_t T, double eps, int64_t latency, const double* sq_norms,
                         double* theta_out, int64_t* mass_bytes, int64_t* broadcasts) {
    DistProtocol p(m, eps, latency);
    p.advance(T, sq_norms, theta_out);
    if (mass_bytes) *mass_bytes = p.bytes;
    if (broadcasts) *broadcasts = p.broadcasts;
}

Coordinator::Coordinator(int d, int m, int device, void* comm, int64_t window, int64_t latency)
    : d_(d), m_(m), dev_(device), comm_(comm), window_(window), latency_(latency) {
    if (d < 1) throw InvalidInput("CoordinatorState: d must be >= 1");
    if (m < 1) throw InvalidInput("CoordinatorState: site count must be >= 1");
    if (window < 0 || latency < 0) throw InvalidInput("CoordinatorState: window and latency must be >= 0");
    AERO_CUDA(cudaSetDevice(dev_));
    AERO_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    B_.alloc((size_t)d * d);
    fill_zero(st_, B_.p, (int64_t)d * d);
    AERO_CUDA(cudaStreamSynchronize(st_));
}
Coordinator::~Coordinator() {
    cudaSetDevice(dev_);
    if (st_) {
        cudaStreamSynchronize(st_);
        eigh_forget(st_);
        cudaStreamDestroy(st_);
    }
}
Coordinator::SiteBook& Coordinator::book(const Sketch* s) {
    for (auto& kv : books_)
        if (kv.first == s) return kv.second;
    books_.emplace_back(s, SiteBook{});
    return books_.back().second;
}
// The site ships every snapshot as it is produced (distributed.cpp:74-85);
// bytes = Message::bytes (distributed.hpp:33-42). Whole-stream mode folds the
// delivered ones (t + latency <= clock) into B (CoordinatorState::receive,
// distributed.cpp:124-136). Window mode also counts the Expire notices sent by
// the site's update at tick t + window (distributed.cpp:87-97) and drops the
// contributions whose Expire has been delivered (t + window + latency <= clock).
int64_t Coordinator::absorb(Sketch& site) {
    if (site.d() != d_) throw ProtocolError("SnapshotUpdate: inconsistent payload shapes");
    AERO_CUDA(cudaSetDevice(dev_));
    SiteBook& bk = book(&site);
    const int64_t clock = site.clock();
    int64_t bytes = 0;
    for (const SnapRec& r : site.snaps()) {
        if (r.t <= bk.shipped_t) continue;
        bytes += 8 * (2 * (int64_t)d_ * r.xi) + 16;
        if (window_ > 0) bk.unexpired.push_back(r.t);
    }
    if (!site.snaps().empty()) bk.shipped_t = std::max(bk.shipped_t, site.snaps().back().t);
    if (window_ > 0) {
        while (!bk.unexpired.empty() && bk.unexpired.front() + window_ <= clock) {
            bytes += 8 + 16;  // Expire
            bk.unexpired.pop_front();
        }
        while (site.snap_count() > 0 && site.snaps().front().t + window_ + latency_ <= clock)
            site.snap_pop_front();
        return bytes;
    }
    int64_t ns = 0;
    while (ns < site.snap_count() && site.snaps()[ns].t + latency_ <= clock) ++ns;
    if (ns > 0) {
        site.synchronize();
        site.accumulate_restore(B_.p, 0, ns);  // on the site's stream
        site.synchronize();
        for (int64_t i = 0; i < ns; ++i) site.snap_pop_front();
    }
    return bytes;
}
void Coordinator::probe(const std::vector<Sketch*>& sites, int root, int ell, double* out_host,
                        double* gram_host) {
    AERO_CUDA(cudaSetDevice(dev_));
    P_.alloc((size_t)d_ * d_);
    copy_matrix(st_, d_, d_, B_.p, d_, P_.p, d_);
    AERO_CUDA(cudaStreamSynchronize(st_));
    for (Sketch* site : sites) {  // residual Grams (distributed.cpp:162-165)
        site->accumulate_residual(P_.p, 1.0);
        if (window_ > 0) {  // live (delivered, unexpired) contributions (:166-172)
            const int64_t clock = site->clock();
            int64_t lo = 0, hi = 0;
            const int64_t ns = site->snap_count();
            while (lo < ns && site->snaps()[lo].t + window_ + latency_ <= clock) ++lo;
            hi = lo;
            while (hi < ns && site->snaps()[hi].t + latency_ <= clock) ++hi;
            if (hi > lo) site->accumulate_restore(P_.p, lo, hi);
        }
        site->synchronize();
    }
    double* G = P_.p;
    int rank = 0;
    if (comm_) {
        ncclComm_t c = static_cast<ncclComm_t>(comm_);
        ncclCommUserRank(c, &rank);
        W_.alloc((size_t)d_ * d_);
        if (ncclReduce(P_.p, W_.p, (size_t)d_ * d_, ncclDouble, ncclSum, root, c, st_) != ncclSuccess)
            throw CudaError("ncclReduce failed");
        G = W_.p;
    }
    if (rank == root) {
        if (gram_host) {
            AERO_CUDA(cudaMemcpyAsync(gram_host, G, sizeof(double) * d_ * d_, cudaMemcpyDeviceToHost, st_));
            AERO_CUDA(cudaStreamSynchronize(st_));
        }
        if (out_host && ell > 0) {
            out_.alloc((size_t)ell * d_ + d_);
            shrink_device(st_, d_, ell, G, out_.p + (size_t)ell * d_, out_.p);
            AERO_CUDA(cudaMemcpyAsync(out_host, out_.p, sizeof(double) * ell * d_, cudaMemcpyDeviceToHost, st_));
        }
    }
    AERO_CUDA(cudaStreamSynchronize(st_));
}

void Coordinator::shrink(const double* gram_host, int ell, double* out_host) {
    if (ell < 1) throw InvalidInput("shrink_to_sketch: ell must be >= 1");
    AERO_CUDA(cudaSetDevice(dev_));
    P_.alloc((size_t)d_ * d_);
    out_.alloc((size_t)ell * d_ + d_);
    AERO_CUDA(cudaMemcpyAsync(P_.p, gram_host, sizeof(double) * d_ * d_, cudaMemcpyHostToDevice, st_));
    shrink_device(st_, d_, ell, P_.p, out_.p + (size_t)ell * d_, out_.p);
    AERO_CUDA(cudaMemcpyAsync(out_host, out_.p, sizeof(double) * ell * d_, cudaMemcpyDeviceToHost, st_));
    AERO_CUDA(cudaStreamSynchronize(st_));
}

void nccl_unique_id(char* id128) {
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) throw CudaError("ncclGetUniqueId failed");
    std::memcpy(id128, id.internal, 128);
}
void* nccl_comm_init(const char* id128, int nranks, int rank, int device) {
    AERO_CUDA(cudaSetDevice(device));
    ncclUniqueId id;
    std::memcpy(id.internal, id128, 128);
    ncclComm_t c = nullptr;
    if (ncclCommInitRank(&c, nranks, id, rank) != ncclSuccess) throw CudaError("ncclCommInitRank failed");
    return c;
}
void nccl_comm_destroy(void* comm) {
    if (comm) ncclCommDestroy(static_cast<ncclComm_t>(comm));
}

// ============================================================================
// generator
// ============================================================================
namespace {
// host RngState (rng.hpp:21-87) for the basis draws
struct HostRng {
    uint64_t state;
    bool spare_ok = false;
    double spare = 0.0;
    HostRng(uint64_t seed, uint64_t stream) : state(rng_state0(seed, stream)) {}
    double uniform() {
        state += kGolden;
        return static_cast<double>((mix_out(state) >> 11) + 1) * 0x1.0p-53;
    }
    double gaussian() {
        if (spare_ok) {
            spare_ok = false;
            return spare;
        }
        const double u1 = uniform(), u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 6.283185307179586476925286766559 * u2;
        spare = r * std::sin(a);
        spare_ok = true;
        return r * std::cos(a);
    }
};
// U (k x d row-major, orthonormal rows) = Q^T of the thin QR (R diag >= 0) of a
// d x k Gaussian drawn row-major (DESIGN.md GENERATOR spec; oracle gen_basis)
std::vector<double> host_basis(uint64_t seed, uint64_t basis_id, int d, int k) {
    HostRng rng(seed, 0xB000000000000000ULL ^ basis_id);
    std::vector<double> a((size_t)d * k);  // column-major d x k
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < k; ++j) a[i + (size_t)j * d] = rng.gaussian();
    // modified Householder QR, Q formed explicitly
    std::vector<double> v((size_t)d * k), tau(k), rdiag(k);
    for (int j = 0; j < k; ++j) {
        double* col = &a[(size_t)j * d];
        double nrm = 0.0;
        for (int i = j; i < d; ++i) nrm += col[i] * col[i];
        nrm = std::sqrt(nrm);
        const double alpha = col[j];
        const double beta = (alpha >= 0.0) ? -nrm : nrm;
        double* vj = &v[(size_t)j * d];
        for (int i = 0; i < j; ++i) vj[i] = 0.0;
        vj[j] = alpha - beta;
        for (int i = j + 1; i < d; ++i) vj[i] = col[i];
        double vn = 0.0;
        for (int i = j; i < d; ++i) vn += vj[i] * vj[i];
        tau[j] = vn > 0.0 ? 2.0 / vn : 0.0;
        rdiag[j] = beta;
        for (int c = j; c < k; ++c) {
            double* cc = &a[(size_t)c * d];
            double s = 0.0;
            for (int i = j; i < d; ++i) s += vj[i] * cc[i];
            s *= tau[j];
            for (int i = j; i < d; ++i) cc[i] -= s * vj[i];
        }
    }
    std::vector<double> q((size_t)d * k, 0.0);
    for (int j = 0; j < k; ++j) q[j + (size_t)j * d] = 1.0;
    for (int j = k - 1; j >= 0; --j) {
        const double* vj = &v[(size_t)j * d];
        for (int c = 0; c < k; ++c) {
            double* qc = &q[(size_t)c * d];
            double s = 0.0;
            for (int i = j; i < d; ++i) s += vj[i] * qc[i];
            s *= tau[j];
            for (int i = j; i < d; ++i) qc[i] -= s * vj[i];
        }
    }
    std::vector<double> u((size_t)k * d);
    for (int j = 0; j < k; ++j) {
        const double sg = (rdiag[j] < 0.0) ? -1.0 : 1.0;  // qr(): R diag >= 0 (linalg.cpp:86-92)
        for (int i = 0; i < d; ++i) u[(size_t)j * d + i] = sg * q[i + (size_t)j * d];
    }
    return u;
}
}  // namespace

void gen_rows_device(const aero_gen_params& p, int64_t t0, int64_t n, double* out, int device) {
    if (p.d < 1 || p.k < 0 || p.k2 < 0 || n < 0 || t0 < 1) throw InvalidInput("gen_rows: bad params");
    AERO_CUDA(cudaSetDevice(device));
    cudaStream_t st;
    AERO_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    double *u1 = nullptr, *u2 = nullptr;
    AERO_CUDA(cudaMalloc(&u1, sizeof(double) * std::max<size_t>((size_t)p.k * p.d, 1)));
    AERO_CUDA(cudaMalloc(&u2, sizeof(double) * std::max<size_t>((size_t)p.k2 * p.d, 1)));
    if (p.k2 > 0) {
        const auto h2 = host_basis(p.seed, (1ULL << 40) + p.stream, p.d, p.k2);
        AERO_CUDA(cudaMemcpy(u2, h2.data(), sizeof(double) * h2.size(), cudaMemcpyHostToDevice));
    }
    int64_t q = 0;
    while (q < n) {
        const int64_t t = t0 + q;
        const int64_t epoch = p.drift_period > 0 ? (t - 1) / p.drift_period : 0;
        int64_t seg = n - q;
        if (p.drift_period > 0) seg = std::min(seg, (epoch + 1) * p.drift_period + 1 - t);
        if (p.k > 0) {
            const auto h1 = host_basis(p.seed, (p.basis_stream << 20) + (uint64_t)epoch, p.d, p.k);
            AERO_CUDA(cudaMemcpy(u1, h1.data(), sizeof(double) * h1.size(), cudaMemcpyHostToDevice));
        }
        gen_rows(st, p.d, p.k, p.k2, u1, u2, p.rho, p.rho2, p.scale2, p.noise, p.r_max, p.seed,
                 p.stream, t, seg, out + q * p.d);
        AERO_CUDA(cudaStreamSynchronize(st));
        q += seg;
    }
    cudaFree(u1);
    cudaFree(u2);
    cudaStreamDestroy(st);
}

// ============================================================================
// CodState -- see cod.cu
// ============================================================================

}  // namespace aero_b200
