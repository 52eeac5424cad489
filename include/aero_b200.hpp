// aero_b200.hpp -- header-only C++ shim over the C-ABI (aero_b200.h) that
// mirrors the reference's C++ sketch API (/root/reference/proj/include/aero):
//   aero::b200::AeroState   <-> aero::AeroState   (sketch.hpp:42-99)
//   aero::b200::AttpState   <-> aero::AttpState   (attp.hpp:15-43)
//   aero::b200::MlState     <-> aero::MlState     (sliding_window.hpp:39-81)
//   aero::b200::CodState    <-> aero::CodState    (amm.hpp:35-69)
//   aero::b200::AdaptiveState <-> aero::AdaptiveState (amm.hpp:71-93)
// Status codes are rethrown as the reference's exception types
// (errors.hpp:15-33). Vectors are raw pointers / std::vector (row-major), so a
// maintainer keeps the Eigen call sites by passing a.data().
#ifndef AERO_B200_HPP
#define AERO_B200_HPP

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "aero_b200.h"

namespace aero {
namespace b200 {

struct InvalidInput : std::invalid_argument {
    explicit InvalidInput(const std::string& w) : std::invalid_argument(w) {}
};
struct FormatError : std::runtime_error {
    explicit FormatError(const std::string& w) : std::runtime_error(w) {}
};
struct ProtocolError : std::runtime_error {
    explicit ProtocolError(const std::string& w) : std::runtime_error(w) {}
};
struct OracleCapExceeded : std::runtime_error {
    explicit OracleCapExceeded(const std::string& w) : std::runtime_error(w) {}
};
struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};

inline void check(int rc) {
    if (rc == AERO_OK) return;
    const std::string msg = aero_last_error();
    switch (rc) {
        case AERO_INVALID_INPUT: throw InvalidInput(msg);
        case AERO_FORMAT_ERROR: throw FormatError(msg);
        case AERO_PROTOCOL_ERROR: throw ProtocolError(msg);
        case AERO_ORACLE_CAP_EXCEEDED: throw OracleCapExceeded(msg);
        case AERO_CUDA_ERROR: throw CudaError(msg);
        default: throw std::runtime_error(msg);
    }
}

using UpdateStats = aero_event;  // doubling_steps, simul_calls, gate_fired, dumped, reduced

struct Snapshot {
    std::vector<double> z;  // d x xi row-major
    std::vector<double> m;  // xi x d row-major
    int xi = 0;
    std::int64_t s = 0, t = 0;
    double theta = 0.0;
};

class AeroState {
  public:
    // AeroState(d, eps, theta, RngState(seed, stream)) (sketch.cpp:22-31)
    // delta > 0: probability amplification (sketch.hpp:44-46)
    AeroState(int d, double eps, double theta, std::uint64_t seed, std::uint64_t stream,
              int device = 0, int theta_mode = AERO_THETA_FIXED, double delta = 0.0) {
        aero_cfg c{};
        c.d = d;
        c.eps = eps;
        c.theta = theta;
        c.seed = seed;
        c.stream = stream;
        c.device = device;
        c.theta_mode = theta_mode;
        c.delta = delta;
        check(aero_create(&c, &h_));
    }
    AeroState(const AeroState&) = delete;
    AeroState& operator=(const AeroState&) = delete;
    AeroState(AeroState&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    virtual ~AeroState() { aero_destroy(h_); }

    void update(const double* a, std::int64_t i) { check(aero_update_block(h_, a, 1, d(), &i, nullptr, nullptr)); }
    void update(const std::vector<double>& a, std::int64_t i) {
        if ((int)a.size() != d()) throw InvalidInput("AeroState: row dimension mismatch");
        update(a.data(), i);
    }
    // sketch.cpp:45-48
    void update_amplified(const double* a, std::int64_t i) {
        check(aero_update_block_amplified(h_, a, 1, d(), &i, nullptr, nullptr));
    }
    // caller-owned random projections (aero_set_rng_fill)
    void set_rng_fill(aero_rng_fill fn, void* ctx) { check(aero_set_rng_fill(h_, fn, ctx)); }
    // n sequential updates of row-major rows (the block API the reference lacks)
    void update_block(const double* rows, std::int64_t n, const std::int64_t* t,
                      std::vector<UpdateStats>* log = nullptr) {
        if (log) log->resize(n);
        check(aero_update_block(h_, rows, n, d(), t, nullptr, log ? log->data() : nullptr));
    }
    // ell x d row-major (sketch.cpp:143-160)
    std::vector<double> query(std::int64_t lb, std::int64_t ub) const {
        std::vector<double> out((size_t)ell() * d());
        check(aero_query(h_, lb, ub, out.data()));
        return out;
    }
    void set_theta(double theta) { check(aero_set_theta(h_, theta)); }
    int d() const { return info().d; }
    int ell() const { return info().ell; }
    double theta() const { return info().theta; }
    std::int64_t clock() const { return info().clock; }
    std::int64_t last_dump_time() const { return info().last_dump_t; }
    std::vector<double> residual() const {
        const aero_info i = info();
        std::vector<double> out((size_t)i.rows * i.d);
        check(aero_residual(h_, out.data(), i.rows));
        return out;
    }
    std::int64_t snap_count() const {
        std::int64_t n = 0;
        check(aero_snap_count(h_, &n));
        return n;
    }
    Snapshot snap(std::int64_t idx) const {
        Snapshot s;
        check(aero_snap_info(h_, idx, &s.xi, &s.s, &s.t, &s.theta));
        s.z.resize((size_t)d() * s.xi);
        s.m.resize((size_t)d() * s.xi);
        check(aero_snap_get(h_, idx, s.z.data(), s.m.data()));
        return s;
    }
    void snap_pop_front() { check(aero_snap_pop_front(h_)); }
    UpdateStats last_update_stats() const {
        UpdateStats e{};
        check(aero_last_stats(h_, &e));
        return e;
    }
    aero_info info() const {
        aero_info i{};
        check(aero_get_info(h_, &i));
        return i;
    }
    aero_sketch* handle() const { return h_; }

  protected:
    explicit AeroState(aero_sketch* h) : h_(h) {}
    aero_sketch* h_ = nullptr;
};

// AttpState (attp.hpp:15-43): theta = eps * running mass, query(t) = prefix sketch
class AttpState : public AeroState {
  public:
    AttpState(int d, double eps, std::uint64_t seed, std::uint64_t stream, int device = 0)
        : AeroState(d, eps, 0.0, seed, stream, device, AERO_THETA_ATTP) {}
    std::vector<double> query(std::int64_t t) const {
        std::vector<double> out((size_t)ell() * d());
        check(aero_attp_query(h_, t, out.data()));
        return out;
    }
    double fro_mass() const { return info().fro_mass; }
};

// MlState (sliding_window.hpp:39-81)
class MlState {
  public:
    MlState(int d, std::int64_t n, double r_max, double eps, std::uint64_t seed,
            std::uint64_t stream, int device = 0)
        : d_(d) {
        check(aero_ml_create(d, n, r_max, eps, seed, stream, device, &h_));
    }
    MlState(const MlState&) = delete;
    MlState& operator=(const MlState&) = delete;
    ~MlState() { aero_ml_destroy(h_); }
    void update(const double* a, std::int64_t i) { check(aero_ml_update_block(h_, a, 1, d_, &i)); }
    void update_block(const double* rows, std::int64_t n, const std::int64_t* t) {
        check(aero_ml_update_block(h_, rows, n, d_, t));
    }
    struct QueryResult {
        std::vector<double> sketch;  // ell x d
        int level = 0;
        bool fallback = false;
        std::int64_t xi_sum = 0;
        int heavy_used = 0;
    };
    QueryResult query() const {
        aero_ml_info inf{};
        check(aero_ml_get_info(h_, &inf));
        QueryResult q;
        q.sketch.resize((size_t)inf.ell * d_);
        aero_ml_query_result r{};
        check(aero_ml_query(h_, q.sketch.data(), &r));
        q.level = r.level;
        q.fallback = r.fallback != 0;
        q.xi_sum = r.xi_sum;
        q.heavy_used = r.heavy_used;
        return q;
    }
    int levels() const {
        aero_ml_info inf{};
        check(aero_ml_get_info(h_, &inf));
        return inf.levels;
    }
    double theta(int j) const { return aero_ml_theta(h_, j); }

  private:
    int d_;
    aero_ml* h_ = nullptr;
};

// CodState (amm.hpp:35-69)
class CodState {
  public:
    CodState(int dx, int dy, double eps, double theta, std::int64_t n, std::uint64_t seed,
             std::uint64_t stream, int device = 0)
        : dx_(dx), dy_(dy) {
        check(aero_cod_create(dx, dy, eps, theta, n, seed, stream, device, &h_));
    }
    CodState(const CodState&) = delete;
    CodState& operator=(const CodState&) = delete;
    ~CodState() { aero_cod_destroy(h_); }
    void update(const double* x, const double* y, std::int64_t i) {
        check(aero_cod_update_block(h_, x, y, 1, &i, nullptr));
    }
    // (a*: dx x ell, b*: dy x ell) row-major
    std::pair<std::vector<double>, std::vector<double>> query() const {
        std::int32_t ell = 0;
        check(aero_cod_info(h_, &ell, nullptr, nullptr, nullptr));
        std::vector<double> a((size_t)dx_ * ell), b((size_t)dy_ * ell);
        check(aero_cod_query(h_, a.data(), b.data()));
        return {std::move(a), std::move(b)};
    }

    double theta() const {
        double t = 0.0;
        check(aero_cod_theta(h_, &t));
        return t;
    }
    void set_theta(double theta) { check(aero_cod_set_theta(h_, theta)); }

  private:
    int dx_, dy_;
    aero_cod* h_ = nullptr;
};

// AdaptiveState (amm.hpp:71-93): main/aux CodState pair, threshold doubling /
// halving with main's queue length
class AdaptiveState {
  public:
    AdaptiveState(int dx, int dy, double eps, double theta0, std::int64_t n, std::uint64_t seed,
                  std::uint64_t stream, int device = 0)
        : dx_(dx), dy_(dy), ell_(static_cast<int>(std::ceil(2.0 / eps))) {
        check(aero_adaptive_create(dx, dy, eps, theta0, n, seed, stream, device, &h_));
    }
    AdaptiveState(const AdaptiveState&) = delete;
    AdaptiveState& operator=(const AdaptiveState&) = delete;
    ~AdaptiveState() { aero_adaptive_destroy(h_); }
    void update(const double* x, const double* y, std::int64_t i) {
        check(aero_adaptive_update_block(h_, x, y, 1, &i, nullptr, nullptr));
    }
    int level() const {
        std::int32_t lv = 0;
        check(aero_adaptive_info(h_, &lv, nullptr, nullptr, nullptr, nullptr));
        return lv;
    }
    std::pair<std::vector<double>, std::vector<double>> query() const {
        std::vector<double> a((size_t)dx_ * ell_), b((size_t)dy_ * ell_);
        check(aero_adaptive_query(h_, a.data(), b.data()));
        return {std::move(a), std::move(b)};
    }

  private:
    int dx_, dy_, ell_;
    aero_adaptive* h_ = nullptr;
};

}  // namespace b200
}  // namespace aero

#endif  // AERO_B200_HPP
