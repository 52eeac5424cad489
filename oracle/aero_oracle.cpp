// =============================================================================
// aero_oracle.cpp -- CPU ORACLE (test infrastructure only; see header).
// Each function cites the reference file:line it restates. LAPACK/BLAS come
// from the scipy wheel's OpenBLAS (LP64, scipy_-prefixed symbols).
// =============================================================================
#include "aero_oracle.hpp"

#include <algorithm>
#include <cstring>
#include <limits>

extern "C" {
void scipy_dgemm_(const char*, const char*, const int*, const int*, const int*, const double*,
                  const double*, const int*, const double*, const int*, const double*, double*,
                  const int*, size_t, size_t);
void scipy_dgemv_(const char*, const int*, const int*, const double*, const double*, const int*,
                  const double*, const int*, const double*, double*, const int*, size_t);
void scipy_dgesdd_(const char*, const int*, const int*, double*, const int*, double*, double*,
                   const int*, double*, const int*, double*, const int*, int*, int*, size_t);
void scipy_dsyevd_(const char*, const char*, const int*, double*, const int*, double*, double*,
                   const int*, int*, const int*, int*, size_t, size_t);
void scipy_dgeqrf_(const int*, const int*, double*, const int*, double*, double*, const int*,
                   int*);
void scipy_dorgqr_(const int*, const int*, const int*, double*, const int*, const double*,
                   double*, const int*, int*);
void scipy_openblas_set_num_threads(int);
}

namespace orc {

// ---------------------------------------------------------------- helpers
double fro_norm(const Mat& a) {
    double s = 0.0;
    for (double x : a.v) s += x * x;
    return std::sqrt(s);
}
static double sq_norm(const double* x, std::int64_t n) {
    double s = 0.0;
    for (std::int64_t i = 0; i < n; ++i) s += x[i] * x[i];
    return s;
}
bool all_finite(const double* x, std::int64_t n) {
    for (std::int64_t i = 0; i < n; ++i)
        if (!std::isfinite(x[i])) return false;
    return true;
}
bool all_finite(const Mat& a) { return all_finite(a.data(), a.size()); }
Mat transpose(const Mat& a) {
    Mat t(a.c, a.r);
    for (std::int64_t j = 0; j < a.c; ++j)
        for (std::int64_t i = 0; i < a.r; ++i) t(j, i) = a(i, j);
    return t;
}
void set_threads(int n) { scipy_openblas_set_num_threads(n); }

Mat matmul(const Mat& a, const Mat& b, bool ta, bool tb) {
    const std::int64_t m = ta ? a.c : a.r, ka = ta ? a.r : a.c;
    const std::int64_t kb = tb ? b.c : b.r, n = tb ? b.r : b.c;
    if (ka != kb) throw InvalidInput("matmul: inner dimension mismatch");
    Mat c(m, n);
    if (m == 0 || n == 0) return c;
    if (ka == 0) return c;
    const int M = (int)m, N = (int)n, K = (int)ka;
    const int lda = std::max<int>(1, (int)a.r), ldb = std::max<int>(1, (int)b.r),
              ldc = std::max<int>(1, M);
    const double one = 1.0, zero = 0.0;
    scipy_dgemm_(ta ? "T" : "N", tb ? "T" : "N", &M, &N, &K, &one, a.data(), &lda, b.data(), &ldb,
                 &zero, c.data(), &ldc, 1, 1);
    return c;
}
static void gemv(bool trans, const Mat& a, const double* x, double* y) {
    const int M = (int)a.r, N = (int)a.c, lda = std::max<int>(1, M), inc = 1;
    const double one = 1.0, zero = 0.0;
    scipy_dgemv_(trans ? "T" : "N", &M, &N, &one, a.data(), &lda, x, &inc, &zero, y, &inc, 1);
}

// ---------------------------------------------------------------- linalg
// reference linalg.cpp:17-26 (largest-magnitude entry of each column made
// positive; first index on ties, like Eigen's maxCoeff)
static void fix_column_signs(Mat& m, Mat* paired_rows = nullptr) {
    for (std::int64_t j = 0; j < m.c; ++j) {
        std::int64_t at = 0;
        double best = -1.0;
        for (std::int64_t i = 0; i < m.r; ++i) {
            const double v = std::fabs(m(i, j));
            if (v > best) { best = v; at = i; }
        }
        if (m.r > 0 && m(at, j) < 0.0) {
            for (std::int64_t i = 0; i < m.r; ++i) m(i, j) = -m(i, j);
            if (paired_rows)
                for (std::int64_t c = 0; c < paired_rows->c; ++c)
                    (*paired_rows)(j, c) = -(*paired_rows)(j, c);
        }
    }
}

void check_finite(const Mat& a, const char* who) {
    if (!all_finite(a)) throw InvalidInput(std::string(who) + ": non-finite entry");
}

// reference linalg.cpp:48-58 (BDCSVD thin -> dgesdd 'S')
SvdResult svd(const Mat& a) {
    if (a.size() == 0) throw InvalidInput("svd: empty input");
    check_finite(a, "svd");
    const int m = (int)a.r, n = (int)a.c, k = std::min(m, n);
    Mat w = a;
    SvdResult out;
    out.sigma.assign(k, 0.0);
    out.u = Mat(m, k);
    out.vt = Mat(k, n);
    std::vector<int> iwork(8 * (size_t)k);
    int lwork = -1, info = 0;
    double wq = 0.0;
    const int lda = std::max(1, m), ldu = std::max(1, m), ldvt = std::max(1, k);
    scipy_dgesdd_("S", &m, &n, w.data(), &lda, out.sigma.data(), out.u.data(), &ldu,
                  out.vt.data(), &ldvt, &wq, &lwork, iwork.data(), &info, 1);
    lwork = (int)wq + 1;
    std::vector<double> work(lwork);
    scipy_dgesdd_("S", &m, &n, w.data(), &lda, out.sigma.data(), out.u.data(), &ldu,
                  out.vt.data(), &ldvt, work.data(), &lwork, iwork.data(), &info, 1);
    if (info != 0) throw std::runtime_error("svd: dgesdd failed");
    fix_column_signs(out.u, &out.vt);
    return out;
}

// reference linalg.cpp:60-77 (eigh of (B+B^T)/2, descending, sign-fixed)
EighResult eigh(const Mat& b) {
    if (b.size() == 0) throw InvalidInput("eigh: empty input");
    if (b.r != b.c) throw InvalidInput("eigh: input not square");
    check_finite(b, "eigh");
    const int n = (int)b.r;
    Mat sym(n, n);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) sym(i, j) = 0.5 * (b(i, j) + b(j, i));
    std::vector<double> w(n);
    int lwork = -1, liwork = -1, info = 0, iwq = 0;
    double wq = 0.0;
    scipy_dsyevd_("V", "L", &n, sym.data(), &n, w.data(), &wq, &lwork, &iwq, &liwork, &info, 1,
                  1);
    lwork = (int)wq + 1;
    liwork = iwq + 1;
    std::vector<double> work(lwork);
    std::vector<int> iwork(liwork);
    scipy_dsyevd_("V", "L", &n, sym.data(), &n, w.data(), work.data(), &lwork, iwork.data(),
                  &liwork, &info, 1, 1);
    if (info != 0) throw std::runtime_error("eigh: dsyevd failed");
    EighResult out;
    out.lambda.assign(n, 0.0);
    out.v = Mat(n, n);
    for (int i = 0; i < n; ++i) {
        out.lambda[i] = w[n - 1 - i];
        std::memcpy(&out.v(0, i), &sym(0, n - 1 - i), sizeof(double) * n);
    }
    fix_column_signs(out.v);
    return out;
}

// Householder thin Q (rows >= cols): dgeqrf + dorgqr; returns (Q, packed QR)
static void householder_qr(const Mat& a, Mat& q, Mat* r) {
    const int m = (int)a.r, n = (int)a.c, k = std::min(m, n);
    Mat f = a;
    std::vector<double> tau(std::max(1, k));
    int lwork = -1, info = 0;
    double wq = 0.0;
    const int lda = std::max(1, m);
    scipy_dgeqrf_(&m, &n, f.data(), &lda, tau.data(), &wq, &lwork, &info);
    lwork = std::max(1, (int)wq);
    std::vector<double> work(lwork);
    scipy_dgeqrf_(&m, &n, f.data(), &lda, tau.data(), work.data(), &lwork, &info);
    if (r) {
        *r = Mat(k, n);
        for (int j = 0; j < n; ++j)
            for (int i = 0; i <= std::min(j, k - 1); ++i) (*r)(i, j) = f(i, j);
    }
    q = Mat(m, k);
    for (int j = 0; j < k; ++j) std::memcpy(&q(0, j), &f(0, j), sizeof(double) * m);
    lwork = -1;
    scipy_dorgqr_(&m, &k, &k, q.data(), &lda, tau.data(), &wq, &lwork, &info);
    lwork = std::max(1, (int)wq);
    work.assign(lwork, 0.0);
    scipy_dorgqr_(&m, &k, &k, q.data(), &lda, tau.data(), work.data(), &lwork, &info);
    if (info != 0) throw std::runtime_error("qr: dorgqr failed");
}

// reference linalg.cpp:29-33 (no sign fix)
Mat orthonormalize(const Mat& g) {
    Mat q;
    householder_qr(g, q, nullptr);
    return q;
}

// reference linalg.cpp:79-94 (nonnegative diag(R))
std::pair<Mat, Mat> qr(const Mat& a) {
    if (a.size() == 0) throw InvalidInput("qr: empty input");
    if (a.r < a.c) throw InvalidInput("qr: rows < cols (pad or transpose first)");
    check_finite(a, "qr");
    Mat q, r;
    householder_qr(a, q, &r);
    for (std::int64_t i = 0; i < r.r; ++i) {
        if (r(i, i) < 0.0) {
            for (std::int64_t j = 0; j < r.c; ++j) r(i, j) = -r(i, j);
            for (std::int64_t j = 0; j < q.r; ++j) q(j, i) = -q(j, i);
        }
    }
    return {std::move(q), std::move(r)};
}

// reference linalg.cpp:35-40 (row-major fill)
static Mat gaussian_matrix(std::int64_t rows, std::int64_t cols, RngState& rng) {
    Mat g(rows, cols);
    for (std::int64_t i = 0; i < rows; ++i)
        for (std::int64_t j = 0; j < cols; ++j) g(i, j) = rng.gaussian();
    return g;
}

// reference linalg.cpp:96-121
std::pair<double, Vec> power_iteration(const Mat& a, int k, RngState rng) {
    if (k < 1) throw InvalidInput("power_iteration: k must be >= 1");
    if (a.size() == 0) throw InvalidInput("power_iteration: empty input");
    check_finite(a, "power_iteration");
    const std::int64_t n = a.c;
    if (fro_norm(a) == 0.0) {
        Vec e1(n, 0.0);
        e1[0] = 1.0;
        return {0.0, e1};
    }
    Vec x(n), ax(a.r), y(n);
    for (std::int64_t i = 0; i < n; ++i) x[i] = rng.gaussian();
    {
        const double nx = std::sqrt(sq_norm(x.data(), n));
        if (nx > 0.0)
            for (double& v : x) v /= nx;
    }
    for (int it = 0; it < k; ++it) {
        gemv(false, a, x.data(), ax.data());
        gemv(true, a, ax.data(), y.data());
        const double nrm = std::sqrt(sq_norm(y.data(), n));
        if (nrm < 1e-300) {
            Vec e1(n, 0.0);
            e1[0] = 1.0;
            return {0.0, e1};
        }
        for (std::int64_t i = 0; i < n; ++i) x[i] = y[i] / nrm;
    }
    gemv(false, a, x.data(), ax.data());
    return {sq_norm(ax.data(), a.r), x};
}

// reference linalg.cpp:123-152
SimulIterResult simul_iter(const Mat& a, int k, double eps_si, RngState rng) {
    if (a.size() == 0) throw InvalidInput("simul_iter: empty input");
    if (k < 1 || k > std::min(a.r, a.c)) throw InvalidInput("simul_iter: k out of range");
    if (!(eps_si > 0.0 && eps_si < 1.0)) throw InvalidInput("simul_iter: eps_si out of (0,1)");
    check_finite(a, "simul_iter");
    const std::int64_t d = a.r;
    SimulIterResult out;
    if (fro_norm(a) == 0.0) {
        out.z = Mat::identity(d, k);
        out.sigma_hat.assign(k, 0.0);
        return out;
    }
    const int q = static_cast<int>(std::ceil(
        kSimulIterQConstant * std::log2(static_cast<double>(std::max<std::int64_t>(d, 2))) /
        eps_si));
    Mat pi = gaussian_matrix(a.c, k, rng);
    Mat g = orthonormalize(matmul(a, pi));
    for (int it = 0; it < q; ++it) g = orthonormalize(matmul(a, matmul(a, g, true, false)));
    const Mat w = matmul(a, g, true, false);
    const EighResult m = eigh(matmul(w, w, true, false));
    out.sigma_hat.assign(k, 0.0);
    for (int i = 0; i < k; ++i) out.sigma_hat[i] = std::sqrt(std::max(m.lambda[i], 0.0));
    out.z = matmul(g, m.v);
    fix_column_signs(out.z);
    return out;
}

// reference linalg.cpp:154-159
double spectral_norm_sym(const Mat& s) {
    if (s.size() == 0) return 0.0;
    const int n = (int)s.r;
    Mat sym(n, n);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) sym(i, j) = 0.5 * (s(i, j) + s(j, i));
    std::vector<double> w(n);
    int lwork = -1, liwork = -1, info = 0, iwq = 0;
    double wq = 0.0;
    scipy_dsyevd_("N", "L", &n, sym.data(), &n, w.data(), &wq, &lwork, &iwq, &liwork, &info, 1,
                  1);
    lwork = (int)wq + 1;
    liwork = iwq + 1;
    std::vector<double> work(lwork);
    std::vector<int> iwork(liwork);
    scipy_dsyevd_("N", "L", &n, sym.data(), &n, w.data(), work.data(), &lwork, iwork.data(),
                  &liwork, &info, 1, 1);
    double best = 0.0;
    for (double x : w) best = std::max(best, std::fabs(x));
    return best;
}

// reference linalg.cpp:161-165
double spectral_norm(const Mat& a) {
    if (a.size() == 0 || fro_norm(a) == 0.0) return 0.0;
    const int m = (int)a.r, n = (int)a.c, k = std::min(m, n);
    Mat w = a;
    std::vector<double> s(k);
    std::vector<int> iwork(8 * (size_t)k);
    int lwork = -1, info = 0, one = 1;
    double wq = 0.0, dummy = 0.0;
    scipy_dgesdd_("N", &m, &n, w.data(), &m, s.data(), &dummy, &one, &dummy, &one, &wq, &lwork,
                  iwork.data(), &info, 1);
    lwork = (int)wq + 1;
    std::vector<double> work(lwork);
    scipy_dgesdd_("N", &m, &n, w.data(), &m, s.data(), &dummy, &one, &dummy, &one, work.data(),
                  &lwork, iwork.data(), &info, 1);
    return s[0];
}

// ---------------------------------------------------------------- fd
// reference fd.cpp:13-29
Mat fd_reduce(const Mat& b, int ell) {
    if (ell < 1) throw InvalidInput("fd_reduce: ell must be >= 1");
    if (b.r != 2 * (std::int64_t)ell)
        throw InvalidInput("fd_reduce: buffer must have exactly 2*ell rows");
    check_finite(b, "fd_reduce");
    if (fro_norm(b) == 0.0) return Mat(b.r, b.c);
    const SvdResult fac = svd(b);
    const std::int64_t nsv = (std::int64_t)fac.sigma.size();
    const double cut = (ell <= nsv) ? fac.sigma[ell - 1] * fac.sigma[ell - 1] : 0.0;
    Mat out(b.r, b.c);
    for (std::int64_t i = 0; i < nsv; ++i) {
        const double s2 = fac.sigma[i] * fac.sigma[i] - cut;
        if (s2 > 0.0) {
            const double w = std::sqrt(s2);
            for (std::int64_t j = 0; j < b.c; ++j) out(i, j) = w * fac.vt(i, j);
        }
    }
    return out;
}

// reference fd.cpp:56-86
std::pair<Mat, Mat> cod_reduce(const Mat& a, const Mat& b, int ell) {
    if (ell < 1) throw InvalidInput("cod_reduce: ell must be >= 1");
    if (a.c != b.c) throw InvalidInput("cod_reduce: column-count mismatch");
    check_finite(a, "cod_reduce");
    check_finite(b, "cod_reduce");
    if (fro_norm(a) == 0.0 || fro_norm(b) == 0.0) return {Mat(a.r, a.c), Mat(b.r, b.c)};
    auto thin_qr = [](const Mat& m) {
        Mat q;
        householder_qr(m, q, nullptr);
        Mat r = matmul(q, m, true, false);
        return std::make_pair(std::move(q), std::move(r));
    };
    const auto [qa, ra] = thin_qr(a);
    const auto [qb, rb] = thin_qr(b);
    const SvdResult fac = svd(matmul(ra, rb, false, true));
    const std::int64_t nsv = (std::int64_t)fac.sigma.size();
    const double cut = (ell <= nsv) ? fac.sigma[ell - 1] : 0.0;
    Vec w(nsv, 0.0);
    for (std::int64_t i = 0; i < nsv; ++i) w[i] = std::sqrt(std::max(fac.sigma[i] - cut, 0.0));
    Mat uw = fac.u;
    for (std::int64_t j = 0; j < nsv; ++j)
        for (std::int64_t i = 0; i < uw.r; ++i) uw(i, j) *= w[j];
    Mat vw(fac.vt.c, nsv);
    for (std::int64_t j = 0; j < nsv; ++j)
        for (std::int64_t i = 0; i < vw.r; ++i) vw(i, j) = fac.vt(j, i) * w[j];
    const Mat ap = matmul(qa, uw), bp = matmul(qb, vw);
    Mat aprime(a.r, a.c), bprime(b.r, b.c);
    for (std::int64_t j = 0; j < nsv; ++j) {
        std::memcpy(&aprime(0, j), ap.data() + j * a.r, sizeof(double) * a.r);
        std::memcpy(&bprime(0, j), bp.data() + j * b.r, sizeof(double) * b.r);
    }
    return {std::move(aprime), std::move(bprime)};
}

// ---------------------------------------------------------------- sketch
// reference sketch.cpp:16-18
int power_iter_count(int d) {
    return static_cast<int>(std::ceil(std::log2(static_cast<double>(std::max(d, 2))))) + 1;
}

// reference sketch.cpp:22-31
AeroState::AeroState(int d, double eps, double theta, RngState rng, double delta)
    : d_(d), eps_(eps), ell_(0), theta_(theta), eps_si_(0.4), ct_(Mat(d > 0 ? d : 0, 0)),
      clock_(0), last_dump_t_(0), rng_(rng) {
    if (d < 1) throw InvalidInput("AeroState: d must be >= 1");
    if (!(eps > 0.0 && eps <= 1.0)) throw InvalidInput("AeroState: eps out of (0,1]");
    if (theta < 0.0) throw InvalidInput("AeroState: theta must be >= 0");
    if (delta != 0.0 && !(delta > 0.0 && delta < 1.0)) throw InvalidInput("AeroState: delta out of (0, 1)");
    delta_ = delta;
    ell_ = static_cast<int>(std::ceil(2.0 / eps));
}

// reference sketch.cpp:45-48
void AeroState::update_amplified(const double* a, std::int64_t i) {
    if (delta_ == 0.0) throw InvalidInput("AeroState: amplification requested without delta");
    update_impl(a, i, true);
}

void AeroState::import_state(const double* rows_rm, std::int64_t r, std::uint64_t forks, std::int64_t clock,
                             std::int64_t last_dump_t, double theta) {
    if (r < 0 || r > 2 * (std::int64_t)ell_) throw InvalidInput("import_state: rows out of range");
    ct_ = Mat(d_, r);
    std::copy(rows_rm, rows_rm + r * d_, ct_.v.begin());  // C row-major == C^T column-major
    snaps_.clear();
    rng_.set_forks(forks);
    clock_ = clock;
    last_dump_t_ = last_dump_t;
    theta_ = theta;
}

void AeroState::set_theta(double theta) {
    if (theta < 0.0) throw InvalidInput("AeroState: theta must be >= 0");
    theta_ = theta;
}

// reference sketch.cpp:50-80: plain simul_iter, or r candidates at eps_si=0.2
// whose residual C'^T - z z^T C'^T is scored by the max of s power
// iterations; the smallest score wins (the first on ties)
SimulIterResult AeroState::factorize(const Mat& at, int k, bool amplified) {
    if (!amplified) {
        ++stats_.simul_calls;
        return simul_iter(at, k, eps_si_, rng_.fork());
    }
    const double delta = delta_;
    const int r = static_cast<int>(std::ceil(std::log(2.0 / delta) / std::log(100.0)));
    if (r <= 1) {
        ++stats_.simul_calls;
        return simul_iter(at, k, 0.2, rng_.fork());
    }
    const int s = static_cast<int>(std::ceil(2.0 * std::log(2.0 / delta) / std::log(3.0)));
    const int kp = power_iter_count(d_);
    SimulIterResult best;
    double best_cost = 0.0;
    for (int h = 0; h < r; ++h) {
        ++stats_.simul_calls;
        SimulIterResult cand = simul_iter(at, k, 0.2, rng_.fork());
        // at_res = at - z (z^T at)   (d x r)
        const Mat zt_at = matmul(cand.z, at, true, false);   // k x r
        const Mat proj = matmul(cand.z, zt_at, false, false);  // d x r
        Mat at_res = at;
        for (std::int64_t q = 0; q < at_res.size(); ++q) at_res.v[q] -= proj.v[q];
        double cost = 0.0;
        for (int rep = 0; rep < s; ++rep) cost = std::max(cost, power_iteration(at_res, kp, rng_.fork()).first);
        if (h == 0 || cost < best_cost) {
            best_cost = cost;
            best = std::move(cand);
        }
    }
    return best;
}

// reference sketch.cpp:82-141. The buffer is held as C'^T (d x r, column-major)
// which is C' in row-major order; every product below is the reference's.
void AeroState::update_impl(const double* a, std::int64_t i, bool amplified) {
    if (!all_finite(a, d_)) throw InvalidInput("AeroState: non-finite row");
    if (i <= clock_) throw InvalidInput("AeroState: timestamp regression");
    stats_ = UpdateStats{};
    ev_ = Event{};
    ev_.t = i;
    ev_.theta = theta_;
    ev_.forks_before = (std::int64_t)rng_.forks();

    // insert into the buffer; reduce when full (sketch.cpp:89-95)
    Mat cp(d_, ct_.c + 1);
    std::memcpy(cp.data(), ct_.data(), sizeof(double) * ct_.size());
    std::memcpy(&cp(0, ct_.c), a, sizeof(double) * d_);
    if (cp.c == 2 * (std::int64_t)ell_) {
        const Mat red = fd_reduce(transpose(cp), ell_);  // 2ell x d
        const std::int64_t keep = std::max(ell_ - 1, 1);
        Mat nc(d_, keep);
        for (std::int64_t r = 0; r < keep; ++r)
            for (std::int64_t j = 0; j < d_; ++j) nc(j, r) = red(r, j);
        cp = std::move(nc);
        stats_.reduced = true;
    }

    // gate (sketch.cpp:97-106)
    const int kp = power_iter_count(d_);
    const double sigma1_sq = power_iteration(cp, kp, rng_.fork()).first;
    stats_.gate_fired = sigma1_sq >= 0.5 * theta_;
    ev_.sigma1_sq = sigma1_sq;

    if (stats_.gate_fired) {
        // doubling search (sketch.cpp:108-139)
        const int kmax = (int)std::min<std::int64_t>({(std::int64_t)ell_, (std::int64_t)d_, cp.c});
        int k = std::min(2, kmax);
        while (true) {
            ++stats_.doubling_steps;
            const SimulIterResult fac = factorize(cp, k, amplified);
            const double tail = fac.sigma_hat[k - 1] * fac.sigma_hat[k - 1];
            ev_.k_last = k;
            ev_.tail_sq = tail;
            if (tail < theta_ || k == kmax) {
                int xi = 0;
                for (int j = 0; j < k; ++j) {
                    if (fac.sigma_hat[j] * fac.sigma_hat[j] >= theta_) xi = j + 1;
                    else break;
                }
                ev_.xi = xi;
                if (xi >= 1) {
                    Snapshot snap;
                    snap.z = Mat(d_, xi);
                    std::memcpy(snap.z.data(), fac.z.data(), sizeof(double) * d_ * xi);
                    const Mat cz = matmul(cp, snap.z, true, false);  // C' z (r x xi)
                    snap.m = matmul(cz, cp, true, true);            // (C'z)^T C' (xi x d)
                    snap.s = last_dump_t_ + 1;
                    snap.t = i;
                    snap.theta = theta_;
                    last_dump_t_ = i;
                    const Mat zczt = matmul(snap.z, cz, false, true);  // z (C'z)^T (d x r)
                    for (std::int64_t q = 0; q < cp.size(); ++q) cp.v[q] -= zczt.v[q];
                    snaps_.push_back(std::move(snap));
                    stats_.dumped = true;
                }
                break;
            }
            k = std::min(2 * k, kmax);
        }
    }
    ct_ = std::move(cp);
    clock_ = i;
    ev_.forks_after = (std::int64_t)rng_.forks();
    ev_.rows_after = (std::int32_t)ct_.c;
    ev_.reduced = stats_.reduced;
    ev_.gate_fired = stats_.gate_fired;
    ev_.dumped = stats_.dumped;
    ev_.doubling_steps = stats_.doubling_steps;
    ev_.simul_calls = stats_.simul_calls;
}

// reference sketch.cpp:162-165
Mat restore_contribution(const Snapshot& snap) {
    Mat b(snap.z.r, snap.z.r);
    add_restore_contribution(b, snap, 1.0);
    return b;
}
void add_restore_contribution(Mat& b, const Snapshot& snap, double sign) {
    const Mat zm = matmul(snap.z, snap.m);           // d x d
    const Mat mz = matmul(snap.m, snap.z);           // xi x xi
    const Mat zmz = matmul(matmul(snap.z, mz), snap.z, false, true);  // d x d
    const std::int64_t d = snap.z.r;
    for (std::int64_t j = 0; j < d; ++j)
        for (std::int64_t i = 0; i < d; ++i)
            b(i, j) += sign * (zm(i, j) + zm(j, i) - zmz(i, j));
}

// reference sketch.cpp:143-160 (before the final shrink)
Mat AeroState::query_gram(std::int64_t lb, std::int64_t ub) const {
    if (lb >= ub) throw InvalidInput("AeroState: query needs lb < ub");
    if (ub > clock_) throw InvalidInput("AeroState: query beyond clock");
    Mat b(d_, d_);
    if (ub == clock_ && ct_.c > 0) b = matmul(ct_, ct_, false, true);
    auto first = std::lower_bound(snaps_.begin(), snaps_.end(), lb,
                                  [](const Snapshot& s, std::int64_t v) { return s.t <= v; });
    for (auto it = first; it != snaps_.end() && it->t <= ub; ++it)
        add_restore_contribution(b, *it, 1.0);
    return b;
}
Mat AeroState::query(std::int64_t lb, std::int64_t ub) const {
    return shrink_to_sketch(query_gram(lb, ub), ell_);
}

// reference sketch.cpp:167-178
Mat shrink_to_sketch(const Mat& b, int ell) {
    const EighResult fac = eigh(b);
    const std::int64_t d = b.r;
    Vec lam = fac.lambda;
    for (double& x : lam) x = std::max(x, 0.0);
    const double cut = (ell <= d) ? lam[ell - 1] : 0.0;
    Mat out(ell, d);
    for (std::int64_t i = 0; i < std::min<std::int64_t>(ell, d); ++i) {
        const double w = lam[i] - cut;
        if (w > 0.0) {
            const double s = std::sqrt(w);
            for (std::int64_t j = 0; j < d; ++j) out(i, j) = s * fac.v(j, i);
        }
    }
    return out;
}

// ---------------------------------------------------------------- attp
// reference attp.hpp:21-32
void AttpState::update(const double* a, std::int64_t i) {
    fro_mass_ += sq_norm(a, inner_.d());
    inner_.set_theta(inner_.eps() * fro_mass_);
    if (inner_.delta() != 0.0) inner_.update_amplified(a, i);  // attp.hpp:24
    else inner_.update(a, i);
}
Mat AttpState::query(std::int64_t t) const {
    if (t < 1 || t > inner_.clock()) throw InvalidInput("AttpState: t out of range");
    return inner_.query(0, t);
}

// ---------------------------------------------------------------- sliding window
// reference sliding_window.cpp:15-30
MlState::MlState(int d, std::int64_t n, double r_max, double eps, RngState rng, double delta)
    : d_(d), n_(n), r_max_(r_max), eps_(eps), ell_(0), cap_(0), clock_(0), window_mass_(0.0),
      norm_warnings_(0) {
    if (n < 1) throw InvalidInput("MlState: window size must be >= 1");
    if (r_max < 1.0) throw InvalidInput("MlState: r_max must be >= 1 (squared norms in [1, R])");
    if (!(eps > 0.0 && eps <= 1.0)) throw InvalidInput("MlState: eps out of (0,1]");
    ell_ = static_cast<int>(std::ceil(2.0 / eps));
    cap_ = static_cast<std::int64_t>(std::ceil(8.0 / eps));
    const int big_l = static_cast<int>(std::ceil(std::log2(std::max(r_max, 2.0))));
    for (int j = 0; j < std::max(big_l, 1); ++j) {
        const double theta_j = std::pow(2.0, j) * eps * static_cast<double>(n);
        levels_.emplace_back(d, eps, theta_j, rng.fork(), delta);
        heavy_.emplace_back();
    }
}
// reference sliding_window.cpp:32-65
std::int64_t MlState::combined_len(int j) const {
    return (std::int64_t)(levels_[j].snaps().size() + heavy_[j].size());
}
std::int64_t MlState::front_t(int j) const {
    std::int64_t t = std::numeric_limits<std::int64_t>::max();
    if (!levels_[j].snaps().empty()) t = std::min(t, levels_[j].snaps().front().t);
    if (!heavy_[j].empty()) t = std::min(t, heavy_[j].front().t);
    return t;
}
std::int64_t MlState::front_s(int j) const {
    const auto& snaps = levels_[j].snaps();
    const auto& hv = heavy_[j];
    if (snaps.empty() && hv.empty()) return std::numeric_limits<std::int64_t>::max();
    if (snaps.empty()) return hv.front().s;
    if (hv.empty()) return snaps.front().s;
    return (snaps.front().t <= hv.front().t) ? snaps.front().s : hv.front().s;
}
std::int64_t MlState::tail_t(int j) const {
    std::int64_t t = 0;
    if (!levels_[j].snaps().empty()) t = std::max(t, levels_[j].snaps().back().t);
    if (!heavy_[j].empty()) t = std::max(t, heavy_[j].back().t);
    return t;
}
void MlState::pop_front(int j) {
    auto& snaps = levels_[j].snaps();
    auto& hv = heavy_[j];
    if (snaps.empty() && hv.empty()) return;
    if (hv.empty() || (!snaps.empty() && snaps.front().t <= hv.front().t)) snaps.pop_front();
    else hv.pop_front();
}
// reference sliding_window.cpp:67-100
void MlState::update(const double* a, std::int64_t i) {
    if (!all_finite(a, d_)) throw InvalidInput("MlState: non-finite row");
    if (i <= clock_) throw InvalidInput("MlState: timestamp regression");
    const double nsq = sq_norm(a, d_);
    if (nsq < 1.0 || nsq > r_max_) ++norm_warnings_;
    ring_.push_back(nsq);
    window_mass_ += nsq;
    while ((std::int64_t)ring_.size() > n_) {
        window_mass_ -= ring_.front();
        ring_.pop_front();
    }
    for (int j = 0; j < levels(); ++j) {
        while (combined_len(j) > 0 && front_t(j) <= i - n_) pop_front(j);
        if (nsq >= levels_[j].theta()) {
            heavy_[j].push_back(HeavyRow{Vec(a, a + d_), tail_t(j) + 1, i});
        } else {
            if (levels_[j].delta() != 0.0) levels_[j].update_amplified(a, i);  // sliding_window.cpp:90-91
            else levels_[j].update(a, i);
        }
        while (combined_len(j) > cap_) pop_front(j);
    }
    clock_ = i;
}
// reference sliding_window.cpp:102-146
MlQueryResult MlState::query() const {
    if (clock_ == 0) throw InvalidInput("MlState: query before any update");
    const std::int64_t t_now = clock_;
    const std::int64_t wstart = t_now - n_;
    const std::int64_t head = std::max<std::int64_t>(wstart + 1, 1);
    MlQueryResult out;
    int pick = -1;
    for (int j = 0; j < levels(); ++j) {
        if (combined_len(j) == 0) continue;
        const std::int64_t s0 = front_s(j);
        if (s0 >= 1 && s0 <= head) { pick = j; break; }
    }
    if (pick < 0) {
        out.fallback = true;
        double guess = 0.0;
        if (window_mass_ > 0.0) guess = std::floor(std::log2(window_mass_ / (double)n_));
        pick = (int)std::clamp(guess, 0.0, (double)(levels() - 1));
    }
    out.level = pick;
    const AeroState& lv = levels_[pick];
    const std::int64_t lb = std::max<std::int64_t>(wstart, 0);
    Mat base(ell_, d_);
    if (lv.clock() > lb) base = lv.query(lb, lv.clock());
    for (const Snapshot& s : lv.snaps())
        if (s.t > wstart && s.t <= t_now) out.xi_sum += s.z.c;
    std::vector<const HeavyRow*> hv;
    for (const HeavyRow& h : heavy_[pick])
        if (h.t > wstart && h.t <= t_now) hv.push_back(&h);
    out.heavy_used = (int)hv.size();
    Mat stack(base.r + (std::int64_t)hv.size(), d_);
    for (std::int64_t r = 0; r < base.r; ++r)
        for (std::int64_t j = 0; j < d_; ++j) stack(r, j) = base(r, j);
    for (std::size_t r = 0; r < hv.size(); ++r)
        for (std::int64_t j = 0; j < d_; ++j) stack(base.r + (std::int64_t)r, j) = hv[r]->row[j];
    out.sketch = shrink_to_sketch(matmul(stack, stack, true, false), ell_);
    return out;
}
std::int64_t MlState::stored_floats() const {
    std::int64_t total = (std::int64_t)ring_.size();
    for (int j = 0; j < levels(); ++j) {
        total += levels_[j].residual_t().size();
        for (const Snapshot& s : levels_[j].snaps()) total += s.z.size() + s.m.size();
        total += (std::int64_t)heavy_[j].size() * d_;
    }
    return total;
}

// ---------------------------------------------------------------- distributed
// reference distributed.cpp:16-24
SiteState::SiteState(int id, int d, double eps, int m, RngState rng,
                     std::optional<std::int64_t> window)
    : id_(id), m_(m), eps_(eps), window_(window), inner_(d, eps, 0.0, rng), f_local_(0.0),
      f_self_sent_(0.0), f_hat_known_(0.0), w_local_(0.0), w_last_sent_(0.0) {
    if (id < 0) throw InvalidInput("SiteState: negative site id");
    if (m < 1) throw InvalidInput("SiteState: site count must be >= 1");
}
void SiteState::on_broadcast(double f_hat) {
    f_hat_known_ = window_ ? f_hat : std::max(f_hat_known_, f_hat);
}
// reference distributed.cpp:31-98
void SiteState::update(const double* a, std::int64_t i, std::vector<Message>& outbox) {
    const double nsq = sq_norm(a, inner_.d());
    if (window_) {
        ring_.push_back(nsq);
        w_local_ += nsq;
        while ((std::int64_t)ring_.size() > *window_) {
            w_local_ -= ring_.front();
            ring_.pop_front();
        }
        const double delta = w_local_ - w_last_sent_;
        if (std::abs(delta) >= (eps_ / m_) * f_hat_known_) {
            Message msg;
            msg.kind = MsgKind::FroMass;
            msg.from = id_;
            msg.f = delta;
            outbox.push_back(std::move(msg));
            w_last_sent_ = w_local_;
        }
        inner_.set_theta(eps_ * w_local_);
    } else {
        f_local_ += nsq;
        if (f_local_ >= (eps_ / m_) * f_hat_known_) {
            Message msg;
            msg.kind = MsgKind::FroMass;
            msg.from = id_;
            msg.f = f_local_;
            outbox.push_back(std::move(msg));
            f_self_sent_ += f_local_;
            f_local_ = 0.0;
        }
        inner_.set_theta(eps_ * std::max(f_hat_known_, f_self_sent_ + f_local_));
    }
    inner_.update(a, i);
    auto& q = const_cast<AeroState&>(inner_).snaps();
    while (!q.empty()) {
        Snapshot snap = std::move(q.front());
        q.pop_front();
        Message msg;
        msg.kind = MsgKind::SnapshotUpdate;
        msg.from = id_;
        msg.z = std::move(snap.z);
        msg.m = std::move(snap.m);
        msg.t = snap.t;
        outbox.push_back(std::move(msg));
        if (window_) sent_snap_times_.push_back(snap.t);
    }
    if (window_) {
        while (!sent_snap_times_.empty() && sent_snap_times_.front() <= i - *window_) {
            Message msg;
            msg.kind = MsgKind::Expire;
            msg.from = id_;
            msg.t = sent_snap_times_.front();
            sent_snap_times_.pop_front();
            outbox.push_back(std::move(msg));
        }
    }
}
// reference distributed.cpp:100-105
CoordinatorState::CoordinatorState(int d, int m, bool window_mode)
    : d_(d), m_(m), window_mode_(window_mode), b_(Mat(d > 0 ? d : 0, d > 0 ? d : 0)), f_hat_(0.0),
      msg_count_(0), broadcasts_(0) {
    if (d < 1) throw InvalidInput("CoordinatorState: d must be >= 1");
    if (m < 1) throw InvalidInput("CoordinatorState: site count must be >= 1");
}
// reference distributed.cpp:107-149
std::optional<Message> CoordinatorState::receive(const Message& msg) {
    switch (msg.kind) {
        case MsgKind::FroMass: {
            if (!window_mode_ && !(msg.f >= 0.0)) throw ProtocolError("FroMass: negative mass");
            f_hat_ = std::max(f_hat_ + msg.f, 0.0);
            if (++msg_count_ >= m_) {
                msg_count_ = 0;
                ++broadcasts_;
                Message bc;
                bc.kind = MsgKind::FroBroadcast;
                bc.from = -1;
                bc.f = f_hat_;
                return bc;
            }
            return std::nullopt;
        }
        case MsgKind::SnapshotUpdate: {
            if (msg.z.c == 0 || msg.z.r != d_ || msg.m.r != msg.z.c || msg.m.c != d_)
                throw ProtocolError("SnapshotUpdate: inconsistent payload shapes");
            Snapshot s;
            s.z = msg.z;
            s.m = msg.m;
            Mat contrib = restore_contribution(s);
            for (std::int64_t q = 0; q < b_.size(); ++q) b_.v[q] += contrib.v[q];
            contributions_[{msg.from, msg.t}] = std::move(contrib);
            return std::nullopt;
        }
        case MsgKind::Expire: {
            if (!window_mode_) throw ProtocolError("Expire outside sliding-window mode");
            const auto it = contributions_.find({msg.from, msg.t});
            if (it == contributions_.end()) throw ProtocolError("Expire: unknown contribution");
            for (std::int64_t q = 0; q < b_.size(); ++q) b_.v[q] -= it->second.v[q];
            contributions_.erase(it);
            return std::nullopt;
        }
        case MsgKind::FroBroadcast: throw ProtocolError("coordinator received a broadcast");
    }
    throw ProtocolError("unknown message kind");
}

// ---------------------------------------------------------------- amm
// reference amm.cpp:22-25
Mat cod_restore_contribution(const CodSnapshot& s) {
    Mat out = matmul(s.z, s.zm);
    const Mat mh_ht = matmul(s.mh, s.h, false, true);
    const Mat z_zmh_ht = matmul(matmul(s.z, matmul(s.zm, s.h)), s.h, false, true);
    for (std::int64_t q = 0; q < out.size(); ++q) out.v[q] += mh_ht.v[q] - z_zmh_ht.v[q];
    return out;
}
// reference amm.cpp:27-36
CodState::CodState(int d_x, int d_y, double eps, double theta, std::int64_t n, RngState rng)
    : dx_(d_x), dy_(d_y), eps_(eps), ell_(0), theta_(theta), n_(n),
      a_(Mat(d_x > 0 ? d_x : 0, 0)), b_(Mat(d_y > 0 ? d_y : 0, 0)), clock_(0), last_dump_t_(0),
      rng_(rng) {
    if (d_x < 1 || d_y < 1) throw InvalidInput("CodState: dimensions must be >= 1");
    if (!(eps > 0.0 && eps <= 1.0)) throw InvalidInput("CodState: eps out of (0,1]");
    if (theta < 0.0) throw InvalidInput("CodState: theta must be >= 0");
    if (n < 1) throw InvalidInput("CodState: window size must be >= 1");
    ell_ = static_cast<int>(std::ceil(2.0 / eps));
}
// reference amm.cpp:38-41
void CodState::set_theta(double theta) {
    if (theta < 0.0) throw InvalidInput("CodState: theta must be >= 0");
    theta_ = theta;
}
static Mat append_col(const Mat& m, const double* x) {
    Mat out(m.r, m.c + 1);
    std::memcpy(out.data(), m.data(), sizeof(double) * m.size());
    std::memcpy(&out(0, m.c), x, sizeof(double) * m.r);
    return out;
}
static Mat left_cols(const Mat& m, std::int64_t k) {
    Mat out(m.r, k);
    std::memcpy(out.data(), m.data(), sizeof(double) * m.r * k);
    return out;
}
// reference amm.cpp:42-103
void CodState::update(const double* x, const double* y, std::int64_t i) {
    if (!all_finite(x, dx_) || !all_finite(y, dy_))
        throw InvalidInput("CodState: non-finite input");
    if (i <= clock_) throw InvalidInput("CodState: timestamp regression");
    ev_ = Event{};
    ev_.t = i;
    ev_.theta = theta_;
    ev_.forks_before = (std::int64_t)rng_.forks();
    while (!snaps_.empty() && snaps_.front().t + n_ <= i) snaps_.pop_front();
    a_ = append_col(a_, x);
    b_ = append_col(b_, y);
    if (a_.c == 2 * (std::int64_t)ell_) {
        auto [ap, bp] = cod_reduce(a_, b_, ell_);
        const std::int64_t keep = std::max(ell_ - 1, 1);
        a_ = left_cols(ap, keep);
        b_ = left_cols(bp, keep);
        ev_.reduced = 1;
    }
    const Mat p = matmul(a_, b_, false, true);
    const int kp = power_iter_count(ell_);
    const double sigma1 = std::sqrt(power_iteration(p, kp, rng_.fork()).first);
    ev_.sigma1_sq = sigma1 * sigma1;
    if (sigma1 < 0.5 * theta_) {
        clock_ = i;
        ev_.forks_after = (std::int64_t)rng_.forks();
        ev_.rows_after = (std::int32_t)a_.c;
        return;
    }
    ev_.gate_fired = 1;
    const int kmax = (int)std::min<std::int64_t>({(std::int64_t)ell_, (std::int64_t)dx_,
                                                  (std::int64_t)dy_, a_.c});
    int k = std::min(2, kmax);
    while (true) {
        ++ev_.doubling_steps;
        const SimulIterResult zfac = simul_iter(p, k, 0.4, rng_.fork());
        const SimulIterResult hfac = simul_iter(transpose(p), k, 0.4, rng_.fork());
        ev_.simul_calls += 2;
        ev_.k_last = k;
        ev_.tail_sq = zfac.sigma_hat[k - 1];
        if (zfac.sigma_hat[k - 1] < theta_ || k == kmax) {
            int xi = 0;
            for (int j = 0; j < k; ++j) {
                if (zfac.sigma_hat[j] >= theta_) xi = j + 1;
                else break;
            }
            ev_.xi = xi;
            if (xi >= 1) {
                CodSnapshot snap;
                snap.z = left_cols(zfac.z, xi);
                snap.h = left_cols(hfac.z, xi);
                snap.zm = matmul(snap.z, p, true, false);
                snap.mh = matmul(p, snap.h);
                snap.s = last_dump_t_ + 1;
                snap.t = i;
                last_dump_t_ = i;
                const Mat za = matmul(snap.z, matmul(snap.z, a_, true, false));
                const Mat hb = matmul(snap.h, matmul(snap.h, b_, true, false));
                for (std::int64_t q = 0; q < a_.size(); ++q) a_.v[q] -= za.v[q];
                for (std::int64_t q = 0; q < b_.size(); ++q) b_.v[q] -= hb.v[q];
                snaps_.push_back(std::move(snap));
                ev_.dumped = 1;
            }
            break;
        }
        k = std::min(2 * k, kmax);
    }
    clock_ = i;
    ev_.forks_after = (std::int64_t)rng_.forks();
    ev_.rows_after = (std::int32_t)a_.c;
}
// reference amm.cpp:105-122
Mat CodState::query_product() const {
    Mat p = matmul(a_, b_, false, true);
    for (const CodSnapshot& s : snaps_) {
        const Mat c = cod_restore_contribution(s);
        for (std::int64_t q = 0; q < p.size(); ++q) p.v[q] += c.v[q];
    }
    return p;
}
std::pair<Mat, Mat> CodState::query() const {
    const Mat p = query_product();
    Mat astar(dx_, ell_), bstar(dy_, ell_);
    if (fro_norm(p) > 0.0) {
        const SvdResult fac = svd(p);
        const std::int64_t nsv = (std::int64_t)fac.sigma.size();
        const double cut = (ell_ <= nsv) ? fac.sigma[ell_ - 1] : 0.0;
        for (std::int64_t j = 0; j < std::min<std::int64_t>(ell_, nsv); ++j) {
            const double w = std::sqrt(std::max(fac.sigma[j] - cut, 0.0));
            for (std::int64_t i = 0; i < dx_; ++i) astar(i, j) = w * fac.u(i, j);
            for (std::int64_t i = 0; i < dy_; ++i) bstar(i, j) = w * fac.vt(j, i);
        }
    }
    return {std::move(astar), std::move(bstar)};
}

// reference amm.cpp:131-138. Member order fixes the fork order: main_ takes
// the parameter's first fork, aux_ its second, rng_ keeps the parent.
AdaptiveState::AdaptiveState(int d_x, int d_y, double eps, double theta0, std::int64_t n,
                             RngState rng)
    : eps_(eps), theta0_(theta0), n_(n), level_(1),
      main_(d_x, d_y, eps, theta0, n, rng.fork()),
      aux_(d_x, d_y, eps, theta0, n, rng.fork()),
      rng_(rng) {
    if (theta0 <= 0.0) throw InvalidInput("AdaptiveState: theta0 must be > 0");
}
// reference amm.cpp:140-159
void AdaptiveState::update(const double* x, const double* y, std::int64_t i) {
    if (i > 1 && (i % n_) == 1) {  // window boundary: aux becomes main
        main_ = aux_;
        aux_ = CodState(main_.d_x(), main_.d_y(), eps_, main_.theta(), n_, rng_.fork());
    }
    main_.update(x, y, i);
    aux_.update(x, y, i);
    const double qlen = static_cast<double>(main_.snaps().size());
    if (qlen >= static_cast<double>(level_) / eps_) {
        ++level_;
        main_.set_theta(2.0 * main_.theta());
        aux_.set_theta(2.0 * aux_.theta());
    } else if (level_ > 1 && qlen <= static_cast<double>(level_ - 1) / eps_) {
        --level_;
        main_.set_theta(0.5 * main_.theta());
        aux_.set_theta(0.5 * aux_.theta());
    }
}

// ---------------------------------------------------------------- exact oracle
// reference oracle.hpp:28-53
OracleGram::OracleGram(int d, std::optional<std::int64_t> window, std::int64_t cap)
    : d_(d), window_(window), cap_(cap), capped_(false), g_(Mat(d, d)), mass_(0.0), rows_(0) {}
void OracleGram::add(const double* row, std::int64_t t) {
    if (capped_) return;
    ++rows_;
    for (int j = 0; j < d_; ++j)
        for (int i = 0; i < d_; ++i) g_(i, j) += row[i] * row[j];
    mass_ += sq_norm(row, d_);
    if (window_) {
        held_.push_back({t, Vec(row, row + d_)});
        while (!held_.empty() && held_.front().t + *window_ <= t) {
            const Vec& old = held_.front().row;
            for (int j = 0; j < d_; ++j)
                for (int i = 0; i < d_; ++i) g_(i, j) -= old[i] * old[j];
            mass_ -= sq_norm(old.data(), d_);
            held_.pop_front();
            --rows_;
        }
    }
    if (rows_ > cap_) capped_ = true;
}
double OracleGram::error(const Mat& sketch) const {
    if (capped_) throw OracleCapExceeded("oracle row cap exceeded");
    if (mass_ <= 0.0) return 0.0;
    const Mat btb = matmul(sketch, sketch, true, false);
    Mat diff = g_;
    for (std::int64_t q = 0; q < diff.size(); ++q) diff.v[q] -= btb.v[q];
    return spectral_norm_sym(diff) / mass_;
}
double OracleGram::error_gram(const Mat& gram_hat) const {
    if (capped_) throw OracleCapExceeded("oracle row cap exceeded");
    if (mass_ <= 0.0) return 0.0;
    Mat diff = g_;
    for (std::int64_t q = 0; q < diff.size(); ++q) diff.v[q] -= gram_hat.v[q];
    return spectral_norm_sym(diff) / mass_;
}

// ---------------------------------------------------------------- generators
Mat gen_basis(std::uint64_t seed, std::uint64_t basis_id, int d, int k) {
    RngState rng(seed, 0xB000000000000000ULL ^ basis_id);
    Mat g = gaussian_matrix(d, k, rng);
    const Mat q = qr(g).first;  // d x k, R diag >= 0 (unique)
    return transpose(q);        // k x d, orthonormal rows
}
static std::uint64_t row_stream(std::uint64_t stream, std::int64_t t) {
    return (stream << 32) + (std::uint64_t)t;
}
void gen_rows(const GenParams& p, std::int64_t t0, std::int64_t n, double* out) {
    const int d = p.d;
    std::int64_t cur_epoch = -1;
    Mat u1, u2;
    if (p.k2 > 0) u2 = gen_basis(p.seed, (1ULL << 40) + p.stream, d, p.k2);
    Vec s(p.k), s2(p.k2), g(d);
    for (std::int64_t q = 0; q < n; ++q) {
        const std::int64_t t = t0 + q;
        const std::int64_t epoch = p.drift_period > 0 ? (t - 1) / p.drift_period : 0;
        if (epoch != cur_epoch) {
            u1 = gen_basis(p.seed, (p.basis_stream << 20) + (std::uint64_t)epoch, d, p.k);
            cur_epoch = epoch;
        }
        RngState rs(p.seed, row_stream(p.stream, t));
        for (int j = 0; j < p.k; ++j) s[j] = rs.gaussian();
        for (int j = 0; j < p.k2; ++j) s2[j] = rs.gaussian();
        for (int j = 0; j < d; ++j) g[j] = rs.gaussian();
        const double u = rs.uniform();
        double* a = out + q * d;
        for (int j = 0; j < d; ++j) a[j] = p.noise * g[j];
        double sig = 1.0;
        for (int l = 0; l < p.k; ++l) {
            const double c = s[l] * sig;
            for (int j = 0; j < d; ++j) a[j] += c * u1(l, j);
            sig *= p.rho;
        }
        sig = p.scale2;
        for (int l = 0; l < p.k2; ++l) {
            const double c = s2[l] * sig;
            for (int j = 0; j < d; ++j) a[j] += c * u2(l, j);
            sig *= p.rho2;
        }
        const double target = std::pow(p.r_max, u);
        const double scale = std::sqrt(target / sq_norm(a, d));
        for (int j = 0; j < d; ++j) a[j] *= scale;
    }
}
void gen_amm_rows(std::uint64_t seed, int dx, int dy, int latent, double noise, double r_max,
                  std::int64_t t0, std::int64_t n, double* x_out, double* y_out) {
    RngState wr(seed, 0xA000000000000000ULL);
    const Mat wx = gaussian_matrix(latent, dx, wr);
    const Mat wy = gaussian_matrix(latent, dy, wr);
    Vec z(latent), g(dx), h(dy);
    for (std::int64_t q = 0; q < n; ++q) {
        const std::int64_t t = t0 + q;
        RngState rs(seed, row_stream(0xA, t));
        for (int j = 0; j < latent; ++j) z[j] = rs.gaussian();
        for (int j = 0; j < dx; ++j) g[j] = rs.gaussian();
        for (int j = 0; j < dy; ++j) h[j] = rs.gaussian();
        const double ux = rs.uniform(), uy = rs.uniform();
        double* x = x_out + q * dx;
        double* y = y_out + q * dy;
        for (int j = 0; j < dx; ++j) x[j] = noise * g[j];
        for (int j = 0; j < dy; ++j) y[j] = noise * h[j];
        for (int l = 0; l < latent; ++l) {
            for (int j = 0; j < dx; ++j) x[j] += z[l] * wx(l, j);
            for (int j = 0; j < dy; ++j) y[j] += z[l] * wy(l, j);
        }
        const double sx = std::sqrt(std::pow(r_max, ux) / sq_norm(x, dx));
        const double sy = std::sqrt(std::pow(r_max, uy) / sq_norm(y, dy));
        for (int j = 0; j < dx; ++j) x[j] *= sx;
        for (int j = 0; j < dy; ++j) y[j] *= sy;
    }
}

}  // namespace orc
