// =============================================================================
// oracle_capi.cpp -- extern "C" surface of the CPU ORACLE for ctypes-driven
// tests (test infrastructure only; never linked by the product). Matrices
// crossing this boundary are row-major.
// =============================================================================
#include <algorithm>
#include <cstring>
#include <memory>
#include <string>

#include "aero_oracle.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const InvalidInput& e) {
        g_err = e.what();
        return 1;
    } catch (const FormatError& e) {
        g_err = e.what();
        return 2;
    } catch (const ProtocolError& e) {
        g_err = e.what();
        return 3;
    } catch (const OracleCapExceeded& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}
Mat from_rm(const double* p, std::int64_t r, std::int64_t c) {
    Mat m(r, c);
    for (std::int64_t i = 0; i < r; ++i)
        for (std::int64_t j = 0; j < c; ++j) m(i, j) = p[i * c + j];
    return m;
}
void to_rm(const Mat& m, double* p) {
    for (std::int64_t i = 0; i < m.r; ++i)
        for (std::int64_t j = 0; j < m.c; ++j) p[i * m.c + j] = m(i, j);
}
struct Site {
    std::unique_ptr<SiteState> s;
    std::vector<Message> outbox;
};
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
void orc_set_threads(int n) { set_threads(n); }
int orc_event_size() { return (int)sizeof(Event); }

// ---- rng: draws of fork #fork_index of RngState(seed, stream) (0 = parent)
int orc_rng_draw(std::uint64_t seed, std::uint64_t stream, std::int64_t fork_index,
                 std::int64_t count, int kind, double* out) {
    return guard([&] {
        RngState root(seed, stream);
        RngState r = root;
        for (std::int64_t f = 0; f < fork_index; ++f) r = root.fork();
        for (std::int64_t i = 0; i < count; ++i) out[i] = kind == 0 ? r.gaussian() : r.uniform();
    });
}

// ---- linalg known-answer surface
int orc_svd(const double* a, int m, int n, double* u, double* s, double* vt) {
    return guard([&] {
        const SvdResult f = svd(from_rm(a, m, n));
        to_rm(f.u, u);
        std::memcpy(s, f.sigma.data(), sizeof(double) * f.sigma.size());
        to_rm(f.vt, vt);
    });
}
int orc_eigh(const double* b, int n, double* lam, double* v) {
    return guard([&] {
        const EighResult f = eigh(from_rm(b, n, n));
        std::memcpy(lam, f.lambda.data(), sizeof(double) * n);
        to_rm(f.v, v);
    });
}
int orc_qr(const double* a, int m, int n, double* q, double* r) {
    return guard([&] {
        const auto f = qr(from_rm(a, m, n));
        to_rm(f.first, q);
        to_rm(f.second, r);
    });
}
int orc_power_iteration(const double* a, int m, int n, int k, std::uint64_t seed,
                        std::uint64_t stream, double* s2, double* x) {
    return guard([&] {
        const auto f = power_iteration(from_rm(a, m, n), k, RngState(seed, stream));
        *s2 = f.first;
        std::memcpy(x, f.second.data(), sizeof(double) * f.second.size());
    });
}
int orc_simul_iter(const double* a, int m, int n, int k, double eps_si, std::uint64_t seed,
                   std::uint64_t stream, double* z, double* sh) {
    return guard([&] {
        const auto f = simul_iter(from_rm(a, m, n), k, eps_si, RngState(seed, stream));
        to_rm(f.z, z);
        std::memcpy(sh, f.sigma_hat.data(), sizeof(double) * k);
    });
}
int orc_fd_reduce(const double* b, int rows, int cols, int ell, double* out) {
    return guard([&] { to_rm(fd_reduce(from_rm(b, rows, cols), ell), out); });
}
int orc_cod_reduce(const double* a, int dx, const double* b, int dy, int cols, int ell,
                   double* ap, double* bp) {
    return guard([&] {
        const auto f = cod_reduce(from_rm(a, dx, cols), from_rm(b, dy, cols), ell);
        to_rm(f.first, ap);
        to_rm(f.second, bp);
    });
}
double orc_spectral_norm_sym(const double* s, int n) { return spectral_norm_sym(from_rm(s, n, n)); }
double orc_spectral_norm(const double* a, int m, int n) { return spectral_norm(from_rm(a, m, n)); }
int orc_shrink_to_sketch(const double* b, int d, int ell, double* out) {
    return guard([&] { to_rm(shrink_to_sketch(from_rm(b, d, d), ell), out); });
}
int orc_restore_contribution(const double* z, const double* m, int d, int xi, double* out) {
    return guard([&] {
        Snapshot s;
        s.z = from_rm(z, d, xi);
        s.m = from_rm(m, xi, d);
        to_rm(restore_contribution(s), out);
    });
}

// ---- AeroState
void* orc_aero_create(int d, double eps, double theta, std::uint64_t seed, std::uint64_t stream) {
    AeroState* p = nullptr;
    if (guard([&] { p = new AeroState(d, eps, theta, RngState(seed, stream)); }) != 0)
        return nullptr;
    return p;
}
void* orc_aero_create2(int d, double eps, double theta, std::uint64_t seed, std::uint64_t stream, double delta) {
    AeroState* p = nullptr;
    if (guard([&] { p = new AeroState(d, eps, theta, RngState(seed, stream), delta); }) != 0)
        return nullptr;
    return p;
}
int orc_aero_update_block_amplified(void* h, const double* rows, std::int64_t n, const std::int64_t* t,
                                    const double* theta, Event* ev) {
    return guard([&] {
        auto* s = static_cast<AeroState*>(h);
        for (std::int64_t q = 0; q < n; ++q) {
            if (theta) s->set_theta(theta[q]);
            s->update_amplified(rows + q * s->d(), t[q]);
            if (ev) ev[q] = s->last_event();
        }
    });
}
void* orc_attp_create2(int d, double eps, std::uint64_t seed, std::uint64_t stream, double delta) {
    AttpState* p = nullptr;
    if (guard([&] { p = new AttpState(d, eps, RngState(seed, stream), delta); }) != 0) return nullptr;
    return p;
}
void* orc_ml_create2(int d, std::int64_t n, double rmax, double eps, std::uint64_t seed, std::uint64_t stream,
                     double delta) {
    MlState* p = nullptr;
    if (guard([&] { p = new MlState(d, n, rmax, eps, RngState(seed, stream), delta); }) != 0) return nullptr;
    return p;
}
void orc_aero_destroy(void* h) { delete static_cast<AeroState*>(h); }
int orc_aero_set_theta(void* h, double th) {
    return guard([&] { static_cast<AeroState*>(h)->set_theta(th); });
}
int orc_aero_update_block(void* h, const double* rows, std::int64_t n, const std::int64_t* t,
                          const double* theta, Event* ev) {
    return guard([&] {
        auto* s = static_cast<AeroState*>(h);
        for (std::int64_t q = 0; q < n; ++q) {
            if (theta) s->set_theta(theta[q]);
            s->update(rows + q * s->d(), t[q]);
            if (ev) ev[q] = s->last_event();
        }
    });
}
int orc_aero_query(void* h, std::int64_t lb, std::int64_t ub, double* out) {
    return guard([&] { to_rm(static_cast<AeroState*>(h)->query(lb, ub), out); });
}
int orc_aero_query_gram(void* h, std::int64_t lb, std::int64_t ub, double* out) {
    return guard([&] { to_rm(static_cast<AeroState*>(h)->query_gram(lb, ub), out); });
}
std::int64_t orc_aero_rows(void* h) { return static_cast<AeroState*>(h)->rows(); }
int orc_aero_residual(void* h, double* out) {
    return guard([&] {
        const Mat& ct = static_cast<AeroState*>(h)->residual_t();
        std::memcpy(out, ct.data(), sizeof(double) * ct.size());  // C row-major == C^T col-major
    });
}
std::int64_t orc_aero_snap_count(void* h) {
    return (std::int64_t) static_cast<AeroState*>(h)->snaps().size();
}
int orc_aero_snap_info(void* h, std::int64_t idx, int* xi, std::int64_t* s, std::int64_t* t,
                       double* theta) {
    return guard([&] {
        const Snapshot& sn = static_cast<AeroState*>(h)->snaps().at(idx);
        *xi = (int)sn.z.c;
        *s = sn.s;
        *t = sn.t;
        *theta = sn.theta;
    });
}
int orc_aero_snap_get(void* h, std::int64_t idx, double* z, double* m) {
    return guard([&] {
        const Snapshot& sn = static_cast<AeroState*>(h)->snaps().at(idx);
        if (z) to_rm(sn.z, z);
        if (m) to_rm(sn.m, m);
    });
}
int orc_aero_snap_pop_front(void* h) {
    return guard([&] {
        auto& q = static_cast<AeroState*>(h)->snaps();
        if (!q.empty()) q.pop_front();
    });
}
int orc_aero_info(void* h, int* d, int* ell, std::int64_t* clock, double* theta,
                  std::int64_t* forks, std::int64_t* last_dump) {
    auto* s = static_cast<AeroState*>(h);
    *d = s->d();
    *ell = s->ell();
    *clock = s->clock();
    *theta = s->theta();
    *forks = (std::int64_t)s->forks();
    *last_dump = s->last_dump_time();
    return 0;
}

// ---- AttpState
void* orc_attp_create(int d, double eps, std::uint64_t seed, std::uint64_t stream) {
    AttpState* p = nullptr;
    if (guard([&] { p = new AttpState(d, eps, RngState(seed, stream)); }) != 0) return nullptr;
    return p;
}
void orc_attp_destroy(void* h) { delete static_cast<AttpState*>(h); }
int orc_attp_update_block(void* h, const double* rows, std::int64_t n, const std::int64_t* t,
                          Event* ev) {
    return guard([&] {
        auto* s = static_cast<AttpState*>(h);
        const int d = s->inner().d();
        for (std::int64_t q = 0; q < n; ++q) {
            s->update(rows + q * d, t[q]);
            if (ev) ev[q] = s->inner().last_event();
        }
    });
}
int orc_attp_query(void* h, std::int64_t t, double* out) {
    return guard([&] { to_rm(static_cast<AttpState*>(h)->query(t), out); });
}
double orc_attp_mass(void* h) { return static_cast<AttpState*>(h)->fro_mass(); }
int orc_attp_import(void* h, const double* rows, std::int64_t r, std::uint64_t forks, std::int64_t clock,
                    std::int64_t last_dump_t, double theta, double fro_mass) {
    return guard([&] {
        auto* s = static_cast<AttpState*>(h);
        s->inner().import_state(rows, r, forks, clock, last_dump_t, theta);
        s->set_fro_mass(fro_mass);
    });
}
void* orc_attp_inner(void* h) { return &static_cast<AttpState*>(h)->inner(); }

// ---- MlState
void* orc_ml_create(int d, std::int64_t n, double rmax, double eps, std::uint64_t seed,
                    std::uint64_t stream) {
    MlState* p = nullptr;
    if (guard([&] { p = new MlState(d, n, rmax, eps, RngState(seed, stream)); }) != 0)
        return nullptr;
    return p;
}
void orc_ml_destroy(void* h) { delete static_cast<MlState*>(h); }
int orc_ml_update_block(void* h, const double* rows, std::int64_t n, const std::int64_t* t) {
    return guard([&] {
        auto* s = static_cast<MlState*>(h);
        for (std::int64_t q = 0; q < n; ++q) s->update(rows + q * s->d(), t[q]);
    });
}
int orc_ml_query(void* h, double* sketch, int* level, int* fallback, std::int64_t* xi_sum,
                 int* heavy_used) {
    return guard([&] {
        const MlQueryResult r = static_cast<MlState*>(h)->query();
        to_rm(r.sketch, sketch);
        *level = r.level;
        *fallback = r.fallback;
        *xi_sum = r.xi_sum;
        *heavy_used = r.heavy_used;
    });
}
int orc_ml_info(void* h, int* levels, int* ell, double* window_mass, std::int64_t* norm_warnings,
                std::int64_t* cap, std::int64_t* clock) {
    auto* s = static_cast<MlState*>(h);
    *levels = s->levels();
    *ell = s->ell();
    *window_mass = s->window_mass();
    *norm_warnings = s->norm_warnings();
    *cap = s->cap();
    *clock = s->clock();
    return 0;
}
double orc_ml_theta(void* h, int j) { return static_cast<MlState*>(h)->theta(j); }
void* orc_ml_level(void* h, int j) {
    return const_cast<AeroState*>(&static_cast<MlState*>(h)->level_state(j));
}
std::int64_t orc_ml_heavy_count(void* h, int j) {
    return (std::int64_t) static_cast<MlState*>(h)->heavy(j).size();
}
int orc_ml_heavy_get(void* h, int j, std::int64_t idx, double* row, std::int64_t* s,
                     std::int64_t* t) {
    return guard([&] {
        const HeavyRow& hr = static_cast<MlState*>(h)->heavy(j).at(idx);
        if (row) std::memcpy(row, hr.row.data(), sizeof(double) * hr.row.size());
        *s = hr.s;
        *t = hr.t;
    });
}
std::int64_t orc_ml_stored_floats(void* h) { return static_cast<MlState*>(h)->stored_floats(); }

// ---- CodState
void* orc_cod_create(int dx, int dy, double eps, double theta, std::int64_t n, std::uint64_t seed,
                     std::uint64_t stream) {
    CodState* p = nullptr;
    if (guard([&] { p = new CodState(dx, dy, eps, theta, n, RngState(seed, stream)); }) != 0)
        return nullptr;
    return p;
}
void orc_cod_destroy(void* h) { delete static_cast<CodState*>(h); }
int orc_cod_update_block(void* h, const double* x, const double* y, int dx, int dy,
                         std::int64_t n, const std::int64_t* t, Event* ev) {
    return guard([&] {
        auto* s = static_cast<CodState*>(h);
        for (std::int64_t q = 0; q < n; ++q) {
            s->update(x + q * dx, y + q * dy, t[q]);
            if (ev) ev[q] = s->last_event();
        }
    });
}
int orc_cod_query(void* h, double* astar, double* bstar) {
    return guard([&] {
        const auto r = static_cast<CodState*>(h)->query();
        to_rm(r.first, astar);
        to_rm(r.second, bstar);
    });
}
int orc_cod_query_product(void* h, double* p) {
    return guard([&] { to_rm(static_cast<CodState*>(h)->query_product(), p); });
}
int orc_cod_info(void* h, int* ell, std::int64_t* cols, std::int64_t* nsnaps, std::int64_t* clock) {
    auto* s = static_cast<CodState*>(h);
    *ell = s->ell();
    *cols = s->a().c;
    *nsnaps = (std::int64_t)s->snaps().size();
    *clock = s->clock();
    return 0;
}
int orc_cod_get_ab(void* h, double* a, double* b) {
    return guard([&] {
        auto* s = static_cast<CodState*>(h);
        to_rm(s->a(), a);
        to_rm(s->b(), b);
    });
}

// ---- AdaptiveState (reference amm.hpp:71-93)
void* orc_adaptive_create(int dx, int dy, double eps, double theta0, std::int64_t n,
                          std::uint64_t seed, std::uint64_t stream) {
    AdaptiveState* p = nullptr;
    if (guard([&] { p = new AdaptiveState(dx, dy, eps, theta0, n, RngState(seed, stream)); }) != 0)
        return nullptr;
    return p;
}
void orc_adaptive_destroy(void* h) { delete static_cast<AdaptiveState*>(h); }
// per row: level after the row, main's theta and snapshot count after the row
int orc_adaptive_update_block(void* h, const double* x, const double* y, int dx, int dy,
                              std::int64_t n, const std::int64_t* t, Event* ev, int* level,
                              double* theta, std::int64_t* nsnaps) {
    return guard([&] {
        auto* s = static_cast<AdaptiveState*>(h);
        for (std::int64_t q = 0; q < n; ++q) {
            s->update(x + q * dx, y + q * dy, t[q]);
            if (ev) ev[q] = s->main().last_event();
            if (level) level[q] = s->level();
            if (theta) theta[q] = s->main().theta();
            if (nsnaps) nsnaps[q] = (std::int64_t)s->main().snaps().size();
        }
    });
}
int orc_adaptive_query(void* h, double* astar, double* bstar) {
    return guard([&] {
        const auto r = static_cast<AdaptiveState*>(h)->query();
        to_rm(r.first, astar);
        to_rm(r.second, bstar);
    });
}
int orc_adaptive_query_product(void* h, double* p) {
    return guard([&] { to_rm(static_cast<AdaptiveState*>(h)->main().query_product(), p); });
}

// ---- distributed: site / coordinator objects and the tick simulator
void* orc_site_create(int id, int d, double eps, int m, std::uint64_t seed, std::uint64_t stream,
                      std::int64_t window) {
    Site* p = nullptr;
    if (guard([&] {
            p = new Site;
            p->s.reset(new SiteState(id, d, eps, m, RngState(seed, stream),
                                     window > 0 ? std::optional<std::int64_t>(window)
                                                : std::nullopt));
        }) != 0)
        return nullptr;
    return p;
}
void orc_site_destroy(void* h) { delete static_cast<Site*>(h); }
// update; returns the outbox length (messages are retained in the site until
// the next update and can be read with orc_site_msg)
int orc_site_update(void* h, const double* row, std::int64_t t, int* n_msgs) {
    return guard([&] {
        auto* s = static_cast<Site*>(h);
        s->outbox.clear();
        s->s->update(row, t, s->outbox);
        *n_msgs = (int)s->outbox.size();
    });
}
int orc_site_msg(void* h, int idx, int* kind, double* f, std::int64_t* t, int* xi,
                 std::int64_t* bytes, double* z, double* m) {
    return guard([&] {
        const Message& msg = static_cast<Site*>(h)->outbox.at(idx);
        *kind = (int)msg.kind;
        *f = msg.f;
        *t = msg.t;
        *xi = (int)msg.z.c;
        *bytes = msg.bytes();
        if (z && msg.z.size()) to_rm(msg.z, z);
        if (m && msg.m.size()) to_rm(msg.m, m);
    });
}
void orc_site_on_broadcast(void* h, double f) { static_cast<Site*>(h)->s->on_broadcast(f); }
double orc_site_theta(void* h) { return static_cast<Site*>(h)->s->inner().theta(); }
void* orc_site_inner(void* h) { return const_cast<AeroState*>(&static_cast<Site*>(h)->s->inner()); }

int orc_dist_run(int m, int d, double eps, std::int64_t window, std::int64_t query_every,
                 std::int64_t latency, std::uint64_t seed, const double* streams, std::int64_t T,
                 std::int64_t oracle_cap, double* probe_err, std::int64_t* probe_bytes,
                 std::int64_t* comm_bytes_out, std::int64_t* broadcasts_out, double* theta_out,
                 double* final_gram) {
    // reference distributed.cpp:177-269 (update-only timing omitted)
    return guard([&] {
        const bool window_mode = window > 0;
        const int ell = static_cast<int>(std::ceil(2.0 / eps));
        std::vector<SiteState> sites;
        for (int j = 0; j < m; ++j)
            sites.emplace_back(j, d, eps, m, RngState(seed, kSketchStreamBase + j),
                               window_mode ? std::optional<std::int64_t>(window) : std::nullopt);
        CoordinatorState coord(d, m, window_mode);
        OracleGram oracle(d, window_mode ? std::optional<std::int64_t>(window) : std::nullopt,
                          oracle_cap);
        std::deque<std::pair<std::int64_t, Message>> to_coord, to_sites;
        std::int64_t comm_bytes = 0, probe = 0;
        for (std::int64_t i = 1; i <= T; ++i) {
            while (!to_sites.empty() && to_sites.front().first <= i) {
                for (SiteState& s : sites) s.on_broadcast(to_sites.front().second.f);
                to_sites.pop_front();
            }
            std::vector<Message> outbox;
            for (int j = 0; j < m; ++j) {
                const double* row = streams + ((std::int64_t)j * T + (i - 1)) * d;
                sites[j].update(row, i, outbox);
                if (theta_out) theta_out[(std::int64_t)j * T + (i - 1)] = sites[j].inner().theta();
                if (probe_err) oracle.add(row, i);
            }
            for (Message& msg : outbox) {
                comm_bytes += msg.bytes();
                to_coord.emplace_back(i + latency, std::move(msg));
            }
            while (!to_coord.empty() && to_coord.front().first <= i) {
                std::optional<Message> bc = coord.receive(to_coord.front().second);
                to_coord.pop_front();
                if (bc) {
                    comm_bytes += (std::int64_t)m * bc->bytes();
                    to_sites.emplace_back(i + 1 + latency, std::move(*bc));
                }
            }
            if (query_every > 0 && i % query_every == 0 && probe_err) {
                // probe_gram: residual Grams + contributions sorted by (t, site)
                Mat b(d, d);
                for (const SiteState& s : sites) {
                    const Mat& ct = s.inner().residual_t();
                    if (ct.c > 0) {
                        const Mat g = matmul(ct, ct, false, true);
                        for (std::int64_t q = 0; q < b.size(); ++q) b.v[q] += g.v[q];
                    }
                }
                std::vector<const std::pair<const std::pair<int, std::int64_t>, Mat>*> live;
                for (const auto& kv : coord.contributions()) live.push_back(&kv);
                std::sort(live.begin(), live.end(), [](const auto* x, const auto* y) {
                    if (x->first.second != y->first.second) return x->first.second < y->first.second;
                    return x->first.first < y->first.first;
                });
                for (const auto* kv : live)
                    for (std::int64_t q = 0; q < b.size(); ++q) b.v[q] += kv->second.v[q];
                const Mat sk = shrink_to_sketch(b, ell);
                double err = -1.0;
                try {
                    err = oracle.error(sk);
                } catch (const OracleCapExceeded&) {
                }
                probe_err[probe] = err;
                if (probe_bytes) probe_bytes[probe] = comm_bytes;
                ++probe;
                if (final_gram) to_rm(b, final_gram);
            }
        }
        *comm_bytes_out = comm_bytes;
        *broadcasts_out = coord.broadcasts();
    });
}

// ---- exact Gram oracle
void* orc_gram_create(int d, std::int64_t window, std::int64_t cap) {
    return new OracleGram(d, window > 0 ? std::optional<std::int64_t>(window) : std::nullopt, cap);
}
void orc_gram_destroy(void* h) { delete static_cast<OracleGram*>(h); }
int orc_gram_add_block(void* h, const double* rows, int d, std::int64_t n, const std::int64_t* t) {
    return guard([&] {
        for (std::int64_t q = 0; q < n; ++q) static_cast<OracleGram*>(h)->add(rows + q * d, t[q]);
    });
}
int orc_gram_error(void* h, const double* sketch, std::int64_t rows, int d, double* err) {
    return guard([&] { *err = static_cast<OracleGram*>(h)->error(from_rm(sketch, rows, d)); });
}
double orc_gram_mass(void* h) { return static_cast<OracleGram*>(h)->mass(); }
int orc_gram_get(void* h, double* g) {
    return guard([&] { to_rm(static_cast<OracleGram*>(h)->gram(), g); });
}

// ---- generators
int orc_gen_rows(int d, int k, double rho, double noise, double rmax, std::uint64_t seed,
                 std::uint64_t stream, std::int64_t drift, int k2, double rho2, double scale2,
                 std::uint64_t basis_stream, std::int64_t t0, std::int64_t n, double* out) {
    return guard([&] {
        GenParams p;
        p.d = d;
        p.k = k;
        p.rho = rho;
        p.noise = noise;
        p.r_max = rmax;
        p.seed = seed;
        p.stream = stream;
        p.drift_period = drift;
        p.k2 = k2;
        p.rho2 = rho2;
        p.scale2 = scale2;
        p.basis_stream = basis_stream;
        gen_rows(p, t0, n, out);
    });
}
int orc_gen_basis(std::uint64_t seed, std::uint64_t basis_id, int d, int k, double* out) {
    return guard([&] { to_rm(gen_basis(seed, basis_id, d, k), out); });
}
int orc_gen_amm_rows(std::uint64_t seed, int dx, int dy, int latent, double noise, double rmax,
                     std::int64_t t0, std::int64_t n, double* x, double* y) {
    return guard([&] { gen_amm_rows(seed, dx, dy, latent, noise, rmax, t0, n, x, y); });
}

}  // extern "C"
