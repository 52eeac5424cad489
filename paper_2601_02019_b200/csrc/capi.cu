// extern "C" boundary (include/aero_b200.h): maps the reference's exceptions
// (errors.hpp:15-33) to status codes; no torch types cross this line.
#include <cstring>
#include <string>
#include <vector>

#include "aero_common.cuh"
#include "aeroio.hpp"
#include "engines.hpp"
#include "sketch.hpp"
#include "rng_panels.hpp"

using namespace aero_b200;

struct aero_sketch {
    Sketch* s;
    bool owned;
};

namespace aero_b200 {
long long launches_total();
thread_local std::string g_last_error;
}  // namespace aero_b200

namespace {
template <typename F>
int guard(F&& f) {
    try {
        f();
        return AERO_OK;
    } catch (const InvalidInput& e) {
        g_last_error = e.what();
        return AERO_INVALID_INPUT;
    } catch (const ProtocolError& e) {
        g_last_error = e.what();
        return AERO_PROTOCOL_ERROR;
    } catch (const FormatError& e) {
        g_last_error = e.what();
        return AERO_FORMAT_ERROR;
    } catch (const CudaError& e) {
        g_last_error = e.what();
        return AERO_CUDA_ERROR;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return AERO_INTERNAL_ERROR;
    }
}
int require(const void* p, const char* what) {
    if (!p) {
        g_last_error = std::string(what) + ": null handle";
        return AERO_INVALID_INPUT;
    }
    return AERO_OK;
}
#define REQ(p)                                   \
    do {                                         \
        int _rc = require((p), __func__);        \
        if (_rc != AERO_OK) return _rc;          \
    } while (0)
}  // namespace

extern "C" {

const char* aero_last_error(void) { return g_last_error.c_str(); }
const char* aero_version(void) { return "aero_b200 0.1 (sm_100a, fp64)"; }
int64_t aero_kernel_launches(void) { return (int64_t)launches_total(); }

int aero_create(const aero_cfg* cfg, aero_sketch** out) {
    REQ(cfg);
    REQ(out);
    return guard([&] {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw CudaError("no CUDA device: the AeroSketch B200 path has no CPU fallback");
        *out = new aero_sketch{new Sketch(*cfg), true};
    });
}
int aero_destroy(aero_sketch* h) {
    if (!h) return AERO_OK;
    return guard([&] {
        if (h->owned) delete h->s;
        delete h;
    });
}
int aero_set_theta(aero_sketch* h, double theta) {
    REQ(h);
    return guard([&] { h->s->set_theta(theta); });
}
int aero_set_grid_share(aero_sketch* h, int32_t share) {
    REQ(h);
    h->s->set_grid_share(share);
    return AERO_OK;
}
int aero_set_rng_fill(aero_sketch* h, aero_rng_fill fn, void* ctx) {
    REQ(h);
    return guard([&] { h->s->set_rng_source(h->s->host_rng_default(), fn, ctx); });
}
int aero_update_block(aero_sketch* h, const double* rows, int64_t n, int64_t ld, const int64_t* t,
                      const double* theta_per_row, aero_event* log_out) {
    REQ(h);
    if (n > 0) {
        REQ(rows);
        REQ(t);
    }
    return guard([&] { h->s->update_block(rows, false, n, ld, t, theta_per_row, log_out); });
}
int aero_update_block_amplified(aero_sketch* h, const double* rows, int64_t n, int64_t ld, const int64_t* t,
                                const double* theta_per_row, aero_event* log_out) {
    REQ(h);
    if (n > 0) {
        REQ(rows);
        REQ(t);
    }
    return guard([&] { h->s->update_block(rows, false, n, ld, t, theta_per_row, log_out, true); });
}
int aero_update_block_device(aero_sketch* h, const double* rows_device, int64_t n, int64_t ld,
                             const int64_t* t, const double* theta_per_row, aero_event* log_out) {
    REQ(h);
    if (n > 0) {
        REQ(rows_device);
        REQ(t);
    }
    return guard([&] { h->s->update_block(rows_device, true, n, ld, t, theta_per_row, log_out); });
}
int aero_query(aero_sketch* h, int64_t lb, int64_t ub, double* out) {
    REQ(h);
    REQ(out);
    return guard([&] { h->s->query(lb, ub, out); });
}
int aero_query_gram(aero_sketch* h, int64_t lb, int64_t ub, double* out) {
    REQ(h);
    REQ(out);
    return guard([&] { h->s->query_gram(lb, ub, out); });
}
int aero_attp_query(aero_sketch* h, int64_t t, double* out) {  // attp.hpp:29-32
    REQ(h);
    REQ(out);
    return guard([&] {
        if (t < 1 || t > h->s->clock()) throw InvalidInput("AttpState: t out of range");
        h->s->query(0, t, out);
    });
}
int aero_residual(aero_sketch* h, double* out, int64_t max_rows) {
    REQ(h);
    return guard([&] {
        if (h->s->rows() > 0 && max_rows > 0) {
            if (!out) throw InvalidInput("aero_residual: null output");
            h->s->residual(out, max_rows);
        }
    });
}
int aero_snap_count(aero_sketch* h, int64_t* count) {
    REQ(h);
    REQ(count);
    *count = h->s->snap_count();
    return AERO_OK;
}
int aero_snap_info(aero_sketch* h, int64_t idx, int32_t* xi, int64_t* s, int64_t* t, double* theta) {
    REQ(h);
    return guard([&] {
        const SnapRec& r = h->s->snap(idx);
        if (xi) *xi = r.xi;
        if (s) *s = r.s;
        if (t) *t = r.t;
        if (theta) *theta = r.theta;
    });
}
int aero_snap_get(aero_sketch* h, int64_t idx, double* z, double* m) {
    REQ(h);
    return guard([&] { h->s->snap_get(idx, z, m); });
}
int aero_snap_pop_front(aero_sketch* h) {
    REQ(h);
    return guard([&] { h->s->snap_pop_front(); });
}
int aero_last_stats(aero_sketch* h, aero_event* out) {
    REQ(h);
    REQ(out);
    *out = h->s->last_event();
    return AERO_OK;
}
int aero_get_info(aero_sketch* h, aero_info* out) {
    REQ(h);
    REQ(out);
    h->s->info(out);
    return AERO_OK;
}
int aero_synchronize(aero_sketch* h) {
    REQ(h);
    return guard([&] { h->s->synchronize(); });
}

void* aero_stream(aero_sketch* h) { return h ? (void*)h->s->stream() : nullptr; }
int aero_get_profile(aero_sketch* h, aero_profile* out) {
    REQ(h);
    REQ(out);
    *out = h->s->prof;
    return AERO_OK;
}
int aero_reset_profile(aero_sketch* h) {
    REQ(h);
    h->s->prof = aero_profile{};
    return AERO_OK;
}

int aero_dev_product(int32_t r, int32_t n, const double* g, const double* x, const int32_t* colmask,
                     int32_t mode, double* y, double* device_ms) {
    REQ(g);
    REQ(x);
    REQ(y);
    return guard([&] {
        if (r < 1 || n < 1) throw InvalidInput("product: empty input");
        if (mode != 0 && mode != 1) throw InvalidInput("product: mode must be 0 or 1");
        const int ld = r + (r & 1);
        double *dG, *dX, *dY, *dW;
        int* dM = nullptr;
        const size_t wsn = product_workspace_doubles(r, n);
        AERO_CUDA(cudaMalloc(&dG, sizeof(double) * (size_t)ld * r));
        AERO_CUDA(cudaMalloc(&dX, sizeof(double) * (size_t)ld * n));
        AERO_CUDA(cudaMalloc(&dY, sizeof(double) * (size_t)ld * n));
        AERO_CUDA(cudaMalloc(&dW, sizeof(double) * wsn));
        AERO_CUDA(cudaMemcpy2D(dG, sizeof(double) * ld, g, sizeof(double) * r, sizeof(double) * r, r,
                               cudaMemcpyHostToDevice));
        AERO_CUDA(cudaMemcpy2D(dX, sizeof(double) * ld, x, sizeof(double) * r, sizeof(double) * r, n,
                               cudaMemcpyHostToDevice));
        if (colmask) {
            AERO_CUDA(cudaMalloc(&dM, sizeof(int) * n));
            AERO_CUDA(cudaMemcpy(dM, colmask, sizeof(int) * n, cudaMemcpyHostToDevice));
        }
        OzakiGram oz;
        cudaStream_t st = 0;
        if (mode == 0) oz.prepare(st, r, dG, ld);
        auto run = [&] {
            if (mode == 0) oz.product(st, n, dX, ld, dM, dY, ld, dW, wsn);
            else gemm_product(st, r, n, r, dG, ld, dX, ld, dY, ld, dM, dW, wsn);
        };
        run();
        AERO_CUDA(cudaStreamSynchronize(st));
        AERO_CUDA(cudaMemcpy2D(y, sizeof(double) * r, dY, sizeof(double) * ld, sizeof(double) * r, n,
                               cudaMemcpyDeviceToHost));
        if (device_ms) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0, st);
            for (int it = 0; it < 20; ++it) run();
            cudaEventRecord(e1, st);
            AERO_CUDA(cudaEventSynchronize(e1));
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            *device_ms = ms / 20.0;
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
        }
        oz.release();
        cudaFree(dG);
        cudaFree(dX);
        cudaFree(dY);
        cudaFree(dW);
        if (dM) cudaFree(dM);
    });
}

int aero_eigh(int32_t n, const double* a, double* w, double* v, double* device_ms) {
    REQ(a);
    REQ(w);
    REQ(v);
    return guard([&] {
        if (n < 1) throw InvalidInput("eigh: empty input");
        double *dA = nullptr, *dw = nullptr;
        AERO_CUDA(cudaMalloc(&dA, sizeof(double) * (size_t)n * n));
        AERO_CUDA(cudaMalloc(&dw, sizeof(double) * n));
        // row-major symmetric input == its column-major transpose
        AERO_CUDA(cudaMemcpy(dA, a, sizeof(double) * (size_t)n * n, cudaMemcpyHostToDevice));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, 0);
        eigh(0, n, dA, n, dw);
        cudaEventRecord(e1, 0);
        AERO_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (device_ms) *device_ms = ms;
        std::vector<double> cm((size_t)n * n);
        AERO_CUDA(cudaMemcpy(cm.data(), dA, sizeof(double) * cm.size(), cudaMemcpyDeviceToHost));
        AERO_CUDA(cudaMemcpy(w, dw, sizeof(double) * n, cudaMemcpyDeviceToHost));
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) v[(size_t)i * n + j] = cm[i + (size_t)j * n];
        cudaFree(dA);
        cudaFree(dw);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    });
}

int aero_rng_gaussians(uint64_t seed, uint64_t stream, int64_t fork, int64_t count, double* out) {
    REQ(out);
    return guard([&] {
        uint64_t s = stream;
        if (fork > 0) s = fork_stream(stream, (uint64_t)fork);
        double* d = nullptr;
        AERO_CUDA(cudaMalloc(&d, sizeof(double) * std::max<int64_t>(count, 1)));
        gen_gaussian_matrix(0, rng_state0(seed, s), count, d);
        AERO_CUDA(cudaMemcpy(out, d, sizeof(double) * count, cudaMemcpyDeviceToHost));
        cudaFree(d);
    });
}

int aero_rng_gaussians_host(uint64_t seed, uint64_t stream, int64_t fork, int64_t count, double* out) {
    REQ(out);
    return guard([&] {
        const uint64_t s = (fork > 0) ? fork_stream(stream, (uint64_t)fork) : stream;
        const uint64_t s0 = rng_state0(seed, s);
        for (int64_t i = 0; i < count; ++i) out[i] = host_gaussian_at(s0, (uint64_t)i);
    });
}

// ---- MlState ----------------------------------------------------------------
struct aero_ml {
    MlEngine* e;
    std::vector<aero_sketch> levels;
};
int aero_ml_create(int32_t d, int64_t window, double r_max, double eps, uint64_t seed,
                   uint64_t stream, int32_t device, aero_ml** out) {
    return aero_ml_create_amplified(d, window, r_max, eps, 0.0, seed, stream, device, out);
}
int aero_ml_create_amplified(int32_t d, int64_t window, double r_max, double eps, double delta,
                             uint64_t seed, uint64_t stream, int32_t device, aero_ml** out) {
    REQ(out);
    return guard([&] {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw CudaError("no CUDA device: the AeroSketch B200 path has no CPU fallback");
        auto* h = new aero_ml;
        h->e = new MlEngine(d, window, r_max, eps, seed, stream, device, delta);
        for (int j = 0; j < h->e->levels(); ++j) h->levels.push_back(aero_sketch{&h->e->level(j), false});
        *out = h;
    });
}
int aero_ml_destroy(aero_ml* h) {
    if (!h) return AERO_OK;
    return guard([&] {
        delete h->e;
        delete h;
    });
}
int aero_ml_update_block(aero_ml* h, const double* rows, int64_t n, int64_t ld, const int64_t* t) {
    REQ(h);
    return guard([&] { h->e->update_block(rows, false, n, ld, t); });
}
int aero_ml_update_block_device(aero_ml* h, const double* rows, int64_t n, int64_t ld,
                                const int64_t* t) {
    REQ(h);
    return guard([&] { h->e->update_block(rows, true, n, ld, t); });
}
int aero_ml_query(aero_ml* h, double* out, aero_ml_query_result* res) {
    REQ(h);
    REQ(out);
    return guard([&] { h->e->query(out, res); });
}
int aero_ml_get_info(aero_ml* h, aero_ml_info* out) {
    REQ(h);
    REQ(out);
    h->e->info(out);
    return AERO_OK;
}
double aero_ml_theta(aero_ml* h, int32_t level) {
    if (!h || level < 0 || level >= h->e->levels()) return -1.0;
    return h->e->level(level).theta();
}
aero_sketch* aero_ml_level(aero_ml* h, int32_t level) {
    if (!h || level < 0 || level >= (int)h->levels.size()) return nullptr;
    return &h->levels[level];
}
int aero_ml_heavy_count(aero_ml* h, int32_t level, int64_t* count) {
    REQ(h);
    REQ(count);
    return guard([&] { *count = h->e->heavy_count(level); });
}
int aero_ml_heavy_get(aero_ml* h, int32_t level, int64_t idx, double* row, int64_t* s, int64_t* t) {
    REQ(h);
    return guard([&] { h->e->heavy_get(level, idx, row, s, t); });
}

// ---- distributed ---------------------------------------------------------------
int aero_dist_theta_schedule(int32_t m, int64_t T, double eps, int64_t latency,
                             const double* sq_norms, double* theta_out, int64_t* mass_bytes,
                             int64_t* broadcasts) {
    REQ(sq_norms);
    REQ(theta_out);
    return guard([&] {
        dist_theta_schedule(m, T, eps, latency, sq_norms, theta_out, mass_bytes, broadcasts);
    });
}
struct aero_dist_protocol {
    DistProtocol* p;
};
int aero_dist_protocol_create(int32_t m, double eps, int64_t latency, aero_dist_protocol** out) {
    REQ(out);
    return guard([&] { *out = new aero_dist_protocol{new DistProtocol(m, eps, latency)}; });
}
int aero_dist_protocol_create_window(int32_t m, double eps, int64_t latency, int64_t window,
                                     aero_dist_protocol** out) {
    REQ(out);
    return guard([&] { *out = new aero_dist_protocol{new DistProtocol(m, eps, latency, window)}; });
}
int aero_dist_protocol_destroy(aero_dist_protocol* h) {
    if (!h) return AERO_OK;
    delete h->p;
    delete h;
    return AERO_OK;
}
int aero_dist_protocol_advance(aero_dist_protocol* h, int64_t T, const double* sq_norms,
                               double* theta_out) {
    REQ(h);
    if (T > 0) {
        REQ(sq_norms);
        REQ(theta_out);
    }
    return guard([&] { h->p->advance(T, sq_norms, theta_out); });
}
int aero_dist_protocol_info(aero_dist_protocol* h, int64_t* ticks, int64_t* mass_bytes,
                            int64_t* broadcasts, double* f_hat) {
    REQ(h);
    if (ticks) *ticks = h->p->ticks;
    if (mass_bytes) *mass_bytes = h->p->bytes;
    if (broadcasts) *broadcasts = h->p->broadcasts;
    if (f_hat) *f_hat = h->p->f_hat;
    return AERO_OK;
}
int aero_row_sq_norms_device(const double* rows_device, int64_t n, int64_t ld, int32_t d,
                             int32_t device, double* out_host) {
    REQ(rows_device);
    REQ(out_host);
    return guard([&] {
        AERO_CUDA(cudaSetDevice(device));
        double* nrm = nullptr;
        int* bad = nullptr;
        AERO_CUDA(cudaMalloc(&nrm, sizeof(double) * std::max<int64_t>(n, 1)));
        AERO_CUDA(cudaMalloc(&bad, sizeof(int) * std::max<int64_t>(n, 1)));
        ingest_rows(0, rows_device, n, ld, d, nrm, bad);
        AERO_CUDA(cudaMemcpy(out_host, nrm, sizeof(double) * n, cudaMemcpyDeviceToHost));
        cudaFree(nrm);
        cudaFree(bad);
    });
}

struct aero_coord {
    Coordinator* c;
};
int aero_coord_create(int32_t d, int32_t m, int32_t device, void* nccl_comm, aero_coord** out) {
    REQ(out);
    return guard([&] { *out = new aero_coord{new Coordinator(d, m, device, nccl_comm)}; });
}
int aero_coord_create_window(int32_t d, int32_t m, int32_t device, void* nccl_comm, int64_t window,
                             int64_t latency, aero_coord** out) {
    REQ(out);
    return guard([&] { *out = new aero_coord{new Coordinator(d, m, device, nccl_comm, window, latency)}; });
}
int aero_coord_destroy(aero_coord* h) {
    if (!h) return AERO_OK;
    return guard([&] {
        delete h->c;
        delete h;
    });
}
int aero_coord_absorb_snapshots(aero_coord* h, aero_sketch* site, int64_t* bytes) {
    REQ(h);
    REQ(site);
    return guard([&] {
        const int64_t b = h->c->absorb(*site->s);
        if (bytes) *bytes = b;
    });
}
int aero_coord_probe(aero_coord* h, aero_sketch* const* sites, int32_t nsites, int32_t root,
                     int32_t ell, double* out, double* gram) {
    REQ(h);
    return guard([&] {
        std::vector<Sketch*> ss;
        for (int i = 0; i < nsites; ++i)
            if (sites && sites[i]) ss.push_back(sites[i]->s);
        h->c->probe(ss, root, ell, out, gram);
    });
}
int aero_coord_shrink(aero_coord* h, const double* gram, int32_t ell, double* out) {
    REQ(h);
    REQ(gram);
    REQ(out);
    return guard([&] { h->c->shrink(gram, ell, out); });
}
int aero_nccl_get_unique_id(char* id128) {
    REQ(id128);
    return guard([&] { nccl_unique_id(id128); });
}
int aero_nccl_comm_init(const char* id128, int32_t nranks, int32_t rank, int32_t device,
                        void** comm_out) {
    REQ(id128);
    REQ(comm_out);
    return guard([&] { *comm_out = nccl_comm_init(id128, nranks, rank, device); });
}
int aero_nccl_comm_destroy(void* comm) {
    return guard([&] { nccl_comm_destroy(comm); });
}

// ---- CodState --------------------------------------------------------------
struct aero_cod {
    CodEngine* e;
};
int aero_cod_create(int32_t dx, int32_t dy, double eps, double theta, int64_t window,
                    uint64_t seed, uint64_t stream, int32_t device, aero_cod** out) {
    REQ(out);
    return guard([&] {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw CudaError("no CUDA device: the AeroSketch B200 path has no CPU fallback");
        *out = new aero_cod{new CodEngine(dx, dy, eps, theta, window, seed, stream, device)};
    });
}
int aero_cod_destroy(aero_cod* h) {
    if (!h) return AERO_OK;
    return guard([&] {
        delete h->e;
        delete h;
    });
}
int aero_cod_update_block(aero_cod* h, const double* xs, const double* ys, int64_t n,
                          const int64_t* t, aero_event* log_out) {
    REQ(h);
    return guard([&] { h->e->update_block(xs, ys, n, t, log_out); });
}
int aero_cod_query(aero_cod* h, double* astar, double* bstar) {
    REQ(h);
    return guard([&] { h->e->query(astar, bstar); });
}
int aero_cod_query_product(aero_cod* h, double* p) {
    REQ(h);
    return guard([&] { h->e->query_product(p); });
}
int aero_cod_info(aero_cod* h, int32_t* ell, int64_t* cols, int64_t* snaps, int64_t* clock) {
    REQ(h);
    h->e->info(ell, cols, snaps, clock);
    return AERO_OK;
}

int aero_cod_theta(aero_cod* h, double* theta) {
    REQ(h);
    REQ(theta);
    *theta = h->e->theta();
    return AERO_OK;
}
int aero_cod_set_theta(aero_cod* h, double theta) {
    REQ(h);
    return guard([&] { h->e->set_theta(theta); });
}

// ---- AdaptiveState -------------------------------------------------------------
struct aero_adaptive {
    AdaptiveEngine* e;
};
int aero_adaptive_create(int32_t dx, int32_t dy, double eps, double theta0, int64_t window,
                         uint64_t seed, uint64_t stream, int32_t device, aero_adaptive** out) {
    REQ(out);
    return guard([&] {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw CudaError("no CUDA device: the AeroSketch B200 path has no CPU fallback");
        *out = new aero_adaptive{new AdaptiveEngine(dx, dy, eps, theta0, window, seed, stream, device)};
    });
}
int aero_adaptive_destroy(aero_adaptive* h) {
    if (!h) return AERO_OK;
    return guard([&] {
        delete h->e;
        delete h;
    });
}
int aero_adaptive_update_block(aero_adaptive* h, const double* xs, const double* ys, int64_t n,
                               const int64_t* t, aero_event* log_out, int32_t* level_out) {
    REQ(h);
    if (n > 0) {
        REQ(xs);
        REQ(ys);
        REQ(t);
    }
    return guard([&] { h->e->update_block(xs, ys, n, t, log_out, level_out); });
}
int aero_adaptive_query(aero_adaptive* h, double* astar, double* bstar) {
    REQ(h);
    return guard([&] { h->e->main().query(astar, bstar); });
}
int aero_adaptive_query_product(aero_adaptive* h, double* p) {
    REQ(h);
    return guard([&] { h->e->main().query_product(p); });
}
int aero_adaptive_info(aero_adaptive* h, int32_t* level, double* theta_main, double* theta_aux,
                       int64_t* snaps_main, int64_t* snaps_aux) {
    REQ(h);
    if (level) *level = h->e->level();
    if (theta_main) *theta_main = h->e->main().theta();
    if (theta_aux) *theta_aux = h->e->aux().theta();
    if (snaps_main) *snaps_main = h->e->main().snap_count();
    if (snaps_aux) *snaps_aux = h->e->aux().snap_count();
    return AERO_OK;
}

// ---- AERO files ------------------------------------------------------------------
struct aero_file {
    AeroFile* f;
};
int aero_file_open(const char* path, aero_file** out, int32_t* d, uint64_t* n_header) {
    REQ(path);
    REQ(out);
    return guard([&] {
        AeroFile* f = new AeroFile(path);
        if (d) *d = (int32_t)f->d();
        if (n_header) *n_header = f->n_header();
        *out = new aero_file{f};
    });
}
int aero_file_read(aero_file* h, double* rows, int64_t max_rows, int64_t* got) {
    REQ(h);
    REQ(got);
    if (max_rows > 0) REQ(rows);
    return guard([&] { *got = h->f->read(rows, max_rows); });
}
int aero_file_close(aero_file* h) {
    if (!h) return AERO_OK;
    delete h->f;
    delete h;
    return AERO_OK;
}
int aero_file_write(const char* path, const double* rows, int64_t n, int32_t d) {
    REQ(path);
    if (n > 0) REQ(rows);
    return guard([&] { aero_file_write(std::string(path), rows, n, d); });
}
int aero_update_from_file(aero_sketch* h, const char* path, int64_t t0, int64_t chunk_rows,
                          aero_event* log_out, int64_t log_cap, int64_t* rows_out) {
    REQ(h);
    REQ(path);
    return guard([&] {
        const int64_t n = aero_file_update(*h->s, path, t0, chunk_rows, log_out, log_cap);
        if (rows_out) *rows_out = n;
    });
}

// ---- generator -----------------------------------------------------------------
int aero_gen_rows_device(const aero_gen_params* p, int64_t t0, int64_t n, double* out_device,
                         int32_t device) {
    REQ(p);
    REQ(out_device);
    return guard([&] { gen_rows_device(*p, t0, n, out_device, device); });
}

}  // extern "C"
