/*
 * aero_b200.h -- C-ABI of the B200-native AeroSketch update path.
 *
 * Drop-in boundary for the reference C++ sketch API (arXiv 2601.02019,
 * /root/reference/proj/include/aero). The reference has no FFI layer of its
 * own; each entry point below replaces one reference member function, cited
 * as file:line. All pointers are HOST pointers unless the name ends in
 * _device. Matrices are row-major with an explicit leading dimension.
 * Every call returns a status code (0 = ok) mirroring the reference's
 * exception taxonomy (errors.hpp:15-33); aero_last_error() gives the text.
 * There is no CPU fallback: without a CUDA device every compute entry point
 * returns AERO_CUDA_ERROR.
 */
#ifndef AERO_B200_H
#define AERO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (errors.hpp:15-33) */
#define AERO_OK 0
#define AERO_INVALID_INPUT 1        /* aero::InvalidInput  */
#define AERO_FORMAT_ERROR 2         /* aero::FormatError   */
#define AERO_PROTOCOL_ERROR 3       /* aero::ProtocolError */
#define AERO_ORACLE_CAP_EXCEEDED 4  /* aero::OracleCapExceeded */
#define AERO_CUDA_ERROR 10
#define AERO_INTERNAL_ERROR 11

/* threshold modes */
#define AERO_THETA_FIXED 0  /* AeroState: theta set by aero_set_theta / per-row array */
#define AERO_THETA_ATTP 1   /* AttpState (attp.hpp:21-26): theta = eps * running ||A||_F^2 */

/* flags */
#define AERO_FLAG_EXACT 1   /* no speculative row batching (one row per device step) */
#define AERO_FLAG_PROFILE 2 /* time the batched G.X products with CUDA events */
/* random projections from the host: the start vectors of every power_iteration
 * and the Pi of every simul_iter are drawn on the host by this library's
 * restatement of rng.hpp:54-78 (host libm) and uploaded, instead of being drawn
 * on the device (see aero_set_rng_fill for a caller-owned source) */
#define AERO_FLAG_HOST_RNG 4

typedef struct aero_sketch aero_sketch; /* opaque AeroState / AttpState */

typedef struct aero_cfg {
    int32_t d;          /* row dimension (sketch.cpp:22-31) */
    int32_t ell;        /* 0: ell = ceil(2/eps) (sketch.cpp:30) */
    double eps;         /* (0, 1] */
    double theta;       /* initial threshold >= 0 */
    double eps_si;      /* simul_iter accuracy; 0 -> 0.4 (sketch.cpp:23) */
    uint64_t seed;      /* RngState(seed, stream) of the sketch (rng.hpp:45-48) */
    uint64_t stream;
    int32_t device;     /* CUDA device ordinal */
    int32_t theta_mode; /* AERO_THETA_FIXED or AERO_THETA_ATTP */
    int32_t flags;      /* AERO_FLAG_* */
    int32_t max_batch;  /* speculative batch rows (0 = auto) */
    double delta;       /* probability amplification bound in (0, 1) (sketch.hpp:44-46); 0 = none.
                           AttpState with delta amplifies every update (attp.hpp:24) */
} aero_cfg;

/* per-row event record (UpdateStats, sketch.hpp:33-39, plus the trace the
 * parity tests compare); same layout as the oracle's Event */
typedef struct aero_event {
    int64_t t;
    int64_t forks_before, forks_after;
    int32_t rows_after, reduced, gate_fired, dumped;
    int32_t doubling_steps, simul_calls, xi, k_last;
    double theta, sigma1_sq, tail_sq;
} aero_event;

typedef struct aero_info {
    int32_t d, ell, rows;       /* rows = residual buffer rows */
    int64_t clock, last_dump_t; /* sketch.hpp:74,86 */
    int64_t forks;              /* RngState fork counter */
    int64_t snaps;              /* snapshot queue length */
    int64_t snap_cols;          /* sum of snapshot widths (xi) in the queue */
    double theta, fro_mass;     /* fro_mass: AttpState::fro_mass (attp.hpp:34) */
    int64_t device_rows_processed, device_batches, device_mispredicts;
    /* batch-ending causes: predicted fire but the gate did not; predicted no
     * fire but it did; a larger doubling rank was needed; a dump */
    int64_t end_nofire, end_fired, end_doubling, end_dump;
} aero_info;

/* ---- AeroState / AttpState --------------------------------------------- */
/* AeroState(d, eps, theta, rng) (sketch.cpp:22-31); AttpState(d, eps, rng)
 * when theta_mode == AERO_THETA_ATTP (attp.hpp:17-19) */
int aero_create(const aero_cfg* cfg, aero_sketch** out);
int aero_destroy(aero_sketch* h);
/* AeroState::set_theta (sketch.cpp:33-36) */
int aero_set_theta(aero_sketch* h, double theta);
/* performance hint, no semantic effect: `share` sketches run concurrently on
 * this GPU (e.g. co-hosted distributed sites); their persistent cooperative
 * iterate kernels then use at most 1/share of the resident CTAs each */
int aero_set_grid_share(aero_sketch* h, int32_t share);
/* Caller-owned random projections (north star: "projection
 * matrices passed in through the FFI"). The sketch consumes one RngState fork
 * per power_iteration (sketch.cpp:99, linalg.cpp:106-108: first r Gaussians)
 * and per simul_iter (sketch.cpp:53, linalg.cpp:141: the r x k Pi, row-major,
 * i.e. the first r*k Gaussians). The library asks for them as
 *   fill(ctx, n, out, count): out[0..count) = the first `count` Gaussians of
 *   fork #n (n >= 1) of the sketch's RngState(seed, stream) (rng.hpp:54-57),
 * returning 0 on success (nonzero -> AERO_INVALID_INPUT from the update).
 * fill is called from library threads, concurrently for distinct forks.
 * fn == NULL reverts to the default (device draws, or AERO_FLAG_HOST_RNG). */
typedef int (*aero_rng_fill)(void* ctx, uint64_t fork_index, double* out, int64_t count);
int aero_set_rng_fill(aero_sketch* h, aero_rng_fill fn, void* ctx);
/* n sequential AeroState::update / AttpState::update calls (sketch.cpp:82-141,
 * attp.hpp:21-26). t: n strictly increasing timestamps > clock. theta_per_row
 * (nullable, fixed mode only) sets the threshold before each row. log_out
 * (nullable) receives one aero_event per row. */
int aero_update_block(aero_sketch* h, const double* rows, int64_t n, int64_t ld, const int64_t* t,
                      const double* theta_per_row, aero_event* log_out);
/* n sequential AeroState::update_amplified calls (sketch.cpp:45-48; needs
 * cfg.delta > 0, else AERO_INVALID_INPUT before any row is absorbed) */
int aero_update_block_amplified(aero_sketch* h, const double* rows, int64_t n, int64_t ld,
                                const int64_t* t, const double* theta_per_row, aero_event* log_out);
/* same, rows already resident in device memory (ld in elements). The rows
 * are read on aero_stream(h): the caller must order their producer before it
 * (cudaStreamWaitEvent on aero_stream(h), or a completed producer stream). */
int aero_update_block_device(aero_sketch* h, const double* rows_device, int64_t n, int64_t ld,
                             const int64_t* t, const double* theta_per_row, aero_event* log_out);
/* AeroState::query(lb, ub) (sketch.cpp:143-160): ell x d row-major */
int aero_query(aero_sketch* h, int64_t lb, int64_t ub, double* out_ell_by_d);
/* the restored Gram before the final shrink (d x d row-major, symmetric) */
int aero_query_gram(aero_sketch* h, int64_t lb, int64_t ub, double* out_d_by_d);
/* AeroState::residual() (sketch.hpp:77): rows x d row-major */
int aero_residual(aero_sketch* h, double* out, int64_t max_rows);
/* snapshot queue access (sketch.hpp:78-79; callers pop it: sliding_window.cpp:59-65,
 * distributed.cpp:74-77). z: d x xi row-major, m: xi x d row-major (nullable). */
int aero_snap_count(aero_sketch* h, int64_t* count);
int aero_snap_info(aero_sketch* h, int64_t idx, int32_t* xi, int64_t* s, int64_t* t, double* theta);
int aero_snap_get(aero_sketch* h, int64_t idx, double* z, double* m);
int aero_snap_pop_front(aero_sketch* h);
/* AeroState::last_update_stats (sketch.hpp:80) as an event record */
int aero_last_stats(aero_sketch* h, aero_event* out);
int aero_get_info(aero_sketch* h, aero_info* out);
/* wait for all device work of this sketch */
int aero_synchronize(aero_sketch* h);
/* the cudaStream_t this sketch launches its kernels on */
void* aero_stream(aero_sketch* h);
/* AERO_FLAG_PROFILE: CUDA-event time, launches, useful flops (sum over the
 * active job columns of 2 r_j^2 k_j) and compulsory bytes of the batched
 * power/subspace-iteration products (the dominant kernel), plus batch counts */
typedef struct aero_profile {
    double product_ms;
    int64_t product_launches;
    double product_flops, product_bytes;
    double iterate_ms;   /* init + products + normalizations */
    double reduce_ms;    /* FD reduce (eigensolver + rotation) */
    int64_t reduces;
} aero_profile;
int aero_get_profile(aero_sketch* h, aero_profile* out);
int aero_reset_profile(aero_sketch* h);

/* ---- AttpState::query(t) (attp.hpp:29-32): prefix sketch at time t ---- */
int aero_attp_query(aero_sketch* h, int64_t t, double* out_ell_by_d);

/* ---- MlState: sliding-window multi-level sketch
 * (sliding_window.hpp:39-81, sliding_window.cpp:15-156) ---------------- */
typedef struct aero_ml aero_ml;
typedef struct aero_ml_query_result {
    int32_t level, fallback, heavy_used, _pad;
    int64_t xi_sum;
} aero_ml_query_result;
typedef struct aero_ml_info {
    int32_t d, ell, levels, _pad;
    int64_t n, cap, clock, norm_warnings, stored_floats;
    double window_mass;
} aero_ml_info;
int aero_ml_create(int32_t d, int64_t window, double r_max, double eps, uint64_t seed,
                   uint64_t stream, int32_t device, aero_ml** out);
/* MlState(d, n, r_max, eps, rng, delta) with amplified level updates
 * (sliding_window.cpp:15-30, 90-91) */
int aero_ml_create_amplified(int32_t d, int64_t window, double r_max, double eps, double delta,
                             uint64_t seed, uint64_t stream, int32_t device, aero_ml** out);
int aero_ml_destroy(aero_ml* h);
int aero_ml_update_block(aero_ml* h, const double* rows, int64_t n, int64_t ld, const int64_t* t);
int aero_ml_update_block_device(aero_ml* h, const double* rows_device, int64_t n, int64_t ld,
                                const int64_t* t);
int aero_ml_query(aero_ml* h, double* out_ell_by_d, aero_ml_query_result* res);
int aero_ml_get_info(aero_ml* h, aero_ml_info* out);
double aero_ml_theta(aero_ml* h, int32_t level);
/* level j's AeroState (borrowed handle, owned by the MlState) */
aero_sketch* aero_ml_level(aero_ml* h, int32_t level);
int aero_ml_heavy_count(aero_ml* h, int32_t level, int64_t* count);
int aero_ml_heavy_get(aero_ml* h, int32_t level, int64_t idx, double* row, int64_t* s, int64_t* t);

/* ---- distributed: site -> coordinator merge (distributed.hpp:23-135,
 * distributed.cpp:16-269), one site per GPU ------------------------------ */
/* Norm-only replay of the FroMass / broadcast protocol (distributed.cpp:31-69,
 * 107-123, 201-239): given every site's squared row norms (m x T, row-major),
 * returns each site's threshold per tick (m x T) and the protocol byte count
 * of the mass messages and broadcasts. Pure host integer/fp64 logic. */
int aero_dist_theta_schedule(int32_t m, int64_t T, double eps, int64_t latency,
                             const double* sq_norms, double* theta_out, int64_t* mass_bytes,
                             int64_t* broadcasts);
/* the same replay, streaming: state persists across calls; advance() consumes
 * the next T ticks of every site's squared norms (m x T row-major) */
typedef struct aero_dist_protocol aero_dist_protocol;
int aero_dist_protocol_create(int32_t m, double eps, int64_t latency, aero_dist_protocol** out);
/* sliding-window protocol (SiteState with window, distributed.cpp:33-55,
 * 27-30, 107-123): exact per-site window mass, signed FroMass deltas,
 * theta = eps * own window mass. window = 0 is the whole-stream protocol. */
int aero_dist_protocol_create_window(int32_t m, double eps, int64_t latency, int64_t window,
                                     aero_dist_protocol** out);
int aero_dist_protocol_destroy(aero_dist_protocol* h);
int aero_dist_protocol_advance(aero_dist_protocol* h, int64_t T, const double* sq_norms,
                               double* theta_out);
int aero_dist_protocol_info(aero_dist_protocol* h, int64_t* ticks, int64_t* mass_bytes,
                            int64_t* broadcasts, double* f_hat);
/* squared norms of n device rows (row-major, ld) into host memory (K1) */
int aero_row_sq_norms_device(const double* rows_device, int64_t n, int64_t ld, int32_t d,
                             int32_t device, double* out_host);
typedef struct aero_coord aero_coord;
/* coordinator accumulator B (d x d fp64) on `device`; nccl_comm is an
 * ncclComm_t (or NULL for single-process use) */
int aero_coord_create(int32_t d, int32_t m, int32_t device, void* nccl_comm, aero_coord** out);
/* CoordinatorState(d, m, window_mode) (distributed.hpp:78-105) with the
 * simulator's delivery latency (distributed.cpp:226-239): window > 0 keeps a
 * contribution live from tick t + latency until its Expire is delivered at
 * t + window + latency (distributed.cpp:87-97, 137-144); absorb() then also
 * counts the Expire messages' bytes. */
int aero_coord_create_window(int32_t d, int32_t m, int32_t device, void* nccl_comm, int64_t window,
                             int64_t latency, aero_coord** out);
int aero_coord_destroy(aero_coord* h);
/* CoordinatorState::receive(SnapshotUpdate) for every snapshot queued in the
 * site sketch (distributed.cpp:124-136), popping them (distributed.cpp:74-77);
 * returns the protocol bytes 8*(d*xi + xi*d) + 16 per message */
int aero_coord_absorb_snapshots(aero_coord* h, aero_sketch* site, int64_t* bytes);
/* probe_gram (distributed.cpp:159-173): this rank's absorbed contributions
 * plus the residual Grams of its `nsites` site sketches, summed over ranks with
 * ncclReduce to `root`; on root, shrink_to_sketch(B, ell) -> out (ell x d
 * row-major, nullable) and the d x d Gram (nullable) */
int aero_coord_probe(aero_coord* h, aero_sketch* const* sites, int32_t nsites, int32_t root,
                     int32_t ell, double* out_ell_by_d, double* out_gram);
/* shrink_to_sketch (sketch.cpp:167-178) of a merged d x d Gram
 * given in host memory, on the coordinator's device -> out (ell x d): the
 * root's last step when the per-rank Grams were summed over a process group
 * without NCCL (gloo) */
int aero_coord_shrink(aero_coord* h, const double* gram, int32_t ell, double* out);
/* NCCL helpers so callers need no NCCL headers: 128-byte unique id */
int aero_nccl_get_unique_id(char* id128);
int aero_nccl_comm_init(const char* id128, int32_t nranks, int32_t rank, int32_t device,
                        void** comm_out);
int aero_nccl_comm_destroy(void* comm);

/* ---- CodState: sliding-window AMM (amm.hpp:35-69, amm.cpp:27-122) ----- */
typedef struct aero_cod aero_cod;
int aero_cod_create(int32_t dx, int32_t dy, double eps, double theta, int64_t window,
                    uint64_t seed, uint64_t stream, int32_t device, aero_cod** out);
int aero_cod_destroy(aero_cod* h);
int aero_cod_update_block(aero_cod* h, const double* xs, const double* ys, int64_t n,
                          const int64_t* t, aero_event* log_out);
/* CodState::query: a* (dx x ell) and b* (dy x ell), row-major */
int aero_cod_query(aero_cod* h, double* astar, double* bstar);
int aero_cod_query_product(aero_cod* h, double* p_dx_by_dy);
int aero_cod_info(aero_cod* h, int32_t* ell, int64_t* cols, int64_t* snaps, int64_t* clock);
/* CodState::theta / set_theta (amm.hpp:52-53, amm.cpp:38-41) */
int aero_cod_theta(aero_cod* h, double* theta);
int aero_cod_set_theta(aero_cod* h, double theta);

/* ---- AdaptiveState: main/aux CodState pair with queue-length-driven
 * threshold doubling / halving (amm.hpp:71-93, amm.cpp:131-161).
 * aero_adaptive_create mirrors AdaptiveState(d_x, d_y, eps, theta0, n,
 * RngState(seed, stream)); update_block = n sequential update(x, y, i) calls
 * (xs n x dx, ys n x dy row-major, host); log_out (nullable) receives main's
 * per-row events, level_out (nullable) level() after each row. Query and
 * product come from the main sketch (amm.hpp:79). */
typedef struct aero_adaptive aero_adaptive;
int aero_adaptive_create(int32_t dx, int32_t dy, double eps, double theta0, int64_t window,
                         uint64_t seed, uint64_t stream, int32_t device, aero_adaptive** out);
int aero_adaptive_destroy(aero_adaptive* h);
int aero_adaptive_update_block(aero_adaptive* h, const double* xs, const double* ys, int64_t n,
                               const int64_t* t, aero_event* log_out, int32_t* level_out);
int aero_adaptive_query(aero_adaptive* h, double* astar, double* bstar);
int aero_adaptive_query_product(aero_adaptive* h, double* p_dx_by_dy);
/* level(), main().theta(), aux().theta(), main().snaps().size(), aux().snaps().size() */
int aero_adaptive_info(aero_adaptive* h, int32_t* level, double* theta_main, double* theta_aux,
                       int64_t* snaps_main, int64_t* snaps_aux);

/* ---- AERO binary stream files (streams.cpp:105-168, streams.hpp:45-47:
 * load_stream / save_stream with StreamFormat::Aero): "AERO", version 0x01,
 * u32 d, u64 n (0 = until EOF), n rows of d LE fp64. Read in chunks (the
 * configs' inputs do not fit in memory); FormatError (AERO_FORMAT_ERROR) for
 * bad magic / version, truncated header or row, zero dimension, non-finite
 * value -- raised by the chunk that holds it. */
typedef struct aero_file aero_file;
int aero_file_open(const char* path, aero_file** out, int32_t* d, uint64_t* n_header);
/* next rows (max_rows x d row-major) -> *got (0 at the end) */
int aero_file_read(aero_file* h, double* rows, int64_t max_rows, int64_t* got);
int aero_file_close(aero_file* h);
int aero_file_write(const char* path, const double* rows, int64_t n, int32_t d);
/* stream a file through a sketch: row q gets t0 + q; chunk k+1 is read into a
 * pinned buffer by a reader thread while chunk k is absorbed (n sequential
 * updates, like aero_update_block). log_out (nullable) holds log_cap events;
 * *rows_out = rows absorbed. */
int aero_update_from_file(aero_sketch* h, const char* path, int64_t t0, int64_t chunk_rows,
                          aero_event* log_out, int64_t log_cap, int64_t* rows_out);

/* ---- stream generators (BASELINE.json configs; DESIGN.md GENERATOR spec) */
typedef struct aero_gen_params {
    int32_t d, k, k2, _pad;
    double rho, noise, r_max, rho2, scale2;
    uint64_t seed, stream, basis_stream;
    int64_t drift_period;
} aero_gen_params;
/* rows t0 .. t0+n-1 into device memory (n x d row-major) */
int aero_gen_rows_device(const aero_gen_params* p, int64_t t0, int64_t n, double* out_device,
                         int32_t device);

/* ---- misc ---------------------------------------------------------------- */
const char* aero_last_error(void);  /* thread-local text of the last failure */
const char* aero_version(void);
/* device kernels launched by this library so far (all handles, this process) */
int64_t aero_kernel_launches(void);
/* symmetric eigensolver used by the FD reduce and the query shrink (test
 * hook; linalg.cpp:60-77 semantics): a is n x n row-major (symmetrized),
 * w descending, v columns = eigenvectors sign-fixed; device_ms (nullable)
 * receives the device time of the solve */
int aero_eigh(int32_t n, const double* a, double* w, double* v, double* device_ms);
/* The iteration product Y = G X (test hook): mode 0 = int8 tensor cores by
 * exact slicing (ozaki.cu), mode 1 = fp64 DMMA (product.cu). g is r x r symmetric, x is r x n column-major
 * (column j = x + j*r), colmask (nullable) gives each column's prefix length
 * (entries of x at k >= colmask[j] are treated as 0; output rows i >=
 * colmask[j] are 0); y is r x n column-major; device_ms (nullable) receives
 * the mean device time of one product over 20 launches after a warm-up
 * (mode 0: slicing of x, MMA and split-K sum; the slicing of g is done once
 * before, as the engine does once per batch). */
int aero_dev_product(int32_t r, int32_t n, const double* g, const double* x, const int32_t* colmask,
                     int32_t mode, double* y, double* device_ms);
/* RngState draws on the device (test hook): count gaussians of fork #fork of
 * RngState(seed, stream) (fork 0 = the root), to host memory */
int aero_rng_gaussians(uint64_t seed, uint64_t stream, int64_t fork, int64_t count, double* out);
/* the same draws by the host restatement AERO_FLAG_HOST_RNG uses (rng.hpp:60-78
 * with the host libm; needs no GPU) */
int aero_rng_gaussians_host(uint64_t seed, uint64_t stream, int64_t fork, int64_t count, double* out);

#ifdef __cplusplus
}
#endif
#endif /* AERO_B200_H */
