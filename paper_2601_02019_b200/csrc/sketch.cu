// AeroState engine on one B200 (see sketch.hpp). Control flow restates
// /root/reference/proj/src/sketch.cpp:82-141 row by row; device work is
// batched speculatively across rows.
#include <chrono>
#include <cstdio>
#include <algorithm>
#include <cmath>
#include <cstring>

#include "aero_common.cuh"
#include "sketch.hpp"

namespace aero_b200 {

void DeviceBuf::alloc(size_t count) {
    if (count <= n && p) return;
    release();
    AERO_CUDA(cudaMalloc(&p, sizeof(double) * std::max<size_t>(count, 1)));
    n = count;
}
void DeviceBuf::release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
}

namespace {
int power_iter_count(int d) {  // sketch.cpp:16-18
    return static_cast<int>(std::ceil(std::log2(static_cast<double>(std::max(d, 2))))) + 1;
}
int simul_q(int d, double eps_si) {  // linalg.cpp:138-139
    return static_cast<int>(
        std::ceil(1.0 * std::log2(static_cast<double>(std::max(d, 2))) / eps_si));
}
template <typename T>
T* pinned(size_t n) {
    T* p = nullptr;
    AERO_CUDA(cudaMallocHost(&p, sizeof(T) * std::max<size_t>(n, 1)));
    return p;
}
template <typename T>
T* dev_alloc(size_t n) {
    T* p = nullptr;
    AERO_CUDA(cudaMalloc(&p, sizeof(T) * std::max<size_t>(n, 1)));
    return p;
}
}  // namespace

__global__ void k_sym_fill(int r0, int B, double* G, int ldg) {
    // G[r0+j, i] = G[i, r0+j] for i < r0 (lower-left block of the new rows)
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)r0 * B) return;
    const int i = (int)(e % r0), j = (int)(e / r0);
    G[(r0 + j) + (int64_t)i * ldg] = G[i + (int64_t)(r0 + j) * ldg];
}
__global__ void k_inv_sqrt_clamp(const double* lam, int k, double* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double lmax = 0.0;
    for (int i = 0; i < k; ++i) lmax = fmax(lmax, lam[i]);
    for (int i = 0; i < k; ++i) {
        const double l = lam[i];
        out[i] = (l > 0.0 && l > 1e-14 * lmax) ? 1.0 / sqrt(l) : 0.0;
    }
}
__global__ void k_sqrt_clamp(const double* lam, int k, double* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < k) out[i] = sqrt(fmax(lam[i], 0.0));
}
__global__ void k_identity_cols(int d, int xi, double* z, int ld) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)d * xi) return;
    const int i = (int)(e % d), j = (int)(e / d);
    z[i + (int64_t)j * ld] = (i == j) ? 1.0 : 0.0;
}

Sketch::Sketch(const aero_cfg& cfg) {
    if (cfg.d < 1) throw InvalidInput("AeroState: d must be >= 1");
    if (!(cfg.eps > 0.0 && cfg.eps <= 1.0)) throw InvalidInput("AeroState: eps out of (0,1]");
    if (cfg.theta < 0.0) throw InvalidInput("AeroState: theta must be >= 0");
    d_ = cfg.d;
    eps_ = cfg.eps;
    ell_ = cfg.ell > 0 ? cfg.ell : static_cast<int>(std::ceil(2.0 / cfg.eps));  // sketch.cpp:30
    eps_si_ = cfg.eps_si > 0.0 ? cfg.eps_si : 0.4;                              // sketch.cpp:23
    if (cfg.delta != 0.0 && !(cfg.delta > 0.0 && cfg.delta < 1.0))
        throw InvalidInput("AeroState: delta out of (0, 1)");  // sketch.cpp:28-29
    delta_ = cfg.delta;
    if (!(eps_si_ > 0.0 && eps_si_ < 1.0)) throw InvalidInput("AeroState: eps_si out of (0,1)");
    theta_ = cfg.theta;
    seed_ = cfg.seed;
    stream_ = cfg.stream;
    mode_ = cfg.theta_mode;
    exact_ = (cfg.flags & AERO_FLAG_EXACT) != 0;
    profiling = (cfg.flags & AERO_FLAG_PROFILE) != 0;
    host_rng_default_ = (cfg.flags & AERO_FLAG_HOST_RNG) != 0;
    if (host_rng_default_) rng_.set_host();
    dev_ = cfg.device;
    cap_ = 2 * ell_;
    kp_ = power_iter_count(d_);
    q_ = simul_q(d_, eps_si_);
    max_batch_ = cfg.max_batch > 0 ? cfg.max_batch : 192;
    cfg_max_batch_ = cfg.max_batch;
    cur_batch_ = std::min(64, max_batch_);
    AERO_CUDA(cudaSetDevice(dev_));
    AERO_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    C_.alloc((size_t)d_ * cap_);
    C2_.alloc((size_t)d_ * cap_);
    G_.alloc((size_t)cap_ * cap_);
    fill_zero(st_, G_.p, (int64_t)cap_ * cap_);
    ldx_ = cap_;
    // job columns: a batch's 3 per row, or one simul_iter at the largest
    // doubling rank kmax = min(ell, d) (sketch.cpp:112-138)
    ncols_ = std::max({3 * max_batch_, 64, std::min(ell_, d_)});
    X_.alloc((size_t)ldx_ * ncols_);
    Y_.alloc((size_t)ldx_ * ncols_);
    H_.alloc((size_t)ldx_ * ncols_);
    ws_.alloc(product_workspace_doubles(cap_, std::max(ncols_, cap_ / 4)));  // split-K partials
    sig_.alloc(ncols_);
    vr_.alloc((size_t)ncols_ * kv_);
    small_.alloc(4 * 64 * 64 + 64);
    if (i8_ && cap_ >= i8_min_rows_) oz_.reserve(cap_, ncols_);
    status_d_ = dev_alloc<int>(ncols_);
    clamp_d_ = dev_alloc<int>(ncols_);
    colmask_d_ = dev_alloc<int>(ncols_);
    jobs_d_ = dev_alloc<IterJob>(ncols_);
    jobs_h_ = pinned<IterJob>(ncols_);
    phase_d_ = dev_alloc<int>(2 * kMaxPhases);
    phase_h_ = pinned<int>(2 * kMaxPhases);
    bar_d_ = dev_alloc<unsigned>(1);
    colmask_h_ = pinned<int>(ncols_);
    sig_h_ = pinned<double>(std::max(ncols_, cap_));
    status_h_ = pinned<int>(ncols_);
    clamp_h_ = pinned<int>(ncols_);
    stage_rows_ = 4096;
    nrm_.alloc(2 * (size_t)stage_rows_);
    bad_d_ = dev_alloc<int>(2 * (size_t)stage_rows_);
    nrm_h_ = pinned<double>(2 * (size_t)stage_rows_);
    bad_h_ = pinned<int>(2 * (size_t)stage_rows_);
    AERO_CUDA(cudaStreamCreateWithFlags(&cs_, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
        AERO_CUDA(cudaEventCreateWithFlags(&ev_ready_[b], cudaEventDisableTiming));
        AERO_CUDA(cudaEventCreateWithFlags(&ev_free_[b], cudaEventDisableTiming));
    }
}

cudaEvent_t Sketch::ev_at(size_t i) {
    while (ev_pool_.size() <= i) {
        cudaEvent_t e;
        AERO_CUDA(cudaEventCreate(&e));
        ev_pool_.push_back(e);
    }
    return ev_pool_[i];
}

Sketch::~Sketch() {
    if (getenv("AERO_HOST_PROF") && host_syncs_ > 0)
        fprintf(stderr, "sketch host: process_rows wall %.1f ms, blocked in iterate syncs %.1f ms over %lld syncs (%.1f us/sync)\n",
                host_wall_s_ * 1e3, host_sync_s_ * 1e3, (long long)host_syncs_, host_sync_s_ * 1e6 / host_syncs_);
    cudaSetDevice(dev_);
    if (st_) cudaStreamSynchronize(st_);
    for (cudaEvent_t e : ev_pool_) cudaEventDestroy(e);
    for (Chunk* c : chunks_) {
        cudaFree(c->z);
        cudaFree(c->mt);
        delete c;
    }
    cudaFree(status_d_);
    cudaFree(phase_d_);
    cudaFree(bar_d_);
    cudaFreeHost(phase_h_);
    cudaFree(clamp_d_);
    cudaFree(colmask_d_);
    cudaFree(jobs_d_);
    cudaFree(bad_d_);
    if (cs_) {
        cudaStreamSynchronize(cs_);
        cudaStreamDestroy(cs_);
    }
    for (int b = 0; b < 2; ++b) {
        if (ev_ready_[b]) cudaEventDestroy(ev_ready_[b]);
        if (ev_free_[b]) cudaEventDestroy(ev_free_[b]);
    }
    cudaFreeHost(jobs_h_);
    cudaFreeHost(colmask_h_);
    cudaFreeHost(sig_h_);
    cudaFreeHost(status_h_);
    cudaFreeHost(clamp_h_);
    cudaFreeHost(nrm_h_);
    cudaFreeHost(bad_h_);
    if (st_) {
        eigh_forget(st_);
        cudaStreamDestroy(st_);
    }
}

void Sketch::set_theta(double th) {  // sketch.cpp:33-36
    if (th < 0.0) throw InvalidInput("AeroState: theta must be >= 0");
    theta_ = th;
}

uint64_t Sketch::fork_state0(uint64_t n) const {
    return rng_state0(seed_, fork_stream(stream_, n));
}

void Sketch::synchronize() { AERO_CUDA(cudaStreamSynchronize(st_)); }

void Sketch::set_rng_source(bool host, aero_rng_fill fn, void* ctx) {
    if (fn) rng_.set_callback(fn, ctx);
    else if (host) rng_.set_host();
    else rng_.set_device();
}

// ---------------------------------------------------------------- arena
Chunk* Sketch::arena_alloc(int xi, int* col) {
    if (chunks_.empty() || chunks_.back()->used + xi > chunks_.back()->cap) {
        Chunk* c = new Chunk;
        c->cap = std::max(xi, std::max(64, (int)std::min<int64_t>(1024, (int64_t)(1 << 24) / d_)));
        AERO_CUDA(cudaMalloc(&c->z, sizeof(double) * (size_t)d_ * c->cap));
        AERO_CUDA(cudaMalloc(&c->mt, sizeof(double) * (size_t)d_ * c->cap));
        chunks_.push_back(c);
    }
    Chunk* c = chunks_.back();
    *col = c->used;
    c->used += xi;
    c->live += xi;
    return c;
}
void Sketch::arena_release(const SnapRec& s) {
    s.chunk->live -= s.xi;
    while (!chunks_.empty() && chunks_.front()->live == 0 && chunks_.front() != chunks_.back()) {
        Chunk* c = chunks_.front();
        AERO_CUDA(cudaStreamSynchronize(st_));
        cudaFree(c->z);
        cudaFree(c->mt);
        delete c;
        chunks_.pop_front();
    }
}

// ---------------------------------------------------------------- append
// C'[:, r..r+B) <- rows; G[0:r+B, r:r+B] = C'^T C'_new; symmetric fill
void Sketch::append_rows(const double* dev_rows, int64_t B) {
    const int r0 = r_;
    AERO_CUDA(cudaMemcpyAsync(C_.p + (size_t)r0 * d_, dev_rows, sizeof(double) * d_ * B,
                              cudaMemcpyDeviceToDevice, st_));
    if (!gemm_big(st_, true, false, r0 + (int)B, (int)B, d_, C_.p, d_, C_.p + (size_t)r0 * d_, d_,
                  G_.p + (size_t)r0 * cap_, cap_, nullptr, ws_.p, ws_.n))
        dgemm(st_, true, false, r0 + (int)B, (int)B, d_, 1.0, C_.p, d_, C_.p + (size_t)r0 * d_, d_,
              0.0, G_.p + (size_t)r0 * cap_, cap_);
    if (r0 > 0) {
        const int64_t tot = (int64_t)r0 * B;
        k_sym_fill<<<(unsigned)((tot + 255) / 256), 256, 0, st_>>>(r0, (int)B, G_.p, cap_);
        AERO_LAUNCHED();
    }
}

// ---------------------------------------------------------------- reduce
// FD reduce of the full 2ell x d buffer (fd.cpp:13-29 via sketch.cpp:92-95):
// eig(C'C'^T) = U diag(sigma^2) U^T; new rows sqrt(sigma_i^2 - sigma_ell^2) v_i^T
// = (w_i u_i^T) C' with w_i = sqrt(s2_i)/sigma_i; keep max(ell-1, 1) rows.
void Sketch::reduce() {
    if (profiling) AERO_CUDA(cudaEventRecord(ev_at(0), st_));
    const int n = cap_;
    const int keep = std::max(ell_ - 1, 1);
    E_.alloc((size_t)n * n);
    ew_.alloc(n);
    fw_.alloc(n);
    copy_matrix(st_, n, n, G_.p, cap_, E_.p, n);
    eigh(st_, n, E_.p, n, ew_.p, 1, 0, keep);  // only the kept directions
    fd_weights(st_, ew_.p, n, ell_, keep, fw_.p);
    scale_columns(st_, n, keep, E_.p, n, fw_.p);
    if (!gemm_big(st_, false, false, d_, keep, n, C_.p, d_, E_.p, n, C2_.p, d_, nullptr, ws_.p, ws_.n))
        dgemm(st_, false, false, d_, keep, n, 1.0, C_.p, d_, E_.p, n, 0.0, C2_.p, d_);
    std::swap(C_.p, C2_.p);
    std::swap(C_.n, C2_.n);
    if (!gemm_big(st_, true, false, keep, keep, d_, C_.p, d_, C_.p, d_, G_.p, cap_, nullptr, ws_.p, ws_.n))
        dgemm(st_, true, false, keep, keep, d_, 1.0, C_.p, d_, C_.p, d_, 0.0, G_.p, cap_);
    r_ = keep;
    if (profiling) {
        AERO_CUDA(cudaEventRecord(ev_at(1), st_));
        AERO_CUDA(cudaEventSynchronize(ev_at(1)));
        float ms = 0.f;
        AERO_CUDA(cudaEventElapsedTime(&ms, ev_at(0), ev_at(1)));
        prof.reduce_ms += ms;
        prof.reduces++;
    }
}

// ---------------------------------------------------------------- iterate
void Sketch::run_iterate(int njobs, int R, int max_k) {
    int maxphase = 0, ncol_total = 0;
    for (int j = 0; j < njobs; ++j) {
        maxphase = std::max(maxphase, jobs_h_[j].nphase);
        ncol_total = std::max(ncol_total, jobs_h_[j].col + jobs_h_[j].k);
    }
    prepare_rng(njobs);
    AERO_CUDA(cudaMemcpyAsync(jobs_d_, jobs_h_, sizeof(IterJob) * njobs, cudaMemcpyHostToDevice, st_));
    AERO_CUDA(cudaMemcpyAsync(colmask_d_, colmask_h_, sizeof(int) * ncol_total,
                              cudaMemcpyHostToDevice, st_));
    // persistent launch when the phases are launch-latency bound (small products);
    // large products run as separate DMMA launches (measured faster there)
    double big = 0.0;
    for (int j = 0; j < njobs; ++j) big = std::max(big, (double)jobs_h_[j].r);
    const bool small_phases = big * big * (double)ncol_total < 1e8;
    // experimental (AERO_CTA_ITER=1): measured slower than the persistent
    // grid kernel at C3/C4 (G chunk loads are not yet double-buffered)
    static const bool use_cta = getenv("AERO_CTA_ITER") != nullptr;
    const bool cta_iter = persistent_ && use_cta && R > 96 && R <= 512 && max_k <= 2 && !(i8_ && R >= i8_min_rows_);
    if (persistent_ && ((R <= 96 && max_k <= 2) || cta_iter)) {
        // small buffer: one warp per job, all phases, G in shared memory;
        // medium buffer (<= 512): 4 jobs per CTA, G streamed through shared memory
        double flops = 0.0;
        for (int j = 0; j < njobs; ++j) flops += 2.0 * jobs_h_[j].r * (double)jobs_h_[j].r * jobs_h_[j].k * jobs_h_[j].nphase;
        if (profiling) AERO_CUDA(cudaEventRecord(ev_at(0), st_));
        iter_init(st_, jobs_d_, njobs, G_.p, cap_, X_.p, ldx_, R, status_d_, panel_d_);
        if (profiling) AERO_CUDA(cudaEventRecord(ev_at(2), st_));
        if (R <= 96)
            iterate_warp(st_, jobs_d_, njobs, G_.p, cap_, R, X_.p, ldx_, H_.p, status_d_, sig_.p, vr_.p, kv_,
                         clamp_d_, max_k);
        else
            iterate_cta(st_, jobs_d_, njobs, G_.p, cap_, R, X_.p, ldx_, H_.p, status_d_, sig_.p, vr_.p, kv_,
                        clamp_d_, max_k);
        if (profiling) {
            AERO_CUDA(cudaEventRecord(ev_at(3), st_));
            prof.product_launches++;
            prof.product_flops += flops;
        }
        maxphase = 1;
    } else if (i8_ && R >= i8_min_rows_ && persistent_ && max_k <= 4 && maxphase <= kMaxPhases) {
        // large buffers: all phases in one cooperative launch, products on the
        // int8 tensor cores (kernels.cu k_iterate_i8)
        oz_.prepare(st_, R, G_.p, cap_);
        double flops = 0.0;
        for (int p = 0; p < maxphase; ++p) {
            int ncol = 0;
            for (int j = 0; j < njobs; ++j)
                if (jobs_h_[j].nphase > p) {
                    ncol = std::max(ncol, jobs_h_[j].col + jobs_h_[j].k);
                    flops += 2.0 * jobs_h_[j].r * (double)jobs_h_[j].r * jobs_h_[j].k;
                }
            ncol = std::max(ncol, 1);
            phase_h_[p] = ncol;
            // effective slices of the phase's products (opt-in experiment, default
            // all slices everywhere): the last oz_tail_ phases of every job run on
            // all slices, the steering phases before them on oz_se_ (AERO_OZ_SE /
            // AERO_OZ_TAIL)
            int se = oz_se_;
            for (int j = 0; j < njobs && se < ozaki_slices(); ++j)
                if (jobs_h_[j].nphase > p && jobs_h_[j].nphase - 1 - p < oz_tail_) se = ozaki_slices();
            phase_h_[kMaxPhases + p] = ozaki_splits(oz_, ncol, ws_.n) | (se << 16);
        }
        oz_.reserve_x(phase_h_[0]);
        AERO_CUDA(cudaMemcpyAsync(phase_d_, phase_h_, sizeof(int) * 2 * kMaxPhases, cudaMemcpyHostToDevice, st_));
        if (profiling) AERO_CUDA(cudaEventRecord(ev_at(0), st_));
        iter_init(st_, jobs_d_, njobs, G_.p, cap_, X_.p, ldx_, R, status_d_, panel_d_);
        if (profiling) AERO_CUDA(cudaEventRecord(ev_at(2), st_));
        static int sms = 0;
        if (!sms) AERO_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev_));
        iterate_i8_persistent(st_, jobs_d_, njobs, maxphase, R, oz_, colmask_d_, X_.p, ldx_, H_.p, status_d_,
                              sig_.p, vr_.p, kv_, clamp_d_, ws_.p, phase_d_, phase_d_ + kMaxPhases, bar_d_, max_k,
                              sms);
        if (profiling) {
            AERO_CUDA(cudaEventRecord(ev_at(3), st_));
            prof.product_launches++;
            prof.product_flops += flops;
        }
        maxphase = 1;  // one timed region below
    } else if (max_k <= 4 && maxphase <= kMaxPhases && persistent_ && small_phases) {
        // all phases in one cooperative launch (kernels.cu k_iterate)
        const int kt = (R + 15) / 16;
        int max_tiles = 1;
        for (int p = 0; p < maxphase; ++p) {
            int ncol = 0;
            for (int j = 0; j < njobs; ++j)
                if (jobs_h_[j].nphase > p) ncol = std::max(ncol, jobs_h_[j].col + jobs_h_[j].k);
            max_tiles = std::max(max_tiles, ((ncol + 63) / 64) * ((R + 127) / 128));
        }
        // CTAs: one per job for the normalizations, ~8 K-splits per product tile
        // the split-K factors (hence every summation order, hence every
        // decision) follow the unshared grid; the launch may use fewer CTAs
        // (grid share: concurrent sketches), which then loop over the items
        const int grid_full = std::min(iterate_grid(R), std::max({njobs, 8 * max_tiles, 16}));
        const int grid = std::min(grid_full, std::max(16, iterate_grid(R) / grid_share_));
        double flops = 0.0;
        for (int p = 0; p < maxphase; ++p) {
            int ncol = 0;
            for (int j = 0; j < njobs; ++j)
                if (jobs_h_[j].nphase > p) {
                    ncol = std::max(ncol, jobs_h_[j].col + jobs_h_[j].k);
                    flops += 2.0 * jobs_h_[j].r * (double)jobs_h_[j].r * jobs_h_[j].k;
                }
            const int tiles = ((ncol + 63) / 64) * ((R + 127) / 128);
            int splits = std::max(1, std::min({grid_full / std::max(tiles, 1), 16, std::max(1, kt / 2)}));
            while (splits > 1 && (size_t)splits * R * ncol > ws_.n) --splits;
            phase_h_[p] = std::max(ncol, 1);
            phase_h_[kMaxPhases + p] = splits;
        }
        AERO_CUDA(cudaMemcpyAsync(phase_d_, phase_h_, sizeof(int) * 2 * kMaxPhases, cudaMemcpyHostToDevice, st_));
        if (profiling) AERO_CUDA(cudaEventRecord(ev_at(0), st_));
        iter_init(st_, jobs_d_, njobs, G_.p, cap_, X_.p, ldx_, R, status_d_, panel_d_);
        if (profiling) AERO_CUDA(cudaEventRecord(ev_at(2), st_));
        iterate_persistent(st_, jobs_d_, njobs, maxphase, R, G_.p, cap_, X_.p, ldx_, H_.p, status_d_, sig_.p,
                           vr_.p, kv_, clamp_d_, ws_.p, phase_d_, phase_d_ + kMaxPhases, bar_d_, max_k, grid);
        if (profiling) {
            AERO_CUDA(cudaEventRecord(ev_at(3), st_));
            prof.product_launches++;
            prof.product_flops += flops;
        }
        maxphase = 1;  // one timed region below
    } else {
    if (profiling) AERO_CUDA(cudaEventRecord(ev_at(0), st_));
    iter_init(st_, jobs_d_, njobs, G_.p, cap_, X_.p, ldx_, R, status_d_, panel_d_);
    // large buffers: G sliced once for all phases, products on the int8 tensor cores
    const bool i8 = i8_ && R >= i8_min_rows_;
    if (i8) oz_.prepare(st_, R, G_.p, cap_);
    for (int p = 0; p < maxphase; ++p) {
        int ncol = 0;
        double flops = 0.0;
        for (int j = 0; j < njobs; ++j)
            if (jobs_h_[j].nphase > p) {
                ncol = std::max(ncol, jobs_h_[j].col + jobs_h_[j].k);
                flops += 2.0 * jobs_h_[j].r * (double)jobs_h_[j].r * jobs_h_[j].k;
            }
        if (profiling) AERO_CUDA(cudaEventRecord(ev_at(2 + 2 * p), st_));
        // (fusing the split-K sum into the per-job normalization measured slower:
        // one CTA per job streams all partials -- profiles/round1_c2_steady_launches.txt)
        constexpr bool kFuseSplitK = false;
        int splits = 1;
        bool fast = true;
        if (i8) {
            oz_.product(st_, ncol, X_.p, ldx_, colmask_d_, Y_.p, ldx_, ws_.p, ws_.n);
        } else {
            fast = gemm_big(st_, false, false, R, ncol, R, G_.p, cap_, X_.p, ldx_, Y_.p, ldx_, colmask_d_,
                            ws_.p, ws_.n, &splits, kFuseSplitK && max_k <= 4);
            if (!fast)
                dgemm(st_, false, false, R, ncol, R, 1.0, G_.p, cap_, X_.p, ldx_, 0.0, Y_.p, ldx_,
                      colmask_d_);
        }
        if (profiling) {
            AERO_CUDA(cudaEventRecord(ev_at(3 + 2 * p), st_));
            prof.product_launches++;
            prof.product_flops += flops;
            prof.product_bytes += 8.0 * ((double)R * R + 2.0 * (double)R * ncol);
        }
        if (kFuseSplitK && fast && splits > 1 && max_k <= 4)  // split-K sum fused into the normalization
            iter_normalize_ws(st_, jobs_d_, njobs, p, X_.p, ldx_, ws_.p, R, ncol, splits, H_.p,
                              status_d_, sig_.p, vr_.p, kv_, clamp_d_, std::max(max_k, 1));
        else
            iter_normalize(st_, jobs_d_, njobs, p, X_.p, Y_.p, ldx_, H_.p, status_d_, sig_.p,
                           vr_.p, kv_, clamp_d_, std::max(max_k, 1));
    }
    }
    if (profiling) AERO_CUDA(cudaEventRecord(ev_at(1), st_));
    AERO_CUDA(cudaMemcpyAsync(sig_h_, sig_.p, sizeof(double) * ncol_total, cudaMemcpyDeviceToHost, st_));
    AERO_CUDA(cudaMemcpyAsync(status_h_, status_d_, sizeof(int) * njobs, cudaMemcpyDeviceToHost, st_));
    AERO_CUDA(cudaMemcpyAsync(clamp_h_, clamp_d_, sizeof(int) * njobs, cudaMemcpyDeviceToHost, st_));
    const auto hs0 = std::chrono::steady_clock::now();
    AERO_CUDA(cudaStreamSynchronize(st_));
    host_sync_s_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - hs0).count();
    host_syncs_++;
    if (profiling) {
        float ms = 0.f;
        AERO_CUDA(cudaEventElapsedTime(&ms, ev_at(0), ev_at(1)));
        prof.iterate_ms += ms;
        for (int p = 0; p < maxphase; ++p) {
            AERO_CUDA(cudaEventElapsedTime(&ms, ev_at(2 + 2 * p), ev_at(3 + 2 * p)));
            prof.product_ms += ms;
        }
    }
}

// simul_iter with k > 64 columns: same r-space iteration, host-driven phases
// with device GEMMs and the general eigensolver for the k x k Grams.
void Sketch::run_simul_large(int k, uint64_t fork, int r, int q) {
    const size_t kk = (size_t)k * k;
    qw_.alloc(3 * kk + 3 * (size_t)k);
    double* S = qw_.p;
    double* Tm = S + kk;
    double* lam = Tm + kk;
    double* sc = lam + k;
    if (vr_.n < kk) vr_.alloc(kk);
    if (k > ncols_) throw InvalidInput("simul_iter: k exceeds work capacity");
    jobs_h_[0] = IterJob{1, r, k, 0, q + 1, -1, fork_state0(fork), fork};
    for (int c = 0; c < k; ++c) colmask_h_[c] = r;
    prepare_rng(1);
    AERO_CUDA(cudaMemcpyAsync(jobs_d_, jobs_h_, sizeof(IterJob), cudaMemcpyHostToDevice, st_));
    AERO_CUDA(cudaMemcpyAsync(colmask_d_, colmask_h_, sizeof(int) * k, cudaMemcpyHostToDevice, st_));
    iter_init(st_, jobs_d_, 1, G_.p, cap_, X_.p, ldx_, r, status_d_, panel_d_);
    AERO_CUDA(cudaMemcpyAsync(status_h_, status_d_, sizeof(int), cudaMemcpyDeviceToHost, st_));
    AERO_CUDA(cudaStreamSynchronize(st_));
    if (status_h_[0] != JOB_ACTIVE) {
        for (int a = 0; a < k; ++a) sig_h_[a] = 0.0;
        return;
    }
    for (int p = 0; p <= q; ++p) {
        gemm_product(st_, r, k, r, G_.p, cap_, X_.p, ldx_, Y_.p, ldx_, colmask_d_, ws_.p, ws_.n);
        dgemm(st_, true, false, k, k, r, 1.0, X_.p, ldx_, Y_.p, ldx_, 0.0, S, k);
        eigh(st_, k, S, k, lam);
        k_inv_sqrt_clamp<<<1, 1, 0, st_>>>(lam, k, sc);
        AERO_LAUNCHED();
        scale_columns(st_, k, k, S, k, sc);  // T = W diag(lam^-1/2)
        if (p == q) dgemm(st_, false, false, r, k, k, 1.0, X_.p, ldx_, S, k, 0.0, H_.p, ldx_);
        dgemm(st_, false, false, r, k, k, 1.0, Y_.p, ldx_, S, k, 0.0, X_.p, ldx_);
    }
    dgemm(st_, true, false, k, k, r, 1.0, X_.p, ldx_, X_.p, ldx_, 0.0, vr_.p, k);
    eigh(st_, k, vr_.p, k, lam);
    k_sqrt_clamp<<<(k + 127) / 128, 128, 0, st_>>>(lam, k, sig_.p);
    AERO_LAUNCHED();
    AERO_CUDA(cudaMemcpyAsync(sig_h_, sig_.p, sizeof(double) * k, cudaMemcpyDeviceToHost, st_));
    AERO_CUDA(cudaStreamSynchronize(st_));
}

// ---------------------------------------------------------------- dump
// sketch.cpp:119-132: z = g V[:, :xi] = C'^T (H V); sign fix (linalg.cpp:150);
// m = (C'z)^T C'; C <- C' - (C'z) z^T; G <- G - 2PP^T + P (z^T z) P^T, P = C'z
void Sketch::dump_from_job(int col, int k, int xi, int64_t t, double theta, bool zero_buffer) {
    int ccol = 0;
    Chunk* ch = arena_alloc(xi, &ccol);
    double* z = ch->z + (size_t)ccol * d_;
    double* mt = ch->mt + (size_t)ccol * d_;
    const int r = r_;
    if (zero_buffer) {  // linalg.cpp:132-135: z = I(d, k), C' = 0 so m = 0
        const int64_t tot = (int64_t)d_ * xi;
        k_identity_cols<<<(unsigned)((tot + 255) / 256), 256, 0, st_>>>(d_, xi, z, d_);
        AERO_LAUNCHED();
        fill_zero(st_, mt, tot);
    } else {
        const int rl = r + (r & 1);  // even leading dimension (16-byte aligned columns)
        qy_.alloc((size_t)rl * xi * 2 + (size_t)xi * xi + 64);
        double* HV = qy_.p;
        double* P = HV + (size_t)rl * xi;
        double* ZZ = P + (size_t)rl * xi;
        const double* vr = (k > 64) ? vr_.p : vr_.p + (size_t)col * kv_;
        auto big = [&](bool ta, bool tb, int M, int N, int K, const double* A, int lda,
                       const double* Bm, int ldb, double* Y, int ldy) {
            if (!gemm_big(st_, ta, tb, M, N, K, A, lda, Bm, ldb, Y, ldy, nullptr, ws_.p, ws_.n))
                dgemm(st_, ta, tb, M, N, K, 1.0, A, lda, Bm, ldb, 0.0, Y, ldy);
        };
        dgemm(st_, false, false, r, xi, k, 1.0, H_.p + (size_t)col * ldx_, ldx_, vr, k, 0.0, HV, rl);
        big(false, false, d_, xi, r, C_.p, d_, HV, rl, z, d_);               // z = C'^T (H V)
        fix_column_signs(st_, d_, xi, z, d_, nullptr);
        big(true, false, r, xi, d_, C_.p, d_, z, d_, P, rl);                 // P = C' z
        big(false, false, d_, xi, r, C_.p, d_, P, rl, mt, d_);               // m^T = C'^T P
        dgemm(st_, false, true, d_, r, xi, -1.0, z, d_, P, rl, 1.0, C_.p, d_);  // C' -= P z^T
        big(true, false, xi, xi, d_, z, d_, z, d_, ZZ, xi);                  // z^T z
        add_identity(st_, xi, ZZ, xi, -2.0);
        dgemm(st_, false, false, r, xi, xi, 1.0, P, rl, ZZ, xi, 0.0, HV, rl);   // P (z^T z - 2I)
        dgemm(st_, false, true, r, r, xi, 1.0, HV, rl, P, rl, 1.0, G_.p, cap_);
        symmetrize(st_, r, G_.p, cap_);
    }
    SnapRec s{xi, last_dump_t_ + 1, t, theta, ch, ccol};
    last_dump_t_ = t;
    snaps_.push_back(s);
}

// ---------------------------------------------------------------- amplification
// sketch.cpp:55-79 in Gram (r-space) form. Candidate h: simul_iter at eps_si =
// 0.2 gives H (r x k), V (k x k), sigma; z = C'^T (H V). Its residual
// at_res = C'^T - z z^T C'^T has Gram  G_res = at_res^T at_res
// = G - 2 P P^T + P (z^T z) P^T  with P = C' z = G (H V) and z^T z = (HV)^T P
// (the dump's downdate formula). s power_iteration gates on G_res (forks
// after the candidate's) score it by their max; the smallest score wins.
bool Sketch::amplified_factorize(int k, aero_event* ev) {
    const double delta = delta_;
    const int rc = static_cast<int>(std::ceil(std::log(2.0 / delta) / std::log(100.0)));
    const int q02 = simul_q(d_, 0.2);
    auto run_candidate = [&](uint64_t f) -> bool {  // -> buffer exactly zero
        ev->simul_calls++;
        if (k <= 64) {
            jobs_h_[0] = IterJob{1, r_, k, 0, q02 + 1, -1, fork_state0(f), f};
            for (int c = 0; c < k; ++c) colmask_h_[c] = r_;
            run_iterate(1, r_, k);
            return status_h_[0] == JOB_ZERO;
        }
        run_simul_large(k, f, r_, q02);
        return status_h_[0] != JOB_ACTIVE;
    };
    if (rc <= 1) return run_candidate(++forks_);  // sketch.cpp:57-60
    const int s = static_cast<int>(std::ceil(2.0 * std::log(2.0 / delta) / std::log(3.0)));
    if (s > ncols_) throw InvalidInput("amplification: s exceeds work capacity");
    const int r = r_, rl = r + (r & 1);
    const size_t kk = (size_t)k * k;
    Gres_.alloc((size_t)cap_ * cap_);
    Hc_.alloc((size_t)rl * k);
    Hb_.alloc((size_t)rl * k);
    vrc_.alloc(kk);
    vrb_.alloc(kk);
    qy_.alloc((size_t)rl * k * 2 + kk + 64);
    double* HV = qy_.p;
    double* P = HV + (size_t)rl * k;
    double* ZZ = P + (size_t)rl * k;
    std::vector<double> best_sig(k), cur_sig(k);
    double best_cost = 0.0;
    bool best_zero = false;
    for (int h = 0; h < rc; ++h) {
        const bool zero = run_candidate(++forks_);
        const double* vr = vr_.p;  // the candidate is job 0 (col 0, k x k at vr_)
        for (int a = 0; a < k; ++a) cur_sig[a] = sig_h_[a];
        // keep the candidate's factors before the scoring gates overwrite H / vr
        AERO_CUDA(cudaMemcpy2DAsync(Hc_.p, sizeof(double) * rl, H_.p, sizeof(double) * ldx_, sizeof(double) * r, k,
                                    cudaMemcpyDeviceToDevice, st_));
        AERO_CUDA(cudaMemcpyAsync(vrc_.p, vr, sizeof(double) * kk, cudaMemcpyDeviceToDevice, st_));
        // residual Gram of this candidate (z = I for an all-zero buffer: G_res = 0)
        if (zero) {
            fill_zero(st_, Gres_.p, (int64_t)cap_ * cap_);
        } else {
            copy_matrix(st_, r, r, G_.p, cap_, Gres_.p, cap_);
            dgemm(st_, false, false, r, k, k, 1.0, Hc_.p, rl, vrc_.p, k, 0.0, HV, rl);  // H V
            dgemm(st_, false, false, r, k, r, 1.0, G_.p, cap_, HV, rl, 0.0, P, rl);      // P = G H V
            dgemm(st_, true, false, k, k, r, 1.0, HV, rl, P, rl, 0.0, ZZ, k);           // z^T z
            add_identity(st_, k, ZZ, k, -2.0);
            dgemm(st_, false, false, r, k, k, 1.0, P, rl, ZZ, k, 0.0, HV, rl);          // P (z^T z - 2I)
            dgemm(st_, false, true, r, r, k, 1.0, HV, rl, P, rl, 1.0, Gres_.p, cap_);
            symmetrize(st_, r, Gres_.p, cap_);
        }
        // s power iterations on the residual (sketch.cpp:67-69), one batched launch
        const uint64_t f0 = forks_;
        for (int i = 0; i < s; ++i) {
            jobs_h_[i] = IterJob{0, r, 1, i, kp_ + 1, -1, fork_state0(f0 + 1 + i), f0 + 1 + i};
            colmask_h_[i] = r;
        }
        forks_ += s;
        std::swap(G_.p, Gres_.p);
        try {
            run_iterate(s, r, 1);
        } catch (...) {
            std::swap(G_.p, Gres_.p);
            throw;
        }
        std::swap(G_.p, Gres_.p);
        double cost = 0.0;
        for (int i = 0; i < s; ++i) cost = std::max(cost, status_h_[i] == JOB_ACTIVE ? sig_h_[i] : 0.0);
        if (h == 0 || cost < best_cost) {
            best_cost = cost;
            best_zero = zero;
            best_sig = cur_sig;
            std::swap(Hb_.p, Hc_.p);
            std::swap(vrb_.p, vrc_.p);
        }
    }
    // the winner back where dump_from_job reads a job-0 factorization
    AERO_CUDA(cudaMemcpy2DAsync(H_.p, sizeof(double) * ldx_, Hb_.p, sizeof(double) * rl, sizeof(double) * r, k,
                                cudaMemcpyDeviceToDevice, st_));
    AERO_CUDA(cudaMemcpyAsync(vr_.p, vrb_.p, sizeof(double) * kk, cudaMemcpyDeviceToDevice, st_));
    for (int a = 0; a < k; ++a) sig_h_[a] = best_sig[a];
    status_h_[0] = best_zero ? JOB_ZERO : JOB_ACTIVE;
    return best_zero;
}

// ---------------------------------------------------------------- doubling
// sketch.cpp:108-139 for one row, starting at rank k (forks consumed so far
// are already in forks_)
void Sketch::doubling(int k, int64_t t, double theta, aero_event* ev) {
    const int kmax = std::min({ell_, d_, r_});
    while (true) {
        ev->doubling_steps++;
        bool zero = false;
        if (amp_) {
            zero = amplified_factorize(k, ev);
        } else if (k <= 64) {
            ev->simul_calls++;
            const uint64_t f = ++forks_;
            jobs_h_[0] = IterJob{1, r_, k, 0, q_ + 1, -1, fork_state0(f), f};
            for (int c = 0; c < k; ++c) colmask_h_[c] = r_;
            run_iterate(1, r_, k);
            zero = status_h_[0] == JOB_ZERO;
        } else {
            ev->simul_calls++;
            const uint64_t f = ++forks_;
            run_simul_large(k, f, r_, q_);
            zero = status_h_[0] != JOB_ACTIVE;
        }
        const double tail = sig_h_[k - 1] * sig_h_[k - 1];
        ev->k_last = k;
        ev->tail_sq = tail;
        if (tail < theta || k == kmax) {
            int xi = 0;
            for (int j = 0; j < k; ++j) {
                if (sig_h_[j] * sig_h_[j] >= theta) xi = j + 1;
                else break;
            }
            ev->xi = xi;
            if (xi >= 1) {
                dump_from_job(0, k, xi, t, theta, zero);
                ev->dumped = 1;
            }
            break;
        }
        k = std::min(2 * k, kmax);
    }
}

// ---------------------------------------------------------------- single row
void Sketch::single_row(const double* dev_row, int64_t t, double theta, aero_event* ev) {
    ev->forks_before = (int64_t)forks_;
    append_rows(dev_row, 1);
    r_ += 1;
    if (r_ == cap_) {
        reduce();
        ev->reduced = 1;
    }
    const uint64_t f = ++forks_;
    jobs_h_[0] = IterJob{0, r_, 1, 0, kp_ + 1, -1, fork_state0(f), f};
    colmask_h_[0] = r_;
    run_iterate(1, r_, 1);
    const double s1 = (status_h_[0] == JOB_ACTIVE) ? sig_h_[0] : 0.0;
    ev->sigma1_sq = s1;
    if (s1 >= 0.5 * theta) {  // sketch.cpp:100
        ev->gate_fired = 1;
        doubling(std::min(2, std::min({ell_, d_, r_})), t, theta, ev);
    }
    clock_ = t;
    ev->forks_after = (int64_t)forks_;
    ev->rows_after = r_;
}

// ---------------------------------------------------------------- batch
// Speculative batch of B rows (no reduce inside): every row's gate (and, under
// the FIRE1 pattern, its first doubling step at k = min(2, kmax)) is computed
// at once on the masked prefix of the batch-final Gram; rows are then
// validated in order and the first row whose outcome differs from the
// prediction (or that dumps) ends the batch. Returns rows consumed (>= 1).
int64_t Sketch::run_batch(const double* dev_rows, int64_t B, const int64_t* t,
                          const double* thetas, aero_event* log) {
    const int r0 = r_;
    const uint64_t F = forks_;
    // predict the majority outcome of recent rows (a lone non-firing row in a
    // firing regime ends one batch, not two)
    // (amplified rows finish every fired gate exactly: r candidates + scoring)
    const Pattern pat = (!amp_ && fire_ema_ >= 0.5) ? FIRE1 : NOFIRE;
    const auto pa = std::chrono::steady_clock::now();
    append_rows(dev_rows, B);
    if (host_prof_) {
        AERO_CUDA(cudaStreamSynchronize(st_));
        prof_append_ms_ = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - pa).count();
    }
    const int R = r0 + (int)B;
    int njobs = 0;
    const int gate_base = (pat == FIRE1) ? 2 * (int)B : 0;
    if (pat == FIRE1) {
        for (int j = 0; j < B; ++j) {
            const int rj = r0 + j + 1;
            const int kj = std::min(2, std::min({ell_, d_, rj}));
            jobs_h_[njobs++] = IterJob{1, rj, kj, 2 * j, q_ + 1, -1, fork_state0(F + 2 * j + 2), F + 2 * j + 2};
            colmask_h_[2 * j] = rj;
            colmask_h_[2 * j + 1] = (kj == 2) ? rj : 0;
        }
    }
    for (int j = 0; j < B; ++j) {
        const int rj = r0 + j + 1;
        const uint64_t gf = (pat == FIRE1) ? F + 2 * j + 1 : F + j + 1;
        jobs_h_[njobs++] = IterJob{0, rj, 1, gate_base + j, kp_ + 1, -1, fork_state0(gf), gf};
        colmask_h_[gate_base + j] = rj;
    }
    const auto pi = std::chrono::steady_clock::now();
    run_iterate(njobs, R, 2);
    if (host_prof_)
        prof_iter_ms_ = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - pi).count();
    batches++;
    const int simul_job0 = 0, gate_job0 = (pat == FIRE1) ? (int)B : 0;
    uint64_t forks = F;
    for (int64_t j = 0; j < B; ++j) {
        aero_event* ev = log + j;
        *ev = aero_event{};
        ev->t = t[j];
        ev->theta = thetas[j];
        ev->forks_before = (int64_t)forks;
        const double theta = thetas[j];
        const int gj = gate_job0 + (int)j;
        const double s1 = (status_h_[gj] == JOB_ACTIVE) ? sig_h_[gate_base + j] : 0.0;
        ev->sigma1_sq = s1;
        const bool fire = s1 >= 0.5 * theta;
        const int rj = r0 + (int)j + 1;
        auto commit = [&]() {
            fire_ema_ = 0.95 * fire_ema_ + 0.05 * (ev->gate_fired ? 1.0 : 0.0);
            r_ = rj;
            clock_ = t[j];
            ev->forks_after = (int64_t)forks_;
            ev->rows_after = r_;
            theta_ = theta;
            rows_processed++;
        };
        if (pat == NOFIRE) {
            forks = F + j + 1;
            forks_ = forks;
            if (fire) {  // mispredicted: finish this row exactly, drop the rest
                r_ = rj;
                ev->gate_fired = 1;
                doubling(std::min(2, std::min({ell_, d_, rj})), t[j], theta, ev);
                commit();
                pattern_ = FIRE1;
                mispredicts++;
                end_fired++;
                return j + 1;
            }
            commit();
            continue;
        }
        // FIRE1
        forks = F + 2 * j + 1;
        forks_ = forks;
        if (!fire) {
            commit();
            pattern_ = NOFIRE;
            mispredicts++;
            end_nofire++;
            return j + 1;
        }
        ev->gate_fired = 1;
        ev->doubling_steps = 1;
        ev->simul_calls = 1;
        forks = F + 2 * j + 2;
        forks_ = forks;
        const int kmax = std::min({ell_, d_, rj});
        const int k = std::min(2, kmax);
        const int sj = simul_job0 + (int)j;
        const double* sg = sig_h_ + 2 * j;
        const bool zero = status_h_[sj] == JOB_ZERO;
        const double tail = sg[k - 1] * sg[k - 1];
        ev->k_last = k;
        ev->tail_sq = tail;
        if (tail < theta || k == kmax) {
            int xi = 0;
            for (int a = 0; a < k; ++a) {
                if (sg[a] * sg[a] >= theta) xi = a + 1;
                else break;
            }
            ev->xi = xi;
            if (xi >= 1) {  // state changes: dump, end the batch after this row
                r_ = rj;
                dump_from_job(2 * (int)j, k, xi, t[j], theta, zero);
                ev->dumped = 1;
                commit();
                pattern_ = FIRE1;
                if (j + 1 < B) {
                    mispredicts++;
                    end_dump++;
                }
                return j + 1;
            }
            commit();
            continue;
        }
        // needs a larger rank: continue the doubling for this row exactly
        r_ = rj;
        doubling(std::min(2 * k, kmax), t[j], theta, ev);
        commit();
        pattern_ = FIRE1;
        mispredicts++;
        end_doubling++;
        return j + 1;
    }
    pattern_ = pat;
    return B;
}

void Sketch::process_rows(const double* dev_rows, int64_t n, const int64_t* t,
                          const double* thetas, aero_event* log) {
    const auto hw0 = std::chrono::steady_clock::now();
    struct WallAcc {  // dev instrumentation (AERO_HOST_PROF): wall time of process_rows
        double& acc;
        std::chrono::steady_clock::time_point t0;
        ~WallAcc() { acc += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); }
    } wall_acc{host_wall_s_, hw0};
    int64_t pos = 0;
    while (pos < n) {
        const int64_t room = (int64_t)cap_ - 1 - r_;  // rows that fit before a reduce
        if (exact_ || room < 2 || n - pos < 2) {
            aero_event* ev = log + pos;
            *ev = aero_event{};
            ev->t = t[pos];
            ev->theta = thetas[pos];
            theta_ = thetas[pos];
            const auto s0 = std::chrono::steady_clock::now();
            single_row(dev_rows + (size_t)pos * d_, t[pos], thetas[pos], ev);
            if (host_prof_) {
                const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - s0).count();
                if (ms > 40.0) fprintf(stderr, "  slow single_row t=%lld r=%d reduce=%d: %.1f ms\n", (long long)t[pos], r_, ev->reduced, ms);
            }
            fire_ema_ = 0.95 * fire_ema_ + 0.05 * (ev->gate_fired ? 1.0 : 0.0);
            rows_processed++;
            pos++;
            continue;
        }
        // batch size from the observed rate p of batch-ending rows: a batch
        // costs ~alpha + beta*B (alpha = the fixed phase latency, ~40 rows'
        // worth of products) and commits (1-(1-p)^B)/p rows on average, which
        // is cheapest per row near B* = sqrt(2 alpha / (beta p))
        const double p = std::max(end_rate_, 1e-4);
        static const double two_alpha = getenv("AERO_BATCH_2ALPHA") ? atof(getenv("AERO_BATCH_2ALPHA")) : 52.0;
        // int8 iterate (r >= i8_min_rows_): cap a batch at one column per
        // job slot of a 64-wide MMA tile row -- 3 x 64 columns (FIRE1: 3 per
        // row) or 192 (NOFIRE) -- which also keeps the jobs <= the 148 CTAs, so
        // no CTA normalizes two jobs in a phase (C2 sweep: 64 rows 1858 ms vs
        // 192 rows 1938 ms per 40960 rows; 48: 2120, 96: 1909)
        int cap = max_batch_;
        if (i8_ && r_ + 1 >= i8_min_rows_ && persistent_ && cfg_max_batch_ == 0)
        {
            // dev knob AERO_I8_BATCH_CAP: rows per FIRE1 batch (sweep in DESIGN.md 5)
            static const int fire_cap = getenv("AERO_I8_BATCH_CAP") ? std::max(16, atoi(getenv("AERO_I8_BATCH_CAP"))) : 64;
            cap = std::min(cap, (!amp_ && fire_ema_ >= 0.5) ? fire_cap : 192);
        }
        cur_batch_ = (int)std::clamp(std::sqrt(two_alpha / p), 16.0, (double)cap);
        const int64_t B = std::min<int64_t>({(int64_t)cur_batch_, n - pos, room});
        const int64_t mp0 = mispredicts;
        const auto b0 = std::chrono::steady_clock::now();
        const int64_t used = run_batch(dev_rows + (size_t)pos * d_, B, t + pos, thetas + pos, log + pos);
        if (host_prof_) {
            const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - b0).count();
            if (ms > 40.0) fprintf(stderr, "  slow batch t=%lld B=%lld used=%lld r=%d: %.1f ms (append %.1f iterate %.1f)\n", (long long)t[pos], (long long)B, (long long)used, r_, ms, prof_append_ms_, prof_iter_ms_);
        }
        const double ended = (mispredicts > mp0) ? 1.0 : 0.0;
        const double w = std::min(1.0, (double)used / 256.0);  // EMA over ~256 rows
        end_rate_ = (1.0 - w) * end_rate_ + w * (ended / (double)used);
        pos += used;
    }
    if (n > 0) last_ev_ = log[n - 1];
}

// ---------------------------------------------------------------- update
void Sketch::update_block(const double* rows, bool device, int64_t n, int64_t ld, const int64_t* t,
                          const double* theta_per_row, aero_event* log, bool amplified) {
    if (n <= 0) return;
    if (ld < d_) throw InvalidInput("AeroState: row dimension mismatch");
    if (amplified && delta_ == 0.0)  // sketch.cpp:46
        throw InvalidInput("AeroState: amplification requested without delta");
    amp_ = amplified || (mode_ == AERO_THETA_ATTP && delta_ > 0.0);  // attp.hpp:24
    AERO_CUDA(cudaSetDevice(dev_));
    std::vector<aero_event> local;
    if (!log) {
        local.resize(n);
        log = local.data();
    }
    // Chunks of stage_rows_ rows through two staging buffers: the H2D copy
    // (pinned host rows: DMA) and the K1 norm/finiteness pass of chunk k+1 run
    // on the staging stream while chunk k is processed. Device rows with
    // ld == d are read in place (no staging copy).
    const int64_t nchunks = (n + stage_rows_ - 1) / stage_rows_;
    const bool in_place = device && ld == d_;
    const double* src[2] = {nullptr, nullptr};
    auto prefetch = [&](int64_t k) {
        const int b = (int)(k & 1);
        const int64_t off = k * stage_rows_, cnt = std::min<int64_t>(stage_rows_, n - off);
        if (in_place) {
            src[b] = rows + off * ld;
            AERO_CUDA(cudaStreamWaitEvent(cs_, ev_free_[b], 0));
        } else {
            stage_[b].alloc((size_t)stage_rows_ * d_);
            AERO_CUDA(cudaStreamWaitEvent(cs_, ev_free_[b], 0));  // chunk k-2 is done with it
            AERO_CUDA(cudaMemcpy2DAsync(stage_[b].p, sizeof(double) * d_, rows + off * ld, sizeof(double) * ld,
                                        sizeof(double) * d_, cnt,
                                        device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, cs_));
            src[b] = stage_[b].p;
        }
        double* nd = nrm_.p + (size_t)b * stage_rows_;
        int* bd = bad_d_ + (size_t)b * stage_rows_;
        ingest_rows(cs_, src[b], cnt, d_, d_, nd, bd);
        AERO_CUDA(cudaMemcpyAsync(nrm_h_ + (size_t)b * stage_rows_, nd, sizeof(double) * cnt, cudaMemcpyDeviceToHost, cs_));
        AERO_CUDA(cudaMemcpyAsync(bad_h_ + (size_t)b * stage_rows_, bd, sizeof(int) * cnt, cudaMemcpyDeviceToHost, cs_));
        AERO_CUDA(cudaEventRecord(ev_ready_[b], cs_));
    };
    // events start "free": record them once on the sketch stream
    for (int b = 0; b < 2; ++b) AERO_CUDA(cudaEventRecord(ev_free_[b], st_));
    std::vector<double> th;
    prefetch(0);
    for (int64_t k = 0; k < nchunks; ++k) {
        const int b = (int)(k & 1);
        const int64_t off = k * stage_rows_, cnt = std::min<int64_t>(stage_rows_, n - off);
        if (k + 1 < nchunks) prefetch(k + 1);
        AERO_CUDA(cudaEventSynchronize(ev_ready_[b]));
        const double* nrm_h = nrm_h_ + (size_t)b * stage_rows_;
        const int* bad_h = bad_h_ + (size_t)b * stage_rows_;
        // validation in row order (sketch.cpp:83-85): the first offending row
        // raises after the rows before it were absorbed
        int64_t good = cnt;
        std::string err;
        int64_t prev = (off == 0) ? clock_ : t[off - 1];
        for (int64_t j = 0; j < cnt; ++j) {
            if (bad_h[j]) { good = j; err = "AeroState: non-finite row"; break; }
            if (t[off + j] <= prev) { good = j; err = "AeroState: timestamp regression"; break; }
            if (mode_ != AERO_THETA_ATTP && theta_per_row && theta_per_row[off + j] < 0.0) {
                good = j;  // set_theta throws before this row's update (sketch.cpp:33-36)
                err = "AeroState: theta must be >= 0";
                break;
            }
            prev = t[off + j];
        }
        th.resize(good);
        for (int64_t j = 0; j < good; ++j) {
            if (mode_ == AERO_THETA_ATTP) {  // attp.hpp:22-23
                fro_mass_ += nrm_h[j];
                th[j] = eps_ * fro_mass_;
            } else if (theta_per_row) {
                th[j] = theta_per_row[off + j];
            } else {
                th[j] = theta_;
            }
        }
        AERO_CUDA(cudaStreamWaitEvent(st_, ev_ready_[b], 0));
        try {
            process_rows(src[b], good, t + off, th.data(), log + off);
        } catch (...) {
            cudaStreamSynchronize(cs_);  // no DMA from the caller's rows after we return
            throw;
        }
        AERO_CUDA(cudaEventRecord(ev_free_[b], st_));
        if (good < cnt) {
            AERO_CUDA(cudaStreamSynchronize(cs_));
            throw InvalidInput(err);
        }
    }
    AERO_CUDA(cudaStreamSynchronize(cs_));
}

// ---------------------------------------------------------------- queries
void Sketch::ensure_query_buffers() {
    Bq_.alloc((size_t)d_ * d_);
    Wq_.alloc((size_t)d_ * d_ + d_);
}

void Sketch::accumulate_residual(double* B, double beta_first) {
    if (r_ > 0)
        gemm_acc(st_, false, true, d_, d_, r_, 1.0, C_.p, d_, C_.p, d_, beta_first, B, d_, ws_.p, ws_.n);
    else if (beta_first == 0.0)
        fill_zero(st_, B, (int64_t)d_ * d_);
}

// sketch.cpp:162-165 summed over snaps [first, last): B += Z M + (Z M)^T - Z (M Z) Z^T
void Sketch::accumulate_restore(double* B, int64_t first, int64_t last) {
    int64_t i = first;
    std::vector<int> offs, wids;
    while (i < last) {
        const Chunk* ch = snaps_[i].chunk;
        const int c0 = snaps_[i].col;
        int64_t j = i;
        int cols = 0;
        offs.clear();
        wids.clear();
        while (j < last && snaps_[j].chunk == ch && snaps_[j].col == c0 + cols) {
            offs.push_back(snaps_[j].col);
            wids.push_back(snaps_[j].xi);
            cols += snaps_[j].xi;
            ++j;
        }
        const double* Z = ch->z + (size_t)c0 * d_;
        const double* Mt = ch->mt + (size_t)c0 * d_;
        // the d x d restore products on the fp64 DMMA engine (split-K, fixed order)
        gemm_acc(st_, false, true, d_, d_, cols, 1.0, Z, d_, Mt, d_, 1.0, B, d_, ws_.p, ws_.n);   // Z M
        gemm_acc(st_, false, true, d_, d_, cols, 1.0, Mt, d_, Z, d_, 1.0, B, d_, ws_.p, ws_.n);   // (Z M)^T
        qy_.alloc((size_t)d_ * ch->cap + 2 * (size_t)ch->cap + 64);
        double* Yk = qy_.p;
        // per-snapshot K terms (batched kernel for xi <= 64, GEMMs otherwise)
        std::vector<int> so, sw;
        for (size_t s = 0; s < offs.size(); ++s) {
            if (wids[s] <= 64) {
                so.push_back(offs[s]);
                sw.push_back(wids[s]);
            } else {
                const int xi = wids[s];
                double* zs = ch->z + (size_t)offs[s] * d_;
                double* ms = ch->mt + (size_t)offs[s] * d_;
                qw_.alloc((size_t)xi * xi);
                dgemm(st_, true, false, xi, xi, d_, 1.0, ms, d_, zs, d_, 0.0, qw_.p, xi);
                dgemm(st_, false, false, d_, xi, xi, 1.0, zs, d_, qw_.p, xi, 0.0,
                      Yk + (size_t)offs[s] * d_, d_);
            }
        }
        if (!so.empty()) {
            int* dso = nullptr;
            AERO_CUDA(cudaMallocAsync(&dso, sizeof(int) * 2 * so.size(), st_));
            AERO_CUDA(cudaMemcpyAsync(dso, so.data(), sizeof(int) * so.size(), cudaMemcpyHostToDevice, st_));
            AERO_CUDA(cudaMemcpyAsync(dso + so.size(), sw.data(), sizeof(int) * sw.size(),
                                      cudaMemcpyHostToDevice, st_));
            restore_k_terms(st_, d_, ch->z, ch->mt, d_, dso, dso + so.size(), (int)so.size(), Yk);
            AERO_CUDA(cudaFreeAsync(dso, st_));
            AERO_CUDA(cudaStreamSynchronize(st_));
        }
        gemm_acc(st_, false, true, d_, d_, cols, -1.0, Yk + (size_t)c0 * d_, d_, Z, d_, 1.0, B, d_, ws_.p, ws_.n);
        i = j;
    }
}

const double* Sketch::query_gram_device(int64_t lb, int64_t ub) {
    if (lb >= ub) throw InvalidInput("AeroState: query needs lb < ub");
    if (ub > clock_) throw InvalidInput("AeroState: query beyond clock");
    AERO_CUDA(cudaSetDevice(dev_));
    ensure_query_buffers();
    fill_zero(st_, Bq_.p, (int64_t)d_ * d_);
    if (ub == clock_ && r_ > 0) accumulate_residual(Bq_.p, 0.0);  // sketch.cpp:150
    // first snapshot with t > lb (sketch.cpp:153-157), then while t <= ub
    int64_t first = 0, last = 0;
    while (first < (int64_t)snaps_.size() && snaps_[first].t <= lb) ++first;
    last = first;
    while (last < (int64_t)snaps_.size() && snaps_[last].t <= ub) ++last;
    accumulate_restore(Bq_.p, first, last);
    return Bq_.p;
}

void Sketch::query_gram(int64_t lb, int64_t ub, double* out_host) {
    const double* B = query_gram_device(lb, ub);
    AERO_CUDA(cudaMemcpyAsync(out_host, B, sizeof(double) * d_ * d_, cudaMemcpyDeviceToHost, st_));
    AERO_CUDA(cudaStreamSynchronize(st_));  // symmetric: column-major == row-major
}

// shrink_to_sketch (sketch.cpp:167-178)
void Sketch::query(int64_t lb, int64_t ub, double* out_host) {
    const double* B = query_gram_device(lb, ub);
    copy_matrix(st_, d_, d_, B, d_, Wq_.p, d_);
    double* w = Wq_.p + (size_t)d_ * d_;
    eigh(st_, d_, Wq_.p, d_, w, 1, 0, std::min(ell_, d_));
    qy_.alloc((size_t)ell_ * d_);
    shrink_rows(st_, w, Wq_.p, d_, d_, ell_, qy_.p);
    AERO_CUDA(cudaMemcpyAsync(out_host, qy_.p, sizeof(double) * ell_ * d_, cudaMemcpyDeviceToHost, st_));
    AERO_CUDA(cudaStreamSynchronize(st_));
}

void Sketch::residual(double* out, int64_t max_rows) {
    const int64_t rows = std::min<int64_t>(r_, max_rows);
    AERO_CUDA(cudaMemcpyAsync(out, C_.p, sizeof(double) * d_ * rows, cudaMemcpyDeviceToHost, st_));
    AERO_CUDA(cudaStreamSynchronize(st_));
}

const SnapRec& Sketch::snap(int64_t i) const {
    if (i < 0 || i >= (int64_t)snaps_.size()) throw InvalidInput("snapshot index out of range");
    return snaps_[i];
}
void Sketch::snap_get(int64_t i, double* z, double* m) {
    const SnapRec& s = snap(i);
    if (z) {  // device z is d x xi column-major; the ABI wants d x xi row-major
        std::vector<double> tmp((size_t)d_ * s.xi);
        AERO_CUDA(cudaMemcpyAsync(tmp.data(), s.chunk->z + (size_t)s.col * d_,
                                  sizeof(double) * tmp.size(), cudaMemcpyDeviceToHost, st_));
        AERO_CUDA(cudaStreamSynchronize(st_));
        for (int j = 0; j < s.xi; ++j)
            for (int i2 = 0; i2 < d_; ++i2) z[(size_t)i2 * s.xi + j] = tmp[(size_t)j * d_ + i2];
    }
    if (m) {  // m^T column-major d x xi == m row-major xi x d
        AERO_CUDA(cudaMemcpyAsync(m, s.chunk->mt + (size_t)s.col * d_,
                                  sizeof(double) * (size_t)d_ * s.xi, cudaMemcpyDeviceToHost, st_));
        AERO_CUDA(cudaStreamSynchronize(st_));
    }
}
void Sketch::snap_pop_front() {
    if (snaps_.empty()) return;
    const SnapRec s = snaps_.front();
    snaps_.pop_front();
    arena_release(s);
}

void Sketch::info(aero_info* o) const {
    o->d = d_;
    o->ell = ell_;
    o->rows = r_;
    o->clock = clock_;
    o->last_dump_t = last_dump_t_;
    o->forks = (int64_t)forks_;
    o->snaps = (int64_t)snaps_.size();
    int64_t cols = 0;
    for (const SnapRec& s : snaps_) cols += s.xi;
    o->snap_cols = cols;
    o->theta = theta_;
    o->fro_mass = fro_mass_;
    o->device_rows_processed = rows_processed;
    o->device_batches = batches;
    o->device_mispredicts = mispredicts;
    o->end_nofire = end_nofire;
    o->end_fired = end_fired;
    o->end_doubling = end_doubling;
    o->end_dump = end_dump;
}

}  // namespace aero_b200
