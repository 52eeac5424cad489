// Launchers for the B200 AeroSketch device kernels (kernels.cu, eigh.cu).
// All matrices are column-major (BLAS convention) unless stated: the residual
// buffer C' (r x d, reference row-major semantics) is held as C'^T, a d x cap
// column-major array whose column i is row i of C'.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace aero_b200 {

// D = alpha * op(A) * op(B) + beta * D (fp64, column-major). If colmask is
// non-null, output rows i >= colmask[j] of column j are written as 0.
void dgemm(cudaStream_t st, bool ta, bool tb, int m, int n, int k, double alpha, const double* A,
           int lda, const double* B, int ldb, double beta, double* D, int ldd,
           const int* colmask = nullptr);

// the dominant product Y = A B (A: M x K, B: K x N, column-major) with the
// per-column row mask; split-K partials go through ws (product.cu)
size_t product_workspace_doubles(int M, int N);
// Y = op(A) op(B) on the fast path (alpha = 1, beta = 0); returns false (and
// does nothing) when operand alignment rules it out -- callers then use dgemm
// (defer_reduce: leave split-K partials in ws, ws[z*M*N + i + j*M], and report
// the split count; the caller's consumer sums them -- iter_normalize_ws)
bool gemm_big(cudaStream_t st, bool ta, bool tb, int M, int N, int K, const double* A, int lda,
              const double* B, int ldb, double* Y, int ldy, const int* colmask, double* ws,
              size_t ws_doubles, int* splits_used = nullptr, bool defer_reduce = false);
// Y = alpha op(A) op(B) + beta Y on the fast path (falls back to dgemm when
// operand alignment rules the fast path out)
void gemm_acc(cudaStream_t st, bool ta, bool tb, int M, int N, int K, double alpha, const double* A,
              int lda, const double* B, int ldb, double beta, double* Y, int ldy, double* ws,
              size_t ws_doubles);
void gemm_product(cudaStream_t st, int M, int N, int K, const double* A, int lda, const double* B,
                  int ldb, double* Y, int ldy, const int* colmask, double* ws, size_t ws_doubles);

// Y = G X (fp64 in and out) on the int8 tensor cores by exact slicing
// (Ozaki scheme, ozaki.cu). prepare() slices G (r x r, symmetric, column i =
// row i at G + i*ldg) once per Gram; product() slices X (R x N, column j
// masked to rows < colmask[j]) and runs the tcgen05 kind::i8 kernel; output
// rows i >= colmask[j] of column j are 0. Split-K partials go through ws.
struct OzakiGram {
    int R = 0, Rp = 0, Kp = 0;
    int8_t *a = nullptr, *b = nullptr;
    int *ea = nullptr, *fb = nullptr;
    size_t a_bytes = 0, b_bytes = 0, ea_n = 0, fb_n = 0;
    void prepare(cudaStream_t st, int R, const double* G, int ldg);
    void product(cudaStream_t st, int N, const double* X, int ldx, const int* colmask, double* Y, int ldy,
                 double* ws, size_t ws_doubles);
    void reserve_x(int N);  // X slice buffers for N columns
    // allocate the slice buffers for up to Rmax rows and Nmax columns once
    // (growing them on demand costs a cudaFree -- a device-wide sync -- plus a
    // cudaMalloc inside the update loop)
    void reserve(int Rmax, int Nmax);
    void release();
    ~OzakiGram() { release(); }
};
int ozaki_slices();

// dst[q] = src[idx_d[q]] (rows of d doubles, src row stride lds, dst contiguous)
void gather_rows(cudaStream_t st, const double* src, int64_t lds, const int64_t* idx_d, int64_t n, int d,
                 double* dst);
// per-row squared norm and finiteness of n rows (row-major, ld) -> nrm2[n], bad[n]
void ingest_rows(cudaStream_t st, const double* rows, int64_t n, int64_t ld, int d, double* nrm2,
                 int* bad);

// ---- batched power / subspace iteration engine ---------------------------
struct IterJob {
    int type;       // 0 = gate (power_iteration, linalg.cpp:96-121), 1 = simul (linalg.cpp:123-152)
    int r;          // prefix rows of G (buffer rows for this row's update)
    int k;          // columns (1 for gate)
    int col;        // first column in the X / Y work arrays
    int nphase;     // number of G products: kp + 1 (gate) or q + 1 (simul)
    int panel;      // offset of the job's host-supplied Gaussians (rng_panels.hpp), -1: device draws
    uint64_t rng0;  // splitmix state0 of the fork that seeds this job
    uint64_t fork;  // the fork's index in the sketch's RngState (rng.hpp:54-57)
};
// job status codes (device int per job)
enum : int { JOB_ACTIVE = 0, JOB_ZERO = 1, JOB_DEAD = 2 };

// init: X columns <- first r Gaussians of the job's fork (gate: normalized;
// simul: Pi row-major r x k), zero below r; status from trace(G[0:r,0:r]).
// panel (nullable): host-supplied Gaussians, job j's at panel + jobs[j].panel
void iter_init(cudaStream_t st, const IterJob* jobs, int njobs, const double* G, int ldg,
               double* X, int ldx, int R, int* status, const double* panel = nullptr);
// normalization after product phase `phase` (Y = G X already computed):
//  gate : phase < nphase-1 -> X <- Y / ||Y|| (1e-300 check); last -> s1sq = X.Y
//  simul: S = X^T Y, T = S^{-1/2} (eig, clamped), [last: H = X T], X <- Y T,
//         [last: Ritz values of (X)^T X -> sig, Vr]
// out_sig: per column value (gate s1sq at col; simul sigma_hat[0..k) at col..),
// out_vr : per simul job k x k (col-major, ld kv) at out_vr + col * kv
void iter_normalize(cudaStream_t st, const IterJob* jobs, int njobs, int phase, double* X,
                    const double* Y, int ldx, double* H, int* status, double* out_sig,
                    double* out_vr, int kv, int* out_clamped, int max_k);
// same, with Y given as `splits` split-K partials of an M x N product in ws
// (summed in fixed order per job, cached in shared memory): fuses the split-K
// reduction into the normalization (k <= 4)
void iter_normalize_ws(cudaStream_t st, const IterJob* jobs, int njobs, int phase, double* X,
                       int ldx, const double* ws, int M, int N, int splits, double* H, int* status,
                       double* out_sig, double* out_vr, int kv, int* out_clamped, int max_k);

// all phases of a batch in one persistent cooperative launch (max_k <= 4):
// split-K DMMA products into ws (phase_splits[p] * R * phase_ncol[p] doubles)
// and per-job normalization separated by grid barriers; same results as the
// per-phase gemm_big + iter_normalize_ws sequence. `grid` (<= iterate_grid(R),
// the co-resident maximum) is sized to the work so small problems leave the
// rest of the GPU to concurrent streams (MlState levels)
int iterate_grid(int R);
// all phases of a batch in one persistent cooperative launch with the products
// on the int8 tensor cores (ozaki.cuh tiles; G sliced by oz.prepare, X sliced
// in the kernel: phase 0 up front, later phases by the normalization as it
// writes each new iterate); phase_splits[p] split-K ways per phase (partials
// in ws, summed by the per-job normalization); grid <= number of SMs
void iterate_i8_persistent(cudaStream_t st, const IterJob* jobs, int njobs, int maxphase, int R, const OzakiGram& oz,
                           const int* colmask, double* X, int ldx, double* H, int* status, double* out_sig,
                           double* out_vr, int kv, int* out_clamped, double* ws, const int* phase_ncol,
                           const int* phase_splits, unsigned* bar, int max_k, int grid);
// split-K ways of an int8 tensor-core product of R rows x N columns (K = R)
int ozaki_splits(const OzakiGram& oz, int N, size_t ws_doubles);
void iterate_persistent(cudaStream_t st, const IterJob* jobs, int njobs, int maxphase, int R, const double* G,
                        int ldg, double* X, int ldx, double* H, int* status, double* out_sig, double* out_vr,
                        int kv, int* out_clamped, double* ws, const int* phase_ncol, const int* phase_splits,
                        unsigned* bar, int max_k, int grid);

// buffers of <= 96 rows and k <= 2: one warp per job runs all its phases with
// G in shared memory (no phase synchronisation); returns false if not applicable
bool iterate_warp(cudaStream_t st, const IterJob* jobs, int njobs, const double* G, int ldg, int R, double* X,
                  int ldx, double* H, int* status, double* out_sig, double* out_vr, int kv, int* out_clamped,
                  int max_k);
// 96 < R <= 512, k <= 2: one CTA per 4 jobs, all phases, G streamed through shared memory
bool iterate_cta(cudaStream_t st, const IterJob* jobs, int njobs, const double* G, int ldg, int R, double* X,
                 int ldx, double* H, int* status, double* out_sig, double* out_vr, int kv, int* out_clamped,
                 int max_k);

// ---- small dense helpers ---------------------------------------------------
// symmetric eigendecomposition of `batch` n x n matrices (column-major, ld,
// stride between matrices): eigenvalues descending, eigenvector columns
// sign-fixed (largest-magnitude entry positive, linalg.cpp:17-26). A is
// overwritten by V. One-CTA Jacobi for n <= kSmallEigMax, the tridiagonal
// solver of syev.cu otherwise; nvec > 0 limits the eigenvectors to the top
// nvec (columns nvec.. of A are then unspecified; all n eigenvalues returned).
constexpr int kSmallEigMax = 32;
constexpr int kBatchedJacobiMax = 96;
void eigh(cudaStream_t st, int n, double* A, int lda, double* w, int batch = 1,
          int64_t stride = 0, int nvec = 0);
void eigh_forget(cudaStream_t st);  // free the solver cached for one stream

// columns of V (n x ncol, ld) scaled: V[:, i] *= scale[i]
void scale_columns(cudaStream_t st, int n, int ncol, double* V, int ld, const double* scale);
// rows scaled: V[i, :] *= scale[i]
void scale_rows(cudaStream_t st, int n, int ncol, double* V, int ld, const double* scale);
// FD reduce weights (fd.cpp:20-27 via eig of C'C'^T): from eigenvalues lam
// (descending) compute w_i = sqrt(s2_i)/sigma_i with sigma_i = sqrt(max(lam,0)),
// s2_i = sigma_i^2 - sigma_{ell-1}^2 (0 if <= 0), for i < keep
void fd_weights(cudaStream_t st, const double* lam, int n, int ell, int keep, double* w);
// make the largest-magnitude entry of each column of Z (d x k, ld) positive;
// flips[j] = +-1 written (linalg.cpp:17-26)
void fix_column_signs(cudaStream_t st, int d, int k, double* Z, int ld, double* flips);
// symmetrize square matrix in place: A <- (A + A^T)/2 (eigh, linalg.cpp:64)
void symmetrize(cudaStream_t st, int n, double* A, int lda);
// copy / fill helpers
void fill_zero(cudaStream_t st, double* p, int64_t count);
void copy_matrix(cudaStream_t st, int m, int n, const double* A, int lda, double* B, int ldb);
// rows (row-major, ld) -> columns of Ct (d x n, ld = ldc), i.e. a 2-D copy
void rows_to_cols(cudaStream_t st, const double* rows, int64_t n, int64_t ld, int d, double* Ct,
                  int ldc);
// add a multiple of the identity to a k x k block: A += alpha I
void add_identity(cudaStream_t st, int k, double* A, int lda, double alpha);
// shrink_to_sketch epilogue (sketch.cpp:167-178): rows i < min(ell, d):
// out_rm[i, :] = sqrt(max(lam_i,0) - cut) * V[:, i]^T (row-major ell x d)
void shrink_rows(cudaStream_t st, const double* lam, const double* V, int ldv, int d, int ell,
                 double* out_rm);
// per-snapshot K_s = M_s^T Z_s (xi x xi) then Y_s = Z_s K_s (d x xi) for a run
// of snapshots stored contiguously: Z, Mt are d x ncols; widths[s] per snapshot
void restore_k_terms(cudaStream_t st, int d, const double* Z, const double* Mt, int ld,
                     const int* offsets, const int* widths, int nsnap, double* Y);

// ---- stream generator (DESIGN.md GENERATOR spec) ---------------------------
// raw latent rows: out[t][j] = sum_l s_l sigma_l U[l, j] + noise * g_j, then
// rescaled to ||a||^2 = r_max^u. U1 (k x d row-major), U2 (k2 x d) on device.
void gen_rows(cudaStream_t st, int d, int k, int k2, const double* U1, const double* U2,
              double rho, double rho2, double scale2, double noise, double r_max, uint64_t seed,
              uint64_t stream, int64_t t0, int64_t n, double* out);
// Gaussian matrix rows x cols row-major from RngState(seed, stream) (fork 0)
void gen_gaussian_matrix(cudaStream_t st, uint64_t state0, int64_t count, double* out);

}  // namespace aero_b200
