// Symmetric eigensolver dispatch for the FD reduce (K3), the simul Ritz step
// and the query shrink (K6): n <= kSmallEigMax -> one-CTA shared-memory
// Jacobi (kernels.cu, also batches of n <= 96); larger n -> tridiagonalization + multisection +
// twisted-factorization eigenvectors + WY back-transform (syev.cu).
#include "aero_common.cuh"
#include "kernels.cuh"

namespace aero_b200 {

void eigh_small(cudaStream_t st, int n, double* A, int lda, double* w, int batch, int64_t stride);
void eigh_large(cudaStream_t st, int n, double* A, int lda, double* w, int nvec);
void eigh_large_forget(cudaStream_t st);

void eigh(cudaStream_t st, int n, double* A, int lda, double* w, int batch, int64_t stride, int nvec) {
    if (n <= 0 || batch <= 0) return;
    symmetrize(st, n, A, lda);  // (B + B^T)/2, linalg.cpp:64
    for (int b = 1; b < batch; ++b) symmetrize(st, n, A + b * stride, lda);
    if (n <= kSmallEigMax || (batch > 1 && n <= kBatchedJacobiMax)) {  // one launch for the batch
        eigh_small(st, n, A, lda, w, batch, stride);
        return;
    }
    for (int b = 0; b < batch; ++b) eigh_large(st, n, A + b * stride, lda, w + (int64_t)b * n, nvec);
}

void eigh_forget(cudaStream_t st) { eigh_large_forget(st); }

}  // namespace aero_b200
