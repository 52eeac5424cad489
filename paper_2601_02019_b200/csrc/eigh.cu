// Symmetric eigensolver dispatch for the FD reduce (K3) and query shrink (K6).
// n <= kSmallEigMax: one-CTA shared-memory Jacobi (kernels.cu, own code).
// n >  kSmallEigMax: cuSOLVER syevd -- ROUND-1 STOPGAP, documented in
// DESIGN.md; replaced by an own tridiagonal/divide-and-conquer solver next.
#include <cusolverDn.h>

#include <mutex>
#include <unordered_map>

#include "aero_common.cuh"
#include "kernels.cuh"

namespace aero_b200 {

void eigh_small(cudaStream_t st, int n, double* A, int lda, double* w, int batch, int64_t stride);

namespace {
struct Solver {
    cusolverDnHandle_t h = nullptr;
    double* work = nullptr;
    int lwork = 0;
    int* info = nullptr;
    double* tmpw = nullptr;
    int tmpw_n = 0;
};
std::mutex g_mu;
// one solver (handle + workspace) per stream: sketches on different host
// threads (MlState levels) must not share a workspace
std::unordered_map<cudaStream_t, Solver> g_solvers;

// reverse to descending order and fix signs (linalg.cpp:17-26, 66-75)
__global__ void k_reverse_fix(int n, double* A, int lda, const double* wasc, double* wdesc) {
    // one CTA per output column
    __shared__ double bv[32];
    __shared__ int bi[32];
    const int col = blockIdx.x;
    const int src = n - 1 - col;
    if (threadIdx.x == 0) wdesc[col] = wasc[src];
    // columns col and src swap: handle only col <= src pair once
    if (col > src) return;
    double* a = A + (int64_t)col * lda;
    double* b = A + (int64_t)src * lda;
    for (int i = threadIdx.x; i < n && col != src; i += blockDim.x) {
        const double t = a[i];
        a[i] = b[i];
        b[i] = t;
    }
    __syncthreads();
    for (int pass = 0; pass < (col == src ? 1 : 2); ++pass) {
        double* z = pass == 0 ? a : b;
        double best = -1.0;
        int at = 0x7fffffff;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const double v = fabs(z[i]);
            if (v > best) { best = v; at = i; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, at, o);
            if (ov > best || (ov == best && oi < at)) { best = ov; at = oi; }
        }
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
        if (lane == 0) { bv[wid] = best; bi[wid] = at; }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int w = 1; w < nw; ++w)
                if (bv[w] > bv[0] || (bv[w] == bv[0] && bi[w] < bi[0])) { bv[0] = bv[w]; bi[0] = bi[w]; }
        __syncthreads();
        const bool flip = bi[0] < n && z[bi[0]] < 0.0;
        __syncthreads();
        if (flip)
            for (int i = threadIdx.x; i < n; i += blockDim.x) z[i] = -z[i];
        __syncthreads();
    }
}
}  // namespace

void eigh(cudaStream_t st, int n, double* A, int lda, double* w, int batch, int64_t stride) {
    if (n <= 0 || batch <= 0) return;
    symmetrize(st, n, A, lda);  // (B + B^T)/2, linalg.cpp:64
    for (int b = 1; b < batch; ++b) symmetrize(st, n, A + b * stride, lda);
    if (n <= kSmallEigMax) {
        eigh_small(st, n, A, lda, w, batch, stride);
        return;
    }
    Solver* sp;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        sp = &g_solvers[st];  // node-based map: the reference stays valid
    }
    Solver& s = *sp;
    if (!s.h) {
        if (cusolverDnCreate(&s.h) != CUSOLVER_STATUS_SUCCESS) throw CudaError("cusolverDnCreate");
        AERO_CUDA(cudaMalloc(&s.info, sizeof(int)));
    }
    cusolverDnSetStream(s.h, st);
    for (int b = 0; b < batch; ++b) {
        double* Ab = A + b * stride;
        double* wb = w + (int64_t)b * n;
        int lwork = 0;
        if (cusolverDnDsyevd_bufferSize(s.h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n,
                                        Ab, lda, wb, &lwork) != CUSOLVER_STATUS_SUCCESS)
            throw CudaError("cusolverDnDsyevd_bufferSize");
        if (lwork > s.lwork) {
            if (s.work) cudaFree(s.work);
            AERO_CUDA(cudaMalloc(&s.work, sizeof(double) * (size_t)lwork));
            s.lwork = lwork;
        }
        if (n > s.tmpw_n) {
            if (s.tmpw) cudaFree(s.tmpw);
            AERO_CUDA(cudaMalloc(&s.tmpw, sizeof(double) * (size_t)n));
            s.tmpw_n = n;
        }
        if (cusolverDnDsyevd(s.h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, Ab, lda,
                             s.tmpw, s.work, s.lwork, s.info) != CUSOLVER_STATUS_SUCCESS)
            throw CudaError("cusolverDnDsyevd");
        note_launch();
        k_reverse_fix<<<n, 256, 0, st>>>(n, Ab, lda, s.tmpw, wb);
        AERO_LAUNCHED();
    }
}

void eigh_forget(cudaStream_t st) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_solvers.find(st);
    if (it == g_solvers.end()) return;
    Solver& s = it->second;
    if (s.work) cudaFree(s.work);
    if (s.tmpw) cudaFree(s.tmpw);
    if (s.info) cudaFree(s.info);
    if (s.h) cusolverDnDestroy(s.h);
    g_solvers.erase(it);
}

void eigh_release() {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& kv : g_solvers) {
        Solver& s = kv.second;
        if (s.work) cudaFree(s.work);
        if (s.tmpw) cudaFree(s.tmpw);
        if (s.info) cudaFree(s.info);
        if (s.h) cusolverDnDestroy(s.h);
    }
    g_solvers.clear();
}

}  // namespace aero_b200
