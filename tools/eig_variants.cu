// Times cuSOLVER symmetric eigensolver variants at n = 2048 (FD reduce size at C2).
#include <cusolverDn.h>
#include <cstdio>
#include <vector>
#include <random>
#define CK(x) do { auto e_ = (x); if (e_ != 0) printf("err %d at %s\n", (int)e_, #x); } while (0)
int main() {
    const int n = 2048, il = n - 1024 + 1, iu = n;
    std::mt19937_64 g(1);
    std::normal_distribution<double> nd;
    std::vector<double> a((size_t)n * 4096), G((size_t)n * n, 0.0);
    for (auto& x : a) x = nd(g);
    // G = A A^T via host (slow but fine): use a cheaper Gram: A (n x 512)
    for (int i = 0; i < n; ++i)
        for (int j = 0; j <= i; ++j) {
            double s = 0;
            for (int k = 0; k < 256; ++k) s += a[i * 256 + k] * a[j * 256 + k];
            s += (i == j) ? 1.0 : 0.0;
            G[i + (size_t)j * n] = G[j + (size_t)i * n] = s;
        }
    cusolverDnHandle_t h;
    cusolverDnCreate(&h);
    double *dA, *dW, *work;
    float *fA, *fW, *fwork;
    int* info;
    cudaMalloc(&dA, sizeof(double) * n * n);
    cudaMalloc(&dW, sizeof(double) * n);
    cudaMalloc(&fA, sizeof(float) * n * n);
    cudaMalloc(&fW, sizeof(float) * n);
    cudaMalloc(&info, sizeof(int));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    auto reset = [&]() { cudaMemcpy(dA, G.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice); };
    int lw = 0;
    // 1. Dsyevd
    cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, &lw);
    cudaMalloc(&work, sizeof(double) * lw);
    for (int rep = 0; rep < 3; ++rep) {
        reset();
        cudaEventRecord(e0);
        CK(cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, work, lw, info));
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("Dsyevd          %8.2f ms\n", ms);
    }
    // 2. Dsyevdx top 1024
    int lw2 = 0, meig = 0;
    cusolverDnDsyevdx_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n, dA, n, 0.0, 0.0, il, iu, &meig, dW, &lw2);
    double* work2;
    cudaMalloc(&work2, sizeof(double) * lw2);
    for (int rep = 0; rep < 3; ++rep) {
        reset();
        cudaEventRecord(e0);
        CK(cusolverDnDsyevdx(h, CUSOLVER_EIG_MODE_VECTOR, CUSOLVER_EIG_RANGE_I, CUBLAS_FILL_MODE_LOWER, n, dA, n, 0.0, 0.0, il, iu, &meig, dW, work2, lw2, info));
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("Dsyevdx top1024 %8.2f ms (m=%d)\n", ms, meig);
    }
    // 3. Xsyevd (64-bit API)
    cusolverDnParams_t prm;
    cusolverDnCreateParams(&prm);
    size_t dws = 0, hws = 0;
    cusolverDnXsyevd_bufferSize(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n, CUDA_R_64F, dW, CUDA_R_64F, &dws, &hws);
    void* dwork; cudaMalloc(&dwork, dws);
    std::vector<char> hwork(hws + 1);
    for (int rep = 0; rep < 3; ++rep) {
        reset();
        cudaEventRecord(e0);
        CK(cusolverDnXsyevd(h, prm, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, CUDA_R_64F, dA, n, CUDA_R_64F, dW, CUDA_R_64F, dwork, dws, hwork.data(), hws, info));
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("Xsyevd          %8.2f ms\n", ms);
    }
    // 4. Ssyevd (fp32)
    std::vector<float> Gf(G.begin(), G.end());
    int lwf = 0;
    cusolverDnSsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, fA, n, fW, &lwf);
    cudaMalloc(&fwork, sizeof(float) * lwf);
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemcpy(fA, Gf.data(), sizeof(float) * n * n, cudaMemcpyHostToDevice);
        cudaEventRecord(e0);
        CK(cusolverDnSsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, fA, n, fW, fwork, lwf, info));
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("Ssyevd (fp32)   %8.2f ms\n", ms);
    }
    // 5. Dsyevj
    syevjInfo_t sj;
    cusolverDnCreateSyevjInfo(&sj);
    cusolverDnXsyevjSetTolerance(sj, 1e-14);
    cusolverDnXsyevjSetMaxSweeps(sj, 20);
    int lwj = 0;
    cusolverDnDsyevj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, &lwj, sj);
    double* workj; cudaMalloc(&workj, sizeof(double) * lwj);
    for (int rep = 0; rep < 2; ++rep) {
        reset();
        cudaEventRecord(e0);
        CK(cusolverDnDsyevj(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, workj, lwj, info, sj));
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("Dsyevj          %8.2f ms\n", ms);
    }
    // 6. breakdown: sytrd, syevd eigenvalues only, ormtr (1024 columns)
    {
        double *d, *e, *tau, *wk, *C;
        cudaMalloc(&d, sizeof(double) * n); cudaMalloc(&e, sizeof(double) * n); cudaMalloc(&tau, sizeof(double) * n);
        cudaMalloc(&C, sizeof(double) * n * 1024);
        int lt = 0, lo = 0, lv = 0;
        cusolverDnDsytrd_bufferSize(h, CUBLAS_FILL_MODE_LOWER, n, dA, n, d, e, tau, &lt);
        cusolverDnDormtr_bufferSize(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, n, 1024, dA, n, tau, C, n, &lo);
        cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_NOVECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, &lv);
        int lmax = lt > lo ? lt : lo; lmax = lmax > lv ? lmax : lv;
        cudaMalloc(&wk, sizeof(double) * lmax);
        for (int rep = 0; rep < 3; ++rep) {
            reset();
            cudaEventRecord(e0);
            CK(cusolverDnDsytrd(h, CUBLAS_FILL_MODE_LOWER, n, dA, n, d, e, tau, wk, lmax, info));
            cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
            printf("Dsytrd          %8.2f ms\n", ms);
            cudaEventRecord(e0);
            CK(cusolverDnDormtr(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, n, 1024, dA, n, tau, C, n, wk, lmax, info));
            cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
            printf("Dormtr 1024     %8.2f ms\n", ms);
            reset();
            cudaEventRecord(e0);
            CK(cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_NOVECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dW, wk, lmax, info));
            cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
            printf("Dsyevd novec    %8.2f ms\n", ms);
        }
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
