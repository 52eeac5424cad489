// Microbenchmark: k_product (product.cu) vs cuBLAS DGEMM on the C2 shapes.
#include <cublas_v2.h>
#include <cstdio>
#include <vector>
#include <cmath>
#include "../paper_2601_02019_b200/csrc/kernels.cuh"
using namespace aero_b200;
int main() {
    cublasHandle_t hb;
    cublasCreate(&hb);
    const int cap = 2048;
    double *G, *X, *Y, *ws;
    cudaMalloc(&G, sizeof(double) * cap * cap);
    cudaMalloc(&X, sizeof(double) * cap * 192);
    cudaMalloc(&Y, sizeof(double) * cap * 192);
    size_t wsn = product_workspace_doubles(cap, 192);
    cudaMalloc(&ws, sizeof(double) * wsn);
    std::vector<double> h((size_t)cap * cap);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)((i * 2654435761ull) % 1000) / 1000.0;
    cudaMemcpy(G, h.data(), sizeof(double) * cap * cap, cudaMemcpyHostToDevice);
    cudaMemcpy(X, h.data(), sizeof(double) * cap * 192, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int R : {1024, 1536, 2000}) {
        for (int N : {32, 64, 128, 192}) {
            const double fl = 2.0 * R * (double)R * N;
            float ms = 0.f, best = 1e9f, bestc = 1e9f;
            for (int rep = 0; rep < 20; ++rep) {
                cudaEventRecord(e0);
                gemm_product(0, R, N, R, G, cap, X, cap, Y, cap, nullptr, ws, wsn);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
                best = ms < best ? ms : best;
                const double one = 1.0, zero = 0.0;
                cudaEventRecord(e0);
                cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, R, N, R, &one, G, cap, X, cap, &zero, Y, cap);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
                bestc = ms < bestc ? ms : bestc;
            }
            // correctness vs cuBLAS
            double *Y2;
            cudaMalloc(&Y2, sizeof(double) * cap * N);
            gemm_product(0, R, N, R, G, cap, X, cap, Y2, cap, nullptr, ws, wsn);
            const double one = 1.0, zero = 0.0;
            cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, R, N, R, &one, G, cap, X, cap, &zero, Y, cap);
            std::vector<double> h1((size_t)cap * N), h2((size_t)cap * N);
            cudaMemcpy(h1.data(), Y, sizeof(double) * cap * N, cudaMemcpyDeviceToHost);
            cudaMemcpy(h2.data(), Y2, sizeof(double) * cap * N, cudaMemcpyDeviceToHost);
            double md = 0, mx = 0;
            for (int j = 0; j < N; ++j)
                for (int i = 0; i < R; ++i) {
                    md = fmax(md, fabs(h1[i + (size_t)j * cap] - h2[i + (size_t)j * cap]));
                    mx = fmax(mx, fabs(h1[i + (size_t)j * cap]));
                }
            cudaFree(Y2);
            printf("R=%4d N=%3d  ours %7.1f us %6.2f TF/s   cublas %7.1f us %6.2f TF/s  relmax %.1e\n", R, N,
                   best * 1e3, fl / (best * 1e-3) / 1e12, bestc * 1e3, fl / (bestc * 1e-3) / 1e12, md / mx);
        }
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
