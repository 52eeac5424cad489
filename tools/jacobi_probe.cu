// Standalone probe: sweeps and time of the one-CTA Jacobi (kernels.cu).
#include "../paper_2601_02019_b200/csrc/kernels.cu"
#include <cstdio>
#include <random>
#include <vector>
using namespace aero_b200;
int main() {
    for (int n : {8, 16, 32, 64, 96}) {
        std::mt19937_64 g(1);
        std::normal_distribution<double> nd;
        std::vector<double> a((size_t)(n + 5) * n), b((size_t)n * n, 0.0);
        for (auto& x : a) x = nd(g);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                for (int r = 0; r < n + 5; ++r) b[i + j * n] += a[r * n + i] * a[r * n + j];
        double *dA, *dw;
        cudaMalloc(&dA, sizeof(double) * n * n);
        cudaMalloc(&dw, sizeof(double) * n);
        int zero = 0;
        float best = 1e9;
        int sw = 0;
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemcpy(dA, b.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice);
            cudaMemcpyToSymbol(g_jacobi_sweeps, &zero, sizeof(int));
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            eigh_small(0, n, dA, n, dw, 1, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
            cudaMemcpyFromSymbol(&sw, g_jacobi_sweeps, sizeof(int));
        }
        printf("n=%d sweeps=%d ms=%.3f err=%s\n", n, sw, best, cudaGetErrorString(cudaGetLastError()));
    }
}
