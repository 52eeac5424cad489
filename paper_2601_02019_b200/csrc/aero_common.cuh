// Shared device/host helpers for the B200 AeroSketch engine.
#pragma once

#include <cuda/atomic>

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace aero_b200 {

// exception taxonomy mirrored from the reference (errors.hpp:15-33)
struct InvalidInput : std::invalid_argument {
    explicit InvalidInput(const std::string& w) : std::invalid_argument(w) {}
};
struct FormatError : std::runtime_error {  // errors.hpp: malformed stream file
    using std::runtime_error::runtime_error;
};
struct ProtocolError : std::runtime_error {
    explicit ProtocolError(const std::string& w) : std::runtime_error(w) {}
};
struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};

#define AERO_CUDA(expr)                                                                       \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess)                                                                \
            throw ::aero_b200::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

void note_launch(int n = 1);  // launch counter (aero_kernel_launches)
#define AERO_LAUNCHED()                                                                   \
    do {                                                                                  \
        ::aero_b200::note_launch();                                                       \
        cudaError_t _e = cudaGetLastError();                                              \
        if (_e != cudaSuccess)                                                            \
            throw ::aero_b200::CudaError(std::string("kernel launch: ") + cudaGetErrorString(_e)); \
    } while (0)

// ---- RngState restatement (reference rng.hpp:21-87) ------------------------
constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;

__host__ __device__ inline uint64_t mix_out(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
// stationary mix64 (rng.hpp:32-35)
__host__ __device__ inline uint64_t mix64(uint64_t x) { return mix_out(x + kGolden); }
// initial splitmix state of RngState(seed, stream) (rng.hpp:45-48)
__host__ __device__ inline uint64_t rng_state0(uint64_t seed, uint64_t stream) {
    return mix64(seed) ^ mix64(mix64(stream) + 0x632be59bd9b4e019ULL);
}
// stream id of the n-th fork (n >= 1) of a state with stream id `stream` (rng.hpp:54-57)
__host__ __device__ inline uint64_t fork_stream(uint64_t stream, uint64_t n) {
    return mix64(stream ^ mix64(n));
}
// m-th uniform draw (m >= 1) of a state: random access into the splitmix sequence
__host__ __device__ inline double rng_uniform_at(uint64_t state0, uint64_t m) {
    const uint64_t bits = mix_out(state0 + m * kGolden) >> 11;
    return static_cast<double>(bits + 1) * 0x1.0p-53;
}
// i-th gaussian (0-based) of a fresh state (Box-Muller pairs, rng.hpp:66-78)
__device__ inline double rng_gaussian_at(uint64_t state0, uint64_t i) {
    const uint64_t p = i >> 1;
    const double u1 = rng_uniform_at(state0, 2 * p + 1);
    const double u2 = rng_uniform_at(state0, 2 * p + 2);
    const double r = sqrt(-2.0 * log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    double s, c;
    sincos(a, &s, &c);
    return (i & 1) ? r * s : r * c;
}

// ---- warp / block reductions -------------------------------------------------
__device__ inline double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
// block-wide sum; `scratch` must hold blockDim.x/32 doubles; result broadcast
__device__ inline double block_sum(double v, double* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    double t = 0.0;
    for (int i = 0; i < nw; ++i) t += scratch[i];
    __syncthreads();
    return t;
}

// grid-wide barrier for persistent cooperative kernels: monotone arrival
// counter (zeroed before the launch), release-add, acquire-spin (~1.2 us on a
// B200 across both dies, tools/barrier_bench.cu)
__device__ __forceinline__ void grid_sync(unsigned* ctr, unsigned& epoch, unsigned nblocks) {
    __syncthreads();
    epoch += nblocks;
    if (threadIdx.x == 0) {
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> c(*ctr);
        c.fetch_add(1u, cuda::memory_order_release);
        // relaxed polling (an acquire load per poll would invalidate L1 under
        // the co-resident CTA every iteration), one acquire fence at the end
        while (c.load(cuda::memory_order_relaxed) < epoch) {
        }
        cuda::atomic_thread_fence(cuda::memory_order_acquire, cuda::thread_scope_device);
    }
    __syncthreads();
}

// grid barrier for kernels whose next phase reads, through the async proxy
// (cp.async.bulk), data this phase wrote with generic stores (k_iterate_i8):
// every thread orders its generic writes (global and shared) before the async
// proxy ahead of the release, and the acquiring thread fences again before its
// CTA issues bulk copies
__device__ __forceinline__ void grid_sync_async(unsigned* ctr, unsigned& epoch, unsigned nblocks) {
    asm volatile("fence.proxy.async;\n" ::: "memory");
    grid_sync(ctr, epoch, nblocks);
    asm volatile("fence.proxy.async;\n" ::: "memory");
}

}  // namespace aero_b200
