// Grid-barrier latency on the B200 (atomic counter + generation flag), by grid size.
#include <cuda/atomic>
#include <cstdio>
struct GridBar { unsigned count, gen; };
__device__ __forceinline__ void grid_barrier(GridBar* b, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> gen(b->gen), cnt(b->count);
        const unsigned g = gen.load(cuda::memory_order_relaxed);
        __threadfence();
        if (cnt.fetch_add(1u, cuda::memory_order_acq_rel) == nblocks - 1) {
            cnt.store(0u, cuda::memory_order_relaxed);
            gen.fetch_add(1u, cuda::memory_order_release);
        } else {
            while (gen.load(cuda::memory_order_acquire) == g) {}
        }
        __threadfence();
    }
    __syncthreads();
}
// variant: per-CTA flag array, CTA 0 gathers and releases
__device__ __forceinline__ void grid_barrier2(unsigned* flags, unsigned* rel, unsigned epoch, unsigned nblocks) {
    __syncthreads();
    if (blockIdx.x == 0) {
        if (threadIdx.x < nblocks && threadIdx.x > 0) {
            cuda::atomic_ref<unsigned, cuda::thread_scope_device> f(flags[threadIdx.x * 32]);
            while (f.load(cuda::memory_order_acquire) != epoch) {}
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            cuda::atomic_ref<unsigned, cuda::thread_scope_device> r(*rel);
            r.store(epoch, cuda::memory_order_release);
        }
    } else if (threadIdx.x == 0) {
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> f(flags[blockIdx.x * 32]);
        f.store(epoch, cuda::memory_order_release);
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> r(*rel);
        while (r.load(cuda::memory_order_acquire) != epoch) {}
    }
    __syncthreads();
}
// variant 3: no explicit fences, release arrival / acquire spin
__device__ __forceinline__ void grid_barrier3(GridBar* b, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> gen(b->gen), cnt(b->count);
        const unsigned g = gen.load(cuda::memory_order_relaxed);
        if (cnt.fetch_add(1u, cuda::memory_order_acq_rel) == nblocks - 1) {
            cnt.store(0u, cuda::memory_order_relaxed);
            gen.store(g + 1, cuda::memory_order_release);
        } else {
            while (gen.load(cuda::memory_order_acquire) == g) {}
        }
    }
    __syncthreads();
}
// variant 4: monotone counter (no reset): arrive with release add, spin until count >= target
__device__ __forceinline__ void grid_barrier4(unsigned* ctr, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> c(*ctr);
        c.fetch_add(1u, cuda::memory_order_release);
        while (c.load(cuda::memory_order_acquire) < target) {}
    }
    __syncthreads();
}
// variant 5: release add, relaxed spin, then one acquire fence
__device__ __forceinline__ void grid_barrier5(unsigned* ctr, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> c(*ctr);
        c.fetch_add(1u, cuda::memory_order_release);
        while (c.load(cuda::memory_order_relaxed) < target) {}
        cuda::atomic_thread_fence(cuda::memory_order_acquire, cuda::thread_scope_device);
    }
    __syncthreads();
}
// variant 6: red.release (no return) + relaxed volatile spin + fence
__device__ __forceinline__ void grid_barrier6(unsigned* ctr, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        unsigned v;
        do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
}
__global__ void k_bar5(unsigned* ctr, int iters) {
    for (int i = 0; i < iters; ++i) grid_barrier5(ctr, (unsigned)(i + 1) * gridDim.x);
}
__global__ void k_bar6(unsigned* ctr, int iters) {
    for (int i = 0; i < iters; ++i) grid_barrier6(ctr, (unsigned)(i + 1) * gridDim.x);
}
__global__ void k_bar3(GridBar* b, int iters) {
    for (int i = 0; i < iters; ++i) grid_barrier3(b, gridDim.x);
}
__global__ void k_bar4(unsigned* ctr, int iters) {
    for (int i = 0; i < iters; ++i) grid_barrier4(ctr, (unsigned)(i + 1) * gridDim.x);
}
__global__ void k_bar(GridBar* b, int iters) {
    for (int i = 0; i < iters; ++i) grid_barrier(b, gridDim.x);
}
__global__ void k_bar2(unsigned* flags, unsigned* rel, int iters) {
    for (int i = 0; i < iters; ++i) grid_barrier2(flags, rel, (unsigned)i + 1, gridDim.x);
}
int main() {
    GridBar* b; unsigned *flags, *rel;
    cudaMalloc(&b, sizeof(GridBar)); cudaMemset(b, 0, sizeof(GridBar));
    cudaMalloc(&flags, 4 * 32 * 256); cudaMalloc(&rel, 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000;
    for (int G : {8, 16, 32, 64, 128, 148}) {
        for (int v = 3; v < 6; ++v) {
            cudaMemset(flags, 0, 4 * 32 * 256); cudaMemset(rel, 0, 4);
            void* a1[] = {&b, (void*)&iters};
            void* a2[] = {&flags, &rel, (void*)&iters};
            cudaEventRecord(e0);
            if (v == 0) cudaLaunchCooperativeKernel((void*)k_bar, dim3(G), dim3(256), a1, 0, 0);
            else if (v == 1) cudaLaunchCooperativeKernel((void*)k_bar2, dim3(G), dim3(256), a2, 0, 0);
            else if (v == 2) cudaLaunchCooperativeKernel((void*)k_bar3, dim3(G), dim3(256), a1, 0, 0);
            else { void* a4[] = {&rel, (void*)&iters};
                   cudaLaunchCooperativeKernel(v == 3 ? (void*)k_bar4 : v == 4 ? (void*)k_bar5 : (void*)k_bar6, dim3(G), dim3(256), a4, 0, 0); }
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("G=%3d variant %d: %.3f us/barrier  (%s)\n", G, v, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
        }
    }
}
