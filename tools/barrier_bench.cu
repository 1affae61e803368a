// Grid-barrier micro-benchmark (B200): time per barrier of a persistent grid
// (148 CTAs x 768 threads, one CTA per SM, like the solver) for barrier
// variants.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/barrier_bench.cu -o tools/barrier_bench
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// variant 0: the solver's barrier (red.release arrive, ld.acquire poll, fence)
// variant 1: red.release arrive, relaxed poll, one acquire fence after
// variant 2: cooperative_groups grid.sync()
// variant 3: as 0 with __nanosleep(32) in the poll loop
template <int V>
__global__ void __launch_bounds__(768, 1) k_bar(unsigned long long* ctr, int iters, unsigned long long* out) {
    __shared__ int dummy;
    unsigned gen = 0;
    auto grid = cg::this_grid();
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (V == 2) {
            grid.sync();
            continue;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned long long target = (unsigned long long)(gen + 1) * gridDim.x;
            asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
            if (V == 1) {
                while (ld_relaxed(ctr) < target) {
                }
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            } else {
                while (ld_acquire(ctr) < target) {
                    if (V == 3) __nanosleep(32);
                }
                __threadfence();
            }
            ++gen;
            dummy = gen;
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[V] = clock64() - t0;
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *ctr, *out;
    cudaMalloc(&ctr, 8);
    cudaMalloc(&out, 64);
    const int iters = 20000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    void (*ks[4])(unsigned long long*, int, unsigned long long*) = {k_bar<0>, k_bar<1>, k_bar<2>, k_bar<3>};
    const char* names[4] = {"red.release + ld.acquire poll (solver)", "red.release + relaxed poll + fence",
                            "cooperative_groups grid.sync", "solver + nanosleep(32)"};
    for (int rep = 0; rep < 2; ++rep)
        for (int v = 0; v < 4; ++v) {
            cudaMemset(ctr, 0, 8);
            int it = iters;
            void* args[] = {&ctr, &it, &out};
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)ks[v], nsm, 768, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            if (cudaGetLastError() != cudaSuccess) {
                printf("launch failed\n");
                return 1;
            }
            printf("%-42s %.3f us per barrier\n", names[v], ms * 1e3 / iters);
        }
    return 0;
}
