// common.cuh -- shared device helpers for the sm_100a delta-stepping library.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ds {

// Block shape of the persistent solver (warp-granular work inside; the block
// size only sets how many CTAs arrive at each grid barrier).
#ifndef DS_THREADS
#define DS_THREADS 768
#endif
#ifndef DS_MIN_BLOCKS
#define DS_MIN_BLOCKS (768 / DS_THREADS)
#endif
constexpr int kThreads = DS_THREADS;

constexpr unsigned long long kMask48 = (1ull << 48) - 1;

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// L2-coherent loads for data written by other CTAs inside the same launch
// (L1 is not coherent across SMs).
__device__ __forceinline__ unsigned ldcg(const unsigned* p) { return __ldcg(p); }
__device__ __forceinline__ int ldcg(const int* p) { return __ldcg(p); }
__device__ __forceinline__ unsigned long long ldcg(const unsigned long long* p) { return __ldcg(p); }
__device__ __forceinline__ long long ldcg(const long long* p) { return __ldcg(p); }

// Fixed-point threshold: smallest integer >= x, clamped to the INF code.
__device__ __host__ __forceinline__ unsigned ceil_u32_clamped(double x) {
    if (!(x < 4294967295.0)) return 0xFFFFFFFFu;
    double c = ceil(x);
    return c >= 4294967295.0 ? 0xFFFFFFFFu : (unsigned)c;
}

// _bucket_index_of (sssp.py:230-236): the unique i with fl(i*delta) <= v < fl((i+1)*delta).
__device__ __host__ __forceinline__ long long bucket_index_of(double value, double delta) {
    long long idx = (long long)floor(value / delta);
    while ((double)idx * delta > value) --idx;
    while ((double)(idx + 1) * delta <= value) ++idx;
    return idx;
}

}  // namespace ds
