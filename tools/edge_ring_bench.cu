// edge_ring_bench.cu -- does a bulk-copy (TMA unit, cp.async.bulk + mbarrier) edge ring pay for the
// relax step on B200 (sm_100a)?  Best case for the ring: every 256-edge chunk is one contiguous
// 2 KB run (a hub row).  Both kernels do the relax step's work per edge -- (col, w) pair in, one
// divergent 4-byte pre-check read of dist[col], an atomicMin when the candidate improves -- and
// differ only in how the edge pairs reach the lanes:
//   lanes : 8 coalesced 8-byte ld.global.nc.L1::no_allocate per lane (what relax_step does)
//   ring  : lane 0 issues cp.async.bulk of the chunk STAGES-1 chunks ahead into the warp's
//           shared-memory ring (mbarrier complete_tx), lanes read the pairs with ld.shared.v2
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/edge_ring_bench tools/edge_ring_bench.cu
//   cuobjdump -sass tools/edge_ring_bench | grep -c UBLKCP     (the ring's bulk copies)
//   tools/edge_ring_bench [M edges, default 128] [dist MiB, default 35] [improving %, default 30]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess) {                                                   \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                               \
        }                                                                          \
    } while (0)

constexpr int kThreads = 768, kWarps = kThreads / 32, kChunk = 256, kPer = kChunk / 32;

__device__ __forceinline__ unsigned mix(unsigned x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

// edges: col skewed towards a hub prefix like a degree-sorted R-MAT (38% of the targets in the
// first 16 K ids), weight in [1, 2^20)
__global__ void k_fill_edges(uint2* e, unsigned long long m, unsigned n) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < m;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned r = mix((unsigned)i * 2654435761u + (unsigned)(i >> 32));
        const unsigned c = (r & 255u) < 97u ? (r >> 8) % 16384u : 16384u + (r >> 8) % (n - 16384u);
        e[i] = make_uint2(c, 1u + (mix(r) & 0xFFFFFu));
    }
}
// dist: a share `improve_pct` of the targets holds a value any candidate improves
__global__ void k_fill_dist(unsigned* d, unsigned n, unsigned improve_pct) {
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        d[i] = (mix(i) % 100u) < improve_pct ? 0xFFFFFFF0u : 0u;
}

__device__ __forceinline__ void relax8(const uint2 (&ed)[kPer], unsigned du, unsigned* dist) {
    unsigned cur[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) cur[j] = dist[ed[j].x];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const unsigned nd = du + ed[j].y;
        if (nd < cur[j]) atomicMin(dist + ed[j].x, nd | 0x80000000u);  // stays "improvable": steady state
    }
}

__global__ void __launch_bounds__(kThreads, 1) k_lanes(const uint2* edges, unsigned long long nchunk, unsigned* dist) {
    const int lane = threadIdx.x & 31;
    const unsigned long long gw = (unsigned long long)blockIdx.x * kWarps + (threadIdx.x >> 5);
    const unsigned long long nw = (unsigned long long)gridDim.x * kWarps;
    for (unsigned long long c = gw; c < nchunk; c += nw) {
        uint2 ed[kPer];
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const uint2* p = edges + c * kChunk + lane + 32 * j;
            asm("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(ed[j].x), "=r"(ed[j].y) : "l"(p));
        }
        relax8(ed, (unsigned)c & 0xFFFFu, dist);
    }
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int STAGES>
__global__ void __launch_bounds__(kThreads, 1) k_ring(const uint2* edges, unsigned long long nchunk, unsigned* dist) {
    extern __shared__ __align__(128) unsigned char raw[];
    // per warp: STAGES x 2 KB of pairs, then STAGES mbarriers
    uint2* ring = reinterpret_cast<uint2*>(raw) + (size_t)(threadIdx.x >> 5) * STAGES * kChunk;
    unsigned long long* bars =
        reinterpret_cast<unsigned long long*>(raw + (size_t)kWarps * STAGES * kChunk * sizeof(uint2)) +
        (threadIdx.x >> 5) * STAGES;
    const int lane = threadIdx.x & 31;
    const unsigned long long gw = (unsigned long long)blockIdx.x * kWarps + (threadIdx.x >> 5);
    const unsigned long long nw = (unsigned long long)gridDim.x * kWarps;
    if (lane == 0) {
        for (int s = 0; s < STAGES; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + s)));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // inits visible to the async proxy
    }
    __syncwarp();
    auto issue = [&](unsigned long long c, int s) {  // lane 0
        const unsigned bar = smem_u32(bars + s);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"((unsigned)(kChunk * sizeof(uint2)))
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(ring + s * kChunk)),
                     "l"(edges + c * kChunk), "r"((unsigned)(kChunk * sizeof(uint2))), "r"(bar)
                     : "memory");
    };
    // prologue: STAGES - 1 chunks in flight
    unsigned long long cn = gw;
    int sn = 0;
    if (lane == 0)
        for (int k = 0; k < STAGES - 1 && cn < nchunk; ++k, cn += nw, sn = (sn + 1) % STAGES) issue(cn, sn);
    cn = __shfl_sync(0xffffffffu, cn, 0);
    sn = __shfl_sync(0xffffffffu, sn, 0);
    int s = 0;
    unsigned phase = 0;
    for (unsigned long long c = gw; c < nchunk; c += nw) {
        // the slot refilled now was consumed one iteration ago (all lanes passed the __syncwarp)
        if (lane == 0 && cn < nchunk) issue(cn, sn);
        cn += nw;
        sn = (sn + 1) % STAGES;
        const unsigned bar = smem_u32(bars + s);
        unsigned done = 0;
        while (!done)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(bar), "r"(phase)
                : "memory");
        uint2 ed[kPer];
#pragma unroll
        for (int j = 0; j < kPer; ++j) ed[j] = ring[s * kChunk + lane + 32 * j];
        __syncwarp();  // every lane holds its pairs: the slot may be refilled
        relax8(ed, (unsigned)c & 0xFFFFu, dist);
        if (++s == STAGES) {
            s = 0;
            phase ^= 1u;
        }
    }
}

template <class F>
static float time_it(F launch) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    launch();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int i = 0; i < 5; ++i) launch();
    CK(cudaEventRecord(e1));
    CK(cudaDeviceSynchronize());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    return ms / 5;
}

template <int STAGES>
static void run_ring(const uint2* e, unsigned long long nchunk, unsigned* d, int nsm, double edges) {
    const int smem = kWarps * STAGES * (kChunk * (int)sizeof(uint2) + 8);
    CK(cudaFuncSetAttribute(k_ring<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const float ms = time_it([&] { k_ring<STAGES><<<nsm, kThreads, smem>>>(e, nchunk, d); });
    printf("ring, %d stages (%3d KB smem/CTA)   %8.3f ms  %7.1f G edges/s\n", STAGES, smem / 1024, ms,
           edges / (ms * 1e-3) / 1e9);
}

int main(int argc, char** argv) {
    const unsigned long long m = (argc > 1 ? (unsigned long long)atoll(argv[1]) : 128ull) << 20;
    const unsigned n = (argc > 2 ? (unsigned)atoi(argv[2]) : 35u) * (1u << 18);
    const unsigned pct = argc > 3 ? (unsigned)atoi(argv[3]) : 30u;
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    const int nsm = prop.multiProcessorCount;
    uint2* e;
    unsigned* d;
    CK(cudaMalloc(&e, sizeof(uint2) * m));
    CK(cudaMalloc(&d, sizeof(unsigned) * (size_t)n));
    k_fill_edges<<<nsm * 8, 256>>>(e, m, n);
    k_fill_dist<<<nsm * 8, 256>>>(d, n, pct);
    CK(cudaDeviceSynchronize());
    const unsigned long long nchunk = m / kChunk;
    printf("%s, %d SMs; %llu M edges (%.1f GB stream), dist %u MiB, %u%% of the targets improvable\n", prop.name, nsm,
           m >> 20, (double)m * 8 / 1e9, n >> 18, pct);
    const float ms = time_it([&] { k_lanes<<<nsm, kThreads>>>(e, nchunk, d); });
    printf("lanes (8 x ld.global.nc.v2 per lane)   %8.3f ms  %7.1f G edges/s\n", ms, (double)m / (ms * 1e-3) / 1e9);
    run_ring<2>(e, nchunk, d, nsm, (double)m);
    run_ring<3>(e, nchunk, d, nsm, (double)m);
    run_ring<4>(e, nchunk, d, nsm, (double)m);
    return 0;
}
