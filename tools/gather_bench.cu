// gather_bench.cu -- per-SM rate of divergent 4-byte reads on B200 (sm_100a), the access the
// relax step's pre-check makes once per edge.  Compares the global-load paths (L1-allocating,
// L2-only, non-coherent), the texture path, shared memory, and a mix where a share of the lanes
// is served from shared memory (a hub cache) and the rest from global memory.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/gather_bench tools/gather_bench.cu
//   tools/gather_bench [array MiB, default 35] [hub entries, default 16384]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess) {                                                   \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                               \
        }                                                                          \
    } while (0)

constexpr int kThreads = 768;
constexpr int kPer = 8;      // independent loads in flight per lane and round
constexpr int kRounds = 64;  // rounds per thread

__device__ __forceinline__ unsigned mix(unsigned x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

// skewed index: with probability hub_pct/256 the target is one of the first `hub` entries
__device__ __forceinline__ unsigned pick(unsigned h, unsigned n, unsigned hub, unsigned hub_pct) {
    const unsigned r = mix(h);
    if ((r & 255u) < hub_pct) return (r >> 8) % hub;
    return hub + (r >> 8) % (n - hub);
}

enum Path { LDG_CA = 0, LDG_CG = 1, LDG_NC = 2, TEX = 3, MIXED = 4, LDS_ONLY = 5 };

template <int PATH>
__global__ void __launch_bounds__(kThreads, 1)
k_gather(const unsigned* __restrict__ a, cudaTextureObject_t tex, unsigned n, unsigned hub, unsigned hub_pct,
         unsigned long long* out) {
    extern __shared__ unsigned sh[];
    if (PATH == MIXED || PATH == LDS_ONLY) {
        for (unsigned i = threadIdx.x; i < hub; i += kThreads) sh[i] = a[i];
        __syncthreads();
    }
    const unsigned tid = blockIdx.x * kThreads + threadIdx.x;
    unsigned long long acc = 0;
    for (int r = 0; r < kRounds; ++r) {
        unsigned v[kPer];
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const unsigned i = pick(tid * 2654435761u + (unsigned)(r * kPer + j) * 40503u, n, hub, hub_pct);
            if (PATH == LDG_CA) {
                v[j] = a[i];
            } else if (PATH == LDG_CG) {
                v[j] = __ldcg(a + i);
            } else if (PATH == LDG_NC) {
                v[j] = __ldg(a + i);
            } else if (PATH == TEX) {
                v[j] = tex1Dfetch<unsigned>(tex, (int)i);
            } else if (PATH == MIXED) {
                v[j] = i < hub ? sh[i] : __ldcg(a + i);
            } else {
                v[j] = sh[i % hub];
            }
        }
#pragma unroll
        for (int j = 0; j < kPer; ++j) acc += v[j];
    }
    if (acc == 0x123456789ull) out[0] = acc;  // keep the loads
}

template <int PATH>
static void run(const char* name, const unsigned* a, cudaTextureObject_t tex, unsigned n, unsigned hub,
                unsigned hub_pct, unsigned long long* out, int nsm, float mhz) {
    const size_t smem = (PATH == MIXED || PATH == LDS_ONLY) ? hub * sizeof(unsigned) : 0;
    CK(cudaFuncSetAttribute(k_gather<PATH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    k_gather<PATH><<<nsm, kThreads, smem>>>(a, tex, n, hub, hub_pct, out);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    const int reps = 5;
    for (int i = 0; i < reps; ++i) k_gather<PATH><<<nsm, kThreads, smem>>>(a, tex, n, hub, hub_pct, out);
    CK(cudaEventRecord(e1));
    CK(cudaDeviceSynchronize());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= reps;
    const double loads = (double)nsm * kThreads * kRounds * kPer;
    const double gps = loads / (ms * 1e-3) / 1e9;
    printf("%-34s hub%%=%3u  %8.3f ms  %7.1f G reads/s  %5.2f cycles per lane-read per SM\n", name,
           hub_pct * 100 / 256, ms, gps, (double)nsm * mhz * 1e6 / (gps * 1e9));
}

int main(int argc, char** argv) {
    const unsigned mib = argc > 1 ? (unsigned)atoi(argv[1]) : 35;
    const unsigned hub = argc > 2 ? (unsigned)atoi(argv[2]) : 16384;
    const unsigned n = mib * (1u << 18);
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    int khz = 0;
    CK(cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0));
    const float mhz = khz / 1000.f;
    printf("%s, %d SMs, %.0f MHz nominal; array %u MiB (%u words), hub %u entries\n", prop.name,
           prop.multiProcessorCount, mhz, mib, n, hub);
    unsigned* a;
    unsigned long long* out;
    CK(cudaMalloc(&a, sizeof(unsigned) * (size_t)n));
    CK(cudaMalloc(&out, 8));
    CK(cudaMemset(a, 1, sizeof(unsigned) * (size_t)n));
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = a;
    rd.res.linear.desc = cudaCreateChannelDesc<unsigned>();
    rd.res.linear.sizeInBytes = sizeof(unsigned) * (size_t)n;
    cudaTextureDesc td{};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex = 0;
    CK(cudaCreateTextureObject(&tex, &rd, &td, nullptr));
    const int nsm = prop.multiProcessorCount;
    for (unsigned pct : {0u, 72u, 97u}) {  // share of the reads aimed at the hub prefix: 0 / 28% / 38%
        run<LDG_CA>("ld.global (L1 allocating)", a, tex, n, hub, pct, out, nsm, mhz);
        run<LDG_CG>("ld.global.cg (L2 only)", a, tex, n, hub, pct, out, nsm, mhz);
        run<LDG_NC>("ld.global.nc", a, tex, n, hub, pct, out, nsm, mhz);
        run<TEX>("tex1Dfetch", a, tex, n, hub, pct, out, nsm, mhz);
        run<MIXED>("hub from smem, rest ld.global.cg", a, tex, n, hub, pct, out, nsm, mhz);
    }
    run<LDS_ONLY>("shared memory only", a, tex, n, hub, 0, out, nsm, mhz);
    return 0;
}
