// gen.cu -- on-device synthetic R-MAT construction.
//
// Bit-identical to paper_1911_06895_b200.graphs.rmat (counter-based
// splitmix64 per (edge, level); Graph500 quadrant thresholds as 32-bit
// integers; bijective vertex scramble; weight per undirected pair).  Builds
// symmetrised + deduplicated CSR with CUB radix sort / unique and hands the
// arrays to a new graph handle without a host round trip.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include "../../include/dsssp.h"

int ds_internal_adopt(ds_graph** out, int device, void* stream, long long n, long long nnz,
                      long long* indptr, int* col, double* w);
int ds_internal_set_err(int code, const char* msg);

namespace {

constexpr unsigned long long kGolden = 0x9E3779B97F4A7C15ull;
// int(p * 2**32) for a, b, c = .57, .19, .19 (graphs.RMAT_A/B/C)
constexpr long long kA = 2448131358LL;
constexpr long long kB = 816043786LL;
constexpr long long kC = 816043786LL;

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
    unsigned long long z = x + kGolden;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ unsigned long long scramble(unsigned long long v, int scale,
                                                       unsigned long long seed) {
    const unsigned long long mask = (1ull << scale) - 1;
    const int half = max(1, (scale + 1) / 2);
    unsigned long long x = (v * (kGolden | 1ull)) & mask;
    x ^= x >> half;
    x = (x * 0xD6E8FEB86659FD93ull) & mask;
    x ^= x >> half;
    x = (x + seed * 0x632BE59BD9B4E019ull) & mask;
    return x;
}

__global__ void k_rmat_keys(long long m, int scale, unsigned long long seed,
                            unsigned long long* keys) {
    const unsigned long long sentinel = (1ull << scale) << 32;  // > every valid key
    const unsigned long long seed_mix = seed * kGolden;
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < m;
         k += (long long)gridDim.x * blockDim.x) {
        unsigned long long s = 0, d = 0;
        for (int level = 0; level < scale; ++level) {
            const unsigned long long h =
                splitmix64(((unsigned long long)k * 64ull + (unsigned long long)level) ^ seed_mix);
            const long long r = (long long)(h >> 32);
            const unsigned long long bit = 1ull << (scale - 1 - level);
            if (r >= kA + kB) s |= bit;
            if ((r >= kA && r < kA + kB) || r >= kA + kB + kC) d |= bit;
        }
        s = scramble(s, scale, seed);
        d = scramble(d, scale, seed);
        if (s == d) {
            keys[2 * k] = sentinel;
            keys[2 * k + 1] = sentinel;
        } else {
            keys[2 * k] = (s << 32) | d;
            keys[2 * k + 1] = (d << 32) | s;
        }
    }
}

__global__ void k_rmat_csr(const unsigned long long* keys, long long m, long long n,
                           unsigned long long wseed, long long* indptr, int* col, double* w) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long key = keys[i];
        const long long u = (long long)(key >> 32);
        const unsigned long long v = key & 0xFFFFFFFFull;
        const long long uprev = i == 0 ? -1 : (long long)(keys[i - 1] >> 32);
        for (long long r = uprev + 1; r <= u; ++r) indptr[r] = i;
        if (i == m - 1)
            for (long long r = u + 1; r <= n; ++r) indptr[r] = m;
        col[i] = (int)v;
        const unsigned long long lo = (unsigned long long)u < v ? (unsigned long long)u : v;
        const unsigned long long hi = (unsigned long long)u < v ? v : (unsigned long long)u;
        const unsigned long long h = splitmix64(((lo << 32) | hi) ^ (wseed * 0xD1B54A32D192ED03ull));
        unsigned long long kq = h >> 40;
        if (kq == 0) kq = 1;
        w[i] = ldexp((double)kq, -24);
    }
}

__global__ void k_fill_indptr_empty(long long* indptr, long long n) {
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r <= n;
         r += (long long)gridDim.x * blockDim.x)
        indptr[r] = 0;
}

}  // namespace

#define GCK(call)                                                               \
    do {                                                                        \
        cudaError_t e_ = (call);                                                \
        if (e_ != cudaSuccess) {                                                \
            rc = ds_internal_set_err(e_ == cudaErrorMemoryAllocation ? DS_ENOMEM \
                                                                     : DS_ECUDA, \
                                     cudaGetErrorString(e_));                   \
            goto cleanup;                                                       \
        }                                                                       \
    } while (0)

extern "C" int ds_gen_rmat(int32_t scale, int32_t edge_factor, uint64_t seed, uint64_t weight_seed,
                           int device, void* stream, ds_graph** out) {
    if (!out) return ds_internal_set_err(DS_EINVAL, "null output handle");
    if (scale < 1 || scale > 30 || edge_factor < 1)
        return ds_internal_set_err(DS_EINVAL, "scale must be in [1, 30] and edge_factor >= 1");
    int rc = DS_OK;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaStream_t st = (cudaStream_t)stream;
    const long long n = 1LL << scale;
    const long long m = (long long)edge_factor << scale;
    const long long m2 = 2 * m;
    unsigned long long *keys = nullptr, *keys2 = nullptr, *uniq = nullptr, *nsel = nullptr;
    void* tmp = nullptr;
    size_t tbytes = 0, t2 = 0;
    long long* indptr = nullptr;
    int* col = nullptr;
    double* w = nullptr;
    unsigned long long h_nsel = 0, h_last = 0;
    long long nnz = 0;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    const unsigned grid = (unsigned)nsm * 8;
    const int end_bit = 32 + scale + 1;
    GCK(cudaMalloc(&keys, sizeof(unsigned long long) * m2));
    GCK(cudaMalloc(&keys2, sizeof(unsigned long long) * m2));
    k_rmat_keys<<<grid, 256, 0, st>>>(m, scale, seed, keys);
    GCK(cudaGetLastError());
    {
        cub::DoubleBuffer<unsigned long long> db(keys, keys2);
        GCK(cub::DeviceRadixSort::SortKeys(nullptr, tbytes, db, m2, 0, end_bit, st));
        GCK(cub::DeviceSelect::Unique(nullptr, t2, keys, keys2, nsel, m2, st));
        tbytes = tbytes > t2 ? tbytes : t2;
        GCK(cudaMalloc(&tmp, tbytes));
        GCK(cub::DeviceRadixSort::SortKeys(tmp, tbytes, db, m2, 0, end_bit, st));
        unsigned long long* sorted = db.Current();
        uniq = db.Alternate();
        GCK(cudaMalloc(&nsel, sizeof(unsigned long long)));
        GCK(cub::DeviceSelect::Unique(tmp, tbytes, sorted, uniq, nsel, m2, st));
        GCK(cudaMemcpyAsync(&h_nsel, nsel, sizeof(h_nsel), cudaMemcpyDeviceToHost, st));
        GCK(cudaStreamSynchronize(st));
        if (h_nsel > 0) {
            GCK(cudaMemcpyAsync(&h_last, uniq + (h_nsel - 1), sizeof(h_last), cudaMemcpyDeviceToHost, st));
            GCK(cudaStreamSynchronize(st));
        }
        nnz = (long long)h_nsel;
        if (nnz > 0 && (h_last >> 32) >= (unsigned long long)n) --nnz;  // drop the self-loop sentinel
        GCK(cudaMalloc(&indptr, sizeof(long long) * (n + 1)));
        GCK(cudaMalloc(&col, sizeof(int) * (nnz > 0 ? nnz : 1)));
        GCK(cudaMalloc(&w, sizeof(double) * (nnz > 0 ? nnz : 1)));
        if (nnz > 0) {
            k_rmat_csr<<<grid, 256, 0, st>>>(uniq, nnz, n, weight_seed, indptr, col, w);
        } else {
            k_fill_indptr_empty<<<grid, 256, 0, st>>>(indptr, n);
        }
        GCK(cudaGetLastError());
        GCK(cudaStreamSynchronize(st));
        // sorted/uniq alias keys/keys2; both freed below
    }
    cudaFree(keys);
    cudaFree(keys2);
    cudaFree(tmp);
    cudaFree(nsel);
    keys = keys2 = nsel = nullptr;
    tmp = nullptr;
    rc = ds_internal_adopt(out, device, stream, n, nnz, indptr, col, w);
    if (rc == DS_OK) {
        indptr = nullptr;
        col = nullptr;
        w = nullptr;
    }
cleanup:
    if (keys) cudaFree(keys);
    if (keys2) cudaFree(keys2);
    if (tmp) cudaFree(tmp);
    if (nsel) cudaFree(nsel);
    if (rc != DS_OK) {
        if (indptr) cudaFree(indptr);
        if (col) cudaFree(col);
        if (w) cudaFree(w);
    }
    cudaSetDevice(prev);
    return rc;
}
