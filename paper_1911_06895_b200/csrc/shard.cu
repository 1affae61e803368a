// shard.cu -- one rank's part of the 1-D vertex-partitioned delta-stepping
// solver ("destination owner computes").
//
// Rank r owns the vertex range [v0, v0 + n_local) of the input ids and stores
// every edge (u -> v) whose TARGET v it owns, as a CSR over all n_global
// sources (rows = global source ids, columns = local target ids).  Each phase
// the host exchanges the global frontier (ids + captured values) between
// ranks (NCCL all-gather over NVLink, or gloo), and every rank pushes the
// frontier's edges into its own targets with local atomics only.  Heavy
// phases need no data exchange: every rank accumulated the same S from the
// exchanged frontiers.  The control decisions (bucket index, phase loop,
// termination) are made identically on every rank from all-reduced scalars,
// so distances and counters equal the single-GPU solver's.
//
// The step kernels are plain launches driven from the host (one exchange per
// phase is a host-visible synchronisation point anyway); the push reuses the
// single-GPU solver's edge-balanced capture/relax device code.
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "../../include/dsssp.h"
#include "common.cuh"
#include "sssp_kernel.cuh"

using namespace ds;

int ds_internal_set_err(int code, const char* msg);

#define SCK(call)                                                                         \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return ds_internal_set_err(                                                   \
                e_ == cudaErrorMemoryAllocation ? DS_ENOMEM : DS_ECUDA, cudaGetErrorString(e_)); \
    } while (0)

struct ds_shard {
    int device = 0;
    unsigned long long launches = 0;  // solver kernels launched (begin .. result)
    cudaStream_t stream = nullptr;
    long long n = 0, v0 = 0, nl = 0, nnz = 0;  // global n, owned range, local edges
    int nsm = 148;
    long long* indptr = nullptr;  // n + 1, rows = global sources
    int* col = nullptr;           // local target ids
    double* w = nullptr;
    // split
    bool prepared = false;
    double delta = 0;
    int mode = DS_MODE_FIXED32, frac = 0;
    long long nL = 0, nH = 0;
    long long* Lptr = nullptr;
    long long* Hptr = nullptr;
    void* Ledges = nullptr;
    void* Hedges = nullptr;
    // state
    void* dist = nullptr;       // nl entries of D
    unsigned* fbits = nullptr;  // nl/32 + 1 words
    unsigned* sbits = nullptr;  // n/32 + 1 words (global S membership)
    unsigned long long* sval = nullptr;  // n entries: S values (u64, D-widened)
    int* slist = nullptr;                // n entries
    unsigned long long* counters = nullptr;  // device scalars
    unsigned long long h_counters[8];
    long long scount = 0;
    int* tmp_ids = nullptr;             // nl
    unsigned long long* tmp_vals = nullptr;  // nl
    long long* cnt_scratch = nullptr;
    // edge-balanced push (the single-GPU solver's capture/relax machinery)
    long long* Rpre = nullptr;   // n entries
    long long* Rbase = nullptr;  // n entries
    void* Rd = nullptr;          // n entries of D
    unsigned* chunk_start = nullptr;
    StepSlot* slot = nullptr;
    int grid_fixed = 0, grid_f64 = 0;
};

namespace {

constexpr int kT = 256;

template <class M>
__global__ void k_shard_init(typename M::D* dist, long long nl, long long src_local) {
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nl;
         v += (long long)gridDim.x * blockDim.x)
        dist[v] = (v == src_local) ? (typename M::D)0 : M::INF;
}

// local bucket extraction: owned vertices with L <= d < H (global ids + values)
// and the minimum owned value >= H
template <class M>
__global__ void k_shard_scan(const typename M::D* dist, long long nl, long long v0, typename M::D L,
                             typename M::D H, int* out_ids, unsigned long long* out_vals,
                             unsigned long long* counters) {
    using D = typename M::D;
    unsigned long long mn = ~0ull;
    const int lane = threadIdx.x & 31;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v - lane < nl;
         v += (long long)gridDim.x * blockDim.x) {
        const D d = v < nl ? dist[v] : M::INF;
        const bool in = v < nl && d >= L && d < H;
        if (v < nl && d >= H && d != M::INF && (unsigned long long)d < mn) mn = (unsigned long long)d;
        const unsigned m = __ballot_sync(0xffffffffu, in);
        if (m) {
            unsigned long long b = 0;
            if (lane == 0) b = atomicAdd(&counters[0], (unsigned long long)__popc(m));
            b = __shfl_sync(0xffffffffu, b, 0);
            if (in) {
                const unsigned pos = (unsigned)b + __popc(m & ((1u << lane) - 1u));
                out_ids[pos] = (int)(v + v0);
                out_vals[pos] = (unsigned long long)d;
            }
        }
    }
    mn = warp_min(mn);
    if (lane == 0 && mn != ~0ull) atomicMin(&counters[1], mn);
}

// add an exchanged frontier to S (bitmap dedup) with its captured values
__global__ void k_shard_s_add(const int* ids, const unsigned long long* vals, long long count,
                              unsigned* sbits, unsigned long long* sval, int* slist,
                              unsigned long long* counters) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x) {
        const int u = ids[i];
        sval[u] = vals[i];  // a later frontier carries the smaller, current value
        if (claim_bit(sbits, (unsigned)u)) slist[atomicAdd(&counters[2], 1ull)] = u;
    }
}

__global__ void k_shard_s_clear(const int* slist, long long count, unsigned* sbits) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned u = (unsigned)slist[i];
        sbits[u >> 5] = 0u;
    }
}

__global__ void k_shard_gather_s(const int* slist, long long count, const unsigned long long* sval,
                                 unsigned long long* out_vals) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x)
        out_vals[i] = sval[slist[i]];
}

// next frontier: local ids -> global ids + final values; clear their dedup bits
template <class M>
__global__ void k_shard_emit(const int* local, long long count, const typename M::D* dist, long long v0,
                             unsigned* fbits, int* out_ids, unsigned long long* out_vals) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x) {
        const int v = local[i];
        out_ids[i] = (int)(v + v0);
        out_vals[i] = (unsigned long long)dist[v];
        fbits[(unsigned)v >> 5] = 0u;
    }
}

template <class M>
__global__ void k_shard_result(const typename M::D* dist, long long nl, int frac, double* out) {
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < nl;
         v += (long long)gridDim.x * blockDim.x)
        out[v] = M::to_f64(dist[v], frac);
}

__device__ __forceinline__ bool sh_light(double w, double delta) { return w > 0.0 && w <= delta; }
__device__ __forceinline__ bool sh_heavy(double w, double delta) { return w > delta && w < CUDART_INF; }

__global__ void k_shard_probe(const double* w, long long nnz, double delta, unsigned long long* out) {
    // out: [0] min light bits, [1] max weight bits, [2] max frac bits, [3] nL, [4] nH
    unsigned long long mn = ~0ull, mx = 0, nl = 0, nh = 0;
    int frac = 0;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz;
         e += (long long)gridDim.x * blockDim.x) {
        const double x = w[e];
        const bool L = sh_light(x, delta), H = sh_heavy(x, delta);
        nl += L;
        nh += H;
        if (L || H) {
            const unsigned long long b = (unsigned long long)__double_as_longlong(x);
            if (L && b < mn) mn = b;
            if (b > mx) mx = b;
            const int ex = (int)((b >> 52) & 0x7FF);
            unsigned long long m = b & ((1ull << 52) - 1);
            int e2;
            if (ex == 0) e2 = -1074;
            else {
                m |= 1ull << 52;
                e2 = ex - 1075;
            }
            const int low = e2 + (__ffsll((long long)m) - 1);
            frac = max(frac, low < 0 ? -low : 0);
        }
    }
    mn = warp_min(mn);
    mx = warp_max(mx);
    nl = warp_sum(nl);
    nh = warp_sum(nh);
    for (int o = 16; o; o >>= 1) frac = max(frac, __shfl_xor_sync(0xffffffffu, frac, o));
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&out[0], mn);
        atomicMax(&out[1], mx);
        atomicMax(&out[2], (unsigned long long)frac);
        atomicAdd(&out[3], nl);
        atomicAdd(&out[4], nh);
    }
}

__global__ void k_shard_count(long long n, const long long* indptr, const double* w, double delta,
                              long long* Lc, long long* Hc) {
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n;
         r += (long long)gridDim.x * blockDim.x) {
        long long l = 0, h = 0;
        for (long long e = indptr[r]; e < indptr[r + 1]; ++e) {
            l += sh_light(w[e], delta);
            h += sh_heavy(w[e], delta);
        }
        Lc[r] = l;
        Hc[r] = h;
    }
}

template <class Edge>
__device__ __forceinline__ Edge make_e(int c, double x, int frac);
template <>
__device__ __forceinline__ uint2 make_e<uint2>(int c, double x, int frac) {
    return make_uint2((unsigned)c, (unsigned)ldexp(x, frac));
}
template <>
__device__ __forceinline__ EdgeF64 make_e<EdgeF64>(int c, double x, int) {
    EdgeF64 e;
    e.col = (unsigned)c;
    e.pad = 0;
    e.w = x;
    return e;
}

template <class Edge>
__global__ void k_shard_scatter(long long n, const long long* indptr, const int* col, const double* w,
                                double delta, int frac, const long long* Lptr, const long long* Hptr,
                                Edge* Lo, Edge* Ho) {
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n;
         r += (long long)gridDim.x * blockDim.x) {
        long long l = Lptr[r], h = Hptr[r];
        for (long long e = indptr[r]; e < indptr[r + 1]; ++e) {
            const double x = w[e];
            if (sh_light(x, delta)) Lo[l++] = make_e<Edge>(col[e], x, frac);
            else if (sh_heavy(x, delta)) Ho[h++] = make_e<Edge>(col[e], x, frac);
        }
    }
}

// Capture of an exchanged frontier (global source ids + u64-widened values):
// degrees from the shard's CSR rows, entries + chunk map for relax_step.
template <class M>
__global__ void __launch_bounds__(kThreads) k_shard_capture(const KParams<M> p, StepSlot* slot,
                                                            const int* ids,
                                                            const unsigned long long* vals,
                                                            long long count, const long long* ptr) {
    using D = typename M::D;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const unsigned long long per_chunk = 32ull * kListPer;
    const unsigned long long nchunk = ((unsigned long long)count + per_chunk - 1) / per_chunk;
    const unsigned long long gw = (unsigned long long)blockIdx.x * kWarps + wib;
    const unsigned long long nw = (unsigned long long)gridDim.x * kWarps;
    for (unsigned long long c = gw; c < nchunk; c += nw) {
        D dv[kListPer];
        long long off[kListPer], deg[kListPer];
#pragma unroll
        for (int j = 0; j < kListPer; ++j) {
            const unsigned long long idx = c * per_chunk + lane + 32ull * j;
            const bool in = idx < (unsigned long long)count;
            const int u = in ? ids[idx] : 0;
            dv[j] = in ? (D)vals[idx] : (D)0;
            off[j] = in ? __ldg(ptr + u) : 0;
            deg[j] = in ? __ldg(ptr + u + 1) - off[j] : 0;
        }
        capture_emit<M, kListPer>(p, slot, lane, dv, off, deg);
    }
}

template <class M, bool LIGHT>
__global__ void __launch_bounds__(kThreads) k_shard_relax(const KParams<M> p, StepSlot* slot,
                                                          unsigned long long E, unsigned long long Rc,
                                                          const typename M::Edge* edges,
                                                          typename M::D H, int* out_list,
                                                          unsigned* fbits) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem<typename M::D>& sm = *reinterpret_cast<Smem<typename M::D>*>(smem_raw);
    relax_step<M, LIGHT>(p, sm, slot, E, Rc, edges, H, out_list, fbits);
}

}  // namespace

static unsigned sgrid(ds_shard* s) { return (unsigned)(s->nsm * 8); }

extern "C" int ds_shard_create(int64_t n_global, int64_t v0, int64_t n_local, int64_t nnz,
                               const int64_t* indptr, const int32_t* col_local, const double* val,
                               int device, void* stream, ds_shard** out) {
    if (!out) return ds_internal_set_err(DS_EINVAL, "null output handle");
    if (n_global < 1 || v0 < 0 || n_local < 0 || v0 + n_local > n_global || nnz < 0)
        return ds_internal_set_err(DS_EINVAL, "bad shard geometry");
    cudaSetDevice(device);
    ds_shard* s = new ds_shard();
    s->device = device;
    s->stream = (cudaStream_t)stream;
    s->n = n_global;
    s->v0 = v0;
    s->nl = n_local;
    s->nnz = nnz;
    cudaDeviceGetAttribute(&s->nsm, cudaDevAttrMultiProcessorCount, device);
    const long long nl1 = std::max<long long>(n_local, 1LL);
    auto fail = [&](int rc) {
        ds_shard_destroy(s);
        return rc;
    };
#define SCF(call)                                                                          \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return fail(ds_internal_set_err(e_ == cudaErrorMemoryAllocation ? DS_ENOMEM     \
                                                                            : DS_ECUDA,     \
                                            cudaGetErrorString(e_)));                      \
    } while (0)
    SCF(cudaMalloc(&s->indptr, sizeof(long long) * (n_global + 1)));
    SCF(cudaMalloc(&s->col, sizeof(int) * std::max<long long>(nnz, 1LL)));
    SCF(cudaMalloc(&s->w, sizeof(double) * std::max<long long>(nnz, 1LL)));
    SCF(cudaMemcpyAsync(s->indptr, indptr, sizeof(long long) * (n_global + 1), cudaMemcpyDefault,
                        s->stream));
    if (nnz) {
        SCF(cudaMemcpyAsync(s->col, col_local, sizeof(int) * nnz, cudaMemcpyDefault, s->stream));
        SCF(cudaMemcpyAsync(s->w, val, sizeof(double) * nnz, cudaMemcpyDefault, s->stream));
    }
    SCF(cudaMalloc(&s->Lptr, sizeof(long long) * (n_global + 1)));
    SCF(cudaMalloc(&s->Hptr, sizeof(long long) * (n_global + 1)));
    SCF(cudaMalloc(&s->dist, sizeof(unsigned long long) * nl1));
    SCF(cudaMalloc(&s->fbits, sizeof(unsigned) * (nl1 / 32 + 1)));
    SCF(cudaMalloc(&s->sbits, sizeof(unsigned) * (n_global / 32 + 1)));
    SCF(cudaMalloc(&s->sval, sizeof(unsigned long long) * n_global));
    SCF(cudaMalloc(&s->slist, sizeof(int) * n_global));
    SCF(cudaMalloc(&s->counters, sizeof(unsigned long long) * 8));
    SCF(cudaMalloc(&s->tmp_ids, sizeof(int) * nl1));
    SCF(cudaMalloc(&s->tmp_vals, sizeof(unsigned long long) * nl1));
    SCF(cudaMalloc(&s->cnt_scratch, sizeof(long long) * 2 * (n_global + 1)));
    SCF(cudaMalloc(&s->Rpre, sizeof(long long) * n_global));
    SCF(cudaMalloc(&s->Rbase, sizeof(long long) * n_global));
    SCF(cudaMalloc(&s->Rd, sizeof(unsigned long long) * n_global));
    SCF(cudaMalloc(&s->chunk_start, sizeof(unsigned) * (std::max<long long>(nnz, 1LL) / kChunk + 4)));
    SCF(cudaMalloc(&s->slot, sizeof(StepSlot)));
    SCF(cudaFuncSetAttribute(k_shard_relax<ModeFixed, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(Smem<unsigned>)));
    SCF(cudaFuncSetAttribute(k_shard_relax<ModeFixed, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(Smem<unsigned>)));
    SCF(cudaFuncSetAttribute(k_shard_relax<ModeF64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(Smem<unsigned long long>)));
    SCF(cudaFuncSetAttribute(k_shard_relax<ModeF64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(Smem<unsigned long long>)));
    SCF(cudaMemsetAsync(s->fbits, 0, sizeof(unsigned) * (nl1 / 32 + 1), s->stream));
    SCF(cudaMemsetAsync(s->sbits, 0, sizeof(unsigned) * (n_global / 32 + 1), s->stream));
    SCF(cudaStreamSynchronize(s->stream));
#undef SCF
    *out = s;
    return DS_OK;
}

extern "C" void ds_shard_destroy(ds_shard* s) {
    if (!s) return;
    cudaSetDevice(s->device);
    cudaStreamSynchronize(s->stream);
    void* ptrs[] = {s->indptr, s->col, s->w, s->Lptr, s->Hptr, s->Ledges, s->Hedges, s->dist,
                    s->fbits, s->sbits, s->sval, s->slist, s->counters, s->tmp_ids, s->tmp_vals,
                    s->cnt_scratch, s->Rpre, s->Rbase, s->Rd, s->chunk_start, s->slot};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    delete s;
}

extern "C" int ds_shard_probe(ds_shard* s, double delta, uint64_t* out5) {
    if (!s) return ds_internal_set_err(DS_EINVAL, "null shard");
    cudaSetDevice(s->device);
    unsigned long long init[5] = {~0ull, 0, 0, 0, 0};
    SCK(cudaMemcpyAsync(s->counters, init, sizeof(init), cudaMemcpyHostToDevice, s->stream));
    if (s->nnz) k_shard_probe<<<sgrid(s), kT, 0, s->stream>>>(s->w, s->nnz, delta, s->counters);
    SCK(cudaGetLastError());
    SCK(cudaMemcpyAsync(out5, s->counters, 5 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                        s->stream));
    SCK(cudaStreamSynchronize(s->stream));
    return DS_OK;
}

extern "C" int ds_shard_prepare(ds_shard* s, double delta, int mode, int frac) {
    if (!s) return ds_internal_set_err(DS_EINVAL, "null shard");
    if (!(delta > 0) || !std::isfinite(delta))
        return ds_internal_set_err(DS_EINVAL, "delta must be a positive finite number");
    cudaSetDevice(s->device);
    const long long n = s->n;
    long long* Lc = s->cnt_scratch;
    long long* Hc = s->cnt_scratch + (n + 1);
    k_shard_count<<<sgrid(s), kT, 0, s->stream>>>(n, s->indptr, s->w, delta, Lc, Hc);
    SCK(cudaGetLastError());
    SCK(cudaMemsetAsync(s->Lptr, 0, sizeof(long long), s->stream));
    SCK(cudaMemsetAsync(s->Hptr, 0, sizeof(long long), s->stream));
    void* tmp = nullptr;
    size_t bytes = 0;
    SCK(cub::DeviceScan::InclusiveSum(nullptr, bytes, Lc, s->Lptr + 1, n, s->stream));
    SCK(cudaMalloc(&tmp, bytes));
    SCK(cub::DeviceScan::InclusiveSum(tmp, bytes, Lc, s->Lptr + 1, n, s->stream));
    SCK(cub::DeviceScan::InclusiveSum(tmp, bytes, Hc, s->Hptr + 1, n, s->stream));
    SCK(cudaMemcpyAsync(&s->nL, s->Lptr + n, sizeof(long long), cudaMemcpyDeviceToHost, s->stream));
    SCK(cudaMemcpyAsync(&s->nH, s->Hptr + n, sizeof(long long), cudaMemcpyDeviceToHost, s->stream));
    SCK(cudaStreamSynchronize(s->stream));
    cudaFree(tmp);
    if (s->Ledges) cudaFree(s->Ledges);
    if (s->Hedges) cudaFree(s->Hedges);
    s->Ledges = s->Hedges = nullptr;
    const size_t es = mode == DS_MODE_FIXED32 ? sizeof(uint2) : sizeof(EdgeF64);
    SCK(cudaMalloc(&s->Ledges, es * std::max<long long>(s->nL, 1LL)));
    SCK(cudaMalloc(&s->Hedges, es * std::max<long long>(s->nH, 1LL)));
    if (mode == DS_MODE_FIXED32)
        k_shard_scatter<uint2><<<sgrid(s), kT, 0, s->stream>>>(n, s->indptr, s->col, s->w, delta, frac,
                                                                s->Lptr, s->Hptr, (uint2*)s->Ledges,
                                                                (uint2*)s->Hedges);
    else
        k_shard_scatter<EdgeF64><<<sgrid(s), kT, 0, s->stream>>>(n, s->indptr, s->col, s->w, delta, 0,
                                                                  s->Lptr, s->Hptr, (EdgeF64*)s->Ledges,
                                                                  (EdgeF64*)s->Hedges);
    SCK(cudaGetLastError());
    SCK(cudaStreamSynchronize(s->stream));
    s->mode = mode;
    s->frac = mode == DS_MODE_FIXED32 ? frac : 0;
    s->delta = delta;
    s->prepared = true;
    return DS_OK;
}

extern "C" int ds_shard_begin(ds_shard* s, int64_t source) {
    if (!s || !s->prepared) return ds_internal_set_err(DS_EINVAL, "shard not prepared");
    if (!(source >= 0 && source < s->n)) return ds_internal_set_err(DS_EINVAL, "source out of range");
    cudaSetDevice(s->device);
    const long long sl = (source >= s->v0 && source < s->v0 + s->nl) ? source - s->v0 : -1;
    if (s->mode == DS_MODE_FIXED32)
        (++s->launches), k_shard_init<ModeFixed><<<sgrid(s), kT, 0, s->stream>>>((unsigned*)s->dist, s->nl, sl);
    else
        (++s->launches), k_shard_init<ModeF64><<<sgrid(s), kT, 0, s->stream>>>((unsigned long long*)s->dist, s->nl, sl);
    SCK(cudaGetLastError());
    SCK(cudaMemsetAsync(s->fbits, 0, sizeof(unsigned) * (std::max<long long>(s->nl, 1LL) / 32 + 1), s->stream));
    SCK(cudaMemsetAsync(s->sbits, 0, sizeof(unsigned) * (s->n / 32 + 1), s->stream));
    s->scount = 0;
    SCK(cudaStreamSynchronize(s->stream));
    return DS_OK;
}

// Owned vertices in [L, H) -> out_ids/out_vals (device buffers of nl entries);
// *count, *next_min (owned min value >= H, ~0 if none).  L/H are D values
// widened to u64 (fixed: integer thresholds; f64: bit patterns).
extern "C" int ds_shard_scan(ds_shard* s, uint64_t L, uint64_t H, int32_t* out_ids, uint64_t* out_vals,
                             int64_t* count, uint64_t* next_min) {
    if (!s) return ds_internal_set_err(DS_EINVAL, "null shard");
    cudaSetDevice(s->device);
    unsigned long long init[2] = {0, ~0ull};
    SCK(cudaMemcpyAsync(s->counters, init, sizeof(init), cudaMemcpyHostToDevice, s->stream));
    if (s->nl) {
        if (s->mode == DS_MODE_FIXED32)
            (++s->launches), k_shard_scan<ModeFixed><<<sgrid(s), kT, 0, s->stream>>>(
                (const unsigned*)s->dist, s->nl, s->v0, (unsigned)L, (unsigned)H, out_ids,
                (unsigned long long*)out_vals, s->counters);
        else
            (++s->launches), k_shard_scan<ModeF64><<<sgrid(s), kT, 0, s->stream>>>(
                (const unsigned long long*)s->dist, s->nl, s->v0, L, H, out_ids,
                (unsigned long long*)out_vals, s->counters);
    }
    SCK(cudaGetLastError());
    SCK(cudaMemcpyAsync(s->h_counters, s->counters, 2 * sizeof(unsigned long long),
                        cudaMemcpyDeviceToHost, s->stream));
    SCK(cudaStreamSynchronize(s->stream));
    *count = (int64_t)s->h_counters[0];
    *next_min = s->h_counters[1];
    return DS_OK;
}

// Add an exchanged (global) frontier to S.
extern "C" int ds_shard_s_add(ds_shard* s, const int32_t* ids, const uint64_t* vals, int64_t count) {
    if (!s) return ds_internal_set_err(DS_EINVAL, "null shard");
    cudaSetDevice(s->device);
    unsigned long long c2 = (unsigned long long)s->scount;
    SCK(cudaMemcpyAsync(s->counters + 2, &c2, sizeof(c2), cudaMemcpyHostToDevice, s->stream));
    if (count > 0)
        (++s->launches), k_shard_s_add<<<sgrid(s), kT, 0, s->stream>>>(ids, (const unsigned long long*)vals, count,
                                                       s->sbits, s->sval, s->slist, s->counters);
    SCK(cudaGetLastError());
    SCK(cudaMemcpyAsync(&c2, s->counters + 2, sizeof(c2), cudaMemcpyDeviceToHost, s->stream));
    SCK(cudaStreamSynchronize(s->stream));
    s->scount = (long long)c2;
    return DS_OK;
}


// Edge-balanced push of (ids, vals) through the shard's light or heavy CSR.
// Light: the owned part of the next frontier lands in s->tmp_ids and its size
// in *nf.  Returns DS_OK; *ovf gets the fixed-point overflow flag.
template <class M>
static int shard_push(ds_shard* s, bool light, const int* ids, const unsigned long long* vals,
                      long long count, typename M::D H, long long* nf, int* ovf) {
    KParams<M> p{};
    p.dist = (typename M::D*)s->dist;
    p.Rent = reinterpret_cast<uint2*>(s->Rpre);  // n entries of 8 B
    p.Rd = (typename M::D*)s->Rd;
    p.chunk_start = s->chunk_start;
    SCK(cudaMemsetAsync(s->slot, 0, sizeof(StepSlot), s->stream));
    const unsigned grid = (unsigned)(s->nsm * 4);
    (++s->launches), k_shard_capture<M><<<grid, kThreads, 0, s->stream>>>(p, s->slot, ids, vals, count,
                                                         light ? s->Lptr : s->Hptr);
    SCK(cudaGetLastError());
    StepSlot h{};
    SCK(cudaMemcpyAsync(&h, s->slot, sizeof(StepSlot), cudaMemcpyDeviceToHost, s->stream));
    SCK(cudaStreamSynchronize(s->stream));
    const unsigned long long E = h.re_packed & kMask33, Rc = h.re_packed >> kPackShift;
    *nf = 0;
    *ovf = 0;
    if (E == 0) return DS_OK;
    const size_t smem = sizeof(Smem<typename M::D>);
    int occ = 1;
    if (light)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_shard_relax<M, true>, kThreads, smem);
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_shard_relax<M, false>, kThreads, smem);
    const unsigned rgrid = (unsigned)(s->nsm * std::max(occ, 1));
    if (light)
        (++s->launches), k_shard_relax<M, true><<<rgrid, kThreads, smem, s->stream>>>(
            p, s->slot, E, Rc, (const typename M::Edge*)s->Ledges, H, s->tmp_ids, s->fbits);
    else
        (++s->launches), k_shard_relax<M, false><<<rgrid, kThreads, smem, s->stream>>>(
            p, s->slot, E, Rc, (const typename M::Edge*)s->Hedges, H, nullptr, nullptr);
    SCK(cudaGetLastError());
    SCK(cudaMemcpyAsync(&h, s->slot, sizeof(StepSlot), cudaMemcpyDeviceToHost, s->stream));
    SCK(cudaStreamSynchronize(s->stream));
    *nf = (long long)h.append_count;
    *ovf = (int)(h.flags & 1u);
    return DS_OK;
}

// Light relaxation of an exchanged frontier (global ids + captured values)
// into the owned targets; the owned part of the next frontier comes back as
// global ids + final values (out buffers hold nl entries).  heavy=1 relaxes
// the heavy edges of the accumulated S instead (no output) and retires S.
extern "C" int ds_shard_relax(ds_shard* s, int heavy, const int32_t* ids, const uint64_t* vals,
                              int64_t count, uint64_t H, int32_t* out_ids, uint64_t* out_vals,
                              int64_t* out_count, int32_t* overflow) {
    if (!s) return ds_internal_set_err(DS_EINVAL, "null shard");
    cudaSetDevice(s->device);
    const bool fx = s->mode == DS_MODE_FIXED32;
    long long nf = 0;
    int ovf = 0, rc = DS_OK;
    if (heavy) {
        const long long sc = s->scount;
        if (sc > 0) {
            unsigned long long* sv = (unsigned long long*)s->cnt_scratch;
            (++s->launches), k_shard_gather_s<<<sgrid(s), kT, 0, s->stream>>>(s->slist, sc, s->sval, sv);
            SCK(cudaGetLastError());
            rc = fx ? shard_push<ModeFixed>(s, false, s->slist, sv, sc, 0u, &nf, &ovf)
                    : shard_push<ModeF64>(s, false, s->slist, sv, sc, 0ull, &nf, &ovf);
            if (rc) return rc;
            (++s->launches), k_shard_s_clear<<<sgrid(s), kT, 0, s->stream>>>(s->slist, sc, s->sbits);
            SCK(cudaGetLastError());
            SCK(cudaStreamSynchronize(s->stream));
        }
        s->scount = 0;
        if (out_count) *out_count = 0;
        if (overflow) *overflow = ovf;
        return DS_OK;
    }
    if (count > 0) {
        rc = fx ? shard_push<ModeFixed>(s, true, ids, (const unsigned long long*)vals, count,
                                        (unsigned)H, &nf, &ovf)
                : shard_push<ModeF64>(s, true, ids, (const unsigned long long*)vals, count, H, &nf,
                                      &ovf);
        if (rc) return rc;
    }
    if (nf > 0) {
        if (fx)
            (++s->launches), k_shard_emit<ModeFixed><<<sgrid(s), kT, 0, s->stream>>>(s->tmp_ids, nf, (const unsigned*)s->dist,
                                                                   s->v0, s->fbits, out_ids,
                                                                   (unsigned long long*)out_vals);
        else
            (++s->launches), k_shard_emit<ModeF64><<<sgrid(s), kT, 0, s->stream>>>(
                s->tmp_ids, nf, (const unsigned long long*)s->dist, s->v0, s->fbits, out_ids,
                (unsigned long long*)out_vals);
        SCK(cudaGetLastError());
        SCK(cudaStreamSynchronize(s->stream));
    }
    *out_count = nf;
    if (overflow) *overflow = ovf;
    return DS_OK;
}

// Owned distances as float64 (+inf = unreachable), out holds nl doubles.
extern "C" int64_t ds_shard_launches(const ds_shard* s) { return s ? (int64_t)s->launches : 0; }

extern "C" int ds_shard_result(ds_shard* s, double* out) {
    if (!s) return ds_internal_set_err(DS_EINVAL, "null shard");
    cudaSetDevice(s->device);
    if (s->nl) {
        double* d = nullptr;
        SCK(cudaMalloc(&d, sizeof(double) * s->nl));
        if (s->mode == DS_MODE_FIXED32)
            (++s->launches), k_shard_result<ModeFixed><<<sgrid(s), kT, 0, s->stream>>>((const unsigned*)s->dist, s->nl,
                                                                      s->frac, d);
        else
            (++s->launches), k_shard_result<ModeF64><<<sgrid(s), kT, 0, s->stream>>>((const unsigned long long*)s->dist,
                                                                    s->nl, 0, d);
        SCK(cudaGetLastError());
        SCK(cudaMemcpyAsync(out, d, sizeof(double) * s->nl, cudaMemcpyDefault, s->stream));
        SCK(cudaStreamSynchronize(s->stream));
        cudaFree(d);
    }
    return DS_OK;
}

// ---------------------------------------------------------------- shard from a device graph

int ds_internal_graph_csr(ds_graph* g, long long** indptr, int** col, double** w, long long* n,
                          long long* nnz, int* device, void** stream);

namespace {
__global__ void k_slice_count(const long long* indptr, const int* col, long long n, int v0, int v1,
                              long long* counts) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long r = warp; r < n; r += nwarps) {
        unsigned long long c = 0;
        for (long long e = indptr[r] + lane; e < indptr[r + 1]; e += 32) {
            const int v = col[e];
            c += (v >= v0 && v < v1);
        }
        c = warp_sum(c);
        if (lane == 0) counts[r] = (long long)c;
    }
}

__global__ void k_slice_scatter(const long long* indptr, const int* col, const double* w, long long n,
                                int v0, int v1, const long long* optr, int* ocol, double* ow) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    const unsigned lt = (1u << lane) - 1u;
    for (long long r = warp; r < n; r += nwarps) {
        long long o = optr[r];
        for (long long e0 = indptr[r]; e0 < indptr[r + 1]; e0 += 32) {
            const long long e = e0 + lane;
            const int v = e < indptr[r + 1] ? col[e] : -1;
            const bool keep = v >= v0 && v < v1;
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const long long k = o + __popc(m & lt);
                ocol[k] = v - v0;
                ow[k] = w[e];
            }
            o += __popc(m);
        }
    }
}
}  // namespace

// Shard [v0, v1) of a graph already resident on the device (no host copy).
extern "C" int ds_shard_from_graph(ds_graph* g, int64_t v0, int64_t v1, ds_shard** out) {
    long long *indptr = nullptr, n = 0, nnz = 0;
    int* col = nullptr;
    double* w = nullptr;
    int device = 0;
    void* stream = nullptr;
    int rc = ds_internal_graph_csr(g, &indptr, &col, &w, &n, &nnz, &device, &stream);
    if (rc) return rc;
    if (!(0 <= v0 && v0 <= v1 && v1 <= n)) return ds_internal_set_err(DS_EINVAL, "bad shard range");
    cudaSetDevice(device);
    cudaStream_t st = (cudaStream_t)stream;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    long long *counts = nullptr, *optr = nullptr;
    int* ocol = nullptr;
    double* ow = nullptr;
    void* tmp = nullptr;
    size_t bytes = 0;
    long long m = 0;
    SCK(cudaMalloc(&counts, sizeof(long long) * (n + 1)));
    SCK(cudaMalloc(&optr, sizeof(long long) * (n + 1)));
    k_slice_count<<<nsm * 16, 256, 0, st>>>(indptr, col, n, (int)v0, (int)v1, counts);
    SCK(cudaGetLastError());
    SCK(cudaMemsetAsync(optr, 0, sizeof(long long), st));
    SCK(cub::DeviceScan::InclusiveSum(nullptr, bytes, counts, optr + 1, n, st));
    SCK(cudaMalloc(&tmp, bytes));
    SCK(cub::DeviceScan::InclusiveSum(tmp, bytes, counts, optr + 1, n, st));
    SCK(cudaMemcpyAsync(&m, optr + n, sizeof(long long), cudaMemcpyDeviceToHost, st));
    SCK(cudaStreamSynchronize(st));
    SCK(cudaMalloc(&ocol, sizeof(int) * (m > 0 ? m : 1)));
    SCK(cudaMalloc(&ow, sizeof(double) * (m > 0 ? m : 1)));
    k_slice_scatter<<<nsm * 16, 256, 0, st>>>(indptr, col, w, n, (int)v0, (int)v1, optr, ocol, ow);
    SCK(cudaGetLastError());
    SCK(cudaStreamSynchronize(st));
    rc = ds_shard_create(n, v0, v1 - v0, m, (const int64_t*)optr, ocol, ow, device, stream, out);
    cudaFree(counts);
    cudaFree(optr);
    cudaFree(ocol);
    cudaFree(ow);
    cudaFree(tmp);
    return rc;
}
