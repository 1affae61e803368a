// sssp_kernel.cuh -- persistent, device-resident delta-stepping solver (sm_100a).
//
// One cooperative launch solves one source: bucket selection, every light
// phase, the heavy relaxation and termination all run on the device with
// grid-wide barriers between steps -- no host round trip per phase.
//
// Reference semantics reproduced (SURVEY.md §8(a) "parity semantics"):
//  * light predicate 0 < w <= delta / heavy delta < w, in f64 (sssp.py:96-97)
//    -- applied once by the split kernels (prepare.cu);
//  * bucket window [i*delta, (i+1)*delta) recomputed in f64 from i every time
//    (bucket_bounds, fused.py:58-61);
//  * a light phase relaxes the bucket's frontier with the distance values
//    CAPTURED before the merge (t o t_Bi then vxm, sssp.py:183-203): the
//    capture step below snapshots dist[u] after a grid barrier, the relax
//    step pushes from the snapshot;
//  * the next frontier is {v : lo <= r_v < hi and r_v < t_old(v)}
//    (fused_bucket_update, fused.py:187-190) -- realised as "some atomicMin
//    push with nd in the window succeeded", deduplicated by a phase stamp;
//  * S accumulates every frontier of the bucket (sssp.py:191, reset :285) and
//    the heavy edges are relaxed once per bucket from S with CURRENT t
//    (sssp.py:218-227);
//  * buckets are visited in increasing order; empty ones are skipped
//    internally (same distances, test_sssp.py:365-375) and the reference's
//    non-skip outer_iterations is recovered on the host from max(t_final).
//
// Work decomposition per step (all steps grid-stride over the persistent grid):
//  capture : frontier ids -> (captured d, row base, degree prefix) entries.
//            Each CTA tile scans its degrees in shared memory and reserves
//            its (entries, edges) ranges with ONE packed 64-bit atomicAdd, so
//            entry ranks and edge prefixes stay consistent without a global
//            scan; it also writes a tile->first-entry map for the relax step.
//  relax   : edge-balanced; each CTA stages one tile's entries in shared
//            memory, each thread maps kRelItems consecutive virtual edges to
//            their rows, then issues all edge loads, all distance loads and
//            finally the atomicMin pushes (three batched latency stages).
//  Appends (next frontier, S) are staged in a per-CTA shared-memory queue and
//  flushed with one global atomic per tile.
#pragma once

#include <cooperative_groups.h>
#include <cub/block/block_scan.cuh>
#include <math_constants.h>

#include "common.cuh"

namespace ds {

namespace cg = cooperative_groups;

// ---------------------------------------------------------------- modes

// Exact 32-bit fixed point: distance d is stored as D = d * 2^frac (an
// integer); every reference add fl64(d + w) is exact in this regime, so the
// integer sum is bit-identical after conversion.
struct ModeFixed {
    using D = unsigned;
    using Edge = uint2;  // x = column, y = weight * 2^frac
    static constexpr D INF = 0xFFFFFFFFu;
    __device__ __forceinline__ static Edge load(const Edge* p, unsigned long long pol) {
        Edge r;
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
                     : "=r"(r.x), "=r"(r.y)
                     : "l"(p), "l"(pol));
        return r;
    }
    __device__ __forceinline__ static unsigned col(const Edge& e) { return e.x; }
    __device__ __forceinline__ static bool add(D du, const Edge& e, D& nd) {
        unsigned long long s = (unsigned long long)du + e.y;
        if (s >= 0xFFFFFFFFull) return false;  // overflow -> rerun in f64 mode
        nd = (unsigned)s;
        return true;
    }
    __device__ __forceinline__ static double to_f64(D d, int frac) {
        return d == INF ? CUDART_INF : ldexp((double)d, -frac);
    }
    __device__ __forceinline__ static void window(double lo, double hi, int frac, D& L, D& H) {
        L = ceil_u32_clamped(ldexp(lo, frac));
        H = ceil_u32_clamped(ldexp(hi, frac));
    }
};

struct __align__(16) EdgeF64 {
    unsigned col;
    unsigned pad;
    double w;
};

// IEEE binary64 distances held as their bit patterns: for non-negative
// doubles the u64 order equals the numeric order, so atomicMin on the bits is
// an exact f64 min.  Adds are round-to-nearest like numpy.
struct ModeF64 {
    using D = unsigned long long;
    using Edge = EdgeF64;
    static constexpr D INF = 0x7FF0000000000000ull;
    __device__ __forceinline__ static Edge load(const Edge* p, unsigned long long pol) {
        uint4 q;
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                     : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w)
                     : "l"(p), "l"(pol));
        Edge e;
        e.col = q.x;
        e.pad = 0;
        e.w = __hiloint2double((int)q.w, (int)q.z);
        return e;
    }
    __device__ __forceinline__ static unsigned col(const Edge& e) { return e.col; }
    __device__ __forceinline__ static bool add(D du, const Edge& e, D& nd) {
        nd = (D)__double_as_longlong(__dadd_rn(__longlong_as_double((long long)du), e.w));
        return true;
    }
    __device__ __forceinline__ static double to_f64(D d, int) {
        return __longlong_as_double((long long)d);
    }
    __device__ __forceinline__ static void window(double lo, double hi, int, D& L, D& H) {
        L = (D)__double_as_longlong(lo);
        H = (D)__double_as_longlong(hi);
    }
};

// ---------------------------------------------------------------- control block

constexpr int kPackShift = 33;  // capture reservation: (entries << 33) | edges
constexpr unsigned long long kMask33 = (1ull << kPackShift) - 1;

struct StepSlot {
    unsigned long long re_packed;     // capture: reserved (entries << 33) | edges
    unsigned long long front_count;   // capture (range mode): frontier size
    unsigned long long next_min;      // capture (range mode): min D >= H
    unsigned long long append_count;  // relax (light): next-frontier size
    unsigned int flags;               // bit0: fixed-point overflow
    unsigned int pad;
    unsigned long long pad2[3];
};

struct Ctl {
    unsigned bar_count;
    unsigned bar_gen;
    unsigned abort;
    int status;  // DS_* code raised on the device
    StepSlot slot[3];
    unsigned long long s_count[2];
    unsigned long long reached, edges_reached, max_d;
    unsigned long long phases, visited, edges_scanned, barriers, steps;
    long long last_bucket;
};

constexpr int kDevOverflow = 100;  // internal status: fixed-point overflow

template <class M>
struct KParams {
    using D = typename M::D;
    using Edge = typename M::Edge;
    long long n;
    long long source;
    double delta;
    int frac;
    int pad;
    long long ceiling;
    unsigned long long timeout_ns;
    const long long* indptr;  // original CSR row offsets (for m_r)
    const long long* Lptr;
    const Edge* Ledges;
    const long long* Hptr;
    const Edge* Hedges;
    D* dist;
    unsigned* fstamp;
    unsigned* sstamp;
    int* F0;
    int* F1;
    int* S;
    long long* Rpre;
    long long* Rbase;
    D* Rd;
    unsigned* tile_start;
    Ctl* ctl;
    double* out;
    unsigned long long* trace;  // optional per-step timeline (2 words / step)
    unsigned long long trace_cap;
    unsigned pser0, bser0;
};

constexpr int kQCap = 1024;  // per-CTA append staging (overflow spills to global)

template <class D>
struct SmemRelax {
    long long base[kRelTile + 1];
    D d[kRelTile + 1];
    int rel[kRelTile + 1];
    unsigned short row[kRelTile];  // tile-local edge -> staged entry
};

using BlockScanU64 = cub::BlockScan<unsigned long long, kThreads>;

template <class D>
struct Smem {
    union {
        SmemRelax<D> rx;
        typename BlockScanU64::TempStorage scan;
    } u;
    int qbuf[kQCap];
    unsigned qcnt;
    unsigned qn;
    unsigned long long qbase;
    unsigned long long red[kThreads / 32];
    unsigned long long red2[kThreads / 32];
    unsigned long long pc, pd;
    int ok;
};

// ---------------------------------------------------------------- block utils

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ unsigned long long warp_min(unsigned long long v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}
__device__ __forceinline__ unsigned long long warp_max(unsigned long long v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}

// op: 0 sum, 1 min, 2 max; result valid in thread 0
template <int OP>
__device__ __forceinline__ unsigned long long block_reduce(unsigned long long v,
                                                           unsigned long long* buf) {
    v = OP == 0 ? warp_sum(v) : OP == 1 ? warp_min(v) : warp_max(v);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) buf[w] = v;
    __syncthreads();
    if (w == 0) {
        v = lane < kThreads / 32 ? buf[lane] : (OP == 1 ? ~0ull : 0ull);
        v = OP == 0 ? warp_sum(v) : OP == 1 ? warp_min(v) : warp_max(v);
    }
    return v;
}

__device__ __forceinline__ unsigned long long evict_first_policy() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// Grid-wide barrier over a co-resident (cooperative) grid.  Returns false if
// the solve was aborted (watchdog deadline or another CTA's abort).
template <class S>
__device__ __forceinline__ bool grid_sync(Ctl* c, unsigned& gen, unsigned long long deadline,
                                          S& sm) {
    __syncthreads();
    if (threadIdx.x == 0) {
        int ok = 1;
        const unsigned target = gen + 1;
        __threadfence();
        const unsigned prev = atomicAdd(&c->bar_count, 1u);
        if (prev == gridDim.x - 1) {
            c->bar_count = 0;
            st_release_u32(&c->bar_gen, target);
        } else {
            unsigned spins = 0;
            while (ld_acquire_u32(&c->bar_gen) != target) {
                if ((++spins & 1023u) == 0) {
                    if (ld_acquire_u32(&c->abort)) {
                        ok = 0;
                        break;
                    }
                    if (globaltimer_ns() > deadline) {
                        atomicExch(&c->abort, 1u);
                        ok = 0;
                        break;
                    }
                }
            }
        }
        __threadfence();
        gen = target;
        if (ld_acquire_u32(&c->abort)) ok = 0;
        sm.ok = ok;
    }
    __syncthreads();
    return sm.ok != 0;
}

// Stage v in the CTA's shared-memory queue (warp-aggregated); spill straight
// to the global list when the queue is full.
template <class S>
__device__ __forceinline__ void q_push(S& sm, int* list, unsigned long long* counter, int v) {
    cg::coalesced_group g = cg::coalesced_threads();
    unsigned pos = 0;
    if (g.thread_rank() == 0) pos = atomicAdd(&sm.qcnt, (unsigned)g.size());
    pos = g.shfl(pos, 0) + g.thread_rank();
    if (pos < (unsigned)kQCap) {
        sm.qbuf[pos] = v;
    } else {
        cg::coalesced_group h = cg::coalesced_threads();
        unsigned long long b = 0;
        if (h.thread_rank() == 0) b = atomicAdd(counter, (unsigned long long)h.size());
        b = h.shfl(b, 0);
        list[b + h.thread_rank()] = v;
    }
}

// Reserve global space for the staged queue (thread 0); call between two
// __syncthreads, then q_copy after the second.
template <class S>
__device__ __forceinline__ void q_reserve(S& sm, unsigned long long* counter) {
    const unsigned c = sm.qcnt < (unsigned)kQCap ? sm.qcnt : (unsigned)kQCap;
    sm.qn = c;
    sm.qbase = c ? atomicAdd(counter, (unsigned long long)c) : 0ull;
    sm.qcnt = 0;
}
template <class S>
__device__ __forceinline__ void q_copy(S& sm, int* list) {
    const unsigned c = sm.qn;
    for (unsigned i = threadIdx.x; i < c; i += kThreads) list[sm.qbase + i] = sm.qbuf[i];
}

// ---------------------------------------------------------------- capture step
//
// Input: a frontier given as an id list (LIST) or as "all vertices whose
// distance lies in [L, H)" (RANGE: compute_bucket, sssp.py:153-158).
// Output: compacted entries (captured d, row base, degree prefix) of the
// frontier vertices with at least one edge in `ptr`'s CSR, the relax tile
// map, and the slot totals.  APPEND_S adds every frontier vertex to S
// (S = S + t_Bi, sssp.py:191; dedup by the bucket stamp).

template <class M, bool RANGE, bool APPEND_S>
__device__ void capture_step(const KParams<M>& p, Smem<typename M::D>& sm, StepSlot* slot,
                             const int* list, unsigned long long count, typename M::D L,
                             typename M::D H, const long long* ptr, unsigned bser,
                             unsigned long long* s_counter) {
    using D = typename M::D;
    const unsigned long long total = RANGE ? (unsigned long long)p.n : count;
    const unsigned long long ntiles = (total + kCapTile - 1) / kCapTile;
    unsigned long long local_fc = 0;
    unsigned long long local_min = ~0ull;

    for (unsigned long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        __syncthreads();  // shared queue / scan storage reuse across tiles
        const unsigned long long base = tile * kCapTile + (unsigned long long)threadIdx.x * kCapItems;
        int vtx[kCapItems];
        D dv[kCapItems];
        bool in[kCapItems];
#pragma unroll
        for (int j = 0; j < kCapItems; ++j) {
            const unsigned long long idx = base + j;
            in[j] = idx < total;
            vtx[j] = in[j] ? (RANGE ? (int)idx : ldcg(list + idx)) : 0;
        }
#pragma unroll
        for (int j = 0; j < kCapItems; ++j) dv[j] = in[j] ? __ldcg(p.dist + vtx[j]) : M::INF;
        long long off[kCapItems];
        long long deg[kCapItems];
        unsigned long long packed = 0;  // (count << 48) | degree within the tile
#pragma unroll
        for (int j = 0; j < kCapItems; ++j) {
            if (RANGE && in[j]) {
                const D d = dv[j];
                if (d >= H && d != M::INF && (unsigned long long)d < local_min)
                    local_min = (unsigned long long)d;
                in[j] = (d >= L) && (d < H);
            }
            off[j] = in[j] ? __ldg(ptr + vtx[j]) : 0;
            deg[j] = in[j] ? __ldg(ptr + vtx[j] + 1) : 0;
        }
#pragma unroll
        for (int j = 0; j < kCapItems; ++j) {
            if (in[j]) {
                ++local_fc;
                if (APPEND_S) {
                    if (atomicExch(p.sstamp + vtx[j], bser) != bser) q_push(sm, p.S, s_counter, vtx[j]);
                }
                deg[j] -= off[j];
                if (deg[j] > 0) packed += (1ull << 48) + (unsigned long long)deg[j];
            } else {
                deg[j] = 0;
            }
        }
        unsigned long long excl, agg;
        BlockScanU64(sm.u.scan).ExclusiveSum(packed, excl, agg);
        __syncthreads();
        if (threadIdx.x == 0) {
            // one packed reservation keeps entry ranks and edge prefixes in
            // the same order across tiles
            if (agg) {
                const unsigned long long want = ((agg >> 48) << kPackShift) | (agg & kMask48);
                const unsigned long long r = atomicAdd(&slot->re_packed, want);
                sm.pc = r >> kPackShift;
                sm.pd = r & kMask33;
            }
            if (APPEND_S) q_reserve(sm, s_counter);
        }
        __syncthreads();
        if (APPEND_S) q_copy(sm, p.S);
        if (agg) {
            unsigned long long rank = sm.pc + (excl >> 48);
            unsigned long long pre = sm.pd + (excl & kMask48);
#pragma unroll
            for (int j = 0; j < kCapItems; ++j) {
                if (deg[j] > 0) {
                    p.Rpre[rank] = (long long)pre;
                    p.Rbase[rank] = off[j] - (long long)pre;
                    p.Rd[rank] = dv[j];
                    const unsigned long long t0 = (pre + kRelTile - 1) / kRelTile;
                    const unsigned long long t1 = (pre + (unsigned long long)deg[j] - 1) / kRelTile;
                    for (unsigned long long t = t0; t <= t1; ++t) p.tile_start[t] = (unsigned)rank;
                    ++rank;
                    pre += (unsigned long long)deg[j];
                }
            }
        }
    }
    if (RANGE) {
        const unsigned long long fc = block_reduce<0>(local_fc, sm.red);
        const unsigned long long mn = block_reduce<1>(local_min, sm.red2);
        if (threadIdx.x == 0) {
            if (fc) atomicAdd(&slot->front_count, fc);
            if (mn != ~0ull) atomicMin(&slot->next_min, mn);
        }
    }
}

// ---------------------------------------------------------------- relax step
//
// Edge-balanced push over the entries of the last capture.  LIGHT: successful
// improvements that land inside the window join the next frontier once
// (fstamp dedup); HEAVY: min-merge only (results land beyond the window).

template <class M, bool LIGHT>
__device__ void relax_step(const KParams<M>& p, Smem<typename M::D>& sm, StepSlot* slot,
                           unsigned long long E, unsigned long long Rc,
                           const typename M::Edge* edges, typename M::D H, int* out_list,
                           unsigned pser) {
    using D = typename M::D;
    using Edge = typename M::Edge;
    const unsigned long long ntile = (E + kRelTile - 1) / kRelTile;
    const unsigned long long pol = evict_first_policy();
    bool overflow = false;
    for (unsigned long long t = blockIdx.x; t < ntile; t += gridDim.x) {
        const unsigned long long r0 = ldcg(p.tile_start + t);
        const unsigned long long r1 = (t + 1 < ntile) ? ldcg(p.tile_start + t + 1) : Rc - 1;
        const int ne = (int)(r1 - r0 + 1);
        const long long tb = (long long)(t * kRelTile);
        for (int k = threadIdx.x; k < ne; k += kThreads) {
            const unsigned long long r = r0 + k;
            const long long rel = ldcg(p.Rpre + r) - tb;
            sm.u.rx.rel[k] = rel < 0 ? 0 : (int)rel;
            sm.u.rx.base[k] = ldcg(p.Rbase + r);
            sm.u.rx.d[k] = __ldcg(p.Rd + r);
        }
        __syncthreads();
        // row map: thread t resolves the staged entry of tile edges
        // [8t, 8t+8) with one binary search and a short walk
        {
            const int rel0 = threadIdx.x * kRelItems;
            int lo = 0, hi = ne;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (sm.u.rx.rel[mid] <= rel0) lo = mid;
                else hi = mid;
            }
            int k = lo;
#pragma unroll
            for (int j = 0; j < kRelItems; ++j) {
                while (k + 1 < ne && sm.u.rx.rel[k + 1] <= rel0 + j) ++k;
                sm.u.rx.row[rel0 + j] = (unsigned short)k;
            }
        }
        __syncthreads();
        // edges are taken lane-strided (edge = tb + tid + 256 j) so every warp
        // load instruction reads 32 consecutive (col, w) pairs
        const long long left = (long long)E - tb - threadIdx.x;  // > 256 j  <=>  edge j exists
        if (left > 0) {
            int kk[kRelItems];
            Edge ed[kRelItems];
#pragma unroll
            for (int j = 0; j < kRelItems; ++j) {
                const int r = threadIdx.x + j * kThreads;
                kk[j] = sm.u.rx.row[r];
                if (j * kThreads < left) ed[j] = M::load(edges + (sm.u.rx.base[kk[j]] + tb + r), pol);
            }
            // stage 2: candidate distances and current values
            D nd[kRelItems], cur[kRelItems];
#pragma unroll
            for (int j = 0; j < kRelItems; ++j) {
                cur[j] = (D)0;
                if (j * kThreads < left) {
                    if (M::add(sm.u.rx.d[kk[j]], ed[j], nd[j])) {
                        cur[j] = __ldcg(p.dist + M::col(ed[j]));
                    } else {
                        overflow = true;
                    }
                }
            }
            // stage 3: pushes
#pragma unroll
            for (int j = 0; j < kRelItems; ++j) {
                if (j * kThreads < left && nd[j] < cur[j]) {
                    const unsigned v = M::col(ed[j]);
                    if (LIGHT) {
                        const D old = atomicMin(p.dist + v, nd[j]);
                        if (nd[j] < old && nd[j] < H) {
                            if (atomicExch(p.fstamp + v, pser) != pser)
                                q_push(sm, out_list, &slot->append_count, (int)v);
                        }
                    } else {
                        atomicMin(p.dist + v, nd[j]);
                    }
                }
            }
        }
        __syncthreads();
        if (LIGHT) {
            if (threadIdx.x == 0) q_reserve(sm, &slot->append_count);
            __syncthreads();
            q_copy(sm, out_list);
        }
    }
    if (overflow) atomicOr(&slot->flags, 1u);
}

// ---------------------------------------------------------------- the solver

template <class M>
__global__ void __launch_bounds__(kThreads, 3)
    sssp_persistent_kernel(const KParams<M> p) {
    using D = typename M::D;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem<D>& sm = *reinterpret_cast<Smem<D>*>(smem_raw);
    Ctl* const c = p.ctl;
    unsigned gen = 0;
    unsigned long long deadline = 0;
    if (threadIdx.x == 0) {
        deadline = globaltimer_ns() + p.timeout_ns;
        sm.qcnt = 0;
    }

    // ---- init: t = {source: 0} (sssp.py:276), all else +inf
    {
        const long long stride = (long long)gridDim.x * kThreads;
        for (long long v = (long long)blockIdx.x * kThreads + threadIdx.x; v < p.n; v += stride)
            p.dist[v] = (v == p.source) ? (D)0 : M::INF;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            for (int k = 0; k < 3; ++k) {
                StepSlot* s = &c->slot[k];
                s->re_packed = s->front_count = s->append_count = 0;
                s->flags = 0;
                s->next_min = ~0ull;
            }
            c->s_count[0] = c->s_count[1] = 0;
        }
    }
    if (!grid_sync(c, gen, deadline, sm)) return;
    if (p.trace && blockIdx.x == 0 && threadIdx.x == 0) c->last_bucket = (long long)globaltimer_ns();

    unsigned long long st = 0;  // step counter (identical on every CTA)
    unsigned long long nbar = 1, escanned = 0;
    long long idx = 0;  // bucket index
    unsigned long long phases = 0, visited = 0;
    unsigned pser = p.pser0, bser = p.bser0;
    int pp = 0;
    int status = 0;

    auto end_step = [&](unsigned long long kind, unsigned long long work) -> bool {
        if (blockIdx.x == 0 && threadIdx.x == 0) {  // recycle the slot two steps ahead
            StepSlot* s = &c->slot[(st + 1) % 3];
            s->re_packed = s->front_count = s->append_count = 0;
            s->flags = 0;
            s->next_min = ~0ull;
        }
        const bool ok = grid_sync(c, gen, deadline, sm);
        if (p.trace && blockIdx.x == 0 && threadIdx.x == 0 && st < p.trace_cap) {
            p.trace[2 * st] = globaltimer_ns();
            p.trace[2 * st + 1] = (kind << 56) | (work & ((1ull << 56) - 1));
        }
        ++st;
        ++nbar;
        return ok;
    };
    auto prev = [&]() -> StepSlot* { return &c->slot[(st + 2) % 3]; };

    for (;;) {
        const double lo = (double)idx * p.delta;
        const double hi = (double)(idx + 1) * p.delta;
        D L, H;
        M::window(lo, hi, p.frac, L, H);

        // ---- bucket extraction: t_Bi = {v : lo <= t[v] < hi}; S starts empty
        if (blockIdx.x == 0 && threadIdx.x == 0) c->s_count[(bser & 1) ^ 1] = 0;
        capture_step<M, true, true>(p, sm, &c->slot[st % 3], nullptr, 0, L, H, p.Lptr, bser,
                                    &c->s_count[bser & 1]);
        if (!end_step(0, (unsigned long long)p.n)) return;
        const unsigned long long fc = ldcg(&prev()->front_count);
        unsigned long long re = ldcg(&prev()->re_packed);
        if (fc == 0) {
            const unsigned long long nm = ldcg(&prev()->next_min);
            if (nm == ~0ull) break;  // nothing stored beyond: done
            idx = bucket_index_of(M::to_f64((D)nm, p.frac), p.delta);
            continue;
        }
        ++visited;

        // ---- light phases (sssp.py:292-301)
        for (;;) {
            ++phases;
            if ((long long)phases > p.ceiling) {
                status = 2;  // DS_ENOCONVERGE
                break;
            }
            unsigned long long nf = 0;
            const unsigned long long E = re & kMask33;
            if (E > 0) {
                escanned += E;
                relax_step<M, true>(p, sm, &c->slot[st % 3], E, re >> kPackShift, p.Ledges, H,
                                    pp ? p.F1 : p.F0, pser);
                if (!end_step(1, E)) return;
                if (ldcg(&prev()->flags) & 1u) {
                    status = kDevOverflow;
                    break;
                }
                nf = ldcg(&prev()->append_count);
            }
            ++pser;
            if (nf == 0) break;
            capture_step<M, false, true>(p, sm, &c->slot[st % 3], pp ? p.F1 : p.F0, nf, L, H,
                                         p.Lptr, bser, &c->s_count[bser & 1]);
            if (!end_step(2, nf)) return;
            re = ldcg(&prev()->re_packed);
            pp ^= 1;
        }
        if (status) break;

        // ---- heavy relaxation from S with current t (sssp.py:218-227)
        const unsigned long long scount = ldcg(&c->s_count[bser & 1]);
        capture_step<M, false, false>(p, sm, &c->slot[st % 3], p.S, scount, L, H, p.Hptr, bser,
                                      nullptr);
        if (!end_step(3, scount)) return;
        re = ldcg(&prev()->re_packed);
        const unsigned long long E = re & kMask33;
        if (E > 0) {
            escanned += E;
            relax_step<M, false>(p, sm, &c->slot[st % 3], E, re >> kPackShift, p.Hedges, H,
                                 nullptr, pser);
            if (!end_step(4, E)) return;
            if (ldcg(&prev()->flags) & 1u) {
                status = kDevOverflow;
                break;
            }
        }
        ++bser;
        ++idx;
    }

    if (status) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            c->status = status;
            c->phases = phases;
            c->steps = st;
        }
        return;
    }

    // ---- finalize: fp64 output, n_r, m_r, max distance (SsspResult, sssp.py:312-313)
    {
        unsigned long long cnt = 0, m = 0, mx = 0;
        const long long stride = (long long)gridDim.x * kThreads;
        for (long long v = (long long)blockIdx.x * kThreads + threadIdx.x; v < p.n; v += stride) {
            const D d = __ldcg(p.dist + v);
            if (d != M::INF) {
                ++cnt;
                m += (unsigned long long)(__ldg(p.indptr + v + 1) - __ldg(p.indptr + v));
                if ((unsigned long long)d > mx) mx = (unsigned long long)d;
            }
            p.out[v] = M::to_f64(d, p.frac);
        }
        cnt = block_reduce<0>(cnt, sm.red);
        m = block_reduce<0>(m, sm.red2);
        mx = block_reduce<2>(mx, sm.red);
        if (threadIdx.x == 0) {
            atomicAdd(&c->reached, cnt);
            atomicAdd(&c->edges_reached, m);
            atomicMax(&c->max_d, mx);
            if (blockIdx.x == 0) {
                c->phases = phases;
                c->visited = visited;
                c->edges_scanned = escanned;
                c->barriers = nbar;
                c->steps = st;
                if (!p.trace) c->last_bucket = idx;
                c->status = 0;
            }
        }
    }
}

}  // namespace ds
