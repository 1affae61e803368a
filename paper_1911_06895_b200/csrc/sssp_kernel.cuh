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
// Work decomposition per step: every step is warp-granular -- warps of the
// persistent grid take chunks independently and never wait on each other
// inside a step (no __syncthreads); steps are separated by grid barriers.
//  capture : frontier ids -> (captured d, row base, degree prefix) entries.
//            A warp scans its chunk's degrees with shuffles and reserves its
//            (entries, edges) ranges with ONE packed 64-bit atomicAdd, so entry
//            ranks and edge prefixes stay consistent without a global scan; it
//            also writes the chunk map (first entry of every 256-edge chunk).
//  relax   : edge-balanced; a warp stages one 256-edge chunk's entries in its
//            shared-memory slice, maps each edge to its row, then issues
//            lane-strided (coalesced) edge loads, the distance loads and the
//            atomicMin pushes as three batched latency stages.
//  Dedup of the next frontier uses 1 bit per vertex (an L2-resident bitmap),
//  cleared by the step that consumes the list; S needs none in the push builds
//  (the one push that brings a vertex into the window tags its entry).  Appends
//  are staged in the warp's shared-memory queue (ballot prefix) and flushed
//  with one global atomic per chunk.
//
// Schedules.  Binary64 graphs run exactly the reference's bucket / phase
// schedule above.  Fixed-point graphs run the "lex" schedule (see "lex mode"):
// distance words carry a hop count, from which the reference's counters are
// recovered whatever the processing order -- ksub internal buckets per
// reference bucket while the buckets are large, then (see "wide windows" and
// "bidirectional step") the latency-bound tail as one label-correcting
// closure over every edge of the frontier rows.
#pragma once

#include <cooperative_groups.h>
#include <cub/block/block_scan.cuh>
#include <math_constants.h>

#include <climits>
#include <type_traits>

#include "common.cuh"

// DS_CHECKS=1 builds (tools/build_variant.py chk -DDS_CHECKS=1): device-side
// bounds checks on the indices the solver computes -- entry ranks, chunk-map
// slots, edge offsets, targets, list lengths, window tables -- that print the
// failing condition and trap.  compute-sanitizer is not available on the GPU
// pool; the GPU test suite and the fuzzer run against this build instead.
#ifndef DS_CHECKS
#define DS_CHECKS 0
#endif
#if DS_CHECKS
#include <cstdio>
#define DS_ASSERT(cond)                                                                              \
    do {                                                                                             \
        if (!(cond)) {                                                                               \
            printf("DS_ASSERT failed: %s (line %d) block %d thread %d\n", #cond, __LINE__, blockIdx.x, \
                   threadIdx.x);                                                                     \
            __trap();                                                                                \
        }                                                                                            \
    } while (0)
#else
#define DS_ASSERT(cond) \
    do {                \
    } while (0)
#endif

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
    // every heavy result t_u + w with t_u >= L lands at or beyond H
    __device__ __forceinline__ static bool heavy_beyond(D L, D H, double, double, unsigned long long minW) {
        return (unsigned long long)L + minW >= (unsigned long long)H;
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
    // fl(t_u + w) >= fl(lo + min w) >= hi for every t_u >= lo (monotone rounding)
    __device__ __forceinline__ static bool heavy_beyond(D, D, double lo, double hi, unsigned long long minW) {
        return __dadd_rn(lo, __longlong_as_double((long long)minW)) >= hi;
    }
};

// ---------------------------------------------------------------- lex mode
//
// The reference's counters (outer_iterations, inner_phases) follow its
// Jacobi light phases inside each bucket [i*delta, (i+1)*delta) -- a schedule
// that re-pushes a vertex's light row every time it improves (R-MAT 24:
// 6x nnz(A_L)).  Lex mode computes the same distances with ksub finer internal
// buckets per reference bucket (fewer re-pushes) and recovers the counters
// exactly from hop counts carried in the distance word:
//   key = (D << kHopBits) | h,   min over keys = min D, then min h.
// A push u -> v with weight W carries h_u + 1 when the edge is a reference-
// light edge (W <= WD) landing in u's reference bucket (D_u + W < HD), else 0
// (the value is part of a later bucket's starting state).  Integer adds are
// exact, so the lexicographic minimum over walks is schedule-independent and
// h(v) is the fewest light hops over the walks achieving D(v) inside the
// bucket, counted from the bucket's starting values.  The reference's k-th
// phase of bucket i is non-empty iff some vertex of the bucket has h >= k
// (Jacobi round k finds exactly the <= k-hop walks), so the bucket runs
// 1 + max h phases; a bucket is visited iff some final value lies in it.
// Keys need D < 2^(32 - kHopBits) - 1 and h < 2^kHopBits: a larger sum or
// hop count raises the overflow flag and the solve reruns in binary64 mode.
constexpr int kHopBits = 6;
constexpr unsigned kHopMask = (1u << kHopBits) - 1;
constexpr unsigned long long kLexDLimit = (1ull << (32 - kHopBits)) - 1;
constexpr unsigned kLexSat = (unsigned)(kLexDLimit << kHopBits);  // < INF (0xFFFFFFFF)

template <class M>
struct KParams;

// push candidate: plain add, or the lex key (fixed point, p.lex)
template <bool LEX, class M>
__device__ __forceinline__ bool padd(const KParams<M>& p, typename M::D ku, const typename M::Edge& e,
                                     typename M::D hd, typename M::D& nd) {
    if constexpr (LEX && std::is_same<M, ModeFixed>::value) {
        // 32-bit: D < 2^26 and every weight W < 2^26 (checked at prepare)
        // Hops saturate at kHopMask: a saturated key still orders below every
        // longer walk of the same distance, and only a FINAL key of the
        // bucket at kHopMask (checked at its S capture) is unusable.
        // A sum beyond the key range becomes kLexSat: larger than every real
        // key (so any real path replaces it) but still "reached"; should one
        // survive until the solver reaches it, the solve reruns without lex
        // (its true distance is not representable).
        const unsigned s = (ku >> kHopBits) + e.y;
        const unsigned hu = ku & kHopMask;
        const unsigned h = (e.y <= p.WD && s < hd) ? hu + (hu < kHopMask ? 1u : 0u) : 0u;
        nd = s < (unsigned)kLexDLimit ? (s << kHopBits) | h : kLexSat;
        return true;
    }
    return M::add(ku, e, nd);
}

// ---------------------------------------------------------------- control block

constexpr int kPackShift = 33;  // capture reservation: (entries << 33) | edges
constexpr unsigned long long kMask33 = (1ull << kPackShift) - 1;
constexpr int kWarps = kThreads / 32;
// standalone giant-push kernel: its own block shape (uses Smem::w[0 .. warps))
#ifndef DS_BIG_THREADS
#define DS_BIG_THREADS DS_THREADS
#endif
#ifndef DS_BIG_MINB
#define DS_BIG_MINB 1
#endif
constexpr int kBigThreads = DS_BIG_THREADS;
static_assert(kBigThreads % 32 == 0 && kBigThreads <= kThreads, "standalone push block shape");
#ifndef DS_CHUNK
#define DS_CHUNK 256
#endif
constexpr int kChunk = DS_CHUNK;  // relax / pull: edges per warp chunk (32 lanes x kRelPer)
constexpr int kRelPer = kChunk / 32;
#ifndef DS_LIST_PER
#define DS_LIST_PER 2
#endif
constexpr int kListPer = DS_LIST_PER;  // capture (range): entries per lane per round
#ifndef DS_CAP_PER
#define DS_CAP_PER DS_LIST_PER
#endif
constexpr int kCapPer = DS_CAP_PER;  // capture (list): entries per lane per round
#ifndef DS_QUEUE
#define DS_QUEUE 256
#endif
#ifndef DS_BULK_CLEAR
#define DS_BULK_CLEAR 16384  // frontier lists at least this long clear the dedup bitmap as a whole
#endif
constexpr unsigned long long kBulkClearMin = DS_BULK_CLEAR;
constexpr int kRangePer = 16;     // capture (range): vertices per lane
constexpr int kQueue = DS_QUEUE;  // per-warp append staging (overflow spills to global)
#ifndef DS_HEAVY_RED
#define DS_HEAVY_RED 0
#endif
#ifndef DS_PRECHECK_L1
#define DS_PRECHECK_L1 1
#endif
constexpr bool kHeavyRed = DS_HEAVY_RED != 0;
// Pull (vxm) forms compiled into the solver.  Both are correct (parity tests
// run with them on) but on R-MAT 24 they cost more than they save: the extra
// code raises register pressure (spills) in every step of this persistent
// kernel, so they are opt-in builds (-DDS_PULL_LIGHT=1 / -DDS_PULL_HEAVY=1).
#ifndef DS_PULL_LIGHT
#define DS_PULL_LIGHT 0
#endif
#ifndef DS_PULL_HEAVY
#define DS_PULL_HEAVY 0
#endif
// DS_CSUM: the high-diameter (SMALL) kernel keeps, per 512-vertex scan chunk,
// a lower bound of the stored values beyond the current window, so a bucket
// scan reads only the chunks that can hold in-window vertices (the dense scan
// of every vertex per bucket dominated many-bucket graphs).  Push builds only:
// the pull forms write beyond-window values without maintaining the bound.
#ifndef DS_CSUM
#define DS_CSUM 1
#endif
#ifndef DS_CSUM_RED
#define DS_CSUM_RED 1
#endif
constexpr bool kCsum = DS_CSUM && !(DS_PULL_LIGHT || DS_PULL_HEAVY);
// S (the bucket's settled set, sssp.py:191) without a membership bitmap: a
// vertex joins S exactly once per bucket -- either the bucket scan finds it in
// the window, or ONE push brings it from at-or-beyond hi to below hi (values
// only decrease, atomicMin serialises the pushes, so exactly one sees
// old >= hi > new).  That push tags its next-frontier entry (bit 31) and the
// capture of that frontier appends the vertex to S; a tagging push that loses
// the frontier dedup claim appends to S directly.  Replaces one returning
// atomicOr per frontier vertex and phase plus one atomicAnd per S member and
// bucket.  The pull builds gate on the S bitmap and keep the claims.
#ifndef DS_S_ENTRY
#define DS_S_ENTRY 1
#endif
constexpr bool kSEntry = DS_S_ENTRY && !(DS_PULL_LIGHT || DS_PULL_HEAVY);
constexpr unsigned kSTag = 0x80000000u;
#ifndef DS_ROWMAP_SCAN
#define DS_ROWMAP_SCAN 1  // 1: push row map by marks + warp max-scan (0: search + walk)
#endif
#ifndef DS_CS_PREFETCH
#define DS_CS_PREFETCH 1  // 1: prefetch the next chunk's chunk-map words
#endif
#ifndef DS_DEFER_APPEND
#define DS_DEFER_APPEND 1  // 1: consume a chunk's dedup claims after the next chunk's loads
#endif
#ifndef DS_LATE_FLUSH
#define DS_LATE_FLUSH 1  // 1: flush warp append queues when half full, not per chunk
#endif
#ifndef DS_BARRIER
#define DS_BARRIER 1  // 1: monotonic-counter grid barrier (0: counter + generation pair)
#endif
#ifndef DS_BARRIER_SLEEP
#define DS_BARRIER_SLEEP 0
#endif
#ifndef DS_PIPE
#define DS_PIPE 0  // software-pipelined push: next chunk's entries load under this chunk's edges
#endif
#ifndef DS_PRECHECK_CUT
#define DS_PRECHECK_CUT 32768  // > 0: only pre-check reads of solver ids below it go through L1 (measured -2%)
#endif
#ifndef DS_COUNT
#define DS_COUNT 0  // count the light push atomics (diagnostics build)
#endif
#ifndef DS_L2PF
#define DS_L2PF 0  // bulk L2 prefetch of the next chunk's edges (measured slower: 5.34 -> 5.40 ms)
#endif

#ifndef DS_BIDIR_BUILD
#define DS_BIDIR_BUILD 1  // 0: compile the bidirectional step out (register-pressure A/B)
#endif
#ifndef DS_WIDE_REF
#define DS_WIDE_REF 256
#endif
constexpr int kWideRef = DS_WIDE_REF;  // reference buckets one wide window may span

struct StepSlot {
    unsigned long long re_packed;     // capture: reserved (entries << 33) | edges
    unsigned long long front_count;   // capture (range mode): frontier size
    unsigned long long next_min;      // capture (range mode): min D >= H
    unsigned long long append_count;  // relax / pull (light): next-frontier size
    unsigned int flags;               // bit0: fixed-point overflow
    unsigned int hopmax;              // lex mode: largest hop count of a captured S
    unsigned long long pad2[3];
};

struct Ctl {
    unsigned bar_count;
    unsigned bar_gen;
    unsigned long long bar_arrive;  // DS_BARRIER=1: monotonic arrival counter
    unsigned abort;
    int status;  // DS_* code raised on the device
    StepSlot slot[3];
    unsigned long long s_count[2];
    unsigned long long reached, edges_reached, max_d;
    unsigned long long phases, visited, edges_scanned, barriers, steps;
    long long last_bucket;
    unsigned long long pulls;  // light/heavy steps run as pulls
    unsigned long long cnt_atomics, cnt_improved;  // DS_COUNT=1 builds: light atomics issued / improving
    // resumable solver: the persistent kernel hands a giant push to a
    // standalone launch (k_big_relax) and is relaunched where it left off
    unsigned long long rs_pos, rs_req, rs_E, rs_Rc;
    unsigned long long rs_st, rs_phases, rs_visited, rs_escanned, rs_nbar, rs_npull;
    unsigned long long rs_re, rs_scount, rs_old_scount, rs_pp, rs_bpar, rs_hset;
    long long rs_idx;
    StepSlot xslot;  // results of the standalone push
    StepSlot lslot[2];  // block-local mode (CTA 0 alone)
    // results of the block-local steps; light and heavy publish to separate
    // fields so a slow CTA still reading the light result is never overwritten
    // by CTA 0 racing ahead into the local heavy step
    unsigned long long h_phases, h_re, h_pp, h_done, h_status, h_escanned;
    unsigned long long hh_re, hh_done, hh_status;
    unsigned long long t_enter, t_exit;  // DS_TRACE: kernel entry / last CTA's finalize end
    unsigned lexsat;  // lex mode: a final key held an out-of-range sum (rerun without lex)
    // wide windows (lex mode): per reference bucket of the window, 1 + the
    // largest final hop count (0: no final value in the bucket); two sets,
    // alternating between windows
    unsigned whm[2][kWideRef];
    unsigned long long wide_windows, wide_edges;  // stats: windows run wide / edges they pushed
};

enum : int { POS_FRESH = 0, POS_BUCKET = 1, POS_PHASE = 2, POS_AFTER_LIGHT = 3, POS_HEAVY = 4,
             POS_AFTER_HEAVY = 5 };

constexpr int kDevOverflow = 100;  // internal status: fixed-point overflow
constexpr int kDevLexFail = 101;   // internal status: lex keys out of range (rerun without lex)

// Pull schedule of one CSR (light or heavy) in solver order: the rows with
// at least one edge, their offsets, the row holding the first edge of every
// 256-edge chunk, and the rows that cross a chunk boundary (their partial
// minima meet in `req` and are finished by the commit step).
struct PullPlan {
    const int* rowid;           // compacted row -> solver vertex id
    const long long* cptr;      // compacted offsets (n_nz + 1)
    const unsigned* chunk_row;  // nchunk + 1 entries
    const int* span;            // compacted rows crossing a chunk boundary
    long long n_nz, nspan, nnz;
};

template <class M>
struct KParams {
    using D = typename M::D;
    using Edge = typename M::Edge;
    long long n;
    long long source;
    double delta;
    int frac;
    int pull_enabled;
    float pull_light, pull_heavy;  // pull when push volume > frac * nnz
    unsigned long long big_light, big_heavy;  // pushes with >= this many edges run standalone
    int heavy_pull;  // standalone heavy step as a pull (k_big_pull/k_big_commit; A^T == A)
    unsigned long long local_edges, local_entries;  // SMALL kernel: CTA-0-only steps below these
    long long ceiling;
    unsigned long long timeout_ns;
    // direction-optimised heavy step: pull into the unsettled rows when the
    // push over S would stream more edges (symmetric graphs)
    int hpull;
    float hpull_ratio;
    unsigned long long hpull_min;
    unsigned long long nH;
    unsigned long long nL, nA;     // edges in A_L / the merged rows (DS_CHECKS bounds)
    unsigned long long cap_chunks;  // slots of chunk_start (DS_CHECKS bounds)
    unsigned long long min_heavy;  // smallest heavy weight: fixed W, or f64 bits
    // Sub-bucketed solve with lexicographic keys (fixed point only; see
    // "lex mode" below): ksub internal buckets per reference bucket, dist
    // words hold (D << kHopBits) | hops, WD = largest reference-light W.
    int lex;
    int ksub_log2;  // ksub = 1 << ksub_log2 (shifts, no 64-bit divisions)
    unsigned WD;
    const long long* indptr;  // original CSR row offsets (for m_r)
    const long long* Lptr;
    const Edge* Ledges;
    const long long* Hptr;
    const Edge* Hedges;
    // per row {offset mod 2^32, degree} of the light / heavy CSR: the captures
    // read a row's extent with ONE 8-byte load (two int64 offsets were two
    // divergent loads per frontier vertex; the L1 wavefront rate is the bound)
    const uint2* Linfo;
    const uint2* Hinfo;
    // wide windows (lex mode; see "wide windows" at the solver loop): every
    // row of A in solver order, light edges first (null: disabled)
    const Edge* Aedges;
    const uint2* Ainfo;
    unsigned long long wide_enter;  // a bucket that pushed fewer edges than this switches to wide windows
    unsigned long long wide_lo, wide_hi;  // a window below wide_lo doubles the next one, above wide_hi halves it
    unsigned wide_g0, wide_gmax;  // first / largest window, in internal buckets
    int wide_force;               // tests: wide windows after the first bucket, whatever its size
    int bidir;                    // enter the wide tail through the bidirectional step
    unsigned long long wide_unsettled;  // ... and at most this many heavy edges in rows not yet settled
    unsigned long long wide_all;        // at most this many: the first window takes the largest size
    PullPlan Lpull, Hpull;
    D* dist;
    D* csum;             // SMALL kernel (kCsum): per scan chunk, <= every stored value >= the window
    D* req;              // pull partial minima (INF when idle), n_nz entries
    unsigned* fbits[2];  // next-frontier dedup bitmaps (alternating phases)
    unsigned* sbits;     // S membership / dedup bitmap
    int* F[2];           // frontier lists
    D* Fv[2];            // frontier values (lists produced by a pull)
    int* S[2];           // S lists (alternating buckets)
    uint2* Rent;  // capture entries {edge prefix, row base - prefix}, both mod 2^32
                  // (a step's edges and the split arrays stay below 2^32, checked at prepare)
    D* Rd;
    unsigned* chunk_start;
    const int* perm;      // input id -> solver id (degree-sorted relabeling)
    const unsigned* sdeg; // solver id -> out-degree in A (m_r)
    long long n_active;   // solver ids >= n_active have no edges at all
    Ctl* ctl;
    double* out;
    unsigned long long* trace;  // optional per-step timeline (2 words / step)
    unsigned long long trace_cap;
    unsigned long long* cta_done;  // DS_TRACE=2: per step and CTA, the time its warps finished the step
};

template <class D>
struct WarpSmem {
    unsigned base[kChunk + 1];  // push: (row base + chunk offset) mod 2^32; pull: row end
                                // (light / heavy edge arrays hold < 2^32 edges; checked at prepare)
    D d[kChunk + 1];
    short rel[kChunk + 1];  // chunk-relative row starts, clamped to [-1, kChunk]
    alignas(16) unsigned short row[kChunk];
    int q[kQueue];
#if DS_PULL_LIGHT || DS_PULL_HEAVY
    D qv[kQueue];  // values travelling with pull-produced lists
#endif
#if DS_PIPE
    D du[kChunk];  // pipelined push: per-edge source value of the chunk in flight
#endif
};
template <class D>
__device__ __forceinline__ D* queue_vals(WarpSmem<D>& ws) {
#if DS_PULL_LIGHT || DS_PULL_HEAVY
    return ws.qv;
#else
    return nullptr;
#endif
}

// lex-mode accounting of the reference buckets (kept by thread 0 of every
// CTA in shared memory: the values are uniform, and registers are scarce in
// the persistent kernel)
struct LexAcc {
    long long cur_ref;  // reference bucket being accumulated
    unsigned long long phases, visited;
    unsigned hop_acc;
    int any;
    int over;  // the reference's phase count exceeded the ceiling
};

template <class D>
struct Smem {
    WarpSmem<D> w[kWarps];
    unsigned long long red[kWarps];
    unsigned long long red2[kWarps];
    int ok;
    LexAcc lx;
    // wide windows: D thresholds of the window's reference buckets (wn + 1
    // entries) and the per-bucket hop maxima of the hop pass
    unsigned wthr[kWideRef + 1];
    unsigned whm[kWideRef];
    int wn;
    int wfail;
    unsigned wpar;             // which Ctl::whm set the current window reports into
    unsigned long long bwork;  // edges pushed by the current bucket / window (thread 0 adds)
};
static_assert(kWarps <= 32, "one warp scans the CTA's per-warp totals");

// ---------------------------------------------------------------- warp / block utils

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
__device__ __forceinline__ unsigned long long warp_incl_scan(unsigned long long v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
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
        v = lane < kWarps ? buf[lane] : (OP == 1 ? ~0ull : 0ull);
        v = OP == 0 ? warp_sum(v) : OP == 1 ? warp_min(v) : warp_max(v);
    }
    return v;
}

__device__ __forceinline__ unsigned long long evict_first_policy() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

#ifndef DS_LIGHT_POL
#define DS_LIGHT_POL 0  // L2 policy of light-edge loads: 0 evict_first, 1 evict_normal, 2 evict_last
#endif
__device__ __forceinline__ unsigned long long light_policy() {
    unsigned long long pol;
#if DS_LIGHT_POL == 2
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#elif DS_LIGHT_POL == 1
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
#else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#endif
    return pol;
}

// set bit v; true iff it was clear (first claim this phase / bucket)
__device__ __forceinline__ bool claim_bit(unsigned* bits, unsigned v) {
    const unsigned m = 1u << (v & 31);
    return (atomicOr(bits + (v >> 5), m) & m) == 0;
}
__device__ __forceinline__ bool test_bit(const unsigned* bits, unsigned v) {
    return (__ldcg(bits + (v >> 5)) >> (v & 31)) & 1u;
}

// Grid-wide barrier over a co-resident (cooperative) grid.  Returns false if
// the solve was aborted (watchdog deadline or another CTA's abort).
template <class S>
__device__ __forceinline__ bool grid_sync(Ctl* c, unsigned& gen, unsigned long long deadline,
                                          S& sm) {
    __syncthreads();
#if DS_BARRIER == 1
    // monotonic counter: arrive with a fire-and-forget release add, wait until
    // every CTA's arrival for this generation is visible (no reset, no second
    // release store, one round trip less than the counter + generation pair)
    if (threadIdx.x == 0) {
        int ok = 1;
        const unsigned long long target = (unsigned long long)(gen + 1) * gridDim.x;
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(&c->bar_arrive) : "memory");
        unsigned spins = 0;
        while (ld_acquire_u64(&c->bar_arrive) < target) {
#if DS_BARRIER_SLEEP
            __nanosleep(DS_BARRIER_SLEEP);
#endif
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
        __threadfence();
        gen += 1;
        if (ld_acquire_u32(&c->abort)) ok = 0;
        sm.ok = ok;
    }
    __syncthreads();
    return sm.ok != 0;
#else
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
#endif
}

// Warp-uniform append: every lane calls it; lanes with `want` land in the
// warp's queue at ballot-prefix positions (optionally with a value).  Spills
// to the global list when the queue is full.
template <class D, bool VAL>
__device__ __forceinline__ void wq_push(int* q, D* qv, unsigned& qn, bool want, int v, D val,
                                        int lane, int* list, D* vlist,
                                        unsigned long long* counter) {
    const unsigned m = __ballot_sync(0xffffffffu, want);
    if (!m) return;
    const unsigned cnt = __popc(m);
    const unsigned below = __popc(m & ((1u << lane) - 1u));
    if (qn + cnt <= (unsigned)kQueue) {
        if (want) {
            q[qn + below] = v;
            if (VAL) qv[qn + below] = val;
        }
        qn += cnt;
    } else {
        unsigned long long b = 0;
        if (lane == 0) b = atomicAdd(counter, (unsigned long long)cnt);
        b = __shfl_sync(0xffffffffu, b, 0);
        if (want) {
            list[b + below] = v;
            if (VAL) vlist[b + below] = val;
        }
    }
}

template <class D, bool VAL>
__device__ __forceinline__ void wq_flush(int* q, D* qv, unsigned& qn, int lane, int* list,
                                         D* vlist, unsigned long long* counter) {
    if (!qn) return;
    __syncwarp();
    unsigned long long b = 0;
    if (lane == 0) b = atomicAdd(counter, (unsigned long long)qn);
    b = __shfl_sync(0xffffffffu, b, 0);
    for (unsigned i = lane; i < qn; i += 32) {
        list[b + i] = q[i];
        if (VAL) vlist[b + i] = qv[i];
    }
    __syncwarp();
    qn = 0;
}

// ---------------------------------------------------------------- capture step
//
// Input: a frontier given as an id list (LIST) or as "all vertices whose
// distance lies in [L, H)" (RANGE: compute_bucket, sssp.py:153-158).
// Output: compacted entries (captured d, row base, degree prefix) of the
// frontier vertices with at least one edge in `ptr`'s CSR, the relax chunk
// map, and the slot totals.  APPEND_S adds every frontier vertex to S
// (S = S + t_Bi, sssp.py:191; dedup by the S bitmap).

template <class M, int PER>
__device__ __forceinline__ void capture_emit(const KParams<M>& p, StepSlot* slot, int lane,
                                             const typename M::D (&dv)[PER],
                                             const long long (&off)[PER], const long long (&deg)[PER]) {
    unsigned long long packed = 0;  // (count << 48) | degree within the warp chunk
#pragma unroll
    for (int j = 0; j < PER; ++j)
        if (deg[j] > 0) packed += (1ull << 48) + (unsigned long long)deg[j];
    const unsigned long long incl = warp_incl_scan(packed, lane);
    const unsigned long long tot = __shfl_sync(0xffffffffu, incl, 31);
    if (!tot) return;
    unsigned long long r = 0;
    if (lane == 31) {
        // one packed reservation keeps entry ranks and edge prefixes in the
        // same order across warps
        const unsigned long long want = ((tot >> 48) << kPackShift) | (tot & kMask48);
        r = atomicAdd(&slot->re_packed, want);
    }
    r = __shfl_sync(0xffffffffu, r, 31);
    const unsigned long long excl = incl - packed;
    unsigned long long rank = (r >> kPackShift) + (excl >> 48);
    unsigned long long pre = (r & kMask33) + (excl & kMask48);
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        if (deg[j] > 0) {
            DS_ASSERT(rank < (unsigned long long)p.n);
            p.Rent[rank] = make_uint2((unsigned)pre, (unsigned)(off[j] - (long long)pre));
            p.Rd[rank] = dv[j];
            const unsigned long long t0 = (pre + kChunk - 1) / kChunk;
            const unsigned long long t1 = (pre + (unsigned long long)deg[j] - 1) / kChunk;
            DS_ASSERT(t1 < p.cap_chunks);
            for (unsigned long long t = t0; t <= t1; ++t) p.chunk_start[t] = (unsigned)rank;
            ++rank;
            pre += (unsigned long long)deg[j];
        }
    }
}

// CTA-cooperative form of capture_emit: every warp of the CTA calls it once
// per round; the warps' totals are scanned in shared memory and the CTA makes
// ONE packed reservation for all of them.  (Per-warp reservations all hit one
// counter: at R-MAT 24 they were ~16% of the solver's stall samples.)
template <class M, int PER>
__device__ __forceinline__ void capture_emit_cta(const KParams<M>& p, Smem<typename M::D>& sm,
                                                 StepSlot* slot, int lane, int wib,
                                                 const typename M::D (&dv)[PER],
                                                 const long long (&off)[PER], const long long (&deg)[PER]) {
    unsigned long long packed = 0;  // (count << 48) | degree within the warp chunk
#pragma unroll
    for (int j = 0; j < PER; ++j)
        if (deg[j] > 0) packed += (1ull << 48) + (unsigned long long)deg[j];
    const unsigned long long incl = warp_incl_scan(packed, lane);
    if (lane == 31) sm.red[wib] = incl;
    __syncthreads();
    if (wib == 0) {
        const unsigned long long wt = lane < kWarps ? sm.red[lane] : 0ull;
        const unsigned long long wi = warp_incl_scan(wt, lane);
        const unsigned long long all = __shfl_sync(0xffffffffu, wi, 31);
        unsigned long long r = 0;
        if (lane == 31 && all) r = atomicAdd(&slot->re_packed, ((all >> 48) << kPackShift) | (all & kMask48));
        r = __shfl_sync(0xffffffffu, r, 31);
        const unsigned long long we = wi - wt;  // warps before this one
        if (lane < kWarps) {
            sm.red[lane] = (r >> kPackShift) + (we >> 48);  // first entry rank
            sm.red2[lane] = (r & kMask33) + (we & kMask48);  // first edge prefix
        }
    }
    __syncthreads();
    const unsigned long long excl = incl - packed;
    unsigned long long rank = sm.red[wib] + (excl >> 48);
    unsigned long long pre = sm.red2[wib] + (excl & kMask48);
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        if (deg[j] > 0) {
            DS_ASSERT(rank < (unsigned long long)p.n);
            p.Rent[rank] = make_uint2((unsigned)pre, (unsigned)(off[j] - (long long)pre));
            p.Rd[rank] = dv[j];
            const unsigned long long t0 = (pre + kChunk - 1) / kChunk;
            const unsigned long long t1 = (pre + (unsigned long long)deg[j] - 1) / kChunk;
            DS_ASSERT(t1 < p.cap_chunks);
            for (unsigned long long t = t0; t <= t1; ++t) p.chunk_start[t] = (unsigned)rank;
            ++rank;
            pre += (unsigned long long)deg[j];
        }
    }
}

// Dense-scan register layout: a warp's scan chunk is 32 x kRangePer consecutive
// vertices; register slot j of a lane holds the vertex scan_vertex(chunk base,
// lane, j) -- lane-interleaved 16-byte groups, so every load instruction of the
// warp covers 512 contiguous bytes (a lane reading its own 64 contiguous bytes
// made each instruction touch every line of the chunk: 4x the L1 tag requests).
template <class D>
__device__ __forceinline__ unsigned long long scan_vertex(unsigned long long cbase, int lane, int j) {
    constexpr int V = 16 / (int)sizeof(D);
    return cbase + (unsigned long long)((j / V) * (32 * V) + lane * V + (j % V));
}
template <class D>
__device__ __forceinline__ void load_run(const D* chunk, int lane, D (&out)[kRangePer]);
template <>
__device__ __forceinline__ void load_run<unsigned>(const unsigned* chunk, int lane, unsigned (&out)[kRangePer]) {
#pragma unroll
    for (int i = 0; i < kRangePer / 4; ++i) {
        const uint4 q = __ldcg(reinterpret_cast<const uint4*>(chunk) + i * 32 + lane);
        out[4 * i] = q.x;
        out[4 * i + 1] = q.y;
        out[4 * i + 2] = q.z;
        out[4 * i + 3] = q.w;
    }
}
template <>
__device__ __forceinline__ void load_run<unsigned long long>(const unsigned long long* chunk, int lane,
                                                             unsigned long long (&out)[kRangePer]) {
#pragma unroll
    for (int i = 0; i < kRangePer / 2; ++i) {
        const ulonglong2 q = __ldcg(reinterpret_cast<const ulonglong2*>(chunk) + i * 32 + lane);
        out[2 * i] = q.x;
        out[2 * i + 1] = q.y;
    }
}

// RANGE capture: bucket extraction by a dense scan of the distance array.
// Also retires the previous bucket's S bits (atomicAnd: disjoint from the
// new bucket's S, which only holds vertices with values >= the old hi).
// UNSET: instead capture every row whose value is >= L (unsettled, INF
// included) over `ptr`, with the row's solver id as the entry value -- the
// rows a heavy pull gathers into (see pull_gather in relax_step).
template <class M, bool SUM = false, bool UNSET = false>
__device__ void capture_range(const KParams<M>& p, Smem<typename M::D>& sm, StepSlot* slot,
                              typename M::D L, typename M::D H, int* S, unsigned long long* s_counter,
                              unsigned long long n_scan, const int* old_S, unsigned long long old_count,
                              const uint2* ptr) {
    using D = typename M::D;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    WarpSmem<D>& ws = sm.w[wib];
    unsigned qn = 0;
    const unsigned long long gw = (unsigned long long)blockIdx.x * kWarps + wib;
    const unsigned long long nw = (unsigned long long)gridDim.x * kWarps;
    if (!kSEntry) {
        for (unsigned long long i = gw * 32 + lane; i < old_count; i += nw * 32) {
            const unsigned v = (unsigned)ldcg(old_S + i);
            atomicAnd(p.sbits + (v >> 5), ~(1u << (v & 31)));
        }
    }
    const unsigned long long n = n_scan;
    const unsigned long long per_chunk = 32ull * kRangePer;
    const unsigned long long nchunk = (n + per_chunk - 1) / per_chunk;
    unsigned long long local_fc = 0;
    D local_min = M::INF;  // smallest stored value beyond the window (INF: none)
    // !SUM: per scan chunk a "settled" flag (in csum's storage): every value of
    // the chunk is below the window, hence final -- later scans skip the chunk
    unsigned* const chunk_done = reinterpret_cast<unsigned*>(p.csum);
    auto scan_chunk = [&](unsigned long long c) {
        const unsigned long long cbase = c * per_chunk;
        D dv[kRangePer];
        const bool full = cbase + per_chunk <= n;
        if (full) {
            load_run<D>(p.dist + cbase, lane, dv);
        } else {
#pragma unroll
            for (int j = 0; j < kRangePer; ++j) {
                const unsigned long long vj = scan_vertex<D>(cbase, lane, j);
                dv[j] = vj < n ? __ldcg(p.dist + vj) : M::INF;
            }
        }
        unsigned hits = 0;
        D cmin = M::INF;
        bool settled = true;
#pragma unroll
        for (int j = 0; j < kRangePer; ++j) {
            const D d = dv[j];
            if (UNSET) {
                if (d >= L && scan_vertex<D>(cbase, lane, j) < n) hits |= 1u << j;
                continue;
            }
            const bool below = d < L;
            const bool inw = !below && d < H;
            if (inw) hits |= 1u << j;
            const D beyond = (below || inw) ? M::INF : d;  // INF stays INF: "none"
            cmin = beyond < cmin ? beyond : cmin;
            settled = settled && below;
        }
        if (cmin < local_min) local_min = cmin;
        if (SUM && !UNSET) {  // exact bound for the chunk (no relaxation runs during this step)
            unsigned long long wm = warp_min((unsigned long long)cmin);
            if (lane == 0) p.csum[c] = (D)wm;
        }
        if (!SUM && !UNSET && full && __all_sync(0xffffffffu, settled)) {
            if (lane == 0) chunk_done[c] = 1u;
            return;
        }
        if (!__any_sync(0xffffffffu, hits != 0)) return;
        local_fc += __popc(hits);
        // in-window vertices of this chunk, kListPer per lane per round
        D cd[kListPer];
        long long off[kListPer], deg[kListPer];
        unsigned rem = hits;
        while (__any_sync(0xffffffffu, rem != 0)) {
            int vtx[kListPer];
#pragma unroll
            for (int j = 0; j < kListPer; ++j) {
                deg[j] = 0;
                off[j] = 0;
                vtx[j] = -1;
                cd[j] = 0;
                if (rem) {
                    const int b = __ffs(rem) - 1;
                    rem &= rem - 1;
                    vtx[j] = (int)scan_vertex<D>(cbase, lane, b);
                    if (UNSET) {
                        cd[j] = (D)vtx[j];  // the entry carries the row id
                    } else {
                        // select, not dv[b]: a dynamic index would move dv[] to local memory
                        D x = dv[0];
#pragma unroll
                        for (int i = 1; i < kRangePer; ++i) x = (b == i) ? dv[i] : x;
                        cd[j] = x;
                    }
                }
            }
            bool news[kListPer];
#pragma unroll
            for (int j = 0; j < kListPer; ++j) {
                const bool in = vtx[j] >= 0;
                if (in) {
                    const uint2 ri = __ldg(ptr + vtx[j]);  // {row offset mod 2^32, degree}: one load
                    off[j] = ri.x;
                    deg[j] = ri.y;
                }
                // kSEntry: the scan meets every vertex once -- no claim needed
                news[j] = !UNSET && in && (kSEntry || claim_bit(p.sbits, (unsigned)vtx[j]));
            }
            if (!UNSET) {
#pragma unroll
                for (int j = 0; j < kListPer; ++j)
                    wq_push<D, false>(ws.q, queue_vals(ws), qn, news[j], vtx[j], (D)0, lane, S, nullptr,
                                      s_counter);
            }
            capture_emit<M, kListPer>(p, slot, lane, cd, off, deg);
        }
        if (!UNSET && (!DS_LATE_FLUSH || qn > (unsigned)kQueue / 2))
            wq_flush<D, false>(ws.q, queue_vals(ws), qn, lane, S, nullptr, s_counter);
    };
    if (SUM && !UNSET) {
        // the warp's chunks are the usual grid-strided ones; each lane reads the
        // bound of one of them (one round trip for up to 32 chunks) and the
        // warp scans only the chunks whose bound is below hi.  Every stored value >= lo of a chunk is >= its
        // bound, so a bound >= hi means no in-window vertex, and it stands in
        // for the chunk's beyond-window minimum (a lower bound of it: a low
        // bound only makes the solver visit an empty bucket, which is not
        // counted and rescans that chunk exactly)
        for (unsigned long long g = gw; g < nchunk; g += 32 * nw) {
            const unsigned long long cl = g + lane * nw;
            const D s = cl < nchunk ? __ldcg(p.csum + cl) : M::INF;
            const bool act = s < H;
            if (!act && s < local_min) local_min = s;
            unsigned mask = __ballot_sync(0xffffffffu, act);
            while (mask) {
                const int b = __ffs(mask) - 1;
                mask &= mask - 1;
                scan_chunk(g + (unsigned long long)b * nw);
            }
        }
    } else if (UNSET) {
        for (unsigned long long c = gw; c < nchunk; c += nw) scan_chunk(c);
    } else {
        // each lane reads the settled flag of one of the warp's next 32 chunks
        for (unsigned long long g = gw; g < nchunk; g += 32 * nw) {
            const unsigned long long cl = g + lane * nw;
            const unsigned f = cl < nchunk ? ldcg(chunk_done + cl) : 1u;
            unsigned mask = __ballot_sync(0xffffffffu, f == 0u);
            while (mask) {
                const int b = __ffs(mask) - 1;
                mask &= mask - 1;
                scan_chunk(g + (unsigned long long)b * nw);
            }
        }
    }
    if (UNSET) return;  // the entry / edge totals are in slot->re_packed
    wq_flush<D, false>(ws.q, queue_vals(ws), qn, lane, S, nullptr, s_counter);
    const unsigned long long fc = block_reduce<0>(local_fc, sm.red);
    const unsigned long long mn =
        block_reduce<1>(local_min == M::INF ? ~0ull : (unsigned long long)local_min, sm.red2);
    if (threadIdx.x == 0) {
        if (fc) atomicAdd(&slot->front_count, fc);
        if (mn != ~0ull) atomicMin(&slot->next_min, mn);
    }
}

// UNSETTLED capture for the heavy gather (dense: most rows of the active
// prefix are unsettled at a giant bucket): CTA-uniform rounds of 32 x kUnsetPer
// consecutive rows per warp (coalesced dist / offset reads), one entry
// reservation per CTA round.  Entries carry the row id; rows >= n_scan and
// rows without heavy edges get none.
constexpr int kUnsetPer = 4;
// `info`: the rows' extents (A_H, or the merged rows for the bidirectional
// step).  S != null: rows whose value already lies in [T, HW) -- reached by
// light pushes beyond the bucket -- are appended to S (the coming wide
// window's settled set; everything else enters it by a tagged push).
template <class M>
__device__ void capture_unsettled(const KParams<M>& p, Smem<typename M::D>& sm, StepSlot* slot,
                                  typename M::D T, unsigned long long n_scan, const uint2* info,
                                  typename M::D HW = 0, int* S = nullptr,
                                  unsigned long long* s_counter = nullptr) {
    using D = typename M::D;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    WarpSmem<D>& ws = sm.w[wib];
    unsigned qn = 0;
    const unsigned long long per_warp = 32ull * kUnsetPer;
    const unsigned long long nblk = (n_scan + per_warp - 1) / per_warp;
    const unsigned long long nw = (unsigned long long)gridDim.x * kWarps;
    for (unsigned long long cbase = (unsigned long long)blockIdx.x * kWarps; cbase < nblk; cbase += nw) {
        const unsigned long long c = cbase + wib;
        D cd[kUnsetPer];
        long long off[kUnsetPer], deg[kUnsetPer];
#pragma unroll
        for (int j = 0; j < kUnsetPer; ++j) {
            const unsigned long long v = c * per_warp + lane + 32ull * j;
            const bool in = c < nblk && v < n_scan;
            const D d = in ? __ldcg(p.dist + v) : (D)0;
            const bool un = in && d >= T;
            cd[j] = (D)v;
            const uint2 ri = un ? __ldg(info + v) : make_uint2(0u, 0u);
            off[j] = ri.x;
            deg[j] = ri.y;
            if (S) wq_push<D, false>(ws.q, queue_vals(ws), qn, un && d < HW, (int)v, (D)0, lane, S, nullptr, s_counter);
        }
        capture_emit_cta<M, kUnsetPer>(p, sm, slot, lane, wib, cd, off, deg);
    }
    if (S) wq_flush<D, false>(ws.q, queue_vals(ws), qn, lane, S, nullptr, s_counter);
}

// LIST capture: a frontier / S list.  Snapshots d after the barrier that
// ended the previous phase (VALS: the list carries values produced by a pull
// and this step commits them to t first), looks up degrees in `ptr`, clears
// the next-frontier dedup bits for their next use, optionally adds to S.
template <class M, bool APPEND_S, bool VALS, bool LOCALW = false, bool HOPS = false>
__device__ void capture_list(const KParams<M>& p, Smem<typename M::D>& sm, StepSlot* slot,
                             const int* list, const typename M::D* vals, unsigned long long count,
                             const uint2* ptr, unsigned* clear_bits, int* S,
                             unsigned long long* s_counter, unsigned long long clear_words = 0) {
    using D = typename M::D;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    WarpSmem<D>& ws = sm.w[wib];
    unsigned qn = 0;
    // clear_words > 0 (large lists): the dedup bitmap is zeroed as a whole by
    // coalesced stores instead of one divergent store per list entry
    if (!LOCALW && clear_bits && clear_words) {
        for (unsigned long long k = (unsigned long long)blockIdx.x * kThreads + threadIdx.x; k < clear_words;
             k += (unsigned long long)gridDim.x * kThreads)
            clear_bits[k] = 0u;
        clear_bits = nullptr;
    }
    const unsigned long long per_chunk = 32ull * kCapPer;
    const unsigned long long nchunk = (count + per_chunk - 1) / per_chunk;
    // LOCALW: only this CTA's warps take part (block-local small-frontier mode)
    // CTA-uniform rounds (capture_emit_cta synchronises the CTA's warps):
    // warp w of the CTA takes chunk cbase + w
    const unsigned long long cb0 = LOCALW ? 0ull : (unsigned long long)blockIdx.x * kWarps;
    const unsigned long long nw = LOCALW ? kWarps : (unsigned long long)gridDim.x * kWarps;
    unsigned hop_cta = 0;  // lex S capture: largest hop count seen by this warp
    for (unsigned long long cbase = cb0; cbase < nchunk; cbase += nw) {
        const unsigned long long c = cbase + wib;
        int vtx[kCapPer];
        bool in[kCapPer];
        D dv[kCapPer];
#pragma unroll
        for (int j = 0; j < kCapPer; ++j) {
            const unsigned long long idx = c * per_chunk + lane + 32ull * j;
            in[j] = c < nchunk && idx < count;
            vtx[j] = in[j] ? ldcg(list + idx) : 0;
            if (VALS) dv[j] = in[j] ? __ldcg(vals + idx) : (D)0;
        }
        bool tagged[kCapPer];  // kSEntry: the entry's push brought the vertex into the window
#pragma unroll
        for (int j = 0; j < kCapPer; ++j) {
            tagged[j] = false;
            if (kSEntry && APPEND_S) {
                tagged[j] = in[j] && ((unsigned)vtx[j] & kSTag);
                vtx[j] = (int)((unsigned)vtx[j] & ~kSTag);
            }
        }
        long long off[kCapPer], deg[kCapPer];
#pragma unroll
        for (int j = 0; j < kCapPer; ++j) {
            if (VALS) {
                if (in[j]) p.dist[vtx[j]] = dv[j];
            } else {
                dv[j] = in[j] ? __ldcg(p.dist + vtx[j]) : (D)0;
            }
            const uint2 ri = in[j] ? __ldg(ptr + vtx[j]) : make_uint2(0u, 0u);
            off[j] = ri.x;
            deg[j] = ri.y;
            if (in[j] && clear_bits) clear_bits[(unsigned)vtx[j] >> 5] = 0u;
        }
        if (HOPS && std::is_same<M, ModeFixed>::value) {
            // lex mode, S capture of an internal bucket: its largest hop count
            // (S holds the bucket's final keys)
            if (p.lex) {
#pragma unroll
                for (int j = 0; j < kCapPer; ++j)
                    if (in[j]) hop_cta = max(hop_cta, (unsigned)dv[j] & kHopMask);
            }
        }
        if (APPEND_S) {
            bool news[kCapPer];
#pragma unroll
            for (int j = 0; j < kCapPer; ++j)
                news[j] = kSEntry ? tagged[j] : (in[j] && claim_bit(p.sbits, (unsigned)vtx[j]));
#pragma unroll
            for (int j = 0; j < kCapPer; ++j)
                wq_push<D, false>(ws.q, queue_vals(ws), qn, news[j], vtx[j], (D)0, lane, S, nullptr, s_counter);
            if (!DS_LATE_FLUSH || qn > (unsigned)kQueue / 2)
                wq_flush<D, false>(ws.q, queue_vals(ws), qn, lane, S, nullptr, s_counter);
        }
        capture_emit_cta<M, kCapPer>(p, sm, slot, lane, wib, dv, off, deg);
    }
    if (APPEND_S) wq_flush<D, false>(ws.q, queue_vals(ws), qn, lane, S, nullptr, s_counter);
    if (HOPS && std::is_same<M, ModeFixed>::value && p.lex) {
#pragma unroll
        for (int o = 16; o; o >>= 1) hop_cta = max(hop_cta, __shfl_xor_sync(0xffffffffu, hop_cta, o));
        if (lane == 0 && hop_cta) atomicMax(&slot->hopmax, hop_cta);  // once per warp and capture
    }
}

// ---------------------------------------------------------------- relax step (push)
//
// Edge-balanced push over the entries of the last capture.  LIGHT: successful
// improvements that land inside the window join the next frontier once
// (bitmap dedup); HEAVY: min-merge only (results land beyond the window).

#ifndef DS_RELAX_INLINE
#define DS_RELAX_INLINE __forceinline__
#endif
// Inlined: a __noinline__ push measured 25% slower (the kernel parameters
// then live in a local-memory frame).
template <class M>
__device__ __forceinline__ void csum_lower(const KParams<M>& p, unsigned v, typename M::D nd) {
    typename M::D* b = p.csum + v / (32u * kRangePer);
#if DS_CSUM_RED
    atomicMin(b, nd);  // result unused: a fire-and-forget reduction, no round trip
#else
    if (nd < *b) atomicMin(b, nd);  // a stale (L1) bound is >= the current one
#endif
}

// Row map of a warp chunk from the entries' start marks: every chunk edge takes
// the largest mark at or before it (one warp max-scan instead of a per-lane
// search and walk).  ws.row holds the marks on entry, the entry index per edge
// on return; the caller syncs the warp around it.
template <class D>
__device__ __forceinline__ void rowmap_scan(WarpSmem<D>& ws, int lane) {
    static_assert(kRelPer == 8 || kRelPer == 4, "row-map scan: 4 or 8 edges per lane");
    unsigned w[kRelPer / 2];  // the lane's kRelPer marks, two per word
    if constexpr (kRelPer == 8) {
        const uint4 m4 = reinterpret_cast<uint4*>(ws.row)[lane];
        w[0] = m4.x; w[1] = m4.y; w[2] = m4.z; w[3] = m4.w;
    } else {
        const uint2 m2 = reinterpret_cast<uint2*>(ws.row)[lane];
        w[0] = m2.x; w[1] = m2.y;
    }
    unsigned v[kRelPer];
#pragma unroll
    for (int j = 0; j < kRelPer; ++j) v[j] = (j & 1) ? (w[j / 2] >> 16) : (w[j / 2] & 0xFFFFu);
#pragma unroll
    for (int j = 1; j < kRelPer; ++j) v[j] = max(v[j], v[j - 1]);
    unsigned run = v[kRelPer - 1];  // inclusive max-scan of the lanes' maxima
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, run, o);
        if (lane >= o) run = max(run, t);
    }
    unsigned carry = __shfl_up_sync(0xffffffffu, run, 1);
    if (lane == 0) carry = 0;
#pragma unroll
    for (int j = 0; j < kRelPer; ++j) v[j] = max(v[j], carry);
#pragma unroll
    for (int j = 0; j < kRelPer / 2; ++j) w[j] = v[2 * j] | (v[2 * j + 1] << 16);
    if constexpr (kRelPer == 8)
        reinterpret_cast<uint4*>(ws.row)[lane] = make_uint4(w[0], w[1], w[2], w[3]);
    else
        reinterpret_cast<uint2*>(ws.row)[lane] = make_uint2(w[0], w[1]);
}

// SUM: also lower the scan-chunk bound of every target that may have received
// a value beyond the window (SMALL kernel, see capture_range).
// PULL (heavy only): the entries are the UNSETTLED rows v (capture_range
// UNSET, entry value = v) and every edge v->u of A_H (= A_H^T, symmetric
// graphs) gathers t[u] + w when u is settled (t[u] < H): the reference's own
// pulled form of the heavy relaxation, r = A_H^T (t o S) (sssp.py:206-227),
// restricted to the rows it can still lower.  See the direction choice at
// POS_HEAVY for why this is exact.
// STAG (light, kSEntry): the push that brings a vertex from at-or-beyond H to
// below H tags its next-frontier entry with kSTag (the capture of that list
// appends the vertex to S); if it loses the dedup claim it appends to
// S[sidx] directly.
// WIDE (lex mode, light): the window spans several reference buckets, so the
// hop rule's bound -- the upper end of the SOURCE's reference bucket -- is
// looked up per captured entry in the window's threshold table (sm.wthr) and
// kept as an index in the warp's rel[] slots (no entry pipelining: the wide
// steps are latency-bound tails with about one chunk per warp).
template <class M, bool LIGHT, bool LOCALW = false, bool SUM = false, bool PULL = false, bool LEX = false,
          bool STAG = false, bool WIDE = false>
__device__ DS_RELAX_INLINE void relax_step(const KParams<M>& p, Smem<typename M::D>& sm, StepSlot* slot,
                           unsigned long long E, unsigned long long Rc,
                           const typename M::Edge* edges, typename M::D H, int* out_list,
                           unsigned* fbits, typename M::D HD = 0, unsigned sidx = 0) {
    static_assert(!STAG || (LIGHT && DS_DEFER_APPEND), "S tags ride on the deferred light appends");
    static_assert(!WIDE || (LIGHT && LEX && !PULL && DS_ROWMAP_SCAN), "wide windows: lex-mode light pushes");
    constexpr bool kPipe = DS_PIPE != 0 && !WIDE;
    using D = typename M::D;
    using Edge = typename M::Edge;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    WarpSmem<D>& ws = sm.w[wib];
    unsigned qn = 0;
    const unsigned long long nchunk = (E + kChunk - 1) / kChunk;
    // warps per block from the launch: the standalone push may run narrower blocks
    const unsigned wpb = LOCALW ? (unsigned)kWarps : (blockDim.x >> 5);
    const unsigned long long gw = LOCALW ? wib : (unsigned long long)blockIdx.x * wpb + wib;
    const unsigned long long nw = LOCALW ? kWarps : (unsigned long long)gridDim.x * wpb;
    const unsigned long long pol = LIGHT ? light_policy() : evict_first_policy();
    bool overflow = false;
    // entries of chunk c -> this warp's smem (offset, row base, captured d)
    // and the row map: lane resolves the entry of chunk edges [8 lane, 8 lane + 8)
    // DS_CS_PREFETCH: the chunk map words of a warp's next chunk are loaded one
    // iteration early (two registers), taking a round trip off the chain
#if DS_CHECKS
    int ne_chk = 0;  // entries of the chunk in flight
#endif
    unsigned cs0 = 0, cs1 = 0;
    auto cs_fetch = [&](unsigned long long c) {
        if (c < nchunk) {
            cs0 = ldcg(p.chunk_start + c);
            cs1 = (c + 1 < nchunk) ? ldcg(p.chunk_start + c + 1) : (unsigned)(Rc - 1);
        }
    };
    if (DS_CS_PREFETCH) cs_fetch(gw);
    auto load_meta = [&](unsigned long long c) {
        unsigned long long r0, r1;
        if (DS_CS_PREFETCH) {
            r0 = cs0;
            r1 = cs1;
            cs_fetch(c + nw);
        } else {
            r0 = ldcg(p.chunk_start + c);
            r1 = (c + 1 < nchunk) ? ldcg(p.chunk_start + c + 1) : Rc - 1;
        }
        const int ne = (int)(r1 - r0 + 1);
        const long long cb = (long long)(c * kChunk);
        DS_ASSERT(ne >= 1 && ne <= kChunk + 1 && r1 < Rc);
#if DS_CHECKS
        ne_chk = ne;
#endif
#if DS_ROWMAP_SCAN
        // row map by marks + prefix max: entry k marks the chunk edge where
        // its row starts, then every edge takes the largest mark at or
        // before it (one warp scan instead of a per-lane search and walk)
        static_assert(kRelPer == 8 || kRelPer == 4, "row-map scan: 4 or 8 edges per lane");
        if (kRelPer == 8)
            reinterpret_cast<uint4*>(ws.row)[lane] = make_uint4(0u, 0u, 0u, 0u);
        else
            reinterpret_cast<uint2*>(ws.row)[lane] = make_uint2(0u, 0u);
        __syncwarp();
        for (int k = lane; k < ne; k += 32) {
            const unsigned long long r = r0 + k;
            const uint2 en = __ldcg(p.Rent + r);
            const long long rel = (long long)en.x - cb;
            // the entry of chunk_start[c + 1] may begin exactly at the next chunk
            if (rel < kChunk) ws.row[rel < 0 ? 0 : rel] = (unsigned short)k;
            ws.base[k] = en.y + (unsigned)cb;
            const D dk = __ldcg(p.Rd + r);
            ws.d[k] = dk;
            if constexpr (WIDE) {
                // upper end of the reference bucket holding the entry's distance
                const unsigned Du = (unsigned)(dk >> kHopBits);
                int a = 0, b = sm.wn;
                while (b - a > 1) {
                    const int m = (a + b) >> 1;
                    if (sm.wthr[m] <= Du) a = m;
                    else b = m;
                }
                ws.rel[k] = (short)(a + 1);  // index of that bound in sm.wthr (rel[] is free: DS_ROWMAP_SCAN)
            }
        }
        __syncwarp();
        rowmap_scan<D>(ws, lane);
        __syncwarp();
#else
        for (int k = lane; k < ne; k += 32) {
            const unsigned long long r = r0 + k;
            const uint2 en = __ldcg(p.Rent + r);
            const long long rel = (long long)en.x - cb;
            ws.rel[k] = (short)(rel < 0 ? 0 : rel);
            ws.base[k] = en.y + (unsigned)cb;
            ws.d[k] = __ldcg(p.Rd + r);
        }
        __syncwarp();
        const int rel0 = lane * kRelPer;
        int lo = 0, hi = ne;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (ws.rel[mid] <= rel0) lo = mid;
            else hi = mid;
        }
        int k = lo;
#pragma unroll
        for (int j = 0; j < kRelPer; ++j) {
            while (k + 1 < ne && ws.rel[k + 1] <= rel0 + j) ++k;
            ws.row[rel0 + j] = (unsigned short)k;
        }
        __syncwarp();
#endif
    };
    if constexpr (kPipe) {
        if (gw < nchunk) load_meta(gw);
    }
    // DS_DEFER_APPEND (light): a chunk's dedup claims are consumed (appended)
    // only after the next chunk's edge loads are out, hiding their round trip
    unsigned p_col[kRelPer], p_ret[kRelPer];
    unsigned p_req = 0, p_tag = 0;  // claims requested / of those, the pushes that brought a vertex into the window
#pragma unroll
    for (int j = 0; j < kRelPer; ++j) p_col[j] = p_ret[j] = 0u;
    auto drain = [&]() {
        unsigned gm = 0;
#pragma unroll
        for (int j = 0; j < kRelPer; ++j) {
            const bool g = ((p_req >> j) & 1u) && !(p_ret[j] & (1u << (p_col[j] & 31)));
            wq_push<D, false>(ws.q, queue_vals(ws), qn, g, (int)p_col[j], (D)0, lane, out_list, nullptr,
                              &slot->append_count);
            gm |= (g ? 1u : 0u) << j;
        }
        // STAG: entered the window but lost the frontier claim (rare)
        const unsigned lostbits = STAG ? (p_tag & ~gm) : 0u;
        if (STAG && __any_sync(0xffffffffu, lostbits != 0u)) {
            // those go to S directly, one reservation for the warp
            const unsigned cnt = __popc(lostbits);
            unsigned incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            unsigned long long b = 0;
            if (lane == 31) b = atomicAdd(&p.ctl->s_count[sidx], (unsigned long long)incl);
            b = __shfl_sync(0xffffffffu, b, 31) + (incl - cnt);
#pragma unroll
            for (int j = 0; j < kRelPer; ++j)
                if ((lostbits >> j) & 1u) p.S[sidx][b++] = (int)(p_col[j] & ~kSTag);
        }
        p_req = 0;
        p_tag = 0;
        if (!DS_LATE_FLUSH || qn > (unsigned)kQueue / 2)
            wq_flush<D, false>(ws.q, queue_vals(ws), qn, lane, out_list, nullptr, &slot->append_count);
    };
    for (unsigned long long c = gw; c < nchunk; c += nw) {
        const long long cb = (long long)(c * kChunk);
        if constexpr (!kPipe) load_meta(c);
        const long long left = (long long)E - cb - lane;  // edge j exists iff 32 j < left
        Edge ed[kRelPer];
        int kk[kRelPer];  // !kPipe: the edges' entries
#if DS_PIPE
        if constexpr (kPipe) {
        // issue this chunk's edge loads, park the per-edge source values in
        // smem, then fetch the next chunk's entries while the edges are in flight
#pragma unroll
        for (int j = 0; j < kRelPer; ++j) {
            const int r = lane + 32 * j;
            const int kj = ws.row[r];
            kk[j] = 0;
            // unconditional definition: a conditionally assigned ed[] is
            // loop-carried and was spilled to local memory
            ed[j] = (32 * j < left) ? M::load(edges + (unsigned)(ws.base[kj] + r), pol) : Edge{};
            ws.du[r] = ws.d[kj];
        }
        __syncwarp();
        if (c + nw < nchunk) load_meta(c + nw);
        } else
#endif
        {
#pragma unroll
        for (int j = 0; j < kRelPer; ++j) {
            const int r = lane + 32 * j;
            kk[j] = ws.row[r];
#if DS_CHECKS
            if (32 * j < left) {
                const unsigned long long lim =
                    edges == p.Ledges ? p.nL : (edges == p.Hedges ? p.nH : (edges == p.Aedges ? p.nA : ~0ull));
                DS_ASSERT(kk[j] < ne_chk);
                // (the partitioned solver's parameter blocks carry no counts: 0 = unchecked)
                DS_ASSERT(lim == 0 || (unsigned long long)(unsigned)(ws.base[kk[j]] + r) < lim);
            }
#endif
            // unconditional definition: a conditionally assigned ed[] is
            // loop-carried and was spilled to local memory
            ed[j] = (32 * j < left) ? M::load(edges + (unsigned)(ws.base[kk[j]] + r), pol) : Edge{};
#if DS_CHECKS
            if (32 * j < left) DS_ASSERT((long long)M::col(ed[j]) < p.n);
#endif
        }
#if DS_L2PF
        // L2 prefetch of this warp's next chunk: cs0 already holds its first
        // entry (cs_fetch above); from that entry's {prefix, base - prefix}
        // its first edge is at base + chunk offset, and hub rows make the
        // chunk one contiguous 256-edge run.  The bulk prefetch goes through
        // the TMA unit, not the SM's L1 miss queue, so the edge loads of the
        // next iteration hit L2 instead of HBM.
        if (DS_CS_PREFETCH && lane == 0 && c + nw < nchunk) {
            const uint2 en = __ldcg(p.Rent + cs0);
            const unsigned long long cbn = (c + nw) * kChunk;
            const unsigned long long a =
                reinterpret_cast<unsigned long long>(edges + (unsigned)(en.y + (unsigned)cbn)) & ~15ull;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((unsigned)(kChunk * sizeof(Edge) + 16))
                         : "memory");
        }
#endif
        }
#if DS_PIPE
#define DS_DU(j) (kPipe ? ws.du[lane + 32 * (j)] : ws.d[kk[j]])
#else
#define DS_DU(j) ws.d[kk[j]]
#endif
#define DS_HD(j) (WIDE ? (D)sm.wthr[ws.rel[kk[j]]] : HD)
        if constexpr (PULL) {
            // gather: source value t[u] (settled iff < H; settled values are
            // final, so an L1 copy is exact) and the row's own value (a stale
            // copy is >= the current one: at worst a redundant atomic)
            D du[kRelPer], cur[kRelPer];
#pragma unroll
            for (int j = 0; j < kRelPer; ++j) {
                du[j] = M::INF;
                cur[j] = (D)0;
                if (32 * j < left) {
                    du[j] = p.dist[M::col(ed[j])];
                    cur[j] = p.dist[(unsigned)DS_DU(j)];
                }
            }
#pragma unroll
            for (int j = 0; j < kRelPer; ++j) {
                if (32 * j < left && du[j] < H) {
                    D nd;
                    if (!padd<LEX>(p, du[j], ed[j], HD, nd)) {
                        overflow = true;
                    } else if (nd < cur[j]) {
                        const unsigned v = (unsigned)DS_DU(j);
                        atomicMin(p.dist + v, nd);
                        if (SUM) csum_lower(p, v, nd);
                    }
                }
            }
            __syncwarp();
            continue;
        }
        if (LIGHT && DS_DEFER_APPEND) drain();  // previous chunk's claims, edges in flight
        D nd[kRelPer], cur[kRelPer];
#pragma unroll
        for (int j = 0; j < kRelPer; ++j) {
            cur[j] = (D)0;
            nd[j] = (D)0;  // defined on every path (see ed[] above)
            if (32 * j < left) {
                if (padd<LEX>(p, DS_DU(j), ed[j], DS_HD(j), nd[j])) {
                    // a stale (L1) value is >= the current one: it can only
                    // cause a redundant atomic, never a missed improvement
                    const unsigned v = M::col(ed[j]);
#if DS_PRECHECK_CUT
                    // hub targets (solver ids below the cut) through L1, the rest
                    // straight from L2 so they do not evict the hub lines
                    cur[j] = v < (unsigned)DS_PRECHECK_CUT ? p.dist[v] : __ldcg(p.dist + v);
#else
                    cur[j] = (LIGHT || !kHeavyRed) ? (DS_PRECHECK_L1 ? p.dist[v] : __ldcg(p.dist + v))
                                                   : M::INF;
#endif
                } else {
                    overflow = true;
                }
            }
        }
        if (LIGHT) {
            // all pushes first, then all dedup claims, then the appends: the
            // returning atomics of one chunk overlap instead of serialising
            // behind a warp vote per edge
            D old[kRelPer];
#pragma unroll
            for (int j = 0; j < kRelPer; ++j) {
                old[j] = nd[j];
                if (32 * j < left && nd[j] < cur[j]) old[j] = atomicMin(p.dist + M::col(ed[j]), nd[j]);
            }
#if DS_COUNT
            {
                unsigned long long na = 0, ni = 0;
#pragma unroll
                for (int j = 0; j < kRelPer; ++j) {
                    if (32 * j < left && nd[j] < cur[j]) ++na;
                    if (32 * j < left && nd[j] < old[j]) ++ni;
                }
                na = warp_sum(na);
                ni = warp_sum(ni);
                if (lane == 0) {
                    atomicAdd(&p.ctl->cnt_atomics, na);
                    atomicAdd(&p.ctl->cnt_improved, ni);
                }
            }
#endif
#if DS_DEFER_APPEND
#pragma unroll
            for (int j = 0; j < kRelPer; ++j) {
                const unsigned v = M::col(ed[j]);
                const bool want = 32 * j < left && nd[j] < old[j] && nd[j] < H;
                if (SUM && 32 * j < left && nd[j] < old[j] && nd[j] >= H) csum_lower(p, v, nd[j]);
                const bool tag = STAG && want && old[j] >= H;
                p_col[j] = tag ? (v | kSTag) : v;
                p_ret[j] = want ? atomicOr(fbits + (v >> 5), 1u << (v & 31)) : 0u;
                p_req |= (want ? 1u : 0u) << j;
                p_tag |= (tag ? 1u : 0u) << j;
            }
#else
            unsigned got[kRelPer];
#pragma unroll
            for (int j = 0; j < kRelPer; ++j) {
                got[j] = 0;
                if (32 * j < left && nd[j] < old[j] && nd[j] < H) {
                    const unsigned v = M::col(ed[j]);
                    got[j] = atomicOr(fbits + (v >> 5), 1u << (v & 31)) & (1u << (v & 31));
                    got[j] = got[j] ? 0u : 1u;
                }
                if (SUM && 32 * j < left && nd[j] < old[j] && nd[j] >= H) csum_lower(p, M::col(ed[j]), nd[j]);
            }
#pragma unroll
            for (int j = 0; j < kRelPer; ++j)
                wq_push<D, false>(ws.q, queue_vals(ws), qn, got[j] != 0, (int)M::col(ed[j]), (D)0, lane,
                                  out_list, nullptr, &slot->append_count);
            if (!DS_LATE_FLUSH || qn > (unsigned)kQueue / 2)
                wq_flush<D, false>(ws.q, queue_vals(ws), qn, lane, out_list, nullptr, &slot->append_count);
#endif
        } else {
#pragma unroll
            for (int j = 0; j < kRelPer; ++j)
                if (32 * j < left && nd[j] < cur[j]) {
                    atomicMin(p.dist + M::col(ed[j]), nd[j]);
                    if (SUM) csum_lower(p, M::col(ed[j]), nd[j]);  // heavy values are >= hi
                }
        }
        __syncwarp();
#undef DS_DU
#undef DS_HD
    }
    if (LIGHT && DS_DEFER_APPEND) drain();
    // DS_LATE_FLUSH: appends stay in the warp queue across chunks until it
    // is half full, so most chunks skip the reservation round trip
    if (LIGHT) wq_flush<D, false>(ws.q, queue_vals(ws), qn, lane, out_list, nullptr, &slot->append_count);
    if (__any_sync(0xffffffffu, overflow) && lane == 0) atomicOr(&slot->flags, LEX ? 2u : 1u);
}

// ---------------------------------------------------------------- bidirectional step
//
// Entry into the wide tail (lex mode, symmetric graphs), replacing the heavy
// gather + the window's scan + its first push round.  Entries are the
// UNSETTLED rows v (value >= HN) over the merged rows (A); one pass reads
// t[u] for every edge (v,u) ONCE and uses it in both directions:
//  A  gather: u settled (t[u] < HN) contributes t[u] + w to v (the bucket's
//     heavy step; the light edges of settled sources were pushed with their
//     final values already, so re-applying them is a no-op), min-reduced per
//     row in the warp's shared memory;
//  B  per entry: one atomicMin commits a lowered row; rows lying inside this
//     warp chunk are complete, rows crossing a chunk boundary join the next
//     frontier when they hold a value in the window, and push from there;
//  C  push back: t[v] + w to every neighbour it improves -- the window's
//     first round, with t[u] from A as the pre-check.
// Every edge between two unsettled rows is seen from both ends, and a vertex
// lowered after its own row was processed joins the next frontier, so after
// the step "t[b] <= t[a] + w, or a is in the frontier" holds for every edge:
// the wide window continues with ordinary rounds.  S of the window: rows
// already inside it at the capture (capture_unsettled), plus the one atomic
// that brings a vertex from at-or-beyond HW to below it (returned old value).
template <class M>
__device__ void bidir_step(const KParams<M>& p, Smem<typename M::D>& sm, StepSlot* slot,
                           unsigned long long E, unsigned long long Rc, typename M::D HN,
                           typename M::D HW, typename M::D HD, int* out_list, unsigned* fbits,
                           unsigned sidx) {
    using D = typename M::D;
    using Edge = typename M::Edge;
    static_assert(kRelPer == 8 && DS_ROWMAP_SCAN, "bidirectional step: 256-edge chunks, scanned row map");
    static_assert(std::is_same<D, unsigned>::value, "bidirectional step: lex mode (32-bit keys)");
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    WarpSmem<D>& ws = sm.w[wib];
    unsigned qn = 0;
    const unsigned long long nchunk = (E + kChunk - 1) / kChunk;
    const unsigned long long gw = (unsigned long long)blockIdx.x * kWarps + wib;
    const unsigned long long nw = (unsigned long long)gridDim.x * kWarps;
    const unsigned long long pol = evict_first_policy();
    // one reservation per warp for direct S appends
    auto s_append = [&](unsigned bits, const unsigned (&ids)[kRelPer]) {
        if (!__any_sync(0xffffffffu, bits != 0u)) return;
        const unsigned cnt = __popc(bits);
        unsigned incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        unsigned long long b = 0;
        if (lane == 31) b = atomicAdd(&p.ctl->s_count[sidx], (unsigned long long)incl);
        b = __shfl_sync(0xffffffffu, b, 31) + (incl - cnt);
#pragma unroll
        for (int j = 0; j < kRelPer; ++j)
            if ((bits >> j) & 1u) p.S[sidx][b++] = (int)ids[j];
    };
    for (unsigned long long c = gw; c < nchunk; c += nw) {
        const long long cb = (long long)(c * kChunk);
        const unsigned long long r0 = ldcg(p.chunk_start + c);
        const unsigned long long r1 = (c + 1 < nchunk) ? ldcg(p.chunk_start + c + 1) : Rc - 1;
        const int ne = (int)(r1 - r0 + 1);
        DS_ASSERT(ne >= 1 && ne <= kChunk + 1 && r1 < Rc);
        reinterpret_cast<uint4*>(ws.row)[lane] = make_uint4(0u, 0u, 0u, 0u);
        __syncwarp();
        for (int k = lane; k < ne; k += 32) {
            const unsigned long long r = r0 + k;
            const uint2 en = __ldcg(p.Rent + r);
            const long long rel = (long long)en.x - cb;
            if (rel < kChunk) ws.row[rel < 0 ? 0 : rel] = (unsigned short)k;
            ws.base[k] = en.y + (unsigned)cb;
            ws.d[k] = __ldcg(p.Rd + r);  // the row id
            // the row ends where the next entry starts (the step's last row at E)
            const long long end = (r + 1 < Rc) ? (long long)__ldcg(p.Rent + r + 1).x : (long long)E;
            ws.rel[k] = (short)((rel >= 0 && end - cb <= kChunk) ? 1 : 0);  // 1: the whole row lies in this chunk
        }
        __syncwarp();
        rowmap_scan<D>(ws, lane);
        __syncwarp();
        const long long left = (long long)E - cb - lane;  // edge j exists iff 32 j < left
        Edge ed[kRelPer];
        int kk[kRelPer];
#pragma unroll
        for (int j = 0; j < kRelPer; ++j) {
            const int r = lane + 32 * j;
            kk[j] = ws.row[r];
            if (32 * j < left) {
                DS_ASSERT(kk[j] < ne && kk[j] < kChunk);
                DS_ASSERT((unsigned long long)(unsigned)(ws.base[kk[j]] + r) < p.nA);
            }
            ed[j] = (32 * j < left) ? M::load(p.Aedges + (unsigned)(ws.base[kk[j]] + r), pol) : Edge{};
            if (32 * j < left) DS_ASSERT((long long)M::col(ed[j]) < p.n);
        }
        __syncwarp();  // every lane holds its entries and addresses: base[] and row[] are free
        // the rows' current values, min-reduced in shared memory by the gather
        // (base[k]); row[k]: the gather lowered it
        for (int k = lane; k < ne; k += 32) {
            ws.base[k] = (unsigned)__ldcg(p.dist + (unsigned)ws.d[k]);
            if (k < kChunk) ws.row[k] = 0;
        }
        D du[kRelPer];
#pragma unroll
        for (int j = 0; j < kRelPer; ++j)  // settled values are final; the rest only pre-check (stale is >=)
            du[j] = (32 * j < left) ? p.dist[M::col(ed[j])] : M::INF;
        __syncwarp();
        // ---- A: gather from the settled neighbours
#pragma unroll
        for (int j = 0; j < kRelPer; ++j) {
            if (32 * j < left && du[j] < HN) {
                D nd;
                padd<true>(p, du[j], ed[j], HD, nd);
                if ((unsigned)nd < atomicMin(&ws.base[kk[j]], (unsigned)nd)) ws.row[kk[j]] = 1;
            }
        }
        __syncwarp();
        // ---- B: per row, commit the gathered value; what the row does next
        for (int k0 = 0; k0 < ne; k0 += 32) {
            const int k = k0 + lane;
            bool fr = false, sev = false;
            unsigned v = 0;
            if (k < ne) {
                v = (unsigned)ws.d[k];
                const bool whole = ws.rel[k] != 0;
                D tv = (D)ws.base[k];
                if (k < kChunk && ws.row[k]) {
                    const D old = atomicMin(p.dist + v, tv);
                    sev = old >= HW && tv < HW;  // the one atomic that brings it into the window
                    tv = old < tv ? old : tv;
                }
                D keep = M::INF;
                if (tv < HW) {
                    if (whole) {
                        keep = tv;
                        const unsigned Du = (unsigned)(tv >> kHopBits);
                        int a = 0, b = sm.wn;
                        while (b - a > 1) {
                            const int m = (a + b) >> 1;
                            if (sm.wthr[m] <= Du) a = m;
                            else b = m;
                        }
                        ws.rel[k] = (short)(a + 1);  // the bound of its reference bucket, in sm.wthr
                    } else {
                        fr = claim_bit(fbits, v);  // crosses a chunk boundary: pushes from the next frontier
                    }
                }
                ws.base[k] = (unsigned)keep;
            }
            const unsigned sm_ = __ballot_sync(0xffffffffu, sev);
            if (sm_) {
                unsigned long long b = 0;
                if (lane == 0) b = atomicAdd(&p.ctl->s_count[sidx], (unsigned long long)__popc(sm_));
                b = __shfl_sync(0xffffffffu, b, 0);
                if (sev) p.S[sidx][b + __popc(sm_ & ((1u << lane) - 1u))] = (int)v;
            }
            wq_push<D, false>(ws.q, queue_vals(ws), qn, fr, (int)v, (D)0, lane, out_list, nullptr,
                              &slot->append_count);
        }
        __syncwarp();
        // ---- C: push back
        {
            D nd[kRelPer], old[kRelPer];
            unsigned tgt[kRelPer];
            unsigned want = 0;
#pragma unroll
            for (int j = 0; j < kRelPer; ++j) {
                nd[j] = old[j] = (D)0;
                tgt[j] = M::col(ed[j]);
                const D tv = (D)ws.base[kk[j]];
                if (32 * j < left && tv != M::INF) {
                    padd<true>(p, tv, ed[j], (D)sm.wthr[ws.rel[kk[j]]], nd[j]);
                    old[j] = nd[j];
                    if (nd[j] < du[j]) old[j] = atomicMin(p.dist + tgt[j], nd[j]);
                    if (nd[j] < old[j] && nd[j] < HW) want |= 1u << j;
                }
            }
            unsigned ret[kRelPer];
#pragma unroll
            for (int j = 0; j < kRelPer; ++j)
                ret[j] = ((want >> j) & 1u) ? atomicOr(fbits + (tgt[j] >> 5), 1u << (tgt[j] & 31)) : 0u;
            unsigned lost = 0;  // entered the window but lost the frontier claim: S directly
#pragma unroll
            for (int j = 0; j < kRelPer; ++j) {
                const bool w = (want >> j) & 1u;
                const bool g = w && !(ret[j] & (1u << (tgt[j] & 31)));
                const bool tag = w && old[j] >= HW;
                wq_push<D, false>(ws.q, queue_vals(ws), qn, g, (int)(tag ? (tgt[j] | kSTag) : tgt[j]), (D)0, lane,
                                  out_list, nullptr, &slot->append_count);
                if (tag && !g) lost |= 1u << j;
            }
            s_append(lost, tgt);
        }
        if (qn > (unsigned)kQueue / 2)
            wq_flush<D, false>(ws.q, queue_vals(ws), qn, lane, out_list, nullptr, &slot->append_count);
        __syncwarp();
    }
    wq_flush<D, false>(ws.q, queue_vals(ws), qn, lane, out_list, nullptr, &slot->append_count);
}

// ---------------------------------------------------------------- pull step
//
// The reference's own formulation of a relaxation -- a (min,+) product
// gathered through the transposed matrix (fused_masked_relax,
// fused.py:127-161; vxm_min_plus, ops.py:238-271) -- used when the frontier
// touches a large share of the edges.  Needs A^T = A (symmetric graphs).
//  LIGHT: an edge u->v contributes iff t[u] lies in the bucket window.  That
//    gates a superset of the frontier, but every in-window vertex outside the
//    frontier already pushed its current value, so the improving minima are
//    exactly the frontier's.  In-window improvements are NOT written to t
//    (they would change the gate mid-phase): they become the next frontier
//    with their values and the next capture commits them.  Improvements
//    beyond the window are written directly (they never pass the gate).
//  HEAVY: u contributes iff u is in S (bitmap); S values are final.
// Rows are reduced per 256-edge chunk in shared memory; rows crossing a
// chunk boundary combine partial minima in `req` for the commit step.

template <class M, bool LIGHT>
__device__ __forceinline__ void pull_row_commit(const KParams<M>& p, typename M::D rmin, int rr,
                                                typename M::D H, bool& want, typename M::D& val) {
    const typename M::D cur = __ldcg(p.dist + rr);
    if (rmin < cur) {
        if (LIGHT && rmin < H) {
            want = true;
            val = rmin;
        } else {
            p.dist[rr] = rmin;
        }
    }
}

template <class M, bool LIGHT>
__device__ void pull_step(const KParams<M>& p, Smem<typename M::D>& sm, StepSlot* slot,
                          const PullPlan& pl, const typename M::Edge* edges, typename M::D L,
                          typename M::D H, int* out_list, typename M::D* out_vals) {
    using D = typename M::D;
    using Edge = typename M::Edge;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    WarpSmem<D>& ws = sm.w[wib];
    unsigned qn = 0;
    const unsigned long long nchunk = ((unsigned long long)pl.nnz + kChunk - 1) / kChunk;
    const unsigned long long gw = (unsigned long long)blockIdx.x * (blockDim.x >> 5) + wib;
    const unsigned long long nw = (unsigned long long)gridDim.x * (blockDim.x >> 5);
    const unsigned long long pol = evict_first_policy();
    bool overflow = false;
    for (unsigned long long c = gw; c < nchunk; c += nw) {
        const long long e0 = (long long)(c * kChunk);
        const long long e1 = e0 + kChunk < pl.nnz ? e0 + kChunk : pl.nnz;
        const int k0 = (int)__ldg(pl.chunk_row + c);
        const int k1 = (int)__ldg(pl.chunk_row + c + 1);
        const int ne = k1 - k0 + 1;
        for (int i = lane; i < ne; i += 32) {
            const long long rs = __ldg(pl.cptr + k0 + i) - e0;  // < 0: row began earlier
            ws.rel[i] = (short)(rs < 0 ? -1 : rs);
            ws.base[i] = (unsigned)__ldg(pl.cptr + k0 + i + 1);  // row end
            ws.d[i] = M::INF;                                   // row minimum
        }
        __syncwarp();
        {   // row map
            const int rel0 = lane * kRelPer;
            int lo = 0, hi = ne;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (ws.rel[mid] <= rel0) lo = mid;
                else hi = mid;
            }
            int k = lo;
#pragma unroll
            for (int j = 0; j < kRelPer; ++j) {
                while (k + 1 < ne && ws.rel[k + 1] <= rel0 + j) ++k;
                ws.row[rel0 + j] = (unsigned short)k;
            }
        }
        __syncwarp();
        const long long left = e1 - e0 - lane;
        Edge ed[kRelPer];
#pragma unroll
        for (int j = 0; j < kRelPer; ++j)  // defined on every path (no loop-carried spill)
            ed[j] = (32 * j < left) ? M::load(edges + (e0 + lane + 32 * j), pol) : Edge{};
        // Heavy gate reads go through L1: within a heavy pull the S bits and S
        // values are frozen, and L1 is invalidated at every grid barrier
        // (gpu-scope fence -> CCTL.IVALL).
        D du[kRelPer];
        bool gate[kRelPer];
#pragma unroll
        for (int j = 0; j < kRelPer; ++j) {
            gate[j] = false;
            du[j] = (D)0;
            if (32 * j < left) {
                const unsigned u = M::col(ed[j]);
                if (LIGHT) {
                    du[j] = __ldcg(p.dist + u);
                    gate[j] = du[j] >= L && du[j] < H;
                } else if (kSEntry) {
                    // no S bitmap: S is exactly the vertices whose (final) value
                    // lies in the window
                    du[j] = p.dist[u];
                    gate[j] = du[j] >= L && du[j] < H;
                } else {
                    gate[j] = (p.sbits[u >> 5] >> (u & 31)) & 1u;
                    du[j] = gate[j] ? p.dist[u] : (D)0;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < kRelPer; ++j) {
            // segmented min over the lanes of this 32-edge window (rows are
            // contiguous runs), then one shared atomic per run
            D val = M::INF;
            if (gate[j]) {
                D nd;
                if (M::add(du[j], ed[j], nd)) val = nd;
                else overflow = true;
            }
            const int k = ws.row[lane + 32 * j];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const D ov = __shfl_up_sync(0xffffffffu, val, o);
                const int ok = __shfl_up_sync(0xffffffffu, k, o);
                if (lane >= o && ok == k && ov < val) val = ov;
            }
            const int kn = __shfl_down_sync(0xffffffffu, k, 1);
            if ((lane == 31 || kn != k) && val != M::INF) atomicMin(&ws.d[k], val);
        }
        __syncwarp();
        for (int b = 0; b < ne; b += 32) {
            const int i = b + lane;
            bool want = false;
            D val = (D)0;
            int rr = 0;
            if (i < ne) {
                const D rmin = ws.d[i];
                if (rmin != M::INF) {
                    rr = __ldg(pl.rowid + k0 + i);
                    if (ws.rel[i] >= 0 && (long long)ws.base[i] <= e1) {
                        pull_row_commit<M, LIGHT>(p, rmin, rr, H, want, val);
                    } else {
                        atomicMin(p.req + (k0 + i), rmin);  // row continues in other chunks
                    }
                }
            }
            if (LIGHT)
                wq_push<D, true>(ws.q, queue_vals(ws), qn, want, rr, val, lane, out_list, out_vals,
                                 &slot->append_count);
        }
        if (LIGHT) wq_flush<D, true>(ws.q, queue_vals(ws), qn, lane, out_list, out_vals, &slot->append_count);
        __syncwarp();
    }
    if (__any_sync(0xffffffffu, overflow) && lane == 0) atomicOr(&slot->flags, 1u);
}

// Finish rows that crossed chunk boundaries (after the pull step's barrier).
template <class M, bool LIGHT>
__device__ void commit_step(const KParams<M>& p, Smem<typename M::D>& sm, StepSlot* slot,
                            const PullPlan& pl, typename M::D H, int* out_list,
                            typename M::D* out_vals) {
    using D = typename M::D;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    WarpSmem<D>& ws = sm.w[wib];
    unsigned qn = 0;
    const unsigned long long gw = (unsigned long long)blockIdx.x * (blockDim.x >> 5) + wib;
    const unsigned long long nw = (unsigned long long)gridDim.x * (blockDim.x >> 5);
    for (unsigned long long b = gw * 32; b < (unsigned long long)pl.nspan; b += nw * 32) {
        const unsigned long long i = b + lane;
        bool want = false;
        D val = (D)0;
        int rr = 0;
        if (i < (unsigned long long)pl.nspan) {
            const int k = __ldg(pl.span + i);
            const D rmin = __ldcg(p.req + k);
            if (rmin != M::INF) {
                p.req[k] = M::INF;
                rr = __ldg(pl.rowid + k);
                const D cur = __ldcg(p.dist + rr);
                if (rmin < cur) {
                    p.dist[rr] = rmin;
                    if (LIGHT && rmin < H) {
                        want = true;
                        val = rmin;
                    }
                }
            }
        }
        if (LIGHT)
            wq_push<D, true>(ws.q, queue_vals(ws), qn, want, rr, val, lane, out_list, out_vals,
                             &slot->append_count);
    }
    if (LIGHT) wq_flush<D, true>(ws.q, queue_vals(ws), qn, lane, out_list, out_vals, &slot->append_count);
}

// ---------------------------------------------------------------- the solver

// Wide windows (lex mode).  The hop-count keys make the reference's counters a
// function of the final keys alone, so the schedule is free: once the buckets
// get small (the latency-bound tail of a power-law graph: ~75 us of barriers
// and round trips per bucket for a few thousand improving vertices) the solver
// merges G internal buckets into one window [L, H) and runs ONE closure over
// it that pushes every edge of a frontier row (A, not A_L: a window wider than
// the light threshold has no "heavy lands beyond" guarantee, and needs no
// heavy step).  Pushes landing below H join the next frontier, the rest only
// lower t -- label-correcting, same least fixpoint of the (D, h) keys.  After
// the closure one pass over the window's S (every vertex whose final key lies
// in it) takes the largest hop count per REFERENCE bucket, from which the
// bucket's phase count and visit follow as in the narrow schedule.
template <class M>
__device__ void wide_hop_pass(const KParams<M>& p, Smem<typename M::D>& sm, const int* S,
                              unsigned long long count, unsigned* out) {
    for (int j = threadIdx.x; j < kWideRef; j += kThreads) sm.whm[j] = 0u;
    __syncthreads();
    const int wn = sm.wn;
    const unsigned long long stride = (unsigned long long)gridDim.x * kThreads;
    for (unsigned long long i = (unsigned long long)blockIdx.x * kThreads + threadIdx.x; i < count; i += stride) {
        const unsigned v = (unsigned)ldcg(S + i);
        const unsigned long long key = (unsigned long long)__ldcg(p.dist + v);
        const unsigned Du = (unsigned)(key >> kHopBits);
        int a = 0, b = wn;
        while (b - a > 1) {
            const int m = (a + b) >> 1;
            if (sm.wthr[m] <= Du) a = m;
            else b = m;
        }
        DS_ASSERT(a >= 0 && a < wn && wn <= kWideRef && (long long)v < p.n);
        DS_ASSERT(Du >= sm.wthr[0] && Du < sm.wthr[wn]);  // every S member's final key lies in the window
        atomicMax(&sm.whm[a], (unsigned)(key & kHopMask) + 1u);
    }
    __syncthreads();
    if ((int)threadIdx.x < wn && sm.whm[threadIdx.x]) atomicMax(out + threadIdx.x, sm.whm[threadIdx.x]);
}

// Window of internal bucket idx: keys [L, H) and the reference bucket's upper
// bound HD in distance units.  Classic: idx is the reference bucket (keys =
// distances).  Lex: reference bucket idx / ksub split into ksub integer
// sub-windows, shifted into key space.
template <class M>
__device__ __forceinline__ void lex_window(const KParams<M>& p, bool lex, long long idx, double& lo,
                                           double& hi, typename M::D& L, typename M::D& H,
                                           typename M::D& HD) {
    using D = typename M::D;
    const int kl = lex ? p.ksub_log2 : 0;
    const long long ridx = idx >> kl;
    lo = (double)ridx * p.delta;
    hi = (double)(ridx + 1) * p.delta;
    D LD;
    M::window(lo, hi, p.frac, LD, HD);
    if (!lex) {
        L = LD;
        H = HD;
        return;
    }
    const unsigned long long w = (unsigned long long)HD - LD;
    const unsigned long long t = (unsigned long long)idx & ((1ull << kl) - 1);
    const unsigned long long a = LD + ((t * w) >> kl);
    const unsigned long long b = t + 1 == (1ull << kl) ? (unsigned long long)HD : LD + (((t + 1) * w) >> kl);
    L = (D)min(a << kHopBits, (unsigned long long)M::INF);
    H = (D)min(b << kHopBits, (unsigned long long)M::INF);
}

template <class M, bool SMALL, bool LEX = false>
__global__ void __launch_bounds__(kThreads, DS_MIN_BLOCKS)
    sssp_persistent_kernel(const KParams<M> p) {
    using D = typename M::D;
    constexpr bool kSum = SMALL && kCsum;  // scan-chunk bounds (high-diameter kernel only)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem<D>& sm = *reinterpret_cast<Smem<D>*>(smem_raw);
    Ctl* const c = p.ctl;
    unsigned gen = 0;
    unsigned long long deadline = 0;
    const int pos0 = (int)ldcg(&c->rs_pos);
    if (p.trace && blockIdx.x == 0 && threadIdx.x == 0 && pos0 == POS_FRESH) c->t_enter = globaltimer_ns();
    if (threadIdx.x == 0) {
        const unsigned long long now = globaltimer_ns();
        deadline = p.timeout_ns > ~0ull - now ? ~0ull : now + p.timeout_ns;  // saturating: ~0 = unarmed
        // resumed launches continue the barrier sequence
#if DS_BARRIER == 1
        gen = (unsigned)(ldcg(&c->bar_arrive) / gridDim.x);
#else
        gen = ldcg(&c->bar_gen);
#endif
    }

    // ---- init: t = {source: 0} (sssp.py:276), all else +inf.  Only solver
    // ids below n_scan can ever be reached (the source may be an isolated
    // vertex outside the active prefix).
    const long long src = __ldg(p.perm + p.source);
    const long long n_scan = p.n_active > src + 1 ? p.n_active : src + 1;
    if (pos0 == POS_FRESH) {
        const long long stride = (long long)gridDim.x * kThreads;
        for (long long v = (long long)blockIdx.x * kThreads + threadIdx.x; v < n_scan; v += stride)
            p.dist[v] = (v == src) ? (D)0 : M::INF;
        // dedup bitmaps start clear: a previous solve on these buffers may
        // have stopped mid-bucket (overflow / rerun), and pipelined batches
        // queue this launch before the host has seen that solve's status
        for (long long k = (long long)blockIdx.x * kThreads + threadIdx.x; k < (n_scan + 31) / 32; k += stride) {
            p.fbits[0][k] = 0u;
            p.fbits[1][k] = 0u;
            p.sbits[k] = 0u;
        }
        if (kSum) {
            const long long per = 32ll * kRangePer;
            for (long long k = (long long)blockIdx.x * kThreads + threadIdx.x; k < (n_scan + per - 1) / per;
                 k += stride)
                p.csum[k] = (k == src / per) ? (D)0 : M::INF;
        } else {
            // settled flags of the scan chunks (capture_range)
            unsigned* const chunk_done = reinterpret_cast<unsigned*>(p.csum);
            const long long per = 32ll * kRangePer;
            for (long long k = (long long)blockIdx.x * kThreads + threadIdx.x; k < (n_scan + per - 1) / per;
                 k += stride)
                chunk_done[k] = 0u;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            for (int k = 0; k < 3; ++k) {
                StepSlot* s = &c->slot[k];
                s->re_packed = s->front_count = s->append_count = 0;
                s->flags = 0;
                s->hopmax = 0;
                s->next_min = ~0ull;
            }
            c->s_count[0] = c->s_count[1] = 0;
        }
        if (!grid_sync(c, gen, deadline, sm)) return;
        if (p.trace && blockIdx.x == 0 && threadIdx.x == 0) c->last_bucket = (long long)globaltimer_ns();
    }

    // solver state (identical on every CTA; saved to / restored from Ctl)
    unsigned long long st = 0, nbar = 1, escanned = 0, npull = 0;
    long long idx = 0;
    unsigned long long phases = 0, visited = 0;
    unsigned long long re = 0, scount = 0, old_scount = 0;
    unsigned long long hset = 0;  // heavy edges of the rows settled so far
    int pp = 0;
    unsigned bpar = 0;
    int pos = POS_BUCKET;
    bool resumed = false;
    // wide windows (lex mode; no giant-push handoff there, so not saved)
    // (the window's parity and edge count live in shared memory: registers are scarce here)
    unsigned wideG = 0;  // internal buckets per window (0: the narrow schedule)

    if (pos0 != POS_FRESH) {
        st = ldcg(&c->rs_st);
        nbar = ldcg(&c->rs_nbar);
        escanned = ldcg(&c->rs_escanned);
        npull = ldcg(&c->rs_npull);
        idx = ldcg(&c->rs_idx);
        phases = ldcg(&c->rs_phases);
        visited = ldcg(&c->rs_visited);
        re = ldcg(&c->rs_re);
        scount = ldcg(&c->rs_scount);
        old_scount = ldcg(&c->rs_old_scount);
        pp = (int)ldcg(&c->rs_pp);
        bpar = (unsigned)ldcg(&c->rs_bpar);
        hset = ldcg(&c->rs_hset);
        pos = pos0;
        resumed = true;
    }
    int status = 0;

    auto end_step = [&](unsigned long long kind, unsigned long long work) -> bool {
        if (p.cta_done && st < p.trace_cap) {  // load-balance diagnostics (DS_TRACE=2)
            __syncthreads();
            if (threadIdx.x == 0) p.cta_done[st * gridDim.x + blockIdx.x] = globaltimer_ns();
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) {  // recycle the slot two steps ahead
            StepSlot* s = &c->slot[(st + 1) % 3];
            s->re_packed = s->front_count = s->append_count = 0;
            s->flags = 0;
            s->hopmax = 0;
            s->next_min = ~0ull;
        }
        const bool ok = grid_sync(c, gen, deadline, sm);
#if DS_CHECKS
        if (ok && blockIdx.x == 0 && threadIdx.x == 0) {  // the step's list lengths fit their arrays
            const StepSlot* s = &c->slot[st % 3];
            DS_ASSERT(ldcg(&s->append_count) <= (unsigned long long)p.n);
            DS_ASSERT((ldcg(&s->re_packed) >> kPackShift) <= (unsigned long long)p.n);
            DS_ASSERT((ldcg(&s->re_packed) & kMask33) <= p.cap_chunks * (unsigned long long)kChunk);
            DS_ASSERT(ldcg(&c->s_count[0]) <= (unsigned long long)p.n && ldcg(&c->s_count[1]) <= (unsigned long long)p.n);
        }
#endif
        if (p.trace && blockIdx.x == 0 && threadIdx.x == 0 && st < p.trace_cap) {
            p.trace[2 * st] = globaltimer_ns();
            p.trace[2 * st + 1] = (kind << 56) | (work & ((1ull << 56) - 1));
        }
        ++st;
        ++nbar;
        return ok;
    };
    auto prev = [&]() -> StepSlot* { return &c->slot[(st + 2) % 3]; };
    // hand a giant push to the host-launched standalone kernel and stop
    auto handoff = [&](int next_pos, unsigned long long req, unsigned long long E,
                       unsigned long long Rc) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            c->rs_pos = (unsigned long long)next_pos;
            c->rs_req = req;
            c->rs_E = E;
            c->rs_Rc = Rc;
            c->rs_st = st;
            c->rs_nbar = nbar;
            c->rs_escanned = escanned + E;
            c->rs_npull = npull;
            c->rs_idx = idx;
            c->rs_phases = phases;
            c->rs_visited = visited;
            c->rs_re = re;
            c->rs_scount = scount;
            c->rs_old_scount = old_scount;
            c->rs_pp = (unsigned long long)pp;
            c->rs_bpar = bpar;
            c->rs_hset = hset;
            StepSlot* x = &c->xslot;
            x->re_packed = x->front_count = x->append_count = 0;
            x->flags = 0;
            x->hopmax = 0;
            x->next_min = ~0ull;
        }
    };
    const unsigned long long pullL =
        p.pull_enabled ? (unsigned long long)(p.pull_light * (float)p.Lpull.nnz) : ~0ull;
    const unsigned long long pullH =
        p.pull_enabled ? (unsigned long long)(p.pull_heavy * (float)p.Hpull.nnz) : ~0ull;
    unsigned long long nf = 0;

    // lex mode (fixed point, non-SMALL kernel, p.lex): idx counts internal
    // buckets, ksub per reference bucket; the reference's counters are
    // accumulated per reference bucket in sm.lx by thread 0
    constexpr bool kLex = LEX && std::is_same<M, ModeFixed>::value && !SMALL;
    static_assert(!LEX || kLex, "lex mode: fixed point, non-SMALL kernel only");
    if (kLex && threadIdx.x == 0) {
        sm.wpar = 0u;
        sm.bwork = 0ull;
        sm.lx.cur_ref = -1;
        sm.lx.phases = sm.lx.visited = 0;
        sm.lx.hop_acc = 0;
        sm.lx.any = sm.lx.over = 0;
    }
    // close the reference bucket (thread 0): it ran 1 + max h phases
    auto ref_flush = [&]() {
        if (sm.lx.any) {
            sm.lx.phases += 1ull + sm.lx.hop_acc;
            ++sm.lx.visited;
            if ((long long)sm.lx.phases > p.ceiling) sm.lx.over = 1;
        }
        sm.lx.any = 0;
        sm.lx.hop_acc = 0;
    };

    // thresholds of the reference buckets the window [idx0, idx0 + G) spans
    // (kept in shared memory for the window's pushes and its hop pass); false:
    // the rounding corner of the narrow schedule's check, in one of them
    auto wide_setup = [&](long long idx0, unsigned G) -> bool {
        const long long r0 = idx0 >> p.ksub_log2;
        const int wn = (int)(((idx0 + (long long)G - 1) >> p.ksub_log2) - r0 + 1);
        DS_ASSERT(wn >= 1 && wn <= kWideRef);
        __syncthreads();
        if (threadIdx.x == 0) {
            sm.wn = wn;
            sm.wfail = 0;
        }
        __syncthreads();
        if ((int)threadIdx.x < wn) {
            D a, b;
            M::window((double)(r0 + threadIdx.x) * p.delta, (double)(r0 + threadIdx.x + 1) * p.delta, p.frac, a,
                      b);
            sm.wthr[threadIdx.x] = (unsigned)a;
            if ((int)threadIdx.x == wn - 1) sm.wthr[wn] = (unsigned)b;
            if ((unsigned long long)b - a > (unsigned long long)p.WD + 1ull) sm.wfail = 1;
        }
        __syncthreads();
        return sm.wfail == 0;
    };

    for (;;) {
        D L, H, HD;
        double lo, hi;  // the reference bucket's bounds (f64)
        lex_window<M>(p, kLex, idx, lo, hi, L, H, HD);
        const bool wide = kLex && wideG != 0;
        if (kLex && wide) {
            // window = internal buckets [idx, idx + wideG)
            D L2, HD2;
            double lo2, hi2;
            lex_window<M>(p, true, idx + (long long)wideG - 1, lo2, hi2, L2, H, HD2);
            if (pos == POS_BUCKET && !wide_setup(idx, wideG)) {
                status = kDevLexFail;
                break;
            }
        } else if (kLex) {
            D LD, HD2;
            M::window(lo, hi, p.frac, LD, HD2);
            if ((unsigned long long)HD - LD > (unsigned long long)p.WD + 1ull) {
                // a reference-heavy edge could land inside its own bucket (a
                // rounding corner of fl(i*delta)): rerun with the reference schedule
                status = kDevLexFail;
                break;
            }
            const long long ridx = idx >> p.ksub_log2;
            __syncthreads();
            if (threadIdx.x == 0 && ridx != sm.lx.cur_ref) {
                ref_flush();
                sm.lx.cur_ref = ridx;
            }
            __syncthreads();
            if (sm.lx.over) {
                status = 2;  // DS_ENOCONVERGE: the reference's phase count
                break;
            }
        }

        if (pos == POS_BUCKET) {
            // ---- bucket extraction: t_Bi = {v : lo <= t[v] < hi}; S starts empty
            if (blockIdx.x == 0 && threadIdx.x == 0) c->s_count[bpar ^ 1] = 0;
            capture_range<M, kSum>(p, sm, &c->slot[st % 3], L, H, p.S[bpar], &c->s_count[bpar],
                             (unsigned long long)n_scan, p.S[bpar ^ 1], old_scount, wide ? p.Ainfo : p.Linfo);
            old_scount = 0;
            if (kLex && threadIdx.x == 0) sm.bwork = 0ull;
            if (!end_step(0, (unsigned long long)n_scan)) return;
            const unsigned long long fc = ldcg(&prev()->front_count);
            re = ldcg(&prev()->re_packed);
            if (fc == 0) {
                const unsigned long long nm = ldcg(&prev()->next_min);
                if (nm == ~0ull) break;  // nothing stored beyond: done
                if (kLex && nm >= kLexSat) {  // only out-of-range sums remain: not representable
                    status = kDevLexFail;
                    break;
                }
                if (kLex) {
                    // next internal bucket: the reference bucket of the value,
                    // then the sub-window holding it
                    const int kl = p.ksub_log2;
                    const D dn = (D)nm >> kHopBits;
                    const long long rn = bucket_index_of(M::to_f64(dn, p.frac), p.delta);
                    D a, b;
                    M::window((double)rn * p.delta, (double)(rn + 1) * p.delta, p.frac, a, b);
                    const unsigned long long w = (unsigned long long)b - a;
                    long long t = (1ll << kl) - 1;
                    while (t > 0 && (unsigned long long)dn < a + (((unsigned long long)t * w) >> kl)) --t;
                    idx = (rn << kl) + t;
                } else {
                    idx = bucket_index_of(M::to_f64((D)nm, p.frac), p.delta);
                }
                continue;
            }
            ++visited;
            if (kLex && !wide && threadIdx.x == 0) sm.lx.any = 1;
            pos = POS_PHASE;
        }

        if (pos == POS_PHASE) {
            // ---- one light phase (sssp.py:292-301)
            ++phases;
            if ((long long)phases > ((kLex) ? (p.ceiling > LLONG_MAX / 64 ? LLONG_MAX : p.ceiling * 64)
                                                         : p.ceiling)) {
                status = 2;  // DS_ENOCONVERGE
                break;
            }
            nf = 0;
            const unsigned long long E = re & kMask33;
            if (E >= p.big_light) {
                handoff(POS_AFTER_LIGHT, 1, E, re >> kPackShift);
                return;
            }
            if (SMALL && E <= p.local_edges && (re >> kPackShift) <= p.local_entries) {
                // ---- block-local mode (high-diameter graphs: tiny frontiers):
                // CTA 0 runs light phases back to back with block barriers while
                // the frontier stays small; the other CTAs wait at the next
                // grid barrier.  Same steps, same snapshot semantics.
                if (blockIdx.x == 0) {
                    unsigned long long lre = re, lph = phases, lesc = 0;
                    int lpp = pp, done = 0, lst = 0, k = 0;
                    for (;;) {
                        StepSlot* a = &c->lslot[k];
                        if (threadIdx.x == 0) {
                            a->re_packed = a->front_count = a->append_count = 0;
                            a->flags = 0;
                            a->hopmax = 0;
                        }
                        __syncthreads();
                        const unsigned long long lE = lre & kMask33;
                        lesc += lE;
                        if (lE)
                            relax_step<M, true, true, kSum, false, false, kSEntry>(
                                p, sm, a, lE, lre >> kPackShift, p.Ledges, H, p.F[lpp], p.fbits[lph & 1], (D)0,
                                bpar);
                        __syncthreads();
                        if (ldcg(&a->flags) & 1u) {
                            lst = kDevOverflow;
                            break;
                        }
                        const unsigned long long lnf = ldcg(&a->append_count);
                        if (lnf == 0) {
                            done = 1;
                            break;
                        }
                        k ^= 1;
                        StepSlot* b = &c->lslot[k];
                        if (threadIdx.x == 0) {
                            b->re_packed = b->front_count = b->append_count = 0;
                            b->flags = 0;
                            b->hopmax = 0;
                        }
                        __syncthreads();
                        capture_list<M, true, false, true>(p, sm, b, p.F[lpp], nullptr, lnf, p.Linfo,
                                                           p.fbits[lph & 1], p.S[bpar],
                                                           &c->s_count[bpar]);
                        __syncthreads();
                        lre = ldcg(&b->re_packed);
                        lpp ^= 1;
                        if ((lre & kMask33) > p.local_edges || (lre >> kPackShift) > p.local_entries)
                            break;  // grown: the next phase runs on the whole grid
                        ++lph;
                        if ((long long)lph > p.ceiling) {
                            lst = 2;
                            break;
                        }
                    }
                    if (threadIdx.x == 0) {
                        c->h_phases = lph;
                        c->h_re = lre;
                        c->h_pp = (unsigned long long)lpp;
                        c->h_done = (unsigned long long)done;
                        c->h_status = (unsigned long long)lst;
                    }
                    escanned += lesc;
                }
                if (!end_step(9, E)) return;
                phases = ldcg(&c->h_phases);
                re = ldcg(&c->h_re);
                pp = (int)ldcg(&c->h_pp);
                status = (int)ldcg(&c->h_status);
                if (status) break;
                if (ldcg(&c->h_done)) {
                    pos = POS_HEAVY;
                } else {
                    pos = POS_PHASE;
                    continue;
                }
            } else {
            if (DS_PULL_LIGHT && E > pullL) {
                escanned += (unsigned long long)p.Lpull.nnz;
                ++npull;
                const unsigned sl = (unsigned)(st % 3);
                pull_step<M, true>(p, sm, &c->slot[sl], p.Lpull, p.Ledges, L, H, p.F[pp], p.Fv[pp]);
                if (!end_step(5, (unsigned long long)p.Lpull.nnz)) return;
                const bool ovf = ldcg(&prev()->flags) & 1u;
                commit_step<M, true>(p, sm, &c->slot[sl], p.Lpull, H, p.F[pp], p.Fv[pp]);
                if (!end_step(6, (unsigned long long)p.Lpull.nspan)) return;
                if (ovf) {
                    status = kDevOverflow;
                    break;
                }
                nf = ldcg(&c->slot[sl].append_count);
                // values travel with the list; commit them in the next capture
                capture_list<M, true, true>(p, sm, &c->slot[st % 3], p.F[pp], p.Fv[pp], nf, p.Linfo,
                                            p.fbits[phases & 1], p.S[bpar], &c->s_count[bpar]);
                if (nf == 0) {
                    pos = POS_HEAVY;
                    continue;
                }
                if (!end_step(2, nf)) return;
                re = ldcg(&prev()->re_packed);
                pp ^= 1;
                continue;
            } else if (E > 0) {
                escanned += E;
                if (kLex && threadIdx.x == 0) sm.bwork += E;
                if constexpr (kLex) {
                    if (wide)
                        relax_step<M, true, false, false, false, true, kSEntry, true>(
                            p, sm, &c->slot[st % 3], E, re >> kPackShift, p.Aedges, H, p.F[pp],
                            p.fbits[phases & 1], HD, bpar);
                    else
                        relax_step<M, true, false, kSum, false, kLex, kSEntry>(p, sm, &c->slot[st % 3], E,
                                                                              re >> kPackShift, p.Ledges, H,
                                                                              p.F[pp], p.fbits[phases & 1], HD,
                                                                              bpar);
                } else {
                    relax_step<M, true, false, kSum, false, kLex, kSEntry>(p, sm, &c->slot[st % 3], E,
                                                                          re >> kPackShift, p.Ledges, H, p.F[pp],
                                                                          p.fbits[phases & 1], HD, bpar);
                }
                if (!end_step(1, E)) return;
                if (const unsigned fl = ldcg(&prev()->flags) & 3u) {
                    status = (fl & 2u) ? kDevLexFail : kDevOverflow;
                    break;
                }
                nf = ldcg(&prev()->append_count);
            }
            pos = POS_AFTER_LIGHT;
            }
        } else if (pos == POS_AFTER_LIGHT && resumed) {
            // results of the standalone light push
            resumed = false;
            if (ldcg(&c->xslot.flags) & 1u) {
                status = kDevOverflow;
                break;
            }
            nf = ldcg(&c->xslot.append_count);
        }

        if (pos == POS_AFTER_LIGHT) {
            if (nf == 0) {
                pos = POS_HEAVY;
            } else {
                capture_list<M, true, false>(p, sm, &c->slot[st % 3], p.F[pp], nullptr, nf,
                                             wide ? p.Ainfo : p.Linfo, p.fbits[phases & 1], p.S[bpar],
                                             &c->s_count[bpar],
                                             nf >= kBulkClearMin ? (unsigned long long)(n_scan + 31) / 32 : 0ull);
                if (!end_step(2, nf)) return;
                re = ldcg(&prev()->re_packed);
                pp ^= 1;
                pos = POS_PHASE;
                continue;
            }
        }

        if (pos == POS_HEAVY) {
            // ---- heavy relaxation from S with current t (sssp.py:218-227)
            scount = ldcg(&c->s_count[bpar]);
            bool heavy_done = false;
            if (kLex && wide) {
                // ---- end of a wide window: no heavy step (the closure pushed
                // every edge); hop maxima per reference bucket from S
                wide_hop_pass<M>(p, sm, p.S[bpar], scount, c->whm[sm.wpar]);
                if (!end_step(13, scount)) return;
                // the window's hop maxima: loaded by the CTA, accounted by thread 0
                for (int j = threadIdx.x; j < sm.wn; j += kThreads) sm.whm[j] = ldcg(&c->whm[sm.wpar][j]);
                __syncthreads();
                if (threadIdx.x == 0) {
                    const long long r0 = idx >> p.ksub_log2;
                    int sat = 0;
                    for (int j = 0; j < sm.wn; ++j) {
                        const unsigned v = sm.whm[j];
                        if (!v) continue;  // no final value in this reference bucket
                        if (v - 1u >= kHopMask) sat = 1;  // a final hop count saturated
                        if (r0 + j != sm.lx.cur_ref) {
                            ref_flush();
                            sm.lx.cur_ref = r0 + j;
                        }
                        sm.lx.any = 1;
                        sm.lx.hop_acc = max(sm.lx.hop_acc, v - 1u);
                    }
                    sm.wfail = sat;
                    if (blockIdx.x == 0) {
                        // the other set was last read two barriers ago
                        for (int j = 0; j < kWideRef; ++j) c->whm[sm.wpar ^ 1u][j] = 0u;
                        ++c->wide_windows;
                        c->wide_edges += sm.bwork;
                    }
                    sm.wpar ^= 1u;
                }
                __syncthreads();
                if (sm.wfail) {
                    status = kDevLexFail;
                    break;
                }
                if (sm.lx.over) {
                    status = 2;  // DS_ENOCONVERGE: the reference's phase count
                    break;
                }
                old_scount = scount;
                bpar ^= 1;
                idx += (long long)wideG;
                pos = POS_BUCKET;
                // next window: double while the windows stay latency-bound,
                // halve (and finally return to the narrow schedule) when one
                // pushed a throughput-sized amount of edges
                {
                    const unsigned long long bw = sm.bwork;  // reset only after the next window's barriers
                    if (bw < p.wide_lo) wideG = min(wideG * 2u, p.wide_gmax);
                    else if (bw > p.wide_hi) wideG = wideG / 2u;
                }
                continue;
            }
            if (SMALL && scount <= p.local_entries) {
                // block-local heavy step: CTA 0 captures S and, if small, relaxes it
                if (blockIdx.x == 0) {
                    StepSlot* a = &c->lslot[0];
                    if (threadIdx.x == 0) {
                        a->re_packed = a->front_count = a->append_count = 0;
                        a->flags = 0;
                        a->hopmax = 0;
                    }
                    __syncthreads();
                    capture_list<M, false, false, true, true>(p, sm, a, p.S[bpar], nullptr, scount, p.Hinfo,
                                                              nullptr, nullptr, nullptr);
                    __syncthreads();
                    const unsigned long long lre = ldcg(&a->re_packed);
                    int done = 0;
                    if ((lre & kMask33) <= p.local_edges) {
                        escanned += lre & kMask33;
                        if (lre & kMask33)
                            relax_step<M, false, true, kSum>(p, sm, a, lre & kMask33, lre >> kPackShift,
                                                       p.Hedges, H, nullptr, nullptr);
                        __syncthreads();
                        done = 1;
                    }
                    if (threadIdx.x == 0) {
                        c->hh_re = lre;
                        c->hh_done = (unsigned long long)done;
                        c->hh_status = (ldcg(&a->flags) & 1u) ? (unsigned long long)kDevOverflow : 0ull;
                    }
                }
                if (!end_step(10, scount)) return;
                re = ldcg(&c->hh_re);
                status = (int)ldcg(&c->hh_status);
                if (status) break;
                heavy_done = ldcg(&c->hh_done) != 0;
            } else {
                capture_list<M, false, false, false, true>(p, sm, &c->slot[st % 3], p.S[bpar], nullptr, scount,
                                                           p.Hinfo, nullptr, nullptr, nullptr);
                if (!end_step(3, scount)) return;
                re = ldcg(&prev()->re_packed);
                if (kLex) {
                    const unsigned hm = ldcg(&prev()->hopmax);
                    if (hm >= kHopMask) {  // a final hop count saturated: not representable
                        status = kDevLexFail;
                        break;
                    }
                    if (threadIdx.x == 0) sm.lx.hop_acc = max(sm.lx.hop_acc, hm);
                }
            }
            const unsigned long long E = heavy_done ? 0ull : (re & kMask33);
            hset += re & kMask33;  // S's rows are settled: their heavy edges leave the pull volume
            if (kLex && threadIdx.x == 0) sm.bwork += E;
            // ---- direction choice.  The push streams E = |A_H rows of S|; the
            // pull streams only the rows that can still change (t >= H), whose
            // heavy edges are U = nnz(A_H) - (heavy edges of every settled row).
            // Exactness of the pull (same t afterwards as the push):
            //  * heavy_beyond: every t_u + w (t_u >= L, w heavy) is >= H, so
            //    the step changes no value below H -- S's values are fixed
            //    during it (the push reads them captured; the pull live) and
            //    rows below H cannot receive anything;
            //  * gating on t_u < H selects S plus rows settled in earlier
            //    buckets, whose t_u + w were applied then (no-ops now);
            //  * rows >= H are the only possible targets; min is order-free.
            if (!heavy_done && E > 0 && p.hpull && E >= p.hpull_min) {
                const unsigned long long U = p.nH > hset ? p.nH - hset : 0ull;
                D Lw = L, Hw = H;  // the internal window in distance units
                if (kLex) {
                    Lw = L >> kHopBits;
                    Hw = H == M::INF ? (D)kLexDLimit : (D)(H >> kHopBits);
                }
                bool gather = (double)E > (double)p.hpull_ratio * (double)U &&
                              M::heavy_beyond(Lw, Hw, lo, hi, p.min_heavy);
                if constexpr (kLex && kSEntry && DS_BIDIR_BUILD) {
                    // the tail starts here: enter the wide window through the
                    // bidirectional step (heavy gather + scan + first round in one pass)
                    if (gather && p.Aedges && p.bidir && !p.wide_force && U <= p.wide_unsettled) {
                        __syncthreads();  // thread 0's sm.bwork
                        if (sm.bwork < p.wide_enter) {
                            const unsigned G = U <= p.wide_all ? p.wide_gmax : p.wide_g0;
                            if (!wide_setup(idx + 1, G)) {
                                status = kDevLexFail;
                                break;
                            }
                            D L2, HW, HD2;
                            double lo2, hi2;
                            lex_window<M>(p, true, idx + (long long)G, lo2, hi2, L2, HW, HD2);
                            capture_unsettled<M>(p, sm, &c->slot[st % 3], H, (unsigned long long)n_scan, p.Ainfo, HW,
                                                 p.S[bpar ^ 1], &c->s_count[bpar ^ 1]);
                            if (!end_step(11, (unsigned long long)n_scan)) return;
                            const unsigned long long pre = ldcg(&prev()->re_packed);
                            const unsigned long long Ep = pre & kMask33;
                            ++npull;
                            ++phases;  // the window's first round (dedup bitmap parity)
                            nf = 0;
                            if (Ep > 0) {
                                escanned += Ep;
                                bidir_step<M>(p, sm, &c->slot[st % 3], Ep, pre >> kPackShift, H, HW, HD, p.F[pp],
                                              p.fbits[phases & 1], bpar ^ 1);
                                if (!end_step(14, Ep)) return;
                                nf = ldcg(&prev()->append_count);
                            }
                            if (threadIdx.x == 0) sm.bwork = Ep;
                            // no scan opened this window: the S counter the NEXT window will
                            // use (this bucket's, read by every CTA barriers ago) is reset here
                            if (blockIdx.x == 0 && threadIdx.x == 0) c->s_count[bpar] = 0;
                            old_scount = scount;
                            bpar ^= 1;
                            idx += 1;
                            wideG = G;
                            pos = POS_AFTER_LIGHT;
                            continue;
                        }
                    }
                }
                if (gather) {
                    capture_unsettled<M>(p, sm, &c->slot[st % 3], H, (unsigned long long)n_scan, p.Hinfo);
                    if (!end_step(11, (unsigned long long)n_scan)) return;
                    const unsigned long long pre = ldcg(&prev()->re_packed);
                    const unsigned long long Ep = pre & kMask33;
                    ++npull;
                    if (Ep > 0) {
                        escanned += Ep;
                        relax_step<M, false, false, kSum, true, kLex>(p, sm, &c->slot[st % 3], Ep, pre >> kPackShift,
                                                                p.Hedges, H, nullptr, nullptr, HD);
                        if (!end_step(12, Ep)) return;
                        if (const unsigned fl = ldcg(&prev()->flags) & 3u) {
                            status = (fl & 2u) ? kDevLexFail : kDevOverflow;
                            break;
                        }
                    }
                    heavy_done = true;
                }
            }
            if (heavy_done) {
            } else if (E >= p.big_heavy) {
                handoff(POS_AFTER_HEAVY, p.heavy_pull ? 3 : 2, E, re >> kPackShift);
                return;
            } else if (DS_PULL_HEAVY && E > pullH) {
                escanned += (unsigned long long)p.Hpull.nnz;
                ++npull;
                const unsigned sl = (unsigned)(st % 3);
                pull_step<M, false>(p, sm, &c->slot[sl], p.Hpull, p.Hedges, L, H, nullptr, nullptr);
                if (!end_step(7, (unsigned long long)p.Hpull.nnz)) return;
                const bool ovf = ldcg(&prev()->flags) & 1u;
                commit_step<M, false>(p, sm, &c->slot[sl], p.Hpull, H, nullptr, nullptr);
                if (!end_step(8, (unsigned long long)p.Hpull.nspan)) return;
                if (ovf) {
                    status = kDevOverflow;
                    break;
                }
            } else if (E > 0) {
                escanned += E;
                relax_step<M, false, false, kSum, false, kLex>(p, sm, &c->slot[st % 3], E, re >> kPackShift,
                                                              p.Hedges, H, nullptr, nullptr, HD);
                if (!end_step(4, E)) return;
                if (const unsigned fl = ldcg(&prev()->flags) & 3u) {
                    status = (fl & 2u) ? kDevLexFail : kDevOverflow;
                    break;
                }
            }
            pos = POS_AFTER_HEAVY;
        } else if (pos == POS_AFTER_HEAVY && resumed) {
            resumed = false;
            if (ldcg(&c->xslot.flags) & 1u) {
                status = kDevOverflow;
                break;
            }
        }

        if (pos == POS_AFTER_HEAVY) {
            old_scount = scount;
            bpar ^= 1;
            ++idx;
            pos = POS_BUCKET;
            // small bucket and most of the graph settled (by heavy edges): the
            // rest is a latency-bound tail -- wide windows from here
            // (sm.bwork: thread 0's last add precedes the heavy step's barrier)
            if (kLex && p.Aedges) {
                const unsigned long long U = p.nH - min(hset, p.nH);  // heavy edges of the unsettled rows
                if (p.wide_force) wideG = p.wide_g0;
                else if (sm.bwork < p.wide_enter && U <= p.wide_unsettled)
                    wideG = U <= p.wide_all ? p.wide_gmax : p.wide_g0;
            }
        }
    }

    if (kLex) {
        __syncthreads();
        if (threadIdx.x == 0 && !status) ref_flush();
        __syncthreads();
        if (!status && sm.lx.over) status = 2;  // DS_ENOCONVERGE: the reference's count
        phases = sm.lx.phases;
        visited = sm.lx.visited;
    }
    if (status) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            c->status = status;
            c->phases = phases;
            c->steps = st;
            c->rs_req = 0;
        }
        return;
    }

    // ---- finalize: fp64 output, n_r, m_r, max distance (SsspResult, sssp.py:312-313)
    {
        // retire the last bucket's S bits
        const unsigned long long gt = (unsigned long long)blockIdx.x * kThreads + threadIdx.x;
        for (unsigned long long i = gt; !kSEntry && i < old_scount; i += (unsigned long long)gridDim.x * kThreads) {
            const unsigned v = (unsigned)ldcg(p.S[bpar ^ 1] + i);
            atomicAnd(p.sbits + (v >> 5), ~(1u << (v & 31)));
        }
        // 8 vertices per thread and round: independent loads in flight (a
        // one-per-thread loop is a chain of dependent round trips)
        unsigned long long cnt = 0, m = 0, mx = 0;
        const long long tid = (long long)blockIdx.x * kThreads + threadIdx.x;
        const long long stride8 = 8ll * gridDim.x * kThreads;
        // a warp converts 256 consecutive vertices per round, lane-interleaved
        // pairs: every perm load of the warp covers 256 contiguous bytes and
        // every output store 512 (full write combining, also when p.out is
        // mapped host memory: zero-copy batch results)
        {
            const int lane = threadIdx.x & 31;
            const long long wg = (long long)blockIdx.x * kWarps + (threadIdx.x >> 5);
            // a batch row of a caller's array is 16-byte aligned only for even n
            const bool out_al = (reinterpret_cast<unsigned long long>(p.out) & 15ull) == 0;
            for (long long base = wg * 256; base < p.n; base += (long long)gridDim.x * kWarps * 256) {
                int sv[8];
                const bool full = base + 256 <= p.n;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const long long v = base + i * 64 + lane * 2;
                    if (full) {
                        const int2 a = __ldg(reinterpret_cast<const int2*>(p.perm + v));
                        sv[2 * i] = a.x;
                        sv[2 * i + 1] = a.y;
                    } else {
                        sv[2 * i] = v < p.n ? __ldg(p.perm + v) : (int)n_scan;
                        sv[2 * i + 1] = v + 1 < p.n ? __ldg(p.perm + v + 1) : (int)n_scan;
                    }
                }
                D d[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    d[j] = sv[j] < n_scan ? __ldcg(p.dist + sv[j]) : M::INF;
                    if (kLex && d[j] == (D)kLexSat) atomicOr(&c->lexsat, 1u);
                    if (kLex && d[j] != M::INF) d[j] >>= kHopBits;  // key -> distance
                }
                double o[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (d[j] != M::INF) {
                        ++cnt;
                        if ((unsigned long long)d[j] > mx) mx = (unsigned long long)d[j];
                    }
                    o[j] = M::to_f64(d[j], p.frac);
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const long long v = base + i * 64 + lane * 2;
                    if (full && out_al) {
                        *reinterpret_cast<double2*>(p.out + v) = make_double2(o[2 * i], o[2 * i + 1]);
                    } else {
                        if (v < p.n) p.out[v] = o[2 * i];
                        if (v + 1 < p.n) p.out[v + 1] = o[2 * i + 1];
                    }
                }
            }
        }
        // m_r = sum of out-degrees of the reached vertices, in solver order
        for (long long s0 = 8 * tid; s0 < n_scan; s0 += stride8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (s0 + j < n_scan && __ldcg(p.dist + s0 + j) != M::INF) m += __ldg(p.sdeg + s0 + j);
            }
        }
        cnt = block_reduce<0>(cnt, sm.red);
        m = block_reduce<0>(m, sm.red2);
        mx = block_reduce<2>(mx, sm.red);
        if (threadIdx.x == 0) {
            atomicAdd(&c->reached, cnt);
            atomicAdd(&c->edges_reached, m);
            atomicMax(&c->max_d, mx);
            if (p.trace) atomicMax(&c->t_exit, globaltimer_ns());
            if (blockIdx.x == 0) {
                c->phases = phases;
                c->visited = visited;
                c->edges_scanned = escanned;
                c->barriers = nbar;
                c->steps = st;
                c->pulls = npull;
                c->rs_req = 0;
                if (!p.trace) c->last_bucket = idx;
                c->status = 0;
            }
        }
    }
}

// A giant push handed off by the persistent kernel, as its own launch (its
// own register allocation, no spills): the solver state says which list,
// window and CSR; results land in Ctl::xslot.
template <class M, bool LIGHT>
__global__ void __launch_bounds__(kBigThreads, DS_BIG_MINB) k_big_relax(const KParams<M> p) {
    using D = typename M::D;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem<D>& sm = *reinterpret_cast<Smem<D>*>(smem_raw);
    Ctl* const c = p.ctl;
    const long long idx = ldcg(&c->rs_idx);
    const double lo = (double)idx * p.delta;
    const double hi = (double)(idx + 1) * p.delta;
    D L, H;
    M::window(lo, hi, p.frac, L, H);
    const unsigned long long E = ldcg(&c->rs_E), Rc = ldcg(&c->rs_Rc);
    const int pp = (int)ldcg(&c->rs_pp);
    const unsigned long long phases = ldcg(&c->rs_phases);
    if (LIGHT)
        relax_step<M, true, false, false, false, false, kSEntry>(p, sm, &c->xslot, E, Rc, p.Ledges, H, p.F[pp],
                                                                 p.fbits[phases & 1], (typename M::D)0,
                                                                 (unsigned)ldcg(&c->rs_bpar));
    else
        relax_step<M, false>(p, sm, &c->xslot, E, Rc, p.Hedges, H, nullptr, nullptr);
    (void)L;
}

// The handed-off heavy step as the reference's own gathered form
// (vxm_min_plus over A_H^T = A_H, gated by S membership; fused.py:105-124):
// every row of A_H is streamed once (coalesced, evict-first) and the random
// accesses are S-bit and S-value reads of hub ids, which stay in L1 -- versus
// one random target check per pushed edge.  Rows crossing a chunk boundary
// finish in k_big_commit.  Results land in Ctl::xslot like k_big_relax's.
template <class M>
__global__ void __launch_bounds__(kBigThreads, DS_BIG_MINB) k_big_pull(const KParams<M> p) {
    using D = typename M::D;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem<D>& sm = *reinterpret_cast<Smem<D>*>(smem_raw);
    Ctl* const c = p.ctl;
    const long long idx = ldcg(&c->rs_idx);
    D L, H;
    M::window((double)idx * p.delta, (double)(idx + 1) * p.delta, p.frac, L, H);
    pull_step<M, false>(p, sm, &c->xslot, p.Hpull, p.Hedges, L, H, nullptr, nullptr);
}

template <class M>
__global__ void __launch_bounds__(kBigThreads, DS_BIG_MINB) k_big_commit(const KParams<M> p) {
    using D = typename M::D;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem<D>& sm = *reinterpret_cast<Smem<D>*>(smem_raw);
    Ctl* const c = p.ctl;
    const long long idx = ldcg(&c->rs_idx);
    D L, H;
    M::window((double)idx * p.delta, (double)(idx + 1) * p.delta, p.frac, L, H);
    commit_step<M, false>(p, sm, &c->xslot, p.Hpull, H, nullptr, nullptr);
    (void)L;
}

}  // namespace ds
