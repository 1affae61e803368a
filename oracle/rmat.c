/*
 * rmat.c -- TEST / BENCH INFRASTRUCTURE ONLY.  Host R-MAT generator for the
 * reference arm and CPU baseline of bench.py, so that the CPU leg synthesises
 * its input without the product's CUDA library.  A restatement in C (OpenMP)
 * of paper_1911_06895_b200/graphs.py:rmat -- the BASELINE.json R-MAT spec
 * (a,b,c,d = .57,.19,.19,.05; self-loops dropped; symmetrised; duplicates
 * collapsed; fp32-lattice weight k * 2^-24 per undirected pair) -- and pinned
 * bit for bit against it by tests/test_oracle.py (the numpy version takes
 * ~15 min at scale 24; this one seconds).
 *
 * Pipeline: counter-based edge draws (splitmix64 per level), vertex scramble,
 * both directions as packed (row << scale | col) keys, a parallel LSD radix
 * sort, dedup + CSR, weights hashed from the undirected pair.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define GOLDEN 0x9E3779B97F4A7C15ull
/* int(p * 2^32) for p = .57 / .19 / .19, as graphs.py computes them */
#define RMAT_A 2448131358ll
#define RMAT_B 816043786ll
#define RMAT_C 816043786ll

static inline uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + GOLDEN;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* graphs.py:_scramble -- bijection on [0, 2^scale) */
static inline uint64_t scramble(uint64_t x, int scale, uint64_t seed) {
    const uint64_t mask = (scale >= 64) ? ~0ull : ((1ull << scale) - 1);
    const int half = (scale + 1) / 2 > 1 ? (scale + 1) / 2 : 1;
    x = (x * (GOLDEN | 1ull)) & mask;
    x ^= x >> half;
    x = (x * 0xD6E8FEB86659FD93ull) & mask;
    x ^= x >> half;
    x = (x + seed * 0x632BE59BD9B4E019ull) & mask;
    return x;
}

/* graphs.py:lattice_weight -- k = top 24 bits of the pair hash, 0 -> 1 */
static inline float lattice_weight(uint64_t a, uint64_t b, uint64_t wseed) {
    const uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
    const uint64_t h = splitmix64(((lo << 32) | hi) ^ (wseed * 0xD1B54A32D192ED03ull));
    int64_t k = (int64_t)(h >> 40);
    if (k == 0) k = 1;
    return (float)((double)k * 0x1p-24);
}

typedef struct {
    int64_t n, nnz;
    int64_t *indptr;
    int32_t *col;
    float *val;
} oracle_rmat_t;

/* parallel LSD radix sort of 64-bit keys on their low `bits` bits */
static int radix_sort(uint64_t *a, int64_t m, int bits) {
    uint64_t *b = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(m > 0 ? m : 1));
    if (!b) return 1;
    const int R = 16, NB = 1 << 16;
    int T = 1;
#ifdef _OPENMP
    T = omp_get_max_threads();
#endif
    int64_t *hist = (int64_t *)calloc((size_t)T * NB, sizeof(int64_t));
    if (!hist) {
        free(b);
        return 1;
    }
    uint64_t *src = a, *dst = b;
    for (int shift = 0; shift < bits; shift += R) {
        memset(hist, 0, sizeof(int64_t) * (size_t)T * NB);
#pragma omp parallel num_threads(T)
        {
            int t = 0;
#ifdef _OPENMP
            t = omp_get_thread_num();
#endif
            const int64_t lo = m * t / T, hi = m * (t + 1) / T;
            int64_t *h = hist + (size_t)t * NB;
            for (int64_t i = lo; i < hi; ++i) ++h[(src[i] >> shift) & (NB - 1)];
#pragma omp barrier
#pragma omp single
            {
                int64_t run = 0;
                for (int d = 0; d < NB; ++d)
                    for (int u = 0; u < T; ++u) {
                        const int64_t c = hist[(size_t)u * NB + d];
                        hist[(size_t)u * NB + d] = run;
                        run += c;
                    }
            }
            for (int64_t i = lo; i < hi; ++i) dst[h[(src[i] >> shift) & (NB - 1)]++] = src[i];
        }
        uint64_t *tmp = src;
        src = dst;
        dst = tmp;
    }
    if (src != a) memcpy(a, src, sizeof(uint64_t) * (size_t)m);
    free(hist);
    free(b);
    return 0;
}

oracle_rmat_t *oracle_rmat_build(int scale, int edge_factor, uint64_t seed, uint64_t wseed, int threads) {
    if (scale < 1 || scale > 31 || edge_factor < 1) return NULL;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
    const int64_t n = (int64_t)1 << scale;
    const int64_t m = (int64_t)edge_factor << scale;
    uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(2 * m));
    if (!keys) return NULL;
    const uint64_t seed_mix = seed * GOLDEN;
    const uint64_t loop_key = ((uint64_t)(n - 1) << scale) | (uint64_t)(n - 1);  /* a self-loop: dropped */
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < m; ++k) {
        uint64_t s = 0, d = 0;
        for (int level = 0; level < scale; ++level) {
            const uint64_t h = splitmix64(((uint64_t)k * 64ull + (uint64_t)level) ^ seed_mix);
            const int64_t r = (int64_t)(h >> 32);
            const uint64_t bit = 1ull << (scale - 1 - level);
            if (r >= RMAT_A + RMAT_B) s |= bit;
            if ((r >= RMAT_A && r < RMAT_A + RMAT_B) || r >= RMAT_A + RMAT_B + RMAT_C) d |= bit;
        }
        s = scramble(s, scale, seed);
        d = scramble(d, scale, seed);
        if (s == d) {
            keys[2 * k] = keys[2 * k + 1] = loop_key;
        } else {
            keys[2 * k] = (s << scale) | d;
            keys[2 * k + 1] = (d << scale) | s;
        }
    }
    if (radix_sort(keys, 2 * m, 2 * scale)) {
        free(keys);
        return NULL;
    }
    /* dedup in place (sequential pass: memory bound) and drop self-loops */
    int64_t w = 0;
    const uint64_t cmask = (uint64_t)n - 1;
    for (int64_t i = 0; i < 2 * m; ++i) {
        const uint64_t x = keys[i];
        if ((x >> scale) == (x & cmask)) continue;
        if (w > 0 && keys[w - 1] == x) continue;
        keys[w++] = x;
    }
    oracle_rmat_t *g = (oracle_rmat_t *)calloc(1, sizeof(oracle_rmat_t));
    if (!g) {
        free(keys);
        return NULL;
    }
    g->n = n;
    g->nnz = w;
    g->indptr = (int64_t *)calloc((size_t)(n + 1), sizeof(int64_t));
    g->col = (int32_t *)malloc(sizeof(int32_t) * (size_t)(w > 0 ? w : 1));
    g->val = (float *)malloc(sizeof(float) * (size_t)(w > 0 ? w : 1));
    if (!g->indptr || !g->col || !g->val) {
        free(g->indptr);
        free(g->col);
        free(g->val);
        free(g);
        free(keys);
        return NULL;
    }
    for (int64_t i = 0; i < w; ++i) ++g->indptr[(keys[i] >> scale) + 1];
    for (int64_t r = 0; r < n; ++r) g->indptr[r + 1] += g->indptr[r];
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < w; ++i) {
        const uint64_t u = keys[i] >> scale, v = keys[i] & cmask;
        g->col[i] = (int32_t)v;
        g->val[i] = lattice_weight(u, v, wseed);
    }
    free(keys);
    return g;
}

int64_t oracle_rmat_nnz(const oracle_rmat_t *g) { return g ? g->nnz : -1; }

void oracle_rmat_fetch(const oracle_rmat_t *g, int64_t *indptr, int32_t *col, float *val) {
    memcpy(indptr, g->indptr, sizeof(int64_t) * (size_t)(g->n + 1));
    memcpy(col, g->col, sizeof(int32_t) * (size_t)g->nnz);
    memcpy(val, g->val, sizeof(float) * (size_t)g->nnz);
}

void oracle_rmat_free(oracle_rmat_t *g) {
    if (!g) return;
    free(g->indptr);
    free(g->col);
    free(g->val);
    free(g);
}
