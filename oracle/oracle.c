/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference's
 * delta-stepping path (arxiv 1911.06895, `deltasparse` package) used as the
 * parity checker for the sm_100a product path.  Only tests/, smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this file's build.
 * The product library (paper_1911_06895_b200/csrc) never links or calls it.
 *
 * Every routine cites the reference file:line it restates
 * (/root/reference/pkg/src/deltasparse/...).  The reference stores sparse
 * vectors with implicit +inf absence; here the same vectors are dense
 * float64 arrays holding +inf for "absent", which is the identical value
 * domain (SparseVector never stores inf, core.py:109-116).
 *
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py -> tests/golden/ fixtures).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_EINVAL 1       /* ValueError in the reference                 */
#define OR_ENOCONVERGE 2  /* RuntimeError: light phase ceiling exceeded   */
#define OR_ENOMEM 3

typedef struct {
    int64_t n;
    int64_t *indptr; /* n+1 */
    int64_t *col;
    double *val;
} csr_t;

static void csr_free(csr_t *m) {
    free(m->indptr);
    free(m->col);
    free(m->val);
    memset(m, 0, sizeof(*m));
}

/* ops.py:63-72 predicates; sssp.py:96-97 (_split_range) */
static inline int is_light(double w, double delta) { return (w > 0) && (w <= delta); }
static inline int is_heavy(double w, double delta) { return w > delta; }

/* filter_matrix (ops.py:158-176): keep entries satisfying the predicate,
 * per-row order preserved.  which = 0 light, 1 heavy. */
static int filter_matrix(int64_t n, const int64_t *indptr, const int64_t *col,
                         const double *val, double delta, int which, csr_t *out) {
    int64_t nnz = indptr[n], kept = 0;
    for (int64_t e = 0; e < nnz; ++e)
        kept += which ? is_heavy(val[e], delta) : is_light(val[e], delta);
    out->n = n;
    out->indptr = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    out->col = (int64_t *)malloc(sizeof(int64_t) * (size_t)(kept ? kept : 1));
    out->val = (double *)malloc(sizeof(double) * (size_t)(kept ? kept : 1));
    if (!out->indptr || !out->col || !out->val) return OR_ENOMEM;
    int64_t k = 0;
    out->indptr[0] = 0;
    for (int64_t r = 0; r < n; ++r) {
        for (int64_t e = indptr[r]; e < indptr[r + 1]; ++e) {
            int keep = which ? is_heavy(val[e], delta) : is_light(val[e], delta);
            if (keep) {
                out->col[k] = col[e];
                out->val[k] = val[e];
                ++k;
            }
        }
        out->indptr[r + 1] = k;
    }
    return OR_OK;
}

/* matrix_transpose_view (core.py:281-301): entries ordered by (col, row) --
 * lexsort((rows, col)).  A stable counting sort by column over row-major
 * input yields exactly that order. */
static int transpose(const csr_t *a, csr_t *t) {
    int64_t n = a->n, nnz = a->indptr[n];
    t->n = n;
    t->indptr = (int64_t *)calloc((size_t)(n + 1), sizeof(int64_t));
    t->col = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nnz ? nnz : 1));
    t->val = (double *)malloc(sizeof(double) * (size_t)(nnz ? nnz : 1));
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
    if (!t->indptr || !t->col || !t->val || !fill) {
        free(fill);
        return OR_ENOMEM;
    }
    for (int64_t e = 0; e < nnz; ++e) t->indptr[a->col[e] + 1]++;
    for (int64_t j = 0; j < n; ++j) t->indptr[j + 1] += t->indptr[j];
    memcpy(fill, t->indptr, sizeof(int64_t) * (size_t)(n + 1));
    for (int64_t r = 0; r < n; ++r)
        for (int64_t e = a->indptr[r]; e < a->indptr[r + 1]; ++e) {
            int64_t p = fill[a->col[e]]++;
            t->col[p] = r;
            t->val[p] = a->val[e];
        }
    free(fill);
    return OR_OK;
}

/* fused_masked_relax (fused.py:127-161) with _relax_range (fused.py:105-124):
 * gated dense operand (fused.py:149-151) then, per output row j of the
 * transposed matrix, min over its entries of gated[i] + w.  +inf results mean
 * "no request" (fused.py:123-124 keeps only finite mins). */
static void masked_relax(const csr_t *tr, const double *gated, double *req, int threads) {
    int64_t n = tr->n;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(threads)
#endif
    for (int64_t j = 0; j < n; ++j) {
        double m = INFINITY;
        for (int64_t e = tr->indptr[j]; e < tr->indptr[j + 1]; ++e) {
            double g = gated[tr->col[e]];
            double c = g + tr->val[e];
            if (c < m) m = c;
        }
        req[j] = m;
    }
    (void)threads;
}

/* sssp.py:230-236 */
static int64_t bucket_index_of(double value, double delta) {
    int64_t index = (int64_t)floor(value / delta);
    while ((double)index * delta > value) index -= 1;
    while ((double)(index + 1) * delta <= value) index += 1;
    return index;
}

/* delta_stepping (sssp.py:239-313), fused backend (bit-identical to unfused,
 * sssp.py:10-12).  dist_out[n]: +inf = unreachable (absent from the
 * reference's SparseVector).  Returns OR_* status. */
int oracle_delta_stepping(int64_t n, const int64_t *indptr, const int64_t *col,
                          const double *val, int64_t source, double delta,
                          int skip_empty_buckets, int threads, double *dist_out,
                          int64_t *outer_out, int64_t *phases_out) {
    if (threads < 1) threads = 1;
    /* sssp.py:257-260 */
    if (!(source >= 0 && source < n)) return OR_EINVAL;
    if (!(delta > 0) || !isfinite(delta)) return OR_EINVAL;

    csr_t light = {0}, heavy = {0}, lt = {0}, ht = {0};
    int rc = OR_OK;
    /* split_edges (sssp.py:106-150) + transposed views (sssp.py:148-149) */
    if ((rc = filter_matrix(n, indptr, col, val, delta, 0, &light))) goto done;
    if ((rc = filter_matrix(n, indptr, col, val, delta, 1, &heavy))) goto done;
    if ((rc = transpose(&light, &lt))) goto done;
    if ((rc = transpose(&heavy, &ht))) goto done;

    /* phase ceiling (sssp.py:268-274); saturating instead of Python bigints */
    int64_t per_bucket = 2;
    int64_t nnz_l = light.indptr[n];
    if (nnz_l) {
        double mn = INFINITY;
        for (int64_t e = 0; e < nnz_l; ++e)
            if (light.val[e] < mn) mn = light.val[e];
        double q = ceil(delta / mn);
        per_bucket = (q > 4e18) ? INT64_MAX / 4 : (int64_t)q + 2;
    }
    int64_t ceiling = (per_bucket > INT64_MAX / (n > 0 ? n : 1)) ? INT64_MAX : n * per_bucket;

    double *t = dist_out;
    double *gated = (double *)malloc(sizeof(double) * (size_t)n);
    double *req = (double *)malloc(sizeof(double) * (size_t)n);
    unsigned char *bucket = (unsigned char *)malloc((size_t)n);
    unsigned char *settled = (unsigned char *)malloc((size_t)n);
    if (!gated || !req || !bucket || !settled) {
        rc = OR_ENOMEM;
        goto done2;
    }
    /* vector_build(n, [(source, 0.0)]) (sssp.py:276) */
    for (int64_t v = 0; v < n; ++v) t[v] = INFINITY;
    t[source] = 0.0;

    int64_t index = 0, outer = 0, phases = 0;
    for (;;) {
        /* while t.nnz and max(t) >= index*delta  (sssp.py:280) */
        double mx = -INFINITY;
        int any = 0;
        for (int64_t v = 0; v < n; ++v)
            if (t[v] != INFINITY) {
                any = 1;
                if (t[v] > mx) mx = t[v];
            }
        if (!any || !(mx >= (double)index * delta)) break;

        /* bucket_bounds (fused.py:58-61); compute_bucket (sssp.py:153-158) */
        double lo = (double)index * delta, hi = (double)(index + 1) * delta;
        int64_t bcount = 0;
        for (int64_t v = 0; v < n; ++v) {
            bucket[v] = (t[v] != INFINITY) && (t[v] >= lo) && (t[v] < hi);
            bcount += bucket[v];
            settled[v] = 0; /* settled = SparseVector(n) (sssp.py:285) */
        }
        /* inner loop (sssp.py:292-301): _relax_light_phase_fused (:183-203) */
        while (bcount) {
            for (int64_t v = 0; v < n; ++v) gated[v] = bucket[v] ? t[v] : INFINITY;
            masked_relax(&lt, gated, req, threads);
            int64_t nb = 0;
            for (int64_t v = 0; v < n; ++v) {
                settled[v] |= bucket[v]; /* ewise_add(S, B, OR) (sssp.py:191) */
                /* fused_bucket_update (fused.py:164-191): window + improving
                 * (absent t passes by truthiness, r > 0 always) + min merge */
                double r = req[v];
                unsigned char b = 0;
                if (r != INFINITY) {
                    b = (r >= lo) && (r < hi) && (t[v] == INFINITY || r < t[v]) && (r != 0.0);
                    if (r < t[v]) t[v] = r;
                }
                bucket[v] = b;
                nb += b;
            }
            bcount = nb;
            phases += 1;
            if (phases > ceiling) {
                rc = OR_ENOCONVERGE;
                goto done2;
            }
        }
        /* _relax_heavy_fused (sssp.py:218-227): from settled with current t */
        for (int64_t v = 0; v < n; ++v) gated[v] = settled[v] ? t[v] : INFINITY;
        masked_relax(&ht, gated, req, threads);
        for (int64_t v = 0; v < n; ++v)
            if (req[v] < t[v]) t[v] = req[v];
        outer += 1;
        if (skip_empty_buckets) { /* sssp.py:305-309 */
            double mn = INFINITY;
            for (int64_t v = 0; v < n; ++v)
                if (t[v] != INFINITY && t[v] >= hi && t[v] < mn) mn = t[v];
            if (mn == INFINITY) break;
            index = bucket_index_of(mn, delta);
        } else {
            index += 1;
        }
    }
    *outer_out = outer;
    *phases_out = phases;
done2:
    free(gated);
    free(req);
    free(bucket);
    free(settled);
done:
    csr_free(&light);
    csr_free(&heavy);
    csr_free(&lt);
    csr_free(&ht);
    return rc;
}

/* split_edges (sssp.py:106-150) exported for the split parity tests: writes
 * the light (which=0) or heavy (which=1) CSR.  Call with col_out == NULL to
 * get the entry count in *nnz_out first. */
int oracle_split(int64_t n, const int64_t *indptr, const int64_t *col, const double *val,
                 double delta, int which, int64_t *indptr_out, int64_t *col_out,
                 double *val_out, int64_t *nnz_out) {
    if (!(delta > 0) || !isfinite(delta)) return OR_EINVAL;
    csr_t m = {0};
    int rc = filter_matrix(n, indptr, col, val, delta, which, &m);
    if (rc) {
        csr_free(&m);
        return rc;
    }
    *nnz_out = m.indptr[n];
    if (col_out) {
        memcpy(indptr_out, m.indptr, sizeof(int64_t) * (size_t)(n + 1));
        memcpy(col_out, m.col, sizeof(int64_t) * (size_t)m.indptr[n]);
        memcpy(val_out, m.val, sizeof(double) * (size_t)m.indptr[n]);
    }
    csr_free(&m);
    return OR_OK;
}

/* ------------------------------------------------------------------------
 * dijkstra_oracle (sssp.py:316-341): textbook binary-heap Dijkstra with lazy
 * deletion, relaxing with strict '<' on fl64(d + w).  Shares no code with the
 * bucketed solver.  Used where the bucketed restatement is too slow (grid
 * 4096^2, RMAT-24); the reference's own test pins Dijkstra == Bellman-Ford
 * bit-exactly (tests/test_sssp.py:445-452). */
typedef struct {
    double d;
    int64_t u;
} hent;

static void heap_push(hent *h, int64_t *sz, hent x) {
    int64_t i = (*sz)++;
    while (i > 0) {
        int64_t p = (i - 1) >> 1;
        /* heapq orders tuples (d, u): ties broken by vertex id */
        if (h[p].d < x.d || (h[p].d == x.d && h[p].u <= x.u)) break;
        h[i] = h[p];
        i = p;
    }
    h[i] = x;
}

static hent heap_pop(hent *h, int64_t *sz) {
    hent top = h[0];
    hent x = h[--(*sz)];
    int64_t i = 0, n = *sz;
    for (;;) {
        int64_t c = 2 * i + 1;
        if (c >= n) break;
        if (c + 1 < n && (h[c + 1].d < h[c].d || (h[c + 1].d == h[c].d && h[c + 1].u < h[c].u))) c++;
        if (x.d < h[c].d || (x.d == h[c].d && x.u <= h[c].u)) break;
        h[i] = h[c];
        i = c;
    }
    if (n) h[i] = x;
    return top;
}

int oracle_dijkstra(int64_t n, const int64_t *indptr, const int64_t *col, const double *val,
                    int64_t source, double *dist_out) {
    if (!(source >= 0 && source < n)) return OR_EINVAL;
    int64_t nnz = indptr[n];
    int64_t cap = nnz + 1;
    hent *h = (hent *)malloc(sizeof(hent) * (size_t)cap);
    unsigned char *done = (unsigned char *)calloc((size_t)n, 1);
    if (!h || !done) {
        free(h);
        free(done);
        return OR_ENOMEM;
    }
    for (int64_t v = 0; v < n; ++v) dist_out[v] = INFINITY;
    dist_out[source] = 0.0;
    int64_t sz = 0;
    heap_push(h, &sz, (hent){0.0, source});
    while (sz) {
        hent x = heap_pop(h, &sz);
        if (done[x.u] || x.d > dist_out[x.u]) continue;
        done[x.u] = 1;
        for (int64_t e = indptr[x.u]; e < indptr[x.u + 1]; ++e) {
            int64_t v = col[e];
            double nd = x.d + val[e];
            if (nd < dist_out[v]) {
                dist_out[v] = nd;
                heap_push(h, &sz, (hent){nd, v});
            }
        }
    }
    free(h);
    free(done);
    return OR_OK;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
