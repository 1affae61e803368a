/*
 * dsssp.h -- C-ABI of the B200-native delta-stepping SSSP library
 * (libdsssp.so, built from paper_1911_06895_b200/csrc for sm_100a).
 *
 * Drop-in boundary for the reference path `deltasparse.delta_stepping`
 * (/root/reference/pkg/src/deltasparse/sssp.py:239-313).  The reference is
 * pure Python/numpy and has no FFI of its own; these entry points are what a
 * maintainer binds (ctypes stub in INTEGRATION.md) to replace, one for one:
 *
 *   ds_graph_create    <- SparseMatrix(n, indptr, col, val)    core.py:130-137
 *                         (+ the instance cache of derived data, core.py:128)
 *   ds_graph_prepare   <- split_edges(matrix, delta)           sssp.py:106-150
 *                         + phase ceiling                      sssp.py:268-274
 *   ds_sssp            <- delta_stepping(matrix, source, delta,
 *                           skip_empty_buckets=...)            sssp.py:239-313
 *   ds_sssp_batch      <- the callers' per-source loop          cli.py:119-128
 *   ds_result_sparse   <- SsspResult.distances (SparseVector)  sssp.py:82-87,
 *                                                              core.py:46-70
 *   ds_result_dense    <- same, as a dense float64 vector (+inf = absent)
 *   ds_export_split    <- the (light, heavy) SparseMatrix pair of split_edges
 *   ds_last_error      <- exception message text
 *
 * Conventions: plain pointers and sizes, no torch types.  Host pointers are
 * copied (pageable or pinned); device pointers (cudaMalloc'd on the graph's
 * device) are accepted wherever noted.  Every call returns DS_OK (0) or an
 * error code; the message is in ds_last_error() (thread-local).
 *   DS_EINVAL      -> ValueError   (bad source / delta / CSR)
 *   DS_ENOCONVERGE -> RuntimeError ("light phase count exceeded ceiling ...")
 *   DS_ECUDA / DS_ENOMEM / DS_ETIMEOUT -> RuntimeError
 * A handle is bound to one device and one stream; it is not re-entrant.
 */
#ifndef DSSSP_H
#define DSSSP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DS_OK 0
#define DS_EINVAL 1
#define DS_ENOCONVERGE 2
#define DS_ECUDA 3
#define DS_ENOMEM 4
#define DS_ETIMEOUT 5
#define DS_EPARSE 6  /* graph file structure -> deltasparse.io.ParseError      */
#define DS_EVALID 7  /* graph file content   -> deltasparse.io.ValidationError */

/* column-index dtypes */
#define DS_IDX_I32 0
#define DS_IDX_I64 1
/* weight dtypes */
#define DS_W_F32 0
#define DS_W_F64 1
#define DS_W_I32 2

/* ds_sssp flags */
#define DS_FLAG_SKIP_EMPTY 1u /* outer_iterations counts like skip_empty_buckets=True */
#define DS_FLAG_FORCE_F64 2u  /* disable the exact 32-bit fixed-point distance mode */
#define DS_FLAG_NO_LEX 4u     /* keep the reference's bucket schedule (no sub-buckets) */

/* distance modes reported in ds_prep_info / ds_stats */
#define DS_MODE_FIXED32 0 /* d * 2^frac_bits held exactly in uint32 */
#define DS_MODE_F64 1     /* IEEE binary64 bit patterns, u64 atomicMin */

typedef struct ds_graph ds_graph;

typedef struct ds_prep_info {
    int64_t nnz_light;        /* entries with 0 < w <= delta              */
    int64_t nnz_heavy;        /* entries with delta < w < inf             */
    double min_light_weight;  /* +inf when A_L is empty                   */
    int64_t phase_ceiling;    /* n * (ceil(delta / min w_L) + 2), saturating */
    int32_t dist_mode;        /* DS_MODE_*                                */
    int32_t frac_bits;        /* fixed-point scale (DS_MODE_FIXED32)      */
    double prepare_ms;        /* device time of the split                 */
    int32_t sub_buckets;      /* internal buckets per reference bucket (1 = the
                                 reference's schedule; >1 = lex mode)       */
    int32_t reserved;
} ds_prep_info;

typedef struct ds_stats {
    int64_t outer_iterations; /* as the reference's SsspResult            */
    int64_t inner_phases;
    int64_t buckets_visited;  /* non-empty buckets (= skip-mode outer)    */
    int64_t reached;          /* n_r: vertices with finite distance       */
    int64_t edges_reached;    /* m_r: sum of out-degrees of reached ones  */
    int64_t edges_scanned;    /* light + heavy edge visits performed      */
    int64_t grid_barriers;    /* device-wide barriers executed            */
    double max_distance;      /* largest finite distance                  */
    double kernel_ms;         /* device time of the solve (CUDA events)   */
    int32_t dist_mode;        /* mode that produced the result            */
    int32_t fallbacks;        /* 1 if fixed-point overflowed and f64 reran */
    int64_t pull_steps;       /* relaxations run in pull (vxm) form       */
    int64_t launches;         /* solver kernel launches (persistent + handed-off pushes) */
} ds_stats;

/* Upload a CSR adjacency (rows = out-edges).  indptr: n+1 int64; col: nnz
 * entries of col_dtype; val: nnz entries of val_dtype.  Pointers may be host
 * or device memory.  stream: a cudaStream_t (NULL = legacy default stream).
 * Validates indptr monotonicity and column range (DS_EINVAL otherwise). */
int ds_graph_create(int64_t n, int64_t nnz, const int64_t* indptr, const void* col,
                    int col_dtype, const void* val, int val_dtype, int device,
                    void* stream, ds_graph** out);

/* Split into light/heavy device CSRs for delta (cached until delta or mode
 * changes).  info may be NULL. */
int ds_graph_prepare(ds_graph* g, double delta, uint32_t flags, ds_prep_info* info);

/* One source, end to end on the device (prepares if needed).  Result stays
 * on the device until fetched with ds_result_*. stats may be NULL. */
int ds_sssp(ds_graph* g, int64_t source, double delta, uint32_t flags, ds_stats* stats);

/* k sources against one prepared graph (the reference's callers loop over
 * sources: cli.py:119-128, the 64/16-source benchmarks).  Up to `concurrency`
 * sources run at once on SM-disjoint persistent grids, each on its own
 * stream (0 = library default: DS_BATCH_CONC if set, else 8 for graphs below
 * 24 Mi edges or high-diameter graphs, 2 otherwise).  stats: k entries or
 * NULL.  dist_out: k x n float64 (row i = dense distances of sources[i],
 * +inf = unreachable), host or device, or NULL to keep nothing.  A source
 * whose fixed-point solve overflows is rerun in binary64 (stats.fallbacks=1).
 * Leaves no "last result" for ds_result_*. */
int ds_sssp_batch(ds_graph* g, const int64_t* sources, int64_t k, double delta, uint32_t flags,
                  int32_t concurrency, ds_stats* stats, double* dist_out);

/* Dense float64 distances of the last solve (+inf = unreachable); out holds
 * n doubles, host or device. */
int ds_result_dense(ds_graph* g, double* out);

/* Reached vertices of the last solve, ascending: idx[reached] int64 and
 * val[reached] float64 (host or device); sizes from ds_stats.reached. */
int ds_result_sparse(ds_graph* g, int64_t* idx, double* val);

/* Light (which=0) or heavy (which=1) CSR of the current prepare: indptr
 * n+1, col/val nnz_light or nnz_heavy entries (host pointers). */
int ds_export_split(ds_graph* g, int which, int64_t* indptr, int64_t* col, double* val);

/* Rebind the handle to another stream (cudaStream_t). */
int ds_graph_set_stream(ds_graph* g, void* stream);

/* Vertices / stored entries of the handle. */
int ds_graph_size(const ds_graph* g, int64_t* n, int64_t* nnz);

void ds_graph_destroy(ds_graph* g);
/* Graph buffers are pooled per device and reused by later handles; this
 * returns every cached buffer to the driver. */
void ds_release_pool(void);
const char* ds_last_error(void);
int ds_device_count(void);

/* Debug timeline of the last solve when DS_TRACE=1 was set: out holds
 * 1 + 2*cap words = [start_ns, then per grid step (end_ns, kind<<56 | work)]
 * with kind 0 bucket scan, 1 light relax, 2 light capture, 3 heavy capture,
 * 4 heavy relax.  Returns the number of steps written. */
int64_t ds_debug_trace(ds_graph* g, uint64_t* out, int64_t cap);

/* DS_TRACE=2 load-balance diagnostics of the last solve: out[0] = grid size,
 * then for every step the time each CTA's warps finished it (steps x grid
 * words).  Returns the number of words written after out[0]. */
int64_t ds_debug_cta_times(ds_graph* g, uint64_t* out, int64_t cap);

/* On-device synthetic R-MAT (Graph500 a,b,c,d = .57,.19,.19,.05; self-loops
 * dropped; symmetrised; deduplicated; fp32-lattice weight k*2^-24 per
 * undirected pair).  Bit-identical to paper_1911_06895_b200.graphs.rmat.
 * Creates the graph handle directly (no host round trip); the CSR can be
 * fetched with ds_graph_download. */
int ds_gen_rmat(int32_t scale, int32_t edge_factor, uint64_t seed, uint64_t weight_seed,
                int device, void* stream, ds_graph** out);

/* Copy the handle's original CSR to host/device buffers: indptr n+1 int64,
 * col nnz int32, val nnz float32 (weights must be float32-exact).  Any of the
 * three may be NULL (not copied). */
int ds_graph_download(ds_graph* g, int64_t* indptr, int32_t* col, float* val);

/* ------------------------------------------------------------------------
 * Partitioned solver: one shard per rank / GPU.  A shard
 * owns the input-id range [v0, v0 + n_local) and stores the edges whose
 * TARGET it owns as a CSR over all n_global sources (col = local target id).
 * The host exchanges frontiers between ranks (all-gather) once per phase;
 * paper_1911_06895_b200/distributed.py drives the protocol.  Buffers passed
 * to scan/s_add/relax are device pointers; values are distances widened to
 * u64 (fixed-point integers or binary64 bit patterns). */
typedef struct ds_shard ds_shard;

int ds_shard_create(int64_t n_global, int64_t v0, int64_t n_local, int64_t nnz,
                    const int64_t* indptr, const int32_t* col_local, const double* val,
                    int device, void* stream, ds_shard** out);
void ds_shard_destroy(ds_shard* s);
/* out5 = {min light weight bits, max weight bits, max fraction bits, nnz_L, nnz_H} */
int ds_shard_probe(ds_shard* s, double delta, uint64_t* out5);
int ds_shard_prepare(ds_shard* s, double delta, int mode, int frac_bits);
int ds_shard_begin(ds_shard* s, int64_t source);
int ds_shard_scan(ds_shard* s, uint64_t L, uint64_t H, int32_t* out_ids, uint64_t* out_vals,
                  int64_t* count, uint64_t* next_min);
int ds_shard_s_add(ds_shard* s, const int32_t* ids, const uint64_t* vals, int64_t count);
int ds_shard_relax(ds_shard* s, int heavy, const int32_t* ids, const uint64_t* vals, int64_t count,
                   uint64_t H, int32_t* out_ids, uint64_t* out_vals, int64_t* out_count,
                   int32_t* overflow);
int ds_shard_result(ds_shard* s, double* out);
/* Solver kernels this shard has launched so far (begin, scan, s_add, relax, result). */
int64_t ds_shard_launches(const ds_shard* s);
/* Shard [v0, v1) cut on the device from a resident graph handle. */
int ds_shard_from_graph(ds_graph* g, int64_t v0, int64_t v1, ds_shard** out);

/* ---- graph-file ingestion (host side, no device needed) -----------------
 * Native parser for the reference loaders (deltasparse/io.py):
 *   DS_FMT_MTX   <- load_matrix_market(path, default_weight)   io.py:121-193
 *   DS_FMT_EDGES <- load_edge_list(path, directed, default_weight) io.py:196-259
 * over an in-memory file image (`name` is used in messages only).  Errors
 * read "name:lineno: message" (ds_last_error) with the line number also in
 * ds_ingest_error_line(); DS_EPARSE / DS_EVALID mirror ParseError /
 * ValidationError.  The result is the COO entry list in file order (mirrored
 * for symmetric / undirected input, self-loops dropped and counted) and the
 * external label of every internal id; build the CSR with matrix_build
 * semantics (duplicates keep the minimum weight, core.py:247-278). */
#define DS_FMT_MTX 0
#define DS_FMT_EDGES 1
typedef struct ds_ingest ds_ingest;
int ds_ingest_parse(const char* data, int64_t len, int32_t format, int32_t directed,
                    double default_weight, const char* name, ds_ingest** out);
int ds_ingest_info(const ds_ingest* h, int64_t* n, int64_t* entries, int64_t* self_loops);
/* rows/cols/vals: `entries` each; labels: n (any may be NULL) */
int ds_ingest_copy(const ds_ingest* h, int64_t* rows, int64_t* cols, double* vals, int64_t* labels);
int64_t ds_ingest_error_line(void);
void ds_ingest_free(ds_ingest* h);

#ifdef __cplusplus
}
#endif
#endif /* DSSSP_H */
