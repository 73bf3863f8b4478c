/*
 * tcdtw.h -- C ABI of the B200-native TC-DTW hot path (libtcdtw.so).
 *
 * This is the drop-in boundary.  The reference (mvdtw v0.1.0, a pure
 * Python/numpy package; citations are file:line relative to
 * /root/reference/pkg/src/mvdtw) has no native FFI of its own: its operator
 * API is the set of Python functions re-exported in __init__.py:3-38.  Each
 * entry point below replaces one of those functions (or a batch of calls to
 * it) and is bound from Python with ctypes by paper_2101_07731_b200/_lib.py
 * (the binding a maintainer would add is shown in INTEGRATION.md).
 *
 * Conventions
 *  - Plain C types only; every array pointer is a DEVICE pointer unless the
 *    comment says "host".  Series arrays are row-major (count, n, dims) of
 *    element type `dtype` (TCDTW_F32 = float, TCDTW_F64 = double).  Per-pair
 *    entry points pair row p of the first array with row p of the second.
 *  - `stream` is a cudaStream_t (NULL = the legacy default stream).  All
 *    work is enqueued on it; calls are reentrant (no global mutable state)
 *    and return after enqueueing unless noted.
 *  - Inputs are validated on the host before any launch; bad arguments
 *    return TCDTW_INVALID_INPUT (mapped to InvalidInputError, core.py:17).
 *  - Abandon thresholds: NULL means "no abandoning" (abandon_above=None);
 *    otherwise one value per pair, +inf meaning none.
 *  - The library never keeps memory or pointers past a call.  The batched
 *    search works inside a caller-provided workspace whose size
 *    tcdtw_search_workspace_size reports.
 */
#ifndef TCDTW_H_
#define TCDTW_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum tcdtw_status_code {
    TCDTW_OK = 0,
    TCDTW_INVALID_INPUT = 1,
    TCDTW_CUDA_ERROR = 2,
    TCDTW_WORKSPACE_TOO_SMALL = 3,
    TCDTW_NOT_SUPPORTED = 4
};

enum tcdtw_dtype { TCDTW_F32 = 0, TCDTW_F64 = 1 };

/* Method, core.py:21-29 */
enum tcdtw_method {
    TCDTW_METHOD_NONE = 0,
    TCDTW_METHOD_LB_MV = 1,
    TCDTW_METHOD_LB_TI = 2,
    TCDTW_METHOD_LB_PC = 3,
    TCDTW_METHOD_TC_DTW = 4,
    TCDTW_METHOD_LB_AD = 5
};

/* TiVariant, core.py:32-38 */
enum tcdtw_ti_variant { TCDTW_TI_BASIC = 0, TCDTW_TI_TOP = 1, TCDTW_TI_TIP = 2, TCDTW_TI_TIP_TOP = 3 };

const char *tcdtw_strerror(int status);
int tcdtw_abi_version(void);
/* Kernel launches issued by the library so far (statistics only). */
unsigned long long tcdtw_launch_count(void);

/* ---------------------------------------------------------------------- */
/* Per-pair operators (the reference's per-call functions, batched).       */
/* ---------------------------------------------------------------------- */

/* dtw_banded(q, c, window, abandon_above) -> DtwResult(distance, abandoned,
 * cells), dtw.py:45-102.  Row-granular abandoning exactly as the reference
 * (rows index a).  out_distance has dtype `dtype`. */
int tcdtw_dtw_banded(int dtype, const void *a, const void *b, int64_t n_pairs, int32_t n,
                     int32_t dims, int32_t window, const void *abandon_above, void *out_distance,
                     uint8_t *out_abandoned, int64_t *out_cells, void *stream);

/* build_envelope(q, window) -> Envelope(upper, lower), lb_mv.py:74-88.
 * Also the whole-collection envelope (candidate-side index). */
int tcdtw_build_envelope(int dtype, const void *series, int64_t n_series, int32_t n, int32_t dims,
                         int32_t window, void *upper, void *lower, void *stream);

/* lb_mv(c, env, abandon_above) -> BoundResult(value, abandoned), lb_mv.py:98-107.
 * upper/lower are per pair (n_pairs, n, dims). */
int tcdtw_lb_mv(int dtype, const void *c, const void *upper, const void *lower, int64_t n_pairs,
                int32_t n, int32_t dims, const void *abandon_above, void *out_value,
                uint8_t *out_abandoned, void *stream);

/* lb_ad(q, c, window, abandon_above), lb_mv.py:110-128. */
int tcdtw_lb_ad(int dtype, const void *q, const void *c, int64_t n_pairs, int32_t n, int32_t dims,
                int32_t window, const void *abandon_above, void *out_value, uint8_t *out_abandoned,
                void *stream);

/* neighbor_steps(series) -> (n_series, n-1), lb_ti.py:51-55. */
int tcdtw_neighbor_steps(int dtype, const void *series, int64_t n_series, int32_t n, int32_t dims,
                         void *out, void *stream);

/* ti_advance / ti_extend_top elementwise, lb_ti.py:79-93. */
int tcdtw_ti_advance(int dtype, const void *lo, const void *up, const void *step, int64_t count,
                     void *out_lo, void *out_up, void *stream);

/* lb_ti(q, c, window, variant, refresh_period, neighbor, abandon_above),
 * lb_ti.py:96-200.  query_steps (n_pairs, n-1) and cand_steps may be NULL
 * (computed on the fly, as NeighborDistances.build does). */
int tcdtw_lb_ti(int dtype, const void *q, const void *c, int64_t n_pairs, int32_t n, int32_t dims,
                int32_t window, int32_t variant, int32_t refresh_period, const void *query_steps,
                const void *cand_steps, const void *abandon_above, void *out_value,
                uint8_t *out_abandoned, void *stream);

/* build_box_sets(q, window, group_width, levels, max_boxes, min_cell_frac,
 * dim_range), lb_pc.py:239-261, for every series.  Outputs are padded to
 * max_boxes per group: out_lo/out_hi (n_series, G, max_boxes, dims) with
 * +inf/-inf in unused slots (lb_pc.py:229-234), out_counts (n_series, G).
 * G = (n-1)/group_width + 1.  dim_range: NULL (each series' own range) or
 * one shared (dims,) array.  quantize_cluster (lb_pc.py:56-116) is the
 * single-group case window = n-1, group_width = n. */
int tcdtw_build_box_sets(int dtype, const void *series, int64_t n_series, int32_t n, int32_t dims,
                         int32_t window, int32_t group_width, int32_t levels, int32_t max_boxes,
                         double min_cell_frac, const void *dim_range, void *out_lo, void *out_hi,
                         int32_t *out_counts, void *stream);

/* lb_pc(c, grouping, abandon_above), lb_pc.py:264-280; boxes per pair
 * (n_pairs, n_groups, kmax, dims). */
int tcdtw_lb_pc(int dtype, const void *c, const void *box_lo, const void *box_hi, int64_t n_pairs,
                int32_t n, int32_t dims, int32_t n_groups, int32_t kmax, int32_t group_width,
                const void *abandon_above, void *out_value, uint8_t *out_abandoned, void *stream);

/* ---------------------------------------------------------------------- */
/* Batched 1-NN search: nn_search (search.py:75-180) for a batch of        */
/* queries against one (shard of a) candidate collection.                   */
/* ---------------------------------------------------------------------- */

typedef struct tcdtw_search_desc {
    int32_t dtype;          /* TCDTW_F32 (filter + float64 finalist re-score) | TCDTW_F64 */
    int32_t n;              /* series length */
    int32_t dims;
    int32_t window;         /* SearchParams.window; min(window, n-1) applies (core.py:200-201) */
    int32_t method;         /* tcdtw_method */
    int32_t advanced;       /* TC_DTW: resolved bound (LB_TI | LB_PC), search.py:59-68 */
    int32_t refresh_period; /* SearchParams fields, core.py:154-198 */
    int32_t quant_levels;
    int32_t max_boxes;
    int32_t group_width;
    double trigger_ti;
    double trigger_pc;
    double min_cell_frac;
    int64_t n_queries;      /* queries in this call, 1..65535 */
    int64_t n_candidates;   /* candidates in this shard */
    int64_t candidate_base; /* global index of this shard's candidate 0 */
    int32_t seeds;          /* seed DTWs per query (0 = default 8) */
    int32_t flags;          /* TCDTW_FLAG_* */
    float *phase_ms;        /* host, nullable: TCDTW_PHASES per-phase CUDA-event times */
    /* Candidate-side index (ABI version 2): envelopes of
     * this shard's candidates, (n_candidates, n, dims) of `dtype`, built with
     * tcdtw_build_envelope at window min(window, n-1).  Read only with
     * TCDTW_FLAG_REVERSE_LB, which prunes on max(LB_MV(c, env(q)),
     * LB_MV(q, env(c))): DTW is symmetric in its arguments for equal lengths,
     * so both are lower bounds (an extension; the reference's "switch the
     * role" idea).  The in-DTW cascade keeps using the
     * forward terms. */
    const void *cand_upper;
    const void *cand_lower;
    /* Capacity of the completed-DTW list the finalisation visits (0 =
     * default); when it overflows, every survivor tile is scanned instead.
     * Tests set 1 to exercise that path (ABI version 3). */
    int64_t done_cap;
    /* Optional (ABI version 3; trailer since 4): the candidates in the
     * planar layout the LB_MV pass reads, made once per collection with
     * tcdtw_planarize into tcdtw_planar_bytes(...) bytes; NULL = planarised
     * into the workspace on every call.  Ignored with TCDTW_FLAG_F32_FILTER
     * and, for float32, with TCDTW_FLAG_REVERSE_LB. */
    const void *cand_planar;
    /* Candidate-side box sets (ABI version 3): every
     * candidate's LB_PC boxes, (n_candidates, G, max_boxes, dims) lo / hi of
     * `dtype`, +inf / -inf padded, built with tcdtw_build_box_sets using this
     * search's window, group_width, quant_levels, max_boxes, min_cell_frac
     * and dim_range.  Read only with TCDTW_FLAG_REVERSE_PC. */
    const void *cand_box_lo;
    const void *cand_box_hi;
} tcdtw_search_desc;

#define TCDTW_FLAG_TIMING 1     /* fill desc->phase_ms (synchronises the stream) */
#define TCDTW_FLAG_REVERSE_LB 2 /* also prune on the candidate-envelope bound */
/* dtype must be TCDTW_F64.  The filter (bounds, seeds, DTW with abandoning)
 * runs in float32 on float32 roundings of the inputs, made in the workspace
 * by the seed phase; decisions carry an extra absolute slack that covers the
 * rounding (2.5 (2n-1) 2^-24 (max|q| + max|c|)), and the finalists are
 * re-scored in float64 on the original inputs, so best_distance is the
 * reference's float64 value and best_index its lowest-index argmin.  d_best
 * is then float32.  Inputs must lie inside the float32 range.  Not combined
 * with TCDTW_FLAG_REVERSE_LB. */
#define TCDTW_FLAG_F32_FILTER 4
#define TCDTW_FLAG_DEBUG_SYNC 8 /* synchronise + report to stderr after every stage */
/* Prune / abandon against a snapshot of d_best taken before each DTW pass
 * instead of the live value other DTWs keep tightening: the same answers,
 * somewhat more DP cells, and dtw_cells / abandon_count identical from run
 * to run -- what the reference's deterministic work model (search.py:14-19,
 * 102-125) needs when tuning or selecting on the GPU's counters. */
#define TCDTW_FLAG_FROZEN_THRESHOLDS 16
/* DTW abandons on its row minima only, without the LB_MV suffix cascade
 * (an A/B knob: the same answers, more DP cells). */
#define TCDTW_FLAG_NO_CASCADE 32
/* With an LB_PC second stage, also bound every triggered pair by the reverse
 * LB_PC -- the query's points against the candidate's box sets
 * (desc->cand_box_lo/hi) -- and prune on the larger of the two.  DTW is
 * symmetric in its arguments for equal lengths, so both are lower bounds
 * (an extension; "switch the role").  Not combined with
 * TCDTW_FLAG_F32_FILTER. */
#define TCDTW_FLAG_REVERSE_PC 64
#define TCDTW_PHASES 8      /* prep, lb_mv, seeds_topk, seeds_dtw, compact, advanced, dtw, finalize */
#define TCDTW_COUNTERS 9    /* per query: see enum below */

enum tcdtw_counter {
    TCDTW_C_DTW_COMPUTED = 0,  /* NnOutcome.dtw_computed (search.py:46-56) */
    TCDTW_C_DTW_SKIPPED = 1,
    TCDTW_C_LB_MV_EVALS = 2,
    TCDTW_C_ADVANCED_LB_EVALS = 3,
    TCDTW_C_ABANDON_COUNT = 4,
    TCDTW_C_DTW_CELLS = 5,     /* DP cells evaluated, as dtw.py:96 counts them */
    TCDTW_C_FINALISTS = 6,     /* candidates re-scored / tie-checked in float64 */
    TCDTW_C_SURVIVORS = 7,     /* entries left after LB_MV */
    TCDTW_C_CELLS_ISSUED = 8   /* DP cells issued by the DTW kernels incl. lockstep waste */
};

int tcdtw_search_workspace_size(const tcdtw_search_desc *desc, size_t *bytes);

/* Phase 1: per-query prep, LB_MV over every (query, candidate) pair, seed
 * DTWs on the smallest bounds.  Writes each query's best-so-far distance
 * (dtype) to d_best (device, n_queries).  A sharded caller may min-reduce
 * d_best across shards before phase 2. */
int tcdtw_search_seed(const tcdtw_search_desc *desc, const void *queries, const void *candidates,
                      const void *dim_range, void *workspace, size_t ws_bytes, void *d_best,
                      void *stream);

/* Phase 2: survivor compaction against d_best, the advanced bound on the
 * trigger band, DTW with early abandoning, lexicographic (distance, index)
 * reduction with float64 finalist re-scoring.  Purely asynchronous: the
 * survivor and tile counts stay on the device (the grids are sized by their
 * upper bounds), so the host never waits -- a sharded caller's d_best
 * exchange of batch k overlaps the GPU work of batch k+1 (only
 * TCDTW_FLAG_TIMING / TCDTW_FLAG_DEBUG_SYNC synchronise).  best_index is global
 * (candidate_base added; -1 if every candidate of this shard was pruned
 * against a better d_best from another shard, with best_distance +inf).
 * counters: (n_queries, TCDTW_COUNTERS) int64. */
int tcdtw_search_finish(const tcdtw_search_desc *desc, const void *queries, const void *candidates,
                        const void *dim_range, void *workspace, size_t ws_bytes, const void *d_best,
                        int64_t *best_index, double *best_distance, int64_t *counters, void *stream);

/* Both phases (single shard). */
int tcdtw_nn_search(const tcdtw_search_desc *desc, const void *queries, const void *candidates,
                    const void *dim_range, void *workspace, size_t ws_bytes, int64_t *best_index,
                    double *best_distance, int64_t *counters, void *stream);

/* The planar copy of a collection for tcdtw_search_desc.cand_planar:
 * series (n_series, n, dims) -> out (n * dims, n_series), dtype elements,
 * followed by a trailer; `out` holds tcdtw_planar_bytes(...) bytes (ABI
 * version 4).  The copy is opaque: float32 values are multiplied by a power
 * of two sigma that maps the collection's value range into (1/2, 1] (exact),
 * and the trailer keeps {sigma, 1/sigma}.  The LB_MV pass then evaluates a
 * per-dimension envelope deviation as sat(|c - m| - h) on (midpoint, half
 * width) query envelopes -- FADD, FADD.SAT, FFMA instead of the five
 * operations of max(c - u, l - c, 0) (lb_mv.py:91-104) -- with h inflated so
 * the float32 value never exceeds the real deviation by more than two
 * roundings; a deviation above the collection's range saturates (a weaker,
 * still valid bound).  Returns 0 on invalid arguments. */
size_t tcdtw_planar_bytes(int dtype, int64_t n_series, int32_t n, int32_t dims);
int tcdtw_planarize(int dtype, const void *series, int64_t n_series, int32_t n, int32_t dims, void *out,
                    void *stream);

/* Cross-shard combine (no reference counterpart -- the
 * reference is single-process).  records (world, n_queries, 2)
 * int64 on the device: every rank's (float64 best_distance bits, global
 * best_index) as gathered by one all-gather; writes the lexicographic
 * (distance, index) minimum per query -- lowest index on equal distances,
 * search.py:173 -- ignoring index -1 entries. */
int tcdtw_shard_combine(const int64_t *records, int32_t world, int64_t n_queries, int64_t *best_index,
                        double *best_distance, void *stream);

/* Standalone LB_MV matrix (the search's dominant streaming kernel), for
 * benchmarking: out (n_queries, n_candidates) = LB_MV of every pair given
 * query envelopes (n_queries, n, dims). */
int tcdtw_lb_mv_matrix(int dtype, const void *upper, const void *lower, const void *candidates,
                       int64_t n_queries, int64_t n_candidates, int32_t n, int32_t dims, void *out,
                       void *stream);

/* Name of the DTW kernel the survivors pass launches for this shape
 * (informational; a static string). */
const char *tcdtw_dtw_kernel_name(const tcdtw_search_desc *desc);

/* ---------------------------------------------------------------------- */
/* Device-side ingest.                                   */
/* ---------------------------------------------------------------------- */

/* Text datasets -> host float64 values.  Replaces the
 * tokenizing and float() conversion of parse_native (ingest.py:92-126) and
 * parse_ts_subset (ingest.py:157-231); the caller reads the file and turns
 * the error record into the reference's ParseError message (ingest.py in
 * this package).  `text`/`values` are HOST pointers.
 *   values == NULL : validate the layout and report the shape in *info
 *                    (native: header and line count; .ts: the whole file);
 *   values != NULL : also convert into values (num_series, length, dims),
 *                    NaN for missing tokens (NA / NaN / ?), capacity in
 *                    doubles.
 * Returns TCDTW_OK, TCDTW_INVALID_INPUT with info->error set, or
 * TCDTW_WORKSPACE_TOO_SMALL.  Lines are numbered from 1 as the reference
 * numbers them (universal newlines). */
enum tcdtw_text_format { TCDTW_FORMAT_NATIVE = 0, TCDTW_FORMAT_TS = 1 };

enum tcdtw_parse_error {
    TCDTW_PARSE_OK = 0,
    TCDTW_PARSE_EMPTY,            /* "empty file" */
    TCDTW_PARSE_HEADER_FIELDS,    /* header is not three fields */
    TCDTW_PARSE_HEADER_INT,       /* non-integer header field */
    TCDTW_PARSE_HEADER_POSITIVE,  /* header fields must be positive */
    TCDTW_PARSE_LINE_COUNT,       /* expected/found value lines */
    TCDTW_PARSE_ROW_WIDTH,        /* expected/found values on a line */
    TCDTW_PARSE_TOKEN,            /* non-numeric token (tok_off, tok_len) */
    TCDTW_PARSE_TS_AFTER_DATA,    /* directive after @data */
    TCDTW_PARSE_TS_DIRECTIVE,     /* unsupported directive (tok = its name) */
    TCDTW_PARSE_TS_FLAG,          /* expected true/false (tok = the argument) */
    TCDTW_PARSE_TS_TIMESTAMPS,    /* timestamped files are not supported */
    TCDTW_PARSE_TS_UNEQUAL,       /* unequal-length series are not supported */
    TCDTW_PARSE_TS_INT_ARG,       /* @dimensions / @seriesLength argument is not an int */
    TCDTW_PARSE_TS_BEFORE_DATA,   /* data before @data directive */
    TCDTW_PARSE_TS_LABEL,         /* missing class label */
    TCDTW_PARSE_TS_DIMS,          /* expected/found dimensions */
    TCDTW_PARSE_TS_RAGGED,        /* ragged dimensions within one series */
    TCDTW_PARSE_TS_LENGTH,        /* expected/found length */
    TCDTW_PARSE_TS_SHAPE,         /* series shape differs from earlier series */
    TCDTW_PARSE_TS_NO_DATA        /* no data lines */
};

typedef struct tcdtw_parse_info {
    int64_t num_series, length, dims; /* shape on success */
    int64_t line;                     /* 1-based line of the error (0 = whole file) */
    int64_t tok_off, tok_len;         /* offending token's byte range in text (-1 = none) */
    int64_t expected, found;          /* counts of the count/shape errors */
    int64_t name_off, name_len;       /* .ts @problemName argument (-1 = none) */
    int32_t error;                    /* tcdtw_parse_error */
    int32_t reserved;
} tcdtw_parse_info;

int tcdtw_parse_text(int32_t format, const char *text, size_t len, double *values, int64_t capacity,
                     tcdtw_parse_info *info);

/* normalize(ds) -> Dataset(values, dim_ranges), ingest.py:245-261, on the
 * device, bit-identical to the reference: values (n_points, dims) float64
 * with NaN marking missing entries (n_points = num_series * length); out
 * (n_points, dims) z-normalised per dimension with the population mean/std
 * over all points (missing values enter as raw zeros, zero-variance
 * dimensions become all-zeros); mean, std, range (dims,) -- range is the
 * post-normalisation max - min (ingest.py:235-237), the LB_PC dim_range.
 * The sums follow numpy's axis-0 reduction order: a sequential running sum
 * per dimension for dims >= 2, numpy's pairwise summation for dims == 1.
 * out may alias values. */
int tcdtw_normalize_workspace_size(int64_t n_points, int32_t dims, size_t *bytes);
int tcdtw_normalize(const double *values, int64_t n_points, int32_t dims, double *out, double *mean,
                    double *std, double *range, void *workspace, size_t ws_bytes, void *stream);

/* Issue-rate probe: a dependent-chain-free FFMA/DFMA loop, for measuring
 * the ALU roofline on the box.  Returns lane-operations issued. */
int tcdtw_alu_probe(int dtype, int32_t blocks, int32_t iters, void *sink, double *lane_ops,
                    void *stream);

#ifdef __cplusplus
}
#endif

#endif /* TCDTW_H_ */
