// capi.cu -- extern "C" entry points of libtcdtw.so (include/tcdtw.h).
//
// Host-side validation mirrors the reference's InvalidInputError rules
// (core.py:41-57, dtw.py:56-61, lb_mv.py:77-78/105-106/120-121,
// lb_ti.py:124-130, lb_pc.py:80-83/255-258/268-271, search.py:64-66/93-94)
// and runs before any launch.

#include <cuda_runtime.h>

#include "../../include/tcdtw.h"
#include "common.cuh"
#include "dispatch.cuh"

namespace tcdtw {
int pairs_dtw(int, const void*, const void*, int64_t, int, int, int, const void*, void*, uint8_t*, int64_t*,
              cudaStream_t);
int pairs_lb_mv(int, const void*, const void*, const void*, int64_t, int, int, const void*, void*, uint8_t*,
                cudaStream_t);
int pairs_lb_ad(int, const void*, const void*, int64_t, int, int, int, const void*, void*, uint8_t*, cudaStream_t);
int series_steps(int, const void*, int64_t, int, int, void*, cudaStream_t);
int pairs_lb_ti(int, const void*, const void*, int64_t, int, int, int, int, int, const void*, const void*,
                const void*, void*, uint8_t*, cudaStream_t);
int pairs_lb_pc(int, const void*, const void*, const void*, int64_t, int, int, int, int, int, const void*, void*,
                uint8_t*, cudaStream_t);
int series_envelope(int, const void*, int64_t, int, int, int, void*, void*, cudaStream_t);
int ti_advance_elementwise(int, const void*, const void*, const void*, int64_t, void*, void*, cudaStream_t);
int series_box_sets(int, const void*, int64_t, int, int, int, int, int, int, double, const void*, void*, void*,
                    int32_t*, cudaStream_t);
int search_workspace_size(const tcdtw_search_desc*, size_t*);
int search_seed(const tcdtw_search_desc*, const void*, const void*, const void*, void*, size_t, void*,
                cudaStream_t);
int search_finish(const tcdtw_search_desc*, const void*, const void*, const void*, void*, size_t, const void*,
                  int64_t*, double*, int64_t*, cudaStream_t);
int lb_mv_matrix(int, const void*, const void*, const void*, int64_t, int64_t, int, int, void*, cudaStream_t);
int alu_probe(int, int, int, void*, double*, cudaStream_t);
const char* dtw_kernel_name(const tcdtw_search_desc*);
size_t normalize_workspace_bytes(int64_t, int);
int normalize_f64(const double*, int64_t, int, double*, double*, double*, double*, double*, cudaStream_t);
int shard_combine(const int64_t*, int, int64_t, int64_t*, double*, cudaStream_t);
int planarize_series(int, const void*, int64_t, int, int, void*, cudaStream_t);
size_t planar_copy_bytes(int, int64_t, int, int);
}  // namespace tcdtw

using namespace tcdtw;

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
static inline bool dtype_ok(int t) { return t == TCDTW_F32 || t == TCDTW_F64; }
static inline bool shape_ok(int64_t count, int32_t n, int32_t dims) {
    return count >= 0 && n >= 1 && dims >= 1;
}
static inline int eff_window(int32_t window, int32_t n) { return window < n - 1 ? window : n - 1; }

extern "C" {

const char* tcdtw_strerror(int status) {
    switch (status) {
        case TCDTW_OK: return "ok";
        case TCDTW_INVALID_INPUT: return "invalid input";
        case TCDTW_CUDA_ERROR: return "CUDA error";
        case TCDTW_WORKSPACE_TOO_SMALL: return "workspace too small";
        case TCDTW_NOT_SUPPORTED: return "configuration not supported";
        default: return "unknown status";
    }
}

int tcdtw_abi_version(void) { return 4; }  // 4: planar copies carry a scale trailer (tcdtw_planar_bytes)

unsigned long long tcdtw_launch_count(void) { return g_launches.load(); }

int tcdtw_dtw_banded(int dtype, const void* a, const void* b, int64_t n_pairs, int32_t n, int32_t dims,
                     int32_t window, const void* abandon_above, void* out_distance, uint8_t* out_abandoned,
                     int64_t* out_cells, void* stream) {
    if (!dtype_ok(dtype) || !shape_ok(n_pairs, n, dims) || window < 0) return TCDTW_INVALID_INPUT;
    if (n_pairs == 0) return TCDTW_OK;
    if (!a || !b || !out_distance || !out_abandoned || !out_cells) return TCDTW_INVALID_INPUT;
    return pairs_dtw(dtype, a, b, n_pairs, n, dims, eff_window(window, n), abandon_above, out_distance,
                     out_abandoned, out_cells, S(stream));
}

int tcdtw_build_envelope(int dtype, const void* series, int64_t n_series, int32_t n, int32_t dims, int32_t window,
                         void* upper, void* lower, void* stream) {
    if (!dtype_ok(dtype) || !shape_ok(n_series, n, dims) || window < 0) return TCDTW_INVALID_INPUT;
    if (n_series == 0) return TCDTW_OK;
    if (!series || !upper || !lower) return TCDTW_INVALID_INPUT;
    return series_envelope(dtype, series, n_series, n, dims, eff_window(window, n), upper, lower, S(stream));
}

int tcdtw_lb_mv(int dtype, const void* c, const void* upper, const void* lower, int64_t n_pairs, int32_t n,
                int32_t dims, const void* abandon_above, void* out_value, uint8_t* out_abandoned, void* stream) {
    if (!dtype_ok(dtype) || !shape_ok(n_pairs, n, dims)) return TCDTW_INVALID_INPUT;
    if (n_pairs == 0) return TCDTW_OK;
    if (!c || !upper || !lower || !out_value || !out_abandoned) return TCDTW_INVALID_INPUT;
    return pairs_lb_mv(dtype, c, upper, lower, n_pairs, n, dims, abandon_above, out_value, out_abandoned, S(stream));
}

int tcdtw_lb_ad(int dtype, const void* q, const void* c, int64_t n_pairs, int32_t n, int32_t dims, int32_t window,
                const void* abandon_above, void* out_value, uint8_t* out_abandoned, void* stream) {
    if (!dtype_ok(dtype) || !shape_ok(n_pairs, n, dims) || window < 0) return TCDTW_INVALID_INPUT;
    if (n_pairs == 0) return TCDTW_OK;
    if (!q || !c || !out_value || !out_abandoned) return TCDTW_INVALID_INPUT;
    return pairs_lb_ad(dtype, q, c, n_pairs, n, dims, eff_window(window, n), abandon_above, out_value, out_abandoned,
                       S(stream));
}

int tcdtw_neighbor_steps(int dtype, const void* series, int64_t n_series, int32_t n, int32_t dims, void* out,
                         void* stream) {
    if (!dtype_ok(dtype) || !shape_ok(n_series, n, dims)) return TCDTW_INVALID_INPUT;
    if (n_series == 0 || n < 2) return TCDTW_OK;
    if (!series || !out) return TCDTW_INVALID_INPUT;
    return series_steps(dtype, series, n_series, n, dims, out, S(stream));
}

int tcdtw_ti_advance(int dtype, const void* lo, const void* up, const void* step, int64_t count, void* out_lo,
                     void* out_up, void* stream) {
    if (!dtype_ok(dtype) || count < 0) return TCDTW_INVALID_INPUT;
    if (count == 0) return TCDTW_OK;
    if (!lo || !up || !step || !out_lo || !out_up) return TCDTW_INVALID_INPUT;
    return ti_advance_elementwise(dtype, lo, up, step, count, out_lo, out_up, S(stream));
}

int tcdtw_lb_ti(int dtype, const void* q, const void* c, int64_t n_pairs, int32_t n, int32_t dims, int32_t window,
                int32_t variant, int32_t refresh_period, const void* query_steps, const void* cand_steps,
                const void* abandon_above, void* out_value, uint8_t* out_abandoned, void* stream) {
    if (!dtype_ok(dtype) || !shape_ok(n_pairs, n, dims) || window < 0) return TCDTW_INVALID_INPUT;
    if (variant < TCDTW_TI_BASIC || variant > TCDTW_TI_TIP_TOP || refresh_period < 1) return TCDTW_INVALID_INPUT;
    if (n_pairs == 0) return TCDTW_OK;
    if (!q || !c || !out_value || !out_abandoned) return TCDTW_INVALID_INPUT;
    return pairs_lb_ti(dtype, q, c, n_pairs, n, dims, eff_window(window, n), variant, refresh_period, query_steps,
                       cand_steps, abandon_above, out_value, out_abandoned, S(stream));
}

int tcdtw_build_box_sets(int dtype, const void* series, int64_t n_series, int32_t n, int32_t dims, int32_t window,
                         int32_t group_width, int32_t levels, int32_t max_boxes, double min_cell_frac,
                         const void* dim_range, void* out_lo, void* out_hi, int32_t* out_counts, void* stream) {
    if (!dtype_ok(dtype) || !shape_ok(n_series, n, dims) || window < 0) return TCDTW_INVALID_INPUT;
    if (group_width < 1 || levels < 1 || max_boxes < 1) return TCDTW_INVALID_INPUT;
    if (n_series == 0) return TCDTW_OK;
    if (!series || !out_lo || !out_hi || !out_counts) return TCDTW_INVALID_INPUT;
    return series_box_sets(dtype, series, n_series, n, dims, eff_window(window, n), group_width, levels, max_boxes,
                           min_cell_frac, dim_range, out_lo, out_hi, out_counts, S(stream));
}

int tcdtw_lb_pc(int dtype, const void* c, const void* box_lo, const void* box_hi, int64_t n_pairs, int32_t n,
                int32_t dims, int32_t n_groups, int32_t kmax, int32_t group_width, const void* abandon_above,
                void* out_value, uint8_t* out_abandoned, void* stream) {
    if (!dtype_ok(dtype) || !shape_ok(n_pairs, n, dims)) return TCDTW_INVALID_INPUT;
    if (group_width < 1 || kmax < 1 || n_groups != (n - 1) / group_width + 1) return TCDTW_INVALID_INPUT;
    if (n_pairs == 0) return TCDTW_OK;
    if (!c || !box_lo || !box_hi || !out_value || !out_abandoned) return TCDTW_INVALID_INPUT;
    return pairs_lb_pc(dtype, c, box_lo, box_hi, n_pairs, n, dims, n_groups, kmax, group_width, abandon_above,
                       out_value, out_abandoned, S(stream));
}

int tcdtw_search_workspace_size(const tcdtw_search_desc* desc, size_t* bytes) {
    if (!bytes) return TCDTW_INVALID_INPUT;
    return search_workspace_size(desc, bytes);
}

int tcdtw_search_seed(const tcdtw_search_desc* desc, const void* queries, const void* candidates,
                      const void* dim_range, void* workspace, size_t ws_bytes, void* d_best, void* stream) {
    return search_seed(desc, queries, candidates, dim_range, workspace, ws_bytes, d_best, S(stream));
}

int tcdtw_search_finish(const tcdtw_search_desc* desc, const void* queries, const void* candidates,
                        const void* dim_range, void* workspace, size_t ws_bytes, const void* d_best,
                        int64_t* best_index, double* best_distance, int64_t* counters, void* stream) {
    return search_finish(desc, queries, candidates, dim_range, workspace, ws_bytes, d_best, best_index,
                         best_distance, counters, S(stream));
}

int tcdtw_nn_search(const tcdtw_search_desc* desc, const void* queries, const void* candidates,
                    const void* dim_range, void* workspace, size_t ws_bytes, int64_t* best_index,
                    double* best_distance, int64_t* counters, void* stream) {
    int s = search_seed(desc, queries, candidates, dim_range, workspace, ws_bytes, nullptr, S(stream));
    if (s != TCDTW_OK) return s;
    return search_finish(desc, queries, candidates, dim_range, workspace, ws_bytes, nullptr, best_index,
                         best_distance, counters, S(stream));
}

int tcdtw_lb_mv_matrix(int dtype, const void* upper, const void* lower, const void* candidates, int64_t n_queries,
                       int64_t n_candidates, int32_t n, int32_t dims, void* out, void* stream) {
    if (!dtype_ok(dtype) || n_queries < 1 || n_candidates < 1 || n < 1 || dims < 1 || dims > 32)
        return TCDTW_INVALID_INPUT;
    if (!upper || !lower || !candidates || !out) return TCDTW_INVALID_INPUT;
    return lb_mv_matrix(dtype, upper, lower, candidates, n_queries, n_candidates, n, dims, out, S(stream));
}

const char* tcdtw_dtw_kernel_name(const tcdtw_search_desc* desc) {
    if (!desc) return "invalid";
    return dtw_kernel_name(desc);
}

int tcdtw_alu_probe(int dtype, int32_t blocks, int32_t iters, void* sink, double* lane_ops, void* stream) {
    if (!dtype_ok(dtype) || blocks < 1 || iters < 1 || !sink) return TCDTW_INVALID_INPUT;
    return alu_probe(dtype, blocks, iters, sink, lane_ops, S(stream));
}


int tcdtw_normalize_workspace_size(int64_t n_points, int32_t dims, size_t* bytes) {
    if (n_points < 1 || dims < 1 || !bytes) return TCDTW_INVALID_INPUT;
    *bytes = normalize_workspace_bytes(n_points, dims);
    return TCDTW_OK;
}

int tcdtw_normalize(const double* values, int64_t n_points, int32_t dims, double* out, double* mean, double* std_,
                    double* range, void* workspace, size_t ws_bytes, void* stream) {
    if (n_points < 1 || dims < 1) return TCDTW_INVALID_INPUT;  // ingest.py:62-63
    if (!values || !out || !mean || !std_ || !range) return TCDTW_INVALID_INPUT;
    if (!workspace || ws_bytes < normalize_workspace_bytes(n_points, dims)) return TCDTW_WORKSPACE_TOO_SMALL;
    return normalize_f64(values, n_points, dims, out, mean, std_, range, (double*)workspace, S(stream));
}
size_t tcdtw_planar_bytes(int dtype, int64_t n_series, int32_t n, int32_t dims) {
    if (!dtype_ok(dtype) || n_series < 0 || n < 1 || dims < 1) return 0;
    return planar_copy_bytes(dtype, n_series, n, dims);
}
int tcdtw_planarize(int dtype, const void* series, int64_t n_series, int32_t n, int32_t dims, void* out,
                    void* stream) {
    if (!dtype_ok(dtype) || n_series < 0 || n < 1 || dims < 1) return TCDTW_INVALID_INPUT;
    if (n_series > 0 && (!series || !out)) return TCDTW_INVALID_INPUT;
    if (n_series == 0) return TCDTW_OK;
    return planarize_series(dtype, series, n_series, n, dims, out, S(stream));
}

int tcdtw_shard_combine(const int64_t* records, int32_t world, int64_t n_queries, int64_t* best_index,
                        double* best_distance, void* stream) {
    if (world < 1 || n_queries < 0 || (n_queries > 0 && (!records || !best_index || !best_distance)))
        return TCDTW_INVALID_INPUT;
    return shard_combine(records, world, n_queries, best_index, best_distance, S(stream));
}
}  // extern "C"
