// k_search.cu -- host entry points of the batched search (search_impl.cuh);
// the per-dtype template instantiations live in k_search_f32.cu / _f64.cu.
#include "search_impl.cuh"

namespace tcdtw {

int search_seed_f32(const tcdtw_search_desc*, const Plan&, const void*, const void*, const void*, void*, void*,
                    cudaStream_t);
int search_seed_f64(const tcdtw_search_desc*, const Plan&, const void*, const void*, const void*, void*, void*,
                    cudaStream_t);
int search_finish_f32(const tcdtw_search_desc*, const Plan&, const void*, const void*, const void*, void*,
                      const void*, int64_t*, double*, int64_t*, cudaStream_t);
int search_finish_f64(const tcdtw_search_desc*, const Plan&, const void*, const void*, const void*, void*,
                      const void*, int64_t*, double*, int64_t*, cudaStream_t);
int lb_mv_matrix_f32(const void*, const void*, const void*, int64_t, int64_t, int, int, void*, cudaStream_t);
int lb_mv_matrix_f64(const void*, const void*, const void*, int64_t, int64_t, int, int, void*, cudaStream_t);

int search_workspace_size(const tcdtw_search_desc* dsc, size_t* bytes) {
    Plan p;
    TRY(make_plan(dsc, &p));
    *bytes = p.total;
    return TCDTW_OK;
}

static int check_ws(const Plan& p, void* ws, size_t ws_bytes) {
    if (!ws || ws_bytes < p.total) return TCDTW_WORKSPACE_TOO_SMALL;
    return TCDTW_OK;
}

int search_seed(const tcdtw_search_desc* dsc, const void* q, const void* c, const void* dr, void* ws,
                size_t ws_bytes, void* dbest, cudaStream_t st) {
    Plan p;
    TRY(make_plan(dsc, &p));
    TRY(check_ws(p, ws, ws_bytes));
    if (!q || !c) return TCDTW_INVALID_INPUT;
    if (p.d > 32) return TCDTW_NOT_SUPPORTED;
    return p.exact ? search_seed_f64(dsc, p, q, c, dr, ws, dbest, st) : search_seed_f32(dsc, p, q, c, dr, ws, dbest, st);
}

int search_finish(const tcdtw_search_desc* dsc, const void* q, const void* c, const void* dr, void* ws,
                  size_t ws_bytes, const void* dbest, int64_t* bi, double* bd, int64_t* ctr, cudaStream_t st) {
    Plan p;
    TRY(make_plan(dsc, &p));
    TRY(check_ws(p, ws, ws_bytes));
    if (!q || !c || !bi || !bd) return TCDTW_INVALID_INPUT;
    if (p.d > 32) return TCDTW_NOT_SUPPORTED;
    return p.exact ? search_finish_f64(dsc, p, q, c, dr, ws, dbest, bi, bd, ctr, st)
                   : search_finish_f32(dsc, p, q, c, dr, ws, dbest, bi, bd, ctr, st);
}

int lb_mv_matrix(int dtype, const void* up, const void* lo, const void* cands, int64_t Q, int64_t N, int n, int d,
                 void* out, cudaStream_t st) {
    if (dtype == TCDTW_F64) return lb_mv_matrix_f64(up, lo, cands, Q, N, n, d, out, st);
    if (dtype == TCDTW_F32) return lb_mv_matrix_f32(up, lo, cands, Q, N, n, d, out, st);
    return TCDTW_INVALID_INPUT;
}

// Which DTW kernel the survivors pass runs for this shape (launch_dtw's
// order; assumes 16-byte aligned candidates).
const char* dtw_kernel_name(const tcdtw_search_desc* dsc) {
    Plan p;
    if (make_plan(dsc, &p) != TCDTW_OK) return "invalid";
    if (!p.exact) {
        const int r = laner_any_rows_shape(p.n, p.d, p.B);
        if (r == 4) return "dtw_laner_kernel<R=4>";
        if (r == 2) return "dtw_laner_kernel<R=2>";
    }
    bool lane = false;
#define TCDTW_NAME_CASE(TT, DD, BB) lane = lane || ((sizeof(TT) == 8) == p.exact && p.d == DD && p.B == BB);
    TCDTW_LANE_SPECS(TCDTW_NAME_CASE)
#undef TCDTW_NAME_CASE
    if (lane) return "dtw_lane_kernel";
    if (p.B <= 64) return "dtw_tpp_kernel";
    bool wd = false;
#define TCDTW_WAVE_NAME(DD) wd = wd || p.d == DD;
    TCDTW_WAVE_DIMS(TCDTW_WAVE_NAME)
#undef TCDTW_WAVE_NAME
    if (wd) return "dtw_wave_d_kernel";
    return "dtw_wave_kernel";
}

int planarize_series(int dtype, const void* series, int64_t ns, int n, int d, void* out, cudaStream_t st) {
    // elements + trailer {sigma, 1/sigma} (planar_bytes): float32 copies are scaled
    if (dtype == TCDTW_F64) {
        float* scale = reinterpret_cast<float*>(reinterpret_cast<char*>(out) + planar_trailer_off(ns, n * d, 8));
        planar_scale_kernel<<<1, 1, 0, st>>>(nullptr, scale);
        return planarize<double>((const double*)series, ns, n * d, (double*)out, st);
    }
    if (dtype == TCDTW_F32) {
        float* scale = reinterpret_cast<float*>(reinterpret_cast<char*>(out) + planar_trailer_off(ns, n * d, 4));
        const int rc = planar_scale((const float*)series, ns * n * d, scale, st);
        if (rc != TCDTW_OK) return rc;
        return planarize_tiled((const float*)series, ns, n * d, (float*)out, st, scale);
    }
    return TCDTW_INVALID_INPUT;
}

size_t planar_copy_bytes(int dtype, int64_t ns, int n, int d) {
    return planar_bytes(ns, n * d, dtype == TCDTW_F64 ? 8 : 4);
}

int alu_probe(int dtype, int blocks, int iters, void* sink, double* lane_ops, cudaStream_t st) {
    if (dtype == TCDTW_F64) alu_probe_kernel<double><<<blocks, 256, 0, st>>>(iters, (double*)sink);
    else alu_probe_kernel<float><<<blocks, 256, 0, st>>>(iters, (float*)sink);
    if (lane_ops) *lane_ops = (double)blocks * 256.0 * iters * 16.0 * 8.0;
    return launch_status();
}

}  // namespace tcdtw
