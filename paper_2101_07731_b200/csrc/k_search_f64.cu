// k_search_f64.cu -- double instantiation of the batched search (search_impl.cuh).
#include "search_impl.cuh"

namespace tcdtw {

int search_seed_f64(const tcdtw_search_desc* dsc, const Plan& p, const void* q, const void* c, const void* dr,
                     void* ws, void* dbest, cudaStream_t st) {
    return dispatch_search_dims<double>(p.d, SeedOp{}, dsc, p, q, c, dr, ws, dbest, st);
}

int search_finish_f64(const tcdtw_search_desc* dsc, const Plan& p, const void* q, const void* c, const void* dr,
                       void* ws, const void* dbest, int64_t* bi, double* bd, int64_t* ctr, cudaStream_t st) {
    return dispatch_search_dims<double>(p.d, FinishOp{}, dsc, p, q, c, dr, ws, dbest, bi, bd, ctr, st);
}

struct MatrixOp_f64 {
    template <typename T, int DM>
    int run(const void* up, const void* lo, const void* cands, int64_t Q, int64_t N, int n, int d, void* out,
            cudaStream_t st) {
        // planar operands in a stream-ordered temporary
        T* tmp = nullptr;
        const size_t qs = (size_t)Q * n * d, cs = (size_t)N * n * d;
        if (cudaMallocAsync(&tmp, (2 * qs + cs) * sizeof(T), st) != cudaSuccess) return TCDTW_CUDA_ERROR;
        int s = planarize<T>((const T*)up, Q, n * d, tmp, st);
        if (s == TCDTW_OK) s = planarize<T>((const T*)lo, Q, n * d, tmp + qs, st);
        if (s == TCDTW_OK) s = planarize<T>((const T*)cands, N, n * d, tmp + 2 * qs, st);
        if (s == TCDTW_OK)
            s = launch_lbmv_matrix<T, DM, sizeof(T) == 8>(tmp, tmp + qs, nullptr, tmp + 2 * qs, Q, N, n, d, (T*)out,
                                                          nullptr, st);
        cudaFreeAsync(tmp, st);
        return s;
    }
};

int lb_mv_matrix_f64(const void* up, const void* lo, const void* cands, int64_t Q, int64_t N, int n, int d,
                      void* out, cudaStream_t st) {
    return dispatch_search_dims<double>(d, MatrixOp_f64{}, up, lo, cands, Q, N, n, d, out, st);
}

}  // namespace tcdtw
