// dispatch.cuh -- runtime (dtype, dims) -> template instantiation.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>

#include "../../include/tcdtw.h"

namespace tcdtw {

// Calls F.template run<T, DMAX>(args...) for the smallest register bucket
// that holds `dims`.
#define TCDTW_DIMS_BUCKETS(X) X(4) X(8) X(16) X(32) X(64) X(128)

template <typename T, typename F, typename... Args>
int dispatch_dims(int dims, F&& f, Args&&... args) {
#define TCDTW_CASE(DM) \
    if (dims <= DM) return f.template run<T, DM>(args...);
    TCDTW_DIMS_BUCKETS(TCDTW_CASE)
#undef TCDTW_CASE
    return TCDTW_NOT_SUPPORTED;  // a valid input the register buckets do not cover
}

template <typename F, typename... Args>
int dispatch_dtype_dims(int dtype, int dims, F&& f, Args&&... args) {
    if (dtype == TCDTW_F64) return dispatch_dims<double>(dims, f, args...);
    if (dtype == TCDTW_F32) return dispatch_dims<float>(dims, f, args...);
    return TCDTW_INVALID_INPUT;
}

inline int cuda_status(cudaError_t e) { return e == cudaSuccess ? TCDTW_OK : TCDTW_CUDA_ERROR; }

// Kernel launches issued by this library (reported by bench.py as
// gpu_launches).  Monotone statistics counter; no other global state.
inline std::atomic<unsigned long long> g_launches{0};

inline int launch_status() {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TCDTW_OK : TCDTW_CUDA_ERROR;
}

inline int grid_for(int64_t n, int block) {
    int64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > 2147483647LL) g = 2147483647LL;
    return (int)g;
}

}  // namespace tcdtw
