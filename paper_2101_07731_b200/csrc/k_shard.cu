// k_shard.cu -- the cross-shard combine of the sharded search.
//
// Every rank all-gathers one 16-byte record per query, (float64 distance
// bits, global index), in ONE collective; this kernel then reduces the
// (world, Q) records of every query to the lexicographic (distance, index)
// minimum -- the reference's lowest-index tie rule (search.py:173) across
// shards.  A record with index -1 (the shard pruned every candidate against
// a better d_best from another shard) never wins.  Non-negative IEEE doubles
// order like their bit patterns, so the comparison is on integers.
#include <cuda_runtime.h>

#include "dispatch.cuh"

namespace tcdtw {

static __global__ void shard_combine_kernel(const long long* __restrict__ rec, int world, int64_t Q,
                                            int64_t* __restrict__ best_index, double* __restrict__ best_distance) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < Q; q += (int64_t)gridDim.x * blockDim.x) {
        long long bd = 0x7ff0000000000000LL;  // +inf
        long long bi = -1;
        for (int r = 0; r < world; ++r) {
            const long long d = rec[((int64_t)r * Q + q) * 2];
            const long long i = rec[((int64_t)r * Q + q) * 2 + 1];
            if (i < 0) continue;
            if (bi < 0 || d < bd || (d == bd && i < bi)) {
                bd = d;
                bi = i;
            }
        }
        best_index[q] = bi;
        best_distance[q] = __longlong_as_double(bd);
    }
}

int shard_combine(const int64_t* rec, int world, int64_t Q, int64_t* best_index, double* best_distance,
                  cudaStream_t st) {
    if (Q <= 0) return TCDTW_OK;
    shard_combine_kernel<<<grid_for(Q, 256), 256, 0, st>>>(reinterpret_cast<const long long*>(rec), world, Q,
                                                           best_index, best_distance);
    return launch_status();
}

}  // namespace tcdtw
