// k_ingest.cu -- device-side dataset normalisation,
// bit-identical to the reference's numpy computation.
//
// normalize (ingest.py:245-261): missing values (NaN) become raw zeros and
// enter the statistics as zeros; mean = flat.sum(axis=0) / M and
// std = sqrt(((flat - mean)**2).sum(axis=0) / M) over the M = S*n points;
// each value becomes (x - mean) / std, zero-variance dimensions all-zeros;
// the post-normalisation range (max - min, ingest.py:235-237) is recorded.
//
// Floating-point sums depend on their order, so the two sums follow the
// order numpy's axis-0 reduction of a C-contiguous (M, D) array uses
// (measured on numpy 2.3.5):
//   * D >= 2: the reduced axis is the outer loop, so each dimension is a
//     plain running sum acc = acc + x[i] over i = 0..M-1.  A strictly
//     sequential chain cannot be split, so one warp owns one dimension:
//     lanes fetch 32 consecutive rows per round (the next round in flight)
//     and every lane folds the 32 values, broadcast by shuffles, into the
//     same running sum.  The chain runs at one DADD latency per point.
//   * D == 1: the column is contiguous and numpy uses its pairwise
//     summation: blocks of <= 128 values summed with 8 interleaved
//     accumulators, combined by a binary recursion that splits n at
//     n/2 rounded down to a multiple of 8.  The recursion tree is
//     evaluated level by level from the deepest: a thread per tree slot
//     walks its path from the root to find its node, sums it if it is a
//     block, else adds its two children.
// Every operation is an explicitly rounded intrinsic (no contraction), so
// the statistics and the normalised values equal numpy's bit for bit.

#include <cuda_runtime.h>

#include "common.cuh"
#include "dispatch.cuh"

namespace tcdtw {

constexpr int kPwBlock = 128;  // numpy PW_BLOCKSIZE
constexpr int kNormBlocks = 148 * 4;
constexpr int kNormThreads = 256;

// element i of the summed array: the value (NaN -> 0), or its centred square
template <bool SQ>
__device__ __forceinline__ double summand(const double* __restrict__ x, int64_t e, double mean) {
    double v = x[e];
    v = v != v ? 0.0 : v;  // ingest.py:256
    if (SQ) {
        const double c = __dsub_rn(v, mean);
        v = __dmul_rn(c, c);
    }
    return v;
}

// ---------------------------------------------------------------- D >= 2
template <bool SQ>
__global__ void __launch_bounds__(32) seq_colsum_kernel(const double* __restrict__ x, int64_t M, int D,
                                                        const double* __restrict__ mean, double* __restrict__ res) {
    const int k = blockIdx.x, lane = threadIdx.x;
    const double m = SQ ? mean[k] : 0.0;
    double acc = 0.0;  // numpy starts the reduction from the identity
    double cur = lane < M ? summand<SQ>(x, (int64_t)lane * D + k, m) : 0.0;
    for (int64_t r0 = 0; r0 < M; r0 += 32) {
        const int64_t nr = r0 + 32 + lane;
        const double nxt = nr < M ? summand<SQ>(x, nr * D + k, m) : 0.0;  // next round in flight
        const int cnt = M - r0 < 32 ? (int)(M - r0) : 32;
        if (cnt == 32) {
#pragma unroll
            for (int j = 0; j < 32; ++j) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, cur, j));
        } else {
            for (int j = 0; j < cnt; ++j) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, cur, j));
        }
        cur = nxt;
    }
    if (lane == 0) {
        const double q = __ddiv_rn(acc, (double)M);
        res[k] = SQ ? __dsqrt_rn(q) : q;  // mean; population std
    }
}

// ---------------------------------------------------------------- D == 1
__host__ __device__ inline int64_t pw_left(int64_t n) {
    const int64_t h = n / 2;
    return h - h % 8;
}

// depth of the deepest block: the all-right path holds the largest nodes
inline int pw_depth(int64_t n) {
    int k = 0;
    while (n > kPwBlock) {
        n -= pw_left(n);
        ++k;
    }
    return k;
}

// numpy pairwise_sum of a block of n <= 128 values starting at element off
template <bool SQ>
__device__ double pw_block(const double* __restrict__ x, int64_t off, int64_t n, double m) {
    if (n < 8) {
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) s = __dadd_rn(s, summand<SQ>(x, off + i, m));
        return s;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = summand<SQ>(x, off + j, m);
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], summand<SQ>(x, off + i + j, m));
    }
    double s = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) s = __dadd_rn(s, summand<SQ>(x, off + i, m));
    return s;
}

// Tree slot s of level `level` (path bits, MSB = first branch).  Writes the
// node's sum to lv[s]; children sit in lv_next[2s], lv_next[2s+1].
template <bool SQ>
__global__ void pw_level_kernel(const double* __restrict__ x, int64_t M, int level,
                                const double* __restrict__ mean, double* __restrict__ lv,
                                const double* __restrict__ lv_next) {
    const int64_t slot = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (slot >= ((int64_t)1 << level)) return;
    const double m = SQ ? mean[0] : 0.0;
    int64_t off = 0, n = M;
    for (int b = level - 1; b >= 0; --b) {
        if (n <= kPwBlock) return;  // an ancestor is a block: no node here
        const int64_t l = pw_left(n);
        if ((slot >> b) & 1) {
            off += l;
            n -= l;
        } else {
            n = l;
        }
    }
    lv[slot] = n <= kPwBlock ? pw_block<SQ>(x, off, n, m) : __dadd_rn(lv_next[2 * slot], lv_next[2 * slot + 1]);
}

__global__ void pw_finish_kernel(const double* __restrict__ root, int64_t M, bool sq, double* __restrict__ res) {
    const double q = __ddiv_rn(root[0], (double)M);  // numpy: the reduction starts from 0.0; 0 + s == s
    res[0] = sq ? __dsqrt_rn(q) : q;
}

// -------------------------------------------------------------- apply pass
__global__ void __launch_bounds__(kNormThreads) norm_apply_kernel(const double* __restrict__ x, int64_t points, int d,
                                                                  const double* __restrict__ mean,
                                                                  const double* __restrict__ stdv,
                                                                  double* __restrict__ out, double* __restrict__ pmin,
                                                                  double* __restrict__ pmax) {
    __shared__ double rmn[kNormThreads], rmx[kNormThreads];
    const int TP = (kNormThreads / d) * d;  // active threads; thread t <-> dimension t % d
    const int t = threadIdx.x;
    const int k = t % d;
    const int64_t per = (points + gridDim.x - 1) / gridDim.x;
    const int64_t p0 = (int64_t)blockIdx.x * per;
    const int64_t p1 = p0 + per < points ? p0 + per : points;
    double mn = dev_inf<double>(), mx = -dev_inf<double>();
    if (t < TP && p0 < p1) {
        const double m = mean[k], s = stdv[k];
        for (int64_t e = p0 * d + t; e < p1 * d; e += TP) {
            double v = x[e];
            v = v != v ? 0.0 : v;
            const double z = s == 0.0 ? 0.0 : __ddiv_rn(__dsub_rn(v, m), s > 0.0 ? s : 1.0);  // ingest.py:257-259
            out[e] = z;
            mn = z < mn ? z : mn;
            mx = z > mx ? z : mx;
        }
    }
    rmn[t] = mn;
    rmx[t] = mx;
    __syncthreads();
    if (t < d) {  // min/max are order-free
        double a = dev_inf<double>(), b = -dev_inf<double>();
        for (int u = t; u < TP; u += d) {
            a = rmn[u] < a ? rmn[u] : a;
            b = rmx[u] > b ? rmx[u] : b;
        }
        pmin[(int64_t)blockIdx.x * d + t] = a;
        pmax[(int64_t)blockIdx.x * d + t] = b;
    }
}

__global__ void norm_range_kernel(int blocks, int d, const double* __restrict__ pmin, const double* __restrict__ pmax,
                                  double* __restrict__ range) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= d) return;
    double a = dev_inf<double>(), b = -dev_inf<double>();
    for (int bl = 0; bl < blocks; ++bl) {
        a = pmin[(int64_t)bl * d + k] < a ? pmin[(int64_t)bl * d + k] : a;
        b = pmax[(int64_t)bl * d + k] > b ? pmax[(int64_t)bl * d + k] : b;
    }
    range[k] = __dsub_rn(b, a);
}

// d > kNormThreads: a block per dimension, its column read with a stride
__global__ void __launch_bounds__(kNormThreads) norm_apply_wide_kernel(const double* __restrict__ x, int64_t points,
                                                                       int d, const double* __restrict__ mean,
                                                                       const double* __restrict__ stdv,
                                                                       double* __restrict__ out,
                                                                       double* __restrict__ range) {
    __shared__ double rmn[kNormThreads], rmx[kNormThreads];
    const int k = blockIdx.x, t = threadIdx.x;
    const double m = mean[k], s = stdv[k];
    double mn = dev_inf<double>(), mx = -dev_inf<double>();
    for (int64_t p = t; p < points; p += kNormThreads) {
        const int64_t e = p * d + k;
        double v = x[e];
        v = v != v ? 0.0 : v;
        const double z = s == 0.0 ? 0.0 : __ddiv_rn(__dsub_rn(v, m), s > 0.0 ? s : 1.0);
        out[e] = z;
        mn = z < mn ? z : mn;
        mx = z > mx ? z : mx;
    }
    rmn[t] = mn;
    rmx[t] = mx;
    __syncthreads();
    if (t == 0) {
        double a = dev_inf<double>(), b = -dev_inf<double>();
        for (int u = 0; u < kNormThreads; ++u) {
            a = rmn[u] < a ? rmn[u] : a;
            b = rmx[u] > b ? rmx[u] : b;
        }
        range[k] = __dsub_rn(b, a);
    }
}

static size_t pw_slots(int64_t M) { return ((size_t)2 << pw_depth(M)); }  // all levels 0..depth

size_t normalize_workspace_bytes(int64_t points, int d) {
    size_t b = (size_t)2 * kNormBlocks * (d > kNormThreads ? 1 : d) * sizeof(double);
    if (d == 1) b += pw_slots(points) * sizeof(double);
    return b;
}

template <bool SQ>
static void pairwise_sum(const double* x, int64_t M, const double* mean, double* tree, double* res, cudaStream_t st,
                         int& rc) {
    const int depth = pw_depth(M);
    // level k occupies tree[2^k - 1 .. 2^(k+1) - 2]
    for (int k = depth; k >= 0; --k) {
        const int64_t slots = (int64_t)1 << k;
        double* lv = tree + (slots - 1);
        const double* nxt = tree + (2 * slots - 1);
        const int threads = 128;
        pw_level_kernel<SQ><<<(unsigned)((slots + threads - 1) / threads), threads, 0, st>>>(x, M, k, mean, lv, nxt);
        const int r = launch_status();
        if (rc == TCDTW_OK) rc = r;
    }
    pw_finish_kernel<<<1, 1, 0, st>>>(tree, M, SQ, res);
    const int r = launch_status();
    if (rc == TCDTW_OK) rc = r;
}

int normalize_f64(const double* x, int64_t points, int d, double* out, double* mean, double* stdv, double* range,
                  double* ws, cudaStream_t st) {
    const int dw = d > kNormThreads ? 1 : d;
    double* pmin = ws;
    double* pmax = ws + (size_t)kNormBlocks * dw;
    double* tree = pmax + (size_t)kNormBlocks * dw;
    int rc = TCDTW_OK;
    auto chk = [&]() {
        const int r = launch_status();  // counts each launch
        if (rc == TCDTW_OK) rc = r;
    };
    if (d == 1) {
        pairwise_sum<false>(x, points, nullptr, tree, mean, st, rc);
        pairwise_sum<true>(x, points, mean, tree, stdv, st, rc);
    } else {
        seq_colsum_kernel<false><<<d, 32, 0, st>>>(x, points, d, nullptr, mean);
        chk();
        seq_colsum_kernel<true><<<d, 32, 0, st>>>(x, points, d, mean, stdv);
        chk();
    }
    if (d > kNormThreads) {
        norm_apply_wide_kernel<<<d, kNormThreads, 0, st>>>(x, points, d, mean, stdv, out, range);
        chk();
        return rc;
    }
    const int blocks = points < kNormBlocks ? (int)points : kNormBlocks;
    norm_apply_kernel<<<blocks, kNormThreads, 0, st>>>(x, points, d, mean, stdv, out, pmin, pmax);
    chk();
    norm_range_kernel<<<(d + 127) / 128, 128, 0, st>>>(blocks, d, pmin, pmax, range);
    chk();
    return rc;
}

}  // namespace tcdtw
