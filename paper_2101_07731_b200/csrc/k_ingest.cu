// k_ingest.cu -- device-side dataset normalisation.
//
// normalize (ingest.py:245-261): missing values (NaN) become raw zeros and
// enter the statistics as zeros; each dimension is z-normalised with the
// population mean and standard deviation over every point of every series;
// zero-variance dimensions map to all-zeros; the post-normalisation range
// (max - min, ingest.py:235-237) of each dimension is recorded for the
// clustering bound.  float64 throughout.
//
// Three HBM streams over the (points, d) array: sum, centred squares, and the
// normalised write with its per-dimension min/max.  Each is coalesced: a
// block walks its contiguous range of points T' = floor(256/d)*d elements at
// a time, so thread t always sees dimension t % d.  The reductions are
// deterministic (fixed block ranges, fixed in-block and cross-block orders)
// but are tree sums, not numpy's sequential axis-0 accumulation, so the
// statistics agree with the reference to rounding (tests: 1e-12 of the
// dimension's scale), not bit for bit.  Given the statistics, each value is
// the reference's (x - mean) / std, correctly rounded.

#include <cuda_runtime.h>

#include "common.cuh"
#include "dispatch.cuh"

namespace tcdtw {

constexpr int kNormBlocks = 148 * 4;
constexpr int kNormThreads = 256;

enum { kNormSum = 0, kNormVar = 1, kNormApply = 2 };

template <int MODE>
__global__ void __launch_bounds__(kNormThreads) norm_pass_kernel(const double* __restrict__ x, int64_t points, int d,
                                                                 const double* __restrict__ mean,
                                                                 const double* __restrict__ stdv,
                                                                 double* __restrict__ out, double* __restrict__ part,
                                                                 double* __restrict__ pmin,
                                                                 double* __restrict__ pmax) {
    __shared__ double red[kNormThreads], rmn[kNormThreads], rmx[kNormThreads];
    const int TP = (kNormThreads / d) * d;  // active threads; thread t <-> dimension t % d
    const int t = threadIdx.x;
    const int k = t % d;
    const int64_t per = (points + gridDim.x - 1) / gridDim.x;
    const int64_t p0 = (int64_t)blockIdx.x * per;
    const int64_t p1 = p0 + per < points ? p0 + per : points;
    double acc = 0.0, mn = dev_inf<double>(), mx = -dev_inf<double>();
    if (t < TP && p0 < p1) {
        const double m = MODE != kNormSum ? mean[k] : 0.0;
        const double s = MODE == kNormApply ? stdv[k] : 1.0;
        for (int64_t e = p0 * d + t; e < p1 * d; e += TP) {
            double v = x[e];
            v = v != v ? 0.0 : v;  // missing -> raw zero (ingest.py:256)
            if (MODE == kNormSum) {
                acc = __dadd_rn(acc, v);
            } else if (MODE == kNormVar) {
                const double c = __dsub_rn(v, m);
                acc = __dadd_rn(acc, __dmul_rn(c, c));
            } else {
                const double z = s > 0.0 ? __ddiv_rn(__dsub_rn(v, m), s) : 0.0;  // ingest.py:257-259
                out[e] = z;
                mn = z < mn ? z : mn;
                mx = z > mx ? z : mx;
            }
        }
    }
    red[t] = acc;
    rmn[t] = mn;
    rmx[t] = mx;
    __syncthreads();
    if (t < d) {  // fixed order over the threads of dimension t
        double s = 0.0, a = dev_inf<double>(), b = -dev_inf<double>();
        for (int u = t; u < TP; u += d) {
            s = __dadd_rn(s, red[u]);
            a = rmn[u] < a ? rmn[u] : a;
            b = rmx[u] > b ? rmx[u] : b;
        }
        part[(int64_t)blockIdx.x * d + t] = s;
        if (MODE == kNormApply) {
            pmin[(int64_t)blockIdx.x * d + t] = a;
            pmax[(int64_t)blockIdx.x * d + t] = b;
        }
    }
}

template <int MODE>
__global__ void norm_final_kernel(int blocks, int64_t points, int d, const double* __restrict__ part,
                                  const double* __restrict__ pmin, const double* __restrict__ pmax,
                                  double* __restrict__ res) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= d) return;
    if (MODE == kNormApply) {  // range of the normalised values
        double a = dev_inf<double>(), b = -dev_inf<double>();
        for (int bl = 0; bl < blocks; ++bl) {
            a = pmin[(int64_t)bl * d + k] < a ? pmin[(int64_t)bl * d + k] : a;
            b = pmax[(int64_t)bl * d + k] > b ? pmax[(int64_t)bl * d + k] : b;
        }
        res[k] = __dsub_rn(b, a);
        return;
    }
    double s = 0.0;
    for (int bl = 0; bl < blocks; ++bl) s = __dadd_rn(s, part[(int64_t)bl * d + k]);
    const double q = __ddiv_rn(s, (double)points);
    res[k] = MODE == kNormSum ? q : __dsqrt_rn(q);  // mean; population std
}

size_t normalize_workspace_bytes(int d) { return (size_t)3 * kNormBlocks * d * sizeof(double); }

int normalize_f64(const double* x, int64_t points, int d, double* out, double* mean, double* stdv, double* range,
                  double* ws, cudaStream_t st) {
    double* part = ws;
    double* pmin = ws + (size_t)kNormBlocks * d;
    double* pmax = pmin + (size_t)kNormBlocks * d;
    const int blocks = points < kNormBlocks ? (int)points : kNormBlocks;
    const int fb = (d + 127) / 128;
    int rc = TCDTW_OK;
    auto chk = [&]() {
        const int r = launch_status();  // counts each launch
        if (rc == TCDTW_OK) rc = r;
    };
    norm_pass_kernel<kNormSum><<<blocks, kNormThreads, 0, st>>>(x, points, d, nullptr, nullptr, nullptr, part, nullptr,
                                                                nullptr);
    chk();
    norm_final_kernel<kNormSum><<<fb, 128, 0, st>>>(blocks, points, d, part, nullptr, nullptr, mean);
    chk();
    norm_pass_kernel<kNormVar><<<blocks, kNormThreads, 0, st>>>(x, points, d, mean, nullptr, nullptr, part, nullptr,
                                                                nullptr);
    chk();
    norm_final_kernel<kNormVar><<<fb, 128, 0, st>>>(blocks, points, d, part, nullptr, nullptr, stdv);
    chk();
    norm_pass_kernel<kNormApply><<<blocks, kNormThreads, 0, st>>>(x, points, d, mean, stdv, out, part, pmin, pmax);
    chk();
    norm_final_kernel<kNormApply><<<fb, 128, 0, st>>>(blocks, points, d, part, pmin, pmax, range);
    chk();
    return rc;
}

}  // namespace tcdtw
