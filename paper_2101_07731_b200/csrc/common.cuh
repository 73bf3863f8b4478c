// common.cuh -- shared device primitives of the TC-DTW B200 path.
//
// Two arithmetic modes, selected at compile time per kernel:
//
//   EXACT  (float64 search, every per-pair API kernel): reproduces the
//          reference's float64 arithmetic bit for bit.  Each point distance
//          is sqrt(sum_p diff_p^2) with numpy's pairwise summation order for
//          a contiguous last-axis reduction (sequential for D < 8, eight
//          interleaved accumulators for 8 <= D <= 128), multiplies and adds
//          rounded separately (no FMA contraction), IEEE sqrt.  Reference:
//          core.py:104-111 ("every distance flows through this formula so
//          bound values and DTW cell costs are bit-identical").
//
//   FAST   (float32 search filter): FMA chains and sqrt.approx; every
//          pruning decision carries a relative safety margin (see
//          search.cu) and the finalists are re-scored in EXACT float64, so
//          the answers are still the reference's.
//
// Citations are file:line relative to /root/reference/pkg/src/mvdtw.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace tcdtw {

constexpr int kMaxDims = 128;  // numpy's unrecursed pairwise block (PW_BLOCKSIZE)

// +inf, usable from host code (kernel arguments) and device code
__host__ __device__ __forceinline__ float inf_of(float) { return __builtin_huge_valf(); }
__host__ __device__ __forceinline__ double inf_of(double) { return __builtin_huge_val(); }

template <typename T> __host__ __device__ __forceinline__ T dev_inf() { return inf_of(T(0)); }

// ---- correctly rounded, never contracted ----------------------------------
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double sqrt_rn(double a) { return __dsqrt_rn(a); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float sqrt_rn(float a) { return __fsqrt_rn(a); }

__device__ __forceinline__ float fast_sqrt(float a) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
    return r;
}
__device__ __forceinline__ double fast_sqrt(double a) { return __dsqrt_rn(a); }

__device__ __forceinline__ float tmin(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ double tmin(double a, double b) { return fmin(a, b); }
__device__ __forceinline__ float tmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double tmax(double a, double b) { return fmax(a, b); }

// numpy pairwise_sum of sq[0..d) (d <= DMAX <= 128), fully unrolled with
// uniform guards so register indices stay static.
template <typename T, int DMAX>
__device__ __forceinline__ T np_sum(const T (&sq)[DMAX], int d) {
    if (DMAX < 8 || d < 8) {
        T r = T(0);
#pragma unroll
        for (int p = 0; p < (DMAX < 8 ? DMAX : 8); ++p)
            if (p < d) r = add_rn(r, sq[p]);
        return r;
    }
    T r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = sq[j < DMAX ? j : 0];
    const int full = d - (d & 7);
#pragma unroll
    for (int i = 8; i + 8 <= DMAX; i += 8) {
        if (i < full) {
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = add_rn(r[j], sq[i + j]);
        }
    }
    T res = add_rn(add_rn(add_rn(r[0], r[1]), add_rn(r[2], r[3])),
                   add_rn(add_rn(r[4], r[5]), add_rn(r[6], r[7])));
#pragma unroll
    for (int i = 8; i < DMAX; ++i)
        if (i >= full && i < d) res = add_rn(res, sq[i]);
    return res;
}

// Squared point distance, EXACT order (dists_to_rows, core.py:110-111).
template <typename T, int DMAX>
__device__ __forceinline__ T sqdist_exact(const T (&a)[DMAX], const T* __restrict__ b, int d) {
    T sq[DMAX];
#pragma unroll
    for (int p = 0; p < DMAX; ++p) {
        if (p < d) {
            T df = sub_rn(a[p], b[p]);
            sq[p] = mul_rn(df, df);
        } else {
            sq[p] = T(0);
        }
    }
    return np_sum<T, DMAX>(sq, d);
}

template <typename T, int DMAX>
__device__ __forceinline__ T dist_exact(const T (&a)[DMAX], const T* __restrict__ b, int d) {
    return sqrt_rn(sqdist_exact<T, DMAX>(a, b, d));
}

// LB_MV per-point term, EXACT (envelope_deviations, lb_mv.py:91-95):
// sqrt(sum_p max(c-u,0)^2 + max(l-c,0)^2).
template <typename T, int DMAX>
__device__ __forceinline__ T lbmv_term_exact(const T (&c)[DMAX], const T* __restrict__ u,
                                             const T* __restrict__ l, int d) {
    T sq[DMAX];
#pragma unroll
    for (int p = 0; p < DMAX; ++p) {
        if (p < d) {
            T hi = tmax(sub_rn(c[p], u[p]), T(0));
            T lo = tmax(sub_rn(l[p], c[p]), T(0));
            sq[p] = add_rn(mul_rn(hi, hi), mul_rn(lo, lo));
        } else {
            sq[p] = T(0);
        }
    }
    return sqrt_rn(np_sum<T, DMAX>(sq, d));
}

// LB_PC squared box distance, EXACT (lb_pc.py:276-278).
template <typename T, int DMAX>
__device__ __forceinline__ T boxdist2_exact(const T (&c)[DMAX], const T* __restrict__ lo,
                                            const T* __restrict__ hi, int d) {
    T sq[DMAX];
#pragma unroll
    for (int p = 0; p < DMAX; ++p) {
        if (p < d) {
            T dl = tmax(sub_rn(lo[p], c[p]), T(0));
            T dh = tmax(sub_rn(c[p], hi[p]), T(0));
            sq[p] = add_rn(mul_rn(dh, dh), mul_rn(dl, dl));
        } else {
            sq[p] = T(0);
        }
    }
    return np_sum<T, DMAX>(sq, d);
}

template <typename T, int DMAX>
__device__ __forceinline__ void load_point(T (&a)[DMAX], const T* __restrict__ src, int d) {
#pragma unroll
    for (int p = 0; p < DMAX; ++p) a[p] = (p < d) ? src[p] : T(0);
}

// LB_TI propagation (ti_advance, lb_ti.py:79-86; vector form :170-176).
// kSlack is 2^-46 for float64 (the reference's _PROP_SLACK) and 2^-17 for the
// float32 filter (the same 128-ulp headroom at float32 precision).
template <typename T> struct TiSlack;
template <> struct TiSlack<double> { static constexpr double v = 1.4210854715202004e-14; };  // 2^-46
template <> struct TiSlack<float> { static constexpr float v = 7.62939453125e-06f; };        // 2^-17

template <typename T>
__device__ __forceinline__ void ti_advance(T& lo, T& up, T s) {
    if (s == T(0)) return;
    T a = sub_rn(lo, s), b = sub_rn(s, up);
    T base = tmax(tmax(a, b), T(0));
    T t = add_rn(up, s);
    T pad = mul_rn(t, TiSlack<T>::v);
    lo = tmax(sub_rn(base, pad), T(0));
    up = add_rn(t, pad);
}

// non-negative float <-> ordered integer bits (for atomicMin on distances)
__device__ __forceinline__ unsigned int ord_bits(float x) { return __float_as_uint(x); }
__device__ __forceinline__ unsigned long long ord_bits(double x) {
    return (unsigned long long)__double_as_longlong(x);
}
__device__ __forceinline__ float from_bits(unsigned int b, float) { return __uint_as_float(b); }
__device__ __forceinline__ double from_bits(unsigned long long b, double) {
    return __longlong_as_double((long long)b);
}

template <typename T> struct BitsOf;
template <> struct BitsOf<float> { using type = unsigned int; };
template <> struct BitsOf<double> { using type = unsigned long long; };

template <typename T>
__device__ __forceinline__ T atomic_min_nonneg(T* addr, T v) {
    using B = typename BitsOf<T>::type;
    B old = atomicMin(reinterpret_cast<B*>(addr), ord_bits(v));
    return from_bits(old, T(0));
}

template <typename T>
__device__ __forceinline__ T load_volatile(const T* p) {
    return *reinterpret_cast<const volatile T*>(p);
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

}  // namespace tcdtw
