#pragma once
// search_impl.cuh -- the batched 1-NN search (nn_search, search.py:75-180) on B200.
//
// Pipeline per call (a batch of Q queries against one shard of N candidates):
//
//   prep      query envelopes (lb_mv.py:74-88), planar copies for tiling,
//             box sets (lb_pc.py:239-261) / query steps (lb_ti.py:51-55)
//   lb_mv     LB_MV of every (query, candidate) pair: a register-tiled
//             ALU-bound kernel over planar [t][p][*] operands staged in shared
//             memory (lb_mv.py:91-107) -> LB matrix (Q, N) in HBM
//   seeds     per query the S smallest bounds; their exact DTWs seed the
//             device-resident best-so-far d_best (replaces the reference's
//             seed from candidate 0, search.py:127-133)
//   compact   survivors LB <= thr(d_best), written per query in candidate
//             order (prune rule search.py:144, made order-free, see below)
//   advanced  LB_PC / LB_TI / LB_AD on survivors in the trigger band
//             e*d_best < LB_MV (search.py:147-165)
//   dtw       banded DTW of the survivors with early abandoning against the
//             live d_best (atomicMin), thread-per-pair (band in registers)
//             for 2W+1 <= 64, warp-per-pair anti-diagonal wavefront beyond
//   finalize  lexicographic (distance, index) minimum; in float32 the
//             finalists are re-scored in EXACT float64.
//
// Order-free exactness.  The reference returns the linear-scan argmin with
// the lowest index winning ties (search.py:144,163,173; dtw.py:97).  Here:
//   EXACT (float64): every bound and DTW value is bit-identical to the
//     reference's, so pruning with strict '>' against d_best can never drop
//     a candidate whose DTW is <= the final best, and the tie rule is applied
//     by a final lexicographic reduction over completed DTWs.
//   FAST (float32): every decision carries a margin eps = (2n+d+16)*2^-23
//     covering float32 rounding of bounds and DTW: prune / abandon iff
//     value > d_best * (1+3 eps); candidates whose float32 DTW is within
//     (1+2.5 eps) of the best are re-scored in EXACT float64 on the same
//     (float32) inputs, and the lexicographic minimum of those is returned.
//     The answer is therefore the reference's on the float32-rounded data.

#include <cub/device/device_scan.cuh>

#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "dispatch.cuh"

namespace tcdtw {

// host wrappers defined in k_pairs.cu
int series_envelope(int dtype, const void* s, int64_t ns, int n, int d, int w, void* u, void* l,
                    cudaStream_t st);
int series_steps(int dtype, const void* s, int64_t ns, int n, int d, void* out, cudaStream_t st);
int series_box_sets(int dtype, const void* s, int64_t ns, int n, int d, int w, int gw, int levels, int K,
                    double mcf, const void* dr, void* olo, void* ohi, int32_t* counts, cudaStream_t st);

constexpr int kSeedMax = 32;
constexpr int kChunk = 2048;  // compaction chunk (candidates per block)
// Survivor lists are laid out chunk-major: segment (chunk, query) at index
// chunk * Q + q.  Work tiles are consumed in that order, so the warps of the
// whole GPU work on one candidate chunk (kChunk series, a few MB) across all
// queries at a time and read the candidate rows from L2, not HBM.
constexpr int kTile = 32;     // survivors per work tile (one per lane)

// ----------------------------------------------------------- small helpers
__host__ __device__ inline int64_t cells_upto(int r, int n, int w) {
    // sum_{i=0}^{r} (min(n-1, i+w) - max(0, i-w) + 1), dtw.py:96
    const int64_t R = r;
    int64_t a = n - 1 - w;  // last i with i + w <= n-1
    if (a > R) a = R;
    int64_t s1 = 0;
    if (a >= 0) s1 = (a + 1) * (int64_t)w + a * (a + 1) / 2;
    const int64_t s2 = (R - a) * (int64_t)(n - 1);
    int64_t s3 = 0;
    if (R >= w) s3 = (R - w) * (R - w + 1) / 2;
    return (R + 1) + s1 + s2 - s3;
}

// Float32 decisions carry an affine margin: threshold = value * mult + add.
// `mult` covers float32 arithmetic on the inputs as given; `add` (device
// pointer, nullptr = 0) covers the rounding of float64 inputs to float32
// when the float32 filter runs on float64 data (TCDTW_FLAG_F32_FILTER):
// add[0] for prune / abandon thresholds, add[1] for finalists.
struct Margins {
    float prune;  // d_best multiplier for prune / abandon thresholds
    float fin;    // best multiplier for finalists
    const float* add;
};

template <typename T>
__device__ __forceinline__ T scale_up(T v, const Margins& mg);
template <>
__device__ __forceinline__ float scale_up<float>(float v, const Margins& mg) {
    const float t = __fmul_ru(v, mg.prune);
    return mg.add ? __fadd_ru(t, __ldg(mg.add)) : t;
}
template <>
__device__ __forceinline__ double scale_up<double>(double v, const Margins&) {
    return v;  // EXACT: no margin
}
__device__ __forceinline__ float fin_up(float v, const Margins& mg) {
    const float t = __fmul_ru(v, mg.fin);
    return mg.add ? __fadd_ru(t, __ldg(mg.add + 1)) : t;
}

// ------------------------------------------------------- planar transpose
// [s][t][p] -> [t*d+p][s]: operands of the tiled LB_MV kernel.
template <typename T>
__global__ void planar_kernel(const T* __restrict__ in, int64_t S, int rows, T* __restrict__ out) {
    __shared__ T tile[32][33];
    const int64_t s0 = (int64_t)blockIdx.x * 32;
    const int r0 = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int k = ty; k < 32; k += 8) {
        const int64_t s = s0 + k;
        const int r = r0 + tx;
        tile[k][tx] = (s < S && r < rows) ? in[s * rows + r] : T(0);
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
        const int r = r0 + k;
        const int64_t s = s0 + tx;
        if (r < rows && s < S) out[(int64_t)r * S + s] = tile[tx][k];
    }
}

template <typename T>
int planarize(const T* in, int64_t S, int rows, T* out, cudaStream_t st) {
    dim3 grid((unsigned)((S + 31) / 32), (unsigned)((rows + 31) / 32));
    if (grid.y > 65535) return TCDTW_NOT_SUPPORTED;
    planar_kernel<T><<<grid, 256, 0, st>>>(in, S, rows, out);
    return launch_status();
}

// The float32 planar copies of the saturating LB_MV pass are tile-major:
// element (row r, series s) at ((s / 64) * rows + r) * 64 + s % 64, the last
// tile zero-padded -- a tile's rows are contiguous (one TMA bulk copy per
// operand and round) -- and multiplied by scale[0], a power of two (exact).
constexpr int kPlanarTile = 64;
inline int64_t planar_pad(int64_t S) { return (S + kPlanarTile - 1) / kPlanarTile * kPlanarTile; }
static __global__ void planar_tiled_kernel(const float* __restrict__ in, int64_t S, int rows, float* __restrict__ out,
                                           const float* __restrict__ scale) {
    __shared__ float tile[32][33];
    const int64_t s0 = (int64_t)blockIdx.x * 32;
    const int r0 = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    const float sc = __ldg(scale);
    for (int k = ty; k < 32; k += 8) {
        const int64_t s = s0 + k;
        const int r = r0 + tx;
        tile[k][tx] = (s < S && r < rows) ? in[s * rows + r] * sc : 0.f;
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
        const int r = r0 + k;
        const int64_t s = s0 + tx;  // < planar_pad(S): the grid covers whole tiles
        if (r < rows) out[((s / kPlanarTile) * rows + r) * kPlanarTile + (s % kPlanarTile)] = tile[tx][k];
    }
}
static int planarize_tiled(const float* in, int64_t S, int rows, float* out, cudaStream_t st, const float* scale) {
    dim3 grid((unsigned)(planar_pad(S) / 32), (unsigned)((rows + 31) / 32));
    if (grid.y > 65535) return TCDTW_NOT_SUPPORTED;
    planar_tiled_kernel<<<grid, 256, 0, st>>>(in, S, rows, out, scale);
    return launch_status();
}

// A planar copy carries a 256-byte trailer behind its elements: float[2]
// {sigma, 1/sigma}, the power-of-two scale its values were multiplied by
// (1 for float64).  sigma maps the collection's value range into (1/2, 1],
// so a per-dimension envelope deviation of any query inside that range is
// <= 1 in the scaled domain and FADD.SAT clamps only what is negative.
inline size_t planar_trailer_off(int64_t S, int rows, size_t es) {
    const int64_t cols = es == 4 ? planar_pad(S) : S;  // float32 copies are tile-major, padded
    return ((size_t)cols * rows * es + 255) & ~size_t(255);
}
inline size_t planar_bytes(int64_t S, int rows, size_t es) { return planar_trailer_off(S, rows, es) + 256; }

__device__ __forceinline__ unsigned f32_ordered(float v) {  // monotone float -> unsigned
    const unsigned u = __float_as_uint(v);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float f32_unordered(unsigned k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}
// mm[0] = ordered min (init 0xffffffff), mm[1] = ordered max (init 0)
static __global__ void __launch_bounds__(256) value_range_kernel(const float* __restrict__ v, int64_t count,
                                                                 unsigned* __restrict__ mm) {
    unsigned lo = 0xffffffffu, hi = 0u;
    for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < count; e += (int64_t)gridDim.x * 256) {
        const unsigned k = f32_ordered(v[e]);
        lo = k < lo ? k : lo;
        hi = k > hi ? k : hi;
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if ((threadIdx.x & 31) == 0) {
        atomicMin(mm, lo);
        atomicMax(mm + 1, hi);
    }
}
static __global__ void planar_scale_kernel(const unsigned* __restrict__ mm, float* __restrict__ scale) {
    float sg = 1.f;
    if (mm && mm[0] <= mm[1]) {
        const double range = (double)f32_unordered(mm[1]) - (double)f32_unordered(mm[0]);
        if (range > 0.0) {
            int ex;
            frexp(range, &ex);  // range = f * 2^ex, f in [1/2, 1)
            if (ldexp(1.0, ex - 1) == range) --ex;  // an exact power of two maps to 1
            ex = ex > 126 ? 126 : (ex < -126 ? -126 : ex);
            sg = (float)ldexp(1.0, -ex);
        }
    }
    scale[0] = sg;
    scale[1] = 1.f / sg;  // exact
}
// float32 collection -> its scale (mm: 8 bytes of scratch next to `scale`)
static int planar_scale(const float* v, int64_t count, float* scale, cudaStream_t st) {
    unsigned* mm = reinterpret_cast<unsigned*>(scale + 2);
    cudaMemsetAsync(mm, 0xff, 4, st);
    cudaMemsetAsync(mm + 1, 0, 4, st);
    int64_t blocks = (count + 255) / 256;
    blocks = blocks > 148 * 16 ? 148 * 16 : (blocks < 1 ? 1 : blocks);
    value_range_kernel<<<(unsigned)blocks, 256, 0, st>>>(v, count, mm);
    planar_scale_kernel<<<1, 1, 0, st>>>(mm, scale);
    return launch_status();
}

// The query envelopes of the saturating LB_MV pass: planar (upper, lower) ->
// (m, h), in place (scaled, tile-major; the layout does not matter here).  m = the rounded midpoint, h = the
// half width inflated so that max(|c - m| - h, 0), evaluated in float32, is
// <= dist(c, [lower, upper]) (1 + 2^-24)^2 for EVERY float c:
//   h >= (true half width + |m - true midpoint|) (1 + 2^-22) + 2^-120
// covers the rounding of m, of c - m and of |.| - h (the relative part) and
// flushed subnormals of the scaled operands (the absolute part).
static __global__ void __launch_bounds__(256) midhalf_kernel(float* __restrict__ up, float* __restrict__ lo,
                                                             int64_t count) {
    for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < count; e += (int64_t)gridDim.x * 256) {
        const double u = (double)up[e], l = (double)lo[e];  // already scaled (planarize_tiled)
        const double md = 0.5 * (u + l);
        const float m = (float)md;
        const double em = fabs((double)m - md);
        const double hd = (0.5 * (u - l) + em) * (1.0 + 0x1p-22) + 0x1p-120;
        float h = __double2float_ru(hd * (1.0 + 0x1p-50));
        up[e] = m;
        lo[e] = h;
    }
}

// ------------------------------------------------------------ LB_MV matrix
// Block = 16 x 16 threads, tile QT = 16*M queries x CT = 16*M candidates,
// TC time steps staged per round.  Each thread accumulates M x M pairs,
// strictly sequentially over t (the reference's cumsum order, which keeps
// LB <= DTW exact in float64).
//
// With UB, the same pass also accumulates the diagonal-path cost
// sum_t ||q_t - c_t||: the cost of one admissible warping path, hence an
// UPPER bound of the banded DTW (exactly so in float64, where it is the
// DP's own sum along that path).  Its per-query minimum seeds d_best and its
// smallest entries pick the seed candidates.
template <typename T, int DMAX, bool EXACT>
struct MvTile {
    static constexpr int M = EXACT ? (DMAX <= 8 ? 2 : 1) : 4;
    static constexpr int QT = 16 * M;
    static constexpr int CT = 16 * M;
};

template <typename T, int DMAX, bool EXACT, bool UB, int DX, bool SAT>
__device__ __forceinline__ void lbmv_matrix_kernel_body(const T* __restrict__ UT, const T* __restrict__ LT,
                                                        const T* __restrict__ QTP, const T* __restrict__ CT_,
                                                        int64_t Q, int64_t N, int n, int d, int TC,
                                                        T* __restrict__ out, T* __restrict__ ub_out, int64_t q0,
                                                        int64_t c0, bool v16, bool trans, int64_t ub_n, int ub_stride,
                                                        const float* __restrict__ scale);

// asynchronous global -> shared copies; src_bytes < bytes zero-fills the rest
__device__ __forceinline__ void cp_async_ca(void* dst, const void* src, int bytes, int src_bytes) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
    if (bytes == 4)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(sa), "l"(src), "r"(src_bytes) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_cg16(void* dst, const void* src, int src_bytes) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(NPEND) : "memory"); }
// TMA bulk copies (global -> shared, bytes a multiple of 16) completing on an mbarrier
__device__ __forceinline__ unsigned mv_saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mv_bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     mv_saddr(dst)),
                 "l"(src), "r"(bytes), "r"(mv_saddr(bar))
                 : "memory");
}
__device__ __forceinline__ void mv_bar_expect(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mv_saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mv_bar_wait(uint64_t* bar, unsigned parity) {
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(mv_saddr(bar)), "r"(parity)
            : "memory");
    }
}

// DX > 0: the dimension count is a compile-time constant (fully unrolled
// per-dimension loop for the hot shapes); DX == 0: runtime d.
template <typename T, int DMAX, bool EXACT, bool UB, int DX, bool SAT>
__global__ void __launch_bounds__(256, (SAT && DX > 0 && DX <= 8) ? 3 : 1) lbmv_matrix_kernel(const T* __restrict__ UT, const T* __restrict__ LT,
                                                          const T* __restrict__ QTP, const T* __restrict__ CT_,
                                                          int64_t Q, int64_t N, int n, int d, int TC,
                                                          T* __restrict__ out, T* __restrict__ ub_out, int ub_stride,
                                                          bool v16, bool trans, int64_t ub_n,
                                                          const float* __restrict__ scale) {
    using Tile = MvTile<T, DMAX, EXACT>;
    constexpr int QT = Tile::QT, CTL = Tile::CT;
    // query tiles vary fastest: concurrently resident blocks share one
    // candidate tile, so each candidate byte leaves HBM once per batch and the
    // (small) envelope tiles are re-read from L2.
    const int64_t nqt = (Q + QT - 1) / QT;
    const int64_t q0 = ((int64_t)blockIdx.x % nqt) * QT;
    const int64_t c0 = ((int64_t)blockIdx.x / nqt) * CTL;
    // the upper bound only seeds d_best: compute it on every ub_stride-th
    // candidate tile (block-uniform)
    if constexpr (UB) {
        if (((int64_t)blockIdx.x / nqt) % ub_stride != 0) {
            lbmv_matrix_kernel_body<T, DMAX, EXACT, false, DX, SAT>(UT, LT, QTP, CT_, Q, N, n, d, TC, out, ub_out, q0,
                                                                    c0, v16, trans, ub_n, ub_stride, scale);
            return;
        }
    }
    lbmv_matrix_kernel_body<T, DMAX, EXACT, UB, DX, SAT>(UT, LT, QTP, CT_, Q, N, n, d, TC, out, ub_out, q0, c0, v16,
                                                         trans, ub_n, ub_stride, scale);
}

template <typename T, int DMAX, bool EXACT, bool UB, int DX, bool SAT>
__device__ __forceinline__ void lbmv_matrix_kernel_body(const T* __restrict__ UT, const T* __restrict__ LT,
                                                        const T* __restrict__ QTP, const T* __restrict__ CT_,
                                                        int64_t Q, int64_t N, int n, int d, int TC,
                                                        T* __restrict__ out, T* __restrict__ ub_out, int64_t q0,
                                                        int64_t c0, bool v16, bool trans, int64_t ub_n, int ub_stride,
                                                        const float* __restrict__ scale) {
    using Tile = MvTile<T, DMAX, EXACT>;
    constexpr int M = Tile::M, QT = Tile::QT, CTL = Tile::CT;
    constexpr int VN = 16 / (int)sizeof(T);  // elements per 16-byte copy
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // two staging buffers (double buffering): round k+1's rows
    // stream in while round k is consumed.  Buffer layout: us | ls | cs | qs
    const size_t buf_elems = (size_t)TC * d * (3 * QT + CTL);
    const int tid = threadIdx.x;
    // SAT: the operands are tile-major planar copies (planar_tiled_kernel) --
    // the rows of one 64-series tile are contiguous, so a round of every
    // operand is ONE TMA bulk copy issued by thread 0, completing on the
    // buffer's mbarrier; no staging instructions in the compute warps.
    uint64_t* const bars = reinterpret_cast<uint64_t*>(reinterpret_cast<T*>(smem_raw) + 2 * buf_elems);
    constexpr bool tma = SAT;
    auto stage = [&](int t0, int buf) {
        T* us = reinterpret_cast<T*>(smem_raw) + buf * buf_elems;
        T* ls = us + (size_t)TC * d * QT;
        T* cs = ls + (size_t)TC * d * QT;
        T* qs = cs + (size_t)TC * d * CTL;
        const int tcn = (n - t0) < TC ? (n - t0) : TC;
        const int rows = tcn * d;
        const int64_t rbase = (int64_t)t0 * d;
        if constexpr (tma) {
            static_assert(!SAT || (QT == kPlanarTile && CTL == kPlanarTile), "tile-major planar width");
            if (tid != 0) return;
            const unsigned bytes = (unsigned)rows * QT * (unsigned)sizeof(T);
            const int64_t qoff = ((q0 / QT) * (int64_t)n * d + rbase) * QT;
            const int64_t coff = ((c0 / CTL) * (int64_t)n * d + rbase) * CTL;
            mv_bar_expect(bars + buf, (UB ? 4u : 3u) * bytes);
            mv_bulk_load(us, UT + qoff, bytes, bars + buf);
            mv_bulk_load(ls, LT + qoff, bytes, bars + buf);
            if constexpr (UB) mv_bulk_load(qs, QTP + qoff, bytes, bars + buf);
            mv_bulk_load(cs, CT_ + coff, bytes, bars + buf);
            return;
        }
        if (v16) {
            for (int e = tid * VN; e < rows * QT; e += 256 * VN) {
                const int r = e / QT, qq = e - (e / QT) * QT;
                const int64_t q = q0 + qq;
                const int64_t left = Q - q;
                const int sb = left <= 0 ? 0 : (left >= VN ? 16 : (int)left * (int)sizeof(T));
                const int64_t off = (rbase + r) * Q + (sb ? q : 0);
                cp_async_cg16(us + e, UT + off, sb);
                cp_async_cg16(ls + e, LT + off, sb);
                if constexpr (UB) cp_async_cg16(qs + e, QTP + off, sb);
            }
            for (int e = tid * VN; e < rows * CTL; e += 256 * VN) {
                const int r = e / CTL, cc = e - (e / CTL) * CTL;
                const int64_t c = c0 + cc;
                const int64_t left = N - c;
                const int sb = left <= 0 ? 0 : (left >= VN ? 16 : (int)left * (int)sizeof(T));
                cp_async_cg16(cs + e, CT_ + (rbase + r) * N + (sb ? c : 0), sb);
            }
        } else {
            for (int e = tid; e < rows * QT; e += 256) {
                const int r = e / QT, qq = e - (e / QT) * QT;
                const int64_t q = q0 + qq;
                const int sb = q < Q ? (int)sizeof(T) : 0;
                const int64_t off = (rbase + r) * Q + (sb ? q : 0);
                cp_async_ca(us + e, UT + off, (int)sizeof(T), sb);
                cp_async_ca(ls + e, LT + off, (int)sizeof(T), sb);
                if constexpr (UB) cp_async_ca(qs + e, QTP + off, (int)sizeof(T), sb);
            }
            for (int e = tid; e < rows * CTL; e += 256) {
                const int r = e / CTL, cc = e - (e / CTL) * CTL;
                const int64_t c = c0 + cc;
                const int sb = c < N ? (int)sizeof(T) : 0;
                cp_async_ca(cs + e, CT_ + (rbase + r) * N + (sb ? c : 0), (int)sizeof(T), sb);
            }
        }
        cp_async_commit();
    };
    const int tq = tid & 15, tc = tid >> 4;
    T total[M][M], ubt[M][M];
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
        for (int j = 0; j < M; ++j) total[i][j] = ubt[i][j] = T(0);

    if constexpr (tma) {
        if (tid == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mv_saddr(bars)) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mv_saddr(bars + 1)) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    stage(0, 0);
    int buf = 0, round = 0;
    for (int t0 = 0; t0 < n; t0 += TC, buf ^= 1, ++round) {
        const int tcn = (n - t0) < TC ? (n - t0) : TC;
        if constexpr (tma) {
            if (t0 + TC < n) stage(t0 + TC, buf ^ 1);  // the other buffer was released by the barrier closing the last round
            mv_bar_wait(bars + buf, (unsigned)(round >> 1) & 1u);
        } else {
            if (t0 + TC < n) {
                stage(t0 + TC, buf ^ 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
        }
        const T* us = reinterpret_cast<const T*>(smem_raw) + buf * buf_elems;
        const T* ls = us + (size_t)TC * d * QT;
        const T* cs = ls + (size_t)TC * d * QT;
        const T* qs = cs + (size_t)TC * d * CTL;
        for (int tt = 0; tt < tcn; ++tt) {
            if constexpr (EXACT) {
                T sq[M][M][DMAX], sd[M][M][DMAX];
#pragma unroll
                for (int p = 0; p < DMAX; ++p) {
                    if (p < d) {
                        const int r = tt * d + p;
                        T u[M], l[M], c[M], qv[M];
#pragma unroll
                        for (int i = 0; i < M; ++i) {
                            u[i] = us[r * QT + tq * M + i];
                            l[i] = ls[r * QT + tq * M + i];
                            c[i] = cs[r * CTL + tc * M + i];
                            if constexpr (UB) qv[i] = qs[r * QT + tq * M + i];
                        }
#pragma unroll
                        for (int i = 0; i < M; ++i)
#pragma unroll
                            for (int j = 0; j < M; ++j) {
                                const T hi = tmax(sub_rn(c[j], u[i]), T(0));
                                const T lo = tmax(sub_rn(l[i], c[j]), T(0));
                                sq[i][j][p] = add_rn(mul_rn(hi, hi), mul_rn(lo, lo));
                                if constexpr (UB) {
                                    const T df = sub_rn(qv[i], c[j]);  // cost_band order: q - c
                                    sd[i][j][p] = mul_rn(df, df);
                                }
                            }
                    } else {
#pragma unroll
                        for (int i = 0; i < M; ++i)
#pragma unroll
                            for (int j = 0; j < M; ++j) sq[i][j][p] = sd[i][j][p] = T(0);
                    }
                }
#pragma unroll
                for (int i = 0; i < M; ++i)
#pragma unroll
                    for (int j = 0; j < M; ++j) {
                        total[i][j] = add_rn(total[i][j], sqrt_rn(np_sum<T, DMAX>(sq[i][j], d)));
                        if constexpr (UB) ubt[i][j] = add_rn(ubt[i][j], sqrt_rn(np_sum<T, DMAX>(sd[i][j], d)));
                    }
            } else {
                T s[M][M], sd[M][M];
#pragma unroll
                for (int i = 0; i < M; ++i)
#pragma unroll
                    for (int j = 0; j < M; ++j) s[i][j] = sd[i][j] = T(0);
                constexpr int PU = DX > 0 ? DX : 1;
#pragma unroll PU
                for (int p = 0; p < (DX > 0 ? DX : d); ++p) {
                    const int r = tt * (DX > 0 ? DX : d) + p;
                    T u[M], l[M], c[M], qv[M];
                    if constexpr (M == 4 && sizeof(T) == 4) {
                        const float4 u4 = *reinterpret_cast<const float4*>(us + r * QT + tq * 4);
                        const float4 l4 = *reinterpret_cast<const float4*>(ls + r * QT + tq * 4);
                        const float4 c4 = *reinterpret_cast<const float4*>(cs + r * CTL + tc * 4);
                        u[0] = u4.x; u[1] = u4.y; u[2] = u4.z; u[3] = u4.w;
                        l[0] = l4.x; l[1] = l4.y; l[2] = l4.z; l[3] = l4.w;
                        c[0] = c4.x; c[1] = c4.y; c[2] = c4.z; c[3] = c4.w;
                        if constexpr (UB) {
                            const float4 q4 = *reinterpret_cast<const float4*>(qs + r * QT + tq * 4);
                            qv[0] = q4.x; qv[1] = q4.y; qv[2] = q4.z; qv[3] = q4.w;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < M; ++i) {
                            u[i] = us[r * QT + tq * M + i];
                            l[i] = ls[r * QT + tq * M + i];
                            c[i] = cs[r * CTL + tc * M + i];
                            if constexpr (UB) qv[i] = qs[r * QT + tq * M + i];
                        }
                    }
#pragma unroll
                    for (int i = 0; i < M; ++i)
#pragma unroll
                        for (int j = 0; j < M; ++j) {
                            T dev;
                            if constexpr (SAT) {
                                // u = midpoint, l = inflated half width (midhalf_kernel), scaled
                                // domain: FADD, FADD.SAT with |.|, FFMA -- 3 issue slots per term
                                dev = __saturatef(fabsf(c[j] - u[i]) - l[i]);
                            } else {
                                // u >= l, so at most one of (c-u, l-c) is positive
                                dev = tmax(tmax(c[j] - u[i], l[i] - c[j]), T(0));
                            }
                            s[i][j] = fma(dev, dev, s[i][j]);
                            if constexpr (UB) {
                                const T df = qv[i] - c[j];
                                sd[i][j] = fma(df, df, sd[i][j]);
                            }
                        }
                }
#pragma unroll
                for (int i = 0; i < M; ++i)
#pragma unroll
                    for (int j = 0; j < M; ++j) {
                        total[i][j] += fast_sqrt(s[i][j]);
                        if constexpr (UB) ubt[i][j] += fast_sqrt(sd[i][j]);
                    }
            }
        }
        __syncthreads();
    }
    if constexpr (SAT) {  // back from the scaled domain (a power of two: exact)
        const T inv = (T)__ldg(scale + 1);
#pragma unroll
        for (int i = 0; i < M; ++i)
#pragma unroll
            for (int j = 0; j < M; ++j) {
                total[i][j] *= inv;
                // the upper bound seeds d_best directly (topk_kernel): a term whose scaled
                // square sum is subnormal is flushed by sqrt.approx.ftz, losing < 2^-63 --
                // give it back so the seed never falls below the path's cost
                if constexpr (UB) ubt[i][j] = (ubt[i][j] + (T)n * (T)0x1p-62) * inv;
            }
    }
#pragma unroll
    for (int i = 0; i < M; ++i) {
        const int64_t q = q0 + tq * M + i;
        if (q >= Q) continue;
#pragma unroll
        for (int j = 0; j < M; ++j) {
            const int64_t c = c0 + tc * M + j;
            if (c < N) {
                // trans: the reverse bound (envelope side = candidates) lands
                // in the (query, candidate) layout of the forward matrix
                out[trans ? c * Q + q : q * N + c] = total[i][j];
                // upper bounds only on the sampled candidate tiles, stored
                // compactly: (q, sampled tile, column) -> q * ub_n + ...
                if constexpr (UB) ub_out[q * ub_n + (c0 / CTL / ub_stride) * CTL + (c - c0)] = ubt[i][j];
            }
        }
    }
}

template <typename T, int DMAX, bool EXACT>
int launch_lbmv_matrix(const T* UT, const T* LT, const T* QTP, const T* CT, int64_t Q, int64_t N, int n, int d,
                       T* out, T* ub_out, cudaStream_t st, int ub_stride = 1, bool trans = false, int64_t ub_n = 0,
                       const float* scale = nullptr) {
    using Tile = MvTile<T, DMAX, EXACT>;
    const bool ub = ub_out != nullptr;
    // two staging buffers of TC time steps each (layout us | ls | cs | qs)
    const size_t per_t = (size_t)d * (3 * Tile::QT + Tile::CT) * sizeof(T);
    // SAT with a compile-time d <= 8: three blocks per SM (80 registers by launch bounds), so 72 KB of
    // staging each (C4 LB_MV 99.3 -> 93.8 ms per 1k queries; d = 20 spills at 80 registers and keeps two)
    const bool three = scale != nullptr && (d == 3 || d == 4 || d == 5 || d == 6 || d == 8) && d <= DMAX;
    int TC = (int)(((three ? 72 : 96) * 1024) / (2 * per_t));
    TC = TC < 1 ? 1 : (TC > 16 ? 16 : TC);
    TC = TC > n ? n : TC;
    const size_t smem = 2 * per_t * TC + 16;  // + the two mbarriers of the TMA staging
    constexpr int VN = 16 / (int)sizeof(T);
    const bool v16 = Q % VN == 0 && N % VN == 0 && (reinterpret_cast<uintptr_t>(UT) | reinterpret_cast<uintptr_t>(LT) |
                                                     reinterpret_cast<uintptr_t>(QTP) | reinterpret_cast<uintptr_t>(CT)) % 16 == 0 &&
                     (Tile::QT % VN) == 0 && (Tile::CT % VN) == 0;
    // scale != nullptr: the saturating form (operands prepared by midhalf_kernel / scaled planarize)
    constexpr bool CAN_SAT = !EXACT && std::is_same<T, float>::value;
    const bool sat = CAN_SAT && scale != nullptr;
    if (scale != nullptr && !sat) return TCDTW_NOT_SUPPORTED;
    auto kern = ub ? lbmv_matrix_kernel<T, DMAX, EXACT, true, 0, false> : lbmv_matrix_kernel<T, DMAX, EXACT, false, 0, false>;
    if constexpr (CAN_SAT) {
        if (sat) kern = ub ? lbmv_matrix_kernel<T, DMAX, EXACT, true, 0, true> : lbmv_matrix_kernel<T, DMAX, EXACT, false, 0, true>;
    }
    if constexpr (!EXACT) {
#define TCDTW_MV_DX(DD)                                                                                    \
        if (d == DD && DD <= DMAX) {                                                                       \
            constexpr int DXV = DD <= DMAX ? DD : 0;                                                       \
            kern = ub ? lbmv_matrix_kernel<T, DMAX, EXACT, true, DXV, false>                               \
                      : lbmv_matrix_kernel<T, DMAX, EXACT, false, DXV, false>;                             \
            if constexpr (CAN_SAT) {                                                                       \
                if (sat)                                                                                   \
                    kern = ub ? lbmv_matrix_kernel<T, DMAX, EXACT, true, DXV, true>                        \
                              : lbmv_matrix_kernel<T, DMAX, EXACT, false, DXV, true>;                      \
            }                                                                                              \
        }
        TCDTW_MV_DX(3) TCDTW_MV_DX(4) TCDTW_MV_DX(5) TCDTW_MV_DX(6) TCDTW_MV_DX(8) TCDTW_MV_DX(20)
#undef TCDTW_MV_DX
    }
    if (smem > 48 * 1024) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return TCDTW_CUDA_ERROR;
    }
    const int64_t nqt = (Q + Tile::QT - 1) / Tile::QT;
    const int64_t nct = (N + Tile::CT - 1) / Tile::CT;
    if (nqt * nct > 2147483647LL) return TCDTW_NOT_SUPPORTED;
    const unsigned grid = (unsigned)(nqt * nct);
    kern<<<grid, 256, smem, st>>>(UT, LT, QTP, CT, Q, N, n, d, TC, out, ub_out, ub_stride, v16, trans, ub_n, scale);
    return launch_status();
}

// ------------------------------------------------------------ seeds (top-S)
template <typename T, int S>
__global__ void __launch_bounds__(256) topk_kernel(const T* __restrict__ lb, int64_t N, int s_eff, T* __restrict__ dbest,
                                                   uint32_t* __restrict__ seeds, int32_t* __restrict__ seed_cnt,
                                                   int ct, int stride) {
    const int64_t q = blockIdx.x;
    const int64_t ub_n = ((N / ((int64_t)ct * stride)) * ct) +
                         ((N % ((int64_t)ct * stride)) < ct ? (N % ((int64_t)ct * stride)) : ct);  // sampled columns
    const T* row = lb + q * ub_n;
    T bv[S];
    uint32_t bi[S];
#pragma unroll
    for (int k = 0; k < S; ++k) {
        bv[k] = dev_inf<T>();
        bi[k] = 0xffffffffu;
    }
    // keys exist on every stride-th tile of ct candidates, stored compactly
    for (int64_t k = threadIdx.x; k < ub_n; k += blockDim.x) {
        const int64_t c = (k / ct) * ct * stride + (k % ct);
        const T v = row[k];
        if (v < bv[S - 1]) {
            bv[S - 1] = v;
            bi[S - 1] = (uint32_t)c;
#pragma unroll
            for (int k = S - 1; k > 0; --k) {
                if (bv[k] < bv[k - 1]) {
                    T tv = bv[k]; bv[k] = bv[k - 1]; bv[k - 1] = tv;
                    uint32_t ti = bi[k]; bi[k] = bi[k - 1]; bi[k - 1] = ti;
                }
            }
        }
    }
    __shared__ T sv[8];
    __shared__ uint32_t si[8];
    __shared__ T win_v;
    __shared__ uint32_t win_i;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int r = 0; r < s_eff; ++r) {
        T v = bv[0];
        uint32_t i = bi[0];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const T ov = __shfl_xor_sync(0xffffffffu, v, o);
            const uint32_t oi = __shfl_xor_sync(0xffffffffu, i, o);
            if (ov < v || (ov == v && oi < i)) { v = ov; i = oi; }
        }
        if (lane == 0) { sv[wid] = v; si[wid] = i; }
        __syncthreads();
        if (threadIdx.x == 0) {
            T bvv = sv[0];
            uint32_t bii = si[0];
            for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
                if (sv[k] < bvv || (sv[k] == bvv && si[k] < bii)) { bvv = sv[k]; bii = si[k]; }
            win_v = bvv;
            win_i = bii;
            seeds[q * S + r] = bii;
            // keys are diagonal-path upper bounds: the smallest one bounds the
            // final nearest-neighbour distance from above
            if (r == 0 && dbest && bvv < dbest[q]) dbest[q] = bvv;
        }
        __syncthreads();
        if (bi[0] == win_i && win_i != 0xffffffffu) {
#pragma unroll
            for (int k = 0; k < S - 1; ++k) { bv[k] = bv[k + 1]; bi[k] = bi[k + 1]; }
            bv[S - 1] = dev_inf<T>();
            bi[S - 1] = 0xffffffffu;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) seed_cnt[q] = s_eff;
}

// --------------------------------------------------------------- work tiles
struct Tiles {
    uint32_t* q;      // query of the tile
    int64_t* begin;   // first entry
    int32_t* len;     // entries (<= 32)
    // number of tiles on the device (written by the compaction's scan), so
    // the host never waits for it; nullptr: the kernels' n_tiles argument
    const int64_t* count = nullptr;
};

// Tiles a kernel works through: the device count when there is one (the
// host passes an upper bound for grid sizing), else the argument.
__device__ __forceinline__ int64_t tile_count(const Tiles& t, int64_t n_tiles) {
    return t.count ? *t.count : n_tiles;
}

// Survivor piece length of the R-row lane kernel, from the device tile
// count: whole 2048-entry segments when there are at least 4 per resident
// warp, else pieces of about survivors / (4 x warps), at least 128.
static __global__ void laner_seglen_kernel(const int64_t* __restrict__ tiles32, int64_t warps, int* __restrict__ out) {
    const int64_t surv_est = *tiles32 * (int64_t)kTile;
    int seg_len = (int)kChunk;
    if (surv_est / kChunk < 4 * warps) {
        const int64_t want = surv_est / (4 * warps);
        seg_len = 128;
        while (seg_len < want && seg_len < (int)kChunk) seg_len <<= 1;
    }
    *out = seg_len;
}

// seed list: one tile per query (S <= 32 entries at q*S)
static __global__ void seed_tiles_kernel(int64_t Q, int S, const int32_t* __restrict__ seed_cnt, Tiles t) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < Q; q += (int64_t)gridDim.x * blockDim.x) {
        t.q[q] = (uint32_t)q;
        t.begin[q] = q * S;
        t.len[q] = seed_cnt[q];
    }
}

// ------------------------------------------------------------- compaction
template <typename T>
__device__ __forceinline__ bool keep_pred(const T* __restrict__ lbrow, const T* __restrict__ lb2row, int64_t c,
                                          T thr, bool all, const uint32_t* seeds_s, int ns) {
    if (!all) {
        if (!(lbrow[c] <= thr)) return false;
        if (lb2row && !(lb2row[c] <= thr)) return false;  // reverse bound (TCDTW_FLAG_REVERSE_LB)
    }
    for (int k = 0; k < ns; ++k)
        if (seeds_s[k] == (uint32_t)c) return false;
    return true;
}

template <typename T>
__global__ void __launch_bounds__(256) compact_count_kernel(const T* __restrict__ lb, const T* __restrict__ lb2,
                                                            int64_t N, int n_chunks,
                                                            const T* __restrict__ dbest, Margins mg, bool all,
                                                            const uint32_t* __restrict__ seeds, const int32_t* __restrict__ seed_cnt,
                                                            int S, int64_t* __restrict__ chunk_cnt) {
    const int64_t q = blockIdx.y;
    const int chunk = blockIdx.x;
    __shared__ uint32_t sd[kSeedMax];
    __shared__ int wsum[8];
    const int ns = S > 0 ? seed_cnt[q] : 0;
    if (threadIdx.x < ns) sd[threadIdx.x] = seeds[q * S + threadIdx.x];
    __syncthreads();
    const T thr = all ? T(0) : scale_up<T>(dbest[q], mg);
    const T* row = lb ? lb + q * N : nullptr;
    const T* row2 = lb2 ? lb2 + q * N : nullptr;
    const int64_t c0 = (int64_t)chunk * kChunk;
    const int64_t c1 = c0 + kChunk < N ? c0 + kChunk : N;
    int cnt = 0;
    for (int64_t c = c0 + threadIdx.x; c < c1; c += 256) cnt += keep_pred<T>(row, row2, c, thr, all, sd, ns) ? 1 : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        for (int k = 0; k < 8; ++k) s += wsum[k];
        chunk_cnt[(int64_t)chunk * gridDim.y + q] = s;
    }
}

template <typename T>
__global__ void __launch_bounds__(256) compact_write_kernel(const T* __restrict__ lb, const T* __restrict__ lb2,
                                                            int64_t N, int n_chunks,
                                                            const T* __restrict__ dbest, Margins mg, bool all,
                                                            const uint32_t* __restrict__ seeds, const int32_t* __restrict__ seed_cnt,
                                                            int S, const int64_t* __restrict__ chunk_off,
                                                            uint32_t* __restrict__ surv, T* __restrict__ res) {
    const int64_t q = blockIdx.y;
    const int chunk = blockIdx.x;
    __shared__ uint32_t sd[kSeedMax];
    __shared__ int wsum[8];
    __shared__ int64_t base_s;
    const int ns = S > 0 ? seed_cnt[q] : 0;
    if (threadIdx.x < ns) sd[threadIdx.x] = seeds[q * S + threadIdx.x];
    if (threadIdx.x == 0) base_s = chunk_off[(int64_t)chunk * gridDim.y + q];
    __syncthreads();
    const T thr = all ? T(0) : scale_up<T>(dbest[q], mg);
    const T* row = lb ? lb + q * N : nullptr;
    const T* row2 = lb2 ? lb2 + q * N : nullptr;
    const int64_t c0 = (int64_t)chunk * kChunk;
    const int64_t c1 = c0 + kChunk < N ? c0 + kChunk : N;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t base = base_s;
    for (int64_t cb = c0; cb < c1; cb += 256) {
        const int64_t c = cb + threadIdx.x;
        const bool k = c < c1 && keep_pred<T>(row, row2, c, thr, all, sd, ns);
        const unsigned bal = __ballot_sync(0xffffffffu, k);
        if (lane == 0) wsum[wid] = __popc(bal);
        __syncthreads();
        int before = 0, tot = 0;
        for (int w2 = 0; w2 < 8; ++w2) {
            before += (w2 < wid) ? wsum[w2] : 0;
            tot += wsum[w2];
        }
        if (k) {
            const int64_t pos = base + before + __popc(bal & ((1u << lane) - 1u));
            surv[pos] = (uint32_t)c;
            res[pos] = dev_inf<T>();
        }
        base += tot;
        __syncthreads();
    }
}

// Seeds are already computed: mark their LB entries NaN so the compaction
// drops them with the bound test alone (!(NaN <= thr)) instead of comparing
// every (query, candidate) against the query's seed list.  Nothing reads a
// seed's LB after the seed pass.
template <typename T>
__global__ void poison_seeds_kernel(T* __restrict__ lb, int64_t N, int64_t Q, int S,
                                    const uint32_t* __restrict__ seeds, const int32_t* __restrict__ seed_cnt) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= Q * S) return;
    const int64_t q = e / S;
    const int k = (int)(e - q * S);
    if (k < seed_cnt[q])
        lb[q * N + seeds[e]] = sizeof(T) == 4 ? (T)__int_as_float(0x7fc00000)                 // quiet NaN
                                              : (T)__longlong_as_double(0x7ff8000000000000LL);
}

// per-(chunk, query) survivor segments -> tile counts; then fill
static __global__ void seg_tiles_count_kernel(int64_t Q, int n_chunks, const int64_t* __restrict__ chunk_off,
                                       int64_t* __restrict__ tile_cnt, int64_t* __restrict__ counters,
                                       int tile_len = kTile, const int* __restrict__ tile_len_dev = nullptr) {
    const int64_t n_seg = Q * n_chunks;
    if (tile_len_dev) tile_len = *tile_len_dev;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n_seg; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t cnt = chunk_off[g + 1] - chunk_off[g];
        tile_cnt[g] = (cnt + tile_len - 1) / tile_len;
        if (cnt && counters) atomicAdd(reinterpret_cast<unsigned long long*>(counters + (g % Q) * TCDTW_COUNTERS + TCDTW_C_SURVIVORS),
                           (unsigned long long)cnt);
    }
}

static __global__ void seg_tiles_fill_kernel(int64_t Q, int n_chunks, const int64_t* __restrict__ chunk_off,
                                      const int64_t* __restrict__ tile_off, Tiles t, int tile_len = kTile,
                                      const int* __restrict__ tile_len_dev = nullptr) {
    const int64_t n_seg = Q * n_chunks;
    if (tile_len_dev) tile_len = *tile_len_dev;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n_seg; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = chunk_off[g], e = chunk_off[g + 1];
        const int64_t t0 = tile_off[g];
        const int64_t nt = (e - b + tile_len - 1) / tile_len;
        for (int64_t k = 0; k < nt; ++k) {
            const int64_t bb = b + k * tile_len;
            t.q[t0 + k] = (uint32_t)(g % Q);
            t.begin[t0 + k] = bb;
            t.len[t0 + k] = (int32_t)((e - bb) < tile_len ? (e - bb) : tile_len);
        }
    }
}

// ------------------------------------------------- search-wide arguments
template <typename T>
struct SArgs {
    const T* queries;     // (Q, n, d)
    const T* cands;       // (N, n, d)
    const T* lb;          // (Q, N) LB_MV or nullptr
    const T* env_up;      // (Q, n, d) query envelopes (nullptr without LB_MV)
    const T* env_lo;
    T* dbest;             // (Q,)
    // where the prune / abandon thresholds are read: dbest (live: every
    // completed DTW tightens them), or a snapshot taken before each DTW pass
    // (TCDTW_FLAG_FROZEN_THRESHOLDS: run-to-run identical cell counts)
    const T* thr_src;
    const T* box_lo;      // (Q, G, K, d)
    const T* box_hi;
    const T* qsteps;      // (Q, n-1)
    int64_t* counters;    // (Q, TCDTW_COUNTERS)
    int64_t N;
    int n, d, w, G, K, gw, period;
    int method, adv;
    float trigger;
    Margins mg;
    bool abandon;         // false for Method.NONE (search.py:135)
    T casc_lo, casc_hi, casc_thr;  // cascaded-abandon slack (see dtw_tpp_kernel)
    bool cascade;         // abandon on the LB_MV suffix too (off: TCDTW_FLAG_NO_CASCADE)
    // completed (not abandoned) DTWs, (q << 40 | entry), so the finalisation
    // visits only them; nullptr for the seed pass
    unsigned long long* done_list;
    unsigned long long* done_cnt;
    int64_t done_cap;
    int refill_min;  // lane kernel: refill once at least this many lanes are free
    int thr_every;   // lane kernels: re-read the live d_best every this many rows
    // float32: queries as coordinate pairs with W INF columns before and
    // W + 8 after, (Q, qpad_rows, (D+1)/2) float2 with D the lane kernel's dimension count
    // (>= d, zero-padded), staged by the R-row lane kernel
    const float2* qpad;
    int qpad_rows;
    // TCDTW_FLAG_F32_FILTER: the float64 inputs the finalists are re-scored
    // on (queries / cands are then their float32 roundings); else nullptr
    const double* xq;
    const double* xc;
    // R-row lane kernel: per-warp scratch of its head batches (nullptr: none)
    float* lane_scratch;
    // reverse LB_PC: the candidates' box sets (N, G, K, d), nullptr = off
    const T* cbox_lo;
    const T* cbox_hi;
};

template <typename T>
__device__ __forceinline__ void note_done(const SArgs<T>& a, int64_t q, int64_t ent) {
    if (a.done_list) {
        const unsigned long long k = atomicAdd(a.done_cnt, 1ull);
        if ((int64_t)k < a.done_cap) a.done_list[k] = ((unsigned long long)q << 40) | (unsigned long long)ent;
    }
}

__device__ __forceinline__ void warp_add_counter(int64_t* ctr, int64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v != 0) atomicAdd(reinterpret_cast<unsigned long long*>(ctr), (unsigned long long)v);
}

// ----------------------------------------- DTW, thread per pair (2W+1 <= BMAX)
// Rows = candidate points (one per lane, streamed from HBM), columns = the
// tile's query, staged once per warp in shared memory with W points of +inf
// padding on both sides, so every lane reads the same address (broadcast).
// The row's band lives in registers; DTW is symmetric (test_dtw.py:196-207),
// and abandoning on candidate rows is as sound as on query rows (every
// warping path crosses every row).
template <typename T, int DMAX, int BMAX, bool EXACT>
__global__ void __launch_bounds__(256) dtw_tpp_kernel(SArgs<T> a, Tiles tl, int64_t n_tiles,
                                                      const uint32_t* __restrict__ cand_of, T* __restrict__ res,
                                                      int* __restrict__ tile_ctr) {
    n_tiles = tile_count(tl, n_tiles);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int VEC = 16 / sizeof(T);
    const int n = a.n, d = a.d, w = a.w, B = 2 * w + 1;
    const int DP = (d + VEC - 1) / VEC * VEC;
    const int warps = blockDim.x >> 5, wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    T* qs = reinterpret_cast<T*>(smem_raw) + (size_t)wib * (n + 2 * w) * DP;
    const T INF = dev_inf<T>();
    int64_t cached_q = -1;
    while (true) {
        int64_t tile = 0;
        if (lane == 0) tile = atomicAdd(tile_ctr, 1);
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile >= n_tiles) break;
        const int64_t q = tl.q[tile];
        const int64_t e0 = tl.begin[tile];
        const int len = tl.len[tile];
        if (q != cached_q) {
            __syncwarp();
            const T* qsrc = a.queries + q * (int64_t)n * d;
            for (int e = lane; e < (n + 2 * w) * DP; e += 32) {
                const int r = e / DP, p = e - (e / DP) * DP;
                const int j = r - w;
                T v = T(0);
                if (p < d) v = (j >= 0 && j < n) ? qsrc[(int64_t)j * d + p] : INF;
                qs[e] = v;
            }
            cached_q = q;
            __syncwarp();
        }
        const bool has = lane < len;
        const int64_t ent = e0 + lane;
        const int64_t c = has ? (int64_t)cand_of[ent] : 0;
        bool active = has;
        if (has && res[ent] < T(0)) active = false;  // pruned by the advanced bound
        const T* crow = a.cands + c * (int64_t)n * d;
        T band[BMAX];
#pragma unroll
        for (int k = 0; k < BMAX; ++k) band[k] = (k == w) ? T(0) : INF;
        T thr = a.abandon ? scale_up<T>(load_volatile(a.thr_src + q), a.mg) : INF;
        bool done = !active;
        int stop_row = n - 1;
        bool abandoned = false;
        T cpt[DMAX], cnext[DMAX];
        load_point<T, DMAX>(cpt, crow, d);
        // Cascaded abandoning: every warping path visits every later row at a
        // cost >= that row's LB_MV term, so DTW >= rowmin_i + sum_{r>i} term_r
        // (the LB_MV row sum is LB[q][c]).  The suffix is estimated from below
        // with the relative slack a.casc (rounding of both sums).
        const bool casc = a.lb != nullptr && a.abandon && a.cascade;
        const T lbtot = (casc && active) ? a.lb[q * a.N + c] : T(0);
        const T* eu = casc ? a.env_up + q * (int64_t)n * d : nullptr;
        const T* el = casc ? a.env_lo + q * (int64_t)n * d : nullptr;
        T prefix = T(0);
        int iters = 0;
        for (int i = 0; i < n; ++i) {
            ++iters;
            if (i + 1 < n) load_point<T, DMAX>(cnext, crow + (int64_t)(i + 1) * d, d);
            const T* qrow = qs + (size_t)i * DP;
            T left = INF, rmin = INF;
#pragma unroll
            for (int k = 0; k < BMAX; ++k) {
                if (k < B) {
                    const T* qp = qrow + (size_t)k * DP;
                    T cost;
                    if constexpr (EXACT) {
                        cost = dist_exact<T, DMAX>(cpt, qp, d);
                    } else {
                        T s = T(0);
#pragma unroll
                        for (int v = 0; v < DMAX / VEC; ++v) {
                            if (v * VEC < d) {
                                const float4 q4 = *reinterpret_cast<const float4*>(qp + v * VEC);
                                const float qv[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
                                for (int u = 0; u < VEC; ++u) {
                                    if (v * VEC + u < d) {
                                        const T df = cpt[v * VEC + u] - qv[u];
                                        s = fma(df, df, s);
                                    }
                                }
                            }
                        }
                        cost = fast_sqrt(s);
                    }
                    const T up = (k + 1 < BMAX) ? band[k + 1 < BMAX ? k + 1 : 0] : INF;
                    const T best = tmin(tmin(up, band[k]), left);
                    const T v = EXACT ? add_rn(cost, best) : cost + best;
                    band[k] = v;
                    left = v;
                    rmin = tmin(rmin, v);
                }
            }
            T bound = rmin;
            if (casc) {
                T t2 = T(0);
#pragma unroll
                for (int p = 0; p < DMAX; ++p) {
                    if (p < d) {
                        const T dv = tmax(tmax(cpt[p] - __ldg(eu + (int64_t)i * d + p),
                                               __ldg(el + (int64_t)i * d + p) - cpt[p]), T(0));
                        t2 = fma(dv, dv, t2);
                    }
                }
                prefix += fast_sqrt(t2);
                const T suf = tmax(lbtot * a.casc_lo - prefix * a.casc_hi, T(0));
                bound = rmin + suf;
            }
            if (!done && (rmin > thr || bound > thr * a.casc_thr)) {
                done = true;
                abandoned = true;
                stop_row = i;
            }
            if (__all_sync(0xffffffffu, done)) break;
            if ((i & 7) == 7 && a.abandon) thr = scale_up<T>(load_volatile(a.thr_src + q), a.mg);
#pragma unroll
            for (int p = 0; p < DMAX; ++p) cpt[p] = cnext[p];
        }
        T fin = INF;
#pragma unroll
        for (int k = 0; k < BMAX; ++k)
            if (k == w) fin = band[k];
        if (active && !abandoned && fin > thr) {  // dtw.py:101-102
            abandoned = true;
            stop_row = n - 1;
        }
        if (active) res[ent] = abandoned ? INF : fin;
        if (active && !abandoned) note_done(a, q, ent);
        // best-so-far update and counters (warp-aggregated; one query per tile)
        T m = (active && !abandoned) ? fin : INF;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = tmin(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0 && m < INF) atomic_min_nonneg<T>(a.dbest + q, m);
        int64_t* ctr = a.counters + q * TCDTW_COUNTERS;
        warp_add_counter(ctr + TCDTW_C_DTW_COMPUTED, active ? 1 : 0);
        warp_add_counter(ctr + TCDTW_C_ABANDON_COUNT, (active && abandoned) ? 1 : 0);
        warp_add_counter(ctr + TCDTW_C_DTW_CELLS, active ? cells_upto(stop_row, n, w) : 0);
        if (lane == 0)
            atomicAdd(reinterpret_cast<unsigned long long*>(ctr + TCDTW_C_CELLS_ISSUED),
                      (unsigned long long)iters * B * 32);
    }
}

// ------------------------------------ DTW, lane per pair, no lockstep
// Specialised for small (d, 2W+1): each lane keeps its own pair's band AND
// the query window (2W+1 points) in registers and advances its own row, so
// a lane whose DTW is abandoned refills at once from the warp's reservoir of
// work tiles instead of idling until the slowest lane of the warp finishes.
// Rows = candidate points; the window slides one query point per row.
template <typename T, int D>
__device__ __forceinline__ T dist_reg(const T (&a)[D], const T (&b)[D]) {
    if constexpr (sizeof(T) == 8) {
        T sq[D];
#pragma unroll
        for (int p = 0; p < D; ++p) {
            const T df = sub_rn(a[p], b[p]);
            sq[p] = mul_rn(df, df);
        }
        return sqrt_rn(np_sum<T, D>(sq, D));
    } else {
        T s = T(0);
#pragma unroll
        for (int p = 0; p < D; ++p) {
            const T df = a[p] - b[p];
            s = fma(df, df, s);
        }
        return fast_sqrt(s);
    }
}

template <typename T, int D>
__device__ __forceinline__ void load_pt(T (&a)[D], const T* __restrict__ src) {
#pragma unroll
    for (int p = 0; p < D; ++p) a[p] = __ldg(src + p);
}

template <typename T> struct Vec16;
template <> struct Vec16<float> { using type = float4; static constexpr int n = 4; };
template <> struct Vec16<double> { using type = double2; static constexpr int n = 2; };

// rows of a (n, D) series per 16-byte-aligned block: 16 / gcd(16, D*sizeof(T))
template <typename T, int D>
constexpr int rows_per_block() {
    constexpr int b = D * (int)sizeof(T);
    constexpr int g = (b % 16 == 0) ? 16 : ((b % 8 == 0) ? 8 : 4);
    return 16 / g;
}

template <typename T> struct Vec8;
template <> struct Vec8<float> { using type = float2; };
template <> struct Vec8<double> { using type = double2; };

// Loads of two consecutive candidate rows (2D values) starting at an even row:
// 16-byte vectors when 2D*sizeof(T) is a multiple of 16, else 8-byte ones.
template <typename T, int D>
struct PairLoad {
    static constexpr bool v16 = ((2 * D * (int)sizeof(T)) % 16) == 0;
    using V = typename std::conditional<v16, typename Vec16<T>::type, typename Vec8<T>::type>::type;
    static constexpr int per = (int)(sizeof(V) / sizeof(T));
    static constexpr int nv = 2 * D / per;
};

// One DTW step over two consecutive rows (i, i+1) of one lane's pair.  The
// cells (i, j) and (i+1, j) share query column j, so every window point read
// from the ring serves two cells, and the two rows' min chains interleave
// (skewed by one column): half the shared-memory traffic, twice the ILP of a
// row-at-a-time sweep.  P holds row i-1 on entry and row i on exit; N
// receives row i+1.
template <typename T, int D, int B, bool EXACT>
__device__ __forceinline__ void dtw_step2(T (&P)[B], T (&N)[B], const T (&c0)[D], const T (&c1)[D],
                                          const typename Vec8<T>::type* __restrict__ ring, int h,
                                          const T (&x1)[D], T& rmin0, T& rmin1) {
    using T2 = typename Vec8<T>::type;
    constexpr int DP = (D + 1) / 2;
    const T INF = dev_inf<T>();
    const T2* base0 = ring + h * DP * 32;
    const T2* base1 = base0 - B * DP * 32;
    const int lim = B - h;
    T left0 = INF, left1 = INF;
    rmin0 = INF;
    rmin1 = INF;
#pragma unroll
    for (int s = 0; s <= B; ++s) {
        T x[D];
        if (s < B) {
            const T2* qp = (s < lim ? base0 : base1) + s * DP * 32;
#pragma unroll
            for (int pp = 0; pp < DP; ++pp) {
                const T2 v = qp[pp * 32];
                x[2 * pp] = v.x;
                if (2 * pp + 1 < D) x[2 * pp + 1] = v.y;
            }
        } else {
#pragma unroll
            for (int p = 0; p < D; ++p) x[p] = x1[p];
        }
        if (s < B) {  // row i, slot s
            T cost;
            if constexpr (EXACT) {
                T sq[D];
#pragma unroll
                for (int p = 0; p < D; ++p) {
                    const T df = sub_rn(c0[p], x[p]);
                    sq[p] = mul_rn(df, df);
                }
                cost = sqrt_rn(np_sum<T, D>(sq, D));
            } else {
                T acc = T(0);
#pragma unroll
                for (int p = 0; p < D; ++p) {
                    const T df = c0[p] - x[p];
                    acc = fma(df, df, acc);
                }
                cost = fast_sqrt(acc);
            }
            const T up = (s + 1 < B) ? P[s + 1 < B ? s + 1 : 0] : INF;
            const T best = tmin(tmin(up, P[s]), left0);
            const T v = EXACT ? add_rn(cost, best) : cost + best;
            P[s] = v;
            left0 = v;
            rmin0 = tmin(rmin0, v);
        }
        if (s >= 1) {  // row i+1, slot s-1: up = (i, j) just computed, diag = (i, j-1)
            T cost;
            if constexpr (EXACT) {
                T sq[D];
#pragma unroll
                for (int p = 0; p < D; ++p) {
                    const T df = sub_rn(c1[p], x[p]);
                    sq[p] = mul_rn(df, df);
                }
                cost = sqrt_rn(np_sum<T, D>(sq, D));
            } else {
                T acc = T(0);
#pragma unroll
                for (int p = 0; p < D; ++p) {
                    const T df = c1[p] - x[p];
                    acc = fma(df, df, acc);
                }
                cost = fast_sqrt(acc);
            }
            const T up = (s < B) ? P[s < B ? s : 0] : INF;
            const T best = tmin(tmin(up, P[s - 1 >= 0 ? s - 1 : 0]), left1);
            const T v = EXACT ? add_rn(cost, best) : cost + best;
            N[s - 1 >= 0 ? s - 1 : 0] = v;
            left1 = v;
            rmin1 = tmin(rmin1, v);
        }
    }
}

template <typename T, int D, int B, bool EXACT, bool VEC>
__global__ void __launch_bounds__(64) dtw_lane_kernel(SArgs<T> a, Tiles tl, int64_t n_tiles,
                                                      const uint32_t* __restrict__ cand_of, T* __restrict__ res,
                                                      int* __restrict__ tile_ctr) {
    n_tiles = tile_count(tl, n_tiles);
    constexpr int W = (B - 1) / 2;
    constexpr int DP = (D + 1) / 2;     // coordinate pairs per point
    constexpr bool QV = (D % 2 == 0);   // query/envelope rows as pairs
    // large d: do not carry the next step's query columns and envelope rows
    // across steps (register budget); load them inside the step instead
    constexpr bool LEAN = D > 8;
    using T2 = typename Vec8<T>::type;
    using PL = PairLoad<T, D>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = a.n;
    const int lane = threadIdx.x & 31;
    // per-lane query window ring, lane-minor pairs: slot s, pair pp of this
    // lane at ring[(s*DP + pp)*32] -> conflict-free 64/128-bit accesses.
    // Column c lives in slot (c + W) mod B.
    T2* ring = reinterpret_cast<T2*>(smem_raw) + (size_t)(threadIdx.x >> 5) * B * DP * 32 + lane;
    // per-warp copy of the current tile query's columns 0..W (the window of
    // row 0), staged once per tile so new pairs fill their ring from smem
    T2* qstage = reinterpret_cast<T2*>(smem_raw) + (size_t)(blockDim.x >> 5) * B * DP * 32 +
                 (size_t)(threadIdx.x >> 5) * (W + 1) * DP;
    int staged_q = -1;
    const unsigned FULL = 0xffffffffu;
    const T INF = dev_inf<T>();
    const bool casc = a.lb != nullptr && a.abandon && a.cascade;
    // warp reservoir (uniform) with per-tile prefetch held one entry per lane
    int64_t t_begin = 0;
    int t_q = -1, t_len = 0, t_next = 0;
    bool exhausted = false;
    T t_thr_raw = INF;  // best-so-far as loaded; the margin is applied at use
    uint32_t pf_c = 0;
    T pf_lb = T(0), pf_res = T(0);
    T pf_pair[2 * D];
    // lane state
    bool busy = false;
    int64_t ent = 0;
    int q = -1, i = 0, since = 0, h = 0;
    const T* crow = nullptr;
    const T* qser = nullptr;
    T bandA[B], bandB[B];
    T c0[D], c1[D], n0[D], n1[D];
    T thr = INF, thr_pend_raw = INF, lbtot = T(0), prefix = T(0);
    T x1[D], x2[D];             // query columns i+W+1, i+W+2 (loaded one step ahead)
    T eu0[D], el0[D], eu1[D], el1[D];  // envelope rows i, i+1 (loaded one step ahead)
    int cq = -1;
    long long c_comp = 0, c_ab = 0, c_cells = 0, c_issued = 0;
    auto flush = [&]() {
        if (cq >= 0) {
            unsigned long long* ctr = reinterpret_cast<unsigned long long*>(a.counters + (int64_t)cq * TCDTW_COUNTERS);
            if (c_comp) atomicAdd(ctr + TCDTW_C_DTW_COMPUTED, (unsigned long long)c_comp);
            if (c_ab) atomicAdd(ctr + TCDTW_C_ABANDON_COUNT, (unsigned long long)c_ab);
            if (c_cells) atomicAdd(ctr + TCDTW_C_DTW_CELLS, (unsigned long long)c_cells);
            if (c_issued) atomicAdd(ctr + TCDTW_C_CELLS_ISSUED, (unsigned long long)c_issued);
        }
        c_comp = c_ab = c_cells = c_issued = 0;
    };
    // candidate rows (row, row+1) -> dst (2D values); row even; row+1 may be n
    auto load_pair = [&](T (&dst)[2 * D], const T* cr, int row) {
        if constexpr (VEC) {
            if (row + 1 < n) {
                const typename PL::V* src = reinterpret_cast<const typename PL::V*>(cr + (int64_t)row * D);
#pragma unroll
                for (int v = 0; v < PL::nv; ++v) {
                    const typename PL::V x = __ldg(src + v);
                    const T* xs = reinterpret_cast<const T*>(&x);
#pragma unroll
                    for (int u = 0; u < PL::per; ++u) dst[v * PL::per + u] = xs[u];
                }
                return;
            }
        }
#pragma unroll
        for (int u = 0; u < 2 * D; ++u) dst[u] = (row + u / D < n) ? __ldg(cr + (int64_t)row * D + u) : T(0);
    };
    auto load_col = [&](T (&dst)[D], int col) {  // query column (INF past the end)
        if (col < n) {
            if constexpr (QV) {
                const T2* s2 = reinterpret_cast<const T2*>(qser + (int64_t)col * D);
#pragma unroll
                for (int pp = 0; pp < DP; ++pp) {
                    const T2 v = __ldg(s2 + pp);
                    dst[2 * pp] = v.x;
                    dst[2 * pp + 1] = v.y;
                }
            } else {
#pragma unroll
                for (int p = 0; p < D; ++p) dst[p] = __ldg(qser + (int64_t)col * D + p);
            }
        } else {
#pragma unroll
            for (int p = 0; p < D; ++p) dst[p] = INF;
        }
    };
    auto put_col = [&](int slot, const T (&src)[D]) {
        T2* dst = ring + slot * DP * 32;
#pragma unroll
        for (int pp = 0; pp < DP; ++pp) dst[pp * 32] = T2{src[2 * pp], (2 * pp + 1 < D) ? src[2 * pp + 1] : T(0)};
    };
    auto load_env = [&](T (&uv)[D], T (&lv)[D], int row) {  // envelope row of the lane's query
        const T* eu = a.env_up + ((int64_t)q * n + row) * D;
        const T* el = a.env_lo + ((int64_t)q * n + row) * D;
        if constexpr (QV) {
#pragma unroll
            for (int pp = 0; pp < DP; ++pp) {
                const T2 x = __ldg(reinterpret_cast<const T2*>(eu) + pp);
                const T2 y = __ldg(reinterpret_cast<const T2*>(el) + pp);
                uv[2 * pp] = x.x; uv[2 * pp + 1] = x.y;
                lv[2 * pp] = y.x; lv[2 * pp + 1] = y.y;
            }
        } else {
#pragma unroll
            for (int p = 0; p < D; ++p) {
                uv[p] = __ldg(eu + p);
                lv[p] = __ldg(el + p);
            }
        }
    };
    auto lb_term = [&](const T (&c)[D], const T (&uv)[D], const T (&lv)[D]) -> T {  // LB_MV term of one row
        T t2 = T(0);
#pragma unroll
        for (int p = 0; p < D; ++p) {
            const T dv = tmax(tmax(c[p] - uv[p], lv[p] - c[p]), T(0));
            t2 = fma(dv, dv, t2);
        }
        return fast_sqrt(t2);
    };
    // refill free lanes; a new pair starts with `prev` as its row -1 band
    auto refill = [&](T (&prev)[B]) {
        unsigned freem = __ballot_sync(FULL, !busy);
        // the refill path costs the whole warp its instructions however many
        // lanes it serves: batch it until refill_min lanes are free
        if (__popc(freem) < a.refill_min && freem != FULL) return;
        while (freem && !exhausted) {
            if (t_next >= t_len) {
                int64_t tile = 0;
                if (lane == 0) tile = atomicAdd(tile_ctr, 1);
                tile = __shfl_sync(FULL, tile, 0);
                if (tile >= n_tiles) {
                    exhausted = true;
                    break;
                }
                t_q = (int)tl.q[tile];
                t_begin = tl.begin[tile];
                t_len = tl.len[tile];
                t_next = 0;
                // prefetch the tile: lane m holds entry m's candidate, bound,
                // state and first two candidate rows
                if (lane < t_len) {
                    const int64_t e = t_begin + lane;
                    pf_c = cand_of[e];
                    pf_res = res[e];
                    pf_lb = casc ? a.lb[(int64_t)t_q * a.N + pf_c] : T(0);
                    load_pair(pf_pair, a.cands + (int64_t)pf_c * n * D, 0);
                }
                t_thr_raw = a.abandon ? load_volatile(a.thr_src + t_q) : INF;
                if (t_q != staged_q) {
                    __syncwarp();
                    const T* qs = a.queries + (int64_t)t_q * n * D;
                    for (int e = lane; e < (W + 1) * DP; e += 32) {
                        const int col = e / DP, pp = e - (e / DP) * DP;
                        qstage[e] = (col < n) ? T2{__ldg(qs + col * D + 2 * pp),
                                                   (2 * pp + 1 < D) ? __ldg(qs + col * D + 2 * pp + 1) : T(0)}
                                              : T2{INF, INF};
                    }
                    staged_q = t_q;
                    __syncwarp();
                }
            }
            const int take = min(t_len - t_next, __popc(freem));
            const int rank = __popc(freem & ((1u << lane) - 1u));
            const int m = t_next + (rank < take ? rank : 0);  // tile position this lane would take
            const uint32_t c_m = __shfl_sync(FULL, pf_c, m);
            const T lb_m = __shfl_sync(FULL, pf_lb, m);
            const T res_m = __shfl_sync(FULL, pf_res, m);
            T pr_m[2 * D];
#pragma unroll
            for (int u = 0; u < 2 * D; ++u) pr_m[u] = __shfl_sync(FULL, pf_pair[u], m);
            if (!busy && rank < take && !(res_m < T(0))) {  // skip entries pruned by the advanced bound
                if (t_q != cq) {
                    flush();
                    cq = t_q;
                }
                q = t_q;
                ent = t_begin + m;
                crow = a.cands + (int64_t)c_m * n * D;
                qser = a.queries + (int64_t)q * n * D;
                lbtot = lb_m;
                prefix = T(0);
                thr = a.abandon ? scale_up<T>(t_thr_raw, a.mg) : INF;
                thr_pend_raw = t_thr_raw;
#pragma unroll
                for (int k = 0; k < B; ++k) prev[k] = (k == W) ? T(0) : INF;
                // ring: column k-W in slot k (INF for k < W), from the staged copy
#pragma unroll
                for (int k = 0; k < W; ++k)
#pragma unroll
                    for (int pp = 0; pp < DP; ++pp) ring[(k * DP + pp) * 32] = T2{INF, INF};
#pragma unroll
                for (int k = W; k < B; ++k)
#pragma unroll
                    for (int pp = 0; pp < DP; ++pp) ring[(k * DP + pp) * 32] = qstage[(k - W) * DP + pp];
                if constexpr (!LEAN) {
                    load_col(x1, W + 1);
                    load_col(x2, W + 2);
                    if (casc) {
                        load_env(eu0, el0, 0);
                        load_env(eu1, el1, 1 < n ? 1 : 0);
                    }
                }
#pragma unroll
                for (int p = 0; p < D; ++p) {
                    c0[p] = pr_m[p];
                    c1[p] = pr_m[D + p];
                }
                T nx[2 * D];
                load_pair(nx, crow, 2);
#pragma unroll
                for (int p = 0; p < D; ++p) {
                    n0[p] = nx[p];
                    n1[p] = nx[D + p];
                }
                i = 0;
                h = 0;
                since = 0;
                busy = true;
            }
            t_next += take;
            freem = __ballot_sync(FULL, !busy);
        }
    };
    // two rows (i, i+1): P = row i-1 band in, row i out; N = row i+1 out
    auto step = [&](T (&P)[B], T (&N)[B]) {
        const bool two = (i + 1 < n);
        T rmin0, rmin1;
        if constexpr (LEAN) load_col(x1, i + W + 1);
        dtw_step2<T, D, B, EXACT>(P, N, c0, c1, ring, h, x1, rmin0, rmin1);
        if constexpr (LEAN) load_col(x2, i + W + 2);
        // cascade terms of rows i, i+1 from envelope rows loaded a step ago
        T suf0 = T(0), suf1 = T(0);
        if constexpr (LEAN) {
            if (casc) {
                load_env(eu0, el0, i);
                load_env(eu1, el1, i + 1 < n ? i + 1 : i);
            }
        }
        if (casc) {
            prefix += lb_term(c0, eu0, el0);
            suf0 = tmax(lbtot * a.casc_lo - prefix * a.casc_hi, T(0));
            if (two) {
                prefix += lb_term(c1, eu1, el1);
                suf1 = tmax(lbtot * a.casc_lo - prefix * a.casc_hi, T(0));
            }
        }
        const T bound0 = rmin0 + suf0, bound1 = rmin1 + suf1;
        int stop = -1;
        bool abandoned = false;
        T fin = INF;
        if (rmin0 > thr || bound0 > thr * a.casc_thr) {
            stop = i;
            abandoned = true;
        } else if (!two) {  // row i is the last row
            stop = i;
#pragma unroll
            for (int k = 0; k < B; ++k)
                if (k == W) fin = P[k];
            abandoned = fin > thr;  // dtw.py:101-102
        } else if (rmin1 > thr || bound1 > thr * a.casc_thr) {
            stop = i + 1;
            abandoned = true;
        } else if (i + 1 == n - 1) {
            stop = i + 1;
#pragma unroll
            for (int k = 0; k < B; ++k)
                if (k == W) fin = N[k];
            abandoned = fin > thr;
        }
        if (stop >= 0) {
            res[ent] = abandoned ? INF : fin;
            if (!abandoned) {
                atomic_min_nonneg<T>(a.dbest + q, fin);
                note_done(a, q, ent);
            }
            ++c_comp;
            c_ab += abandoned ? 1 : 0;
            c_cells += cells_upto(stop, n, W);
            busy = false;
            return;
        }
        // slide two columns: i+W+1 -> slot of i-W (h), i+W+2 -> slot of i-W+1
        put_col(h, x1);
        put_col(h + 1 == B ? 0 : h + 1, x2);
        i += 2;
        h += 2;
        h = h >= B ? h - B : h;
#pragma unroll
        for (int p = 0; p < D; ++p) {
            c0[p] = n0[p];
            c1[p] = n1[p];
        }
        if (i + 2 < n) {
            T nx[2 * D];
            load_pair(nx, crow, i + 2);
#pragma unroll
            for (int p = 0; p < D; ++p) {
                n0[p] = nx[p];
                n1[p] = nx[D + p];
            }
        }
        // operands of the next step, consumed after its DP
        if constexpr (!LEAN) {
            load_col(x1, i + W + 1);
            load_col(x2, i + W + 2);
            if (casc) {
                load_env(eu0, el0, i);
                load_env(eu1, el1, i + 1 < n ? i + 1 : i);
            }
        }
        since += 2;
        if (since >= 8) {
            // the best-so-far read issued 8 rows ago; issue the next one
            since = 0;
            thr = scale_up<T>(thr_pend_raw, a.mg);
            if (a.abandon) thr_pend_raw = load_volatile(a.thr_src + q);
        }
    };
    // One copy of the step keeps the body inside the 32 KB L1.5 I-cache;
    // row i+1's band moves back into bandA (B register moves per two rows).
    while (true) {
        refill(bandA);
        if (!__any_sync(FULL, busy) && exhausted) break;
        c_issued += 2 * B;
        if (busy) {
            step(bandA, bandB);
#pragma unroll
            for (int k = 0; k < B; ++k) bandA[k] = bandB[k];
        }
    }
    flush();
}

// (T, d, 2W+1) shapes served by dtw_lane_kernel; others use the lockstep
// kernels below.  C0: (double,3,25); C1a: (float,5,25); C2: (float,20,13);
// C4: (float,6,25).
#define TCDTW_LANE_SPECS(X) \
    X(float, 3, 25) X(float, 4, 25) X(float, 5, 25) X(float, 6, 25) X(float, 8, 25) \
    X(float, 3, 13) X(float, 5, 13) X(float, 6, 13) X(float, 8, 13) X(float, 20, 13) X(double, 3, 25)

template <typename T>
static int launch_lane(const SArgs<T>& a, int d, int B, Tiles tl, int64_t n_tiles, const uint32_t* cand_of, T* res,
                       int* tctr, cudaStream_t st) {
    constexpr int threads = 64;
    auto go = [&](auto kern, int DD, int BB) -> int {
        int dev = 0, sms = 148, occ = 1;
        const size_t smem = (size_t)(threads / 32) * ((size_t)BB * ((DD + 1) / 2) * 32 + (size_t)(BB / 2 + 1) * ((DD + 1) / 2)) * 2 * sizeof(T);
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (smem > 227 * 1024) return TCDTW_NOT_SUPPORTED;
        if (smem > 48 * 1024 &&
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return TCDTW_NOT_SUPPORTED;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
        if (occ < 1) return TCDTW_NOT_SUPPORTED;
        int64_t grid = (int64_t)occ * sms;
        const int64_t need = (n_tiles + 1) / 2;
        if (grid > need) grid = need;
        cudaMemsetAsync(tctr, 0, sizeof(int), st);
        kern<<<(int)grid, threads, smem, st>>>(a, tl, n_tiles, cand_of, res, tctr);
        return launch_status();
    };
    // 16-byte candidate-row blocks need aligned rows and whole blocks
    const bool base_ok = (reinterpret_cast<uintptr_t>(a.cands) % 16) == 0;
#define TCDTW_LANE_CASE(TT, DD, BB)                                                                      \
    if constexpr (std::is_same<T, TT>::value) {                                                          \
        if (d == DD && B == BB) {                                                                        \
            constexpr size_t VB = sizeof(typename PairLoad<TT, DD>::V);                                  \
            const bool vec = base_ok && (((int64_t)a.n * DD * sizeof(TT)) % VB) == 0;                    \
            if (vec) return go(dtw_lane_kernel<TT, DD, BB, sizeof(TT) == 8, true>, DD, BB);              \
            return go(dtw_lane_kernel<TT, DD, BB, sizeof(TT) == 8, false>, DD, BB);                      \
        }                                                                                                \
    }
    TCDTW_LANE_SPECS(TCDTW_LANE_CASE)
#undef TCDTW_LANE_CASE
    return TCDTW_NOT_SUPPORTED;
}

// ------------------------- DTW, lane per pair, R rows per step (float32)
// Float32 lane kernel for n % R == 0 (R = 4, or 2 for wide points).  A warp
// works on ONE query at a time: it takes whole (chunk, query) survivor
// segments, and the query (padded with W INF columns before and W+8 after)
// and its LB_MV envelope sit in the warp's shared memory.  Each lane runs
// its own pair; a step advances it by R DP rows i..i+R-1: iteration s reads
// query column i - W + s once and applies it to all R rows (row r at band
// slot s - r), so one window-point read serves R cells.  Row i+R-1's band
// replaces row i-1's in place in a per-lane shared-memory row (row 0 reads
// slot s+1 while row R-1 writes slot s-R+1); intermediate rows live in two
// registers each, so the step is a rolled loop of R-iteration blocks with a
// short unrolled prologue and tail (small code, no I-cache misses).
// Abandoning is tested on row i+R-1 only: row minima never decrease down the
// matrix, so the last row of a step is the strongest test of the step.
// Query columns are grouped by R with a two-word pad (2R*DP + 2 words per
// group: an odd number of 8-byte bank pairs) and the envelope by R rows with
// a pad that makes the group an odd number of 16-byte bank quads, so lanes
// on different rows read shared memory with few conflicts.
static __global__ void qpad_kernel(const float* __restrict__ q, int64_t Q, int n, int d, int w, int rows,
                                   float2* __restrict__ out, int dpad) {
    const int DP = (dpad + 1) / 2;  // dpad >= d: the lane kernel's compile-time dimension count
    const int64_t tot = Q * rows * DP;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
        const int pp = (int)(e % DP);
        const int64_t r = (e / DP) % rows, qi = e / ((int64_t)DP * rows);
        const int64_t col = r - w;
        float2 v = make_float2(dev_inf<float>(), dev_inf<float>());
        if (col >= 0 && col < n) {
            const float* src = q + (qi * n + col) * d;
            v.x = (2 * pp < d) ? src[2 * pp] : 0.f;
            v.y = (2 * pp + 1 < d) ? src[2 * pp + 1] : 0.f;
        }
        out[e] = v;
    }
}

template <int D, int R>
struct LaneRLayout {
    static constexpr int DP = (D + 1) / 2;
    static constexpr int QGS = 2 * R * DP + 2;  // words per R-column query group
    static constexpr int EQ = R * D / 4;        // float4s per R-row envelope half (up or lo)
    static constexpr int EGS = 8 * EQ + 4;      // words per R-row envelope group: 2*EQ + 1 (odd) float4s
    static_assert((R * D) % 4 == 0, "R rows of D floats must be whole float4s");
    __host__ __device__ static int q_words(int qrows) { return (((qrows + R - 1) / R) * QGS + 3) & ~3; }
    __host__ __device__ static int e_words(int n) { return (n + R - 1) / R * EGS; }
    __host__ __device__ static int warp_words(int n, int qrows, int B) { return q_words(qrows) + e_words(n) + B * 32; }
};

// Per-warp global scratch of the lane kernel's head batches: the queued
// pairs' band rows and scalars, lane-interleaved (coalesced).
__host__ __device__ inline int laner_scratch_words(int B) { return 2 * B * 32 + 9 * 32; }
constexpr int kLanerMaxWarps = 148 * 32;

template <int D, int B, int R, bool CASC, int MINB>
__global__ void __launch_bounds__(64, MINB) dtw_laner_kernel(SArgs<float> a, Tiles tl, int64_t n_tiles,
                                                             const uint32_t* __restrict__ cand_of,
                                                             float* __restrict__ res, int* __restrict__ tile_ctr) {
    n_tiles = tile_count(tl, n_tiles);
    using L = LaneRLayout<D, R>;
    constexpr int DP = L::DP, QGS = L::QGS, EGS = L::EGS, EQ = L::EQ, RD = R * D;
    // B == 0 / B == 2: the band is a run-time value with 2W % R == B (even W
    // / odd W for R = 4, any W for R = 2): one instantiation per (D, R, B)
    // serves every such window.  The step is prologue (R iterations), JF full
    // blocks and a tail of R + B iterations whose active-row pattern (tail
    // iteration u: rows r >= u - B) does not depend on W; PB is a stand-in
    // band with that pattern for the compile-time tests of the tail.
    // B > 2: everything folds.
    constexpr bool RT = (B == 0 || B == 2);   // B == 2: run-time band with 2W % R == 2 (odd W at R = 4)
    constexpr int PB = RT ? 4 * R + 1 + B : B;
    constexpr int PST = R * ((PB - 1 - R) / R + 1), NTAIL = PB + R - 1 - PST;
    const int Bv = RT ? 2 * a.w + 1 : B;
    const int W = (Bv - 1) / 2;
    const int JF = (Bv - 1 - R) / R;            // full blocks j = 1..JF (all rows inside the band)
    const int ST = R * (JF + 1);                // first tail iteration
    // Head batches: the first HS steps of a pair (rows 0 .. R*HS-1) start at
    // iteration s0 = W - i >= R (earlier columns are < 0), rounded down to a
    // whole block (j0 = s0 / R).  A warp runs them in lockstep for up to 32
    // fresh pairs, so the trimmed iterations are skipped by the whole warp.
    const int HS = (W >= R) ? W / R : 0;
    static_assert(RT || (B >= R + 1 && (B - 1 - R) / R >= 1), "band too narrow for R rows per step");
    extern __shared__ __align__(16) float smem_f[];
    const int n = a.n;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int qrows = a.qpad_rows;
    float* const qs = smem_f + (size_t)wib * L::warp_words(n, qrows, Bv);  // query groups
    float* const es = qs + L::q_words(qrows);                              // envelope groups
    float* const ps = es + L::e_words(n) + lane;                           // band row: slot k at ps[k*32]
    const unsigned FULL = 0xffffffffu;
    const float INF = dev_inf<float>();
    const int thr_mask = a.thr_every - 1;
    const bool casc = CASC && a.lb != nullptr && a.abandon && a.env_up != nullptr && a.cascade;
    const bool heads = HS > 0 && n > R * (HS + 1) && a.lane_scratch != nullptr;
    float* const scr = a.lane_scratch + (size_t)(blockIdx.x * (blockDim.x >> 5) + wib) * laner_scratch_words(Bv);
    // queued pairs (slot = the lane that ran them): band row, result entry,
    // LB_MV total and cascade prefix in scratch; the candidate and the next
    // row stay in that lane's registers q_cand / q_i (the pop's row loads
    // depend on them)
    float* const q_band = scr;
    int* const q_el = reinterpret_cast<int*>(scr + 32 * Bv);
    int* const q_eh = q_el + 32;
    float* const q_lb = scr + 32 * Bv + 64;
    float* const q_pre = scr + 32 * Bv + 96;
    // warp-uniform work state: current tile, reservoir window, query in smem
    int64_t t_begin = 0;
    int t_q = -1, t_len = 0, t_next = 0, r_base = 0, slot_q = -1;
    bool exhausted = false, have_tile = false;
    float t_thr_raw = INF;
    unsigned q_mask = 0;  // queued slots
    uint32_t q_cand = 0;  // candidate and next row of this lane's queued slot
    int q_i = 0;
    int head_h = -1;      // >= 0: a head batch is running, at head step head_h
    // reservoir: lane m holds entry r_base + m of the tile
    uint32_t pf_c = 0;
    float pf_lb = 0.f, pf_res = 0.f;
    // lane state
    int64_t ent = 0;
    int i = -1;  // next row of the lane's pair; < 0: the lane is free
    uint32_t cand = 0;
    float c[RD], nc[RD];
    float thr = INF, thr_pend_raw = INF, lbtot = 0.f, prefix = 0.f;
    int cq = -1;
    // abandons are counted as computed minus the (rare) completions
    unsigned c_comp = 0, c_cells = 0, c_issued = 0;  // flushed before 2^31
    auto flush = [&]() {
        if (cq >= 0) {
            unsigned long long* ctr = reinterpret_cast<unsigned long long*>(a.counters + (int64_t)cq * TCDTW_COUNTERS);
            if (c_comp) {
                atomicAdd(ctr + TCDTW_C_DTW_COMPUTED, (unsigned long long)c_comp);
                atomicAdd(ctr + TCDTW_C_ABANDON_COUNT, (unsigned long long)c_comp);
            }
            if (c_cells) atomicAdd(ctr + TCDTW_C_DTW_CELLS, (unsigned long long)c_cells);
            if (c_issued) atomicAdd(ctr + TCDTW_C_CELLS_ISSUED, (unsigned long long)c_issued);
        }
        c_comp = c_cells = c_issued = 0;
    };
    // a.d < D: the series have fewer dimensions than the instantiation; the
    // missing ones read as 0 on both sides (they add nothing to a distance or
    // an envelope deviation, so every result is unchanged)
    // (run-time-band instantiations only: the compiled buckets keep dd == D
    // a compile-time fact -- the test cost C4 1% of its DTW time)
    const int dd = RT ? a.d : D;
    // n % R != 0 (run-time-band instantiations only): the pair's last n % R
    // rows follow its last full step (tail rows, below); rows past n - 1 read
    // as 0 and a row stride that breaks the 16-byte alignment goes scalar
    const bool vec_rows = dd == D && (!RT || ((n * D) % 4 == 0));
    auto load_rows = [&](float (&dst)[RD], uint32_t cc, int row) {  // rows row..row+R-1, row % R == 0
        if (vec_rows && (!RT || row + R <= n)) {
            const float4* src = reinterpret_cast<const float4*>(a.cands + ((int64_t)cc * n + row) * D);
#pragma unroll
            for (int v = 0; v < RD / 4; ++v) {
                const float4 x = __ldg(src + v);
                dst[4 * v] = x.x;
                dst[4 * v + 1] = x.y;
                dst[4 * v + 2] = x.z;
                dst[4 * v + 3] = x.w;
            }
        } else {
            const float* src = a.cands + ((int64_t)cc * n + row) * dd;
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int p = 0; p < D; ++p) dst[r * D + p] = (p < dd && row + r < n) ? __ldg(src + r * dd + p) : 0.f;
        }
    };
    auto load_reservoir = [&]() {  // entries r_base .. r_base+31 of the tile, one per lane
        if (r_base + lane < t_len) {
            const int64_t e = t_begin + r_base + lane;
            pf_c = cand_of[e];
            pf_res = res[e];
            pf_lb = casc ? a.lb[(int64_t)t_q * a.N + pf_c] : 0.f;
        }
        t_thr_raw = a.abandon ? load_volatile(a.thr_src + t_q) : INF;
    };
    auto load_query = [&](int q) {  // the warp's query slot (all lanes idle)
        __syncwarp();
        const float2* src = a.qpad + (int64_t)q * qrows * DP;
        for (int e = lane; e < qrows * DP; e += 32) {
            const int col = e / DP, pp = e - (e / DP) * DP;
            *reinterpret_cast<float2*>(qs + (col / R) * QGS + (col % R) * 2 * DP + 2 * pp) = src[e];
        }
        if (casc) {
            const float* eu = a.env_up + (int64_t)q * n * dd;
            const float* el = a.env_lo + (int64_t)q * n * dd;
            for (int e = lane; e < n * D; e += 32) {
                const int row = e / D, p = e - (e / D) * D;
                float* g = es + (row / R) * EGS + (row % R) * D + p;
                g[0] = p < dd ? eu[row * dd + p] : 0.f;
                g[4 * EQ] = p < dd ? el[row * dd + p] : 0.f;
            }
        }
        slot_q = q;
        __syncwarp();
    };
    auto start_pair = [&](int64_t e, uint32_t cc, float lb) {  // row 0 of a fresh pair (band init)
        if (t_q != cq) {
            flush();
            cq = t_q;
        }
        ent = e;
        cand = cc;
        lbtot = lb;
        prefix = 0.f;
        thr = a.abandon ? scale_up<float>(t_thr_raw, a.mg) : INF;
        thr_pend_raw = t_thr_raw;
#pragma unroll
        for (int k = 0; k < Bv; ++k) ps[k * 32] = (k == W) ? 0.f : INF;
        load_rows(c, cc, 0);
        i = 0;
    };
    // next tile (warp-uniform); false when none is left
    auto next_tile = [&]() -> bool {
        int64_t tile = 0;
        if (lane == 0) tile = atomicAdd(tile_ctr, 1);
        tile = __shfl_sync(FULL, tile, 0);
        if (tile >= n_tiles) {
            exhausted = true;
            return false;
        }
        t_q = (int)tl.q[tile];
        t_begin = tl.begin[tile];
        t_len = tl.len[tile];
        t_next = 0;
        r_base = 0;
        have_tile = true;
        load_reservoir();
        return true;
    };
    // Body refill: free lanes take queued pairs; with the queue empty, either
    // a head batch starts (heads) or fresh pairs start at row 0 (no heads).
    auto refill = [&]() {
        unsigned freem = __ballot_sync(FULL, i < 0);
        if (freem == 0) return;
        // queued pairs go to any free lane at once (a pop is a few loads); fresh
        // tile entries wait until refill_min lanes are free
        if (q_mask == 0 && __popc(freem) < a.refill_min && freem != FULL) return;
        while (freem) {
            if (q_mask) {  // pop: the rank-th free lane takes the rank-th queued slot
                const int take = min(__popc(q_mask), __popc(freem));
                const int rank = __popc(freem & ((1u << lane) - 1u));
                const int sl = (int)__fns(q_mask, 0, (rank < take ? rank : 0) + 1);
                const uint32_t cs = __shfl_sync(FULL, q_cand, sl);
                const int is = __shfl_sync(FULL, q_i, sl);
                if (i < 0 && rank < take) {
                    if (slot_q != cq) {  // the lane's last pair may belong to the previous query
                        flush();
                        cq = slot_q;
                    }
                    cand = cs;
                    load_rows(c, cand, is);
                    ent = (int64_t)(uint32_t)q_el[sl] | ((int64_t)q_eh[sl] << 32);
                    lbtot = q_lb[sl];
                    prefix = q_pre[sl];
#pragma unroll
                    for (int k = 0; k < Bv; ++k) ps[k * 32] = q_band[k * 32 + sl];
                    const float raw = a.abandon ? load_volatile(a.thr_src + slot_q) : INF;
                    thr = a.abandon ? scale_up<float>(raw, a.mg) : INF;
                    thr_pend_raw = raw;
                    i = is;
                }
                for (int k = 0; k < take; ++k) q_mask &= q_mask - 1;  // the lowest `take` slots are gone
                freem = __ballot_sync(FULL, i < 0);
                continue;
            }
            if (exhausted) return;
            if (!have_tile || t_next >= t_len) {
                have_tile = false;
                if (!next_tile()) return;
            }
            if (t_q != slot_q) {
                // the slot still serves busy lanes of the previous query: drain first
                if (freem != FULL) return;
                load_query(t_q);
            }
            if (heads) {
                // head batch: the busy lanes' pairs go to the queue (the queue
                // is empty here), every lane takes one of the next (up to) 32
                // entries of the tile -- the reservoir window, lane m <-> entry
                // r_base + m (batches consume whole windows) -- and keeps it
                // after the head steps; free lanes pop the queued pairs
                q_mask = __ballot_sync(FULL, i >= 0);
                if (i >= 0) {
                    q_cand = cand;
                    q_i = i;
                    q_el[lane] = (int)(uint32_t)ent;
                    q_eh[lane] = (int)(ent >> 32);
                    q_lb[lane] = lbtot;
                    q_pre[lane] = prefix;
#pragma unroll
                    for (int k = 0; k < Bv; ++k) q_band[k * 32 + lane] = ps[k * 32];
                }
                __syncwarp();
                i = -1;
                const int avail = min(t_len - t_next, 32);
                const int64_t e0 = t_begin + t_next;
                if (lane < avail && !(pf_res < 0.f)) start_pair(e0 + lane, pf_c, pf_lb);
                t_next += avail;
                if (t_next < t_len) {
                    r_base += 32;
                    load_reservoir();
                }
                head_h = 0;
                return;
            }
            // no head batches (short series / narrow band): start at row 0
            if (t_next >= r_base + 32) {
                r_base += 32;
                load_reservoir();
            }
            const int avail = min(t_len, r_base + 32) - t_next;
            const int take = min(avail, __popc(freem));
            const int rank = __popc(freem & ((1u << lane) - 1u));
            const int m = t_next - r_base + (rank < take ? rank : 0);
            const uint32_t c_m = __shfl_sync(FULL, pf_c, m);
            const float lb_m = __shfl_sync(FULL, pf_lb, m);
            const float res_m = __shfl_sync(FULL, pf_res, m);
            if (i < 0 && rank < take && !(res_m < 0.f))  // skip entries pruned by the advanced bound
                start_pair(t_begin + r_base + m, c_m, lb_m);
            t_next += take;
            freem = __ballot_sync(FULL, i < 0);
        }
    };
    float cur[R], prv[R], pu = 0.f, rmin = INF;
    // iteration s of the step: window column i - W + s for rows i..i+R-1.
    // qx: the column's 2*DP words; pk: band slot s.  With `full`, every row is
    // inside the band and row 0's upper neighbour (slot s+1) exists; otherwise
    // s is a compile-time constant after unrolling and the checks fold.
    auto load_x = [&](float (&x)[2 * DP], const float* qx) {
#pragma unroll
        for (int pp = 0; pp < DP; ++pp) {
            const float2 v = *reinterpret_cast<const float2*>(qx + 2 * pp);
            x[2 * pp] = v.x;
            x[2 * pp + 1] = v.y;
        }
    };
    auto iter_x = [&](int s, bool full, const float (&x)[2 * DP], float* pk) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const bool active = full || (s - r >= 0 && s - r <= PB - 1);
            if (!active) {  // not started (all INF) or past the last slot
                prv[r] = cur[r];
                cur[r] = INF;
                continue;
            }
            // one FMA chain per cell (two partial sums measured 3% slower on C4)
            float acc = 0.f;
#pragma unroll
            for (int p = 0; p < D; ++p) {
                const float df = c[r * D + p] - x[p];
                acc = fmaf(df, df, acc);
            }
            const float cost = fast_sqrt(acc);
            float up, dg;
            if (r == 0) {
                up = (full || s + 1 <= PB - 1) ? pk[32] : INF;
                dg = pu;
                pu = up;
            } else {
                up = cur[r - 1];
                dg = prv[r - 1];
            }
            const float v = cost + fminf(fminf(up, dg), cur[r]);
            prv[r] = cur[r];
            cur[r] = v;
            if (r == R - 1) {
                pk[(1 - R) * 32] = v;  // slot s - R + 1
                rmin = fminf(rmin, v);
            }
        }
    };
    auto iter = [&](int s, bool full, const float* qx, float* pk) {
        float x[2 * DP];
        load_x(x, qx);
        iter_x(s, full, x, pk);
    };
    while (true) {
        if (head_h < 0) {
            refill();
            if (!__any_sync(FULL, i >= 0) && exhausted && q_mask == 0) break;
        }
        // head step h: rows i = R h .. with the first (W - i) / R blocks
        // skipped (their columns are < 0); body steps start at block 0
        const int j0 = head_h >= 0 ? (W - R * head_h) / R : 0;
        c_issued += head_h >= 0 ? R * (Bv - R * j0) + R * (R - 1) / 2 : R * Bv;
        if (c_cells >= (1u << 30) || c_issued >= (1u << 30)) flush();
        if (i >= 0) {
            const bool more = i + R < n;
            if (more) load_rows(nc, cand, i + R);  // consumed after the DP
#pragma unroll
            for (int r = 0; r < R; ++r) cur[r] = prv[r] = INF;
            rmin = INF;
            const float* qg = qs + (i / R) * QGS;  // padded column i + s <-> query column i - W + s
            if (j0 == 0) {
                pu = ps[0];
#pragma unroll
                for (int s = 0; s < R; ++s) iter(s, false, qg + s * 2 * DP, ps + s * 32);
            } else {
                pu = ps[j0 * R * 32];
            }
            if constexpr (D <= 8 || MINB <= 5) {
                // the first column of a block is read one block ahead (its
                // consumer was the step's largest stall site: 9% of the samples)
                float xn[2 * DP];
                load_x(xn, qg + (j0 > 1 ? j0 : 1) * QGS);
#pragma unroll 1
                for (int j = j0 > 1 ? j0 : 1; j <= JF; ++j) {
                    const float* qb = qg + j * QGS;
                    float* pb = ps + j * R * 32;
                    iter_x(j * R, true, xn, pb);
                    load_x(xn, qb + QGS);  // block j+1's (or the tail's) first column
#pragma unroll
                    for (int t = 1; t < R; ++t) iter(j * R + t, true, qb + t * 2 * DP, pb + t * 32);
                }
                iter_x(PST, false, xn, ps + ST * 32);
#pragma unroll
                for (int u = 1; u < NTAIL; ++u)
                    iter(PST + u, false, qg + (ST / R + u / R) * QGS + (u % R) * 2 * DP, ps + (ST + u) * 32);
            } else {  // wide points: no registers to spare for the read-ahead
#pragma unroll 1
                for (int j = j0 > 1 ? j0 : 1; j <= JF; ++j) {
                    const float* qb = qg + j * QGS;
                    float* pb = ps + j * R * 32;
#pragma unroll
                    for (int t = 0; t < R; ++t) iter(j * R + t, true, qb + t * 2 * DP, pb + t * 32);
                }
#pragma unroll
                for (int u = 0; u < NTAIL; ++u)
                    iter(PST + u, false, qg + (ST / R + u / R) * QGS + (u % R) * 2 * DP, ps + (ST + u) * 32);
            }
            // cascade: LB_MV terms of rows i..i+R-1 from the envelope group
            float bound = rmin;
            if (casc) {
                const float4* eg = reinterpret_cast<const float4*>(es + (i / R) * EGS);
                float term[R];
#pragma unroll
                for (int r = 0; r < R; ++r) term[r] = 0.f;
#pragma unroll
                for (int v = 0; v < EQ; ++v) {
                    const float4 u4 = eg[v], l4 = eg[EQ + v];
                    const float uu[4] = {u4.x, u4.y, u4.z, u4.w}, ll[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int f = 4 * v + e, r = f / D;
                        const float cv = c[f];
                        const float dv = fmaxf(fmaxf(cv - uu[e], ll[e] - cv), 0.f);
                        term[r] = fmaf(dv, dv, term[r]);
                    }
                }
#pragma unroll
                for (int r = 0; r < R; ++r) prefix += fast_sqrt(term[r]);
                bound = rmin + fmaxf(lbtot * a.casc_lo - prefix * a.casc_hi, 0.f);
            }
            int stop = -1;
            bool abandoned = false;
            float fin = INF;
            if (!more) {  // row i+R-1 is the last row
                stop = n - 1;
                fin = ps[W * 32];
                abandoned = fin > thr;  // dtw.py:101-102
            } else if (rmin > thr || bound > thr * a.casc_thr) {
                stop = i + R - 1;
                abandoned = true;
            }
            if constexpr (RT) {
                if (stop < 0 && n - (i + R) < R) {
                    // the pair's last n % R rows (in nc): one row at a time, in place in the
                    // band row (slot k: diagonal = old slot k, up = old slot k+1, left = new
                    // slot k-1); only DTWs that run to completion get here
                    const int i2 = i + R, rem = n - i2;
#pragma unroll
                    for (int r = 0; r < R - 1; ++r) {
                        if (r < rem) {
                            float left = INF;
                            for (int k = 0; k < Bv; ++k) {
                                const int col = i2 + r + k;  // padded query column
                                float x[2 * DP];
                                load_x(x, qs + (col / R) * QGS + (col % R) * 2 * DP);
                                float acc = 0.f;
#pragma unroll
                                for (int p = 0; p < D; ++p) {
                                    const float df = nc[r * D + p] - x[p];
                                    acc = fmaf(df, df, acc);
                                }
                                const float up = k + 1 < Bv ? ps[(k + 1) * 32] : INF;
                                const float v = fast_sqrt(acc) + fminf(fminf(up, ps[k * 32]), left);
                                ps[k * 32] = v;
                                left = v;
                            }
                        }
                    }
                    c_issued += rem * Bv;
                    stop = n - 1;
                    fin = ps[W * 32];
                    abandoned = fin > thr;  // dtw.py:101-102
                }
            }
            if (stop >= 0) {
                res[ent] = abandoned ? INF : fin;
                if (!abandoned) {
                    atomic_min_nonneg<float>(a.dbest + cq, fin);
                    note_done(a, cq, ent);
                    atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + (int64_t)cq * TCDTW_COUNTERS) +
                                  TCDTW_C_ABANDON_COUNT,
                              ~0ull);  // one completion: -1 (mod 2^64) against the flushed c_comp
                }
                ++c_comp;
                c_cells += cells_upto(stop, n, W);
                i = -1;
            } else {
                i += R;
#pragma unroll
                for (int u = 0; u < RD; ++u) c[u] = nc[u];
                if ((i & thr_mask) == 0) {  // every thr_every rows (a power of two)
                    thr = scale_up<float>(thr_pend_raw, a.mg);
                    if (a.abandon) thr_pend_raw = load_volatile(a.thr_src + cq);
                }
            }
        }
        if (head_h >= 0 && ++head_h == HS) head_h = -1;  // the fresh pairs carry on in their lanes
    }
    flush();
}

// (d, 2W+1, rows per step) shapes served by dtw_laner_kernel
#define TCDTW_LANER_SPECS(X)                                                                          \
    X(3, 25, 4) X(4, 25, 4) X(5, 25, 4) X(6, 25, 4) X(8, 25, 4) X(3, 13, 4) X(4, 13, 4) X(5, 13, 4) \
    X(6, 13, 4) X(8, 13, 4) X(20, 13, 2) X(5, 103, 4)
// run-time band: (d, rows per step, 2W % R); served when W >= R
#define TCDTW_LANER_RT_SPECS(X)                                                                  \
    X(3, 4, 0) X(4, 4, 0) X(5, 4, 0) X(6, 4, 0) X(8, 4, 0) X(3, 4, 2) X(4, 4, 2) X(5, 4, 2) X(6, 4, 2) \
    X(8, 4, 2) X(4, 2, 0) X(6, 2, 0) X(8, 2, 0) X(12, 2, 0) X(16, 2, 0) X(20, 2, 0)

// The lane-kernel instantiation serving a shape: compile-time dimension
// count DD, rows per step, and whether the band is compiled (the (d, 2W+1,
// R) buckets, exact d) or a run-time value (DD >= d, missing dimensions
// zero-padded on the fly).  The smallest DD wins, then a compiled band, then
// 4 rows.
// A run-time band needs W >= R, n >= 2R when n % R != 0 (tail rows) and at least three
// blocks per SM of shared memory (query + envelope + band row per warp);
// longer bands go to the wavefront kernels.
struct LanerPick {
    int dims = 0, rows = 0;
    bool rt = false;
};
static LanerPick laner_pick(int n, int d, int B) {
    LanerPick best;
    auto better = [&](int DD, int RR, bool rt) {
        if (best.dims == 0) return true;
        if (DD != best.dims) return DD < best.dims;
        if (rt != best.rt) return !rt;
        return RR > best.rows;
    };
#define TCDTW_LANER_OK(DD, BB, RR) \
    if (DD == d && B == BB && n % RR == 0 && better(DD, RR, false)) best = LanerPick{DD, RR, false};
    TCDTW_LANER_SPECS(TCDTW_LANER_OK)
#undef TCDTW_LANER_OK
    if (B >= 3) {
        const int W = (B - 1) / 2, qrows = n + 2 * W + 8;
#define TCDTW_LANER_RT_OK(DD, RR, MM)                                                                     \
    if (DD >= d && (n % RR == 0 || n >= 2 * RR) && W >= RR && (2 * W) % RR == MM &&                       \
        (size_t)2 * LaneRLayout<DD, RR>::warp_words(n, qrows, B) * sizeof(float) <= 76 * 1024 &&         \
        better(DD, RR, true))                                                                             \
        best = LanerPick{DD, RR, true};
        TCDTW_LANER_RT_SPECS(TCDTW_LANER_RT_OK)
#undef TCDTW_LANER_RT_OK
    }
    return best;
}
static int laner_any_rows_shape(int n, int d, int B) { return laner_pick(n, d, B).rows; }

static int laner_rows(const SArgs<float>& a, int d, int B) {
    if (a.qpad == nullptr || (reinterpret_cast<uintptr_t>(a.cands) % 16) != 0) return 0;
    return laner_any_rows_shape(a.n, d, B);
}

#ifndef TCDTW_LANER_MINB
#define TCDTW_LANER_MINB 8
#endif
static int launch_laner(const SArgs<float>& a, int d, int B, Tiles tl, int64_t n_tiles, const uint32_t* cand_of,
                        float* res, int* tctr, cudaStream_t st) {
    constexpr int threads = 64;
    if (laner_rows(a, d, B) == 0) return TCDTW_NOT_SUPPORTED;
    auto go = [&](auto kern, int words_per_warp) -> int {
        const size_t smem = (size_t)(threads / 32) * words_per_warp * sizeof(float);
        int dev = 0, sms = 148, occ = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (smem > 227 * 1024) return TCDTW_NOT_SUPPORTED;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return TCDTW_NOT_SUPPORTED;
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
        if (occ < 1) return TCDTW_NOT_SUPPORTED;
        int64_t grid = (int64_t)occ * sms;
        const int64_t need = (n_tiles + 1) / 2;
        if (grid > need) grid = need;
        cudaMemsetAsync(tctr, 0, sizeof(int), st);
        SArgs<float> a4 = a;
        a4.refill_min = 4;  // refill at 2 or 4 free lanes measured equal, 6 and 8 slower (C4)
        kern<<<(int)grid, threads, smem, st>>>(a4, tl, n_tiles, cand_of, res, tctr);
        return launch_status();
    };
    // new pairs load their first rows themselves (no register prefetch in
    // the reservoir): 126 registers at d=6, 16 warps per SM
    const LanerPick pk = laner_pick(a.n, d, B);
#define TCDTW_LANER_CASE(DD, BB, RR)                                                          \
    if (!pk.rt && pk.dims == DD && B == BB && pk.rows == RR) {                                \
        const int ww = LaneRLayout<DD, RR>::warp_words(a.n, a.qpad_rows, BB);                 \
        return go(dtw_laner_kernel<DD, BB, RR, true, (DD >= 12 ? 5 : (BB >= 64 ? 3 : TCDTW_LANER_MINB))>, ww);                  \
    }
    TCDTW_LANER_SPECS(TCDTW_LANER_CASE)
#undef TCDTW_LANER_CASE
#define TCDTW_LANER_RT_CASE(DD, RR, MM)                                                       \
    if (pk.rt && pk.dims == DD && pk.rows == RR && (B - 1) % RR == MM) {                      \
        const int ww = LaneRLayout<DD, RR>::warp_words(a.n, a.qpad_rows, B);                  \
        return go(dtw_laner_kernel<DD, MM, RR, true, (DD >= 12 ? 5 : TCDTW_LANER_MINB)>, ww);                  \
    }
    TCDTW_LANER_RT_SPECS(TCDTW_LANER_RT_CASE)
#undef TCDTW_LANER_RT_CASE
    return TCDTW_NOT_SUPPORTED;
}

// ------------------------------- DTW, warp per pair, anti-diagonal wavefront
// Lane l owns row i0+l of a 32-row chunk and visits its band slot k at step
// tau = k + 2l, so the cell above (slot k+1 of row i-1) arrives from lane
// l-1 by one shuffle at tau-1 and the diagonal cell (slot k) at tau-2.  The
// chunk's last row is handed to the next chunk through shared memory.
// Abandoning (row min > thr) is evaluated per chunk with the first failing
// row selected, which gives the reference's row-granular result.
template <typename T, int DMAX, bool EXACT>
__global__ void __launch_bounds__(256) dtw_wave_kernel(SArgs<T> a, Tiles tl, int64_t n_tiles,
                                                       const uint32_t* __restrict__ cand_of, T* __restrict__ res,
                                                       int* __restrict__ tile_ctr) {
    n_tiles = tile_count(tl, n_tiles);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = a.n, d = a.d, w = a.w, B = 2 * w + 1;
    const int warps = blockDim.x >> 5, wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // query rows with an odd word stride: consecutive lanes read consecutive
    // columns without bank conflicts (fp64 d=8 was 16-way)
    const int SP = (d % 2 == 1) ? d : d + 1;
    T* qs = reinterpret_cast<T*>(smem_raw);                    // (n + 2w) * SP
    T* prow = qs + (size_t)(n + 2 * w) * SP + (size_t)wib * B;  // per warp: B
    __shared__ int64_t tile_s;
    const T INF = dev_inf<T>();
    int64_t cached_q = -1;
    while (true) {
        __syncthreads();
        if (threadIdx.x == 0) tile_s = atomicAdd(tile_ctr, 1);
        __syncthreads();
        const int64_t tile = tile_s;
        if (tile >= n_tiles) break;
        const int64_t q = tl.q[tile];
        const int64_t e0 = tl.begin[tile];
        const int len = tl.len[tile];
        if (q != cached_q) {
            const T* qsrc = a.queries + q * (int64_t)n * d;
            for (int e = threadIdx.x; e < (n + 2 * w) * d; e += blockDim.x) {
                const int r = e / d, p = e - (e / d) * d;
                const int j = r - w;
                qs[r * SP + p] = (j >= 0 && j < n) ? qsrc[(int64_t)j * d + p] : INF;
            }
            cached_q = q;
            __syncthreads();
        }
        for (int slot = wib; slot < len; slot += warps) {
            const int64_t ent = e0 + slot;
            if (res[ent] < T(0)) continue;  // pruned by the advanced bound (warp-uniform)
            const int64_t c = cand_of[ent];
            const T* crow = a.cands + c * (int64_t)n * d;
            for (int k = lane; k < B; k += 32) prow[k] = (k == w) ? T(0) : INF;
            __syncwarp();
            T thr = a.abandon ? scale_up<T>(load_volatile(a.thr_src + q), a.mg) : INF;
            T fin = INF;
            bool abandoned = false;
            int stop_row = n - 1;
            for (int i0 = 0; i0 < n; i0 += 32) {
                const int i = i0 + lane;
                const bool valid = i < n;
                T rp[DMAX];
                load_point<T, DMAX>(rp, crow + (int64_t)(valid ? i : 0) * d, d);
                T mine = INF, got = INF, rmin = INF;
                const int steps = B + 62;
                for (int tau = 0; tau < steps; ++tau) {
                    const int k = tau - 2 * lane;
                    const T got_prev = got;
                    got = __shfl_up_sync(0xffffffffu, mine, 1);
                    const bool act = valid && k >= 0 && k < B;
                    T v = INF;
                    if (act) {
                        T up, dg;
                        if (lane == 0) {
                            up = (k + 1 < B) ? prow[k + 1] : INF;
                            dg = prow[k];
                        } else {
                            up = got;
                            dg = got_prev;
                        }
                        const T* qp = qs + (size_t)(i + k) * SP;
                        T cost;
                        if constexpr (EXACT) {
                            cost = dist_exact<T, DMAX>(rp, qp, d);
                        } else {
                            T s = T(0);
#pragma unroll
                            for (int p = 0; p < DMAX; ++p)
                                if (p < d) {
                                    const T df = rp[p] - qp[p];
                                    s = fma(df, df, s);
                                }
                            cost = fast_sqrt(s);
                        }
                        const T best = tmin(tmin(up, dg), mine);
                        v = EXACT ? add_rn(cost, best) : cost + best;
                        rmin = tmin(rmin, v);
                        if (i == n - 1 && k == w) fin = v;
                    }
                    mine = v;
                    __syncwarp();
                    if (act && (lane == 31 || i == n - 1)) prow[k] = v;
                    __syncwarp();
                }
                const unsigned bad = __ballot_sync(0xffffffffu, valid && rmin > thr);
                if (bad) {
                    const int first = __ffs(bad) - 1;
                    abandoned = true;
                    stop_row = i0 + first;
                    break;
                }
                if (a.abandon) thr = scale_up<T>(load_volatile(a.thr_src + q), a.mg);
            }
            fin = __shfl_sync(0xffffffffu, fin, (n - 1) & 31);
            if (!abandoned && fin > thr) abandoned = true;  // dtw.py:101-102
            if (lane == 0) {
                res[ent] = abandoned ? INF : fin;
                if (!abandoned) {
                    atomic_min_nonneg<T>(a.dbest + q, fin);
                    note_done(a, q, ent);
                }
                int64_t* ctr = a.counters + q * TCDTW_COUNTERS;
                atomicAdd(reinterpret_cast<unsigned long long*>(ctr + TCDTW_C_DTW_COMPUTED), 1ull);
                if (abandoned) atomicAdd(reinterpret_cast<unsigned long long*>(ctr + TCDTW_C_ABANDON_COUNT), 1ull);
                atomicAdd(reinterpret_cast<unsigned long long*>(ctr + TCDTW_C_DTW_CELLS),
                          (unsigned long long)cells_upto(stop_row, n, w));
            }
            __syncwarp();
        }
    }
}

// Query row layout of dtw_wave_d_kernel: NV 16-byte vectors (VE elements
// each) cover the D values; SP = row stride in elements, an odd number of
// vectors.
template <typename T, int D>
struct WaveRow {
    static constexpr int VE = 16 / (int)sizeof(T);
    static constexpr int NV = (D + VE - 1) / VE;
    static constexpr int SPV = NV % 2 == 1 ? NV : NV + 1;
    static constexpr int SP = SPV * VE;
    using VT = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
};
__host__ inline int wave_row_stride(int es, int d) {
    const int ve = 16 / es, nv = (d + ve - 1) / ve;
    return (nv % 2 == 1 ? nv : nv + 1) * ve;
}

// The same wavefront with the dimension count a compile-time constant and a
// branch-free step (C3: d = 8, 2W+1 = 205; the float32 filter's DTW and the
// float64 EXACT path).  Lane l owns row i0+l of a 32-row chunk and visits its
// band slot k = tau - 2l at step tau; the cell above arrives from lane l-1 by
// the one shuffle per step, the diagonal one step later; lane 0 takes the row
// above from the previous chunk's handoff row.  Per step, per lane:
//   * the query point at column i0 - l - w + tau comes from the staged query,
//     padded with +inf rows so that the address only advances by one row per
//     step (no clamping); lanes outside the band compute on whatever row is
//     there and their result is replaced by +inf;
//   * lane 0 reads one handoff slot (the next step's "up" is this step's
//     "diag"), the handoff row padded with +inf past slot B-1;
//   * float minima are FMNMX (values are never NaN); float64 minima are
//     compare-selects (fmin's NaN handling costs four extra instructions).
// Row-granular abandoning (first row of the chunk whose minimum exceeds the
// threshold) and the float64 arithmetic order are those of dtw_wave_kernel.
// QG: the query is read from global memory (L1) instead of being staged --
// series too long for the staged rows to fit in shared memory.
template <typename T>
__device__ __forceinline__ T step_min(T a, T b) {
    if constexpr (sizeof(T) == 4) return fminf(a, b);
    else return a < b ? a : b;
}

constexpr int kWavePad = 32;  // +inf rows before the staged query (lanes trail lane 0 by <= 31 columns)
__host__ __device__ inline int wave_q_rows(int n, int w) { return n + 2 * w + 2 * kWavePad + 32; }
__host__ __device__ inline int wave_prow_len(int B) { return B + 66; }  // lane 0 reads slot tau+1 <= B + 63

template <typename T, int D, bool EXACT, bool QG = false>
__global__ void __launch_bounds__(256, 2) dtw_wave_d_kernel(SArgs<T> a, Tiles tl, int64_t n_tiles,
                                                         const uint32_t* __restrict__ cand_of, T* __restrict__ res,
                                                         int* __restrict__ tile_ctr) {
    n_tiles = tile_count(tl, n_tiles);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // query rows as whole 16-byte vectors, an odd number of them per row:
    // consecutive lanes read consecutive rows with LDS.128, conflict-free
    // within each quarter warp
    constexpr int SP = WaveRow<T, D>::SP;
    constexpr int VE = WaveRow<T, D>::VE, NV = WaveRow<T, D>::NV;
    using VT = typename WaveRow<T, D>::VT;
    const int n = a.n, w = a.w, B = 2 * w + 1;
    const int PR = wave_prow_len(B);
    const int QR = QG ? 0 : wave_q_rows(n, w);
    const int warps = blockDim.x >> 5, wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    T* qs = reinterpret_cast<T*>(smem_raw);                       // QR * SP: row r <-> query column r - w - kWavePad
    T* prow = qs + (size_t)QR * SP + (size_t)wib * PR;            // per warp handoff row (+inf from slot B on)
    __shared__ int64_t tile_s;
    const T INF = dev_inf<T>();
    const unsigned FULL = 0xffffffffu;
    int64_t cached_q = -1;
    while (true) {
        __syncthreads();
        if (threadIdx.x == 0) tile_s = atomicAdd(tile_ctr, 1);
        __syncthreads();
        const int64_t tile = tile_s;
        if (tile >= n_tiles) break;
        const int64_t q = tl.q[tile];
        const int64_t e0 = tl.begin[tile];
        const int len = tl.len[tile];
        if (!QG && q != cached_q) {
            const T* qsrc = a.queries + q * (int64_t)n * D;
            for (int e = threadIdx.x; e < QR * SP; e += blockDim.x) {
                const int r = e / SP, p = e - (e / SP) * SP;
                const int j = r - w - kWavePad;
                qs[e] = (p < D && j >= 0 && j < n) ? qsrc[(int64_t)j * D + p] : INF;
            }
            cached_q = q;
            __syncthreads();
        }
        for (int slot = wib; slot < len; slot += warps) {
            const int64_t ent = e0 + slot;
            if (res[ent] < T(0)) continue;  // pruned by the advanced bound (warp-uniform)
            const int64_t c = cand_of[ent];
            const T* crow = a.cands + c * (int64_t)n * D;
            for (int k = lane; k < PR; k += 32) prow[k] = (k == w) ? T(0) : INF;
            __syncwarp();
            T thr = a.abandon ? scale_up<T>(load_volatile(a.thr_src + q), a.mg) : INF;
            bool abandoned = false;
            int stop_row = n - 1;
            for (int i0 = 0; i0 < n; i0 += 32) {
                const int i = i0 + lane;
                const bool valid = i < n;
                const bool writer = valid && (lane == 31 || i == n - 1);
                T rp[D];
                {
                    const T* src = crow + (int64_t)(valid ? i : n - 1) * D;
#pragma unroll
                    for (int p = 0; p < D; ++p) rp[p] = src[p];
                }
                const int rows_here = n - i0 < 32 ? n - i0 : 32;
                const int steps = B + 2 * (rows_here - 1);
                T mine = INF, got = INF, rmin = INF;
                T p0 = prow[0];                                          // lane 0: "diag" of step 0
                const T* qrow = qs + (size_t)(i0 - lane + kWavePad) * SP;  // staged row of step 0
                T* wrow = prow - 2 * lane;                                // writer: slot tau - 2 lane
                for (int tau = 0; tau < steps; ++tau) {
                    T qv[NV * VE];
                    if constexpr (QG) {
                        const int col = i0 - lane - w + tau;
                        const bool in = (unsigned)col < (unsigned)n;
                        const T* src = a.queries + ((int64_t)q * n + (in ? col : 0)) * D;
#pragma unroll
                        for (int p = 0; p < D; ++p) qv[p] = in ? __ldg(src + p) : INF;
                    } else {
                        const VT* src = reinterpret_cast<const VT*>(qrow);
#pragma unroll
                        for (int v = 0; v < NV; ++v) {
                            const VT x = src[v];
                            if constexpr (VE == 2) {
                                qv[2 * v] = x.x;
                                qv[2 * v + 1] = x.y;
                            } else {
                                qv[4 * v] = x.x;
                                qv[4 * v + 1] = x.y;
                                qv[4 * v + 2] = x.z;
                                qv[4 * v + 3] = x.w;
                            }
                        }
                        qrow += SP;
                    }
                    T cost;
                    if constexpr (EXACT) {
                        cost = dist_exact<T, D>(rp, qv, D);
                    } else {
                        T sacc = T(0);
#pragma unroll
                        for (int p = 0; p < D; ++p) {
                            const T df = rp[p] - qv[p];
                            sacc = fma(df, df, sacc);
                        }
                        cost = fast_sqrt(sacc);
                    }
                    const T got_prev = got;
                    got = __shfl_up_sync(FULL, mine, 1);
                    T up = got, dg = got_prev;
                    if (lane == 0) {
                        up = prow[tau + 1];  // +inf past the band
                        dg = p0;
                        p0 = up;
                    }
                    const bool act = valid && (unsigned)(tau - 2 * lane) < (unsigned)B;
                    const T best = step_min(step_min(dg, up), mine);
                    T v = EXACT ? add_rn(cost, best) : cost + best;
                    v = act ? v : INF;
                    rmin = step_min(rmin, v);
                    mine = v;
                    if (act && writer) wrow[tau] = v;
                }
                __syncwarp();  // the handoff row is complete for the next chunk
                const unsigned bad = __ballot_sync(FULL, valid && rmin > thr);
                if (bad) {
                    abandoned = true;
                    stop_row = i0 + __ffs(bad) - 1;
                    break;
                }
                if (a.abandon) thr = scale_up<T>(load_volatile(a.thr_src + q), a.mg);
            }
            const T fin = abandoned ? INF : prow[w];  // row n-1, column n-1
            if (!abandoned && fin > thr) abandoned = true;  // dtw.py:101-102
            if (lane == 0) {
                res[ent] = abandoned ? INF : fin;
                if (!abandoned) {
                    atomic_min_nonneg<T>(a.dbest + q, fin);
                    note_done(a, q, ent);
                }
                int64_t* ctr = a.counters + q * TCDTW_COUNTERS;
                atomicAdd(reinterpret_cast<unsigned long long*>(ctr + TCDTW_C_DTW_COMPUTED), 1ull);
                if (abandoned) atomicAdd(reinterpret_cast<unsigned long long*>(ctr + TCDTW_C_ABANDON_COUNT), 1ull);
                atomicAdd(reinterpret_cast<unsigned long long*>(ctr + TCDTW_C_DTW_CELLS),
                          (unsigned long long)cells_upto(stop_row, n, w));
            }
            __syncwarp();
        }
    }
}

// dimension counts with a compile-time wavefront kernel
#define TCDTW_WAVE_DIMS(X) X(3) X(4) X(5) X(6) X(8)

// ------------------------------------------------- advanced bounds (step 2)
// One lane per survivor, the tile's query shared by the warp; evaluated only
// in the trigger band LB_MV > e * d_best (search.py:147).  A survivor whose
// second bound exceeds thr is marked pruned (res = -1).
// LB_TI keeps, per lane, the [L, U] intervals of the distances to the window's
// reference points (the 2W+1 slots) and the column minima; with `ring_smem`
// those rings live in the warp's shared memory (lane-interleaved, conflict
// free) instead of global scratch.
// The LB_MV suffix cascade of the second-stage bounds.  LB_PC, LB_TI and
// LB_AD, like LB_MV, add one nonnegative floor per candidate point, each a
// lower bound of the cheapest window cell that point's DTW row can use; so
// sum_t max(adv_t, mv_t) is a lower bound too, and with the points not yet
// reached bounded by the LB_MV suffix (LB_MV total - LB_MV prefix, the slack
// of the DTW cascade) a pair is dropped as soon as
//   sum_{t < next} max(adv_t, mv_t) + suffix > threshold.
// It only ever prunes more than the reference's bound alone (search.py:163):
// the answers do not change.
template <typename T, int DMAX, bool EXACT>
__device__ __forceinline__ T mv_point(const T (&cp)[DMAX], const T* __restrict__ u, const T* __restrict__ l, int d) {
    if constexpr (EXACT) {
        return lbmv_term_exact<T, DMAX>(cp, u, l, d);
    } else {
        T s = T(0);
#pragma unroll
        for (int p = 0; p < DMAX; ++p)
            if (p < d) {
                const T dv = tmax(tmax(cp[p] - u[p], l[p] - cp[p]), T(0));
                s = fma(dv, dv, s);
            }
        return fast_sqrt(s);
    }
}

template <typename T, bool EXACT>
struct AdvCascade {
    bool on;
    T lbtot, comb = T(0), mv = T(0);
    __device__ __forceinline__ void add(T adv_t, T mv_t) {
        const T m = adv_t > mv_t ? adv_t : mv_t;
        comb = EXACT ? add_rn(comb, m) : comb + m;
        mv = EXACT ? add_rn(mv, mv_t) : mv + mv_t;
    }
    // lower bound of the DTW from the points so far plus the LB_MV suffix
    __device__ __forceinline__ T bound(const SArgs<T>& a) const {
        if (!on) return comb;
        const T suf = lbtot * a.casc_lo - mv * a.casc_hi;
        return comb + (suf > T(0) ? suf : T(0));
    }
    __device__ __forceinline__ bool over(const SArgs<T>& a, T thr) const {
        return on ? bound(a) > thr * a.casc_thr : comb > thr;
    }
};

template <typename T, int DMAX, bool EXACT>
__global__ void __launch_bounds__(256) advanced_kernel(SArgs<T> a, Tiles tl, int64_t n_tiles,
                                                       const uint32_t* __restrict__ cand_of, T* __restrict__ res,
                                                       T* __restrict__ ti_scratch, int* __restrict__ tile_ctr,
                                                       bool ring_smem) {
    n_tiles = tile_count(tl, n_tiles);
    extern __shared__ __align__(16) unsigned char adv_smem[];
    const int n = a.n, d = a.d, w = a.w, B = 2 * w + 1;
    const int lane = threadIdx.x & 31;
    const int64_t gwarp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const T INF = dev_inf<T>();
    while (true) {
        int64_t tile = 0;
        if (lane == 0) tile = atomicAdd(tile_ctr, 1);
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile >= n_tiles) break;
        const int64_t q = tl.q[tile];
        const int64_t ent = tl.begin[tile] + lane;
        const bool has = lane < tl.len[tile];
        const int64_t c = has ? (int64_t)cand_of[ent] : 0;
        const T db = load_volatile(a.thr_src + q);
        const T thr = scale_up<T>(db, a.mg);
        const T lb1 = has ? a.lb[q * a.N + c] : T(0);
        // trigger band: b1 > e * d_best (search.py:147); EXACT uses the
        // reference's float64 product
        bool go = has && (EXACT ? ((double)lb1 > (double)a.trigger * (double)db)
                                : (lb1 > a.trigger * db));
        const T* qa = a.queries + q * (int64_t)n * d;
        const T* ca = a.cands + c * (int64_t)n * d;
        const T* eu = a.env_up ? a.env_up + q * (int64_t)n * d : nullptr;
        const T* el = a.env_lo ? a.env_lo + q * (int64_t)n * d : nullptr;
        AdvCascade<T, EXACT> cas{a.cascade && eu != nullptr, lb1};
        T val = T(0);
        if (a.adv == TCDTW_METHOD_LB_PC) {
            const T* bl = a.box_lo + q * (int64_t)a.G * a.K * d;
            const T* bh = a.box_hi + q * (int64_t)a.G * a.K * d;
            for (int t = 0; t < n && __any_sync(0xffffffffu, go && !cas.over(a, thr)); ++t) {
                T cp[DMAX];
                load_point<T, DMAX>(cp, ca + (int64_t)t * d, d);
                const int g = t / a.gw;
                T best = INF;
                for (int k = 0; k < a.K; ++k) {
                    const T* lo = bl + ((int64_t)g * a.K + k) * d;
                    const T* hi = bh + ((int64_t)g * a.K + k) * d;
                    T v2;
                    if constexpr (EXACT) {
                        v2 = boxdist2_exact<T, DMAX>(cp, lo, hi, d);
                    } else {
                        v2 = T(0);
#pragma unroll
                        for (int p = 0; p < DMAX; ++p)
                            if (p < d) {
                                const T dv = tmax(tmax(lo[p] - cp[p], cp[p] - hi[p]), T(0));
                                v2 = fma(dv, dv, v2);
                            }
                    }
                    best = tmin(best, v2);
                }
                const T pc_t = EXACT ? sqrt_rn(best) : fast_sqrt(best);
                cas.add(pc_t, cas.on ? mv_point<T, DMAX, EXACT>(cp, eu + (int64_t)t * d, el + (int64_t)t * d, d) : T(0));
            }
            val = cas.bound(a);
            if (a.cbox_lo) {
                // reverse LB_PC: the query's points against the candidate's
                // boxes (its own expanded windows), for pairs the forward
                // bound kept; prune on the larger of the two
                const bool fwd_pruned = cas.on ? val > thr * a.casc_thr : val > thr;
                const T* cl = a.cbox_lo + c * (int64_t)a.G * a.K * d;
                const T* ch = a.cbox_hi + c * (int64_t)a.G * a.K * d;
                T rv = T(0);
                bool live = go && !fwd_pruned;
                for (int t = 0; t < n && __any_sync(0xffffffffu, live && rv <= thr); ++t) {
                    T qp[DMAX];
                    load_point<T, DMAX>(qp, qa + (int64_t)t * d, d);
                    const int g = t / a.gw;
                    T best = INF;
                    for (int k = 0; k < a.K; ++k) {
                        const T* lo = cl + ((int64_t)g * a.K + k) * d;
                        const T* hi = ch + ((int64_t)g * a.K + k) * d;
                        T v2;
                        if constexpr (EXACT) {
                            v2 = boxdist2_exact<T, DMAX>(qp, lo, hi, d);
                        } else {
                            v2 = T(0);
#pragma unroll
                            for (int p = 0; p < DMAX; ++p)
                                if (p < d) {
                                    const T dv = tmax(tmax(lo[p] - qp[p], qp[p] - hi[p]), T(0));
                                    v2 = fma(dv, dv, v2);
                                }
                        }
                        best = tmin(best, v2);
                    }
                    rv = EXACT ? add_rn(rv, sqrt_rn(best)) : rv + fast_sqrt(best);
                }
                if (live && rv > thr) val = dev_inf<T>();  // pruned by the reverse bound
            }
        } else if (a.adv == TCDTW_METHOD_LB_AD) {
            for (int t = 0; t < n && __any_sync(0xffffffffu, go && !cas.over(a, thr)); ++t) {
                T cp[DMAX];
                load_point<T, DMAX>(cp, ca + (int64_t)t * d, d);
                const int lo = t - w < 0 ? 0 : t - w;
                const int hi = t + w > n - 1 ? n - 1 : t + w;
                T m = INF;
                for (int j = lo; j <= hi; ++j) {
                    T dj;
                    if constexpr (EXACT) {
                        dj = dist_exact<T, DMAX>(cp, qa + (int64_t)j * d, d);
                    } else {
                        T s = T(0);
#pragma unroll
                        for (int p = 0; p < DMAX; ++p)
                            if (p < d) {
                                const T df = cp[p] - qa[(int64_t)j * d + p];
                                s = fma(df, df, s);
                            }
                        dj = fast_sqrt(s);
                    }
                    m = tmin(m, dj);
                }
                cas.add(m, cas.on ? mv_point<T, DMAX, EXACT>(cp, eu + (int64_t)t * d, el + (int64_t)t * d, d) : T(0));
            }
            val = cas.bound(a);
        } else {
            // LB_TI, TIP_TOP variant (search.py:150-153), lb_ti.py:140-200.
            // Slot rings of size B per lane, interleaved by lane in scratch.
            T* lo_r = ring_smem ? reinterpret_cast<T*>(adv_smem) + (threadIdx.x >> 5) * 3 * (int64_t)B * 32
                                : ti_scratch + gwarp * 3 * (int64_t)B * 32;
            T* up_r = lo_r + (int64_t)B * 32;
            T* cm_r = up_r + (int64_t)B * 32;
            const T* qst = a.qsteps + q * (int64_t)(n - 1);
            T q0[DMAX];
            load_point<T, DMAX>(q0, qa, d);
            int hi = w < n - 1 ? w : n - 1;
            if (go) {
                for (int j = 0; j <= hi; ++j) {
                    T cp[DMAX];
                    load_point<T, DMAX>(cp, ca + (int64_t)j * d, d);
                    T dd;
                    if constexpr (EXACT) dd = dist_exact<T, DMAX>(cp, qa, d);
                    else {
                        T s = T(0);
#pragma unroll
                        for (int p = 0; p < DMAX; ++p) if (p < d) { const T df = cp[p] - q0[p]; s = fma(df, df, s); }
                        dd = fast_sqrt(s);
                    }
                    const int r = j % B;
                    lo_r[r * 32 + lane] = dd;
                    up_r[r * 32 + lane] = dd;
                    cm_r[r * 32 + lane] = dd;
                }
            }
            int next_final = 0, prev_lo = 0, prev_hi = hi;
            bool stop = !go;
            for (int i = 1; i < n && __any_sync(0xffffffffu, !stop); ++i) {
                const int lo = i - w > 0 ? i - w : 0;
                hi = i + w < n - 1 ? i + w : n - 1;
                if (!stop) {
                    T qi[DMAX];
                    load_point<T, DMAX>(qi, qa + (int64_t)i * d, d);
                    auto pdist = [&](int j) -> T {
                        T cp[DMAX];
                        load_point<T, DMAX>(cp, ca + (int64_t)j * d, d);
                        if constexpr (EXACT) return dist_exact<T, DMAX>(cp, qa + (int64_t)i * d, d);
                        T s = T(0);
#pragma unroll
                        for (int p = 0; p < DMAX; ++p) if (p < d) { const T df = cp[p] - qi[p]; s = fma(df, df, s); }
                        return fast_sqrt(s);
                    };
                    if (hi > prev_hi) cm_r[(hi % B) * 32 + lane] = INF;  // a new column enters
                    if (i % a.period == 0) {
                        for (int j = lo; j <= hi; ++j) {
                            const T dd = pdist(j);
                            const int r = j % B;
                            lo_r[r * 32 + lane] = dd;
                            up_r[r * 32 + lane] = dd;
                        }
                    } else {
                        const T s = qst[i - 1];
                        if (s > T(0))
                            for (int j = prev_lo; j <= prev_hi; ++j) {
                                const int r = j % B;
                                T l = lo_r[r * 32 + lane], u = up_r[r * 32 + lane];
                                ti_advance<T>(l, u, s);
                                lo_r[r * 32 + lane] = l;
                                up_r[r * 32 + lane] = u;
                            }
                        if (hi > prev_hi) {
                            const T dd = pdist(hi);
                            const int r = hi % B;
                            lo_r[r * 32 + lane] = dd;
                            up_r[r * 32 + lane] = dd;
                        }
                    }
                    for (int j = lo; j <= hi; ++j) {
                        const int r = j % B;
                        const T l = lo_r[r * 32 + lane];
                        if (l < cm_r[r * 32 + lane]) cm_r[r * 32 + lane] = l;
                    }
                    while (next_final <= i - w) {
                        const T cmv = cm_r[(next_final % B) * 32 + lane];
                        T mvj = T(0);
                        if (cas.on) {
                            T cp[DMAX];
                            load_point<T, DMAX>(cp, ca + (int64_t)next_final * d, d);
                            mvj = mv_point<T, DMAX, EXACT>(cp, eu + (int64_t)next_final * d, el + (int64_t)next_final * d, d);
                        }
                        cas.add(cmv, mvj);
                        ++next_final;
                        if (cas.over(a, thr)) { stop = true; break; }
                    }
                }
                prev_lo = lo;
                prev_hi = hi;
            }
            if (!stop) {
                while (next_final < n) {
                    const T cmv = cm_r[(next_final % B) * 32 + lane];
                    T mvj = T(0);
                    if (cas.on) {
                        T cp[DMAX];
                        load_point<T, DMAX>(cp, ca + (int64_t)next_final * d, d);
                        mvj = mv_point<T, DMAX, EXACT>(cp, eu + (int64_t)next_final * d, el + (int64_t)next_final * d, d);
                    }
                    cas.add(cmv, mvj);
                    ++next_final;
                }
            }
            val = cas.bound(a);
        }
        if (go && (cas.on ? val > thr * a.casc_thr : val > thr)) res[ent] = T(-1);
        int64_t* ctr = a.counters + q * TCDTW_COUNTERS;
        warp_add_counter(ctr + TCDTW_C_ADVANCED_LB_EVALS, go ? 1 : 0);
    }
}

// ------------------------- LB_PC on survivors, boxes staged in shared memory
// Warp per work tile (32 survivors of one query, lane = survivor).  The
// query's box sets (G x K boxes, lb_pc.py:229-234 padding included) are staged
// once per tile query in the warp's shared memory as (lo, hi) pairs; all lanes
// walk the candidate index t in lockstep, so every box read is a broadcast.
// Early exit once every lane's running sum exceeds the threshold.  FAST mode
// only (the float64 path keeps advanced_kernel's exact arithmetic).
template <typename T, int D, bool VEC>
__global__ void __launch_bounds__(256) advanced_pc_kernel(SArgs<T> a, Tiles tl, int64_t n_tiles,
                                                          const uint32_t* __restrict__ cand_of, T* __restrict__ res,
                                                          int* __restrict__ tile_ctr) {
    n_tiles = tile_count(tl, n_tiles);
    using T2 = typename Vec8<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = a.n, G = a.G, K = a.K, gw = a.gw;
    const int lane = threadIdx.x & 31;
    T2* bx = reinterpret_cast<T2*>(smem_raw) + (size_t)(threadIdx.x >> 5) * G * K * D;  // [g][k][p] -> (lo, hi)
    const T INF = dev_inf<T>();
    const unsigned FULL = 0xffffffffu;
    int64_t cached_q = -1;
    while (true) {
        int64_t tile = 0;
        if (lane == 0) tile = atomicAdd(tile_ctr, 1);
        tile = __shfl_sync(FULL, tile, 0);
        if (tile >= n_tiles) break;
        const int64_t q = tl.q[tile];
        const int64_t ent = tl.begin[tile] + lane;
        const bool has = lane < tl.len[tile];
        if (q != cached_q) {
            __syncwarp();
            const T* bl = a.box_lo + q * (int64_t)G * K * D;
            const T* bh = a.box_hi + q * (int64_t)G * K * D;
            for (int e = lane; e < G * K * D; e += 32) bx[e] = T2{bl[e], bh[e]};
            cached_q = q;
            __syncwarp();
        }
        const int64_t c = has ? (int64_t)cand_of[ent] : 0;
        const T db = load_volatile(a.thr_src + q);
        const T thr = scale_up<T>(db, a.mg);
        const T lb1 = has ? a.lb[q * a.N + c] : T(0);
        const bool go = has && !(res[ent] < T(0)) && (lb1 > a.trigger * db);  // trigger band, search.py:147
        const T* crow = a.cands + c * (int64_t)n * D;
        using PL = PairLoad<T, D>;
        const T* eu = a.env_up ? a.env_up + q * (int64_t)n * D : nullptr;
        const T* el = a.env_lo ? a.env_lo + q * (int64_t)n * D : nullptr;
        AdvCascade<T, sizeof(T) == 8> cas{a.cascade && eu != nullptr, lb1};
        // two candidate rows per pass: one vectorised load of 2D values
        for (int t = 0; t < n && __any_sync(FULL, go && !cas.over(a, thr)); t += 2) {
            T cp2[2 * D];
            if (VEC && t + 1 < n) {
                const typename PL::V* src = reinterpret_cast<const typename PL::V*>(crow + (int64_t)t * D);
#pragma unroll
                for (int v = 0; v < PL::nv; ++v) {
                    const typename PL::V x = __ldg(src + v);
                    const T* xs = reinterpret_cast<const T*>(&x);
#pragma unroll
                    for (int u = 0; u < PL::per; ++u) cp2[v * PL::per + u] = xs[u];
                }
            } else {
#pragma unroll
                for (int u = 0; u < 2 * D; ++u) cp2[u] = (t + u / D < n) ? __ldg(crow + (int64_t)t * D + u) : T(0);
            }
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                if (t + r < n) {
                    const T2* gb = bx + (size_t)((t + r) / gw) * K * D;
                    T best = INF;
                    for (int k = 0; k < K; ++k) {
                        T acc = T(0);
#pragma unroll
                        for (int p = 0; p < D; ++p) {
                            const T2 b = gb[k * D + p];
                            const T cv = cp2[r * D + p];
                            const T dv = tmax(tmax(b.x - cv, cv - b.y), T(0));
                            acc = fma(dv, dv, acc);
                        }
                        best = tmin(best, acc);
                    }
                    T mv_t = T(0);
                    if (cas.on) {
                        T cpd[D];
#pragma unroll
                        for (int p = 0; p < D; ++p) cpd[p] = cp2[r * D + p];
                        mv_t = mv_point<T, D, false>(cpd, eu + (int64_t)(t + r) * D, el + (int64_t)(t + r) * D, D);
                    }
                    cas.add(fast_sqrt(best), mv_t);
                }
            }
        }
        if (go && cas.over(a, thr)) res[ent] = T(-1);
        int64_t* ctr = a.counters + q * TCDTW_COUNTERS;
        warp_add_counter(ctr + TCDTW_C_ADVANCED_LB_EVALS, go ? 1 : 0);
    }
}

#define TCDTW_PC_DIMS(X) X(3) X(4) X(5) X(6) X(8) X(20)

template <typename T>
static int launch_advanced_pc(const SArgs<T>& a, int d, Tiles tl, int64_t n_tiles, const uint32_t* cand_of, T* res,
                              int* tctr, cudaStream_t st) {
    if constexpr (sizeof(T) == 8) {
        return TCDTW_NOT_SUPPORTED;
    } else {
        auto go = [&](auto kern, int DD) -> int {
            const size_t smem = (size_t)8 * a.G * a.K * DD * 2 * sizeof(T);
            if (smem > 227 * 1024) return TCDTW_NOT_SUPPORTED;
            if (smem > 48 * 1024 &&
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
                return TCDTW_NOT_SUPPORTED;
            int dev = 0, sms = 148, occ = 1;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
            if (occ < 1) return TCDTW_NOT_SUPPORTED;
            int64_t grid = (int64_t)occ * sms;
            const int64_t need = (n_tiles + 7) / 8;
            if (grid > need) grid = need;
            cudaMemsetAsync(tctr, 0, sizeof(int), st);
            kern<<<(int)grid, 256, smem, st>>>(a, tl, n_tiles, cand_of, res, tctr);
            return launch_status();
        };
        const bool base_ok = (reinterpret_cast<uintptr_t>(a.cands) % 16) == 0;
#define TCDTW_PC_CASE(DD)                                                                                   \
        if (d == DD) {                                                                                      \
            const bool vec = base_ok && (((int64_t)a.n * DD * sizeof(T)) % sizeof(typename PairLoad<T, DD>::V)) == 0; \
            return vec ? go(advanced_pc_kernel<T, DD, true>, DD) : go(advanced_pc_kernel<T, DD, false>, DD); \
        }
        TCDTW_PC_DIMS(TCDTW_PC_CASE)
#undef TCDTW_PC_CASE
        return TCDTW_NOT_SUPPORTED;
    }
}

// --------------------------------------------------------------- finalize
// F1: per query minimum of completed DTWs (seeds and survivors).
template <typename T>
__global__ void fin_min_kernel(Tiles tl, int64_t n_tiles, const T* __restrict__ res, T* __restrict__ minv,
                               const unsigned long long* __restrict__ done_cnt, int64_t done_cap) {
    n_tiles = tile_count(tl, n_tiles);
    if (done_cnt && (int64_t)*done_cnt <= done_cap) return;  // the completed list covers it
    for (int64_t tile = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); tile < n_tiles;
         tile += (int64_t)gridDim.x * (blockDim.x >> 5)) {
        const int lane = threadIdx.x & 31;
        const int64_t q = tl.q[tile];
        T v = dev_inf<T>();
        if (lane < tl.len[tile]) {
            const T r = res[tl.begin[tile] + lane];
            if (r >= T(0)) v = r;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = tmin(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0 && v < dev_inf<T>()) atomic_min_nonneg<T>(minv + q, v);
    }
}

// EXACT float64 DTW of one pair by one thread; band rows in `scratch`
// (2 * (2w+1) doubles).  Same arithmetic as dtw_pairs_kernel.
template <int DMAX, typename TIn>
__device__ double dtw_exact_thread(const TIn* qa, const TIn* ca, int n, int d, int w, double* scratch) {
    const int width = 2 * w + 1;
    double* prev = scratch;
    double* cur = scratch + width;
    const double INF = dev_inf<double>();
    for (int k = 0; k < width; ++k) prev[k] = INF;
    for (int i = 0; i < n; ++i) {
        const int lo = i < w ? 0 : i - w;
        const int hi = i + w >= n ? n - 1 : i + w;
        for (int k = 0; k < width; ++k) cur[k] = INF;
        double qi[DMAX];
#pragma unroll
        for (int p = 0; p < DMAX; ++p) qi[p] = p < d ? (double)qa[(int64_t)i * d + p] : 0.0;
        int k = lo - i + w;
        for (int j = lo; j <= hi; ++j, ++k) {
            double sq[DMAX];
#pragma unroll
            for (int p = 0; p < DMAX; ++p) {
                if (p < d) {
                    const double df = __dsub_rn(qi[p], (double)ca[(int64_t)j * d + p]);
                    sq[p] = __dmul_rn(df, df);
                } else {
                    sq[p] = 0.0;
                }
            }
            const double cost = __dsqrt_rn(np_sum<double, DMAX>(sq, d));
            double v;
            if (i == 0 && j == 0) {
                v = cost;
            } else {
                double best = INF;
                if (i > 0) {
                    if (k + 1 < width) best = prev[k + 1];
                    if (j > 0 && prev[k] < best) best = prev[k];
                }
                if (k > 0 && cur[k - 1] < best) best = cur[k - 1];
                v = __dadd_rn(cost, best);
            }
            cur[k] = v;
        }
        double* t = prev;
        prev = cur;
        cur = t;
    }
    return prev[w];
}

// F2/F3 (FAST): finalists (float32 DTW within the margin of the best) are
// re-scored in float64; pass 0 takes the minimum, pass 1 the lowest index
// attaining it.  EXACT: pass 1 only, on the stored exact values.
template <typename T, int DMAX>
__device__ __forceinline__ void rescore_entry(const SArgs<T>& a, int64_t q, int64_t ent,
                                              const uint32_t* __restrict__ cand_of, const T* __restrict__ res,
                                              const T* __restrict__ minv, const T* __restrict__ dbest_in, int pass,
                                              unsigned long long* __restrict__ min64,
                                              unsigned long long* __restrict__ best_idx, double* my_scratch) {
    const T r = res[ent];
    if (!(r >= T(0)) || r == dev_inf<T>()) return;
    const uint32_t c = cand_of[ent];
    if constexpr (sizeof(T) == 8) {
        // EXACT: stored values are the reference's
        if (r == minv[q]) atomicMin(best_idx + q, (unsigned long long)c);
    } else {
        T bound = minv[q];
        if (dbest_in) bound = tmin(bound, dbest_in[q]);
        const T thr = fin_up(bound, a.mg);
        if (!(r <= thr)) return;
        const int64_t qo = q * (int64_t)a.n * a.d, co = (int64_t)c * a.n * a.d;
        const double d64 = a.xq ? dtw_exact_thread<DMAX, double>(a.xq + qo, a.xc + co, a.n, a.d, a.w, my_scratch)
                                : dtw_exact_thread<DMAX, T>(a.queries + qo, a.cands + co, a.n, a.d, a.w, my_scratch);
        const unsigned long long bits = (unsigned long long)__double_as_longlong(d64);
        if (pass == 0) {
            atomicMin(min64 + q, bits);
            atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + q * TCDTW_COUNTERS + TCDTW_C_FINALISTS), 1ull);
        } else if (bits == min64[q]) {
            atomicMin(best_idx + q, (unsigned long long)c);
        }
    }
}

template <typename T, int DMAX>
__global__ void fin_rescore_kernel(SArgs<T> a, Tiles tl, int64_t n_tiles, const uint32_t* __restrict__ cand_of,
                                   const T* __restrict__ res, const T* __restrict__ minv, const T* __restrict__ dbest_in,
                                   int pass, unsigned long long* __restrict__ min64,
                                   unsigned long long* __restrict__ best_idx, double* __restrict__ scratch,
                                   const unsigned long long* __restrict__ done_cnt, int64_t done_cap) {
    n_tiles = tile_count(tl, n_tiles);
    if (done_cnt && (int64_t)*done_cnt <= done_cap) return;  // the completed list covers it
    const int lane = threadIdx.x & 31;
    const int64_t gthread = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int width = 2 * a.w + 1;
    double* my_scratch = scratch + gthread * 2 * (int64_t)width;
    for (int64_t tile = gthread >> 5; tile < n_tiles; tile += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t q = tl.q[tile];
        const bool has = lane < tl.len[tile];
        const int64_t ent = tl.begin[tile] + lane;
        if (!has) continue;
        rescore_entry<T, DMAX>(a, q, ent, cand_of, res, minv, dbest_in, pass, min64, best_idx, my_scratch);
    }
}

// The same over the completed list (q << 40 | entry), one thread per item.
template <typename T>
__global__ void fin_min_list_kernel(const unsigned long long* __restrict__ list,
                                    const unsigned long long* __restrict__ done_cnt, int64_t done_cap,
                                    const T* __restrict__ res, T* __restrict__ minv) {
    const int64_t cnt = (int64_t)*done_cnt;
    if (cnt > done_cap) return;  // overflowed: the tile kernels run instead
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < cnt; k += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long x = list[k];
        const int64_t q = (int64_t)(x >> 40), ent = (int64_t)(x & ((1ull << 40) - 1));
        const T r = res[ent];
        if (r >= T(0) && r < dev_inf<T>()) atomic_min_nonneg<T>(minv + q, r);
    }
}

template <typename T, int DMAX>
__global__ void fin_rescore_list_kernel(SArgs<T> a, const unsigned long long* __restrict__ list,
                                        const unsigned long long* __restrict__ done_cnt, int64_t done_cap,
                                        const uint32_t* __restrict__ cand_of, const T* __restrict__ res,
                                        const T* __restrict__ minv, const T* __restrict__ dbest_in, int pass,
                                        unsigned long long* __restrict__ min64, unsigned long long* __restrict__ best_idx,
                                        double* __restrict__ scratch) {
    const int64_t cnt = (int64_t)*done_cnt;
    if (cnt > done_cap) return;
    const int64_t gthread = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double* my_scratch = scratch + gthread * 2 * (int64_t)(2 * a.w + 1);
    for (int64_t k = gthread; k < cnt; k += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long x = list[k];
        rescore_entry<T, DMAX>(a, (int64_t)(x >> 40), (int64_t)(x & ((1ull << 40) - 1)), cand_of, res, minv, dbest_in,
                               pass, min64, best_idx, my_scratch);
    }
}

// --- finalists: collected once, re-scored by one warp each, picked ----------
// A finalist is a completed DTW whose float32 value is within the margin of
// the best (FAST), or equal to the best (EXACT).  (q << 40 | entry) with the
// candidate index kept alongside.
struct Finalists {
    unsigned long long* item;  // (q << 40) | candidate
    double* d64;               // float64 DTW (FAST) / stored value (EXACT)
    unsigned long long* cnt;
    int64_t cap;
};

template <typename T>
__device__ __forceinline__ void collect_entry(const SArgs<T>& a, int64_t q, T r, uint32_t c,
                                              const T* __restrict__ minv, const T* __restrict__ dbest_in,
                                              Finalists f) {
    if (!(r >= T(0)) || r == dev_inf<T>()) return;
    bool take;
    if constexpr (sizeof(T) == 8) {
        take = (r == minv[q]);
    } else {
        T bound = minv[q];
        if (dbest_in) bound = tmin(bound, dbest_in[q]);
        take = r <= fin_up(bound, a.mg);
    }
    if (!take) return;
    const unsigned long long k = atomicAdd(f.cnt, 1ull);
    if ((int64_t)k < f.cap) {
        f.item[k] = ((unsigned long long)q << 40) | (unsigned long long)c;
        f.d64[k] = (double)r;
    }
}

// seeds (tile list) and the completed survivors (done list) -> finalists
template <typename T>
__global__ void fin_collect_kernel(SArgs<T> a, Tiles stl, int64_t n_seed_tiles, const uint32_t* __restrict__ seeds,
                                   const T* __restrict__ seedres, const unsigned long long* __restrict__ list,
                                   const unsigned long long* __restrict__ done_cnt, int64_t done_cap,
                                   const uint32_t* __restrict__ cand_of, const T* __restrict__ res,
                                   const T* __restrict__ minv, const T* __restrict__ dbest_in, Finalists f) {
    const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = gt; k < n_seed_tiles * 32; k += stride) {
        const int64_t tile = k >> 5;
        const int lane = (int)(k & 31);
        if (lane < stl.len[tile]) {
            const int64_t ent = stl.begin[tile] + lane;
            collect_entry<T>(a, stl.q[tile], seedres[ent], seeds[ent], minv, dbest_in, f);
        }
    }
    if (list == nullptr) return;
    const int64_t cnt = (int64_t)*done_cnt;
    if (cnt > done_cap) return;
    for (int64_t k = gt; k < cnt; k += stride) {
        const unsigned long long x = list[k];
        const int64_t q = (int64_t)(x >> 40), ent = (int64_t)(x & ((1ull << 40) - 1));
        collect_entry<T>(a, q, res[ent], cand_of[ent], minv, dbest_in, f);
    }
}

// EXACT float64 DTW of one (query, candidate) pair by one warp: lane = row of
// a 32-row chunk, anti-diagonal skew of 2 per lane, one shuffle per step, the
// chunk's last row handed over through shared memory (prow, 2W+2 doubles, the
// last one +inf).  Same per-cell arithmetic as dtw_banded (numpy order, no
// contraction).  Branch-free steps with the NEXT step's cell cost computed
// ahead, so the correctly rounded square root (the long pole) overlaps the
// min/add recurrence instead of sitting on it; lanes outside the band work
// on clamped indices and their result is replaced by +inf.
template <typename TIn, typename TCol, int DMAX, bool VEC = false>
__device__ double dtw_warp_exact(const TIn* __restrict__ rows_s, const TCol* __restrict__ cols_s, int col_stride,
                                 int n, int d, int w, double* prow) {
    const int lane = threadIdx.x & 31;
    const int B = 2 * w + 1;
    const double INF = dev_inf<double>();
    const unsigned FULL = 0xffffffffu;
    for (int k = lane; k <= B; k += 32) prow[k] = (k == w) ? 0.0 : INF;
    __syncwarp();
    for (int i0 = 0; i0 < n; i0 += 32) {
        const int i = i0 + lane;
        const bool valid = i < n;
        const bool writer = valid && (lane == 31 || i == n - 1);
        double rp[DMAX];
        {
            const TIn* src = rows_s + (int64_t)(valid ? i : n - 1) * d;
#pragma unroll
            for (int p = 0; p < DMAX; ++p) rp[p] = p < d ? (double)src[p] : 0.0;
        }
        // cost of this lane's cell at step tau: slot k = tau - 2 lane
        auto cost_at = [&](int tau) -> double {
            const int k = tau - 2 * lane;
            const int j = i - w + k;
            const bool in = valid && (unsigned)k < (unsigned)B && (unsigned)j < (unsigned)n;
            const TCol* col = cols_s + (int64_t)(in ? j : 0) * col_stride;
            double cv[DMAX];
            if constexpr (VEC && sizeof(TCol) == 8) {  // staged rows: 16-byte aligned, odd 16-byte stride
#pragma unroll
                for (int p = 0; p + 1 < DMAX; p += 2) {
                    if (p + 1 < d) {
                        const double2 v2 = *reinterpret_cast<const double2*>(col + p);
                        cv[p] = v2.x;
                        cv[p + 1] = v2.y;
                    } else if (p < d) {
                        cv[p] = (double)col[p];
                    }
                }
                if (DMAX % 2 == 1 && DMAX - 1 < d) cv[DMAX - 1] = (double)col[DMAX - 1];
            } else {
#pragma unroll
                for (int p = 0; p < DMAX; ++p)
                    if (p < d) cv[p] = (double)col[p];
            }
            double sq[DMAX];
#pragma unroll
            for (int p = 0; p < DMAX; ++p) {
                if (p < d) {
                    const double df = __dsub_rn(rp[p], cv[p]);
                    sq[p] = __dmul_rn(df, df);
                } else {
                    sq[p] = 0.0;
                }
            }
            const double c = __dsqrt_rn(np_sum<double, DMAX>(sq, d));
            return in ? c : INF;
        };
        const int rows_here = n - i0 < 32 ? n - i0 : 32;
        const int steps = B + 2 * (rows_here - 1);
        double mine = INF, got = INF;
        double cost = cost_at(0);
        for (int tau = 0; tau < steps; ++tau) {
            const double cost_next = cost_at(tau + 1);  // independent of the recurrence below
            const int k = tau - 2 * lane;
            const double got_prev = got;
            got = __shfl_up_sync(FULL, mine, 1);
            const bool act = valid && (unsigned)k < (unsigned)B;
            const int kc = k < 0 ? 0 : (k > B - 1 ? B - 1 : k);
            double up = got, dg = got_prev;
            if (lane == 0) {
                up = prow[kc + 1];  // prow[B] = +inf
                dg = prow[kc];
            }
            // compare-select minima: never NaN, equal operands are equal values
            const double m1 = dg < up ? dg : up;
            const double best = mine < m1 ? mine : m1;
            double v = __dadd_rn(cost, best);
            v = act ? v : INF;
            mine = v;
            if (act && writer) prow[k] = v;
            cost = cost_next;
        }
        __syncwarp();  // the handoff row is complete for the next chunk
    }
    const double fin = prow[w];  // row n-1, column n-1
    __syncwarp();
    return fin;
}

// Doubles per staged query point: pairs of doubles (16 bytes), an odd number
// of them, so lanes reading consecutive points with 16-byte loads do not
// conflict.
__host__ __device__ inline int rescore_col_stride(int d) {
    const int units = (d + 1) / 2;
    return 2 * (units % 2 == 1 ? units : units + 1);
}

// One warp per finalist.  STAGE: the finalist's query (the DP's columns,
// read at every step) is first copied into the warp's shared memory as
// float64 with rescore_col_stride; else it is read from global memory.
template <typename T, int DMAX, bool STAGE>
__global__ void fin_rescore_warp_kernel(SArgs<T> a, Finalists f, unsigned long long* __restrict__ min64) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warps = blockDim.x >> 5, wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cs = rescore_col_stride(a.d);
    const size_t per_warp = (STAGE ? (size_t)a.n * cs : 0) + (size_t)(2 * a.w + 2);
    double* qs = reinterpret_cast<double*>(smem_raw) + (size_t)wib * per_warp;
    double* prow = qs + (STAGE ? (size_t)a.n * cs : 0);
    const int64_t cnt = min((int64_t)*f.cnt, f.cap);
    for (int64_t k = blockIdx.x * (int64_t)warps + wib; k < cnt; k += (int64_t)gridDim.x * warps) {
        const unsigned long long x = f.item[k];
        const int64_t q = (int64_t)(x >> 40), c = (int64_t)(x & ((1ull << 40) - 1));
        double d64;
        if constexpr (sizeof(T) == 8) {
            d64 = f.d64[k];  // EXACT: the stored value is the reference's
        } else {
            // DTW is symmetric (test_dtw.py:196-207): rows = candidate.  With
            // the float32 filter on float64 data, the float64 originals.
            const int64_t qo = q * (int64_t)a.n * a.d, co = c * (int64_t)a.n * a.d;
            if constexpr (STAGE) {
                __syncwarp();
                for (int e = lane; e < a.n * a.d; e += 32) {
                    const int r = e / a.d, p = e - r * a.d;
                    qs[r * cs + p] = a.xq ? a.xq[qo + e] : (double)a.queries[qo + e];
                }
                __syncwarp();
                d64 = a.xq ? dtw_warp_exact<double, double, DMAX, true>(a.xc + co, qs, cs, a.n, a.d, a.w, prow)
                           : dtw_warp_exact<T, double, DMAX, true>(a.cands + co, qs, cs, a.n, a.d, a.w, prow);
            } else {
                d64 = a.xq ? dtw_warp_exact<double, double, DMAX>(a.xc + co, a.xq + qo, a.d, a.n, a.d, a.w, prow)
                           : dtw_warp_exact<T, T, DMAX>(a.cands + co, a.queries + qo, a.d, a.n, a.d, a.w, prow);
            }
        }
        if (lane == 0) {
            f.d64[k] = d64;
            atomicMin(min64 + q, (unsigned long long)__double_as_longlong(d64));
            if constexpr (sizeof(T) == 4)
                atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + q * TCDTW_COUNTERS + TCDTW_C_FINALISTS),
                          1ull);
        }
    }
}

static __global__ void fin_pick_kernel(Finalists f, const unsigned long long* __restrict__ min64,
                                unsigned long long* __restrict__ best_idx) {
    const int64_t cnt = min((int64_t)*f.cnt, f.cap);
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < cnt; k += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long x = f.item[k];
        const int64_t q = (int64_t)(x >> 40);
        if ((unsigned long long)__double_as_longlong(f.d64[k]) == min64[q])
            atomicMin(best_idx + q, x & ((1ull << 40) - 1));
    }
}

template <typename T>
__global__ void fin_output_kernel(int64_t Q, int64_t N, int64_t base, const T* __restrict__ minv,
                                  const unsigned long long* __restrict__ min64,
                                  const unsigned long long* __restrict__ best_idx, const int64_t* __restrict__ ctr,
                                  int has_lb, int64_t* __restrict__ out_idx, double* __restrict__ out_dist,
                                  int64_t* __restrict__ out_ctr) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < Q; q += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long bi = best_idx[q];
        double dist;
        if constexpr (sizeof(T) == 8) dist = (double)minv[q];
        else dist = __longlong_as_double((long long)min64[q]);
        if (bi == 0xffffffffffffffffull) {
            out_idx[q] = -1;
            out_dist[q] = dev_inf<double>();
        } else {
            out_idx[q] = (int64_t)bi + base;
            out_dist[q] = dist;
        }
        const int64_t* c = ctr + q * TCDTW_COUNTERS;
        int64_t* o = out_ctr ? out_ctr + q * TCDTW_COUNTERS : nullptr;
        if (o) {
            for (int k = 0; k < TCDTW_COUNTERS; ++k) o[k] = c[k];
            o[TCDTW_C_DTW_SKIPPED] = N - c[TCDTW_C_DTW_COMPUTED];
            o[TCDTW_C_LB_MV_EVALS] = has_lb ? N : 0;
        }
    }
}

template <typename T>
__global__ void fill_kernel(T* p, int64_t n, T v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

// ----------------------------------------------------------- ALU probe
template <typename T>
__global__ void alu_probe_kernel(int iters, T* sink) {
    T a0 = T(threadIdx.x) * T(1e-7), a1 = a0 + T(1), a2 = a0 + T(2), a3 = a0 + T(3);
    T a4 = a0 + T(4), a5 = a0 + T(5), a6 = a0 + T(6), a7 = a0 + T(7);
    const T m = T(0.999999), c = T(1e-7);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
            a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
        }
    }
    if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == T(-1)) sink[0] = a0;
}

// ------------------------------------------- float32 filter on float64 data
// Rounded float32 copy of (points, d) float64 values and the largest squared
// point norm (nonnegative doubles order like their bit patterns).
static __global__ void round_points_kernel(const double* __restrict__ in, int64_t points, int d, float* __restrict__ out,
                                    unsigned long long* __restrict__ max_sq_bits) {
    double mx = 0.0;
    for (int64_t pt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pt < points;
         pt += (int64_t)gridDim.x * blockDim.x) {
        const double* x = in + pt * d;
        float* y = out + pt * d;
        double s = 0.0;
        for (int k = 0; k < d; ++k) {
            const double v = x[k];
            y[k] = __double2float_rn(v);
            s = fma(v, v, s);
        }
        mx = fmax(mx, s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(max_sq_bits, (unsigned long long)__double_as_longlong(mx));
}

// Additive slack of the float32 decisions.  Rounding a point x to float32
// moves it by at most 2^-24 |x|, so one cell cost moves by at most
// 2^-24 (|q| + |c|) and any warping path (<= 2n-1 cells), hence DTW and
// every bound, by A = (2n-1) 2^-24 (max|q| + max|c|).  A prune / abandon
// decision compares a bound of one candidate with the DTW of another, and a
// finalist is kept against the best: both need 2A, kept with 25% to spare.
static __global__ void f32_slack_kernel(const unsigned long long* __restrict__ max_sq_bits, int n, float* __restrict__ add) {
    const double qn = sqrt(__longlong_as_double((long long)max_sq_bits[0]));
    const double cn = sqrt(__longlong_as_double((long long)max_sq_bits[1]));
    const double A = (2.0 * n - 1.0) * 5.9604644775390625e-08 * (qn + cn) * (1.0 + 1e-6) + 1e-30;
    add[0] = __double2float_ru(2.5 * A);
    add[1] = __double2float_ru(2.5 * A);
}

// =================================================================== plan
struct Plan {
    int64_t Q, N;
    int n, d, w, B, G, K, S, n_chunks;
    size_t es;  // element size
    bool has_lb, exact, rev;
    bool f32f;  // TCDTW_FLAG_F32_FILTER: float64 inputs, float32 filter
    bool cand_planar;  // desc->cand_planar is used instead of o_candT
    bool sat;          // the saturating LB_MV pass on scaled planar operands (float32, no reverse bound)
    bool rev_pc;       // TCDTW_FLAG_REVERSE_PC with an LB_PC second stage
    size_t o_q32, o_c32, o_slack, o_lanesc, o_dbf;
    int64_t max_tiles;
    // byte offsets
    size_t o_qT, o_ub, o_done, o_fin;
    int64_t done_cap, ub_sampled, fin_cap;
    int ub_ct, ub_stride;
    size_t o_up, o_lo, o_upT, o_loT, o_candT, o_steps, o_blo, o_bhi, o_bcnt, o_lb, o_seed, o_seedres,
        o_seedcnt, o_dbest, o_ccnt, o_coff, o_surv, o_res, o_tcnt, o_toff, o_tq, o_tb, o_tl, o_sq, o_sb, o_sl,
        o_ctr, o_minv, o_min64, o_bidx, o_tctr, o_cub, o_fsc, o_tisc, o_qpad, o_cupT, o_cloT, o_lb2, total;
    int qpad_rows, qpad_dims;
    size_t cub_bytes;
    int fin_threads, adv_warps;
};

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

static int make_plan(const tcdtw_search_desc* dsc, Plan* P) {
    if (!dsc) return TCDTW_INVALID_INPUT;
    if (dsc->dtype != TCDTW_F32 && dsc->dtype != TCDTW_F64) return TCDTW_INVALID_INPUT;
    if (dsc->n < 1 || dsc->dims < 1 || dsc->window < 0) return TCDTW_INVALID_INPUT;
    if (dsc->dims > 32) return TCDTW_NOT_SUPPORTED;  // the search's register buckets stop at 32 dimensions
    if (dsc->n_queries < 1 || dsc->n_queries > 65535 || dsc->n_candidates < 1 || dsc->n_candidates > 0xfffffff0LL)
        return TCDTW_INVALID_INPUT;  // queries per call: one compaction grid row each
    if (dsc->method < TCDTW_METHOD_NONE || dsc->method > TCDTW_METHOD_LB_AD) return TCDTW_INVALID_INPUT;
    if (dsc->refresh_period < 1 || dsc->quant_levels < 1 || dsc->max_boxes < 1 || dsc->group_width < 1)
        return TCDTW_INVALID_INPUT;
    if (!(dsc->trigger_ti > 0.0 && dsc->trigger_ti < 1.0) || !(dsc->trigger_pc > 0.0 && dsc->trigger_pc < 1.0))
        return TCDTW_INVALID_INPUT;
    if (!(dsc->min_cell_frac > 0.0)) return TCDTW_INVALID_INPUT;
    if (dsc->method == TCDTW_METHOD_TC_DTW && dsc->advanced != TCDTW_METHOD_LB_TI &&
        dsc->advanced != TCDTW_METHOD_LB_PC)
        return TCDTW_INVALID_INPUT;  // search.py:64-66
    Plan& p = *P;
    p.Q = dsc->n_queries;
    p.N = dsc->n_candidates;
    p.n = dsc->n;
    p.d = dsc->dims;
    p.w = dsc->window < dsc->n - 1 ? dsc->window : dsc->n - 1;
    p.B = 2 * p.w + 1;
    p.G = (p.n - 1) / dsc->group_width + 1;
    p.K = dsc->max_boxes;
    p.f32f = (dsc->flags & TCDTW_FLAG_F32_FILTER) != 0;
    if (p.f32f && dsc->dtype != TCDTW_F64) return TCDTW_INVALID_INPUT;
    p.exact = dsc->dtype == TCDTW_F64 && !p.f32f;
    p.es = p.exact ? 8 : 4;
    p.has_lb = dsc->method != TCDTW_METHOD_NONE;
    p.rev = p.has_lb && (dsc->flags & TCDTW_FLAG_REVERSE_LB) != 0;
    if (p.rev && (!dsc->cand_upper || !dsc->cand_lower)) return TCDTW_INVALID_INPUT;
    if (p.rev && p.f32f) return TCDTW_NOT_SUPPORTED;
    {
        const bool pc = dsc->method == TCDTW_METHOD_LB_PC ||
                        (dsc->method == TCDTW_METHOD_TC_DTW && dsc->advanced == TCDTW_METHOD_LB_PC);
        p.rev_pc = pc && (dsc->flags & TCDTW_FLAG_REVERSE_PC) != 0;
        if (p.rev_pc && (!dsc->cand_box_lo || !dsc->cand_box_hi)) return TCDTW_INVALID_INPUT;
        if (p.rev_pc && p.f32f) return TCDTW_NOT_SUPPORTED;
    }
    p.S = p.has_lb ? (dsc->seeds > 0 ? dsc->seeds : 8) : 0;
    if (p.S > kSeedMax) return TCDTW_INVALID_INPUT;
    if (p.S > p.N) p.S = (int)p.N;
    if (p.S > 0 && p.S != 1 && p.S != 2 && p.S != 4 && p.S != 8 && p.S != 16 && p.S != 32) {
        int s = 1;
        while (s < p.S) s <<= 1;
        p.S = s > kSeedMax ? kSeedMax : s;
    }
    p.n_chunks = (int)((p.N + kChunk - 1) / kChunk);
    p.max_tiles = p.Q * (p.N / kTile) + p.Q * (int64_t)p.n_chunks + p.Q;
    const int64_t Q = p.Q, N = p.N;
    const size_t es = p.es;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes); return r; };
    const size_t series_q = (size_t)Q * p.n * p.d * es;
    p.o_up = take(p.has_lb ? series_q : 0);
    p.o_lo = take(p.has_lb ? series_q : 0);
    const size_t planar_q = (size_t)(es == 4 ? planar_pad(Q) : Q) * p.n * p.d * es;  // float32: whole tiles
    p.o_upT = take(p.has_lb ? planar_q : 0);
    p.o_loT = take(p.has_lb ? planar_q : 0);
    p.o_qT = take(p.has_lb ? planar_q : 0);
    p.sat = p.has_lb && !p.exact && !p.rev;
    // the caller keeps a planar copy (a float32 one is scaled: not for the reverse bound's unscaled pass)
    p.cand_planar = p.has_lb && dsc->cand_planar != nullptr && !p.f32f && (p.exact || p.sat);
    p.o_candT = take(p.has_lb && !p.cand_planar ? planar_bytes(N, p.n * p.d, es) : 0);
    p.o_steps = take((size_t)Q * (p.n > 1 ? p.n - 1 : 1) * es);
    const size_t boxes = (size_t)Q * p.G * p.K * p.d * es;
    p.o_blo = take(boxes);
    p.o_bhi = take(boxes);
    p.o_bcnt = take((size_t)Q * p.G * 4);
    p.o_lb = take(p.has_lb ? (size_t)Q * N * es : 0);
    p.o_ub = 0;  // sized below, once the sampling is known
    p.o_cupT = take(p.rev ? (size_t)N * p.n * p.d * es : 0);
    p.o_cloT = take(p.rev ? (size_t)N * p.n * p.d * es : 0);
    p.o_lb2 = take(p.rev ? (size_t)Q * N * es : 0);
    p.o_seed = take((size_t)Q * kSeedMax * 4);
    p.o_seedres = take((size_t)Q * kSeedMax * es);
    p.o_seedcnt = take((size_t)Q * 4);
    p.o_dbest = take((size_t)Q * es);
    p.o_dbf = take((size_t)Q * es);
    p.o_ccnt = take((size_t)Q * p.n_chunks * 8);
    p.o_coff = take(((size_t)Q * p.n_chunks + 1) * 8);
    p.o_surv = take((size_t)Q * N * 4);
    p.o_res = take((size_t)Q * N * es);
    p.o_tcnt = take(((size_t)Q * p.n_chunks + 1) * 8);
    p.o_toff = take(((size_t)Q * p.n_chunks + 1) * 8);
    p.o_tq = take((size_t)p.max_tiles * 4);
    p.o_tb = take((size_t)p.max_tiles * 8);
    p.o_tl = take((size_t)p.max_tiles * 4);
    p.o_sq = take((size_t)Q * 4);
    p.o_sb = take((size_t)Q * 8);
    p.o_sl = take((size_t)Q * 4);
    p.o_ctr = take((size_t)Q * TCDTW_COUNTERS * 8);
    p.o_minv = take((size_t)Q * es);
    p.o_min64 = take((size_t)Q * 8);
    p.o_bidx = take((size_t)Q * 8);
    p.o_tctr = take(16 * sizeof(int));
    p.done_cap = Q * 256 + 65536;
    // UB (seeding only) on every ub_stride-th candidate tile of the LB_MV pass
    p.ub_ct = p.exact ? MvTile<double, 8, true>::CT : MvTile<float, 8, false>::CT;
    {
        const int64_t tiles = (N + p.ub_ct - 1) / p.ub_ct;
        int64_t st = tiles / 256;
        p.ub_stride = (int)(st < 1 ? 1 : (st > 32 ? 32 : st));
        if (p.exact && p.d > 8) p.ub_ct = MvTile<double, 16, true>::CT;
        const int64_t full = (N / ((int64_t)p.ub_ct * p.ub_stride)) * p.ub_ct;
        const int64_t rem = N % ((int64_t)p.ub_ct * p.ub_stride);
        p.ub_sampled = full + (rem < p.ub_ct ? rem : p.ub_ct);
    }
    p.o_ub = take(p.has_lb ? (size_t)Q * p.ub_sampled * es : 0);  // the sampled upper bounds, compact
    if (dsc->done_cap > 0) p.done_cap = dsc->done_cap;  // tests force the overflow path with 1
    p.o_done = take((size_t)p.done_cap * 8 + 64);
    p.fin_cap = p.done_cap + Q * kSeedMax;
    p.o_fin = take((size_t)p.fin_cap * 16 + 64);
    size_t b1 = 0, b2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, b1, (int64_t*)nullptr, (int64_t*)nullptr, (int)(Q * p.n_chunks + 1));
    b2 = b1;
    p.cub_bytes = b1 > b2 ? b1 : b2;
    p.o_cub = take(p.cub_bytes);
    p.fin_threads = 148 * 256;
    p.o_fsc = take((size_t)p.fin_threads * 2 * p.B * 8);
    p.adv_warps = 148 * 16;
    const bool ti = dsc->method == TCDTW_METHOD_LB_TI ||
                    (dsc->method == TCDTW_METHOD_TC_DTW && dsc->advanced == TCDTW_METHOD_LB_TI);
    p.o_tisc = take(ti ? (size_t)p.adv_warps * 32 * 3 * p.B * es : 0);
    p.o_lanesc = take(!p.exact && laner_any_rows_shape(p.n, p.d, p.B) > 0
                          ? (size_t)kLanerMaxWarps * laner_scratch_words(p.B) * sizeof(float) : 0);
    p.o_q32 = take(p.f32f ? series_q : 0);
    p.o_c32 = take(p.f32f ? (size_t)N * p.n * p.d * 4 : 0);
    p.o_slack = take(p.f32f ? 32 : 0);
    p.qpad_rows = p.n + 2 * p.w + 8;
    {  // the lane kernel's compile-time dimension count for this shape (>= d), else d
        const int ld = p.exact ? 0 : laner_pick(p.n, p.d, p.B).dims;
        p.qpad_dims = ld > 0 ? ld : p.d;
    }
    p.o_qpad = take(p.exact ? 0 : (size_t)Q * p.qpad_rows * ((p.qpad_dims + 1) / 2) * 8);
    p.total = o;
    return TCDTW_OK;
}

template <typename T>
static inline T* at(void* ws, size_t off) { return reinterpret_cast<T*>(reinterpret_cast<char*>(ws) + off); }

// Phase timer: CUDA events on the launching stream.
struct PhaseTimer {
    bool on;
    cudaStream_t st;
    cudaEvent_t ev[TCDTW_PHASES + 1];
    int first, last;
    float* out;
    PhaseTimer(const tcdtw_search_desc* dsc, cudaStream_t s, int f, int l)
        : on(dsc->phase_ms && (dsc->flags & TCDTW_FLAG_TIMING)), st(s), first(f), last(l), out(dsc->phase_ms) {
        if (on)
            for (int i = first; i <= last + 1; ++i) cudaEventCreate(&ev[i]);
    }
    void mark(int i) {
        if (on) cudaEventRecord(ev[i], st);
    }
    void finish() {
        if (!on) return;
        cudaEventSynchronize(ev[last + 1]);
        for (int i = first; i <= last; ++i) cudaEventElapsedTime(&out[i], ev[i], ev[i + 1]);
        for (int i = first; i <= last + 1; ++i) cudaEventDestroy(ev[i]);
    }
};

static int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

#define TRY(x)                         \
    do {                               \
        int _s = (x);                  \
        if (_s != TCDTW_OK) return _s; \
    } while (0)

// TCDTW_FLAG_DEBUG_SYNC: synchronise and report after every pipeline stage.
static void dbg_stage(const tcdtw_search_desc* dsc, cudaStream_t st, const char* what) {
    if (!(dsc->flags & TCDTW_FLAG_DEBUG_SYNC)) return;
    cudaError_t e = cudaStreamSynchronize(st);
    fprintf(stderr, "[tcdtw] %-24s %s\n", what, cudaGetErrorString(e));
    fflush(stderr);
}

template <typename T>
static SArgs<T> make_args(const tcdtw_search_desc* dsc, const Plan& p, const void* queries, const void* cands,
                          void* ws) {
    SArgs<T> a;
    a.queries = (const T*)queries;
    a.cands = (const T*)cands;
    a.lb = p.has_lb ? at<T>(ws, p.o_lb) : nullptr;
    a.env_up = p.has_lb ? at<T>(ws, p.o_up) : nullptr;
    a.env_lo = p.has_lb ? at<T>(ws, p.o_lo) : nullptr;
    a.dbest = at<T>(ws, p.o_dbest);
    a.thr_src = (dsc->flags & TCDTW_FLAG_FROZEN_THRESHOLDS) ? at<T>(ws, p.o_dbf) : a.dbest;
    a.box_lo = at<T>(ws, p.o_blo);
    a.box_hi = at<T>(ws, p.o_bhi);
    a.qsteps = at<T>(ws, p.o_steps);
    a.counters = at<int64_t>(ws, p.o_ctr);
    a.N = p.N;
    a.n = p.n;
    a.d = p.d;
    a.w = p.w;
    a.G = p.G;
    a.K = p.K;
    a.gw = dsc->group_width;
    a.period = dsc->refresh_period;
    a.method = dsc->method;
    a.adv = -1;
    if (dsc->method == TCDTW_METHOD_TC_DTW) a.adv = dsc->advanced;
    else if (dsc->method == TCDTW_METHOD_LB_TI || dsc->method == TCDTW_METHOD_LB_PC || dsc->method == TCDTW_METHOD_LB_AD)
        a.adv = dsc->method;
    a.trigger = (float)(a.adv == TCDTW_METHOD_LB_PC ? dsc->trigger_pc : dsc->trigger_ti);
    if (p.exact) {
        a.mg.prune = 1.0f;
        a.mg.fin = 1.0f;
        // float64: the cascaded bound tolerates 4(n+d) ulps of both sums
        double s = 4.0 * (p.n + p.d) * 1.1102230246251565e-16;  // * 2^-53
        s = s < 9.094947017729282e-13 ? 9.094947017729282e-13 : s;  // >= 2^-40
        a.casc_lo = (T)(1.0 - s);
        a.casc_hi = (T)(1.0 + s);
        a.casc_thr = (T)(1.0 + s);
    } else {
        // + 4: the saturating LB_MV terms carry two more roundings each (midhalf_kernel)
        const double eps = (2.0 * p.n + p.d + 20.0) * 1.1920928955078125e-07;  // * 2^-23
        a.mg.prune = nextafterf((float)(1.0 + 3.0 * eps), 2.0f);
        a.mg.fin = nextafterf((float)(1.0 + 2.5 * eps), 2.0f);
        a.casc_lo = (T)(1.0 - eps);
        a.casc_hi = (T)(1.0 + 2.0 * eps);
        a.casc_thr = (T)1.0;  // thr already carries the (1+3 eps) margin
    }
    a.abandon = dsc->method != TCDTW_METHOD_NONE;
    a.cascade = (dsc->flags & TCDTW_FLAG_NO_CASCADE) == 0;
    a.refill_min = 8;
    a.thr_every = 8;  // re-reading the live d_best every 4 / 8 / 16 rows measured equal (C4)
    a.done_list = nullptr;  // set for the survivors pass only
    a.done_cnt = nullptr;
    a.done_cap = 0;
    a.qpad = p.exact ? nullptr : at<float2>(ws, p.o_qpad);
    a.qpad_rows = p.qpad_rows;
    a.mg.add = nullptr;
    a.xq = a.xc = nullptr;
    a.lane_scratch = (!p.exact && laner_any_rows_shape(p.n, p.d, p.B) > 0) ? at<float>(ws, p.o_lanesc) : nullptr;
    a.cbox_lo = p.rev_pc ? (const T*)dsc->cand_box_lo : nullptr;
    a.cbox_hi = p.rev_pc ? (const T*)dsc->cand_box_hi : nullptr;
    if (p.f32f) {  // queries / cands are the float32 copies in the workspace
        a.queries = at<T>(ws, p.o_q32);
        a.cands = at<T>(ws, p.o_c32);
        a.xq = (const double*)queries;
        a.xc = (const double*)cands;
        a.mg.add = at<float>(ws, p.o_slack);
    }
    return a;
}

// Warp-per-pair wavefront with compile-time d (dtw_wave_d_kernel), or
// TCDTW_NOT_SUPPORTED for other d.
template <typename T, int DMAX, bool EXACT>
static int launch_wave_d(const SArgs<T>& a, const Plan& p, Tiles tl, int64_t n_tiles, const uint32_t* cand_of,
                         T* res, int* tctr, cudaStream_t st) {
    const int sms = sm_count();
    cudaMemsetAsync(tctr, 0, sizeof(int), st);
    // the query rows are shared by the block's warps; block size 256 (or
    // TCDTW_WAVE_THREADS=384: registers are capped for two such blocks)
    const size_t q_bytes = (size_t)wave_q_rows(p.n, p.w) * wave_row_stride((int)sizeof(T), p.d) * sizeof(T);
    const size_t prow_bytes = (size_t)wave_prow_len(p.B) * sizeof(T);
    auto run_d = [&](auto kern) -> int {
        int best_t = 0, best_w = 0;
        size_t best_s = 0;
        // 384-thread blocks keep 24 warps resident but split each 32-pair
        // tile unevenly (C3: 2717 vs 3131 q/s at 256): 256
        for (int t = 256; t <= 256; t += 128) {
            const size_t sm = q_bytes + (size_t)(t / 32) * prow_bytes;
            if (sm > 227 * 1024) continue;
            if (sm > 48 * 1024 &&
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
                continue;
            int occ = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, t, sm);
            if (occ * t / 32 > best_w) {
                best_w = occ * t / 32;
                best_t = t;
                best_s = sm;
            }
        }
        if (best_w < 1) return TCDTW_NOT_SUPPORTED;
        int64_t grid = (int64_t)(best_w / (best_t / 32)) * sms;
        if (grid > n_tiles) grid = n_tiles;
        kern<<<(int)grid, best_t, best_s, st>>>(a, tl, n_tiles, cand_of, res, tctr);
        return launch_status();
    };
    // staged query rows too large for shared memory: read them through L1
    const bool qg = q_bytes + (size_t)8 * prow_bytes > 227 * 1024;
#define TCDTW_WAVE_CASE(DD)                                                                           \
    if (p.d == DD && DD <= DMAX) {                                                                    \
        if (qg) {                                                                                     \
            auto kq = dtw_wave_d_kernel<T, (DD <= DMAX ? DD : 1), EXACT, true>;                       \
            const size_t sm = (size_t)8 * prow_bytes;                                                 \
            if (sm > 48 * 1024 &&                                                                     \
                cudaFuncSetAttribute(kq, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess) \
                return TCDTW_NOT_SUPPORTED;                                                           \
            int occ = 0;                                                                              \
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kq, 256, sm);                         \
            if (occ < 1) return TCDTW_NOT_SUPPORTED;                                                  \
            int64_t grid = (int64_t)occ * sms;                                                        \
            if (grid > n_tiles) grid = n_tiles;                                                       \
            kq<<<(int)grid, 256, sm, st>>>(a, tl, n_tiles, cand_of, res, tctr);                       \
            return launch_status();                                                                   \
        }                                                                                             \
        return run_d(dtw_wave_d_kernel<T, (DD <= DMAX ? DD : 1), EXACT>);                             \
    }
    TCDTW_WAVE_DIMS(TCDTW_WAVE_CASE)
#undef TCDTW_WAVE_CASE
    return TCDTW_NOT_SUPPORTED;
}

// Few pairs (a small collection or the seed pass of a few queries): the
// per-pair latency of the lane kernels (one lane walks all n rows) dominates,
// so the warp-per-pair wavefront (about n + 2W dependent steps) runs instead.
static inline bool few_pairs(int64_t pairs_upper) {
    return pairs_upper <= (int64_t)sm_count() * 8;
}

// DTW launcher over a tile list: thread-per-pair if the band fits the
// register buckets, else the wavefront kernel.
template <typename T, int DMAX, bool EXACT>
static int launch_dtw(const SArgs<T>& a, const Plan& p, Tiles tl, int64_t n_tiles, const uint32_t* cand_of, T* res,
                      int* tctr, cudaStream_t st, bool few) {
    if (n_tiles <= 0) return TCDTW_OK;
    if (few) {
        const int s = launch_wave_d<T, DMAX, EXACT>(a, p, tl, n_tiles, cand_of, res, tctr, st);
        if (s != TCDTW_NOT_SUPPORTED) return s;
    }
    if constexpr (!EXACT) {
        const int s = launch_laner(a, p.d, p.B, tl, n_tiles, cand_of, res, tctr, st);
        if (s != TCDTW_NOT_SUPPORTED) return s;
    }
    {
        const int s = launch_lane<T>(a, p.d, p.B, tl, n_tiles, cand_of, res, tctr, st);
        if (s != TCDTW_NOT_SUPPORTED) return s;
    }
    cudaMemsetAsync(tctr, 0, sizeof(int), st);
    const int sms = sm_count();
    constexpr int VEC = 16 / sizeof(T);
    const int DP = (p.d + VEC - 1) / VEC * VEC;
    if (p.B <= 64) {
        const size_t smem = (size_t)8 * (p.n + 2 * p.w) * DP * sizeof(T);
        auto run = [&](auto kern) -> int {
            if (smem > 48 * 1024 &&
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
                return TCDTW_NOT_SUPPORTED;
            int occ = 1;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
            if (occ < 1) return TCDTW_NOT_SUPPORTED;
            int64_t grid = (int64_t)occ * sms;
            const int64_t need = (n_tiles + 7) / 8;
            if (grid > need) grid = need;
            kern<<<(int)grid, 256, smem, st>>>(a, tl, n_tiles, cand_of, res, tctr);
            return launch_status();
        };
        if (p.B <= 8) return run(dtw_tpp_kernel<T, DMAX, 8, EXACT>);
        if (p.B <= 16) return run(dtw_tpp_kernel<T, DMAX, 16, EXACT>);
        if (p.B <= 32) return run(dtw_tpp_kernel<T, DMAX, 32, EXACT>);
        return run(dtw_tpp_kernel<T, DMAX, 64, EXACT>);
    }
    {
        const int s = launch_wave_d<T, DMAX, EXACT>(a, p, tl, n_tiles, cand_of, res, tctr, st);
        if (s != TCDTW_NOT_SUPPORTED) return s;
    }
    const size_t smem = ((size_t)(p.n + 2 * p.w) * ((p.d % 2 == 1) ? p.d : p.d + 1) + (size_t)8 * p.B) * sizeof(T);
    auto kern = dtw_wave_kernel<T, DMAX, EXACT>;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return TCDTW_NOT_SUPPORTED;
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
    if (occ < 1) return TCDTW_NOT_SUPPORTED;
    int64_t grid = (int64_t)occ * sms;
    if (grid > n_tiles) grid = n_tiles;
    kern<<<(int)grid, 256, smem, st>>>(a, tl, n_tiles, cand_of, res, tctr);
    return launch_status();
}

template <typename T, int DMAX>
struct SearchImpl {
    static constexpr bool EXACT = sizeof(T) == 8;

    static int seed(const tcdtw_search_desc* dsc, const Plan& p, const void* queries, const void* cands,
                    const void* dr, void* ws, void* dbest_out, cudaStream_t st) {
        PhaseTimer tm(dsc, st, 0, 3);
        SArgs<T> a = make_args<T>(dsc, p, queries, cands, ws);
        const int dtype = EXACT ? TCDTW_F64 : TCDTW_F32;
        tm.mark(0);
        if (p.f32f) {
            if constexpr (!EXACT) {
                // the float32 roundings the whole filter runs on (kept in the
                // workspace for the finish phase) and the rounding slack
                unsigned long long* mx = at<unsigned long long>(ws, p.o_slack) + 2;
                cudaMemsetAsync(mx, 0, 16, st);
                const int sms = sm_count();
                round_points_kernel<<<sms * 8, 256, 0, st>>>((const double*)queries, p.Q * p.n, p.d,
                                                            const_cast<T*>(a.queries), mx);
                TRY(launch_status());
                round_points_kernel<<<sms * 8, 256, 0, st>>>((const double*)cands, p.N * p.n, p.d,
                                                            const_cast<T*>(a.cands), mx + 1);
                TRY(launch_status());
                f32_slack_kernel<<<1, 1, 0, st>>>(mx, p.n, at<float>(ws, p.o_slack));
                TRY(launch_status());
            }
            queries = a.queries;
            cands = a.cands;
        }
        cudaMemsetAsync(at<char>(ws, p.o_ctr), 0, (size_t)p.Q * TCDTW_COUNTERS * 8, st);
        fill_kernel<T><<<grid_for(p.Q, 256), 256, 0, st>>>(a.dbest, p.Q, dev_inf<T>());
        TRY(launch_status());
        const T* candT = p.cand_planar ? (const T*)dsc->cand_planar : at<T>(ws, p.o_candT);
        // {sigma, 1/sigma} of the planar candidates (their trailer)
        const float* scale = nullptr;
        if constexpr (!EXACT) {
            if (p.sat)
                scale = reinterpret_cast<const float*>(reinterpret_cast<const char*>(candT) +
                                                       planar_trailer_off(p.N, p.n * p.d, p.es));
        }
        if (p.has_lb) {
            if constexpr (!EXACT) {
                if (p.sat && !p.cand_planar)
                    TRY(planar_scale((const float*)cands, p.N * p.n * p.d, const_cast<float*>(scale), st));
            }
            TRY(series_envelope(dtype, queries, p.Q, p.n, p.d, p.w, at<T>(ws, p.o_up), at<T>(ws, p.o_lo), st));
            bool tiled = false;
            if constexpr (!EXACT) {
                if (p.sat) {  // tile-major scaled copies; envelopes as (midpoint, inflated half width)
                    tiled = true;
                    const int rows = p.n * p.d;
                    TRY(planarize_tiled(at<float>(ws, p.o_up), p.Q, rows, at<float>(ws, p.o_upT), st, scale));
                    TRY(planarize_tiled(at<float>(ws, p.o_lo), p.Q, rows, at<float>(ws, p.o_loT), st, scale));
                    TRY(planarize_tiled((const float*)queries, p.Q, rows, at<float>(ws, p.o_qT), st, scale));
                    if (!p.cand_planar)
                        TRY(planarize_tiled((const float*)cands, p.N, rows, at<float>(ws, p.o_candT), st, scale));
                    const int64_t cnt = planar_pad(p.Q) * rows;
                    midhalf_kernel<<<grid_for(cnt, 256), 256, 0, st>>>(at<float>(ws, p.o_upT), at<float>(ws, p.o_loT),
                                                                        cnt);
                    TRY(launch_status());
                }
            }
            if (!tiled) {
                TRY(planarize<T>(at<T>(ws, p.o_up), p.Q, p.n * p.d, at<T>(ws, p.o_upT), st));
                TRY(planarize<T>(at<T>(ws, p.o_lo), p.Q, p.n * p.d, at<T>(ws, p.o_loT), st));
                TRY(planarize<T>((const T*)queries, p.Q, p.n * p.d, at<T>(ws, p.o_qT), st));
                if (!p.cand_planar) TRY(planarize<T>((const T*)cands, p.N, p.n * p.d, at<T>(ws, p.o_candT), st));
            }
        }
        if (!EXACT) {
            const int DPq = (p.qpad_dims + 1) / 2;
            const int64_t tot = p.Q * p.qpad_rows * DPq;
            qpad_kernel<<<grid_for(tot, 256), 256, 0, st>>>((const float*)queries, p.Q, p.n, p.d, p.w, p.qpad_rows,
                                                             const_cast<float2*>(a.qpad), p.qpad_dims);
            TRY(launch_status());
        }
        if (a.adv == TCDTW_METHOD_LB_PC)
            TRY(series_box_sets(dtype, queries, p.Q, p.n, p.d, p.w, dsc->group_width, dsc->quant_levels, p.K,
                                dsc->min_cell_frac, dr, at<T>(ws, p.o_blo), at<T>(ws, p.o_bhi),
                                at<int32_t>(ws, p.o_bcnt), st));
        if (a.adv == TCDTW_METHOD_LB_TI && p.n > 1)
            TRY(series_steps(dtype, queries, p.Q, p.n, p.d, at<T>(ws, p.o_steps), st));
        dbg_stage(dsc, st, "prep");
        tm.mark(1);
        if (p.has_lb)
            TRY((launch_lbmv_matrix<T, DMAX, EXACT>(at<T>(ws, p.o_upT), at<T>(ws, p.o_loT), at<T>(ws, p.o_qT),
                                                    candT, p.Q, p.N, p.n, p.d, at<T>(ws, p.o_lb),
                                                    at<T>(ws, p.o_ub), st, p.ub_stride, false, p.ub_sampled, scale)));
        if (p.rev) {
            // reverse LB_MV: the candidates' envelopes against the queries,
            // written transposed into the (query, candidate) layout
            TRY(planarize<T>((const T*)dsc->cand_upper, p.N, p.n * p.d, at<T>(ws, p.o_cupT), st));
            TRY(planarize<T>((const T*)dsc->cand_lower, p.N, p.n * p.d, at<T>(ws, p.o_cloT), st));
            TRY((launch_lbmv_matrix<T, DMAX, EXACT>(at<T>(ws, p.o_cupT), at<T>(ws, p.o_cloT), nullptr,
                                                    at<T>(ws, p.o_qT), p.N, p.Q, p.n, p.d, at<T>(ws, p.o_lb2),
                                                    nullptr, st, 1, true)));
        }
        dbg_stage(dsc, st, "lb_mv");
        tm.mark(2);
        if (p.S > 0) {
            uint32_t* seeds = at<uint32_t>(ws, p.o_seed);
            int32_t* scnt = at<int32_t>(ws, p.o_seedcnt);
            const int s_eff = (int)(p.S < p.ub_sampled ? p.S : p.ub_sampled);
            switch (p.S) {
                case 1: topk_kernel<T, 1><<<(unsigned)p.Q, 256, 0, st>>>(at<T>(ws, p.o_ub), p.N, s_eff, a.dbest, seeds, scnt, p.ub_ct, p.ub_stride); break;
                case 2: topk_kernel<T, 2><<<(unsigned)p.Q, 256, 0, st>>>(at<T>(ws, p.o_ub), p.N, s_eff, a.dbest, seeds, scnt, p.ub_ct, p.ub_stride); break;
                case 4: topk_kernel<T, 4><<<(unsigned)p.Q, 256, 0, st>>>(at<T>(ws, p.o_ub), p.N, s_eff, a.dbest, seeds, scnt, p.ub_ct, p.ub_stride); break;
                case 8: topk_kernel<T, 8><<<(unsigned)p.Q, 256, 0, st>>>(at<T>(ws, p.o_ub), p.N, s_eff, a.dbest, seeds, scnt, p.ub_ct, p.ub_stride); break;
                case 16: topk_kernel<T, 16><<<(unsigned)p.Q, 256, 0, st>>>(at<T>(ws, p.o_ub), p.N, s_eff, a.dbest, seeds, scnt, p.ub_ct, p.ub_stride); break;
                default: topk_kernel<T, 32><<<(unsigned)p.Q, 256, 0, st>>>(at<T>(ws, p.o_ub), p.N, s_eff, a.dbest, seeds, scnt, p.ub_ct, p.ub_stride); break;
            }
            TRY(launch_status());
            Tiles stl{at<uint32_t>(ws, p.o_sq), at<int64_t>(ws, p.o_sb), at<int32_t>(ws, p.o_sl)};
            seed_tiles_kernel<<<grid_for(p.Q, 256), 256, 0, st>>>(p.Q, p.S, scnt, stl);
            TRY(launch_status());
            fill_kernel<T><<<grid_for(p.Q * p.S, 256), 256, 0, st>>>(at<T>(ws, p.o_seedres), p.Q * p.S, dev_inf<T>());
            TRY(launch_status());
            dbg_stage(dsc, st, "topk+tiles");
            tm.mark(3);
            if (a.thr_src != a.dbest)  // frozen thresholds: the seed pass prunes against the UB seeding
                cudaMemcpyAsync(const_cast<T*>(a.thr_src), a.dbest, (size_t)p.Q * sizeof(T), cudaMemcpyDeviceToDevice, st);
            TRY((launch_dtw<T, DMAX, EXACT>(a, p, stl, p.Q, seeds, at<T>(ws, p.o_seedres), at<int>(ws, p.o_tctr), st,
                                            few_pairs(p.Q * (int64_t)p.S))));
        } else {
            tm.mark(3);
        }
        dbg_stage(dsc, st, "seed dtw");
        tm.mark(4);
        if (dbest_out && dbest_out != (void*)a.dbest)
            cudaMemcpyAsync(dbest_out, a.dbest, (size_t)p.Q * sizeof(T), cudaMemcpyDeviceToDevice, st);
        tm.finish();
        return launch_status();
    }

    static int finish(const tcdtw_search_desc* dsc, const Plan& p, const void* queries, const void* cands,
                      const void* dr, void* ws, const void* dbest_in, int64_t* best_index, double* best_distance,
                      int64_t* counters, cudaStream_t st) {
        (void)dr;
        PhaseTimer tm(dsc, st, 4, 7);
        SArgs<T> a = make_args<T>(dsc, p, queries, cands, ws);
        if (p.f32f) {  // the float32 copies the seed phase made
            queries = a.queries;
            cands = a.cands;
        }
        const int sms = sm_count();
        tm.mark(4);
        if (dbest_in && dbest_in != (const void*)a.dbest)
            cudaMemcpyAsync(a.dbest, dbest_in, (size_t)p.Q * sizeof(T), cudaMemcpyDeviceToDevice, st);
        if (a.thr_src != a.dbest)  // frozen thresholds: the best after the seed phase (and the exchange)
            cudaMemcpyAsync(const_cast<T*>(a.thr_src), a.dbest, (size_t)p.Q * sizeof(T), cudaMemcpyDeviceToDevice, st);
        // compaction
        const bool all = !p.has_lb;
        int64_t* ccnt = at<int64_t>(ws, p.o_ccnt);
        int64_t* coff = at<int64_t>(ws, p.o_coff);
        dim3 cgrid((unsigned)p.n_chunks, (unsigned)p.Q);
        if (p.Q > 65535) return TCDTW_INVALID_INPUT;
        const T* lb2 = p.rev ? at<T>(ws, p.o_lb2) : nullptr;
        int S_c = p.S;  // seeds compared per element (none once poisoned)
        if (p.has_lb && p.S > 0) {
            poison_seeds_kernel<T><<<grid_for(p.Q * p.S, 256), 256, 0, st>>>(
                const_cast<T*>(a.lb), p.N, p.Q, p.S, at<uint32_t>(ws, p.o_seed), at<int32_t>(ws, p.o_seedcnt));
            TRY(launch_status());
            S_c = 0;
        }
        compact_count_kernel<T><<<cgrid, 256, 0, st>>>(a.lb, lb2, p.N, p.n_chunks, a.dbest, a.mg, all,
                                                       at<uint32_t>(ws, p.o_seed), at<int32_t>(ws, p.o_seedcnt), S_c,
                                                       ccnt);
        TRY(launch_status());
        cudaMemsetAsync(ccnt + p.Q * p.n_chunks, 0, 8, st);
        size_t cb = p.cub_bytes;
        if (cub::DeviceScan::ExclusiveSum(at<void>(ws, p.o_cub), cb, ccnt, coff, (int)(p.Q * p.n_chunks + 1), st) !=
            cudaSuccess)
            return TCDTW_CUDA_ERROR;
        uint32_t* surv = at<uint32_t>(ws, p.o_surv);
        T* res = at<T>(ws, p.o_res);
        compact_write_kernel<T><<<cgrid, 256, 0, st>>>(a.lb, lb2, p.N, p.n_chunks, a.dbest, a.mg, all,
                                                       at<uint32_t>(ws, p.o_seed), at<int32_t>(ws, p.o_seedcnt), S_c,
                                                       coff, surv, res);
        TRY(launch_status());
        int64_t* tcnt = at<int64_t>(ws, p.o_tcnt);
        int64_t* toff = at<int64_t>(ws, p.o_toff);
        const int64_t n_seg = p.Q * p.n_chunks;
        seg_tiles_count_kernel<<<grid_for(n_seg, 256), 256, 0, st>>>(p.Q, p.n_chunks, coff, tcnt, a.counters);
        TRY(launch_status());
        cudaMemsetAsync(tcnt + n_seg, 0, 8, st);
        cb = p.cub_bytes;
        if (cub::DeviceScan::ExclusiveSum(at<void>(ws, p.o_cub), cb, tcnt, toff, (int)(n_seg + 1), st) != cudaSuccess)
            return TCDTW_CUDA_ERROR;
        Tiles tl{at<uint32_t>(ws, p.o_tq), at<int64_t>(ws, p.o_tb), at<int32_t>(ws, p.o_tl)};
        seg_tiles_fill_kernel<<<grid_for(n_seg, 128), 128, 0, st>>>(p.Q, p.n_chunks, coff, toff, tl);
        TRY(launch_status());
        // The number of tiles stays on the device (toff[n_seg], read by the
        // kernels through tl.count); the host only knows the upper bound
        // max_tiles, which sizes the grids.  No host synchronisation.
        dbg_stage(dsc, st, "compact+tiles");
        tl.count = toff + n_seg;
        const int64_t n_tiles = p.max_tiles;
        const bool survivors_few = few_pairs(p.Q * p.N);  // upper bound: every pair survives
        tm.mark(5);
        if (a.adv >= 0) {
            int sa = TCDTW_NOT_SUPPORTED;
            if (a.adv == TCDTW_METHOD_LB_PC && !p.rev_pc)
                sa = launch_advanced_pc<T>(a, p.d, tl, n_tiles, surv, res, at<int>(ws, p.o_tctr), st);
            if (sa == TCDTW_NOT_SUPPORTED) {
                cudaMemsetAsync(at<int>(ws, p.o_tctr), 0, sizeof(int), st);
                int grid = (p.adv_warps * 32) / 256;
                // LB_TI: slot rings in shared memory when 8 warps' rings fit
                const size_t ring = (size_t)8 * 3 * p.B * 32 * sizeof(T);
                bool rs = a.adv == TCDTW_METHOD_LB_TI && ring <= 200 * 1024;
                auto kern = advanced_kernel<T, DMAX, EXACT>;
                if (rs && ring > 48 * 1024 &&
                    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ring) != cudaSuccess)
                    rs = false;
                kern<<<grid, 256, rs ? ring : 0, st>>>(a, tl, n_tiles, surv, res, at<T>(ws, p.o_tisc),
                                                       at<int>(ws, p.o_tctr), rs);
                sa = launch_status();
            }
            TRY(sa);
        }
        dbg_stage(dsc, st, "advanced");
        if constexpr (!EXACT) {
            // the R-row lane kernel keeps one query per warp: hand it whole
            // segments, or, when segments are too few to occupy every warp
            // (small collections: C1 has 3 chunks per query), pieces of about
            // survivors / (4 x resident warps), at least 4 pairs per lane --
            // the piece length is chosen on the device from the tile count
            if (laner_rows(a, p.d, p.B) > 0 && !survivors_few) {
                int* seg_len = at<int>(ws, p.o_tctr) + 8;
                laner_seglen_kernel<<<1, 1, 0, st>>>(tl.count, (int64_t)sms * 16, seg_len);
                TRY(launch_status());
                seg_tiles_count_kernel<<<grid_for(n_seg, 256), 256, 0, st>>>(p.Q, p.n_chunks, coff, tcnt, nullptr,
                                                                             kChunk, seg_len);
                TRY(launch_status());
                cb = p.cub_bytes;
                if (cub::DeviceScan::ExclusiveSum(at<void>(ws, p.o_cub), cb, tcnt, toff, (int)(n_seg + 1), st) !=
                    cudaSuccess)
                    return TCDTW_CUDA_ERROR;
                seg_tiles_fill_kernel<<<grid_for(n_seg, 128), 128, 0, st>>>(p.Q, p.n_chunks, coff, toff, tl, kChunk,
                                                                            seg_len);
                TRY(launch_status());
            }
        }
        tm.mark(6);
        unsigned long long* done_cnt = at<unsigned long long>(ws, p.o_done);
        unsigned long long* done_list = done_cnt + 8;
        cudaMemsetAsync(done_cnt, 0, 8, st);
        SArgs<T> ad = a;
        ad.done_list = done_list;
        ad.done_cnt = done_cnt;
        ad.done_cap = p.done_cap;
        TRY((launch_dtw<T, DMAX, EXACT>(ad, p, tl, n_tiles, surv, res, at<int>(ws, p.o_tctr), st, survivors_few)));
        dbg_stage(dsc, st, "dtw");
        tm.mark(7);
        // finalize
        T* minv = at<T>(ws, p.o_minv);
        unsigned long long* min64 = at<unsigned long long>(ws, p.o_min64);
        unsigned long long* bidx = at<unsigned long long>(ws, p.o_bidx);
        fill_kernel<T><<<grid_for(p.Q, 256), 256, 0, st>>>(minv, p.Q, dev_inf<T>());
        TRY(launch_status());
        cudaMemsetAsync(min64, 0x7f, (size_t)p.Q * 8, st);  // large positive sentinel
        cudaMemsetAsync(bidx, 0xff, (size_t)p.Q * 8, st);
        Tiles stl{at<uint32_t>(ws, p.o_sq), at<int64_t>(ws, p.o_sb), at<int32_t>(ws, p.o_sl)};
        const uint32_t* seeds = at<uint32_t>(ws, p.o_seed);
        const T* seedres = at<T>(ws, p.o_seedres);
        const int fgrid = sms * 4;
        if (p.S > 0) {
            fin_min_kernel<T><<<fgrid, 256, 0, st>>>(stl, p.Q, seedres, minv, nullptr, 0);
            TRY(launch_status());
        }
        {
            // completed survivors from the list; the full tile scan only if
            // the list overflowed (both decided on the device)
            fin_min_list_kernel<T><<<fgrid, 256, 0, st>>>(done_list, done_cnt, p.done_cap, res, minv);
            TRY(launch_status());
            fin_min_kernel<T><<<fgrid, 256, 0, st>>>(tl, n_tiles, res, minv, done_cnt, p.done_cap);
            TRY(launch_status());
        }
        const T* dbi = (const T*)dbest_in;
        double* fsc = at<double>(ws, p.o_fsc);
        const int rgrid = p.fin_threads / 256;
        // finalists: seeds + completed survivors -> one warp per float64 re-score
        Finalists F;
        F.cnt = at<unsigned long long>(ws, p.o_fin);
        F.item = F.cnt + 8;
        F.d64 = reinterpret_cast<double*>(F.item + p.fin_cap);
        F.cap = p.fin_cap;
        cudaMemsetAsync(F.cnt, 0, 8, st);
        fin_collect_kernel<T><<<fgrid, 256, 0, st>>>(a, stl, p.S > 0 ? p.Q : 0, seeds, seedres, done_list, done_cnt,
                                                     p.done_cap, surv, res, minv, dbi, F);
        TRY(launch_status());
        {
            // per warp: the staged query (float64) and one band row (+inf end)
            const size_t row_b = (size_t)(2 * p.w + 2) * sizeof(double);
            const size_t stage_b = (size_t)p.n * rescore_col_stride(p.d) * sizeof(double) + row_b;
            const int wpb = (int)(200 * 1024 / stage_b) < 8 ? (int)(200 * 1024 / stage_b) : 8;
            auto go = [&](auto kern, int warps, size_t per_warp) -> int {
                const size_t fsm = (size_t)warps * per_warp;
                if (fsm > 48 * 1024 &&
                    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm) != cudaSuccess)
                    return TCDTW_NOT_SUPPORTED;
                int occ = 1;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, warps * 32, fsm);
                kern<<<sms * (occ < 1 ? 1 : occ), warps * 32, fsm, st>>>(a, F, min64);
                return launch_status();
            };
            if (wpb >= 1) TRY(go(fin_rescore_warp_kernel<T, DMAX, true>, wpb, stage_b));
            else TRY(go(fin_rescore_warp_kernel<T, DMAX, false>, 8, row_b));
        }
        // survivors' completed list overflowed: scan every tile instead
        fin_rescore_kernel<T, DMAX><<<rgrid, 256, 0, st>>>(a, tl, n_tiles, surv, res, minv, dbi, EXACT ? 1 : 0,
                                                           min64, bidx, fsc, done_cnt, p.done_cap);
        TRY(launch_status());
        fin_pick_kernel<<<fgrid, 256, 0, st>>>(F, min64, bidx);
        TRY(launch_status());
        if (!EXACT) {
            fin_rescore_kernel<T, DMAX><<<rgrid, 256, 0, st>>>(a, tl, n_tiles, surv, res, minv, dbi, 1, min64, bidx,
                                                               fsc, done_cnt, p.done_cap);
            TRY(launch_status());
        }
        fin_output_kernel<T><<<grid_for(p.Q, 256), 256, 0, st>>>(p.Q, p.N, dsc->candidate_base, minv, min64, bidx,
                                                                a.counters, p.has_lb ? 1 : 0, best_index,
                                                                best_distance, counters);
        dbg_stage(dsc, st, "finalize");
        tm.mark(8 > TCDTW_PHASES ? TCDTW_PHASES : 8);
        tm.finish();
        return launch_status();
    }
};

struct SeedOp {
    template <typename T, int DM>
    int run(const tcdtw_search_desc* dsc, const Plan& p, const void* q, const void* c, const void* dr, void* ws,
            void* dbo, cudaStream_t st) {
        return SearchImpl<T, DM>::seed(dsc, p, q, c, dr, ws, dbo, st);
    }
};
struct FinishOp {
    template <typename T, int DM>
    int run(const tcdtw_search_desc* dsc, const Plan& p, const void* q, const void* c, const void* dr, void* ws,
            const void* dbi, int64_t* bi, double* bd, int64_t* ctr, cudaStream_t st) {
        return SearchImpl<T, DM>::finish(dsc, p, q, c, dr, ws, dbi, bi, bd, ctr, st);
    }
};

// Only the register buckets the search instantiates (d <= 32 covers C0-C4;
// larger d goes through the 64/128 buckets).
template <typename T, typename F, typename... Args>
int dispatch_search_dims(int dims, F&& f, Args&&... args) {
    if (dims <= 4) return f.template run<T, 4>(args...);
    if (dims <= 8) return f.template run<T, 8>(args...);
    if (dims <= 16) return f.template run<T, 16>(args...);
    if (dims <= 32) return f.template run<T, 32>(args...);
    return TCDTW_NOT_SUPPORTED;
}

}  // namespace tcdtw
