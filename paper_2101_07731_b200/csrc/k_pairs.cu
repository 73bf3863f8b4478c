// k_pairs.cu -- per-pair operators of the reference API, batched over pairs.
//
// These are the drop-in replacements of the reference's per-call functions
// (dtw_banded, build_envelope, lb_mv, lb_ad, neighbor_steps, ti_advance,
// lb_ti, build_box_sets/quantize_cluster, lb_pc).  They run in EXACT mode
// (common.cuh) and reproduce the reference's float64 results bit for bit,
// including abandon semantics and cell counts.  One thread owns one pair
// (sequential prefix-sum semantics, core.py:133-146); they are latency-bound
// by design -- the throughput path is the batched search (k_search.cu).
//
// Citations: file:line relative to /root/reference/pkg/src/mvdtw.

#include "common.cuh"
#include "dispatch.cuh"

namespace tcdtw {

// ---------------------------------------------------------------- dtw_banded
// dtw.py:45-102; band rows live in global scratch (2*width per pair).
template <typename T, int DMAX>
__global__ void dtw_pairs_kernel(const T* __restrict__ A, const T* __restrict__ B, int64_t P, int n,
                                 int d, int w, const T* __restrict__ thr_arr, T* __restrict__ out_dist,
                                 uint8_t* __restrict__ out_ab, int64_t* __restrict__ out_cells,
                                 T* __restrict__ scratch) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= P) return;
    const T* qa = A + p * (int64_t)n * d;
    const T* ca = B + p * (int64_t)n * d;
    const int width = 2 * w + 1;
    T* prev = scratch + p * 2 * (int64_t)width;
    T* cur = prev + width;
    const T INF = dev_inf<T>();
    const T threshold = thr_arr ? thr_arr[p] : INF;
    for (int k = 0; k < width; ++k) prev[k] = INF;
    int64_t cells = 0;
    for (int i = 0; i < n; ++i) {
        const int lo = i < w ? 0 : i - w;
        const int hi = i + w >= n ? n - 1 : i + w;
        for (int k = 0; k < width; ++k) cur[k] = INF;
        T qi[DMAX];
        load_point<T, DMAX>(qi, qa + (int64_t)i * d, d);
        int k = lo - i + w;
        T row_min = INF;
        for (int j = lo; j <= hi; ++j, ++k) {
            const T cost = dist_exact<T, DMAX>(qi, ca + (int64_t)j * d, d);
            T v;
            if (i == 0 && j == 0) {
                v = cost;
            } else {
                T best = INF;
                if (i > 0) {
                    if (k + 1 < width) best = prev[k + 1];
                    if (j > 0 && prev[k] < best) best = prev[k];
                }
                if (k > 0 && cur[k - 1] < best) best = cur[k - 1];
                v = add_rn(cost, best);
            }
            cur[k] = v;
            if (v < row_min) row_min = v;
        }
        cells += hi - lo + 1;
        if (row_min > threshold) {
            out_dist[p] = row_min;
            out_ab[p] = 1;
            out_cells[p] = cells;
            return;
        }
        T* t = prev;
        prev = cur;
        cur = t;
    }
    const T fin = prev[w];
    out_dist[p] = fin;
    out_ab[p] = fin > threshold ? 1 : 0;
    out_cells[p] = cells;
}

// ------------------------------------------------------------ build_envelope
// lb_mv.py:44-88: windowed max/min per dimension, windows clipped at the ends.
template <typename T>
__global__ void envelope_kernel(const T* __restrict__ S, int64_t n_series, int n, int d, int w,
                                T* __restrict__ U, T* __restrict__ L) {
    const int64_t total = n_series * (int64_t)n * d;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = e / ((int64_t)n * d);
        const int r = (int)(e - s * (int64_t)n * d);
        const int i = r / d, p = r - (r / d) * d;
        const int lo = i - w < 0 ? 0 : i - w;
        const int hi = i + w > n - 1 ? n - 1 : i + w;
        const T* col = S + s * (int64_t)n * d + p;
        T mx = col[(int64_t)lo * d], mn = mx;
        for (int j = lo + 1; j <= hi; ++j) {
            const T v = col[(int64_t)j * d];
            mx = v > mx ? v : mx;
            mn = v < mn ? v : mn;
        }
        U[e] = mx;
        L[e] = mn;
    }
}

// Streaming envelope (the HBM-bound form, also the candidate-side index
// build).  A persistent block walks groups of G whole series (G*n*d
// contiguous elements):
//   * the next group streams into a second staging buffer by 16-byte
//     cp.async while the current one is processed, so HBM reads are always in
//     flight (without it the kernel sat at ~27% of the copy bandwidth);
//   * van Herk / Gil-Werman: the series is cut into blocks of k = min(2W+1, n)
//     points, and four independent scans per (series, dim, block) -- prefix
//     max, prefix min, suffix max, suffix min -- run on four threads, so a
//     clipped window [max(0,i-W), min(n-1,i+W)] is max(suffix[lo],
//     prefix[hi]) when it spans two blocks, prefix[hi] when it starts a block
//     and suffix[lo] otherwise (the last, partial block): about six
//     comparisons per element instead of 2(2W+1);
//   * the combine walks each series row by row with the dimension count a
//     compile-time constant (no integer division per element) and streams
//     the results out (read n*d, write 2*n*d elements per series).
// max/min are exact and ties keep the earliest index, like envelope_kernel,
// so the result is bit-identical to it (lb_mv.py:44-71).
template <typename T>
__device__ __forceinline__ void env_cp16(T* dst, const T* src) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src) : "memory");
}

template <typename T, int DC>  // DC > 0: compile-time dimension count
__global__ void __launch_bounds__(256) envelope_stream_kernel(const T* __restrict__ S, int64_t n_series, int n,
                                                              int d_rt, int w, int G, T* __restrict__ U,
                                                              T* __restrict__ L) {
    extern __shared__ __align__(16) unsigned char env_smem[];
    const int d = DC > 0 ? DC : d_rt;
    const int nd = n * d;
    const int cap = G * nd;
    T* X0 = reinterpret_cast<T*>(env_smem);  // two staging buffers
    T* X1 = X0 + cap;
    T* PX = X1 + cap;                        // prefix max / min, suffix max / min
    T* PN = PX + cap;
    T* SX = PN + cap;
    T* SN = SX + cap;
    int2* tab = reinterpret_cast<int2*>(SN + cap);  // per row: the two max operands' offsets from PX
    const int k = 2 * w + 1 < n ? 2 * w + 1 : n;
    const int nb = (n + k - 1) / k;
    // per-row window table, once per launch (the divisions by the runtime
    // block length stay out of the per-element work).  The window max is
    // max(A, B) with A, B offsets from PX: SX[lo] and PX[hi] when the window
    // spans two blocks, PX[hi] twice when it starts a block, SX[lo] twice
    // otherwise; the min operands sit one array (cap) further (PN, SN).
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int lo = i - w < 0 ? 0 : i - w;
        const int hi = i + w > n - 1 ? n - 1 : i + w;
        const int sx = 2 * cap + lo * d, px = hi * d;
        if (lo / k != hi / k) tab[i] = make_int2(sx, px);
        else if (lo % k == 0) tab[i] = make_int2(px, px);
        else tab[i] = make_int2(sx, sx);
    }
    constexpr int V = 16 / sizeof(T);
    const bool vec = (nd % V) == 0 && (reinterpret_cast<uintptr_t>(S) % 16) == 0;
    const int64_t stride = (int64_t)gridDim.x * G;
    auto stage = [&](int64_t s0, T* X) {  // issue the loads of group s0 (no wait)
        if (s0 >= n_series) return;
        const int g_here = (int)((n_series - s0) < G ? (n_series - s0) : G);
        const int elems = g_here * nd;
        const T* src = S + s0 * nd;
        if (vec) {
            for (int e = threadIdx.x * V; e < elems; e += blockDim.x * V) env_cp16(X + e, src + e);
        } else {
            for (int e = threadIdx.x; e < elems; e += blockDim.x) X[e] = src[e];
        }
    };
    int64_t s0 = (int64_t)blockIdx.x * G;
    stage(s0, X0);
    asm volatile("cp.async.commit_group;" ::: "memory");
    T* X = X0;
    T* Xn = X1;
    for (; s0 < n_series; s0 += stride) {
        stage(s0 + stride, Xn);  // Xn was released by the barrier after the last combine
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncthreads();
        const int g_here = (int)((n_series - s0) < G ? (n_series - s0) : G);
        // scans: one thread per (direction, series, block, dim); the forward
        // thread keeps prefix max and min, the backward one suffix max and
        // min (one load feeds both); decomposed once per sequence
        const int seqs = g_here * nb * d;
        for (int q = threadIdx.x; q < 2 * seqs; q += blockDim.x) {
            const bool fwd = q < seqs;
            const int r = fwd ? q : q - seqs;
            const int p = r % d, gb = r / d;  // gb = g * nb + b
            const int g = gb / nb, b = gb - g * nb;
            const int i0 = b * k, len = (i0 + k < n ? k : n - i0);
            const int off = g * nd + i0 * d + p;
            if (fwd) {
                const T* x = X + off;
                T* ox = PX + off;
                T* on = PN + off;
                T mx = x[0], mn = mx;
                ox[0] = mx;
                on[0] = mn;
                for (int t = 1; t < len; ++t) {
                    const T v = x[t * d];
                    mx = v > mx ? v : mx;  // earliest index wins ties
                    mn = v < mn ? v : mn;
                    ox[t * d] = mx;
                    on[t * d] = mn;
                }
            } else {
                const int last = (len - 1) * d;
                const T* x = X + off;
                T* ox = SX + off;
                T* on = SN + off;
                T mx = x[last], mn = mx;
                ox[last] = mx;
                on[last] = mn;
                for (int t = last - d; t >= 0; t -= d) {
                    const T v = x[t];
                    mx = v >= mx ? v : mx;  // walking backwards: the earlier index wins ties
                    mn = v <= mn ? v : mn;
                    ox[t] = mx;
                    on[t] = mn;
                }
            }
        }
        __syncthreads();
        // combine, branch-free: consecutive threads -> consecutive elements
        // (conflict-free shared reads, coalesced streaming stores)
        for (int g = 0; g < g_here; ++g) {
            T* du = U + (s0 + g) * nd;
            T* dl = L + (s0 + g) * nd;
            const T* pb = PX + g * nd;
            for (int e = threadIdx.x; e < nd; e += blockDim.x) {
                const int i = e / d, p = e - i * d;  // compile-time d: multiply-shift
                const int2 tb = tab[i];
                const T* pa = pb + tb.x + p;
                const T* pc = pb + tb.y + p;
                const T xa = pa[0], xb = pc[0], na = pa[cap], nbv = pc[cap];
                __stcs(du + e, xb > xa ? xb : xa);  // A is the earlier index: it wins ties
                __stcs(dl + e, nbv < na ? nbv : na);
            }
        }
        __syncthreads();  // scans and combine done: X and the scan arrays may be reused
        T* t = X;
        X = Xn;
        Xn = t;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// TMA-fed van Herk envelope (windows 2W+1 <= 32).  A persistent block walks
// groups of G whole series.  One thread issues a TMA bulk copy
// (cp.async.bulk, completion counted on an mbarrier) per series of the NEXT
// group into the other of two shared-memory buffers while the current group
// is processed; each series lands in a slot padded to 4 words mod 32, so
// the lanes of a warp -- 8 series x 4 dimensions of one row -- hit distinct
// banks.  Rows are indexed in v = row + W, cut into blocks of
// k = 2W+1: the window of row i is v-block b = i / k from offset i % k plus
// v-block b+1 up to offset i % k - 1 (van Herk / Gil-Werman).  One thread
// per (series, dimension, block b): a backward scan of v-block b keeps its
// suffix max/min in registers, a forward scan of v-block b+1 completes the k
// outputs, staged in shared memory (same padded slots, conflict-free) and
// streamed out with coalesced 16-byte stores.  Rows outside [0, n) are the identity, which clips
// the window exactly as lb_mv.py:44-71.  Two block barriers per group of 8
// series (staged outputs complete / stages free).
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_expect(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
    }
}

constexpr int kVhMaxK = 32;  // largest window (2W+1) of the register-resident van Herk path
constexpr int kVhG = 8;      // series per group

// Padded series slot, in elements: 4 words mod 32 (16-byte aligned TMA
// destinations), so the 8 series of a group start in distinct bank quads.
__host__ __device__ inline int vh_slot_elems(int nd, int es) {
    int words = (nd * es / 4 + 3) & ~3;
    words += (4 - words % 32 + 32) % 32;
    return words * 4 / es;
}

template <typename T, int D, int KC>  // KC > 0: the window length 2W+1 as a compile-time constant
__global__ void __launch_bounds__(512) envelope_vh_kernel(const T* __restrict__ S, int64_t n_series, int n, int w,
                                                          T* __restrict__ U, T* __restrict__ Lo) {
    extern __shared__ __align__(128) unsigned char vh_smem[];
    const int nd = n * D;
    const int SS = vh_slot_elems(nd, (int)sizeof(T));
    T* buf = reinterpret_cast<T*>(vh_smem);                              // input [2][G][SS]
    T* ou = buf + 2 * kVhG * SS;                                         // output stages [G][SS] (upper,
    T* ol = ou + kVhG * SS;                                              // lower), same padded slots
    uint64_t* bar = reinterpret_cast<uint64_t*>(ol + kVhG * SS);        // 2 mbarriers
    const int k = KC > 0 ? KC : 2 * w + 1;
    constexpr int KU = KC > 0 ? KC : kVhMaxK;  // unrolled loop length
    const int nb = (n + k - 1) / k;          // output blocks per series
    const int tasks = kVhG * D * nb;         // (block, dim, series), series fastest
    const unsigned ser_bytes = (unsigned)(nd * sizeof(T));
    const T NEG = -dev_inf<T>(), POS = dev_inf<T>();
    const int64_t stride = (int64_t)gridDim.x * kVhG;
    auto issue = [&](int64_t s0, int slot) {  // one thread: TMA bulk copies of group s0
        if (s0 >= n_series) return;
        const int g = (int)((n_series - s0) < kVhG ? (n_series - s0) : kVhG);
        mbar_expect(bar + slot, ser_bytes * g);
        for (int j = 0; j < g; ++j)
            tma_load_1d(buf + ((size_t)slot * kVhG + j) * SS, S + (s0 + j) * (int64_t)nd, ser_bytes, bar + slot);
    };
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar + 1)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        issue((int64_t)blockIdx.x * kVhG, 0);
        issue((int64_t)blockIdx.x * kVhG + stride, 1);
    }
    __syncthreads();
    int it = 0;
    for (int64_t s0 = (int64_t)blockIdx.x * kVhG; s0 < n_series; s0 += stride, ++it) {
        const int slot = it & 1;
        const int g_here = (int)((n_series - s0) < kVhG ? (n_series - s0) : kVhG);
        mbar_wait(bar + slot, (unsigned)(it >> 1) & 1u);
        const T* X = buf + (size_t)slot * kVhG * SS;
        for (int t = threadIdx.x; t < tasks; t += blockDim.x) {
            // series fastest: a warp's lanes read one row of 8 series x 4
            // dimensions, one bank each (slots are 4 words mod 32 apart)
            const int sr = t % kVhG;
            const int p = (t / kVhG) % D;
            const int b = t / (D * kVhG);
            if (sr >= g_here) continue;
            const T* x = X + (size_t)sr * SS + p;
            // v-block b: rows r0 .. r0+k-1 with r0 = b*k - w; suffix extrema.
            // Interior tasks (both v-blocks inside [0, n)) skip the range checks.
            const int r0 = b * k - w;
            const int r1 = r0 + k;  // first row of v-block b+1
            const bool interior = r0 >= 0 && r1 + k - 1 < n;
            T hx[KU], hn[KU];
            T* du = ou + (size_t)sr * SS + p;
            T* dl = ol + (size_t)sr * SS + p;
            T gx = NEG, gn = POS;
            if (interior) {
                T mx = NEG, mn = POS;
#pragma unroll
                for (int j = KU - 1; j >= 0; --j) {
                    if (KC > 0 || j < k) {
                        const T v = x[(r0 + j) * D];
                        mx = v > mx ? v : mx;
                        mn = v < mn ? v : mn;
                    }
                    hx[j] = mx;
                    hn[j] = mn;
                }
                // outputs i = b*k + j: h[j] (v-block b from offset j) with the
                // prefix of v-block b+1 up to offset j-1 (all rows < n here)
#pragma unroll
                for (int j = 0; j < KU; ++j) {
                    if (KC > 0 || j < k) {
                        if (j > 0) {
                            const T v = x[(r1 + j - 1) * D];
                            gx = v > gx ? v : gx;
                            gn = v < gn ? v : gn;
                        }
                        du[(b * k + j) * D] = gx > hx[j] ? gx : hx[j];
                        dl[(b * k + j) * D] = gn < hn[j] ? gn : hn[j];
                    }
                }
            } else {
                T mx = NEG, mn = POS;
#pragma unroll
                for (int j = KU - 1; j >= 0; --j) {
                    if (KC > 0 || j < k) {
                        const int r = r0 + j;
                        if ((unsigned)r < (unsigned)n) {
                            const T v = x[r * D];
                            mx = v > mx ? v : mx;
                            mn = v < mn ? v : mn;
                        }
                    }
                    hx[j] = mx;
                    hn[j] = mn;
                }
#pragma unroll
                for (int j = 0; j < KU; ++j) {
                    if (KC > 0 || j < k) {
                        const int i = b * k + j;
                        if (j > 0) {
                            const int r = r1 + j - 1;
                            if ((unsigned)r < (unsigned)n) {
                                const T v = x[r * D];
                                gx = v > gx ? v : gx;
                                gn = v < gn ? v : gn;
                            }
                        }
                        if (i < n) {
                            du[i * D] = gx > hx[j] ? gx : hx[j];
                            dl[i * D] = gn < hn[j] ? gn : hn[j];
                        }
                    }
                }
            }
        }
        __syncthreads();  // group consumed (its input buffer may be refilled), outputs staged
        if (threadIdx.x == 0) issue(s0 + 2 * stride, slot);
        // coalesced 16-byte streaming stores of the staged series
        {
            constexpr int VE = 16 / (int)sizeof(T);
            using V4 = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
            const int nv = nd / VE;
            for (int e = threadIdx.x; e < g_here * nv; e += blockDim.x) {
                const int sr = e / nv, v = e - sr * nv;
                const V4 xu = *reinterpret_cast<const V4*>(ou + (size_t)sr * SS + v * VE);
                const V4 xl = *reinterpret_cast<const V4*>(ol + (size_t)sr * SS + v * VE);
                __stcs(reinterpret_cast<V4*>(U + (s0 + sr) * (int64_t)nd) + v, xu);
                __stcs(reinterpret_cast<V4*>(Lo + (s0 + sr) * (int64_t)nd) + v, xl);
            }
        }
        __syncthreads();  // output stages free
    }
}

// Sequential prefix sum with first-prefix abandoning (core.py:133-146).
template <typename T>
struct PrefixAbandon {
    T cs = T(0);
    T first = T(0);
    bool found = false;
    bool has;
    T thr;
    __device__ PrefixAbandon(bool h, T t) : has(h), thr(t) {}
    __device__ __forceinline__ void add(T x) {
        cs = add_rn(cs, x);
        if (has && !found && cs > thr) {
            first = cs;
            found = true;
        }
    }
    __device__ __forceinline__ void finish(T* out_v, uint8_t* out_ab) const {
        if (has && cs > thr) {
            *out_v = first;
            *out_ab = 1;
        } else {
            *out_v = cs;
            *out_ab = 0;
        }
    }
};

// ------------------------------------------------------------------- lb_mv
template <typename T, int DMAX>
__global__ void lb_mv_pairs_kernel(const T* __restrict__ C, const T* __restrict__ U,
                                   const T* __restrict__ L, int64_t P, int n, int d,
                                   const T* __restrict__ thr_arr, T* __restrict__ out_v,
                                   uint8_t* __restrict__ out_ab) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= P) return;
    const int64_t base = p * (int64_t)n * d;
    PrefixAbandon<T> acc(thr_arr != nullptr, thr_arr ? thr_arr[p] : T(0));
    for (int t = 0; t < n; ++t) {
        T c[DMAX];
        load_point<T, DMAX>(c, C + base + (int64_t)t * d, d);
        acc.add(lbmv_term_exact<T, DMAX>(c, U + base + (int64_t)t * d, L + base + (int64_t)t * d, d));
    }
    acc.finish(out_v + p, out_ab + p);
}

// ------------------------------------------------------------------- lb_ad
// lb_mv.py:110-128: per candidate index, nearest in-window query point.
template <typename T, int DMAX>
__global__ void lb_ad_pairs_kernel(const T* __restrict__ Q, const T* __restrict__ C, int64_t P, int n,
                                   int d, int w, const T* __restrict__ thr_arr, T* __restrict__ out_v,
                                   uint8_t* __restrict__ out_ab) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= P) return;
    const T* qa = Q + p * (int64_t)n * d;
    const T* ca = C + p * (int64_t)n * d;
    PrefixAbandon<T> acc(thr_arr != nullptr, thr_arr ? thr_arr[p] : T(0));
    for (int t = 0; t < n; ++t) {
        T c[DMAX];
        load_point<T, DMAX>(c, ca + (int64_t)t * d, d);
        const int lo = t - w < 0 ? 0 : t - w;
        const int hi = t + w > n - 1 ? n - 1 : t + w;
        T m = dev_inf<T>();
        for (int j = lo; j <= hi; ++j) {
            const T v = dist_exact<T, DMAX>(c, qa + (int64_t)j * d, d);
            m = v < m ? v : m;
        }
        acc.add(m);
    }
    acc.finish(out_v + p, out_ab + p);
}

// ---------------------------------------------------------- neighbor_steps
template <typename T, int DMAX>
__global__ void steps_kernel(const T* __restrict__ S, int64_t n_series, int n, int d, T* __restrict__ out) {
    const int64_t total = n_series * (int64_t)(n - 1);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = e / (n - 1);
        const int t = (int)(e - s * (n - 1));
        const T* a = S + s * (int64_t)n * d;
        T x[DMAX];
        load_point<T, DMAX>(x, a + (int64_t)(t + 1) * d, d);
        out[e] = dist_exact<T, DMAX>(x, a + (int64_t)t * d, d);
    }
}

template <typename T>
__global__ void ti_advance_kernel(const T* lo, const T* up, const T* st, int64_t count, T* olo, T* oup) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
         e += (int64_t)gridDim.x * blockDim.x) {
        T l = lo[e], u = up[e];
        ti_advance<T>(l, u, st[e]);
        olo[e] = l;
        oup[e] = u;
    }
}

// ------------------------------------------------------------------- lb_ti
// lb_ti.py:96-200.  Interval slots and column minima are indexed by
// candidate column in per-pair global scratch (3n values).
template <typename T, int DMAX>
__global__ void lb_ti_pairs_kernel(const T* __restrict__ Q, const T* __restrict__ C, int64_t P, int n,
                                   int d, int w, int variant, int period, const T* __restrict__ qsteps,
                                   const T* __restrict__ csteps, const T* __restrict__ thr_arr,
                                   T* __restrict__ out_v, uint8_t* __restrict__ out_ab,
                                   T* __restrict__ scratch) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= P) return;
    const T* qa = Q + p * (int64_t)n * d;
    const T* ca = C + p * (int64_t)n * d;
    const T* qs = qsteps ? qsteps + p * (int64_t)(n - 1) : nullptr;
    const T* cs = csteps ? csteps + p * (int64_t)(n - 1) : nullptr;
    T* lo_arr = scratch + p * 3 * (int64_t)n;
    T* up_arr = lo_arr + n;
    T* colmin = up_arr + n;
    const bool refreshing = (variant == TCDTW_TI_TIP || variant == TCDTW_TI_TIP_TOP);
    const bool true_top = (variant == TCDTW_TI_TOP || variant == TCDTW_TI_TIP_TOP);
    const T INF = dev_inf<T>();
    const bool has = thr_arr != nullptr;
    const T threshold = has ? thr_arr[p] : INF;
    for (int j = 0; j < n; ++j) colmin[j] = INF;
    int hi = w < n - 1 ? w : n - 1;
    {
        T q0[DMAX];
        load_point<T, DMAX>(q0, qa, d);
        for (int j = 0; j <= hi; ++j) {
            const T dd = dist_exact<T, DMAX>(q0, ca + (int64_t)j * d, d);
            lo_arr[j] = up_arr[j] = colmin[j] = dd;
        }
    }
    T running = T(0);
    int next_final = 0, prev_lo = 0, prev_hi = hi;
    for (int i = 1; i < n; ++i) {
        const int lo = i - w > 0 ? i - w : 0;
        hi = i + w < n - 1 ? i + w : n - 1;
        T qi[DMAX];
        load_point<T, DMAX>(qi, qa + (int64_t)i * d, d);
        if (refreshing && i % period == 0) {
            for (int j = lo; j <= hi; ++j) {
                const T dd = dist_exact<T, DMAX>(qi, ca + (int64_t)j * d, d);
                lo_arr[j] = up_arr[j] = dd;
            }
        } else {
            T s;
            if (qs) {
                s = qs[i - 1];
            } else {
                s = dist_exact<T, DMAX>(qi, qa + (int64_t)(i - 1) * d, d);
            }
            if (s > T(0))
                for (int j = prev_lo; j <= prev_hi; ++j) ti_advance<T>(lo_arr[j], up_arr[j], s);
            if (hi > prev_hi) {
                if (true_top) {
                    const T dd = dist_exact<T, DMAX>(qi, ca + (int64_t)hi * d, d);
                    lo_arr[hi] = up_arr[hi] = dd;
                } else {
                    T cstep;
                    if (cs) {
                        cstep = cs[hi - 1];
                    } else {
                        T x[DMAX];
                        load_point<T, DMAX>(x, ca + (int64_t)hi * d, d);
                        cstep = dist_exact<T, DMAX>(x, ca + (int64_t)(hi - 1) * d, d);
                    }
                    T l2 = lo_arr[hi - 1], u2 = up_arr[hi - 1];
                    ti_advance<T>(l2, u2, cstep);
                    lo_arr[hi] = l2;
                    up_arr[hi] = u2;
                }
            }
        }
        for (int j = lo; j <= hi; ++j) colmin[j] = lo_arr[j] < colmin[j] ? lo_arr[j] : colmin[j];
        while (next_final <= i - w) {
            running = add_rn(running, colmin[next_final]);
            ++next_final;
            if (running > threshold) {
                out_v[p] = running;
                out_ab[p] = 1;
                return;
            }
        }
        prev_lo = lo;
        prev_hi = hi;
    }
    while (next_final < n) {
        running = add_rn(running, colmin[next_final]);
        ++next_final;
        if (running > threshold) {
            out_v[p] = running;
            out_ab[p] = 1;
            return;
        }
    }
    out_v[p] = running;
    out_ab[p] = 0;
}

// ------------------------------------------------------------ box builder
// build_box_sets / quantize_cluster (lb_pc.py:56-116, :167-261), one warp
// per (series, expanded window).  Cell assignment runs in float64 whatever
// the storage type, exactly as the reference (IEEE division, truncation,
// clip, mixed-radix ids with dimension 0 most significant); cells are
// visited in increasing id order and cells from slot max_boxes-1 on merge.
__device__ __forceinline__ long long warp_min_ll(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        long long x = __shfl_xor_sync(0xffffffffu, v, o);
        v = x < v ? x : v;
    }
    return v;
}
__device__ __forceinline__ double warp_min_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

template <typename T>
__device__ __forceinline__ long long cell_id(const T* pt, int d, const double* mn, const double* seg,
                                             const int* lev, const long long* wgt) {
    long long id = 0;
    for (int p = 0; p < d; ++p) {
        if (lev[p] > 1) {
            const double scaled = __ddiv_rn(__dsub_rn((double)pt[p], mn[p]), seg[p]);
            long long ci = (long long)scaled;  // astype(np.int64): truncation
            ci = ci < 0 ? 0 : ci;
            ci = ci > lev[p] - 1 ? lev[p] - 1 : ci;
            id += ci * wgt[p];
        }
    }
    return id;
}

template <typename T>
__global__ void box_sets_kernel(const T* __restrict__ S, int64_t n_series, int n, int d, int w, int gw,
                                int levels, int K, double mcf, const T* __restrict__ dim_range,
                                T* __restrict__ out_lo, T* __restrict__ out_hi,
                                int32_t* __restrict__ out_counts) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warps = blockDim.x >> 5;
    const int wib = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // per-warp scratch: mn, seg (double), wgt (long long), lev (int)
    double* mn = reinterpret_cast<double*>(smem_raw) + (size_t)wib * d * 3;
    double* seg = mn + d;
    long long* wgt = reinterpret_cast<long long*>(seg + d);
    int* lev = reinterpret_cast<int*>(reinterpret_cast<double*>(smem_raw) + (size_t)warps * d * 3) + wib * d;
    const int G = (n - 1) / gw + 1;
    const int64_t job = blockIdx.x * (int64_t)warps + wib;
    if (job >= n_series * G) return;
    const int64_t s = job / G;
    const int g = (int)(job - s * G);
    const T* qa = S + s * (int64_t)n * d;
    int a = g * gw - w;
    a = a < 0 ? 0 : a;
    int b = g * gw + w + gw - 1;
    b = b > n - 1 ? n - 1 : b;
    T* olo = out_lo + job * (int64_t)K * d;
    T* ohi = out_hi + job * (int64_t)K * d;
    const double DINF = __longlong_as_double(0x7ff0000000000000LL);
    for (int e = lane; e < K * d; e += 32) {
        olo[e] = dev_inf<T>();
        ohi[e] = -dev_inf<T>();
    }
    bool any = false;
    for (int p = 0; p < d; ++p) {
        double lmn = DINF, lmx = -DINF;
        for (int t = a + lane; t <= b; t += 32) {
            const double v = (double)qa[(int64_t)t * d + p];
            lmn = fmin(lmn, v);
            lmx = fmax(lmx, v);
        }
        const double gmn = warp_min_d(lmn), gmx = warp_max_d(lmx);
        double ref;
        if (dim_range) {
            ref = (double)dim_range[p];
        } else {
            double rmn = DINF, rmx = -DINF;
            for (int t = lane; t < n; t += 32) {
                const double v = (double)qa[(int64_t)t * d + p];
                rmn = fmin(rmn, v);
                rmx = fmax(rmx, v);
            }
            ref = __dsub_rn(warp_max_d(rmx), warp_min_d(rmn));
        }
        const double rng = __dsub_rn(gmx, gmn);
        const bool split = (rng > 0.0) && (rng >= __dmul_rn(mcf, ref));
        any |= split;
        if (lane == 0) {
            mn[p] = gmn;
            lev[p] = split ? levels : 1;
            seg[p] = split ? __ddiv_rn(rng, (double)levels) : 1.0;
            olo[p] = (T)gmn;  // the single box, kept when nothing splits
            ohi[p] = (T)gmx;
        }
    }
    __syncwarp();
    if (levels == 1 || !any) {
        if (lane == 0) out_counts[job] = 1;
        return;
    }
    if (lane == 0) {
        wgt[d - 1] = 1;
        for (int p = d - 2; p >= 0; --p) wgt[p] = wgt[p + 1] * (long long)lev[p + 1];
    }
    __syncwarp();
    const long long NONE = 0x7fffffffffffffffLL;
    long long prev = -1;
    int nb = 0;
    while (true) {
        const bool last_slot = (nb == K - 1);
        // smallest cell id above prev (or, for the last slot, all remaining)
        long long lm = NONE;
        for (int t = a + lane; t <= b; t += 32) {
            const long long id = cell_id<T>(qa + (int64_t)t * d, d, mn, seg, lev, wgt);
            if (id > prev && id < lm) lm = id;
        }
        const long long cid = warp_min_ll(lm);
        if (cid == NONE) break;
        for (int p = 0; p < d; ++p) {
            double lmn = DINF, lmx = -DINF;
            for (int t = a + lane; t <= b; t += 32) {
                const T* pt = qa + (int64_t)t * d;
                const long long id = cell_id<T>(pt, d, mn, seg, lev, wgt);
                if (last_slot ? (id > prev) : (id == cid)) {
                    const double v = (double)pt[p];
                    lmn = fmin(lmn, v);
                    lmx = fmax(lmx, v);
                }
            }
            lmn = warp_min_d(lmn);
            lmx = warp_max_d(lmx);
            if (lane == 0) {
                olo[(int64_t)nb * d + p] = (T)lmn;
                ohi[(int64_t)nb * d + p] = (T)lmx;
            }
        }
        ++nb;
        prev = cid;
        if (last_slot) break;
    }
    if (lane == 0) out_counts[job] = nb;
}

// ------------------------------------------------------------------- lb_pc
template <typename T, int DMAX>
__global__ void lb_pc_pairs_kernel(const T* __restrict__ C, const T* __restrict__ BL,
                                   const T* __restrict__ BH, int64_t P, int n, int d, int G, int K,
                                   int gw, const T* __restrict__ thr_arr, T* __restrict__ out_v,
                                   uint8_t* __restrict__ out_ab) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= P) return;
    const T* ca = C + p * (int64_t)n * d;
    const T* bl = BL + p * (int64_t)G * K * d;
    const T* bh = BH + p * (int64_t)G * K * d;
    PrefixAbandon<T> acc(thr_arr != nullptr, thr_arr ? thr_arr[p] : T(0));
    for (int t = 0; t < n; ++t) {
        T c[DMAX];
        load_point<T, DMAX>(c, ca + (int64_t)t * d, d);
        const int g = t / gw;
        T best = dev_inf<T>();
        for (int k = 0; k < K; ++k) {
            const T v = boxdist2_exact<T, DMAX>(c, bl + ((int64_t)g * K + k) * d, bh + ((int64_t)g * K + k) * d, d);
            best = v < best ? v : best;
        }
        acc.add(sqrt_rn(best));
    }
    acc.finish(out_v + p, out_ab + p);
}

// =================================================================== host
namespace {

struct DtwPairsOp {
    template <typename T, int DM>
    int run(const void* a, const void* b, int64_t P, int n, int d, int w, const void* thr, void* out,
            uint8_t* ab, int64_t* cells, cudaStream_t st) {
        const int width = 2 * w + 1;
        T* scratch = nullptr;
        if (cudaMallocAsync(&scratch, sizeof(T) * 2 * (size_t)width * P, st) != cudaSuccess)
            return TCDTW_CUDA_ERROR;
        dtw_pairs_kernel<T, DM><<<grid_for(P, 64), 64, 0, st>>>(
            (const T*)a, (const T*)b, P, n, d, w, (const T*)thr, (T*)out, ab, cells, scratch);
        int s = launch_status();
        cudaFreeAsync(scratch, st);
        return s;
    }
};

struct LbMvPairsOp {
    template <typename T, int DM>
    int run(const void* c, const void* u, const void* l, int64_t P, int n, int d, const void* thr,
            void* out, uint8_t* ab, cudaStream_t st) {
        lb_mv_pairs_kernel<T, DM><<<grid_for(P, 128), 128, 0, st>>>(
            (const T*)c, (const T*)u, (const T*)l, P, n, d, (const T*)thr, (T*)out, ab);
        return launch_status();
    }
};

struct LbAdPairsOp {
    template <typename T, int DM>
    int run(const void* q, const void* c, int64_t P, int n, int d, int w, const void* thr, void* out,
            uint8_t* ab, cudaStream_t st) {
        lb_ad_pairs_kernel<T, DM><<<grid_for(P, 128), 128, 0, st>>>(
            (const T*)q, (const T*)c, P, n, d, w, (const T*)thr, (T*)out, ab);
        return launch_status();
    }
};

struct StepsOp {
    template <typename T, int DM>
    int run(const void* s, int64_t ns, int n, int d, void* out, cudaStream_t st) {
        const int64_t total = ns * (int64_t)(n - 1);
        if (total <= 0) return TCDTW_OK;
        steps_kernel<T, DM><<<grid_for(total, 256) > 65535 ? 65535 : grid_for(total, 256), 256, 0, st>>>(
            (const T*)s, ns, n, d, (T*)out);
        return launch_status();
    }
};

struct LbTiPairsOp {
    template <typename T, int DM>
    int run(const void* q, const void* c, int64_t P, int n, int d, int w, int variant, int period,
            const void* qs, const void* cs, const void* thr, void* out, uint8_t* ab, cudaStream_t st) {
        T* scratch = nullptr;
        if (cudaMallocAsync(&scratch, sizeof(T) * 3 * (size_t)n * P, st) != cudaSuccess)
            return TCDTW_CUDA_ERROR;
        lb_ti_pairs_kernel<T, DM><<<grid_for(P, 64), 64, 0, st>>>(
            (const T*)q, (const T*)c, P, n, d, w, variant, period, (const T*)qs, (const T*)cs,
            (const T*)thr, (T*)out, ab, scratch);
        int s = launch_status();
        cudaFreeAsync(scratch, st);
        return s;
    }
};

struct LbPcPairsOp {
    template <typename T, int DM>
    int run(const void* c, const void* bl, const void* bh, int64_t P, int n, int d, int G, int K, int gw,
            const void* thr, void* out, uint8_t* ab, cudaStream_t st) {
        lb_pc_pairs_kernel<T, DM><<<grid_for(P, 128), 128, 0, st>>>(
            (const T*)c, (const T*)bl, (const T*)bh, P, n, d, G, K, gw, (const T*)thr, (T*)out, ab);
        return launch_status();
    }
};

}  // namespace

int pairs_dtw(int dtype, const void* a, const void* b, int64_t P, int n, int d, int w, const void* thr,
              void* out, uint8_t* ab, int64_t* cells, cudaStream_t st) {
    return dispatch_dtype_dims(dtype, d, DtwPairsOp{}, a, b, P, n, d, w, thr, out, ab, cells, st);
}
int pairs_lb_mv(int dtype, const void* c, const void* u, const void* l, int64_t P, int n, int d,
                const void* thr, void* out, uint8_t* ab, cudaStream_t st) {
    return dispatch_dtype_dims(dtype, d, LbMvPairsOp{}, c, u, l, P, n, d, thr, out, ab, st);
}
int pairs_lb_ad(int dtype, const void* q, const void* c, int64_t P, int n, int d, int w, const void* thr,
                void* out, uint8_t* ab, cudaStream_t st) {
    return dispatch_dtype_dims(dtype, d, LbAdPairsOp{}, q, c, P, n, d, w, thr, out, ab, st);
}
int series_steps(int dtype, const void* s, int64_t ns, int n, int d, void* out, cudaStream_t st) {
    return dispatch_dtype_dims(dtype, d, StepsOp{}, s, ns, n, d, out, st);
}
int pairs_lb_ti(int dtype, const void* q, const void* c, int64_t P, int n, int d, int w, int variant,
                int period, const void* qs, const void* cs, const void* thr, void* out, uint8_t* ab,
                cudaStream_t st) {
    return dispatch_dtype_dims(dtype, d, LbTiPairsOp{}, q, c, P, n, d, w, variant, period, qs, cs, thr, out,
                               ab, st);
}
int pairs_lb_pc(int dtype, const void* c, const void* bl, const void* bh, int64_t P, int n, int d, int G,
                int K, int gw, const void* thr, void* out, uint8_t* ab, cudaStream_t st) {
    return dispatch_dtype_dims(dtype, d, LbPcPairsOp{}, c, bl, bh, P, n, d, G, K, gw, thr, out, ab, st);
}

// The TMA-fed van Herk path: windows up to 32 points, series whose bytes are
// a 16-byte multiple, 16-byte aligned arrays.
static int envelope_vh(int dtype, const void* s, int64_t ns, int n, int d, int w, void* u, void* l,
                       cudaStream_t st) {
    const int es = dtype == TCDTW_F64 ? 8 : 4;
    if (2 * w + 1 > kVhMaxK || ((int64_t)n * d * es) % 16 != 0) return TCDTW_NOT_SUPPORTED;
    if (((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(u) | reinterpret_cast<uintptr_t>(l)) & 15) != 0)
        return TCDTW_NOT_SUPPORTED;
    const size_t smem = (size_t)4 * kVhG * vh_slot_elems(n * d, es) * es + 16;
    if (smem > 200 * 1024) return TCDTW_NOT_SUPPORTED;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // one thread per (series, dimension, block) task of a group
    const int k = 2 * w + 1, tasks = kVhG * d * ((n + k - 1) / k);
    int threads = (tasks + 31) / 32 * 32;
    threads = threads > 512 ? 512 : threads;
    auto go = [&](auto kern, auto* S, auto* U, auto* L) -> int {
        if (smem > 48 * 1024 &&
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return TCDTW_NOT_SUPPORTED;
        int occ = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
        int64_t grid = (int64_t)(occ < 1 ? 1 : occ) * sms;
        const int64_t groups = (ns + kVhG - 1) / kVhG;
        if (grid > groups) grid = groups;
        kern<<<(int)grid, threads, smem, st>>>(S, ns, n, w, U, L);
        return launch_status();
    };
#define TCDTW_VH_K(DD, KK)                                                                              \
    if (k == KK) {                                                                                      \
        if (dtype == TCDTW_F64)                                                                         \
            return go(envelope_vh_kernel<double, DD, KK>, (const double*)s, (double*)u, (double*)l);   \
        return go(envelope_vh_kernel<float, DD, KK>, (const float*)s, (float*)u, (float*)l);           \
    }
#define TCDTW_VH(DD)                                                                                    \
    if (d == DD) {                                                                                      \
        TCDTW_VH_K(DD, 25) TCDTW_VH_K(DD, 13)                                                           \
        if (dtype == TCDTW_F64)                                                                         \
            return go(envelope_vh_kernel<double, DD, 0>, (const double*)s, (double*)u, (double*)l);    \
        return go(envelope_vh_kernel<float, DD, 0>, (const float*)s, (float*)u, (float*)l);            \
    }
    TCDTW_VH(1) TCDTW_VH(2) TCDTW_VH(3) TCDTW_VH(4) TCDTW_VH(5) TCDTW_VH(6) TCDTW_VH(8) TCDTW_VH(20)
#undef TCDTW_VH
#undef TCDTW_VH_K
    return TCDTW_NOT_SUPPORTED;
}

int series_envelope(int dtype, const void* s, int64_t ns, int n, int d, int w, void* u, void* l,
                    cudaStream_t st) {
    if (ns <= 0) return TCDTW_OK;
    {
        const int r = envelope_vh(dtype, s, ns, n, d, w, u, l, st);
        if (r != TCDTW_NOT_SUPPORTED) return r;
    }
    const int64_t total = ns * (int64_t)n * d;
    const size_t es = dtype == TCDTW_F64 ? 8 : 4;
    const size_t per_series = (size_t)6 * n * d * es;  // 2 staging + 4 scan arrays
    if (per_series + (size_t)8 * n <= 200 * 1024 && n < (1 << 30)) {
        // ~72 KB per block (3 resident per SM): each keeps one group of
        // reads in flight while it scans the previous one
        constexpr int kb = 54;  // staging KB per block (18 / 36 / 54 / 72 KB measured: 54 best)
        int G = (int)((kb * 1024) / per_series);
        G = G < 1 ? 1 : G;
        const size_t smem = per_series * G + (size_t)8 * n;  // + the per-row window table
        int dev = 0, sms = 148, occ = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        auto go = [&](auto kern, auto* S, auto* U, auto* L) -> int {
            if (smem > 48 * 1024 &&
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
                return TCDTW_CUDA_ERROR;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
            const int64_t groups = (ns + G - 1) / G;
            int64_t grid = (int64_t)(occ < 1 ? 1 : occ) * sms;
            if (grid > groups) grid = groups;
            kern<<<(int)grid, 256, smem, st>>>(S, ns, n, d, w, G, U, L);
            return launch_status();
        };
#define TCDTW_ENV_CASE(DD)                                                                             \
        if (d == DD) {                                                                                 \
            if (dtype == TCDTW_F64)                                                                    \
                return go(envelope_stream_kernel<double, DD>, (const double*)s, (double*)u, (double*)l); \
            return go(envelope_stream_kernel<float, DD>, (const float*)s, (float*)u, (float*)l);       \
        }
        TCDTW_ENV_CASE(1) TCDTW_ENV_CASE(2) TCDTW_ENV_CASE(3) TCDTW_ENV_CASE(4) TCDTW_ENV_CASE(5)
        TCDTW_ENV_CASE(6) TCDTW_ENV_CASE(8) TCDTW_ENV_CASE(20)
#undef TCDTW_ENV_CASE
        if (dtype == TCDTW_F64)
            return go(envelope_stream_kernel<double, 0>, (const double*)s, (double*)u, (double*)l);
        return go(envelope_stream_kernel<float, 0>, (const float*)s, (float*)u, (float*)l);
    }
    const int grid = grid_for(total, 256) > 148 * 64 ? 148 * 64 : grid_for(total, 256);
    if (dtype == TCDTW_F64)
        envelope_kernel<double><<<grid, 256, 0, st>>>((const double*)s, ns, n, d, w, (double*)u, (double*)l);
    else
        envelope_kernel<float><<<grid, 256, 0, st>>>((const float*)s, ns, n, d, w, (float*)u, (float*)l);
    return launch_status();
}

int ti_advance_elementwise(int dtype, const void* lo, const void* up, const void* st_, int64_t count,
                           void* olo, void* oup, cudaStream_t st) {
    if (count <= 0) return TCDTW_OK;
    const int grid = grid_for(count, 256) > 4096 ? 4096 : grid_for(count, 256);
    if (dtype == TCDTW_F64)
        ti_advance_kernel<double><<<grid, 256, 0, st>>>((const double*)lo, (const double*)up,
                                                        (const double*)st_, count, (double*)olo, (double*)oup);
    else
        ti_advance_kernel<float><<<grid, 256, 0, st>>>((const float*)lo, (const float*)up, (const float*)st_,
                                                       count, (float*)olo, (float*)oup);
    return launch_status();
}

int series_box_sets(int dtype, const void* s, int64_t ns, int n, int d, int w, int gw, int levels, int K,
                    double mcf, const void* dr, void* olo, void* ohi, int32_t* counts, cudaStream_t st) {
    const int G = (n - 1) / gw + 1;
    const int64_t jobs = ns * (int64_t)G;
    const int warps = 4;
    const size_t smem = (size_t)warps * d * (3 * sizeof(double) + sizeof(int));
    const int grid = grid_for(jobs, warps);
    if (dtype == TCDTW_F64)
        box_sets_kernel<double><<<grid, warps * 32, smem, st>>>((const double*)s, ns, n, d, w, gw, levels, K,
                                                                mcf, (const double*)dr, (double*)olo,
                                                                (double*)ohi, counts);
    else
        box_sets_kernel<float><<<grid, warps * 32, smem, st>>>((const float*)s, ns, n, d, w, gw, levels, K, mcf,
                                                               (const float*)dr, (float*)olo, (float*)ohi,
                                                               counts);
    return launch_status();
}

}  // namespace tcdtw
