/*
 * tcdtw_oracle.c -- CPU ORACLE (TEST INFRASTRUCTURE ONLY).
 *
 * This file is the parity checker for the B200 path, never part of it.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product package
 * (paper_2101_07731_b200) never imports, links or calls anything here.
 *
 * It is a plain-C restatement of the reference's hot-path algorithms
 * (mvdtw v0.1.0, /root/reference/pkg/src/mvdtw), written to reproduce the
 * reference's float64 arithmetic bit for bit:
 *   - every point distance is sqrt(sum_p diff_p^2) with numpy's pairwise
 *     summation order for a contiguous last-axis reduction (sequential for
 *     D < 8, eight interleaved accumulators for 8 <= D <= 128), no FMA
 *     contraction (build with -ffp-contract=off), IEEE sqrt;
 *   - every bound is a sequential prefix sum with first-prefix abandoning
 *     (core.py:133-146).
 * Parity is pinned by tests/test_oracle_golden.py against vectors produced
 * by the reference itself (tests/golden/make_golden.py).
 *
 * Citations are file:line relative to /root/reference/pkg/src/mvdtw.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_INF (1.0 / 0.0)

/* ------------------------------------------------------------------ */
/* numpy pairwise sum of n contiguous doubles (numpy loops_utils.h:    */
/* pairwise_sum; n < 8 sequential from 0, else 8 accumulators).        */
/* Used for every reduction over the dimension axis in the reference:  */
/* core.py:110-111, dtw.py:40, lb_mv.py:95, lb_ti.py:55,180,           */
/* lb_pc.py:278.                                                       */
/* ------------------------------------------------------------------ */
static double np_pairwise_sum(const double *a, int n)
{
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; i++) res += a[i];
        return res;
    }
    if (n <= 128) {
        double r[8];
        int i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    }
    /* numpy recursion for blocks > 128: split at n2 = n/2 rounded down to 8 */
    int n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}

#define OR_MAXD 256

/* Euclidean point distance, core.py:104-111 (dists_to_rows) */
static double pdist(const double *a, const double *b, int d)
{
    double sq[OR_MAXD];
    for (int p = 0; p < d; p++) {
        double df = a[p] - b[p];
        sq[p] = df * df;
    }
    return sqrt(np_pairwise_sum(sq, d));
}

/* sum_with_abandon, core.py:133-146: sequential cumsum; if the total     */
/* exceeds the threshold, return the first prefix above it.               */
static void sum_with_abandon(const double *per_point, int n, int has_thr, double thr,
                             double *value, int *abandoned)
{
    double cs = 0.0;
    double first_above = 0.0;
    int found = 0;
    for (int t = 0; t < n; t++) {
        cs += per_point[t];
        if (has_thr && !found && cs > thr) {
            first_above = cs;
            found = 1;
        }
    }
    if (has_thr && cs > thr) {
        *value = first_above;
        *abandoned = 1;
    } else {
        *value = cs;
        *abandoned = 0;
    }
}

/* ------------------------------------------------------------------ */
/* dtw_banded, dtw.py:45-102                                           */
/* ------------------------------------------------------------------ */
void or_dtw_banded(const double *q, const double *c, int n, int d, int window,
                   int has_thr, double thr, double *distance, int *abandoned, int64_t *cells_out)
{
    int w = window < n - 1 ? window : n - 1; /* dtw.py:63 */
    int width = 2 * w + 1;
    double *prev = (double *)malloc(sizeof(double) * width);
    double *cur = (double *)malloc(sizeof(double) * width);
    double threshold = has_thr ? thr : OR_INF;
    int64_t cells = 0;
    for (int k = 0; k < width; k++) prev[k] = cur[k] = OR_INF;
    for (int i = 0; i < n; i++) {
        int lo = i < w ? 0 : i - w;
        int hi = i + w >= n ? n - 1 : i + w;
        for (int k = 0; k < width; k++) cur[k] = OR_INF;
        int k = lo - i + w;
        double row_min = OR_INF;
        for (int j = lo; j <= hi; j++) {
            double cost = pdist(q + (int64_t)i * d, c + (int64_t)j * d, d); /* cost_band dtw.py:33-42 */
            double v;
            if (i == 0 && j == 0) {
                v = cost;
            } else {
                double best = OR_INF;
                if (i > 0) {
                    if (k + 1 < width) best = prev[k + 1];
                    if (j > 0 && prev[k] < best) best = prev[k];
                }
                if (k > 0 && cur[k - 1] < best) best = cur[k - 1];
                v = cost + best;
            }
            cur[k] = v;
            if (v < row_min) row_min = v;
            k++;
        }
        cells += hi - lo + 1;
        if (row_min > threshold) { /* dtw.py:97-98 */
            *distance = row_min;
            *abandoned = 1;
            *cells_out = cells;
            free(prev);
            free(cur);
            return;
        }
        double *tmp = prev;
        prev = cur;
        cur = tmp;
    }
    double fin = prev[w]; /* dtw.py:101 */
    *distance = fin;
    *abandoned = fin > threshold;
    *cells_out = cells;
    free(prev);
    free(cur);
}

/* ------------------------------------------------------------------ */
/* build_envelope, lb_mv.py:74-88 (windowed max/min; exact values)     */
/* ------------------------------------------------------------------ */
void or_build_envelope(const double *q, int n, int d, int window, double *upper, double *lower)
{
    int w = window < n - 1 ? window : n - 1;
    for (int i = 0; i < n; i++) {
        int lo = i - w < 0 ? 0 : i - w;
        int hi = i + w > n - 1 ? n - 1 : i + w;
        for (int p = 0; p < d; p++) {
            double mx = q[(int64_t)lo * d + p], mn = mx;
            for (int j = lo + 1; j <= hi; j++) {
                double v = q[(int64_t)j * d + p];
                if (v > mx) mx = v;
                if (v < mn) mn = v;
            }
            upper[(int64_t)i * d + p] = mx;
            lower[(int64_t)i * d + p] = mn;
        }
    }
}

/* envelope_deviations + lb_mv, lb_mv.py:91-107 */
static double lb_mv_point(const double *cp, const double *up, const double *lp, int d)
{
    double sq[OR_MAXD];
    for (int p = 0; p < d; p++) {
        double hi = cp[p] - up[p];
        double lo = lp[p] - cp[p];
        hi = hi > 0.0 ? hi : 0.0;
        lo = lo > 0.0 ? lo : 0.0;
        sq[p] = hi * hi + lo * lo;
    }
    return sqrt(np_pairwise_sum(sq, d));
}

void or_lb_mv(const double *c, const double *upper, const double *lower, int n, int d,
              int has_thr, double thr, double *value, int *abandoned)
{
    double *pp = (double *)malloc(sizeof(double) * n);
    for (int t = 0; t < n; t++)
        pp[t] = lb_mv_point(c + (int64_t)t * d, upper + (int64_t)t * d, lower + (int64_t)t * d, d);
    sum_with_abandon(pp, n, has_thr, thr, value, abandoned);
    free(pp);
}

/* lb_ad, lb_mv.py:110-128: per candidate index, min distance to in-window query points */
void or_lb_ad(const double *q, const double *c, int n, int d, int window,
              int has_thr, double thr, double *value, int *abandoned)
{
    int w = window < n - 1 ? window : n - 1;
    double *pp = (double *)malloc(sizeof(double) * n);
    for (int t = 0; t < n; t++) {
        int lo = t - w < 0 ? 0 : t - w;
        int hi = t + w > n - 1 ? n - 1 : t + w;
        double m = OR_INF;
        for (int j = lo; j <= hi; j++) {
            double v = pdist(c + (int64_t)t * d, q + (int64_t)j * d, d); /* cross_dists(ca, qa) */
            if (v < m) m = v;
        }
        pp[t] = m;
    }
    sum_with_abandon(pp, n, has_thr, thr, value, abandoned);
    free(pp);
}

/* ------------------------------------------------------------------ */
/* LB_TI, lb_ti.py                                                     */
/* ------------------------------------------------------------------ */
#define PROP_SLACK (1.0 / 70368744177664.0) /* 2**-46, lb_ti.py:46 */

/* neighbor_steps, lb_ti.py:51-55 */
void or_neighbor_steps(const double *s, int n, int d, double *out)
{
    for (int t = 0; t + 1 < n; t++) out[t] = pdist(s + (int64_t)(t + 1) * d, s + (int64_t)t * d, d);
}

/* ti_advance, lb_ti.py:79-86 */
void or_ti_advance(double lo, double up, double step, double *lo_out, double *up_out)
{
    if (step == 0.0) {
        *lo_out = lo;
        *up_out = up;
        return;
    }
    double a = lo - step, b = step - up;
    double base = a;
    if (b > base) base = b;
    if (0.0 > base) base = 0.0;
    double t = up + step;
    double pad = t * PROP_SLACK;
    double l2 = base - pad;
    *lo_out = l2 > 0.0 ? l2 : 0.0;
    *up_out = t + pad;
}

/* vectorised advance, lb_ti.py:170-176 (np.maximum(np.maximum(lo-s, s-up), 0)) */
static inline void ti_adv_vec(double *lo, double *up, double s)
{
    double a = *lo - s, b = s - *up;
    double base = a > b ? a : b; /* np.maximum: NaN-free here */
    base = base > 0.0 ? base : 0.0;
    double t = *up + s;
    double pad = t * PROP_SLACK;
    double l2 = base - pad;
    *lo = l2 > 0.0 ? l2 : 0.0;
    *up = t + pad;
}

enum { TI_BASIC = 0, TI_TOP = 1, TI_TIP = 2, TI_TIP_TOP = 3 };

/* lb_ti, lb_ti.py:96-200 */
void or_lb_ti(const double *q, const double *c, int n, int d, int window, int variant,
              int refresh_period, const double *qsteps_in, int has_thr, double thr,
              double *value, int *abandoned)
{
    int w = window < n - 1 ? window : n - 1;
    double *qsteps = (double *)malloc(sizeof(double) * (n > 1 ? n - 1 : 1));
    double *csteps = (double *)malloc(sizeof(double) * (n > 1 ? n - 1 : 1));
    if (qsteps_in)
        memcpy(qsteps, qsteps_in, sizeof(double) * (n > 1 ? n - 1 : 0));
    else
        or_neighbor_steps(q, n, d, qsteps);
    int refreshing = (variant == TI_TIP || variant == TI_TIP_TOP);
    int true_top = (variant == TI_TOP || variant == TI_TIP_TOP);
    if (!true_top) or_neighbor_steps(c, n, d, csteps);
    double threshold = has_thr ? thr : OR_INF;
    double *lo_arr = (double *)malloc(sizeof(double) * n);
    double *up_arr = (double *)malloc(sizeof(double) * n);
    double *colmin = (double *)malloc(sizeof(double) * n);
    for (int j = 0; j < n; j++) colmin[j] = OR_INF;
    int hi = w < n - 1 ? w : n - 1;
    for (int j = 0; j <= hi; j++) {
        double dd = pdist(c + (int64_t)j * d, q, d); /* dists_to_rows(qa[0], ca[:hi+1]) */
        lo_arr[j] = up_arr[j] = colmin[j] = dd;
    }
    double running = 0.0;
    int next_final = 0, prev_lo = 0, prev_hi = hi;
    for (int i = 1; i < n; i++) {
        int lo = i - w > 0 ? i - w : 0;
        hi = i + w < n - 1 ? i + w : n - 1;
        if (refreshing && i % refresh_period == 0) {
            for (int j = lo; j <= hi; j++) {
                double dd = pdist(c + (int64_t)j * d, q + (int64_t)i * d, d);
                lo_arr[j] = up_arr[j] = dd;
            }
        } else {
            double s = qsteps[i - 1];
            if (s > 0.0)
                for (int j = prev_lo; j <= prev_hi; j++) ti_adv_vec(&lo_arr[j], &up_arr[j], s);
            if (hi > prev_hi) {
                if (true_top) {
                    double dd = pdist(q + (int64_t)i * d, c + (int64_t)hi * d, d);
                    lo_arr[hi] = up_arr[hi] = dd;
                } else {
                    double l2, u2;
                    or_ti_advance(lo_arr[hi - 1], up_arr[hi - 1], csteps[hi - 1], &l2, &u2);
                    lo_arr[hi] = l2;
                    up_arr[hi] = u2;
                }
            }
        }
        for (int j = lo; j <= hi; j++)
            if (lo_arr[j] < colmin[j]) colmin[j] = lo_arr[j];
        while (next_final <= i - w) {
            running += colmin[next_final];
            next_final++;
            if (running > threshold) {
                *value = running;
                *abandoned = 1;
                goto done;
            }
        }
        prev_lo = lo;
        prev_hi = hi;
    }
    while (next_final < n) {
        running += colmin[next_final];
        next_final++;
        if (running > threshold) {
            *value = running;
            *abandoned = 1;
            goto done;
        }
    }
    *value = running;
    *abandoned = 0;
done:
    free(qsteps);
    free(csteps);
    free(lo_arr);
    free(up_arr);
    free(colmin);
}

/* ------------------------------------------------------------------ */
/* LB_PC, lb_pc.py                                                     */
/* ------------------------------------------------------------------ */
typedef struct {
    int64_t id;
    int pos;
} idpos_t;

static int cmp_idpos(const void *a, const void *b)
{
    const idpos_t *x = (const idpos_t *)a, *y = (const idpos_t *)b;
    if (x->id < y->id) return -1;
    if (x->id > y->id) return 1;
    return x->pos - y->pos; /* stable */
}

/* Quantize one point set into <= max_boxes boxes: quantize_cluster        */
/* lb_pc.py:56-116, equivalently one group of _grouped_cells + _cap_cells  */
/* (lb_pc.py:167-236).  Writes up to max_boxes boxes; returns the count.   */
int or_quantize_points(const double *pts, int m, int d, int levels, int max_boxes,
                       double min_cell_frac, const double *ref, double *out_lo, double *out_hi)
{
    double mn[OR_MAXD], mx[OR_MAXD], rng[OR_MAXD], seg[OR_MAXD];
    int split[OR_MAXD], lev[OR_MAXD];
    int any = 0;
    for (int p = 0; p < d; p++) {
        mn[p] = mx[p] = pts[p];
        for (int t = 1; t < m; t++) {
            double v = pts[(int64_t)t * d + p];
            if (v < mn[p]) mn[p] = v;
            if (v > mx[p]) mx[p] = v;
        }
        rng[p] = mx[p] - mn[p];
        double r = ref ? ref[p] : rng[p];
        split[p] = (rng[p] > 0.0) && (rng[p] >= min_cell_frac * r);
        lev[p] = split[p] ? levels : 1;
        seg[p] = split[p] ? rng[p] / (double)lev[p] : 1.0;
        any |= split[p];
    }
    if (levels == 1 || !any) {
        for (int p = 0; p < d; p++) {
            out_lo[p] = mn[p];
            out_hi[p] = mx[p];
        }
        return 1;
    }
    int64_t weights[OR_MAXD];
    weights[d - 1] = 1;
    for (int p = d - 2; p >= 0; p--) weights[p] = weights[p + 1] * lev[p + 1];
    idpos_t *ids = (idpos_t *)malloc(sizeof(idpos_t) * m);
    for (int t = 0; t < m; t++) {
        int64_t id = 0;
        for (int p = 0; p < d; p++) {
            int64_t ci = 0;
            if (split[p]) {
                double scaled = (pts[(int64_t)t * d + p] - mn[p]) / seg[p];
                ci = (int64_t)scaled; /* astype(np.int64): truncation */
                if (ci < 0) ci = 0;
                if (ci > lev[p] - 1) ci = lev[p] - 1;
            }
            id += ci * weights[p];
        }
        ids[t].id = id;
        ids[t].pos = t;
    }
    qsort(ids, m, sizeof(idpos_t), cmp_idpos);
    int nb = 0;
    for (int s = 0; s < m;) {
        int e = s;
        while (e < m && ids[e].id == ids[s].id) e++;
        /* cell [s, e): tight box; cells from slot max_boxes-1 on merge */
        int slot = nb < max_boxes ? nb : max_boxes - 1;
        int fresh = nb < max_boxes;
        for (int k = s; k < e; k++) {
            const double *pt = pts + (int64_t)ids[k].pos * d;
            for (int p = 0; p < d; p++) {
                double *lo = &out_lo[(int64_t)slot * d + p], *hi = &out_hi[(int64_t)slot * d + p];
                if (fresh && k == s) {
                    *lo = pt[p];
                    *hi = pt[p];
                } else {
                    if (pt[p] < *lo) *lo = pt[p];
                    if (pt[p] > *hi) *hi = pt[p];
                }
            }
        }
        if (nb < max_boxes) nb++;
        s = e;
    }
    free(ids);
    return nb;
}

/* build_box_sets, lb_pc.py:239-261 -> padded (G, K, D) arrays (lo=+inf,
 * hi=-inf padding, lb_pc.py:229-234), counts and spans.  out_lo/out_hi
 * must hold G*max_boxes*d doubles. dim_range may be NULL (query's range). */
int or_num_groups(int n, int group_width) { return (n - 1) / group_width + 1; }

void or_build_box_sets(const double *q, int n, int d, int window, int group_width, int levels,
                       int max_boxes, double min_cell_frac, const double *dim_range,
                       double *out_lo, double *out_hi, int *out_counts, int *out_spans)
{
    int w = window < n - 1 ? window : n - 1;
    int G = or_num_groups(n, group_width);
    double ref[OR_MAXD];
    if (dim_range) {
        for (int p = 0; p < d; p++) ref[p] = dim_range[p];
    } else {
        for (int p = 0; p < d; p++) {
            double mn = q[p], mx = q[p];
            for (int t = 1; t < n; t++) {
                double v = q[(int64_t)t * d + p];
                if (v < mn) mn = v;
                if (v > mx) mx = v;
            }
            ref[p] = mx - mn;
        }
    }
    for (int64_t i = 0; i < (int64_t)G * max_boxes * d; i++) {
        out_lo[i] = OR_INF;
        out_hi[i] = -OR_INF;
    }
    for (int g = 0; g < G; g++) {
        int a = g * group_width - w;
        if (a < 0) a = 0;
        int b = g * group_width + w + group_width - 1;
        if (b > n - 1) b = n - 1;
        out_spans[2 * g] = a;
        out_spans[2 * g + 1] = b;
        out_counts[g] = or_quantize_points(q + (int64_t)a * d, b - a + 1, d, levels, max_boxes,
                                           min_cell_frac, ref, out_lo + (int64_t)g * max_boxes * d,
                                           out_hi + (int64_t)g * max_boxes * d);
    }
}

/* lb_pc, lb_pc.py:264-280 */
void or_lb_pc(const double *c, const double *box_lo, const double *box_hi, int n, int d,
              int kmax, int group_width, int has_thr, double thr, double *value, int *abandoned)
{
    double *pp = (double *)malloc(sizeof(double) * n);
    double sq[OR_MAXD];
    for (int t = 0; t < n; t++) {
        int g = t / group_width;
        const double *pt = c + (int64_t)t * d;
        double best = OR_INF;
        for (int b = 0; b < kmax; b++) {
            const double *lo = box_lo + ((int64_t)g * kmax + b) * d;
            const double *hi = box_hi + ((int64_t)g * kmax + b) * d;
            for (int p = 0; p < d; p++) {
                double dl = lo[p] - pt[p];
                double dh = pt[p] - hi[p];
                dl = dl > 0.0 ? dl : 0.0;
                dh = dh > 0.0 ? dh : 0.0;
                sq[p] = dh * dh + dl * dl;
            }
            double d2 = np_pairwise_sum(sq, d);
            if (d2 < best) best = d2;
        }
        pp[t] = sqrt(best);
    }
    sum_with_abandon(pp, n, has_thr, thr, value, abandoned);
    free(pp);
}

/* ------------------------------------------------------------------ */
/* nn_search, search.py:75-180: sequential cascade per query.          */
/* ------------------------------------------------------------------ */
enum { M_NONE = 0, M_LB_MV = 1, M_LB_TI = 2, M_LB_PC = 3, M_TC_DTW = 4, M_LB_AD = 5 };

typedef struct {
    int window;
    int method;
    int refresh_period;
    double trigger_ti;
    double trigger_pc;
    int quant_levels;
    int max_boxes;
    int group_width;
    double min_cell_frac;
} or_params_t;

typedef struct {
    int64_t best_index;
    double best_distance;
    int64_t dtw_computed, dtw_skipped, lb_mv_evals, advanced_lb_evals, abandon_count;
    int64_t dtw_cells;
    double work;
} or_outcome_t;

/* advanced: the resolved second-step bound for TC_DTW (M_LB_TI/M_LB_PC), else ignored.
 * returns 0 on success, 1 on invalid input (unresolved TC_DTW). */
int or_nn_search(const double *q, const double *cands, int64_t n_c, int n, int d,
                 const or_params_t *P, int advanced, const double *dim_range, or_outcome_t *out)
{
    int method = P->method;
    int adv = -1; /* _advanced_method, search.py:59-68 */
    if (method == M_NONE || method == M_LB_MV) adv = -1;
    else if (method == M_TC_DTW) {
        if (advanced != M_LB_TI && advanced != M_LB_PC) return 1;
        adv = advanced;
    } else
        adv = method;
    int w = P->window < n - 1 ? P->window : n - 1;
    memset(out, 0, sizeof(*out));
    double *upper = NULL, *lower = NULL, *qsteps = NULL, *blo = NULL, *bhi = NULL;
    int *bcnt = NULL, *bspans = NULL;
    int G = 0;
    if (method != M_NONE) {
        upper = (double *)malloc(sizeof(double) * n * d);
        lower = (double *)malloc(sizeof(double) * n * d);
        or_build_envelope(q, n, d, w, upper, lower);
        out->work += (double)(n * d);
    }
    if (adv == M_LB_TI) {
        qsteps = (double *)malloc(sizeof(double) * (n > 1 ? n - 1 : 1));
        or_neighbor_steps(q, n, d, qsteps);
        out->work += (double)(n * d);
    } else if (adv == M_LB_PC) {
        G = or_num_groups(n, P->group_width);
        blo = (double *)malloc(sizeof(double) * G * P->max_boxes * d);
        bhi = (double *)malloc(sizeof(double) * G * P->max_boxes * d);
        bcnt = (int *)malloc(sizeof(int) * G);
        bspans = (int *)malloc(sizeof(int) * 2 * G);
        or_build_box_sets(q, n, d, w, P->group_width, P->quant_levels, P->max_boxes,
                          P->min_cell_frac, dim_range, blo, bhi, bcnt, bspans);
        out->work += (double)(n * d * (1 + P->quant_levels));
    }
    double work_mv = (double)(n * d);
    double work_ti = n * (4.0 + (2.0 + (double)w / P->refresh_period) * d);
    double work_pc = (double)(n * P->max_boxes * d);
    double work_ad = n * (2.0 * w + 1.0) * d;
    double trig = adv == M_LB_PC ? P->trigger_pc : P->trigger_ti;

    double dist;
    int ab;
    int64_t cells;
    or_dtw_banded(q, cands, n, d, w, 0, 0.0, &dist, &ab, &cells);
    out->dtw_computed += 1;
    out->dtw_cells += cells;
    out->work += (double)(cells * d);
    double d_best = dist;
    int64_t best_idx = 0;
    int abandon = method != M_NONE;
    for (int64_t k = 1; k < n_c; k++) {
        const double *ca = cands + k * (int64_t)n * d;
        if (method != M_NONE) {
            double b1;
            int a1;
            or_lb_mv(ca, upper, lower, n, d, 1, d_best, &b1, &a1);
            out->lb_mv_evals += 1;
            out->work += work_mv;
            if (b1 >= d_best) {
                out->dtw_skipped += 1;
                continue;
            }
            if (adv >= 0 && b1 > trig * d_best) {
                double b2;
                int a2;
                if (adv == M_LB_TI) {
                    or_lb_ti(q, ca, n, d, w, TI_TIP_TOP, P->refresh_period, qsteps, 1, d_best, &b2, &a2);
                    out->work += work_ti;
                } else if (adv == M_LB_PC) {
                    or_lb_pc(ca, blo, bhi, n, d, P->max_boxes, P->group_width, 1, d_best, &b2, &a2);
                    out->work += work_pc;
                } else {
                    or_lb_ad(q, ca, n, d, w, 1, d_best, &b2, &a2);
                    out->work += work_ad;
                }
                out->advanced_lb_evals += 1;
                if (b2 >= d_best) {
                    out->dtw_skipped += 1;
                    continue;
                }
            }
        }
        or_dtw_banded(q, ca, n, d, w, abandon, d_best, &dist, &ab, &cells);
        out->dtw_computed += 1;
        out->dtw_cells += cells;
        out->work += (double)(cells * d);
        if (ab)
            out->abandon_count += 1;
        else if (dist < d_best) {
            d_best = dist;
            best_idx = k;
        }
    }
    out->best_index = best_idx;
    out->best_distance = d_best;
    free(upper);
    free(lower);
    free(qsteps);
    free(blo);
    free(bhi);
    free(bcnt);
    free(bspans);
    return 0;
}

/* Batch driver: queries (n_q, n, d) against one collection, OpenMP over
 * queries (the reference's per-query independence).  Returns
 * the number of threads used. */
int or_nn_search_batch(const double *queries, int64_t n_q, const double *cands, int64_t n_c, int n,
                       int d, const or_params_t *P, int advanced, const double *dim_range,
                       or_outcome_t *outs, int n_threads, int *status)
{
    int used = 1;
    int bad = 0;
#ifdef _OPENMP
    if (n_threads <= 0) n_threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(n_threads) reduction(| : bad)
    for (int64_t i = 0; i < n_q; i++) {
        bad |= or_nn_search(queries + i * (int64_t)n * d, cands, n_c, n, d, P, advanced, dim_range,
                            &outs[i]);
    }
    used = n_threads;
#else
    for (int64_t i = 0; i < n_q; i++)
        bad |= or_nn_search(queries + i * (int64_t)n * d, cands, n_c, n, d, P, advanced, dim_range,
                            &outs[i]);
#endif
    *status = bad;
    return used;
}

/* Exhaustive banded-DTW distance matrix rows (no abandon) for checking. */
void or_dtw_rows(const double *queries, int64_t n_q, const double *cands, int64_t n_c, int n, int d,
                 int window, double *out, int n_threads)
{
#ifdef _OPENMP
    if (n_threads <= 0) n_threads = omp_get_max_threads();
#pragma omp parallel for collapse(2) schedule(dynamic, 64) num_threads(n_threads)
#endif
    for (int64_t i = 0; i < n_q; i++)
        for (int64_t k = 0; k < n_c; k++) {
            double dist;
            int ab;
            int64_t cells;
            or_dtw_banded(queries + i * (int64_t)n * d, cands + k * (int64_t)n * d, n, d, window, 0, 0.0,
                          &dist, &ab, &cells);
            out[i * n_c + k] = dist;
        }
}
