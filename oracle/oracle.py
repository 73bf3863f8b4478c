"""ctypes front-end of the C oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module, and only as the checker (or the timed CPU reference arm),
never as part of the product path.  The product package
``paper_2101_07731_b200`` does not import it.

Every function restates one reference function (file:line relative to
/root/reference/pkg/src/mvdtw) on float64 data, bit for bit; the C source is
``oracle/tcdtw_oracle.c`` and its pinning tests are
``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libtcdtw_oracle.so"
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_i64p = ctypes.POINTER(ctypes.c_int64)

METHODS = {"none": 0, "lb_mv": 1, "lb_ti": 2, "lb_pc": 3, "tc_dtw": 4, "lb_ad": 5}
TI_VARIANTS = {"basic": 0, "top": 1, "tip": 2, "tip_top": 3}


class OrParams(ctypes.Structure):
    _fields_ = [
        ("window", ctypes.c_int),
        ("method", ctypes.c_int),
        ("refresh_period", ctypes.c_int),
        ("trigger_ti", ctypes.c_double),
        ("trigger_pc", ctypes.c_double),
        ("quant_levels", ctypes.c_int),
        ("max_boxes", ctypes.c_int),
        ("group_width", ctypes.c_int),
        ("min_cell_frac", ctypes.c_double),
    ]


class OrOutcome(ctypes.Structure):
    _fields_ = [
        ("best_index", ctypes.c_int64),
        ("best_distance", ctypes.c_double),
        ("dtw_computed", ctypes.c_int64),
        ("dtw_skipped", ctypes.c_int64),
        ("lb_mv_evals", ctypes.c_int64),
        ("advanced_lb_evals", ctypes.c_int64),
        ("abandon_count", ctypes.c_int64),
        ("dtw_cells", ctypes.c_int64),
        ("work", ctypes.c_double),
    ]


def build() -> Path:
    """Compile the oracle (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        L.or_dtw_banded.argtypes = [_dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_double, _dp, _ip, _i64p]
        L.or_build_envelope.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _dp]
        L.or_lb_mv.argtypes = [_dp, _dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                               _dp, _ip]
        L.or_lb_ad.argtypes = [_dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               ctypes.c_double, _dp, _ip]
        L.or_neighbor_steps.argtypes = [_dp, ctypes.c_int, ctypes.c_int, _dp]
        L.or_ti_advance.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double, _dp, _dp]
        L.or_lb_ti.argtypes = [_dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               ctypes.c_int, _dp, ctypes.c_int, ctypes.c_double, _dp, _ip]
        L.or_quantize_points.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_double, _dp, _dp, _dp]
        L.or_quantize_points.restype = ctypes.c_int
        L.or_num_groups.argtypes = [ctypes.c_int, ctypes.c_int]
        L.or_num_groups.restype = ctypes.c_int
        L.or_build_box_sets.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_int, ctypes.c_double, _dp, _dp, _dp, _ip, _ip]
        L.or_lb_pc.argtypes = [_dp, _dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               ctypes.c_int, ctypes.c_double, _dp, _ip]
        L.or_nn_search.argtypes = [_dp, _dp, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                   ctypes.POINTER(OrParams), ctypes.c_int, _dp, ctypes.POINTER(OrOutcome)]
        L.or_nn_search.restype = ctypes.c_int
        L.or_nn_search_batch.argtypes = [_dp, ctypes.c_int64, _dp, ctypes.c_int64, ctypes.c_int,
                                         ctypes.c_int, ctypes.POINTER(OrParams), ctypes.c_int, _dp,
                                         ctypes.POINTER(OrOutcome), ctypes.c_int, _ip]
        L.or_nn_search_batch.restype = ctypes.c_int
        L.or_dtw_rows.argtypes = [_dp, ctypes.c_int64, _dp, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_int, _dp, ctypes.c_int]
        _lib = L
    return _lib


def _arr(x, ndim=2) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if ndim == 2 and a.ndim == 1:
        a = a[:, None]
    return a


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _thr(abandon_above):
    return (0, 0.0) if abandon_above is None else (1, float(abandon_above))


def dtw_banded(q, c, window, abandon_above=None):
    """dtw.py:45-102 -> (distance, abandoned, cells)."""
    qa, ca = _arr(q), _arr(c)
    n, d = qa.shape
    has, thr = _thr(abandon_above)
    dist, ab, cells = ctypes.c_double(), ctypes.c_int(), ctypes.c_int64()
    lib().or_dtw_banded(_p(qa), _p(ca), n, d, int(window), has, thr, ctypes.byref(dist),
                        ctypes.byref(ab), ctypes.byref(cells))
    return dist.value, bool(ab.value), cells.value


def build_envelope(q, window):
    """lb_mv.py:74-88 -> (upper, lower)."""
    qa = _arr(q)
    n, d = qa.shape
    up, lo = np.empty_like(qa), np.empty_like(qa)
    lib().or_build_envelope(_p(qa), n, d, int(window), _p(up), _p(lo))
    return up, lo


def lb_mv(c, upper, lower, abandon_above=None):
    """lb_mv.py:98-107 -> (value, abandoned)."""
    ca, up, lo = _arr(c), _arr(upper), _arr(lower)
    n, d = ca.shape
    has, thr = _thr(abandon_above)
    v, ab = ctypes.c_double(), ctypes.c_int()
    lib().or_lb_mv(_p(ca), _p(up), _p(lo), n, d, has, thr, ctypes.byref(v), ctypes.byref(ab))
    return v.value, bool(ab.value)


def lb_ad(q, c, window, abandon_above=None):
    """lb_mv.py:110-128 -> (value, abandoned)."""
    qa, ca = _arr(q), _arr(c)
    n, d = qa.shape
    has, thr = _thr(abandon_above)
    v, ab = ctypes.c_double(), ctypes.c_int()
    lib().or_lb_ad(_p(qa), _p(ca), n, d, int(window), has, thr, ctypes.byref(v), ctypes.byref(ab))
    return v.value, bool(ab.value)


def neighbor_steps(s):
    """lb_ti.py:51-55."""
    a = _arr(s)
    n, d = a.shape
    out = np.empty(max(n - 1, 0))
    if n > 1:
        lib().or_neighbor_steps(_p(a), n, d, _p(out))
    return out


def ti_advance(lo, up, step):
    """lb_ti.py:79-86."""
    a, b = ctypes.c_double(), ctypes.c_double()
    lib().or_ti_advance(float(lo), float(up), float(step), ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def lb_ti(q, c, window, variant="tip_top", refresh_period=5, abandon_above=None):
    """lb_ti.py:96-200 -> (value, abandoned)."""
    qa, ca = _arr(q), _arr(c)
    n, d = qa.shape
    has, thr = _thr(abandon_above)
    v, ab = ctypes.c_double(), ctypes.c_int()
    lib().or_lb_ti(_p(qa), _p(ca), n, d, int(window), TI_VARIANTS[str(variant)], int(refresh_period),
                   None, has, thr, ctypes.byref(v), ctypes.byref(ab))
    return v.value, bool(ab.value)


def quantize_cluster(points, levels, max_boxes, min_cell_frac, dim_range=None):
    """lb_pc.py:56-116 -> (los, his)."""
    pts = _arr(points)
    m, d = pts.shape
    lo = np.empty((max_boxes, d))
    hi = np.empty((max_boxes, d))
    ref = None if dim_range is None else _arr(dim_range, ndim=1)
    nb = lib().or_quantize_points(_p(pts), m, d, int(levels), int(max_boxes), float(min_cell_frac),
                                  None if ref is None else _p(ref), _p(lo), _p(hi))
    return lo[:nb].copy(), hi[:nb].copy()


def build_box_sets(q, window, group_width, levels, max_boxes, min_cell_frac, dim_range=None):
    """lb_pc.py:239-261 -> (pad_lo (G,K,D), pad_hi, counts (G,), spans [(a,b)])."""
    qa = _arr(q)
    n, d = qa.shape
    G = lib().or_num_groups(n, int(group_width))
    lo = np.empty((G, max_boxes, d))
    hi = np.empty((G, max_boxes, d))
    counts = np.empty(G, dtype=np.int32)
    spans = np.empty(2 * G, dtype=np.int32)
    ref = None if dim_range is None else _arr(dim_range, ndim=1)
    lib().or_build_box_sets(_p(qa), n, d, int(window), int(group_width), int(levels), int(max_boxes),
                            float(min_cell_frac), None if ref is None else _p(ref), _p(lo), _p(hi),
                            counts.ctypes.data_as(_ip), spans.ctypes.data_as(_ip))
    kmax = int(counts.max())
    return lo[:, :kmax].copy(), hi[:, :kmax].copy(), counts.astype(np.int64), \
        [(int(spans[2 * g]), int(spans[2 * g + 1])) for g in range(G)]


def lb_pc(c, pad_lo, pad_hi, group_width, abandon_above=None):
    """lb_pc.py:264-280 -> (value, abandoned)."""
    ca = _arr(c)
    n, d = ca.shape
    lo = np.ascontiguousarray(pad_lo, dtype=np.float64)
    hi = np.ascontiguousarray(pad_hi, dtype=np.float64)
    has, thr = _thr(abandon_above)
    v, ab = ctypes.c_double(), ctypes.c_int()
    lib().or_lb_pc(_p(ca), _p(lo), _p(hi), n, d, lo.shape[1], int(group_width), has, thr,
                   ctypes.byref(v), ctypes.byref(ab))
    return v.value, bool(ab.value)


@dataclass
class OracleOutcome:
    best_index: int
    best_distance: float
    dtw_computed: int
    dtw_skipped: int
    lb_mv_evals: int
    advanced_lb_evals: int
    abandon_count: int
    dtw_cells: int
    work: float


def make_params(window, method="lb_mv", refresh_period=5, trigger_ti=0.1, trigger_pc=0.1,
                quant_levels=2, max_boxes=6, group_width=6, min_cell_frac=1e-5) -> OrParams:
    return OrParams(int(window), METHODS[str(method)], int(refresh_period), float(trigger_ti),
                    float(trigger_pc), int(quant_levels), int(max_boxes), int(group_width),
                    float(min_cell_frac))


def nn_search_batch(queries, candidates, params: OrParams, advanced=None, dim_range=None,
                    n_threads=0):
    """search.py:75-180 applied to every query (OpenMP over queries).

    Returns (list[OracleOutcome], threads_used)."""
    Q = np.ascontiguousarray(np.asarray(queries, dtype=np.float64))
    C = np.ascontiguousarray(np.asarray(candidates, dtype=np.float64))
    if Q.ndim == 2:
        Q = Q[None]
    n_q, n, d = Q.shape
    n_c = C.shape[0]
    outs = (OrOutcome * n_q)()
    status = ctypes.c_int()
    adv = -1 if advanced is None else METHODS[str(advanced)]
    ref = None if dim_range is None else _arr(dim_range, ndim=1)
    used = lib().or_nn_search_batch(_p(Q), n_q, _p(C), n_c, n, d, ctypes.byref(params), adv,
                                    None if ref is None else _p(ref), outs, int(n_threads),
                                    ctypes.byref(status))
    if status.value:
        raise ValueError("TC_DTW must be resolved with tc_dtw_select first")
    res = [OracleOutcome(o.best_index, o.best_distance, o.dtw_computed, o.dtw_skipped, o.lb_mv_evals,
                         o.advanced_lb_evals, o.abandon_count, o.dtw_cells, o.work) for o in outs]
    return res, used


def dtw_rows(queries, candidates, window, n_threads=0) -> np.ndarray:
    """All-pairs banded DTW (no abandon): the brute-force linear-scan oracle."""
    Q = np.ascontiguousarray(np.asarray(queries, dtype=np.float64))
    C = np.ascontiguousarray(np.asarray(candidates, dtype=np.float64))
    n_q, n, d = Q.shape
    out = np.empty((n_q, C.shape[0]))
    lib().or_dtw_rows(_p(Q), n_q, _p(C), C.shape[0], n, d, int(window), _p(out), int(n_threads))
    return out


# --- the reference CLI's TC-DTW setup stage on the CPU (cli.py:228-235) ---------
# tune_params (search.py:220-272) and tc_dtw_select (search.py:198-217) with the
# reference's deterministic work model, costs from this oracle's nn_search.
TUNE_CANDIDATE_SAMPLE, TUNE_QUERY_SAMPLE = 23, 8
GRIDS = {"trigger_ti": (0.05, 0.1, 0.2), "trigger_pc": (0.1, 0.5), "quant_levels": (2, 3)}


def _draw(items, size, rng):
    """search.py:183-187: seeded subset in the original order."""
    if len(items) <= size:
        return np.asarray(items)
    keep = np.sort(rng.choice(len(items), size=size, replace=False))
    return np.asarray(items)[keep]


def _work(queries, candidates, window, method, advanced, dim_range, **knobs) -> float:
    outs, _ = nn_search_batch(queries, candidates, make_params(window, method, **knobs), advanced, dim_range)
    return float(sum(o.work for o in outs))


def resolve_tc_dtw(queries, candidates, window, dim_range=None, seed=42):
    """(trigger_ti, trigger_pc, quant_levels, advanced) as the reference CLI
    resolves method tc_dtw: the grid search on the seeded sample, then the
    cheaper of LB_TI / LB_PC (ties to LB_PC)."""
    rng = np.random.default_rng(seed)
    sq = _draw(queries, TUNE_QUERY_SAMPLE, rng)
    sc = _draw(candidates, TUNE_CANDIDATE_SAMPLE, rng)
    ti_costs = [_work(sq, sc, window, "lb_ti", None, dim_range, trigger_ti=e) for e in GRIDS["trigger_ti"]]
    e_ti = GRIDS["trigger_ti"][int(np.argmin(ti_costs))]
    pc_grid = [(e, lv) for e in GRIDS["trigger_pc"] for lv in GRIDS["quant_levels"]]
    pc_costs = [_work(sq, sc, window, "lb_pc", None, dim_range, trigger_pc=e, quant_levels=lv) for e, lv in pc_grid]
    e_pc, lv = pc_grid[int(np.argmin(pc_costs))]
    rng = np.random.default_rng(seed)
    sq = _draw(queries, TUNE_QUERY_SAMPLE, rng)
    sc = _draw(candidates, TUNE_CANDIDATE_SAMPLE, rng)
    knobs = dict(trigger_ti=e_ti, trigger_pc=e_pc, quant_levels=lv)
    cost_ti = _work(sq, sc, window, "lb_ti", None, dim_range, **knobs)
    cost_pc = _work(sq, sc, window, "lb_pc", None, dim_range, **knobs)
    return e_ti, e_pc, lv, ("lb_ti" if cost_ti < cost_pc else "lb_pc")


def threads_available() -> int:
    return os.cpu_count() or 1
