"""Bounded DTW 1-NN search (search.py:1-272), batched on the GPU.

``nn_search`` keeps the reference's signature and returns its NnOutcome;
``SearchIndex`` is the batched entry point: the candidate collection stays
resident in HBM and queries are searched in batches through the C ABI
(tcdtw_search_seed / tcdtw_search_finish).  Answers equal the reference's
linear-scan argmin with the lowest index winning ties; the counters describe
the GPU's own (order-free) cascade and may differ from the reference's.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field, replace

import numpy as np

from . import _dev, _lib
from .core import METHOD_CODE, InvalidInputError, Method, SearchParams, as_series

MAX_BATCH = 65535  # queries per search call (tcdtw_search_desc.n_queries, include/tcdtw.h)
TUNE_CANDIDATE_SAMPLE = 23
TUNE_QUERY_SAMPLE = 8


@dataclass
class NnOutcome:
    """Result and instrumentation of one query's search (search.py:37-56)."""

    best_index: int
    best_distance: float
    dtw_computed: int = 0
    dtw_skipped: int = 0
    lb_mv_evals: int = 0
    advanced_lb_evals: int = 0
    abandon_count: int = 0
    lb_time: float = 0.0
    dtw_time: float = 0.0
    total_time: float = 0.0
    work: float = 0.0


@dataclass
class BatchOutcome:
    """Per-query results of a batched search (numpy arrays)."""

    best_index: np.ndarray
    best_distance: np.ndarray
    counters: dict
    phase_ms: dict = field(default_factory=dict)
    total_ms: float = 0.0

    def outcome(self, i: int, work: float = 0.0) -> NnOutcome:
        c = self.counters
        return NnOutcome(int(self.best_index[i]), float(self.best_distance[i]), int(c["dtw_computed"][i]),
                         int(c["dtw_skipped"][i]), int(c["lb_mv_evals"][i]), int(c["advanced_lb_evals"][i]),
                         int(c["abandon_count"][i]), work=work)


_NO_SECOND_BOUND = (Method.NONE, Method.LB_MV)
_TC_DTW_CHOICES = (Method.LB_TI, Method.LB_PC)


def _advanced_method(params: SearchParams, advanced) -> Method | None:
    """The bound the cascade's second step runs, or None (search.py:59-68
    decides the same three cases: no second bound for NONE / LB_MV; TC_DTW
    takes the bound tc_dtw_select picked; any other method is its own
    second bound)."""
    m = params.method
    if m in _NO_SECOND_BOUND:
        return None
    if m != Method.TC_DTW:
        return m
    if advanced in _TC_DTW_CHOICES:
        return Method(advanced)
    raise InvalidInputError("TC_DTW must be resolved with tc_dtw_select first")


def work_model(params: SearchParams, n: int, dims: int, adv: Method | None, counters: dict, i: int) -> float:
    """The reference's deterministic work model (search.py:102-125), fed
    with this search's own counters."""
    w = params.effective_window(n)
    work = 0.0
    if params.method != Method.NONE:
        work += n * dims
    if adv == Method.LB_TI:
        work += n * dims
    elif adv == Method.LB_PC:
        work += n * dims * (1 + params.quant_levels)
    work += counters["lb_mv_evals"][i] * (n * dims)
    per_adv = {Method.LB_TI: n * (4.0 + (2.0 + w / params.refresh_period) * dims),
               Method.LB_PC: n * params.max_boxes * dims,
               Method.LB_AD: n * (2.0 * w + 1.0) * dims}
    if adv is not None:
        work += counters["advanced_lb_evals"][i] * per_adv[adv]
    work += counters["dtw_cells"][i] * dims
    return float(work)


def _stack(candidates) -> np.ndarray:
    try:
        import torch

        if isinstance(candidates, torch.Tensor):
            return candidates
    except ImportError:  # pragma: no cover
        pass
    if isinstance(candidates, np.ndarray) and candidates.ndim == 3:
        if not np.all(np.isfinite(candidates)):
            raise InvalidInputError("series contains non-finite values")
        return candidates
    cas = [as_series(c) for c in candidates]
    if not cas:
        raise InvalidInputError("candidate list is empty")
    shape = cas[0].shape
    for c in cas:
        if c.shape != shape:
            raise InvalidInputError(f"shape mismatch: {c.shape} vs {shape}")
    return np.stack(cas)


class SearchIndex:
    """A candidate collection (or one shard of it) resident on the GPU.

    dtype "f32" stores float32 and runs the float32 filter with float64
    finalist re-scoring (on the float32 values).  dtype "f64" stores float64;
    with ``f32_filter`` (the default when every value fits float32 comfortably)
    the bounds and the DTW filter still run in float32, on a rounded copy the
    library makes per call, with a slack covering the rounding, and the
    finalists are re-scored in float64 on the original values -- the answers
    and distances are the EXACT path's, bit for bit (TCDTW_FLAG_F32_FILTER);
    ``f32_filter=False`` runs every kernel in float64.  `base` is the global
    index of candidate 0 (sharding).
    """

    F32_FILTER_MAX_ABS = 1e30  # float32 copies must stay finite with room to spare

    def __init__(self, candidates, dtype=None, base: int = 0, device=None, f32_filter: bool | None = None):
        t = _dev.torch()
        arr = _stack(candidates)
        if dtype is None:
            dtype = "f32" if getattr(arr, "dtype", None) in (np.float32, t.float32) else "f64"
        self.dtype = "f32" if _lib.dtype_code(dtype) == _lib.F32 else "f64"
        self.tdtype = t.float32 if self.dtype == "f32" else t.float64
        if isinstance(arr, t.Tensor):
            dev = arr.to(device=device or "cuda", dtype=self.tdtype).contiguous()
        else:
            if arr.ndim != 3 or arr.shape[0] < 1:
                raise InvalidInputError("candidate list is empty")
            dev = t.from_numpy(np.ascontiguousarray(arr)).to(device=device or "cuda", dtype=self.tdtype)
        if dev.ndim != 3 or dev.shape[0] < 1:
            raise InvalidInputError("candidate list is empty")
        self.candidates = dev.contiguous()
        if not bool(t.isfinite(self.candidates).all()):
            raise InvalidInputError("series contains non-finite values")
        if self.dtype == "f64":
            fits = float(self.candidates.abs().max()) < self.F32_FILTER_MAX_ABS
            self.f32_filter = fits if f32_filter is None else (bool(f32_filter) and fits)
        else:
            self.f32_filter = False
        self.base = int(base)
        self.done_cap = 0  # completed-DTW list capacity (0 = library default; tests force 1)
        # thresholds frozen per DTW pass: run-to-run identical cell counts (work-model tuning)
        self.frozen_thresholds = False
        self._planar = None  # planar copy of the collection for the LB_MV pass (built on first use)
        self.cascade = True  # DTW also abandons on the LB_MV suffix (False: an A/B knob)
        self._cbox = None  # candidate box sets (f2), per parameter key
        self._csteps = None  # candidate neighbour steps (f2)
        self._reverse_pc = False  # the current search uses the reverse LB_PC (set by search())
        self._reverse_pc_range = None
        self._ws = None
        self._ws_bytes = 0
        self._cenv = None  # (window, upper, lower): candidate-side index

    @property
    def n_candidates(self) -> int:
        return int(self.candidates.shape[0])

    def candidate_envelopes(self, window: int):
        """Candidate-side index: the LB_MV envelope of
        every candidate at the effective window, built once per window by the
        streaming envelope kernel and kept resident next to the collection.
        It enables the reverse bound LB_MV(q, env(c)) (``reverse_bound=True``
        in ``search``), the reference's "switch the role" idea."""
        n = int(self.candidates.shape[1])
        w = min(int(window), n - 1)
        if w < 0:
            raise InvalidInputError("window must be >= 0")
        if self._cenv is None or self._cenv[0] != w:
            self._cenv = None
            up = _dev.empty(tuple(self.candidates.shape), self.tdtype)
            lo = _dev.empty(tuple(self.candidates.shape), self.tdtype)
            N, n, d = self.candidates.shape
            _lib.check(_lib.lib().tcdtw_build_envelope(_lib.dtype_code(self.dtype), self.candidates.data_ptr(), N, n,
                                                       d, w, up.data_ptr(), lo.data_ptr(), _lib.stream_ptr()),
                       "build_envelope")
            self._cenv = (w, up, lo)
        return self._cenv[1], self._cenv[2]

    def _planar_ptr(self, params: SearchParams, flags: int):
        """The collection in the LB_MV pass's planar layout, made once per
        index (tcdtw_planarize) instead of once per call; not for the
        float32 filter on float64 data (its rounded copy is per call)."""
        if params.method == Method.NONE or (flags & _lib.FLAG_F32_FILTER) or not _dev.torch().cuda.is_available():
            return None
        if self._planar is None:
            N, n, d = self.candidates.shape
            nbytes = _lib.lib().tcdtw_planar_bytes(_lib.dtype_code(self.dtype), N, n, d)  # elements + scale trailer
            planar = _dev.torch().empty(nbytes, dtype=_dev.torch().uint8, device=self.candidates.device)
            _lib.check(_lib.lib().tcdtw_planarize(_lib.dtype_code(self.dtype), self.candidates.data_ptr(), N, n, d,
                                                  planar.data_ptr(), _lib.stream_ptr()), "planarize")
            self._planar = planar
        return self._planar.data_ptr()

    def _filtering(self, reverse_bound: bool) -> bool:
        return self.f32_filter and not reverse_bound and not self._reverse_pc

    def work_tdtype(self, reverse_bound: bool = False):
        """Element type of d_best and dim_range: float32 under the filter."""
        t = _dev.torch()
        return t.float32 if self._filtering(reverse_bound) else self.tdtype

    def candidate_box_sets(self, params: SearchParams, dim_range=None):
        """Candidate-side index: every candidate's LB_PC
        box sets (lb_pc.py:239-261 applied to the collection), built once per
        (window, group width, levels, boxes, cell fraction, dim_range) and
        kept resident: (lo, hi, counts) with shapes (N, G, K, D) and (N, G).
        They enable the reverse LB_PC (``search(..., reverse_pc=True)``)."""
        from .lb_pc import build_box_sets_batch

        n = int(self.candidates.shape[1])
        key = (min(int(params.window), n - 1), params.group_width, params.quant_levels, params.max_boxes,
               float(params.min_cell_frac), None if dim_range is None else tuple(np.asarray(dim_range).ravel().tolist()))
        if self._cbox is None or self._cbox[0] != key:
            self._cbox = None
            lo, hi, cnt = build_box_sets_batch(self.candidates, key[0], params.group_width, params.quant_levels,
                                               params.max_boxes, params.min_cell_frac, dim_range, self.tdtype)
            self._cbox = (key, lo, hi, cnt)
        return self._cbox[1], self._cbox[2], self._cbox[3]

    def candidate_steps(self):
        """Candidate-side index (f2): every candidate's neighbour steps
        d(c_{t-1}, c_t) (lb_ti.py:51-55), shape (N, n-1), built once; the
        BASIC / TIP variants of LB_TI take them as candidate steps
        (NeighborDistances, lb_ti.py:58-76)."""
        from .lb_ti import neighbor_steps_batch

        if self._csteps is None:
            self._csteps = neighbor_steps_batch(self.candidates, self.tdtype)
        return self._csteps

    def _desc(self, params: SearchParams, adv: Method | None, n_q: int, seeds: int, timing: bool,
              phase_buf, reverse_bound: bool = False) -> _lib.SearchDesc:
        _, n, d = self.candidates.shape
        flags = _lib.FLAG_TIMING if timing else 0
        if self.frozen_thresholds:
            flags |= _lib.FLAG_FROZEN_THRESHOLDS
        if not self.cascade:
            flags |= _lib.FLAG_NO_CASCADE
        rev = reverse_bound and params.method != Method.NONE
        if self._filtering(rev):
            flags |= _lib.FLAG_F32_FILTER
        cu = cl = None
        if rev:
            cu, cl = self.candidate_envelopes(params.window)
            flags |= _lib.FLAG_REVERSE_LB
        cbl = cbh = None
        uses_pc = params.method == Method.LB_PC or (params.method == Method.TC_DTW and adv == Method.LB_PC)
        if self._reverse_pc and uses_pc:
            cbl, cbh, _ = self.candidate_box_sets(params, self._reverse_pc_range)
            flags |= _lib.FLAG_REVERSE_PC
        return _lib.SearchDesc(
            dtype=_lib.dtype_code(self.dtype), n=n, dims=d, window=int(params.window),
            method=METHOD_CODE[params.method],
            advanced=METHOD_CODE[adv] if (params.method == Method.TC_DTW and adv is not None) else 0,
            refresh_period=params.refresh_period, quant_levels=params.quant_levels,
            max_boxes=params.max_boxes, group_width=params.group_width, trigger_ti=params.trigger_ti,
            trigger_pc=params.trigger_pc, min_cell_frac=params.min_cell_frac, n_queries=n_q,
            n_candidates=self.n_candidates, candidate_base=self.base, seeds=seeds,
            flags=flags, phase_ms=ctypes.cast(phase_buf, ctypes.POINTER(ctypes.c_float)) if timing else None,
            cand_upper=_lib.ptr(cu), cand_lower=_lib.ptr(cl), done_cap=self.done_cap,
            cand_planar=self._planar_ptr(params, flags), cand_box_lo=_lib.ptr(cbl), cand_box_hi=_lib.ptr(cbh))

    def workspace_bytes(self, params: SearchParams, advanced=None, n_q: int = 1, seeds: int = 0,
                        reverse_bound: bool = False) -> int:
        adv = _advanced_method(params, advanced)
        desc = self._desc(params, adv, n_q, seeds, False, None, reverse_bound)
        out = ctypes.c_size_t()
        _lib.check(_lib.load_library().tcdtw_search_workspace_size(ctypes.byref(desc), ctypes.byref(out)),
                   "workspace_size")
        return int(out.value)

    def dtw_kernel(self, params: SearchParams, advanced=None, n_q: int = 1) -> str:
        """Name of the DTW kernel the survivors pass launches for this shape."""
        adv = _advanced_method(params, advanced)
        desc = self._desc(params, adv, n_q, 0, False, None)
        return _lib.load_library().tcdtw_dtw_kernel_name(ctypes.byref(desc)).decode()

    def auto_batch(self, params: SearchParams, advanced=None, n_q: int = 1, budget_bytes: int | None = None,
                   seeds: int = 0, reverse_bound: bool = False) -> int:
        """Largest query batch whose workspace fits the budget (default:
        half of the free device memory)."""
        t = _dev.torch()
        if budget_bytes is None:
            free, _ = t.cuda.mem_get_info()
            budget_bytes = int(free * 0.5)
        lo, hi = 1, max(1, min(int(n_q), MAX_BATCH))
        if self.workspace_bytes(params, advanced, hi, seeds, reverse_bound) <= budget_bytes:
            return hi
        while lo < hi:
            mid = (lo + hi + 1) // 2
            if self.workspace_bytes(params, advanced, mid, seeds, reverse_bound) <= budget_bytes:
                lo = mid
            else:
                hi = mid - 1
        return lo

    def _workspace(self, nbytes: int):
        t = _dev.torch()
        if self._ws is None or self._ws_bytes < nbytes:
            self._ws = None
            self._ws = t.empty(nbytes, dtype=t.uint8, device=self.candidates.device)
            self._ws_bytes = nbytes
        return self._ws

    def release(self):
        self._ws = None
        self._ws_bytes = 0
        self._cenv = None
        self._planar = None
        self._cbox = None
        self._csteps = None

    def prepare_queries(self, queries):
        t = _dev.torch()
        Q = queries if isinstance(queries, t.Tensor) else t.from_numpy(np.ascontiguousarray(
            np.asarray(queries, dtype=np.float32 if self.dtype == "f32" else np.float64)))
        if Q.ndim == 2:
            Q = Q[None]
        Q = Q.to(device=self.candidates.device, dtype=self.tdtype).contiguous()
        if Q.ndim != 3 or Q.shape[1:] != self.candidates.shape[1:]:
            raise InvalidInputError(f"shape mismatch: {tuple(Q.shape[1:])} vs {tuple(self.candidates.shape[1:])}")
        if not bool(t.isfinite(Q).all()):
            raise InvalidInputError("series contains non-finite values")
        if self.f32_filter and float(Q.abs().max()) >= self.F32_FILTER_MAX_ABS:
            self.f32_filter = False  # queries outside the float32 comfort range: exact kernels
        return Q

    def seed_phase(self, qp, params: SearchParams, advanced=None, dim_range=None, seeds: int = 0,
                   timing: bool = False, reverse_bound: bool = False) -> dict:
        """Phase 1 (tcdtw_search_seed) for one query batch already on the
        device; returns the state whose ``dbest`` a sharded caller may
        min-reduce before ``finish_phase``."""
        t = _dev.torch()
        adv = _advanced_method(params, advanced)
        phase_buf = (ctypes.c_float * len(_lib.PHASES))()
        desc = self._desc(params, adv, int(qp.shape[0]), seeds, timing, phase_buf, reverse_bound)
        nbytes = ctypes.c_size_t()
        L = _lib.lib()
        _lib.check(L.tcdtw_search_workspace_size(ctypes.byref(desc), ctypes.byref(nbytes)), "workspace_size")
        ws = self._workspace(int(nbytes.value))
        wt = self.work_tdtype(reverse_bound)
        dr = None
        if dim_range is not None:
            dr = _dev.to_dev(np.asarray(dim_range, dtype=np.float64).reshape(-1), wt)
        dbest = t.empty(int(qp.shape[0]), dtype=wt, device=qp.device)
        _lib.check(L.tcdtw_search_seed(ctypes.byref(desc), qp.data_ptr(), self.candidates.data_ptr(), _lib.ptr(dr),
                                       ws.data_ptr(), ws.numel(), dbest.data_ptr(), _lib.stream_ptr()),
                   "search_seed")
        return {"desc": desc, "ws": ws, "qp": qp, "dr": dr, "dbest": dbest, "phase_buf": phase_buf,
                "seed_ms": list(phase_buf[:4]) if timing else None}

    def finish_phase(self, state: dict, out_idx=None, out_dist=None, out_ctr=None):
        """Phase 2 (tcdtw_search_finish); returns device tensors
        (best_index, best_distance, counters)."""
        t = _dev.torch()
        qp = state["qp"]
        nq = int(qp.shape[0])
        if out_idx is None:
            out_idx = t.empty(nq, dtype=t.int64, device=qp.device)
        if out_dist is None:
            out_dist = t.empty(nq, dtype=t.float64, device=qp.device)
        if out_ctr is None:
            out_ctr = t.empty((nq, len(_lib.COUNTERS)), dtype=t.int64, device=qp.device)
        ws = state["ws"]
        _lib.check(_lib.lib().tcdtw_search_finish(
            ctypes.byref(state["desc"]), qp.data_ptr(), self.candidates.data_ptr(), _lib.ptr(state["dr"]),
            ws.data_ptr(), ws.numel(), state["dbest"].data_ptr(), out_idx.data_ptr(), out_dist.data_ptr(),
            out_ctr.data_ptr(), _lib.stream_ptr()), "search_finish")
        return out_idx, out_dist, out_ctr

    def search(self, queries, params: SearchParams, advanced=None, dim_range=None, batch: int | None = None,
               seeds: int = 0, timing: bool = False, dbest_hook=None, return_device: bool = False,
               reverse_bound: bool = False, reverse_pc: bool = False) -> BatchOutcome:
        """1-NN of every query (see _search).  reverse_pc=True (with an LB_PC
        second stage) also prunes on the reverse LB_PC against the
        candidates' own box sets (candidate_box_sets); the answers are the
        same, only the counters change."""
        self._reverse_pc, self._reverse_pc_range = bool(reverse_pc), dim_range
        try:
            return self._search(queries, params, advanced, dim_range, batch, seeds, timing, dbest_hook,
                                return_device, reverse_bound)
        finally:
            self._reverse_pc, self._reverse_pc_range = False, None

    def _search(self, queries, params: SearchParams, advanced=None, dim_range=None, batch: int | None = None,
                seeds: int = 0, timing: bool = False, dbest_hook=None, return_device: bool = False,
                reverse_bound: bool = False) -> BatchOutcome:
        """1-NN of every query.  `dbest_hook(d_best_tensor)` (optional) may
        tighten the per-query best-so-far between the two phases, e.g. an
        NCCL min-allreduce across shards.  With return_device=True the
        result arrays stay on the GPU (torch tensors).  reverse_bound=True
        also prunes on the candidate-envelope bound (candidate_envelopes);
        the answers are the same, only the counters change."""
        t = _dev.torch()
        _advanced_method(params, advanced)
        Q = self.prepare_queries(queries)
        n_q = Q.shape[0]
        if batch is None:
            batch = self.auto_batch(params, advanced, n_q, seeds=seeds, reverse_bound=reverse_bound)
        batch = max(1, min(int(batch), n_q, MAX_BATCH))
        best_idx = t.empty(n_q, dtype=t.int64, device=Q.device)
        best_dist = t.empty(n_q, dtype=t.float64, device=Q.device)
        counters = t.empty((n_q, len(_lib.COUNTERS)), dtype=t.int64, device=Q.device)
        phase_tot = np.zeros(len(_lib.PHASES))
        t_start = time.perf_counter()
        for q0 in range(0, n_q, batch):
            q1 = min(n_q, q0 + batch)
            st = self.seed_phase(Q[q0:q1], params, advanced, dim_range, seeds, timing, reverse_bound)
            if timing:
                phase_tot[:4] += np.array(st["seed_ms"])
            if dbest_hook is not None:
                dbest_hook(st["dbest"])
            self.finish_phase(st, best_idx[q0:q1], best_dist[q0:q1], counters[q0:q1])
            if timing:
                phase_tot[4:] += np.array(st["phase_buf"][4:])
        phases = dict(zip(_lib.PHASES, phase_tot.tolist()))
        if return_device:
            ctr = {k: counters[:, i] for i, k in enumerate(_lib.COUNTERS)}
            return BatchOutcome(best_idx, best_dist, ctr, phases, (time.perf_counter() - t_start) * 1e3)
        ci = counters.cpu().numpy()
        ctr = {k: ci[:, i] for i, k in enumerate(_lib.COUNTERS)}
        return BatchOutcome(best_idx.cpu().numpy(), best_dist.cpu().numpy(), ctr, phases,
                            (time.perf_counter() - t_start) * 1e3)


def nn_search_batch(queries, candidates, params: SearchParams, advanced: Method | None = None,
                    dim_range=None, dtype=None, batch: int | None = None, timing: bool = False) -> BatchOutcome:
    """Batched nn_search: every query against one collection."""
    index = SearchIndex(candidates, dtype=dtype)
    return index.search(queries, params, advanced=advanced, dim_range=dim_range, batch=batch, timing=timing)


def nn_search(query, candidates, params: SearchParams, advanced: Method | None = None,
              dim_range: np.ndarray | None = None) -> NnOutcome:
    """Nearest candidate of `query` under banded DTW (search.py:75-180),
    float64 on the GPU."""
    t0 = time.perf_counter()
    qa = as_series(query)
    arr = _stack(candidates)
    if arr.shape[0] < 1:
        raise InvalidInputError("candidate list is empty")
    if tuple(arr.shape[1:]) != qa.shape:
        raise InvalidInputError(f"shape mismatch: {qa.shape} vs {tuple(arr.shape[1:])}")
    adv = _advanced_method(params, advanced)
    res = SearchIndex(np.asarray(arr, dtype=np.float64), dtype="f64").search(
        qa[None], params, advanced=advanced, dim_range=dim_range, timing=True)
    n, dims = qa.shape
    out = res.outcome(0, work=work_model(params, n, dims, adv, res.counters, 0))
    ph = res.phase_ms
    out.dtw_time = (ph.get("seeds_dtw", 0.0) + ph.get("dtw", 0.0) + ph.get("finalize", 0.0)) / 1e3
    out.lb_time = (ph.get("prep", 0.0) + ph.get("lb_mv", 0.0) + ph.get("seeds_topk", 0.0)
                   + ph.get("compact", 0.0) + ph.get("advanced", 0.0)) / 1e3
    out.total_time = max(time.perf_counter() - t0, out.lb_time + out.dtw_time)
    return out


def _sample(items: list, size: int, rng: np.random.Generator) -> list:
    """A seeded subset of at most ``size`` items in their original order.
    The draw is ``rng.choice(len, size, replace=False)`` as in
    search.py:183-187, so the tuning sample holds the same series as the
    reference's for the same seed."""
    pool = list(items)
    if size >= len(pool):
        return pool
    keep = np.sort(rng.choice(len(pool), size=size, replace=False))
    return [pool[k] for k in keep]


def _run_sample(queries, candidates, params, advanced, dim_range, metric) -> float:
    """search.py:190-195, one batched GPU search over the sample."""
    if not queries:
        return 0.0
    adv = _advanced_method(params, advanced)
    qarr = np.stack([as_series(q) for q in queries])
    index = SearchIndex(np.asarray(_stack(candidates), dtype=np.float64), dtype="f64")
    # the work model reads DP-cell counts: freeze the thresholds per DTW pass
    # so that one seed gives the same choice and counters on every run (the
    # reference's guarantee, search.py:14-19)
    index.frozen_thresholds = metric != "time"
    res = index.search(qarr, params, advanced=advanced, dim_range=dim_range, timing=(metric == "time"))
    n, dims = qarr.shape[1:]
    if metric == "time":
        return float(sum(res.phase_ms.values())) / 1e3
    return float(sum(work_model(params, n, dims, adv, res.counters, i) for i in range(len(queries))))


def tc_dtw_select(sample_queries, sample_candidates, params: SearchParams, dim_range=None,
                  metric: str = "work") -> Method:
    """Pick the cheaper of LB_TI and LB_PC on a sample (search.py:198-217);
    ties go to LB_PC.  Costs come from the GPU search's own counters."""
    if not sample_queries or not sample_candidates:
        raise InvalidInputError("selection sample is empty")
    cost_ti = _run_sample(sample_queries, sample_candidates, replace(params, method=Method.LB_TI), None, dim_range,
                          metric)
    cost_pc = _run_sample(sample_queries, sample_candidates, replace(params, method=Method.LB_PC), None, dim_range,
                          metric)
    return Method.LB_TI if cost_ti < cost_pc else Method.LB_PC


def select_method(sample_queries, sample_candidates, params: SearchParams, dim_range=None) -> tuple:
    """GPU-cost method choice (an extension of
    tc_dtw_select): time LB_MV alone, TC-DTW with LB_TI and TC-DTW with LB_PC
    on the sample with the search's CUDA-event phase times and return the
    fastest as (params, advanced).  On the GPU the second bound often costs
    more than the DTW work it removes, a case the
    reference's two-way choice cannot express.  Ties go to the simpler
    method (LB_MV, then LB_PC)."""
    if not sample_queries or not sample_candidates:
        raise InvalidInputError("selection sample is empty")
    options = [(replace(params, method=Method.LB_MV), None),
               (replace(params, method=Method.TC_DTW), Method.LB_PC),
               (replace(params, method=Method.TC_DTW), Method.LB_TI)]
    best, best_cost = None, None
    for p, adv in options:
        cost = _run_sample(sample_queries, sample_candidates, p, adv, dim_range, "time")
        if best_cost is None or cost < best_cost:
            best, best_cost = (p, adv), cost
    return best


def _tuning_stages(params: SearchParams, grids: dict) -> list:
    """The grid searches tune_params runs for ``params.method``, as
    (bound to run, [(field overrides), ...]) in the reference's order
    (search.py:256-271): the LB_TI trigger grid for LB_TI / LB_AD / TC_DTW
    (LB_AD tunes the same trigger), then trigger x level for LB_PC / TC_DTW."""
    m = params.method
    stages = []
    ti_bound = {Method.LB_TI: Method.LB_TI, Method.LB_AD: Method.LB_AD, Method.TC_DTW: Method.LB_TI}.get(m)
    if ti_bound is not None:
        stages.append((ti_bound, [{"trigger_ti": e} for e in grids["trigger_ti"]]))
    if m in (Method.LB_PC, Method.TC_DTW):
        stages.append((Method.LB_PC, [{"trigger_pc": e, "quant_levels": lv}
                                      for e in grids["trigger_pc"] for lv in grids["quant_levels"]]))
    return stages


def tune_params(queries, candidates, params: SearchParams, grids: dict | None = None, seed: int = 0,
                dim_range=None, metric: str = "work", log: list | None = None) -> SearchParams:
    """Trigger thresholds (and quantisation level) chosen on a seeded sample
    (search.py:220-272): up to 8 queries and 23 candidates drawn as the
    reference draws them, every grid point costed by one batched GPU search
    of the sample, the first cheapest point of each grid kept.  Each
    evaluation is appended to ``log`` as (bound, params, cost)."""
    from .core import default_grids

    if params.method in _NO_SECOND_BOUND:
        return params
    grids = grids or default_grids()
    rng = np.random.default_rng(seed)
    sample_q = _sample(queries, TUNE_QUERY_SAMPLE, rng)
    sample_c = _sample(candidates, TUNE_CANDIDATE_SAMPLE, rng)
    chosen = {}
    for bound, points in _tuning_stages(params, grids):
        costs = []
        for overrides in points:
            trial = replace(params, **overrides)
            cost = _run_sample(sample_q, sample_c, replace(trial, method=bound), None, dim_range, metric)
            costs.append(cost)
            if log is not None:
                log.append((bound, trial, cost))
        chosen.update(points[int(np.argmin(costs))])  # argmin: the first minimum, as a strict-< scan
    return replace(params, **chosen)
