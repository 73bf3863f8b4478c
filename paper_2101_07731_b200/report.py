"""Benchmark report rows in the reference's schema.

The reference reports, per (dataset, method, window, dims) cell, the skip
rate and the speedup against the plain windowed-DTW scan (method none), in
one schema (cli.py:36-39 CSV_COLUMNS, RunReport cli.py:46-83, emit_report
cli.py:294-321).  This module keeps that schema -- columns, rounding and the
csv / json / table renderings are byte-identical -- and fills rows from the
GPU search (``gpu_rows``), so GPU rows can sit next to the reference's CPU
rows.  Counters come from the GPU cascade (order-free, so skip counts may
differ from the reference's; the nearest neighbours do not); ``lb_time_s`` /
``dtw_time_s`` are CUDA-event phase times, ``total_time_s`` the wall time of
``SearchIndex.search``.  The reference's command-line driver itself is out of
scope.
"""

from __future__ import annotations

import json
import time
from dataclasses import dataclass

import numpy as np

from .core import InvalidInputError, Method, SearchParams

CSV_COLUMNS = ["dataset", "method", "window", "dims", "skip_pct", "speedup", "ideal_speedup", "dtw_computed",
               "dtw_skipped", "lb_time_s", "dtw_time_s", "total_time_s", "seed"]

_ROUND = {"skip_pct": 4, "speedup": 4, "ideal_speedup": 4, "lb_time_s": 6, "dtw_time_s": 6, "total_time_s": 6}


class ConfigError(ValueError):
    """The benchmark configuration is invalid (cli.py:42-43)."""


@dataclass
class RunReport:
    """One result row (cli.py:46-83)."""

    dataset: str
    method: str
    window: int
    dims: int
    skip_pct: float
    speedup: float
    ideal_speedup: float | None
    dtw_computed: int
    dtw_skipped: int
    lb_time_s: float
    dtw_time_s: float
    total_time_s: float
    seed: int
    params: str = ""
    threads: int = 1
    reps: int = 1

    def row(self) -> dict:
        out = {}
        for col in CSV_COLUMNS:
            v = getattr(self, col)
            if col in _ROUND and v is not None:
                v = round(float(v), _ROUND[col])
            out[col] = v
        return out


def _cell(v) -> str:
    """Cell text (cli.py:284-291): '' for None / NaN, floats with six
    decimals and trailing zeros dropped."""
    if v is None:
        return ""
    if isinstance(v, float):
        if v != v:
            return ""
        txt = f"{v:.6f}"
        return txt.rstrip("0").rstrip(".")
    return str(v)


def emit_report(reports: list, fmt: str = "csv", meta: dict | None = None) -> str:
    """csv / json / table renderings, identical to the reference's
    (cli.py:294-321)."""
    meta = dict(meta or {})
    rows = [r.row() for r in reports]
    if fmt == "csv":
        out = [f"# {k}: {v}" for k, v in meta.items()]
        out.append(",".join(CSV_COLUMNS))
        out += [",".join(_cell(r[c]) for c in CSV_COLUMNS) for r in rows]
        return "\n".join(out) + "\n"
    if fmt == "json":
        return json.dumps({"meta": meta, "rows": rows}, indent=2) + "\n"
    if fmt == "table":
        head = CSV_COLUMNS + ["params"]
        body = [[_cell(r[c]) for c in CSV_COLUMNS] + [rep.params] for r, rep in zip(rows, reports)]
        width = [max([len(h)] + [len(b[i]) for b in body]) for i, h in enumerate(head)]
        out = ["  ".join(h.ljust(width[i]) for i, h in enumerate(head)),
               "  ".join("-" * w for w in width)]
        out += ["  ".join(b[i].ljust(width[i]) for i in range(len(head))) for b in body]
        if meta:
            out.append("")
            out += [f"{k}: {v}" for k, v in meta.items()]
        return "\n".join(out) + "\n"
    raise ConfigError(f"unknown report format {fmt!r}")


def describe_params(params: SearchParams, label: str) -> str:
    """The table's params column (cli.py:274-281)."""
    m = params.method
    if m in (Method.NONE, Method.LB_MV):
        return label
    bits = [label]
    if m in (Method.LB_TI, Method.LB_AD, Method.TC_DTW):
        bits.append(f"e_ti={params.trigger_ti}")
    if m in (Method.LB_PC, Method.TC_DTW):
        bits.append(f"e_pc={params.trigger_pc} L={params.quant_levels}")
    bits.append(f"P={params.refresh_period} K={params.max_boxes} w={params.group_width}")
    return " ".join(bits)


def _timed_search(index, queries, params, advanced, dim_range, reps):
    """(last result, mean wall seconds) over ``reps`` searches."""
    res, total = None, 0.0
    for _ in range(max(1, int(reps))):
        t0 = time.perf_counter()
        res = index.search(queries, params, advanced=advanced, dim_range=dim_range, timing=True)
        total += time.perf_counter() - t0
    return res, total / max(1, int(reps))


def _phase_seconds(res):
    """(bound time, DTW time) in seconds from the CUDA-event phases."""
    ph = res.phase_ms
    dtw_ms = sum(ph.get(k, 0.0) for k in ("seeds_dtw", "dtw", "finalize"))
    return (sum(ph.values()) - dtw_ms) / 1e3, dtw_ms / 1e3


def _resolve(method: Method, window: int, queries, candidates, dim_range, seed: int, tune: bool):
    """Params and TC-DTW bound for one cell, chosen on the seeded sample the
    reference CLI uses (cli.py:228-235): tune_params, then tc_dtw_select."""
    from .search import TUNE_CANDIDATE_SAMPLE, TUNE_QUERY_SAMPLE, _sample, tc_dtw_select, tune_params

    params = SearchParams(window=window, method=method)
    if method in (Method.NONE, Method.LB_MV):
        return params, None
    if tune:
        params = tune_params(list(queries), list(candidates), params, seed=seed, dim_range=dim_range)
    if method != Method.TC_DTW:
        return params, None
    rng = np.random.default_rng(seed)
    sq = _sample(list(queries), TUNE_QUERY_SAMPLE, rng)
    sc = _sample(list(candidates), TUNE_CANDIDATE_SAMPLE, rng)
    return params, tc_dtw_select(sq, sc, params, dim_range=dim_range)


def gpu_rows(ds, methods=(Method.TC_DTW,), windows=(10, 20), *, seed: int = 42, reps: int = 1, tune: bool = True,
             ideal: bool = False, query_frac: float = 0.3, dtype: str = "f64") -> list:
    """Report rows of one loaded ``ingest.Dataset`` from the GPU search: the
    reference's seeded query/candidate split, a NONE scan per window as the
    speedup baseline, then every method (f3)."""
    from .ingest import split
    from .search import SearchIndex

    np_t = np.float32 if dtype == "f32" else np.float64
    qs, cs = split(ds, query_frac, seed)
    queries = np.ascontiguousarray(qs.values, dtype=np_t)
    candidates = np.ascontiguousarray(cs.values, dtype=np_t)
    index = SearchIndex(candidates, dtype=dtype)
    rows = []
    for window in windows:
        base_res, base_wall = _timed_search(index, queries, SearchParams(window=window, method=Method.NONE), None,
                                            ds.dim_ranges, reps)
        for m in map(Method, methods):
            if m == Method.NONE:
                res, wall, params, adv = base_res, base_wall, SearchParams(window=window, method=m), None
            else:
                params, adv = _resolve(m, window, queries, candidates, ds.dim_ranges, seed, tune)
                res, wall = _timed_search(index, queries, params, adv, ds.dim_ranges, reps)
            computed = int(res.counters["dtw_computed"].sum())
            skipped = int(res.counters["dtw_skipped"].sum())
            lb_s, dtw_s = _phase_seconds(res)
            ideal_x = sum(_phase_seconds(base_res)) / max(dtw_s, 1e-12) if ideal else None  # cli.py:254-259
            label = m.value if adv is None else f"{m.value}({Method(adv).value})"
            rows.append(RunReport(ds.name, m.value, window, ds.dims, 100.0 * skipped / max(1, computed + skipped),
                                  base_wall / wall, ideal_x, computed, skipped, lb_s, dtw_s, wall, seed,
                                  params=describe_params(params, label), reps=reps))
    return rows
