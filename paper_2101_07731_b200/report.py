"""Benchmark report rows in the reference's schema.

The reference's benchmark layer (cli.py:36-39 CSV_COLUMNS, RunReport
cli.py:46-83, run_benchmark cli.py:165-212, _run_cell cli.py:226-271,
emit_report cli.py:294-321) reports, for every (dataset, method, window,
dims) cell, the skip rate and the speedup against the plain windowed-DTW scan
(method none).  This module produces the same rows from the GPU search --
the same columns, the same rounding, the same csv / json / table renderings
-- so GPU rows can be set next to the reference's CPU rows.  Counters come
from the GPU cascade (order-free, so skip counts may differ from the
reference's; the nearest neighbours do not), times from the batched search:
``lb_time_s`` / ``dtw_time_s`` from the CUDA-event phase times, wall time
around ``SearchIndex.search``.

Exit codes of ``main`` follow cli.py:12: 0 success, 1 configuration error,
2 data error.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time
from dataclasses import dataclass, field

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


@dataclass
class BenchConfig:
    """cli.py:86-104, GPU edition: `dtype` selects the float64 (exact) or
    float32 (filter + float64 re-score) search."""

    data: list
    fmt: str = "native"
    methods: list = field(default_factory=lambda: [Method.TC_DTW])
    windows: list = field(default_factory=lambda: [10, 20])
    dims: list = field(default_factory=lambda: ["all"])
    seed: int = 42
    reps: int = 10
    tune: bool = True
    ideal: bool = False
    emit: str = "csv"
    out: str | None = None
    query_frac: float = 0.3
    dtype: str = "f64"


@dataclass
class _Run:
    res: object
    wall_s: float


def _search(index, queries, params, advanced, dim_range, reps) -> _Run:
    walls, res = [], None
    for _ in range(max(1, reps)):
        t0 = time.perf_counter()
        res = index.search(queries, params, advanced=advanced, dim_range=dim_range, timing=True)
        walls.append(time.perf_counter() - t0)
    return _Run(res, sum(walls) / len(walls))


def _times(res):
    ph = res.phase_ms
    lb = (ph.get("prep", 0) + ph.get("lb_mv", 0) + ph.get("seeds_topk", 0) + ph.get("compact", 0)
          + ph.get("advanced", 0)) / 1e3
    dtw = (ph.get("seeds_dtw", 0) + ph.get("dtw", 0) + ph.get("finalize", 0)) / 1e3
    return lb, dtw


def run_cell(ds, queries, candidates, index, method: Method, window: int, baseline: _Run, config: BenchConfig):
    """One (dataset, method, window, dims) row (cli.py:226-271)."""
    from .search import TUNE_CANDIDATE_SAMPLE, TUNE_QUERY_SAMPLE, _sample, tc_dtw_select, tune_params

    params = SearchParams(window=window, method=method)
    advanced = None
    if method == Method.NONE:
        run = baseline
    else:
        qlist, clist = list(queries), list(candidates)
        if config.tune and method != Method.LB_MV:
            params = tune_params(qlist, clist, params, seed=config.seed, dim_range=ds.dim_ranges)
        if method == Method.TC_DTW:
            rng = np.random.default_rng(config.seed)
            sq = _sample(qlist, TUNE_QUERY_SAMPLE, rng)
            sc = _sample(clist, TUNE_CANDIDATE_SAMPLE, rng)
            advanced = tc_dtw_select(sq, sc, params, dim_range=ds.dim_ranges)
        run = _search(index, queries, params, advanced, ds.dim_ranges, config.reps)
    c = run.res.counters
    computed, skipped = int(c["dtw_computed"].sum()), int(c["dtw_skipped"].sum())
    lb_t, dtw_t = _times(run.res)
    ideal = None
    if config.ideal:
        b_lb, b_dtw = _times(baseline.res)
        ideal = (b_lb + b_dtw) / max(dtw_t, 1e-12)  # bound overhead removed (cli.py:254-259)
    label = method.value if advanced is None else f"{method.value}({advanced.value})"
    return RunReport(dataset=ds.name, method=method.value, window=window, dims=ds.dims,
                     skip_pct=100.0 * skipped / max(1, computed + skipped), speedup=baseline.wall_s / run.wall_s,
                     ideal_speedup=ideal, dtw_computed=computed, dtw_skipped=skipped, lb_time_s=lb_t,
                     dtw_time_s=dtw_t, total_time_s=run.wall_s, seed=config.seed,
                     params=describe_params(params, label), threads=1, reps=config.reps)


def run_benchmark(config: BenchConfig, datasets: list | None = None) -> list:
    """Every configured cell (cli.py:165-212).  `datasets` (already loaded
    Dataset objects) bypasses file loading."""
    from . import ingest
    from .search import SearchIndex

    if not config.data and not datasets:
        raise ConfigError("no dataset files given")
    if not config.methods:
        raise ConfigError("no methods given")
    if not config.windows:
        raise ConfigError("no window sizes given")
    if config.reps < 1:
        raise ConfigError("reps must be >= 1")
    methods = [Method(m) for m in config.methods]
    if datasets is None:
        datasets = []
        for path in config.data:
            if config.fmt not in ("native", "ts"):
                raise ConfigError(f"unknown format {config.fmt!r}")
            datasets.append(ingest.load(path, config.fmt))
    for ds in datasets:
        for spec in config.dims:
            if spec != "all" and not (1 <= int(spec) <= ds.dims):
                raise ConfigError(f"dims={spec} out of range for {ds.name} (D={ds.dims})")
    reports = []
    np_t = np.float32 if config.dtype == "f32" else np.float64
    for full in datasets:
        for spec in config.dims:
            ds = full if spec == "all" else ingest.truncate_dims(full, int(spec))
            qs, cs = ingest.split(ds, config.query_frac, config.seed)
            queries = np.ascontiguousarray(qs.values, dtype=np_t)
            candidates = np.ascontiguousarray(cs.values, dtype=np_t)
            index = SearchIndex(candidates, dtype=config.dtype)
            for window in config.windows:
                base = _search(index, queries, SearchParams(window=window, method=Method.NONE), None,
                               ds.dim_ranges, config.reps)
                for m in methods:
                    reports.append(run_cell(ds, queries, candidates, index, m, window, base, config))
    return reports


def build_parser() -> argparse.ArgumentParser:
    class _P(argparse.ArgumentParser):
        def error(self, message):  # configuration errors exit 1 (cli.py:324-326)
            raise ConfigError(message)

    p = _P(prog="tcdtw-report", description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    p.add_argument("--data", nargs="+", required=True)
    p.add_argument("--format", choices=["native", "ts"], default="native")
    p.add_argument("--method", nargs="+", default=["tc_dtw"], choices=[m.value for m in Method])
    p.add_argument("--window", nargs="+", type=int, default=[10, 20])
    p.add_argument("--dims", nargs="+", default=["all"])
    p.add_argument("--seed", type=int, default=42)
    p.add_argument("--reps", type=int, default=10)
    g = p.add_mutually_exclusive_group()
    g.add_argument("--tune", dest="tune", action="store_true", default=True)
    g.add_argument("--no-tune", dest="tune", action="store_false")
    p.add_argument("--out", default=None)
    p.add_argument("--emit", choices=["csv", "table", "json"], default="csv")
    p.add_argument("--ideal", action="store_true")
    p.add_argument("--dtype", choices=["f64", "f32"], default="f64")
    return p


def main(argv=None) -> int:
    from .ingest import ParseError

    try:
        a = build_parser().parse_args(argv)
        dims = []
        for d in a.dims:
            if d == "all":
                dims.append("all")
                continue
            try:
                dims.append(int(d))
            except ValueError:
                raise ConfigError(f'--dims expects integers or "all", got {d!r}') from None
        if any(w < 0 for w in a.window):
            raise ConfigError("--window must be >= 0")
        cfg = BenchConfig(data=a.data, fmt=a.format, methods=[Method(m) for m in a.method], windows=a.window,
                          dims=dims, seed=a.seed, reps=a.reps, tune=a.tune, ideal=a.ideal, emit=a.emit, out=a.out,
                          dtype=a.dtype)
    except ConfigError as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return 1
    for path in cfg.data:
        if not os.path.exists(path):
            print(f"config error: no such file: {path}", file=sys.stderr)
            return 1
    try:
        reports = run_benchmark(cfg)
    except ConfigError as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return 1
    except (ParseError, InvalidInputError, OSError) as exc:
        print(f"data error: {exc}", file=sys.stderr)
        return 2
    import torch

    meta = {"host": platform.node() or "unknown", "platform": platform.platform(),
            "device": torch.cuda.get_device_name(0), "reps": cfg.reps, "seed": cfg.seed, "dtype": cfg.dtype}
    text = emit_report(reports, cfg.emit, meta)
    if cfg.out:
        with open(cfg.out, "w", encoding="utf-8") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
