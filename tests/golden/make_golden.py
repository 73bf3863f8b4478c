"""Generate golden input/output vectors from the REFERENCE implementation.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports the unmodified reference package ``mvdtw`` read-only, runs its
public functions on seeded inputs and writes compressed fixtures next to this
script.  The fixtures pin the C oracle (tests/test_oracle_golden.py) and are
the known-answer cases of the GPU parity tests.  Nothing at run time on the
GPU box reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import mvdtw  # noqa: E402
from mvdtw import (  # noqa: E402
    Method, SearchParams, TiVariant, build_box_sets, build_envelope, dtw_banded, lb_ad, lb_mv,
    lb_pc, lb_ti, neighbor_steps, nn_search, quantize_cluster, ti_advance,
)
from mvdtw.synth import random_walk_dataset  # noqa: E402

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
from paper_2101_07731_b200.datasets import make_workload  # noqa: E402


def instance(rng, max_n=64, max_dims=10, max_window=20):
    """Seeded (q, c, window) draw over four families: random walk, iid
    noise, shifted near-copy, plateaus of repeated points (the same regimes
    the reference's soundness tests draw, tests/conftest.py:15-41)."""
    n = int(rng.integers(1, max_n + 1))
    dims = int(rng.integers(1, max_dims + 1))
    window = int(rng.integers(0, max_window + 1))
    kind = rng.random()
    if kind < 0.4:
        q = np.cumsum(rng.normal(0, 1, (n, dims)), axis=0)
        c = np.cumsum(rng.normal(0, 1, (n, dims)), axis=0)
    elif kind < 0.75:
        q = rng.normal(0, 1, (n, dims))
        c = rng.normal(0, 1, (n, dims))
    elif kind < 0.88:
        q = np.cumsum(rng.normal(0, 1, (n, dims)), axis=0)
        c = np.roll(q + rng.normal(0, 1e-3, (n, dims)), int(rng.integers(0, 3)), axis=0)
    else:
        k = max(1, n // 3)
        q = np.repeat(rng.normal(0, 1, (k, dims)), 3, axis=0)[:n]
        c = np.repeat(rng.normal(0, 1, (k, dims)), 3, axis=0)[:n]
        if len(q) < n:
            q = np.vstack([q, q[-1:].repeat(n - len(q), 0)])
            c = np.vstack([c, c[-1:].repeat(n - len(c), 0)])
    return np.ascontiguousarray(q), np.ascontiguousarray(c), window


def pack(cases: list[dict]) -> dict:
    """Arrays become npz members; scalars go into one JSON blob (Python's
    float repr round-trips exactly)."""
    out = {"n_cases": np.array(len(cases))}
    scalars = []
    for i, case in enumerate(cases):
        sc = {}
        for k, v in case.items():
            a = np.asarray(v)
            if a.ndim == 0:
                sc[k] = a.item()
            else:
                out[f"c{i}_{k}"] = a
        scalars.append(sc)
    out["scalars"] = np.array(json.dumps(scalars))
    return out


def save(name: str, cases: list[dict]):
    path = HERE / f"{name}.npz"
    np.savez_compressed(path, **pack(cases))
    print(f"  {name}: {len(cases)} cases, {path.stat().st_size / 1024:.1f} KiB")


def thresholds(full: float):
    return [None, full, full * 0.999, full * 0.5]


def gen_dtw(rng):
    cases = []
    for i in range(260):
        q, c, w = instance(rng, max_dims=12 if i % 5 else 24)
        full = dtw_banded(q, c, w)
        case = {"q": q, "c": c, "w": w}
        for j, thr in enumerate(thresholds(full.distance)):
            r = dtw_banded(q, c, w, abandon_above=thr)
            case[f"thr{j}"] = np.nan if thr is None else thr
            case[f"dist{j}"] = r.distance
            case[f"ab{j}"] = r.abandoned
            case[f"cells{j}"] = r.cells
        cases.append(case)
    # hand examples (test_dtw.py:17-23)
    for q, c, w in (([[0.0], [0.0]], [[1.0], [1.0]], 1),
                    ([[0.0, 0.0], [3.0, 4.0]], [[0.0, 0.0], [0.0, 0.0]], 1)):
        r = dtw_banded(q, c, w)
        cases.append({"q": np.array(q), "c": np.array(c), "w": w, "thr0": np.nan,
                      "dist0": r.distance, "ab0": r.abandoned, "cells0": r.cells})
    save("dtw", cases)


def gen_envelope(rng):
    cases = []
    for _ in range(80):
        n = int(rng.integers(1, 70))
        d = int(rng.integers(1, 9))
        w = int(rng.integers(0, 20))
        q = rng.normal(size=(n, d)) if rng.random() < 0.5 else np.cumsum(rng.normal(size=(n, d)), 0)
        env = build_envelope(q, w)
        cases.append({"q": q, "w": w, "upper": env.upper, "lower": env.lower, "weff": env.window})
    env = build_envelope([[1.0], [2.0], [3.0]], 1)
    cases.append({"q": np.array([[1.0], [2.0], [3.0]]), "w": 1, "upper": env.upper, "lower": env.lower,
                  "weff": env.window})
    save("envelope", cases)


def gen_lb_mv_ad(rng):
    cases = []
    for i in range(150):
        q, c, w = instance(rng, max_n=48, max_dims=12 if i % 4 else 22, max_window=12)
        if i % 3 == 0:
            c = c + rng.normal(0, 2.0)
        env = build_envelope(q, w)
        case = {"q": q, "c": c, "w": w}
        mv_full = lb_mv(c, env).value
        ad_full = lb_ad(q, c, w).value
        for j, thr in enumerate([None, mv_full / 2.0, mv_full]):
            r = lb_mv(c, env, abandon_above=thr)
            case[f"mv_thr{j}"] = np.nan if thr is None else thr
            case[f"mv{j}"] = r.value
            case[f"mv_ab{j}"] = r.abandoned
        for j, thr in enumerate([None, ad_full / 2.0, ad_full]):
            r = lb_ad(q, c, w, abandon_above=thr)
            case[f"ad_thr{j}"] = np.nan if thr is None else thr
            case[f"ad{j}"] = r.value
            case[f"ad_ab{j}"] = r.abandoned
        case["steps_q"] = neighbor_steps(q) if len(q) > 1 else np.zeros(0)
        cases.append(case)
    save("lb_mv_ad", cases)


def gen_ti(rng):
    adv = []
    for lo, up, s in ((2.5, 4.0, 0.0), (5.0, 7.0, 2.0), (1.0, 2.0, 10.0), (1.0, 5.0, 2.0), (3.0, 6.0, 0.0),
                      (4.0, 6.0, 1.0)):
        adv.append((lo, up, s, *ti_advance(lo, up, s)))
    for _ in range(400):
        lo = abs(rng.normal()) * 10 ** rng.uniform(-3, 3)
        up = lo + abs(rng.normal()) * 10 ** rng.uniform(-3, 3)
        s = 0.0 if rng.random() < 0.1 else abs(rng.normal()) * 10 ** rng.uniform(-3, 3)
        adv.append((lo, up, s, *ti_advance(lo, up, s)))
    cases = [{"adv": np.array(adv)}]
    for i in range(90):
        q, c, w = instance(rng, max_n=40, max_dims=10 if i % 4 else 20, max_window=10)
        n = len(q)
        case = {"q": q, "c": c, "w": w}
        k = 0
        for variant in TiVariant:
            for period in sorted({1, 2, 3, 5, n}):
                full = lb_ti(q, c, w, variant, period).value
                for thr in (None, full / 2.0):
                    r = lb_ti(q, c, w, variant, period, abandon_above=thr)
                    case[f"v{k}_variant"] = list(TiVariant).index(variant)
                    case[f"v{k}_period"] = period
                    case[f"v{k}_thr"] = np.nan if thr is None else thr
                    case[f"v{k}_val"] = r.value
                    case[f"v{k}_ab"] = r.abandoned
                    k += 1
        case["nv"] = k
        cases.append(case)
    save("lb_ti", cases)


def gen_pc(rng):
    qc = []
    examples = [
        (np.array([[0.0], [0.1], [0.9], [1.0]]), 2, 6, 1e-5, None),
        (np.array([[0.0], [0.2], [0.4], [0.6], [0.8], [1.0]]), 6, 2, 1e-5, None),
        (np.array([[0.0, 0.0], [1.0, 1e-9], [2.0, 2e-9]]), 3, 9, 1e-5, np.array([2.0, 2.0])),
        (np.full((5, 2), 3.25), 4, 6, 1e-5, None),
    ]
    for _ in range(120):
        m = int(rng.integers(1, 40))
        d = int(rng.integers(1, 7)) if rng.random() < 0.8 else int(rng.integers(8, 22))
        pts = rng.normal(size=(m, d)) * rng.choice([0.01, 1.0, 100.0])
        if rng.random() < 0.2:
            pts[:, 0] = pts[0, 0]
        levels = int(rng.integers(1, 5))
        cap = int(rng.integers(1, 8))
        dr = None if rng.random() < 0.5 else np.abs(rng.normal(size=d)) * 3
        examples.append((pts, levels, cap, 1e-5 if rng.random() < 0.8 else 0.3, dr))
    for pts, levels, cap, mcf, dr in examples:
        bs = quantize_cluster(pts, levels, cap, mcf, dim_range=dr)
        qc.append({"pts": pts, "levels": levels, "cap": cap, "mcf": mcf,
                   "dr": np.full(pts.shape[1], np.nan) if dr is None else dr,
                   "los": bs.los, "his": bs.his})
    save("quantize", qc)

    cases = []
    for i in range(120):
        q, c, w = instance(rng, max_n=48, max_dims=8 if i % 4 else 20, max_window=10)
        n, d = q.shape
        gw = int(rng.choice([1, 2, 3, 6]))
        levels = int(rng.choice([1, 2, 3]))
        cap = int(rng.choice([1, 2, 4, 6]))
        dr = None if i % 2 else np.abs(rng.normal(size=d)) * 4 + 0.1
        g = build_box_sets(q, w, gw, levels, cap, 1e-5, dim_range=dr)
        case = {"q": q, "c": c, "w": w, "gw": gw, "levels": levels, "cap": cap,
                "dr": np.full(d, np.nan) if dr is None else dr,
                "pad_lo": g.pad_lo, "pad_hi": g.pad_hi, "counts": g.box_counts,
                "spans": np.array(g.spans)}
        full = lb_pc(c, g).value
        for j, thr in enumerate([None, full / 2.0, full]):
            r = lb_pc(c, g, abandon_above=thr)
            case[f"thr{j}"] = np.nan if thr is None else thr
            case[f"val{j}"] = r.value
            case[f"ab{j}"] = r.abandoned
        cases.append(case)
    save("box_sets", cases)


OUTCOME_FIELDS = ("best_index", "best_distance", "dtw_computed", "dtw_skipped", "lb_mv_evals",
                  "advanced_lb_evals", "abandon_count", "work")

METHOD_RUNS = [("none", None), ("lb_mv", None), ("lb_ti", None), ("lb_pc", None), ("lb_ad", None),
               ("tc_dtw", "lb_ti"), ("tc_dtw", "lb_pc")]


def run_methods(q, cands, w, dim_range=None, runs=METHOD_RUNS, **kw):
    out = {}
    for k, (method, adv) in enumerate(runs):
        params = SearchParams(window=w, method=Method(method), **kw)
        o = nn_search(q, cands, params, advanced=None if adv is None else Method(adv), dim_range=dim_range)
        for f in OUTCOME_FIELDS:
            out[f"m{k}_{f}"] = getattr(o, f)
    return out


def gen_search(rng):
    cases = []
    for seed, window, n_series, n, dims in ((1, 5, 26, 24, 3), (3, 5, 26, 24, 3), (6, 0, 26, 24, 3),
                                             (11, 4, 30, 24, 3), (23, 3, 40, 20, 2), (31, 6, 36, 30, 12)):
        ds = random_walk_dataset(n_series, n, dims, seed=seed)
        series = ds.values
        q, cands = series[0], series[1:]
        case = {"q": q, "cands": cands, "w": window, "dr": ds.dim_ranges}
        case.update(run_methods(q, list(cands), window, dim_range=ds.dim_ranges))
        cases.append(case)
    # trigger-band scenario (test_search.py:103-119)
    q = np.zeros((4, 1))
    cands = np.stack([np.ones((4, 1)), np.full((4, 1), 10.0), np.array([[1.0], [1.0], [0.0], [0.0]]),
                      np.array([[0.0], [0.0], [0.0], [0.1]])])
    case = {"q": q, "cands": cands, "w": 1, "dr": np.full(1, np.nan)}
    case.update(run_methods(q, list(cands), 1, runs=[("lb_ti", None)]))
    cases.append(case)
    # duplicated candidates / exact ties: lowest index must win
    base = np.cumsum(rng.normal(size=(30, 16, 2)), axis=1)
    cands = np.concatenate([base[1:], base[1:6], base[1:6]])
    q = base[0]
    case = {"q": q, "cands": cands, "w": 3, "dr": np.full(2, np.nan)}
    case.update(run_methods(q, list(cands), 3))
    cases.append(case)
    save("search_small", cases)


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def gen_configs():
    """Config-level NN results of the reference on sampled queries of the
    seeded workloads (inputs are regenerated from the seed; the digest pins
    the generator)."""
    cases = []
    plan = [  # (config, window index, query ids, runs)
        ("C0", 0, list(range(20)), METHOD_RUNS),
        ("C1", 0, [0, 1, 2, 3], [("lb_mv", None), ("lb_pc", None)]),
        ("C1", 1, [0, 1], [("lb_mv", None)]),
        ("C2", 0, [0, 1], [("lb_mv", None)]),
        ("C3", 0, [0], [("lb_mv", None)]),
    ]
    for cfg, wi, qids, runs in plan:
        t0 = time.time()
        wl = make_workload(cfg, seed=0)
        w = wl.spec.windows()[wi]
        cands64 = wl.candidates.astype(np.float64)
        cand_list = list(cands64)
        for qi in qids:
            q = wl.queries[qi].astype(np.float64)
            case = {"cfg": cfg, "w": w, "qi": qi, "digest_c": digest(wl.candidates),
                    "digest_q": digest(wl.queries), "dr": wl.dim_range}
            case.update(run_methods(q, cand_list, w, dim_range=wl.dim_range, runs=runs))
            case["runs"] = np.array([f"{m}:{a}" for m, a in runs])
            cases.append(case)
        print(f"    {cfg} W={w}: {len(qids)} queries in {time.time() - t0:.1f}s")
    save("configs", cases)


def main():
    rng = np.random.default_rng(20240817)
    print(f"reference mvdtw from {mvdtw.__file__}")
    gen_dtw(rng)
    gen_envelope(rng)
    gen_lb_mv_ad(rng)
    gen_ti(rng)
    gen_pc(rng)
    gen_search(rng)
    if "--no-configs" not in sys.argv:
        gen_configs()


if __name__ == "__main__":
    main()
