"""Device-side normalisation and GPU report rows (f3).

normalize must equal the reference's numpy result bit for bit: values,
dim_ranges (and through them mean/std), asserted with ``array_equal``
against fixtures the reference produced (tests/golden/make_golden_ingest.py,
make_golden_ingest_fuzz.py)."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = Path(__file__).resolve().parent / "golden" / "ingest"
ARR = np.load(G / "ingest.npz")
FILES = ["native_a.txt", "native_b.txt", "ts_a.ts", "ts_b.ts"]
NORM = json.loads((G / "normalize.json").read_text())


@pytest.mark.parametrize("name", FILES)
def test_normalize_matches_reference(name):
    from paper_2101_07731_b200 import ingest

    raw = ingest.parse_native(G / name) if name.startswith("native") else ingest.parse_ts_subset(G / name)
    ds = ingest.normalize(raw)
    key = name.split(".")[0]
    assert ds.normalized
    assert np.array_equal(ds.values, ARR[f"{key}_norm"])
    assert np.array_equal(ds.dim_ranges, ARR[f"{key}_norm_ranges"])
    q, c = ingest.split(ds, 0.3, 42)
    assert np.array_equal(q.values, ARR[f"{key}_q"]) and np.array_equal(c.values, ARR[f"{key}_c"])


def _normal_raw(seed, S, n, D, spread):
    """tests/golden/make_golden_ingest_fuzz.py::normal_raw (same recipe)."""
    rng = np.random.default_rng(seed)
    v = rng.normal(size=(S, n, D)) * 10.0 ** rng.uniform(-spread, spread, size=(S, n, D)) + rng.normal(size=D) * 50
    v[rng.random(size=v.shape) < 0.01] = np.nan
    if D > 2:
        v[:, :, 1] = 3.25
    return v


@pytest.mark.parametrize("case", NORM, ids=lambda c: f"seed{c['seed']}-D{c['D']}-M{c['S'] * c['n']}")
def test_normalize_bit_exact_summation_order(case):
    """Wide dynamic range makes every summation order visible: D = 1 needs
    numpy's pairwise tree (M up to 210,000 points, depth 11), D >= 2 the
    sequential running sum; zero-variance dimensions and missing values
    included."""
    from paper_2101_07731_b200 import ingest

    raw = _normal_raw(case["seed"], case["S"], case["n"], case["D"], case["spread"])
    ds = ingest.normalize(ingest.RawDataset("x", raw, "native"))
    assert [float(x).hex() for x in ds.dim_ranges] == case["dim_ranges"]
    assert hashlib.sha256(np.ascontiguousarray(ds.values).tobytes()).hexdigest() == case["sha256"]


def test_normalize_edge_cases(rng):
    from paper_2101_07731_b200 import ingest

    # one point, one dimension
    o1, m1, s1, r1 = ingest.normalize_device(np.array([[[2.5]]]))
    assert o1.item() == 0.0 and m1.item() == 2.5 and s1.item() == 0.0 and r1.item() == 0.0
    # a non-finite input makes non-finite output, which Dataset rejects as the reference does
    bad = rng.normal(size=(4, 5, 2))
    bad[1, 2, 0] = np.inf
    with pytest.raises(ingest.InvalidInputError):
        ingest.normalize(ingest.RawDataset("x", bad, "native"))
    # many dimensions (the per-dimension apply path) against numpy
    wide = rng.normal(size=(6, 7, 300))
    ow, mw, sw, rw = ingest.normalize_device(wide)
    flat = wide.reshape(-1, 300)
    assert np.array_equal(mw.cpu().numpy(), flat.mean(axis=0)) and np.array_equal(sw.cpu().numpy(), flat.std(axis=0))
    want = (wide - flat.mean(axis=0)) / flat.std(axis=0)
    assert np.array_equal(ow.cpu().numpy(), want)
    assert np.array_equal(rw.cpu().numpy(), want.reshape(-1, 300).max(0) - want.reshape(-1, 300).min(0))


def test_report_rows_from_gpu_search():
    from oracle import oracle as O
    from paper_2101_07731_b200 import Method, SearchIndex, SearchParams, ingest, report

    ds = ingest.load(G / "native_a.txt")
    rows = report.gpu_rows(ds, ["lb_mv", "lb_pc", "tc_dtw", "none"], [2, 5], seed=3, reps=1, ideal=True)
    q, c = ingest.split(ds, 0.3, 3)
    assert len(rows) == 8
    for r in rows:
        assert r.dtw_computed + r.dtw_skipped == q.num_series * c.num_series
        assert r.dataset == "native_a" and r.dims == 3 and r.ideal_speedup is not None
    text = report.emit_report(rows, "csv", {"host": "x"})
    assert text.splitlines()[1] == ",".join(report.CSV_COLUMNS)
    assert all(r.dtw_skipped == 0 for r in rows if r.method == "none")  # the linear scan skips nothing
    # the searches behind the rows find the oracle's neighbours
    res = SearchIndex(c.values, dtype="f64").search(q.values, SearchParams(window=2, method=Method.LB_MV))
    outs, _ = O.nn_search_batch(q.values, c.values, O.make_params(2, "lb_mv"), None, ds.dim_ranges)
    assert [o.best_index for o in outs] == list(res.best_index)
