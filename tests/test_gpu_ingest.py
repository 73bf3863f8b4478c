"""Device-side normalisation and GPU report rows (f3).

normalize: the statistics are deterministic tree reductions, so they agree
with the reference's numpy sequential sums to rounding; asserted within
1e-12 of each dimension's scale (values are O(1) after normalisation)."""

import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = Path(__file__).resolve().parent / "golden" / "ingest"
ARR = np.load(G / "ingest.npz")
FILES = ["native_a.txt", "native_b.txt", "ts_a.ts", "ts_b.ts"]


@pytest.mark.parametrize("name", FILES)
def test_normalize_matches_reference(name):
    from paper_2101_07731_b200 import ingest

    raw = ingest.parse_native(G / name) if name.startswith("native") else ingest.parse_ts_subset(G / name)
    ds = ingest.normalize(raw)
    key = name.split(".")[0]
    ref, ref_rng = ARR[f"{key}_norm"], ARR[f"{key}_norm_ranges"]
    assert ds.normalized and ds.values.shape == ref.shape
    assert np.max(np.abs(ds.values - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
    assert np.allclose(ds.dim_ranges, ref_rng, rtol=1e-12, atol=1e-12)


def test_normalize_edge_cases(rng):
    from paper_2101_07731_b200 import ingest

    # zero-variance dimension -> zeros; NaN -> raw zero inside the statistics
    v = rng.normal(size=(40, 33, 3))
    v[:, :, 1] = 5.0
    v[3, 4, 2] = np.nan
    out, mean, std, rng_ = ingest.normalize_device(v)
    out = out.cpu().numpy()
    assert np.all(out[:, :, 1] == 0.0) and std.cpu().numpy()[1] == 0.0
    ref = np.where(np.isnan(v), 0.0, v)
    flat = ref.reshape(-1, 3)
    m, s = flat.mean(0), flat.std(0)
    for k in (0, 2):
        want = (ref[:, :, k] - m[k]) / s[k]
        assert np.max(np.abs(out[:, :, k] - want)) <= 1e-12
    assert np.allclose(rng_.cpu().numpy(), out.reshape(-1, 3).max(0) - out.reshape(-1, 3).min(0), rtol=0, atol=0)
    # one point, one dimension; a large collection (many blocks)
    o1, _, s1, r1 = ingest.normalize_device(np.array([[[2.5]]]))
    assert o1.item() == 0.0 and s1.item() == 0.0 and r1.item() == 0.0
    big = rng.normal(size=(5000, 64, 5)) * 3 + 1
    ob, mb, sb, _ = ingest.normalize_device(big)
    fl = big.reshape(-1, 5)
    assert np.allclose(mb.cpu().numpy(), fl.mean(0), rtol=1e-12, atol=1e-13)
    assert np.allclose(sb.cpu().numpy(), fl.std(0), rtol=1e-12)


def test_report_rows_from_gpu_search(tmp_path):
    from oracle import oracle as O
    from paper_2101_07731_b200 import ingest, report

    cfg = report.BenchConfig(data=[str(G / "native_a.txt")], methods=["lb_mv", "lb_pc", "tc_dtw", "none"],
                             windows=[2, 5], reps=1, seed=3)
    rows = report.run_benchmark(cfg)
    ds = ingest.load(G / "native_a.txt")
    q, c = ingest.split(ds, 0.3, 3)
    assert len(rows) == 8
    for r in rows:
        assert r.dtw_computed + r.dtw_skipped == q.num_series * c.num_series
        assert r.dataset == "native_a" and r.dims == 3
    text = report.emit_report(rows, "csv", {"host": "x"})
    assert text.splitlines()[1] == ",".join(report.CSV_COLUMNS)
    # the none rows are the reference's linear scan: no skips
    assert all(r.dtw_skipped == 0 for r in rows if r.method == "none")
    # and the searches behind the rows find the oracle's neighbours
    import paper_2101_07731_b200 as P

    res = P.SearchIndex(c.values, dtype="f64").search(q.values, P.SearchParams(window=2, method=P.Method.LB_MV))
    outs, _ = O.nn_search_batch(q.values, c.values, O.make_params(2, "lb_mv"), None, ds.dim_ranges)
    assert [o.best_index for o in outs] == list(res.best_index)
    assert report.main(["--data", str(G / "native_a.txt"), "--method", "lb_mv", "--window", "3", "--reps", "1",
                        "--out", str(tmp_path / "r.csv")]) == 0
    assert (tmp_path / "r.csv").read_text().count("\n") == 1 + 6 + 1 - 1 + 1  # meta(6) + header + 1 row
    assert report.main(["--data", str(G / "bad_token.txt")]) == 2
