"""Ingest parsers and the report layer against the
reference's own outputs (tests/golden/make_golden_ingest.py).  Host logic
only -- no GPU needed."""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_2101_07731_b200 import ingest, report

G = Path(__file__).resolve().parent / "golden" / "ingest"
META = json.loads((G / "meta.json").read_text())
ARR = np.load(G / "ingest.npz")
FILES = ["native_a.txt", "native_b.txt", "ts_a.ts", "ts_b.ts"]


def _parse(name):
    return ingest.parse_native(G / name) if name.startswith("native") else ingest.parse_ts_subset(G / name)


@pytest.mark.parametrize("name", FILES)
def test_parse_matches_reference(name):
    raw = _parse(name)
    key = name.split(".")[0]
    ref = ARR[f"{key}_raw"]
    assert raw.values.shape == ref.shape
    assert np.array_equal(np.isnan(raw.values), np.isnan(ref))
    assert np.array_equal(np.nan_to_num(raw.values), np.nan_to_num(ref))
    assert raw.name == META["files"][name]["name"]
    assert raw.source_format == META["files"][name]["format"]
    fin = ingest.finalize(raw)
    assert np.array_equal(fin.values, ARR[f"{key}_fin"])
    assert np.array_equal(fin.dim_ranges, ARR[f"{key}_fin_ranges"])
    assert not fin.normalized


@pytest.mark.parametrize("name", FILES)
def test_split_matches_reference(name):
    key = name.split(".")[0]
    ds = ingest.Dataset("x", ARR[f"{key}_norm"], True, ARR[f"{key}_norm_ranges"])
    q, c = ingest.split(ds, 0.3, 42)
    assert np.array_equal(q.values, ARR[f"{key}_q"]) and np.array_equal(c.values, ARR[f"{key}_c"])


@pytest.mark.parametrize("name", sorted(META["errors"]))
def test_parse_errors_match_reference(name):
    fn = ingest.parse_native if name.endswith(".txt") else ingest.parse_ts_subset
    with pytest.raises(ingest.ParseError) as exc:
        fn(G / name)
    assert str(exc.value).replace(str(G / name), "<path>") == META["errors"][name]


FUZZ = json.loads((G / "fuzz.json").read_text())
FUZZ_ARR = np.load(G / "fuzz.npz")


@pytest.mark.parametrize("case", range(len(FUZZ)))
def test_parser_edge_cases_match_reference(case, tmp_path):
    """Lexical corners (line ends, Unicode spaces, number spellings,
    directive forms) against the reference parser's own outcome
    (tests/golden/make_golden_ingest_fuzz.py)."""
    rec = FUZZ[case]
    path = tmp_path / ("case.txt" if rec["fmt"] == "native" else "case.ts")
    path.write_text(rec["text"], encoding="utf-8", newline="")
    fn = ingest.parse_native if rec["fmt"] == "native" else ingest.parse_ts_subset
    if "error" in rec:
        kind, msg = rec["error"]
        with pytest.raises(Exception) as exc:
            fn(path)
        assert type(exc.value).__name__ == kind
        assert str(exc.value).replace(str(path), "<path>") == msg
        return
    raw = fn(path)
    want = FUZZ_ARR[f"c{case}"]
    assert raw.values.shape == tuple(rec["shape"]) and raw.source_format == rec["format"]
    assert raw.name.replace(path.stem, "<stem>") == rec["name"]
    assert np.array_equal(raw.values, want, equal_nan=True)
    assert np.array_equal(np.signbit(raw.values), np.signbit(want))  # -0.0 and -nan keep their sign


def test_parser_is_native_code():
    """The tokenizer is the library's tcdtw_parse_text, not Python."""
    import inspect

    src = inspect.getsource(ingest)
    assert "tcdtw_parse_text" in src and "float(" not in src


def test_write_native_round_trip(tmp_path):
    raw = _parse("native_b.txt")
    ds = ingest.finalize(raw)
    ingest.write_native(ds, tmp_path / "rt.txt")
    again = ingest.parse_native(tmp_path / "rt.txt")
    assert np.array_equal(again.values, ds.values)


def test_dataset_and_split_validation():
    with pytest.raises(ingest.InvalidInputError):
        ingest.Dataset("x", np.zeros((0, 3, 2)), False, np.zeros(2))
    with pytest.raises(ingest.InvalidInputError):
        ingest.Dataset("x", np.full((2, 3, 2), np.nan), False, np.zeros(2))
    ds = ingest.Dataset("x", np.zeros((3, 4, 2)), False, np.zeros(2))
    with pytest.raises(ingest.InvalidInputError):
        ingest.split(ds, 1.0)
    with pytest.raises(ingest.InvalidInputError):
        ingest.split(ds, 0.01)
    with pytest.raises(ingest.InvalidInputError):
        ingest.truncate_dims(ds, 3)
    assert ingest.truncate_dims(ds, 1).dims == 1


def _rows():
    R = report.RunReport
    return [R("synth", "lb_mv", 10, 3, 12.5, 1.75, None, 700, 100, 0.0123, 0.4567, 0.5, 42, params="lb_mv"),
            R("synth", "tc_dtw", 20, 3, 33.3333333, 2.123456789, 3.5, 400, 200, 0.25, 0.125, 0.375, 42,
              params="tc_dtw(lb_pc) e_ti=0.1 e_pc=0.1 L=2 P=5 K=6 w=6")]


@pytest.mark.parametrize("fmt", ["csv", "json", "table"])
def test_emit_report_matches_reference(fmt):
    meta = {"host": "box", "threads": 8, "reps": 1, "seed": 42}
    assert report.emit_report(_rows(), fmt, meta) == META["report"][fmt]


def test_report_schema_and_errors():
    assert report.CSV_COLUMNS == META["report_columns"]
    with pytest.raises(report.ConfigError):
        report.emit_report(_rows(), "xml")
    p = report.describe_params(report.SearchParams(window=3, method=report.Method.TC_DTW), "tc_dtw(lb_pc)")
    assert p == "tc_dtw(lb_pc) e_ti=0.1 e_pc=0.1 L=2 P=5 K=6 w=6"
