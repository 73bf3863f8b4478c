"""CPU-only tests: the C-ABI library loads and exports every declared symbol,
host-side validation and logic, the datasets, and the no-fallback rule."""

import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_library_exports_every_header_symbol():
    from paper_2101_07731_b200 import _lib

    L = _lib.load_library()
    header = (ROOT / "include" / "tcdtw.h").read_text()
    declared = set(re.findall(r"\b(tcdtw_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(L, name), name
    assert set(_lib.EXPORTED) == declared
    assert L.tcdtw_abi_version() == 4
    assert L.tcdtw_strerror(1) == b"invalid input"


# mvdtw.__all__ (reference pkg/src/mvdtw/__init__.py:30-38): every name a caller may import
REFERENCE_ALL = [
    "BoundResult", "BoundingBox", "BoxGrouping", "BoxSet", "Dataset", "DtwResult", "Envelope", "InvalidInputError",
    "Method", "MultivariateSeries", "NeighborDistances", "NnOutcome", "ParseError", "RawDataset", "SearchParams",
    "TiVariant", "build_box_sets", "build_envelope", "dtw_banded", "finalize", "lb_ad", "lb_mv", "lb_pc", "lb_ti",
    "neighbor_steps", "nn_search", "normalize", "parse_native", "parse_ts_subset", "point_distance",
    "quantize_cluster", "split", "tc_dtw_select", "ti_advance", "ti_extend_top", "truncate_dims", "tune_params",
    "write_native",
]


def test_package_exports_the_reference_api():
    import paper_2101_07731_b200 as P

    missing = [n for n in REFERENCE_ALL if n not in P.__all__ or not hasattr(P, n)]
    assert not missing, missing


def test_workspace_size_and_validation_without_gpu():
    import ctypes

    from paper_2101_07731_b200 import _lib

    L = _lib.load_library()
    d = _lib.SearchDesc(dtype=0, n=128, dims=6, window=12, method=1, advanced=0, refresh_period=5,
                        quant_levels=2, max_boxes=6, group_width=6, trigger_ti=0.1, trigger_pc=0.1,
                        min_cell_frac=1e-5, n_queries=64, n_candidates=10000, candidate_base=0, seeds=0, flags=0)
    out = ctypes.c_size_t()
    assert L.tcdtw_search_workspace_size(ctypes.byref(d), ctypes.byref(out)) == 0
    assert out.value > 64 * 10000 * 12  # LB matrix + survivors at least
    bad = _lib.SearchDesc.from_buffer_copy(d)
    bad.method = 4  # TC_DTW without a resolved advanced bound (search.py:64-66)
    assert L.tcdtw_search_workspace_size(ctypes.byref(bad), ctypes.byref(out)) == 1
    bad = _lib.SearchDesc.from_buffer_copy(d)
    bad.trigger_ti = 1.0
    assert L.tcdtw_search_workspace_size(ctypes.byref(bad), ctypes.byref(out)) == 1
    # per-pair entry points reject bad shapes before touching the device
    assert L.tcdtw_dtw_banded(0, None, None, 1, 0, 3, 1, None, None, None, None, None) == 1
    assert L.tcdtw_dtw_banded(0, None, None, 1, 4, 3, -1, None, None, None, None, None) == 1
    assert L.tcdtw_lb_ti(1, None, None, 1, 4, 3, 1, 3, 0, None, None, None, None, None, None) == 1
    assert L.tcdtw_build_box_sets(1, None, 1, 4, 3, 1, 0, 2, 6, 1e-5, None, None, None, None, None) == 1


def test_unsupported_dims_are_not_invalid_input():
    """a valid input beyond the kernels' dimension buckets is
    TCDTW_NOT_SUPPORTED (TcdtwError), not InvalidInputError."""
    import ctypes

    from paper_2101_07731_b200 import _lib

    L = _lib.load_library()
    d = _lib.SearchDesc(dtype=0, n=64, dims=61, window=6, method=1, advanced=0, refresh_period=5, quant_levels=2,
                        max_boxes=6, group_width=6, trigger_ti=0.1, trigger_pc=0.1, min_cell_frac=1e-5,
                        n_queries=4, n_candidates=100, candidate_base=0, seeds=0, flags=0)
    out = ctypes.c_size_t()
    assert L.tcdtw_search_workspace_size(ctypes.byref(d), ctypes.byref(out)) == _lib.TCDTW_NOT_SUPPORTED
    with pytest.raises(_lib.TcdtwError):
        _lib.check(_lib.TCDTW_NOT_SUPPORTED, "search")


def test_search_params_validation():
    from paper_2101_07731_b200 import InvalidInputError, Method, SearchParams

    with pytest.raises(InvalidInputError):
        SearchParams(window=-1)
    with pytest.raises(InvalidInputError):
        SearchParams(window=1, refresh_period=0)
    with pytest.raises(InvalidInputError):
        SearchParams(window=1, trigger_ti=0.0)
    with pytest.raises(InvalidInputError):
        SearchParams(window=1, max_boxes=0)
    with pytest.raises(InvalidInputError):
        SearchParams(window=1, min_cell_frac=0.0)
    with pytest.raises(InvalidInputError):
        SearchParams(window=1, dims_used=0)
    p = SearchParams(window=20, method="lb_pc")
    assert p.method == Method.LB_PC and p.effective_window(8) == 7


def test_host_validation_raises_before_device():
    from paper_2101_07731_b200 import InvalidInputError, as_series, dtw_banded, lb_ti, point_distance

    with pytest.raises(InvalidInputError):
        as_series(np.zeros((0, 2)))
    with pytest.raises(InvalidInputError):
        as_series([[1.0, np.nan]])
    with pytest.raises(InvalidInputError):
        dtw_banded(np.zeros((3, 2)), np.zeros((4, 2)), 1)
    with pytest.raises(InvalidInputError):
        dtw_banded(np.zeros((3, 2)), np.zeros((3, 2)), -1)
    with pytest.raises(InvalidInputError):
        lb_ti(np.zeros((6, 2)), np.zeros((6, 2)), 2, refresh_period=0)
    with pytest.raises(InvalidInputError):
        point_distance([1.0, 2.0], [1.0])


def test_advanced_method_resolution():
    from paper_2101_07731_b200 import InvalidInputError, Method, SearchParams
    from paper_2101_07731_b200.search import _advanced_method

    assert _advanced_method(SearchParams(window=1, method="lb_mv"), None) is None
    assert _advanced_method(SearchParams(window=1, method="none"), Method.LB_TI) is None
    assert _advanced_method(SearchParams(window=1, method="lb_ad"), None) == Method.LB_AD
    assert _advanced_method(SearchParams(window=1, method="tc_dtw"), Method.LB_PC) == Method.LB_PC
    with pytest.raises(InvalidInputError):
        _advanced_method(SearchParams(window=1, method="tc_dtw"), None)


def test_no_cpu_fallback(monkeypatch):
    import torch

    from paper_2101_07731_b200 import _lib, dtw_banded

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.NativeUnavailableError):
        dtw_banded(np.zeros((3, 2)), np.ones((3, 2)), 1)


def test_product_does_not_import_oracle():
    pkg = ROOT / "paper_2101_07731_b200"
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        text = f.read_text()
        assert "import oracle" not in text and "from oracle" not in text, f
        assert "tcdtw_oracle" not in text, f


def test_sample_matches_reference_rule():
    from paper_2101_07731_b200.search import _sample

    items = list(range(100))
    a = _sample(items, 8, np.random.default_rng(0))
    rng = np.random.default_rng(0)
    b = [items[i] for i in sorted(rng.choice(100, size=8, replace=False))]
    assert a == b
    assert _sample(items[:5], 8, np.random.default_rng(0)) == items[:5]


def test_work_model_matches_reference_formula():
    from paper_2101_07731_b200 import Method, SearchParams
    from paper_2101_07731_b200.search import work_model

    p = SearchParams(window=5, method="lb_ti")
    ctr = {"lb_mv_evals": [10], "advanced_lb_evals": [3], "dtw_cells": [100]}
    n, d = 24, 3
    expect = n * d + n * d + 10 * n * d + 3 * n * (4.0 + (2.0 + 5 / 5) * d) + 100 * d
    assert work_model(p, n, d, Method.LB_TI, ctr, 0) == expect


def test_cells_formula():
    # the closed form used by the kernels (k_search.cu cells_upto) against
    # the reference's row loop (dtw.py:82-96)
    def loop(r, n, w):
        return sum(min(n - 1, i + w) - max(0, i - w) + 1 for i in range(r + 1))

    def closed(r, n, w):
        a = min(n - 1 - w, r)
        s1 = (a + 1) * w + a * (a + 1) // 2 if a >= 0 else 0
        s2 = (r - a) * (n - 1)
        s3 = (r - w) * (r - w + 1) // 2 if r >= w else 0
        return (r + 1) + s1 + s2 - s3

    for n in range(1, 40):
        for w in range(0, n):
            for r in range(n):
                assert closed(r, n, w) == loop(r, n, w)


def test_datasets_deterministic_and_normalised():
    from paper_2101_07731_b200.datasets import CONFIGS, make_workload

    a = make_workload("C0")
    b = make_workload("C0")
    assert np.array_equal(a.candidates, b.candidates) and np.array_equal(a.queries, b.queries)
    assert a.candidates.shape == (200, 128, 3) and a.queries.shape == (20, 128, 3)
    allv = np.concatenate([a.candidates, a.queries]).reshape(-1, 3)
    assert np.allclose(allv.mean(0), 0, atol=1e-12) and np.allclose(allv.std(0), 1, atol=1e-12)
    s = make_workload("C4", n_candidates=2000, n_queries=50)
    assert s.candidates.dtype == np.float32 and s.candidates.shape == (2000, 128, 6)
    flat = np.concatenate([s.candidates, s.queries]).reshape(-1, 6).astype(np.float64)
    assert np.allclose(flat.mean(0), 0, atol=1e-5) and np.allclose(flat.std(0), 1, atol=1e-4)
    assert [CONFIGS[k].windows() for k in ("C0", "C1", "C2", "C3", "C4")] == [[12], [12, 51], [6], [102], [12]]


def test_shard_bounds_cover():
    from paper_2101_07731_b200.distributed import shard_bounds

    for n in (1, 7, 1000, 1000001):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


def test_new_entry_points_validate_without_gpu():
    """ABI v2 additions: the reverse-bound flag needs the candidate envelopes;
    tcdtw_normalize validates shapes and workspace before any launch."""
    import ctypes

    from paper_2101_07731_b200 import _lib

    L = _lib.load_library()
    d = _lib.SearchDesc(dtype=0, n=128, dims=6, window=12, method=1, advanced=0, refresh_period=5,
                        quant_levels=2, max_boxes=6, group_width=6, trigger_ti=0.1, trigger_pc=0.1,
                        min_cell_frac=1e-5, n_queries=64, n_candidates=10000, candidate_base=0, seeds=0,
                        flags=_lib.FLAG_REVERSE_LB)
    out = ctypes.c_size_t()
    assert L.tcdtw_search_workspace_size(ctypes.byref(d), ctypes.byref(out)) == 1  # no cand_upper/lower
    d.cand_upper, d.cand_lower = 4096, 8192  # any non-null device addresses: only sizes are computed
    assert L.tcdtw_search_workspace_size(ctypes.byref(d), ctypes.byref(out)) == 0
    with_rev = out.value
    d.flags = 0
    assert L.tcdtw_search_workspace_size(ctypes.byref(d), ctypes.byref(out)) == 0
    assert with_rev - out.value >= 64 * 10000 * 4 + 2 * 10000 * 128 * 6 * 4  # (Q,N) bound + planar envelopes
    nb = ctypes.c_size_t()
    assert L.tcdtw_normalize_workspace_size(100, 0, ctypes.byref(nb)) == 1
    assert L.tcdtw_normalize_workspace_size(0, 6, ctypes.byref(nb)) == 1
    assert L.tcdtw_normalize_workspace_size(100, 6, ctypes.byref(nb)) == 0 and nb.value > 0
    assert L.tcdtw_normalize_workspace_size(210000, 1, ctypes.byref(nb)) == 0  # + the pairwise-sum tree
    assert nb.value >= 8 * (2 << 10)
    assert L.tcdtw_normalize(None, 10, 6, None, None, None, None, None, 0, None) == 1
    assert L.tcdtw_normalize(None, 0, 6, None, None, None, None, None, 0, None) == 1


def test_dtw_kernel_choice_by_shape():
    """The lane kernel's shape coverage (host logic only: tcdtw_dtw_kernel_name
    plans the search, no launch): compiled (d, 2W+1) buckets, run-time bands
    (even W / odd W at 4 rows per step, 2 rows for n % 4 != 0 or d > 8),
    dimension padding, and the shapes left to the other kernels."""
    import ctypes

    from paper_2101_07731_b200 import _lib

    L = _lib.load_library()

    def name(n, d, w, dtype=0, flags=0):
        desc = _lib.SearchDesc(dtype=dtype, n=n, dims=d, window=w, method=1, advanced=0, refresh_period=5,
                               quant_levels=2, max_boxes=6, group_width=6, trigger_ti=0.1, trigger_pc=0.1,
                               min_cell_frac=1e-5, n_queries=64, n_candidates=10000, candidate_base=0, seeds=0,
                               flags=flags)
        return L.tcdtw_dtw_kernel_name(ctypes.byref(desc)).decode()

    four, two = "dtw_laner_kernel<R=4>", "dtw_laner_kernel<R=2>"
    assert name(128, 6, 12) == four  # C4: compiled bucket
    assert name(64, 20, 6) == two  # C2: compiled bucket
    assert name(256, 5, 51) == four  # C1b: compiled bucket
    for w in (4, 10, 11, 16, 25):  # run-time band, even and odd W
        assert name(128, 6, w) == four, w
    assert name(126, 6, 12) == four and name(127, 6, 12) == four  # n % 4 != 0: tail rows
    assert name(63, 20, 6) == two and name(3, 6, 12) not in (four, two)  # n >= 2 x rows per step
    for d in (1, 2, 7):  # padded to 3 / 3 / 8 dimensions
        assert name(128, d, 12) == four, d
    for d in (9, 12, 13, 16, 19):  # padded to 12 / 16 / 20 dimensions at 2 rows per step
        assert name(128, d, 12) == two, d
    assert name(128, 6, 3) == two and name(128, 6, 1) not in (four, two)  # W >= rows per step
    assert name(128, 24, 12) not in (four, two)  # d > 20
    assert name(1024, 8, 102) not in (four, two)  # C3's band row does not fit three blocks per SM
    assert name(128, 6, 12, dtype=1) not in (four, two)  # float64 without the filter: exact kernels
    assert name(128, 6, 12, dtype=1, flags=_lib.FLAG_F32_FILTER) == four
