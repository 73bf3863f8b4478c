"""The reference-side binding and the CPU
baseline's TC-DTW setup, against the unmodified reference package.

These run in the build container, where /root/reference is importable; they
skip elsewhere (the GPU box has no reference).  No GPU: the GPU nn_search is
replaced by a stub that records what the shim passed to it."""

import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.is_dir(), reason="reference package not present")


@pytest.fixture(scope="module")
def mvdtw():
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import mvdtw
    import mvdtw.cli
    import mvdtw.search

    saved = (mvdtw.search.nn_search, mvdtw.cli.nn_search)
    yield mvdtw
    mvdtw.search.nn_search, mvdtw.cli.nn_search = saved


def test_shim_translates_arguments_and_outcome(mvdtw):
    import paper_2101_07731_b200 as P
    from paper_2101_07731_b200 import integration

    calls = []

    def stub(query, candidates, params, advanced=None, dim_range=None):
        calls.append((query, candidates, params, advanced, dim_range))
        return P.NnOutcome(best_index=3, best_distance=1.5, dtw_computed=7, dtw_skipped=2, lb_mv_evals=9,
                           advanced_lb_evals=4, abandon_count=5, lb_time=0.1, dtw_time=0.2, total_time=0.4,
                           work=123.0)

    fn = integration.patch_mvdtw(mvdtw.search, mvdtw.cli, impl=stub)
    assert mvdtw.search.nn_search is fn and mvdtw.cli.nn_search is fn
    ref_params = mvdtw.SearchParams(window=7, method=mvdtw.Method.TC_DTW, refresh_period=3, trigger_ti=0.2,
                                    trigger_pc=0.5, quant_levels=3, max_boxes=4, group_width=5,
                                    min_cell_frac=2e-5)
    q = np.zeros((10, 2))
    cands = [np.ones((10, 2))] * 4
    dr = np.array([1.0, 2.0])
    out = mvdtw.search.nn_search(q, cands, ref_params, advanced=mvdtw.Method.LB_PC, dim_range=dr)
    assert type(out) is mvdtw.search.NnOutcome
    assert (out.best_index, out.best_distance, out.dtw_computed, out.dtw_skipped, out.work) == (3, 1.5, 7, 2, 123.0)
    (_, _, params, adv, dr_seen), = calls
    assert isinstance(params, P.SearchParams) and params.method == P.Method.TC_DTW
    for f in ("window", "refresh_period", "trigger_ti", "trigger_pc", "quant_levels", "max_boxes", "group_width",
              "min_cell_frac", "dims_used"):
        assert getattr(params, f) == getattr(ref_params, f), f
    assert adv == P.Method.LB_PC and dr_seen is dr
    # the reference's own callers go through the patch: its sample runner
    # (search.py:190-195) and tc_dtw_select
    calls.clear()
    choice = mvdtw.search.tc_dtw_select([q], cands, mvdtw.SearchParams(window=2), dim_range=dr)
    assert choice in (mvdtw.Method.LB_TI, mvdtw.Method.LB_PC)
    assert [c[2].method for c in calls] == [P.Method.LB_TI, P.Method.LB_PC]
    # invalid parameters still raise the reference's InvalidInputError family (a ValueError)
    with pytest.raises(ValueError):
        integration.translate_params(type("X", (), {"window": -1, "method": mvdtw.Method.LB_MV})())


def test_cpu_baseline_tc_dtw_setup_matches_reference(mvdtw):
    """oracle.resolve_tc_dtw (the CPU baseline's copy of the reference CLI's
    setup, cli.py:228-235) picks what the reference picks."""
    import importlib

    from oracle import oracle as O

    ref_search = importlib.reload(importlib.import_module("mvdtw.search"))  # unpatched
    rng = np.random.default_rng(4)
    series = np.cumsum(rng.normal(size=(60, 40, 3)), axis=1)
    series = (series - series.reshape(-1, 3).mean(0)) / series.reshape(-1, 3).std(0)
    dr = series.reshape(-1, 3).max(0) - series.reshape(-1, 3).min(0)
    queries, cands = list(series[:20]), list(series[20:])
    params = mvdtw.SearchParams(window=4, method=mvdtw.Method.TC_DTW)
    tuned = ref_search.tune_params(queries, cands, params, seed=42, dim_range=dr)
    rs = np.random.default_rng(42)
    sq = ref_search._sample(queries, ref_search.TUNE_QUERY_SAMPLE, rs)
    sc = ref_search._sample(cands, ref_search.TUNE_CANDIDATE_SAMPLE, rs)
    pick = ref_search.tc_dtw_select(sq, sc, tuned, dim_range=dr)
    e_ti, e_pc, lv, adv = O.resolve_tc_dtw(np.stack(queries), np.stack(cands), 4, dr, seed=42)
    assert (e_ti, e_pc, lv) == (tuned.trigger_ti, tuned.trigger_pc, tuned.quant_levels)
    assert adv == pick.value
