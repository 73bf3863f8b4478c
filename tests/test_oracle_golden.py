"""Pin the C oracle against vectors produced by the reference itself.

Every comparison is bit-exact (==): the oracle restates the reference's
float64 arithmetic including numpy's pairwise summation order.  If these
pass, the oracle is a trustworthy checker for the GPU parity tests.
"""

import numpy as np
import pytest

from golden_io import dr_or_none, load_cases, thr_or_none
from oracle import oracle as O

TI_NAMES = ["basic", "top", "tip", "tip_top"]


def test_dtw_banded_golden():
    for case in load_cases("dtw"):
        j = 0
        while f"dist{j}" in case:
            d, ab, cells = O.dtw_banded(case["q"], case["c"], case["w"], thr_or_none(case[f"thr{j}"]))
            assert d == case[f"dist{j}"]
            assert ab == case[f"ab{j}"]
            assert cells == case[f"cells{j}"]
            j += 1


def test_envelope_golden():
    for case in load_cases("envelope"):
        up, lo = O.build_envelope(case["q"], case["w"])
        assert np.array_equal(up, case["upper"]) and np.array_equal(lo, case["lower"])


def test_lb_mv_lb_ad_steps_golden():
    for case in load_cases("lb_mv_ad"):
        up, lo = O.build_envelope(case["q"], case["w"])
        for j in range(3):
            v, ab = O.lb_mv(case["c"], up, lo, thr_or_none(case[f"mv_thr{j}"]))
            assert v == case[f"mv{j}"] and ab == case[f"mv_ab{j}"]
            v, ab = O.lb_ad(case["q"], case["c"], case["w"], thr_or_none(case[f"ad_thr{j}"]))
            assert v == case[f"ad{j}"] and ab == case[f"ad_ab{j}"]
        assert np.array_equal(O.neighbor_steps(case["q"]), case["steps_q"])


def test_ti_advance_golden():
    adv = load_cases("lb_ti")[0]["adv"]
    for lo, up, s, elo, eup in adv:
        assert O.ti_advance(lo, up, s) == (elo, eup)


def test_lb_ti_golden():
    for case in load_cases("lb_ti")[1:]:
        for k in range(case["nv"]):
            v, ab = O.lb_ti(case["q"], case["c"], case["w"], TI_NAMES[case[f"v{k}_variant"]],
                            case[f"v{k}_period"], thr_or_none(case[f"v{k}_thr"]))
            assert v == case[f"v{k}_val"] and ab == case[f"v{k}_ab"]


def test_quantize_cluster_golden():
    for case in load_cases("quantize"):
        los, his = O.quantize_cluster(case["pts"], case["levels"], case["cap"], case["mcf"],
                                      dr_or_none(case["dr"]))
        assert np.array_equal(los, case["los"]) and np.array_equal(his, case["his"])


def test_box_sets_and_lb_pc_golden():
    for case in load_cases("box_sets"):
        lo, hi, counts, spans = O.build_box_sets(case["q"], case["w"], case["gw"], case["levels"],
                                                 case["cap"], 1e-5, dr_or_none(case["dr"]))
        assert np.array_equal(lo, case["pad_lo"]) and np.array_equal(hi, case["pad_hi"])
        assert np.array_equal(counts, case["counts"])
        assert [list(s) for s in spans] == case["spans"].tolist()
        for j in range(3):
            v, ab = O.lb_pc(case["c"], lo, hi, case["gw"], thr_or_none(case[f"thr{j}"]))
            assert v == case[f"val{j}"] and ab == case[f"ab{j}"]


RUNS = [("none", None), ("lb_mv", None), ("lb_ti", None), ("lb_pc", None), ("lb_ad", None),
        ("tc_dtw", "lb_ti"), ("tc_dtw", "lb_pc")]
FIELDS = ("best_index", "best_distance", "dtw_computed", "dtw_skipped", "lb_mv_evals",
          "advanced_lb_evals", "abandon_count", "work")


def _check_runs(q, cands, w, dr, case, runs):
    for k, (method, adv) in enumerate(runs):
        if f"m{k}_best_index" not in case:
            continue
        params = O.make_params(w, method)
        (out,), _ = O.nn_search_batch(q[None], cands, params, adv, dr, n_threads=1)
        for f in FIELDS:
            assert getattr(out, f) == case[f"m{k}_{f}"], (method, adv, f)


def test_nn_search_small_golden():
    cases = load_cases("search_small")
    for case in cases:
        runs = RUNS if "m1_best_index" in case else [("lb_ti", None)]
        _check_runs(case["q"], case["cands"], case["w"], dr_or_none(case["dr"]), case, runs)


def test_tc_dtw_unresolved_rejected():
    q = np.zeros((4, 1))
    with pytest.raises(ValueError):
        O.nn_search_batch(q[None], np.zeros((2, 4, 1)), O.make_params(1, "tc_dtw"), None)


@pytest.mark.parametrize("cfg", ["C0", "C1", "C2", "C3"])
def test_config_samples_golden(cfg):
    from paper_2101_07731_b200.datasets import make_workload
    import hashlib

    cases = [c for c in load_cases("configs") if c["cfg"] == cfg]
    assert cases
    wl = make_workload(cfg, seed=0)
    dig = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]  # noqa: E731
    assert dig(wl.candidates) == cases[0]["digest_c"] and dig(wl.queries) == cases[0]["digest_q"]
    cands = wl.candidates.astype(np.float64)
    for case in cases:
        runs = [tuple(None if x == "None" else x for x in r.split(":")) for r in case["runs"].tolist()]
        q = wl.queries[case["qi"]].astype(np.float64)
        _check_runs(q, cands, case["w"], wl.dim_range, case, runs)
