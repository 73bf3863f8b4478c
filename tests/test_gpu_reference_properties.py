"""The reference's own known answers and properties (its unit
tests' hand examples and acceptance criteria 1-4, 6, 8; criterion 5, skip
rates rising as W drops, is a statistical property of the reference's data
and is not asserted), run through the GPU
per-pair and search APIs.  Instances are drawn here with this suite's own
generator (four families like the reference's fixtures: random walk, iid,
shifted near-copy, plateaus); the brute-force path enumeration is this
file's own.  Bounds are compared with DTW exactly (no tolerance), as the
reference does."""

import itertools
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TI = ["basic", "top", "tip", "tip_top"]


def family(rng, k, n, d):
    kind = k % 4
    if kind == 0:
        return np.cumsum(rng.normal(size=(n, d)), axis=0)
    if kind == 1:
        return rng.normal(size=(n, d))
    if kind == 2:
        base = np.cumsum(rng.normal(size=(n, d)), axis=0)
        return np.roll(base + rng.normal(0, 1e-3, (n, d)), int(rng.integers(0, 3)), axis=0)
    reps = np.repeat(rng.normal(size=(max(1, n // 3), d)), 3, axis=0)
    return np.concatenate([reps, np.repeat(reps[-1:], n, axis=0)])[:n]


def batch(rng, count, n, d):
    return (np.stack([family(rng, k, n, d) for k in range(count)]),
            np.stack([family(rng, k + 1, n, d) for k in range(count)]))


# ----------------------------------------------------------- hand examples
def test_hand_examples():
    import paper_2101_07731_b200 as P

    assert P.dtw_banded([[0.0], [0.0]], [[1.0], [1.0]], 1).distance == pytest.approx(2.0, abs=1e-12)
    assert P.dtw_banded([[0.0, 0.0], [3.0, 4.0]], [[0.0, 0.0], [0.0, 0.0]], 1).distance == pytest.approx(5.0, abs=1e-12)
    env = P.build_envelope([[1.0], [2.0], [3.0]], 1)
    assert env.upper[:, 0].tolist() == [2.0, 3.0, 3.0] and env.lower[:, 0].tolist() == [1.0, 1.0, 2.0]
    assert P.lb_mv([[5.0], [5.0], [5.0]], env).value == pytest.approx(7.0, abs=1e-12)
    assert P.lb_ad([[1.0], [2.0], [3.0]], [[5.0], [5.0], [5.0]], 1).value == pytest.approx(7.0, abs=1e-12)
    lo, up = P.ti_advance(5.0, 7.0, 2.0)
    assert lo == pytest.approx(3.0, abs=1e-11) and up == pytest.approx(9.0, rel=1e-12) and lo <= 3.0 <= 9.0 <= up
    lo, up = P.ti_advance(1.0, 2.0, 10.0)
    assert lo == pytest.approx(8.0, abs=1e-11) and up == pytest.approx(12.0, rel=1e-12)
    lo, up = P.ti_advance(1.0, 5.0, 2.0)  # both branches negative: clamp at zero
    assert lo == 0.0 and up == pytest.approx(7.0, rel=1e-12)
    lo, up = P.ti_extend_top(4.0, 6.0, 1.0)
    assert lo == pytest.approx(3.0, abs=1e-11) and up == pytest.approx(7.0, rel=1e-12)
    q = np.array([[0.0], [0.1], [0.9], [1.0]])
    g = P.build_box_sets(q, 3, 1, 2, 6, 1e-5)
    c = np.full((4, 1), 0.5)
    assert P.lb_pc(c, g).value == pytest.approx(1.6, rel=1e-12)
    assert P.lb_mv(c, P.build_envelope(q, 3)).value == 0.0


def test_window_zero_cells_and_abandon_contract(rng):
    import paper_2101_07731_b200 as P

    q, c = rng.normal(size=(15, 2)), rng.normal(size=(15, 2))
    pointwise = sum(math.sqrt(((q[i] - c[i]) ** 2).sum()) for i in range(15))
    assert P.dtw_banded(q, c, 0).distance == pytest.approx(pointwise, rel=1e-12)
    q, c = rng.normal(size=(10, 2)), rng.normal(size=(10, 2))
    assert P.dtw_banded(q, c, 2).cells == sum(min(9, i + 2) - max(0, i - 2) + 1 for i in range(10))
    q, c = np.cumsum(rng.normal(size=(20, 3)), 0), np.cumsum(rng.normal(size=(20, 3)), 0)
    full = P.dtw_banded(q, c, 5)
    assert not full.abandoned
    assert not P.dtw_banded(q, c, 5, abandon_above=math.inf).abandoned
    cut = P.dtw_banded(q, c, 5, abandon_above=full.distance * 0.999)
    assert cut.abandoned and full.distance * 0.999 < cut.distance <= full.distance and cut.cells <= full.cells
    assert not P.dtw_banded(q, c, 5, abandon_above=full.distance).abandoned
    for w in (0, 3, 11, 50):
        assert P.dtw_banded(q, q, w).distance == 0.0


# -------------------------------------------------- path enumeration (crit. 2)
def brute_dtw(q, c, w):
    """Minimum over every monotone, continuous warping path inside the band."""
    n = len(q)
    cost = np.array([[math.sqrt(((q[i] - c[j]) ** 2).sum()) for j in range(n)] for i in range(n)])
    best = math.inf

    def walk(i, j, acc):
        nonlocal best
        if abs(i - j) > w or acc >= best:
            return
        acc += cost[i, j]
        if i == n - 1 and j == n - 1:
            best = min(best, acc)
            return
        for di, dj in ((1, 0), (0, 1), (1, 1)):
            if i + di < n and j + dj < n:
                walk(i + di, j + dj, acc)

    walk(0, 0, 0.0)
    return best


def test_dtw_equals_path_enumeration(rng):
    import paper_2101_07731_b200 as P

    for n, d in itertools.product((2, 4, 6, 7), (1, 3)):
        for w in range(0, n):
            A, B = batch(rng, 6, n, d)
            dist, _, _ = P.dtw_banded_pairs(A, B, w)
            for p in range(6):
                assert dist[p] == pytest.approx(brute_dtw(A[p], B[p], w), rel=1e-9)
            # symmetry, bit for bit (the transposed DP does the same operations)
            dist_t, _, _ = P.dtw_banded_pairs(B, A, w)
            assert np.array_equal(dist, dist_t)


# ------------------------------------- soundness and dominance (crit. 1, 4)
@pytest.mark.parametrize("n,d,w", [(1, 2, 0), (5, 1, 2), (16, 3, 4), (24, 5, 10), (33, 2, 33), (48, 8, 6),
                                   (64, 10, 20), (9, 4, 0)])
def test_bound_soundness_and_dominance(rng, n, d, w):
    import paper_2101_07731_b200 as P
    from paper_2101_07731_b200.lb_mv import build_envelopes, lb_ad_pairs, lb_mv_pairs
    from paper_2101_07731_b200.lb_pc import build_box_sets_batch, lb_pc_pairs
    from paper_2101_07731_b200.lb_ti import lb_ti_pairs

    Q, C = batch(rng, 160, n, d)
    exact, _, _ = P.dtw_banded_pairs(Q, C, w)
    up, lo = build_envelopes(Q, min(w, n - 1))
    mv, _ = lb_mv_pairs(C, up, lo)
    ad, _ = lb_ad_pairs(Q, C, w)
    assert np.all(mv <= exact) and np.all(ad <= exact) and np.all(mv <= ad)
    for levels in (1, 2, 3):
        for cap in (1, 4, 6):
            bl, bh, _ = build_box_sets_batch(Q, w, 1, levels, cap, 1e-5)
            pc, _ = lb_pc_pairs(C, bl, bh, 1)
            assert np.all(mv <= pc) and np.all(pc <= ad) and np.all(pc <= exact), (levels, cap)
            bl6, bh6, _ = build_box_sets_batch(Q, w, 6, levels, cap, 1e-5)
            pc6, _ = lb_pc_pairs(C, bl6, bh6, 6)
            assert np.all(pc6 <= exact)
    vals = {}
    for variant in TI:
        for period in (1, 2, 5, n):
            v, _ = lb_ti_pairs(Q, C, w, variant, period)
            assert np.all(v <= ad) and np.all(v <= exact), (variant, period)
            vals[(variant, period)] = v
    # refreshing only every n rows never refreshes: bit-identical to the propagate-only variants
    assert np.array_equal(vals[("tip", n)], vals[("basic", 5)])
    assert np.array_equal(vals[("tip_top", n)], vals[("top", 5)])
    np.testing.assert_allclose(vals[("tip", 1)], ad, rtol=1e-12, atol=1e-12)


# ------------------------------------------------- search-level (crit. 3, 6, 8)
def _dataset(rng, S=200, n=50, d=3, smooth=True):
    if smooth:
        X = np.cumsum(rng.normal(size=(S, n, d)), axis=1)
    else:
        centers = rng.normal(size=(6, n, d)) * 3
        X = centers[rng.integers(0, 6, S)] + rng.normal(size=(S, n, d)) * 0.3
    X = (X - X.reshape(-1, d).mean(0)) / X.reshape(-1, d).std(0)
    return X, X.reshape(-1, d).max(0) - X.reshape(-1, d).min(0)


def test_trigger_band_scenario():
    import paper_2101_07731_b200 as P

    q = np.zeros((4, 1))
    cands = [np.ones((4, 1)), np.full((4, 1), 10.0), np.array([[1.0], [1.0], [0.0], [0.0]]),
             np.array([[0.0], [0.0], [0.0], [0.1]])]
    out = P.nn_search(q, cands, P.SearchParams(window=1, method=P.Method.LB_TI, trigger_ti=0.1))
    assert out.best_index == 3 and out.best_distance == pytest.approx(0.1)
    assert out.dtw_computed + out.dtw_skipped == 4


def test_nn_identity_skip_monotonicity_and_determinism(rng):
    import paper_2101_07731_b200 as P
    from oracle import oracle as O

    for smooth in (True, False):
        X, dr = _dataset(rng, smooth=smooth)
        qs, cs = X[:40], X[40:]
        index = P.SearchIndex(cs, dtype="f64")
        answers = {}
        skipped = {}
        for method, adv in (("none", None), ("lb_mv", None), ("lb_ti", None), ("lb_pc", None), ("lb_ad", None),
                            ("tc_dtw", "lb_ti"), ("tc_dtw", "lb_pc")):
            for w in (10, 20):
                res = index.search(qs, P.SearchParams(window=w, method=P.Method(method)),
                                   advanced=None if adv is None else P.Method(adv), dim_range=dr)
                answers[(method, adv, w)] = (res.best_index.tolist(), res.best_distance.tolist())
                skipped[(method, adv, w)] = int(res.counters["dtw_skipped"].sum())
                again = index.search(qs, P.SearchParams(window=w, method=P.Method(method)),
                                     advanced=None if adv is None else P.Method(adv), dim_range=dr)
                # criterion 8: the reported counters (computed / skipped) are run-to-run identical
                assert np.array_equal(res.counters["dtw_skipped"], again.counters["dtw_skipped"])
                assert np.array_equal(res.counters["dtw_computed"], again.counters["dtw_computed"])
        for w in (10, 20):
            ref = answers[("none", None, w)]
            for key, val in answers.items():
                if key[2] == w:
                    assert val == ref, key  # criterion 3: every method finds the same neighbours
            outs, _ = O.nn_search_batch(qs, cs, O.make_params(w, "none"), None, dr)
            assert ref[0] == [o.best_index for o in outs] and ref[1] == [o.best_distance for o in outs]
            # criterion 6: the cascades skip at least as often as LB_MV alone
            assert skipped[("tc_dtw", "lb_pc", w)] >= skipped[("lb_mv", None, w)]
            assert skipped[("tc_dtw", "lb_ti", w)] >= skipped[("lb_mv", None, w)]
