"""Candidate-side index: whole-collection envelopes and
the reverse LB_MV bound.  The answers must not change (identical indices,
bit-identical distances against the oracle); only the pruning counters may.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _params(P, w, method="lb_mv"):
    return P.SearchParams(window=w, method=P.Method(method))


def test_candidate_envelopes_match_oracle(rng):
    import paper_2101_07731_b200 as P
    from oracle import oracle as O

    for dtype, np_t in (("f64", np.float64), ("f32", np.float32)):
        cands = np.cumsum(rng.normal(size=(300, 40, 3)), axis=1).astype(np_t)
        index = P.SearchIndex(cands, dtype=dtype)
        up, lo = index.candidate_envelopes(7)
        up, lo = up.cpu().numpy(), lo.cpu().numpy()
        for s in (0, 1, 150, 299):
            ou, ol = O.build_envelope(cands[s].astype(np.float64), 7)
            assert np.array_equal(up[s].astype(np.float64), ou)
            assert np.array_equal(lo[s].astype(np.float64), ol)
        # cached per window, rebuilt on a new one
        assert index.candidate_envelopes(7)[0].data_ptr() == index.candidate_envelopes(7)[0].data_ptr()
        assert index.candidate_envelopes(100)[0].shape == up.shape  # W >= n clips to n-1


@pytest.mark.parametrize("cfg,wi,nq,method", [("C0", 0, 20, "lb_mv"), ("C0", 0, 20, "lb_pc"),
                                              ("C1", 0, 64, "lb_mv"), ("C1", 1, 24, "lb_mv"),
                                              ("C2", 0, 16, "lb_mv"), ("C4", 0, 2, "lb_mv")])
def test_reverse_bound_parity(cfg, wi, nq, method):
    import paper_2101_07731_b200 as P
    from oracle import oracle as O
    from paper_2101_07731_b200.datasets import make_workload

    wl = make_workload(cfg)
    w = wl.spec.windows()[wi]
    qsel = wl.queries[:nq]
    index = P.SearchIndex(wl.candidates, dtype=wl.dtype)
    fwd = index.search(qsel, _params(P, w, method), dim_range=wl.dim_range)
    both = index.search(qsel, _params(P, w, method), dim_range=wl.dim_range, reverse_bound=True)
    outs, _ = O.nn_search_batch(qsel.astype(np.float64), wl.candidates.astype(np.float64),
                                O.make_params(w, method), None, wl.dim_range)
    for i, o in enumerate(outs):
        assert both.best_index[i] == o.best_index == fwd.best_index[i], (cfg, i)
        assert both.best_distance[i] == o.best_distance == fwd.best_distance[i], (cfg, i)
    # same seeds, same d_best at compaction: the survivors are a subset
    assert np.all(both.counters["survivors"] <= fwd.counters["survivors"])
    assert np.all(both.counters["dtw_computed"] + both.counters["dtw_skipped"] == len(wl.candidates))


def test_reverse_bound_none_method_ignored(rng):
    import paper_2101_07731_b200 as P

    cands = rng.normal(size=(50, 16, 2))
    q = rng.normal(size=(3, 16, 2))
    index = P.SearchIndex(cands, dtype="f64")
    a = index.search(q, _params(P, 3, "none"), reverse_bound=True)
    b = index.search(q, _params(P, 3, "none"))
    assert np.array_equal(a.best_index, b.best_index) and np.array_equal(a.best_distance, b.best_distance)


def test_candidate_box_sets_and_steps_match_oracle(rng):
    """f2: the collection's box sets and neighbour steps, built once per
    index, equal the per-series reference constructions (oracle)."""
    import paper_2101_07731_b200 as P
    from oracle import oracle as O

    cands = np.cumsum(rng.normal(size=(120, 48, 3)), axis=1)
    dr = cands.reshape(-1, 3).max(0) - cands.reshape(-1, 3).min(0)
    index = P.SearchIndex(cands, dtype="f64")
    params = P.SearchParams(window=5, method="lb_pc", group_width=4, quant_levels=2, max_boxes=6)
    lo, hi, cnt = index.candidate_box_sets(params, dr)
    lo, hi, cnt = lo.cpu().numpy(), hi.cpu().numpy(), cnt.cpu().numpy()
    for s in (0, 7, 119):
        olo, ohi, ocnt, _ = O.build_box_sets(cands[s], 5, 4, 2, 6, params.min_cell_frac, dr)
        k = olo.shape[1]
        assert np.array_equal(cnt[s], ocnt)
        assert np.array_equal(lo[s][:, :k], olo) and np.array_equal(hi[s][:, :k], ohi)
        assert np.all(lo[s][:, k:] == np.inf) and np.all(hi[s][:, k:] == -np.inf)
    assert index.candidate_box_sets(params, dr)[0].data_ptr() == index.candidate_box_sets(params, dr)[0].data_ptr()
    steps = index.candidate_steps().cpu().numpy()
    for s in (0, 60, 119):
        assert np.array_equal(steps[s], O.neighbor_steps(cands[s]))
    # LB_TI's BASIC variant fed with the index's candidate steps (lb_ti.py:58-76)
    q = np.cumsum(rng.normal(size=(48, 3)), axis=0)
    nb = P.NeighborDistances(P.neighbor_steps(q), steps[7])
    got = P.lb_ti(q, cands[7], 5, variant=P.TiVariant.BASIC, neighbor=nb)
    want = O.lb_ti(q, cands[7], 5, variant="basic")
    assert got.value == want[0]


@pytest.mark.parametrize("cfg,wi,nq,method,adv", [("C0", 0, 20, "lb_pc", None), ("C0", 0, 20, "tc_dtw", "lb_pc"),
                                                  ("C1", 0, 48, "lb_pc", None), ("C1", 1, 16, "tc_dtw", "lb_pc"),
                                                  ("C4", 0, 2, "lb_pc", None)])
def test_reverse_pc_parity(cfg, wi, nq, method, adv):
    """The reverse LB_PC (query points vs the candidates' box sets) prunes at
    least as much and never changes an answer."""
    import paper_2101_07731_b200 as P
    from oracle import oracle as O
    from paper_2101_07731_b200.datasets import make_workload

    wl = make_workload(cfg)
    w = wl.spec.windows()[wi]
    qsel = wl.queries[:nq]
    index = P.SearchIndex(wl.candidates, dtype=wl.dtype)
    a = None if adv is None else P.Method(adv)
    fwd = index.search(qsel, _params(P, w, method), advanced=a, dim_range=wl.dim_range)
    both = index.search(qsel, _params(P, w, method), advanced=a, dim_range=wl.dim_range, reverse_pc=True)
    outs, _ = O.nn_search_batch(qsel.astype(np.float64), wl.candidates.astype(np.float64),
                                O.make_params(w, method), adv, wl.dim_range)
    for i, o in enumerate(outs):
        assert both.best_index[i] == o.best_index == fwd.best_index[i], (cfg, i)
        assert both.best_distance[i] == o.best_distance == fwd.best_distance[i], (cfg, i)
    assert np.all(both.counters["dtw_computed"] + both.counters["dtw_skipped"] == len(wl.candidates))
    if wl.dtype == "f32":  # same float32 pipeline: the extra bound only removes DTWs
        assert both.counters["dtw_computed"].sum() <= fwd.counters["dtw_computed"].sum()
