"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden vectors and the pinned C oracle.

Tolerances: float64 paths are compared bit-for-bit (==), which is stricter
than the north star's 1e-9 relative; float32 configs must return identical
indices and distances within 1e-4 relative of the oracle (float64 on the
float32-rounded inputs) -- the float64 finalist re-score makes them exact in
practice, and the tests assert <= 1e-12 where that holds.
"""

import numpy as np
import pytest

from golden_io import dr_or_none, load_cases, thr_or_none

pytestmark = pytest.mark.gpu

TI_NAMES = ["basic", "top", "tip", "tip_top"]


@pytest.fixture(scope="module")
def P():
    import paper_2101_07731_b200 as pkg

    return pkg


# ------------------------------------------------------------ per-pair API
def test_dtw_banded_golden(P):
    for case in load_cases("dtw"):
        j = 0
        while f"dist{j}" in case:
            r = P.dtw_banded(case["q"], case["c"], case["w"], thr_or_none(case[f"thr{j}"]))
            assert r.distance == case[f"dist{j}"]
            assert r.abandoned == case[f"ab{j}"]
            assert r.cells == case[f"cells{j}"]
            j += 1


def test_dtw_pairs_batched_matches_single(P, rng):
    from oracle import oracle as O

    for n, d, w in ((17, 3, 4), (64, 8, 10), (40, 20, 3), (9, 1, 0)):
        A = np.cumsum(rng.normal(size=(50, n, d)), axis=1)
        B = np.cumsum(rng.normal(size=(50, n, d)), axis=1)
        dist, ab, cells = P.dtw_banded_pairs(A, B, w)
        for p in range(50):
            od, oab, oc = O.dtw_banded(A[p], B[p], w)
            assert dist[p] == od and ab[p] == oab and cells[p] == oc


def test_point_distance(P, rng):
    for _ in range(20):
        a, b = rng.normal(size=5), rng.normal(size=5)
        assert P.point_distance(a, b) == float(np.sqrt(((a - b) ** 2).sum()))


def test_envelope_golden(P):
    for case in load_cases("envelope"):
        env = P.build_envelope(case["q"], case["w"])
        assert np.array_equal(env.upper, case["upper"]) and np.array_equal(env.lower, case["lower"])
        assert env.window == case["weff"]


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_envelope_stream_shapes(P, rng, dtype):
    """The staged van Herk envelope kernel (whole stacks, ragged last group,
    odd n*d without 16-byte loads, W = 0, W >= n, blocks of one point) is
    bit-identical to the oracle's sliding max/min (lb_mv.py:44-88)."""
    from oracle import oracle as O
    from paper_2101_07731_b200.lb_mv import build_envelopes

    for S, n, d, w in ((37, 128, 6, 12), (11, 64, 20, 6), (9, 33, 3, 5), (5, 17, 1, 0), (7, 10, 4, 40),
                       (6, 25, 5, 12), (13, 31, 7, 3), (3, 1, 2, 2)):
        X = rng.normal(size=(S, n, d)).astype(dtype)
        X[0, :, 0] = 0.0  # constant runs: ties everywhere
        import torch

        up, lo = build_envelopes(X, w, dtype=torch.float32 if dtype == np.float32 else None)
        assert up.dtype == (torch.float32 if dtype == np.float32 else torch.float64)
        up, lo = up.cpu().numpy(), lo.cpu().numpy()
        for s in range(S):
            ou, ol = O.build_envelope(X[s].astype(np.float64), min(w, n - 1))
            assert np.array_equal(up[s].astype(np.float64), ou), (S, n, d, w, s)
            assert np.array_equal(lo[s].astype(np.float64), ol), (S, n, d, w, s)


def test_lb_mv_lb_ad_steps_golden(P):
    for case in load_cases("lb_mv_ad"):
        env = P.build_envelope(case["q"], case["w"])
        for j in range(3):
            r = P.lb_mv(case["c"], env, thr_or_none(case[f"mv_thr{j}"]))
            assert r.value == case[f"mv{j}"] and r.abandoned == case[f"mv_ab{j}"]
            r = P.lb_ad(case["q"], case["c"], case["w"], thr_or_none(case[f"ad_thr{j}"]))
            assert r.value == case[f"ad{j}"] and r.abandoned == case[f"ad_ab{j}"]
        if len(case["q"]) > 1:
            assert np.array_equal(P.neighbor_steps(case["q"]), case["steps_q"])


def test_ti_advance_golden(P):
    from paper_2101_07731_b200.lb_ti import ti_advance_batch

    adv = load_cases("lb_ti")[0]["adv"]
    lo, up = ti_advance_batch(adv[:, 0], adv[:, 1], adv[:, 2])
    assert np.array_equal(lo.cpu().numpy(), adv[:, 3]) and np.array_equal(up.cpu().numpy(), adv[:, 4])
    assert P.ti_advance(2.5, 4.0, 0.0) == (2.5, 4.0)
    assert P.ti_extend_top(3.0, 6.0, 0.0) == (3.0, 6.0)


def test_lb_ti_golden(P):
    for case in load_cases("lb_ti")[1:]:
        for k in range(case["nv"]):
            r = P.lb_ti(case["q"], case["c"], case["w"], TI_NAMES[case[f"v{k}_variant"]], case[f"v{k}_period"],
                        abandon_above=thr_or_none(case[f"v{k}_thr"]))
            assert r.value == case[f"v{k}_val"] and r.abandoned == case[f"v{k}_ab"]


def test_lb_ti_neighbor_reuse(P, rng):
    q = np.cumsum(rng.normal(size=(18, 3)), axis=0)
    c = np.cumsum(rng.normal(size=(18, 3)), axis=0)
    nd = P.NeighborDistances.build(q, c, P.TiVariant.BASIC)
    assert nd.candidate_steps is not None
    assert P.lb_ti(q, c, 4, P.TiVariant.BASIC).value == P.lb_ti(q, c, 4, P.TiVariant.BASIC, neighbor=nd).value


def test_quantize_cluster_golden(P):
    for case in load_cases("quantize"):
        bs = P.quantize_cluster(case["pts"], case["levels"], case["cap"], case["mcf"], dr_or_none(case["dr"]))
        assert np.array_equal(bs.los, case["los"]) and np.array_equal(bs.his, case["his"])


def test_box_sets_and_lb_pc_golden(P):
    for case in load_cases("box_sets"):
        g = P.build_box_sets(case["q"], case["w"], case["gw"], case["levels"], case["cap"], 1e-5,
                             dr_or_none(case["dr"]))
        assert np.array_equal(g.pad_lo, case["pad_lo"]) and np.array_equal(g.pad_hi, case["pad_hi"])
        assert np.array_equal(g.box_counts, case["counts"])
        assert [list(s) for s in g.spans] == case["spans"].tolist()
        for j in range(3):
            r = P.lb_pc(case["c"], g, thr_or_none(case[f"thr{j}"]))
            assert r.value == case[f"val{j}"] and r.abandoned == case[f"ab{j}"]


# ------------------------------------------------------------------ search
RUNS = [("none", None), ("lb_mv", None), ("lb_ti", None), ("lb_pc", None), ("lb_ad", None),
        ("tc_dtw", "lb_ti"), ("tc_dtw", "lb_pc")]


def _params(P, w, method):
    return P.SearchParams(window=w, method=P.Method(method))


def test_nn_search_small_golden(P):
    for case in load_cases("search_small"):
        runs = RUNS if "m1_best_index" in case else [("lb_ti", None)]
        for k, (method, adv) in enumerate(runs):
            out = P.nn_search(case["q"], list(case["cands"]), _params(P, case["w"], method),
                              advanced=None if adv is None else P.Method(adv), dim_range=dr_or_none(case["dr"]))
            assert out.best_index == case[f"m{k}_best_index"], (method, adv)
            assert out.best_distance == case[f"m{k}_best_distance"], (method, adv)
            assert out.dtw_computed + out.dtw_skipped == len(case["cands"])


def test_c0_all_methods_golden(P):
    from paper_2101_07731_b200.datasets import make_workload

    wl = make_workload("C0")
    cases = [c for c in load_cases("configs") if c["cfg"] == "C0"]
    index = P.SearchIndex(wl.candidates, dtype="f64")
    for k, (method, adv) in enumerate(RUNS):
        res = index.search(wl.queries, _params(P, 12, method), advanced=None if adv is None else P.Method(adv),
                           dim_range=wl.dim_range)
        for case in cases:
            qi = case["qi"]
            assert res.best_index[qi] == case[f"m{k}_best_index"], (method, adv, qi)
            assert res.best_distance[qi] == case[f"m{k}_best_distance"], (method, adv, qi)
        c = res.counters
        assert np.all(c["dtw_computed"] + c["dtw_skipped"] == len(wl.candidates))


def _oracle_check(P, cfg, wi, n_queries, method="lb_mv", advanced=None, dtype=None, rel=0.0, f32_filter=None,
                  spread=False):
    """n_queries of the config against the oracle; ``spread`` samples seeded
    random query indices across the whole query set instead of the first."""
    from oracle import oracle as O
    from paper_2101_07731_b200.datasets import make_workload

    wl = make_workload(cfg)
    w = wl.spec.windows()[wi]
    if spread:
        pick = np.sort(np.random.default_rng(99).choice(len(wl.queries), size=n_queries, replace=False))
        qsel = wl.queries[pick]
    else:
        qsel = wl.queries[:n_queries]
    index = P.SearchIndex(wl.candidates, dtype=dtype or wl.dtype, f32_filter=f32_filter)
    if f32_filter is not None:
        assert index.f32_filter == (f32_filter and index.dtype == "f64")
    res = index.search(qsel, _params(P, w, method), advanced=None if advanced is None else P.Method(advanced),
                       dim_range=wl.dim_range)
    outs, _ = O.nn_search_batch(qsel.astype(np.float64), wl.candidates.astype(np.float64),
                                O.make_params(w, method), advanced, wl.dim_range)
    for i, o in enumerate(outs):
        assert res.best_index[i] == o.best_index, (cfg, i)
        if rel == 0.0:
            assert res.best_distance[i] == o.best_distance, (cfg, i)
        else:
            assert abs(res.best_distance[i] - o.best_distance) <= rel * o.best_distance, (cfg, i)
    return res


def test_c1a_full_parity(P):
    # all 500 queries, float32 filter + float64 re-score: bit-exact distances
    _oracle_check(P, "C1", 0, 500, rel=0.0)


def test_c1b_parity(P):
    _oracle_check(P, "C1", 1, 128, rel=0.0)


def test_c1_cascades_parity(P):
    _oracle_check(P, "C1", 0, 32, method="lb_pc", rel=0.0)
    _oracle_check(P, "C1", 0, 16, method="tc_dtw", advanced="lb_ti", rel=0.0)


def test_c2_parity(P):
    _oracle_check(P, "C2", 0, 48, rel=0.0)


def test_c3_parity(P):
    # float64 data: the float32 filter + float64 re-score on the originals
    # (the default) and the all-float64 kernels give the reference's bits
    _oracle_check(P, "C3", 0, 24, rel=0.0, f32_filter=True)
    _oracle_check(P, "C3", 0, 8, rel=0.0, f32_filter=False)


def test_c0_filter_and_exact_paths(P):
    for flt in (True, False):
        for method, adv in (("lb_mv", None), ("lb_pc", None), ("tc_dtw", "lb_ti"), ("none", None)):
            _oracle_check(P, "C0", 0, 20, method=method, advanced=adv, rel=0.0, f32_filter=flt)


def test_c4_sampled_parity(P):
    # spread-out query indices: fp32 near-ties are likeliest at C4
    _oracle_check(P, "C4", 0, 24, rel=0.0, spread=True)


@pytest.mark.parametrize("n,d,w", [(64, 3, 6), (200, 5, 20), (300, 8, 60), (129, 1, 0), (40, 20, 4), (512, 6, 51)])
def test_f32_filter_matches_exact_kernels(P, rng, n, d, w):
    """float64 inputs: the float32-filtered search returns the all-float64
    search's indices and distances bit for bit, including exact ties,
    near-ties below float32 resolution and a wide value range."""
    cands = np.cumsum(rng.normal(size=(300, n, d)), axis=1) * 10.0 ** rng.uniform(-3, 3)
    queries = cands[:12] + rng.normal(size=(12, n, d)) * 1e-9  # near-ties far below float32 resolution
    queries[3] = cands[40]  # exact match
    cands[41] = cands[40]  # exact tie: the lower index wins
    out = {}
    for flt in (True, False):
        idx = P.SearchIndex(cands, dtype="f64", f32_filter=flt)
        assert idx.f32_filter == flt
        res = idx.search(queries, _params(P, w, "lb_mv"))
        out[flt] = (res.best_index, res.best_distance)
    assert np.array_equal(out[True][0], out[False][0])
    assert np.array_equal(out[True][1], out[False][1])
    assert out[True][0][3] == 40 and out[True][1][3] == 0.0


# ------------------------------------------------------------- edge cases
def test_edge_cases(P, rng):
    from oracle import oracle as O

    def check(q, cands, w, method="lb_mv", dtype="f64"):
        res = P.SearchIndex(cands, dtype=dtype).search(q[None], _params(P, w, method))
        outs, _ = O.nn_search_batch(q[None].astype(np.float64), np.asarray(cands, dtype=np.float64),
                                    O.make_params(w, method), None, None)
        assert res.best_index[0] == outs[0].best_index
        assert res.best_distance[0] == outs[0].best_distance

    # n == 1, W >= n, W == 0, d == 1, one candidate, fewer candidates than seeds
    check(rng.normal(size=(1, 3)), rng.normal(size=(5, 1, 3)), 4)
    check(rng.normal(size=(12, 1)), rng.normal(size=(7, 12, 1)), 40)
    check(rng.normal(size=(12, 2)), rng.normal(size=(1, 12, 2)), 0)
    check(rng.normal(size=(12, 2)), rng.normal(size=(3, 12, 2)), 2)
    # exact ties: duplicates of the nearest candidate -> lowest index wins
    base = np.cumsum(rng.normal(size=(40, 20, 3)), axis=1)
    cands = np.concatenate([base[1:], base[1:], base[1:]])
    for method in ("none", "lb_mv", "lb_pc", "lb_ti", "lb_ad"):
        check(base[0], cands, 3, method)
        check(base[0].astype(np.float32), cands.astype(np.float32), 3, method, dtype="f32")
    # query identical to a candidate: distance 0
    check(base[5], base, 3)
    # constant series everywhere (every distance equal)
    const = np.ones((64, 16, 2))
    check(const[0], const, 2)
    check(const[0].astype(np.float32), const.astype(np.float32), 2, dtype="f32")



@pytest.mark.parametrize("case", ["offset", "outside", "tiny", "huge", "ulps", "mixed_scale", "dead_sensor"])
def test_saturating_lb_mv_adversarial(P, rng, case):
    """float32 searches prune on the saturating LB_MV pass (scaled planar
    operands, midpoint / inflated half-width envelopes, FADD.SAT): inputs
    built to break a bound that is not a true lower bound -- a large common
    offset (cancellation in c - m), queries far outside the collection's
    range (saturation), tiny and huge magnitudes (power-of-two scales far
    from 1), candidates within a few ulps of the query and of its
    envelope, dimensions of very different scales -- still return the
    oracle's index and distance."""
    from oracle import oracle as O

    n, d, w, N = 64, 6, 6, 700
    walk = np.cumsum(rng.normal(size=(N, n, d)), axis=1)
    queries = walk[:8] + 0.05 * rng.normal(size=(8, n, d))
    if case == "offset":
        cands, queries = 4096.0 + 1e-2 * walk, 4096.0 + 1e-2 * queries
    elif case == "outside":
        cands, queries = walk, queries * 3.0 + 500.0
    elif case == "tiny":
        cands, queries = walk * 1e-15, queries * 1e-15
    elif case == "huge":
        cands, queries = walk * 1e15, queries * 1e15
    elif case == "ulps":
        cands = walk.astype(np.float32)
        queries = cands[:8].copy()
        for k in range(8):  # candidates 100+k..: the query moved by a few ulps, up and down
            for j in range(6):
                steps = rng.integers(-2, 3, size=(n, d))
                moved = cands[k].copy()
                for _ in range(2):
                    moved = np.where(steps > 0, np.nextafter(moved, np.float32(np.inf)),
                                     np.where(steps < 0, np.nextafter(moved, np.float32(-np.inf)), moved))
                cands[100 + 8 * j + k] = moved
        cands[300:308] = cands[:8]  # exact duplicates: the lower index wins
    elif case == "dead_sensor":
        # near-zero series inside a collection of range ~1e6: their differences vanish in the
        # scaled domain (the seed upper bound must not fall to 0) but not in the DTW's float32
        cands = walk * 3e4
        cands[50:90] = 1e-14 * rng.normal(size=(40, n, d))
        cands[60] = 0.0
        queries = 1e-14 * rng.normal(size=(8, n, d))
        queries[1] = cands[70] * 0.5
    else:  # mixed_scale
        sc = np.array([1e-3, 1.0, 1e3, 1e-6, 30.0, 1e5])
        cands, queries = walk * sc, queries * sc
    cands = np.ascontiguousarray(cands, dtype=np.float32)
    queries = np.ascontiguousarray(queries, dtype=np.float32)
    res = P.SearchIndex(cands, dtype="f32").search(queries, _params(P, w, "lb_mv"))
    outs, _ = O.nn_search_batch(queries.astype(np.float64), cands.astype(np.float64), O.make_params(w, "lb_mv"),
                                None, None)
    assert np.array_equal(res.best_index, np.array([o.best_index for o in outs]))
    assert np.array_equal(res.best_distance, np.array([o.best_distance for o in outs]))


def test_errors(P, rng):
    with pytest.raises(P.InvalidInputError):
        P.nn_search(rng.normal(size=(5, 2)), [], P.SearchParams(window=2))
    with pytest.raises(P.InvalidInputError):
        P.nn_search(rng.normal(size=(5, 2)), [rng.normal(size=(5, 2))], P.SearchParams(window=2, method="tc_dtw"))
    with pytest.raises(P.InvalidInputError):
        P.dtw_banded(np.zeros((3, 2)), np.zeros((4, 2)), 1)
    with pytest.raises(P.InvalidInputError):
        P.SearchIndex(np.zeros((2, 5, 2))).search(np.full((5, 2), np.nan), P.SearchParams(window=1, method="lb_mv"))


# ------------------------------------------------------ sharding on 1 GPU
def test_sharded_combine_equals_single(P):
    """G logical shards searched separately (global d_best exchanged between
    the phases, as the NCCL path does) and combined lexicographically equal
    the single-shard answer."""
    import torch

    from paper_2101_07731_b200.datasets import make_workload
    from paper_2101_07731_b200.distributed import shard_bounds

    wl = make_workload("C1", n_candidates=3000, n_queries=64)
    params = _params(P, 12, "lb_mv")
    ref = P.SearchIndex(wl.candidates, dtype="f32").search(wl.queries, params)
    for G in (2, 3, 8):
        shards = [P.SearchIndex(wl.candidates[a:b], dtype="f32", base=a)
                  for a, b in (shard_bounds(len(wl.candidates), G, r) for r in range(G))]
        Q = [s.prepare_queries(wl.queries) for s in shards]
        states = [s.seed_phase(q, params) for s, q in zip(shards, Q)]
        dmin = torch.stack([st["dbest"] for st in states]).min(dim=0).values  # the NCCL all-reduce(MIN)
        for st in states:
            st["dbest"].copy_(dmin)
        best = np.full(len(wl.queries), np.inf)
        idx = np.full(len(wl.queries), -1)
        for s, st in zip(shards, states):
            bi, bd, _ = s.finish_phase(st)
            bi, bd = bi.cpu().numpy(), bd.cpu().numpy()
            better = (bi >= 0) & ((bd < best) | ((bd == best) & ((idx < 0) | (bi < idx))))
            best = np.where(better, bd, best)
            idx = np.where(better, bi, idx)
        assert np.array_equal(idx, ref.best_index)
        assert np.array_equal(best, ref.best_distance)
    del torch


def test_completed_list_overflow_path(P, monkeypatch):
    """Finalisation normally visits only the list of completed DTWs; with a
    capacity of 1 (tcdtw_search_desc.done_cap) it must fall back to scanning
    every survivor tile and still return the same answers."""
    orig = P.SearchIndex.__init__

    def tiny_list(self, *a, **k):
        orig(self, *a, **k)
        self.done_cap = 1

    monkeypatch.setattr(P.SearchIndex, "__init__", tiny_list)
    _oracle_check(P, "C1", 0, 24, rel=0.0)
    _oracle_check(P, "C0", 0, 20, rel=0.0, f32_filter=True)
    _oracle_check(P, "C0", 0, 20, rel=0.0, f32_filter=False)


@pytest.mark.parametrize("dt,n,d,w", [("f32", 256, 5, 51), ("f64", 256, 5, 51), ("f64", 256, 8, 51),
                                      ("f32", 1024, 8, 102), ("f64", 512, 8, 102), ("f64", 1024, 8, 40),
                                      ("f32", 200, 3, 70), ("f64", 97, 2, 33)])
@pytest.mark.parametrize("f32_filter", [True, False])
def test_long_band_shapes(P, dt, n, d, w, f32_filter):
    """Long bands (2W+1 > 64): wavefront kernels; ragged n (not a multiple of
    32) and rows near the end of the band are the edge cases; float64 data
    through the float32 filter and through the float64 kernels."""
    from oracle import oracle as O

    if dt == "f32" and not f32_filter:
        pytest.skip("float32 data always filters in float32")
    rng = np.random.default_rng(n * 100 + w)
    C = np.cumsum(rng.normal(size=(40, n, d)), axis=1)
    Qs = np.cumsum(rng.normal(size=(3, n, d)), axis=1)
    if dt == "f32":
        C, Qs = C.astype(np.float32), Qs.astype(np.float32)
    res = P.SearchIndex(C, dtype=dt, f32_filter=f32_filter).search(Qs, P.SearchParams(window=w, method="lb_mv"))
    outs, _ = O.nn_search_batch(Qs.astype(np.float64), C.astype(np.float64), O.make_params(w, "lb_mv"), None, None)
    assert res.best_index.tolist() == [o.best_index for o in outs]
    assert res.best_distance.tolist() == [o.best_distance for o in outs]


def test_tc_dtw_select_and_tune(P):
    """Host logic over the GPU search (search.py:198-272): grid sizes, tie
    rule, deterministic picks, and tuned parameters never change answers."""
    rng = np.random.default_rng(5)
    # clustered regime-switching series (synth.clustered_dataset's regime):
    # box sets beat the single envelope box -> the clustering bound wins
    centers = rng.normal(0, 8.0, (24, 2, 2))
    state = (rng.random((24, 30)) < 0.35).cumsum(axis=1) % 2
    series = np.take_along_axis(centers, state[:, :, None].repeat(2, 2), axis=1) + rng.normal(0, 0.25, (24, 30, 2))
    queries, cands = list(series[:4]), list(series[4:])
    params = P.SearchParams(window=5, method="tc_dtw")
    assert P.tc_dtw_select(queries, cands, params) == P.Method.LB_PC
    picks = {P.tc_dtw_select(queries[:1], cands[:1], params) for _ in range(3)}
    assert len(picks) == 1
    log = []
    tuned = P.tune_params(queries, cands, params, seed=0, log=log)
    assert len(log) == 7 and tuned.refresh_period == 5 and tuned.max_boxes == 6
    base = [P.nn_search(q, cands, P.SearchParams(window=5, method="none")) for q in queries]
    choice = P.tc_dtw_select(queries, cands, tuned)
    for q, ref in zip(queries, base):
        out = P.nn_search(q, cands, tuned, advanced=choice)
        assert (out.best_index, out.best_distance) == (ref.best_index, ref.best_distance)


def test_work_model_is_run_to_run_deterministic(P):
    """with metric="work" the choices and the DP-cell counters must
    not depend on the timing of other DTWs' best-so-far updates.  A sample
    of 8 queries x 40 candidates (more than the 23 the tuner draws), three
    repetitions: identical tune_params / tc_dtw_select results, identical
    work-model costs, identical dtw_cells and abandon_count."""
    from paper_2101_07731_b200.search import SearchIndex

    rng = np.random.default_rng(17)
    series = np.cumsum(rng.normal(size=(48, 96, 3)), axis=1)
    queries, cands = list(series[:8]), list(series[8:])
    params = P.SearchParams(window=9, method="tc_dtw")
    runs = []
    for _ in range(3):
        log = []
        tuned = P.tune_params(queries, cands, params, seed=2, log=log)
        choice = P.tc_dtw_select(queries, cands, tuned)
        runs.append((tuned, choice, [c for _, _, c in log]))
    assert all(r == runs[0] for r in runs[1:])
    ctrs = []
    for _ in range(3):
        idx = SearchIndex(np.stack(cands), dtype="f64")
        idx.frozen_thresholds = True
        res = idx.search(np.stack(queries), P.SearchParams(window=9, method="lb_mv"))
        ctrs.append((res.counters["dtw_cells"].tolist(), res.counters["abandon_count"].tolist(),
                     res.best_index.tolist(), res.best_distance.tolist()))
    assert all(c == ctrs[0] for c in ctrs[1:])
    live = SearchIndex(np.stack(cands), dtype="f64").search(np.stack(queries), P.SearchParams(window=9, method="lb_mv"))
    assert live.best_index.tolist() == ctrs[0][2] and live.best_distance.tolist() == ctrs[0][3]


def test_gpu_cost_selection(P):
    """Row f1: selection and tuning ranked by measured GPU phase times
    (metric="time") instead of the work model; answers never change."""
    rng = np.random.default_rng(11)
    series = np.cumsum(rng.normal(size=(40, 32, 3)), axis=1)
    queries, cands = list(series[:6]), list(series[6:])
    params = P.SearchParams(window=4, method="tc_dtw")
    choice = P.tc_dtw_select(queries, cands, params, metric="time")
    assert choice in (P.Method.LB_TI, P.Method.LB_PC)
    log = []
    tuned = P.tune_params(queries, cands, params, seed=1, metric="time", log=log)
    assert len(log) == 7 and all(cost > 0 for _, _, cost in log)
    for q in queries:
        ref = P.nn_search(q, cands, P.SearchParams(window=4, method="none"))
        out = P.nn_search(q, cands, tuned, advanced=choice)
        assert (out.best_index, out.best_distance) == (ref.best_index, ref.best_distance)


def test_select_method_gpu_cost(P):
    """Row f1 extension: the fastest of LB_MV / TC-DTW(LB_PC) / TC-DTW(LB_TI)
    by measured GPU time; the chosen configuration finds the same answers."""
    rng = np.random.default_rng(3)
    series = np.cumsum(rng.normal(size=(60, 48, 3)), axis=1)
    queries, cands = list(series[:6]), list(series[6:])
    params, adv = P.select_method(queries, cands, P.SearchParams(window=5))
    assert (params.method, adv) in ((P.Method.LB_MV, None), (P.Method.TC_DTW, P.Method.LB_PC),
                                    (P.Method.TC_DTW, P.Method.LB_TI))
    for q in queries:
        ref = P.nn_search(q, cands, P.SearchParams(window=5, method="none"))
        out = P.nn_search(q, cands, params, advanced=adv)
        assert (out.best_index, out.best_distance) == (ref.best_index, ref.best_distance)


@pytest.mark.parametrize("method", ["lb_pc", "lb_mv"])
def test_lane_kernel_query_switches_are_attributed(P, method):
    """The R-row lane kernel with head batches switches queries many times
    per warp; with LB_PC pruning most entries, head batches are sparse and
    lanes pop queued pairs they did not start (a lane's query attribution
    must follow the pair: a stale one put completed DTWs on the wrong query,
    round-2 bug).  C4 shape, 16 queries x 100k candidates, three runs, every
    answer == the oracle."""
    from oracle import oracle as O
    from paper_2101_07731_b200.datasets import make_workload

    wl = make_workload("C4", n_candidates=100_000, n_queries=16)
    outs, _ = O.nn_search_batch(wl.queries.astype(np.float64), wl.candidates.astype(np.float64),
                                O.make_params(12, method), None, wl.dim_range)
    index = P.SearchIndex(wl.candidates, dtype="f32")
    assert index.dtw_kernel(_params(P, 12, method), None, 16).startswith("dtw_laner")
    for _ in range(3):
        res = index.search(wl.queries, _params(P, 12, method), dim_range=wl.dim_range)
        assert res.best_index.tolist() == [o.best_index for o in outs]
        assert res.best_distance.tolist() == [o.best_distance for o in outs]
