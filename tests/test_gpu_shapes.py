"""Search parity over a spread of shapes, so that every DTW kernel the
dispatcher can pick (R-row lane kernel for its compiled shapes and with a
run-time band, two-row lane
kernel, thread-per-pair, compile-time-d wavefront, generic wavefront,
few-pairs path) is checked against the oracle, in float32 and float64."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = [  # (n, d, W)
    (1, 3, 0), (2, 1, 1), (7, 2, 3), (16, 4, 6), (33, 7, 5), (64, 20, 6), (64, 6, 12), (100, 9, 10),
    (128, 6, 12), (128, 5, 51), (128, 3, 6), (128, 8, 12), (200, 12, 40), (64, 32, 3), (96, 16, 30),
    (256, 5, 12), (130, 6, 12), (48, 24, 48),
    # run-time-band lane kernel (no compiled (d, 2W+1) bucket): even W -> 4 rows per step, odd W -> 2
    (128, 6, 10), (128, 6, 16), (128, 6, 11), (64, 20, 4), (256, 6, 24), (96, 4, 7), (128, 8, 30), (64, 3, 8),
    (100, 5, 6), (128, 4, 4), (128, 6, 2),
    # dimension counts between the compiled ones: zero-padded on the fly to the next instantiation
    (128, 7, 12), (128, 2, 12), (128, 1, 6), (64, 16, 6), (64, 13, 6), (128, 12, 12), (64, 9, 5), (128, 7, 10),
    (64, 19, 6), (256, 6, 25), (128, 3, 5), (128, 7, 13), (64, 8, 9),
    # n % rows-per-step != 0: the last rows run one at a time after the last full step
    (127, 6, 12), (129, 5, 10), (131, 8, 13), (63, 20, 6), (101, 3, 7), (126, 6, 12), (9, 4, 4), (65, 12, 6),
]


@pytest.mark.parametrize("n,d,w", SHAPES)
@pytest.mark.parametrize("dtype", ["f32", "f64", "f64-exact"])
def test_search_shapes(n, d, w, dtype):
    import paper_2101_07731_b200 as P
    from oracle import oracle as O

    rng = np.random.default_rng(n * 1000 + d * 10 + w)
    N, Q = 900, 5
    X = np.cumsum(rng.normal(size=(N + Q, n, d)), axis=1)
    X = (X - X.reshape(-1, d).mean(0)) / (X.reshape(-1, d).std(0) + 1e-12)
    np_t = np.float32 if dtype == "f32" else np.float64
    X = X.astype(np_t)
    cands, qs = X[:N], X[N:]
    # f64: the float32 filter on float64 data (default); f64-exact: every kernel in float64
    index = P.SearchIndex(cands, dtype=dtype[:3], f32_filter=None if dtype != "f64-exact" else False)
    res = index.search(qs, P.SearchParams(window=w, method=P.Method.LB_MV))
    outs, _ = O.nn_search_batch(qs.astype(np.float64), cands.astype(np.float64), O.make_params(w, "lb_mv"), None,
                                None)
    for i, o in enumerate(outs):
        assert res.best_index[i] == o.best_index, (n, d, w, dtype, i)
        assert res.best_distance[i] == o.best_distance, (n, d, w, dtype, i)
    c = res.counters
    assert np.all(c["dtw_computed"] + c["dtw_skipped"] == N)


@pytest.mark.parametrize("n,d,w,dtype", [(4096, 8, 409, "f64"), (4096, 8, 409, "f64-exact"), (4096, 6, 409, "f32"),
                                          (2048, 3, 1000, "f64"), (2048, 3, 1000, "f64-exact")])
def test_long_series(n, d, w, dtype):
    """Series whose staged query rows exceed shared memory: the wavefront
    reads them through L1; wide bands: the float64 re-score's band rows."""
    import paper_2101_07731_b200 as P
    from oracle import oracle as O

    rng = np.random.default_rng(n + d + w)
    N, Q = 40, 2
    X = np.cumsum(rng.normal(size=(N + Q, n, d)), axis=1)
    X = ((X - X.reshape(-1, d).mean(0)) / X.reshape(-1, d).std(0)).astype(np.float32 if dtype == "f32" else np.float64)
    index = P.SearchIndex(X[:N], dtype=dtype[:3], f32_filter=None if dtype != "f64-exact" else False)
    res = index.search(X[N:], P.SearchParams(window=w, method=P.Method.LB_MV))
    outs, _ = O.nn_search_batch(X[N:].astype(np.float64), X[:N].astype(np.float64), O.make_params(w, "lb_mv"),
                                None, None)
    assert list(res.best_index) == [o.best_index for o in outs]
    assert list(res.best_distance) == [o.best_distance for o in outs]
