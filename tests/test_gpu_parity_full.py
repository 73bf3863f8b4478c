"""Config-level parity evidence: every query of C0-C3 (C1 at both windows;
the float64 configs through both the float32 filter and the all-float64
kernels) and 256 seeded random C4 queries (spread over all 10,000) searched
on the GPU and by the C oracle, compared
index for index and distance for distance (==).  A few minutes of oracle
work, so it only runs with TCDTW_FULL_PARITY=1:

    TCDTW_FULL_PARITY=1 python -m pytest tests/test_gpu_parity_full.py -m gpu -s

(its per-config lines are kept in profiles/r01_parity_full.log).
"""

import os
import time

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(os.environ.get("TCDTW_FULL_PARITY") != "1",
                                                  reason="set TCDTW_FULL_PARITY=1 (minutes of oracle work)")]


def test_full_parity():
    import paper_2101_07731_b200 as P
    from oracle import oracle as O
    from paper_2101_07731_b200.datasets import make_workload

    runs = [("C0", 0, None, "lb_mv", True), ("C0", 0, None, "lb_pc", True), ("C0", 0, None, "lb_mv", False),
            ("C1", 0, None, "lb_mv", None), ("C1", 1, None, "lb_mv", None), ("C2", 0, None, "lb_mv", None),
            ("C3", 0, None, "lb_mv", True), ("C3", 0, None, "lb_mv", False), ("C4", 0, 256, "lb_mv", None)]
    all_ok = True
    for cfg, wi, nq, method, flt in runs:
        wl = make_workload(cfg)
        w = wl.spec.windows()[wi]
        if nq is None:
            qs = wl.queries
        else:
            qs = wl.queries[np.sort(np.random.default_rng(7).choice(len(wl.queries), size=nq, replace=False))]
        t0 = time.perf_counter()
        res = P.SearchIndex(wl.candidates, dtype=wl.dtype, f32_filter=flt).search(
            qs, P.SearchParams(window=w, method=P.Method(method)), dim_range=wl.dim_range)
        t_gpu = time.perf_counter() - t0
        t0 = time.perf_counter()
        outs, used = O.nn_search_batch(qs.astype(np.float64), wl.candidates.astype(np.float64),
                                       O.make_params(w, method), None, wl.dim_range)
        t_cpu = time.perf_counter() - t0
        oi = np.array([o.best_index for o in outs])
        od = np.array([o.best_distance for o in outs])
        same_i = int((res.best_index == oi).sum())
        same_d = int((res.best_distance == od).sum())
        rel = float(np.max(np.abs(res.best_distance - od) / np.maximum(od, 1e-300)))
        ok = same_i == len(qs) and same_d == len(qs)
        all_ok &= ok
        mode = {True: " f32-filter", False: " exact-f64", None: ""}[flt]
        print(f"{cfg} W={w} {method} {wl.dtype}{mode}: {len(qs)} queries x {len(wl.candidates)} candidates; "
              f"indices equal {same_i}/{len(qs)}, distances equal (==) {same_d}/{len(qs)}, max rel diff {rel:.3g}; "
              f"GPU {t_gpu:.2f} s (incl. upload), oracle {t_cpu:.1f} s on {used} threads -> {'OK' if ok else 'MISMATCH'}",
              flush=True)
    print("ALL OK" if all_ok else "MISMATCHES FOUND")
    assert all_ok


