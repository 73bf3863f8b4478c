"""Config-level parity evidence: every query of C0-C3 (C1 at both windows)
and a 64-query C4 sample searched on the GPU and by the C oracle, compared
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

    runs = [("C0", 0, None, "lb_mv"), ("C0", 0, None, "lb_pc"), ("C1", 0, None, "lb_mv"), ("C1", 1, None, "lb_mv"),
            ("C2", 0, None, "lb_mv"), ("C3", 0, None, "lb_mv"), ("C4", 0, 64, "lb_mv")]
    all_ok = True
    for cfg, wi, nq, method in runs:
        wl = make_workload(cfg)
        w = wl.spec.windows()[wi]
        qs = wl.queries if nq is None else wl.queries[:nq]
        t0 = time.perf_counter()
        res = P.SearchIndex(wl.candidates, dtype=wl.dtype).search(
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
        print(f"{cfg} W={w} {method} {wl.dtype}: {len(qs)} queries x {len(wl.candidates)} candidates; "
              f"indices equal {same_i}/{len(qs)}, distances equal (==) {same_d}/{len(qs)}, max rel diff {rel:.3g}; "
              f"GPU {t_gpu:.2f} s (incl. upload), oracle {t_cpu:.1f} s on {used} threads -> {'OK' if ok else 'MISMATCH'}",
              flush=True)
    print("ALL OK" if all_ok else "MISMATCHES FOUND")
    assert all_ok


