import numpy as np, sys
sys.path.insert(0, '.')
import paper_2101_07731_b200 as P
from oracle import oracle as O
from paper_2101_07731_b200.datasets import make_workload
wl = make_workload("C4"); w = 12
qsel = wl.queries[:4]
outs, _ = O.nn_search_batch(qsel.astype(np.float64), wl.candidates.astype(np.float64), O.make_params(w, "lb_pc"), None, wl.dim_range)
print("oracle", [(o.best_index, o.best_distance) for o in outs], flush=True)
index = P.SearchIndex(wl.candidates, dtype="f32")
for casc in (True, False):
    index.cascade = casc
    for rev in (False, True, False, True):
        r = index.search(qsel, P.SearchParams(window=w, method="lb_pc"), dim_range=wl.dim_range, reverse_pc=rev)
        ok = [int(r.best_index[i]) == outs[i].best_index for i in range(4)]
        print("casc", casc, "rev", rev, list(zip(r.best_index.tolist(), r.best_distance.tolist())), ok, r.counters["advanced_lb_evals"].tolist(), r.counters["dtw_computed"].tolist(), flush=True)
for nq in (1, 2, 8):
    r = index.search(wl.queries[:nq], P.SearchParams(window=w, method="lb_mv"))
    print("lb_mv", nq, r.best_index.tolist()[:4], flush=True)
