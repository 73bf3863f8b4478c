import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2101_07731_b200 as P
from paper_2101_07731_b200.datasets import make_workload
wl = make_workload("C3", n_candidates=64, n_queries=2)
idx = P.SearchIndex(wl.candidates, dtype="f64")
res = idx.search(wl.queries, P.SearchParams(window=102, method="lb_mv"))
print(res.best_index, res.best_distance)
