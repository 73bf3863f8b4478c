"""How much DTW work is due to d_best converging late?  C4 at Q queries:
run 1 normal; run 2 with d_best preset (between the phases) to run 1's answers."""
import sys, json
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2101_07731_b200 as P
from paper_2101_07731_b200.datasets import make_workload

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
wl = make_workload("C4", n_queries=nq)
w = wl.spec.windows()[0]
idx = P.SearchIndex(wl.candidates, dtype=wl.dtype)
prm = P.SearchParams(window=w, method="lb_mv")
Q = wl.queries
seeded = {}
def grab(d):
    seeded["d"] = d.clone()
for rep in range(2):
    r1 = idx.search(Q, prm, timing=True, dbest_hook=grab)
print("normal", json.dumps({k: round(v, 1) for k, v in r1.phase_ms.items()}), "cells", int(r1.counters["dtw_cells"].sum()),
      "issued", int(r1.counters["cells_issued"].sum()), "computed", int(r1.counters["dtw_computed"].sum()))
true = torch.from_numpy(r1.best_distance).cuda()
ratio = (seeded["d"].double() / true).cpu().numpy()
print("seed d_best / final: mean %.4f median %.4f p90 %.4f max %.4f" % (ratio.mean(), np.median(ratio), np.quantile(ratio, .9), ratio.max()))
def preset(d):
    d.copy_(torch.minimum(d.double(), true * (1 + 1e-5)).to(d.dtype))
for rep in range(2):
    r2 = idx.search(Q, prm, timing=True, dbest_hook=preset)
print("oracle", json.dumps({k: round(v, 1) for k, v in r2.phase_ms.items()}), "cells", int(r2.counters["dtw_cells"].sum()),
      "issued", int(r2.counters["cells_issued"].sum()), "computed", int(r2.counters["dtw_computed"].sum()))
assert (r2.best_index == r1.best_index).all() and (r2.best_distance == r1.best_distance).all()
for f in (1.02, 1.05, 1.10):
    def pre(d, f=f):
        d.copy_(torch.minimum(d.double(), true * f).to(d.dtype))
    r3 = idx.search(Q, prm, timing=True, dbest_hook=pre)
    print("preset x%.2f dtw_ms %.1f cells %d" % (f, r3.phase_ms.get("dtw", 0), int(r3.counters["dtw_cells"].sum())))
