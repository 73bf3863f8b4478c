"""Step-by-step search on a tiny problem (debug aid)."""
import faulthandler
import sys

faulthandler.enable()
sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2101_07731_b200 as P
from paper_2101_07731_b200 import _lib

rng = np.random.default_rng(0)
cands = np.cumsum(rng.normal(size=(25, 24, 3)), axis=1)
q = np.cumsum(rng.normal(size=(24, 3)), axis=0)
for dtype in ("f64", "f32"):
    for method in ("none", "lb_mv", "lb_pc", "lb_ti", "lb_ad"):
        print("==", dtype, method, flush=True)
        idx = P.SearchIndex(cands, dtype=dtype)
        params = P.SearchParams(window=5, method=method)
        Q = idx.prepare_queries(q[None])
        print("prepared", flush=True)
        try:
            st = idx.seed_phase(Q, params)
        except BaseException as e:
            print("EXC", repr(e), flush=True)
            raise
        torch.cuda.synchronize()
        print("seeded", st["dbest"].cpu().numpy(), flush=True)
        bi, bd, ctr = idx.finish_phase(st)
        torch.cuda.synchronize()
        print("finished", bi.cpu().numpy(), bd.cpu().numpy(), ctr.cpu().numpy(), flush=True)
        from oracle import oracle as O
        outs, _ = O.nn_search_batch(q[None].astype(np.float32 if dtype == "f32" else np.float64).astype(np.float64),
                                    cands.astype(np.float32 if dtype == "f32" else np.float64).astype(np.float64),
                                    O.make_params(5, method), None, None)
        print("oracle", outs[0].best_index, outs[0].best_distance, flush=True)
print("ALL OK")
