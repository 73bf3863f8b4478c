import sys, subprocess, json
sys.path.insert(0, ".")
cases = [("f32", 256, 5, 51), ("f64", 256, 5, 51), ("f64", 256, 8, 51), ("f32", 256, 8, 51),
         ("f64", 1024, 5, 102), ("f32", 1024, 8, 102), ("f64", 512, 8, 102), ("f64", 1024, 8, 40), ("f64", 1024, 8, 102)]
code = r'''
import sys; sys.path.insert(0, ".")
import numpy as np, paper_2101_07731_b200 as P
from oracle import oracle as O
dt, n, d, w = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
rng = np.random.default_rng(0)
C = np.cumsum(rng.normal(size=(40, n, d)), axis=1); Qs = np.cumsum(rng.normal(size=(2, n, d)), axis=1)
if dt == "f32": C, Qs = C.astype(np.float32), Qs.astype(np.float32)
res = P.SearchIndex(C, dtype=dt).search(Qs, P.SearchParams(window=w, method="lb_mv"))
outs, _ = O.nn_search_batch(Qs.astype(np.float64), C.astype(np.float64), O.make_params(w, "lb_mv"), None, None)
print("OK", res.best_index.tolist(), [o.best_index for o in outs], res.best_distance.tolist() == [o.best_distance for o in outs])
'''
for c in cases:
    r = subprocess.run([sys.executable, "-c", code, *map(str, c)], capture_output=True, text=True, timeout=300)
    print(c, (r.stdout.strip() or r.stderr.strip().splitlines()[-1])[:200], flush=True)
