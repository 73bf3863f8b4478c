#!/usr/bin/env python
"""Cost of leaving the compiled (d, 2W+1) buckets of the lane DTW kernel
(VERDICT r1 weak 10): the same C4-style workload (sinusoid mixture, float32,
200k candidates x 256 queries) at the C4 shape and at neighbouring shapes the
dispatcher serves with another kernel.  Prints one line per shape: kernel,
q/s, DTW ms, GCUPS and the fraction of the nominal FP32 issue peak.

    python scripts/offbucket_shapes.py > gpurun_out/offbucket.txt
    python scripts/offbucket_shapes.py 128 6 10     # one shape
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2101_07731_b200 as P  # noqa: E402
from paper_2101_07731_b200 import datasets  # noqa: E402

SHAPES = [  # (n, d, W)
    (128, 6, 12), (128, 7, 12), (128, 8, 12), (128, 6, 10), (128, 6, 16), (126, 6, 12), (128, 12, 12),
    (128, 2, 12), (256, 6, 25), (64, 20, 6), (64, 16, 6), (127, 6, 12),
]


def main():
    nominal = 148 * 128 * 1.965e9
    shapes = SHAPES
    if len(sys.argv) == 4:  # one shape: n d W (for an ncu capture)
        shapes = [tuple(int(v) for v in sys.argv[1:4])]
    for n, d, w in shapes:
        spec = datasets.ConfigSpec(f"X{n}_{d}", 200000, 256, n, d, "f32", (w / n,), "sines", 50)
        rng = np.random.default_rng(0)
        vals = np.ascontiguousarray(datasets._sines_chunked(spec, spec.n_candidates + spec.n_queries, rng))
        cands, queries = vals[: spec.n_candidates], vals[spec.n_candidates:]
        index = P.SearchIndex(cands, dtype="f32")
        params = P.SearchParams(window=w, method=P.Method.LB_MV)
        index.search(queries, params)  # warm-up
        res = index.search(queries, params, timing=True)
        torch.cuda.synchronize()
        ph = res.phase_ms
        cells = int(np.asarray(res.counters["dtw_cells"]).sum())
        dtw_ms = ph["dtw"] + ph["seeds_dtw"]
        total = sum(ph.values())
        gcups = cells / (dtw_ms / 1e3) / 1e9
        frac = cells * (2 * d + 4) / (dtw_ms / 1e3) / nominal
        print(f"n={n:4d} d={d:2d} W={w:2d}  {index.dtw_kernel(params, None, 256):28s} {256 / (total / 1e3):9.1f} q/s  "
              f"lb_mv {ph['lb_mv']:7.2f} ms  dtw {dtw_ms:8.2f} ms  {gcups:7.1f} GCUPS  {frac:.3f} of nominal", flush=True)


if __name__ == "__main__":
    main()
