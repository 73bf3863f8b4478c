"""Loader for the reference-generated fixtures in tests/golden/*.npz."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def load_cases(name: str) -> tuple:
    z = np.load(GOLDEN / f"{name}.npz", allow_pickle=False)
    scalars = json.loads(str(z["scalars"]))
    cases = []
    for i, sc in enumerate(scalars):
        case = dict(sc)
        prefix = f"c{i}_"
        for k in z.files:
            if k.startswith(prefix):
                case[k[len(prefix):]] = z[k]
        cases.append(case)
    return tuple(cases)


def thr_or_none(x):
    return None if x is None or (isinstance(x, float) and np.isnan(x)) else float(x)


def dr_or_none(a):
    a = np.asarray(a, dtype=np.float64)
    return None if np.all(np.isnan(a)) else a
