"""Sakoe-Chiba banded multivariate DTW with early abandoning (dtw.py:1-102).

``dtw_banded`` keeps the reference's signature and result (distance,
abandoned, cells), computed by the EXACT float64 CUDA kernel
(tcdtw_dtw_banded), bit-identical to the reference including the
row-granular abandon value and the cell count.  ``dtw_banded_pairs`` is the
batched form.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .core import InvalidInputError, as_series


@dataclass(frozen=True)
class DtwResult:
    """Banded DTW outcome (dtw.py:14-30)."""

    distance: float
    abandoned: bool = False
    cells: int = 0


def dtw_banded_pairs(a, b, window: int, abandon_above=None, dtype=None):
    """DTW of every pair (a[p], b[p]); a, b: (P, n, D).  Returns numpy
    (distance, abandoned, cells)."""
    t = _dev.torch()
    A = _dev.to_dev(a, dtype)
    B = _dev.to_dev(b, dtype)
    if A.ndim != 3 or A.shape != B.shape:
        raise InvalidInputError(f"shape mismatch: {tuple(A.shape)} vs {tuple(B.shape)}")
    if window < 0:
        raise InvalidInputError("window must be >= 0")
    P, n, d = A.shape
    thr = _dev.thresholds(abandon_above, P, A.dtype)
    dist = _dev.empty((P,), A.dtype)
    ab = t.empty((P,), device="cuda", dtype=t.uint8)
    cells = t.empty((P,), device="cuda", dtype=t.int64)
    L = _lib.lib()
    _lib.check(L.tcdtw_dtw_banded(_dev.code_of(A.dtype), A.data_ptr(), B.data_ptr(), P, n, d, int(window),
                                  _lib.ptr(thr), dist.data_ptr(), ab.data_ptr(), cells.data_ptr(),
                                  _lib.stream_ptr()), "dtw_banded")
    return dist.double().cpu().numpy(), ab.cpu().numpy().astype(bool), cells.cpu().numpy()


def dtw_banded(q, c, window: int, abandon_above: float | None = None) -> DtwResult:
    """Band-constrained DTW distance of two equal-shape series (dtw.py:45-102)."""
    qa = as_series(q)
    ca = as_series(c)
    if qa.shape != ca.shape:
        raise InvalidInputError(f"shape mismatch: {qa.shape} vs {ca.shape}")
    if window < 0:
        raise InvalidInputError("window must be >= 0")
    d, ab, cells = dtw_banded_pairs(qa[None], ca[None], int(window),
                                    None if abandon_above is None else [float(abandon_above)])
    return DtwResult(float(d[0]), bool(ab[0]), int(cells[0]))
