"""Envelope bound LB_MV and all-distances bound LB_AD (lb_mv.py:1-128).

Same names and results as the reference; computed by EXACT float64 CUDA
kernels (tcdtw_build_envelope, tcdtw_lb_mv, tcdtw_lb_ad).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .core import BoundResult, InvalidInputError, as_series


@dataclass(frozen=True, eq=False)
class Envelope:
    """Windowed max/min tube of a series (lb_mv.py:22-41)."""

    upper: np.ndarray
    lower: np.ndarray
    window: int

    @property
    def n(self) -> int:
        return self.upper.shape[0]

    @property
    def dims(self) -> int:
        return self.upper.shape[1]


def build_envelopes(series, window: int, dtype=None):
    """Envelopes of a stack of series (S, n, D) -> (upper, lower) tensors."""
    S = _dev.to_dev(series, dtype)
    if S.ndim != 3:
        raise InvalidInputError(f"series stack must be (S, n, D), got {tuple(S.shape)}")
    if window < 0:
        raise InvalidInputError("window must be >= 0")
    ns, n, d = S.shape
    up = _dev.empty(S.shape, S.dtype)
    lo = _dev.empty(S.shape, S.dtype)
    _lib.check(_lib.lib().tcdtw_build_envelope(_dev.code_of(S.dtype), S.data_ptr(), ns, n, d, int(window),
                                               up.data_ptr(), lo.data_ptr(), _lib.stream_ptr()), "build_envelope")
    return up, lo


def build_envelope(q, window: int) -> Envelope:
    """Windowed max/min envelope of one series (lb_mv.py:74-88)."""
    qa = as_series(q)
    if window < 0:
        raise InvalidInputError("window must be >= 0")
    n = qa.shape[0]
    w = min(int(window), n - 1)
    up, lo = build_envelopes(qa[None], w)
    return Envelope(upper=up[0].cpu().numpy(), lower=lo[0].cpu().numpy(), window=w)


def _bound_call(fn_name, args, P, tdtype, abandon_above, what):
    t = _dev.torch()
    thr = _dev.thresholds(abandon_above, P, tdtype)
    val = _dev.empty((P,), tdtype)
    ab = t.empty((P,), device="cuda", dtype=t.uint8)
    fn = getattr(_lib.lib(), fn_name)
    _lib.check(fn(*args, _lib.ptr(thr), val.data_ptr(), ab.data_ptr(), _lib.stream_ptr()), what)
    return val.double().cpu().numpy(), ab.cpu().numpy().astype(bool)


def lb_mv_pairs(c, upper, lower, abandon_above=None, dtype=None):
    """LB_MV of every pair (c[p], envelope p); arrays (P, n, D)."""
    C, U, Lo = _dev.to_dev(c, dtype), _dev.to_dev(upper, dtype), _dev.to_dev(lower, dtype)
    if C.shape != U.shape or C.shape != Lo.shape or C.ndim != 3:
        raise InvalidInputError(f"shape mismatch: {tuple(C.shape)} vs {tuple(U.shape)}")
    P, n, d = C.shape
    return _bound_call("tcdtw_lb_mv", (_dev.code_of(C.dtype), C.data_ptr(), U.data_ptr(), Lo.data_ptr(), P, n, d),
                       P, C.dtype, abandon_above, "lb_mv")


def lb_mv(c, env: Envelope, abandon_above: float | None = None) -> BoundResult:
    """Envelope lower bound of the banded DTW distance (lb_mv.py:98-107)."""
    ca = as_series(c)
    if ca.shape != env.upper.shape:
        raise InvalidInputError(f"shape mismatch: {ca.shape} vs {env.upper.shape}")
    v, ab = lb_mv_pairs(ca[None], np.asarray(env.upper)[None], np.asarray(env.lower)[None],
                        None if abandon_above is None else [float(abandon_above)])
    return BoundResult(float(v[0]), bool(ab[0]))


def lb_ad_pairs(q, c, window: int, abandon_above=None, dtype=None):
    Q, C = _dev.to_dev(q, dtype), _dev.to_dev(c, dtype)
    if Q.shape != C.shape or Q.ndim != 3:
        raise InvalidInputError(f"shape mismatch: {tuple(Q.shape)} vs {tuple(C.shape)}")
    if window < 0:
        raise InvalidInputError("window must be >= 0")
    P, n, d = Q.shape
    return _bound_call("tcdtw_lb_ad", (_dev.code_of(Q.dtype), Q.data_ptr(), C.data_ptr(), P, n, d, int(window)),
                       P, Q.dtype, abandon_above, "lb_ad")


def lb_ad(q, c, window: int, abandon_above: float | None = None) -> BoundResult:
    """All-distances lower bound (lb_mv.py:110-128)."""
    qa = as_series(q)
    ca = as_series(c)
    if qa.shape != ca.shape:
        raise InvalidInputError(f"shape mismatch: {qa.shape} vs {ca.shape}")
    v, ab = lb_ad_pairs(qa[None], ca[None], window, None if abandon_above is None else [float(abandon_above)])
    return BoundResult(float(v[0]), bool(ab[0]))
