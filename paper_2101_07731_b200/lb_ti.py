"""Triangle-inequality bound LB_TI and its variants (lb_ti.py:1-200).

Same names, variants, refresh semantics, one-sided 2^-46 safety pad and
abandon rule as the reference, computed by EXACT float64 CUDA kernels
(tcdtw_lb_ti, tcdtw_neighbor_steps, tcdtw_ti_advance).  The reference's
``trace`` test hook has no GPU equivalent and is rejected.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .core import BoundResult, InvalidInputError, TI_CODE, TiVariant, as_series

_PROP_SLACK = 2.0 ** -46


def neighbor_steps_batch(series, dtype=None):
    S = _dev.to_dev(series, dtype)
    ns, n, d = S.shape
    out = _dev.empty((ns, max(n - 1, 0)), S.dtype)
    if n > 1:
        _lib.check(_lib.lib().tcdtw_neighbor_steps(_dev.code_of(S.dtype), S.data_ptr(), ns, n, d, out.data_ptr(),
                                                   _lib.stream_ptr()), "neighbor_steps")
    return out


def neighbor_steps(series) -> np.ndarray:
    """Distances between consecutive points, shape (n-1,) (lb_ti.py:51-55)."""
    a = as_series(series)
    return neighbor_steps_batch(a[None])[0].cpu().numpy()


@dataclass(frozen=True, eq=False)
class NeighborDistances:
    """Adjacent-point distances, built once and reused (lb_ti.py:58-76)."""

    query_steps: np.ndarray
    candidate_steps: np.ndarray | None = None

    @classmethod
    def build(cls, q, c, variant: TiVariant = TiVariant.TIP_TOP) -> "NeighborDistances":
        needs_cand = TiVariant(variant) in (TiVariant.BASIC, TiVariant.TIP)
        return cls(query_steps=neighbor_steps(q), candidate_steps=neighbor_steps(c) if needs_cand else None)


def ti_advance_batch(lo, up, step, dtype=None):
    LO, UP, ST = _dev.to_dev(lo, dtype), _dev.to_dev(up, dtype), _dev.to_dev(step, dtype)
    olo, oup = _dev.empty(LO.shape, LO.dtype), _dev.empty(UP.shape, UP.dtype)
    _lib.check(_lib.lib().tcdtw_ti_advance(_dev.code_of(LO.dtype), LO.data_ptr(), UP.data_ptr(), ST.data_ptr(),
                                           LO.numel(), olo.data_ptr(), oup.data_ptr(), _lib.stream_ptr()),
               "ti_advance")
    return olo, oup


def ti_advance(lo: float, up: float, step: float) -> tuple[float, float]:
    """Advance one [L, U] interval across a query step (lb_ti.py:79-86)."""
    olo, oup = ti_advance_batch(np.array([lo]), np.array([up]), np.array([step]))
    return float(olo[0]), float(oup[0])


def ti_extend_top(lo: float, up: float, step: float) -> tuple[float, float]:
    """Interval of the window's new top slot (lb_ti.py:89-93)."""
    return ti_advance(lo, up, step)


def lb_ti_pairs(q, c, window: int, variant=TiVariant.TIP_TOP, refresh_period: int = 5, query_steps=None,
                cand_steps=None, abandon_above=None, dtype=None):
    Q, C = _dev.to_dev(q, dtype), _dev.to_dev(c, dtype)
    if Q.shape != C.shape or Q.ndim != 3:
        raise InvalidInputError(f"shape mismatch: {tuple(Q.shape)} vs {tuple(C.shape)}")
    variant = TiVariant(variant)
    if refresh_period < 1:
        raise InvalidInputError("refresh_period must be >= 1")
    if window < 0:
        raise InvalidInputError("window must be >= 0")
    P, n, d = Q.shape
    qs = None if query_steps is None else _dev.to_dev(query_steps, Q.dtype)
    cs = None if cand_steps is None else _dev.to_dev(cand_steps, Q.dtype)
    t = _dev.torch()
    thr = _dev.thresholds(abandon_above, P, Q.dtype)
    val = _dev.empty((P,), Q.dtype)
    ab = t.empty((P,), device="cuda", dtype=t.uint8)
    _lib.check(_lib.lib().tcdtw_lb_ti(_dev.code_of(Q.dtype), Q.data_ptr(), C.data_ptr(), P, n, d, int(window),
                                      TI_CODE[variant], int(refresh_period), _lib.ptr(qs), _lib.ptr(cs),
                                      _lib.ptr(thr), val.data_ptr(), ab.data_ptr(), _lib.stream_ptr()), "lb_ti")
    return val.double().cpu().numpy(), ab.cpu().numpy().astype(bool)


def lb_ti(q, c, window: int, variant: TiVariant = TiVariant.TIP_TOP, refresh_period: int = 5,
          neighbor: NeighborDistances | None = None, abandon_above: float | None = None,
          trace: list | None = None) -> BoundResult:
    """Triangle-inequality lower bound of the banded DTW distance (lb_ti.py:96-200)."""
    qa = as_series(q)
    ca = as_series(c)
    if qa.shape != ca.shape:
        raise InvalidInputError(f"shape mismatch: {qa.shape} vs {ca.shape}")
    variant = TiVariant(variant)
    if refresh_period < 1:
        raise InvalidInputError("refresh_period must be >= 1")
    if window < 0:
        raise InvalidInputError("window must be >= 0")
    if trace is not None:
        raise InvalidInputError("the lb_ti trace test hook is not available on the GPU path")
    n = qa.shape[0]
    qs = cs = None
    if neighbor is not None and n > 1:
        qs = np.asarray(neighbor.query_steps, dtype=np.float64)[None]
        if neighbor.candidate_steps is not None:
            cs = np.asarray(neighbor.candidate_steps, dtype=np.float64)[None]
    v, ab = lb_ti_pairs(qa[None], ca[None], window, variant, refresh_period, qs, cs,
                        None if abandon_above is None else [float(abandon_above)])
    return BoundResult(float(v[0]), bool(ab[0]))
