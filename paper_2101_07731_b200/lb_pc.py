"""Point-clustering bound LB_PC (lb_pc.py:1-280).

Box building (quantisation into <= max_boxes tight boxes per expanded
window) and the bound itself run in CUDA (tcdtw_build_box_sets,
tcdtw_lb_pc); cell assignment is float64 with IEEE division, so the boxes
equal the reference's bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dev, _lib
from .core import BoundResult, InvalidInputError, as_series


@dataclass(frozen=True, eq=False)
class BoundingBox:
    lo: np.ndarray
    hi: np.ndarray


@dataclass(frozen=True, eq=False)
class BoxSet:
    """Boxes of one (expanded) window (lb_pc.py:34-53)."""

    los: np.ndarray
    his: np.ndarray
    window_span: tuple[int, int] | None = None

    @property
    def num_boxes(self) -> int:
        return self.los.shape[0]

    @property
    def boxes(self) -> list[BoundingBox]:
        return [BoundingBox(self.los[b], self.his[b]) for b in range(self.num_boxes)]


class BoxGrouping:
    """Box sets of every expanded window of one query (lb_pc.py:119-150)."""

    def __init__(self, group_width: int, window: int, n: int, pad_lo: np.ndarray, pad_hi: np.ndarray,
                 box_counts: np.ndarray, spans: list[tuple[int, int]]):
        self.group_width = group_width
        self.window = window
        self.n = n
        self.pad_lo = pad_lo
        self.pad_hi = pad_hi
        self.box_counts = box_counts
        self.spans = spans
        self._sets = None

    @property
    def sets(self) -> tuple[BoxSet, ...]:
        if self._sets is None:
            self._sets = tuple(BoxSet(self.pad_lo[g, : self.box_counts[g]].copy(),
                                      self.pad_hi[g, : self.box_counts[g]].copy(), self.spans[g])
                               for g in range(len(self.spans)))
        return self._sets

    def set_for_index(self, i: int) -> BoxSet:
        return self.sets[i // self.group_width]


def num_groups(n: int, group_width: int) -> int:
    return (n - 1) // group_width + 1


def spans_of(n: int, window: int, group_width: int) -> list[tuple[int, int]]:
    w = min(int(window), n - 1)
    return [(max(0, g * group_width - w), min(n - 1, g * group_width + w + group_width - 1))
            for g in range(num_groups(n, group_width))]


def build_box_sets_batch(series, window: int, group_width: int, levels: int, max_boxes: int,
                         min_cell_frac: float, dim_range=None, dtype=None):
    """Box sets of a stack of series -> (lo, hi, counts) device tensors with
    shapes (S, G, max_boxes, D) and (S, G)."""
    t = _dev.torch()
    S = _dev.to_dev(series, dtype)
    if window < 0:
        raise InvalidInputError("window must be >= 0")
    if group_width < 1 or levels < 1 or max_boxes < 1:
        raise InvalidInputError("group_width, levels and max_boxes must be >= 1")
    ns, n, d = S.shape
    G = num_groups(n, group_width)
    lo = _dev.empty((ns, G, max_boxes, d), S.dtype)
    hi = _dev.empty((ns, G, max_boxes, d), S.dtype)
    cnt = t.empty((ns, G), device="cuda", dtype=t.int32)
    dr = None if dim_range is None else _dev.to_dev(np.asarray(dim_range, dtype=np.float64).reshape(-1), S.dtype)
    _lib.check(_lib.lib().tcdtw_build_box_sets(_dev.code_of(S.dtype), S.data_ptr(), ns, n, d, int(window),
                                               int(group_width), int(levels), int(max_boxes), float(min_cell_frac),
                                               _lib.ptr(dr), lo.data_ptr(), hi.data_ptr(), cnt.data_ptr(),
                                               _lib.stream_ptr()), "build_box_sets")
    return lo, hi, cnt


def quantize_cluster(points, levels: int, max_boxes: int, min_cell_frac: float,
                     dim_range: np.ndarray | None = None, window_span: tuple[int, int] | None = None) -> BoxSet:
    """Grid-quantise points into <= max_boxes tight boxes (lb_pc.py:56-116):
    the single-window case of the batched builder."""
    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim == 1:
        pts = pts[:, None]
    if pts.size == 0:
        raise InvalidInputError("cannot cluster an empty point list")
    if levels < 1 or max_boxes < 1:
        raise InvalidInputError("levels and max_boxes must be >= 1")
    m = pts.shape[0]
    lo, hi, cnt = build_box_sets_batch(pts[None], m - 1, m, levels, max_boxes, min_cell_frac, dim_range)
    k = int(cnt[0, 0])
    return BoxSet(lo[0, 0, :k].cpu().numpy(), hi[0, 0, :k].cpu().numpy(), window_span)


def build_box_sets(q, window: int, group_width: int, levels: int, max_boxes: int, min_cell_frac: float,
                   dim_range: np.ndarray | None = None) -> BoxGrouping:
    """Cluster a query's expanded windows into box sets (lb_pc.py:239-261)."""
    qa = as_series(q)
    if window < 0:
        raise InvalidInputError("window must be >= 0")
    if group_width < 1 or levels < 1 or max_boxes < 1:
        raise InvalidInputError("group_width, levels and max_boxes must be >= 1")
    n = qa.shape[0]
    w = min(int(window), n - 1)
    lo, hi, cnt = build_box_sets_batch(qa[None], w, group_width, levels, max_boxes, min_cell_frac, dim_range)
    counts = cnt[0].cpu().numpy().astype(np.int64)
    kmax = int(counts.max())
    return BoxGrouping(group_width, w, n, lo[0, :, :kmax].cpu().numpy(), hi[0, :, :kmax].cpu().numpy(), counts,
                       spans_of(n, w, group_width))


def lb_pc_pairs(c, box_lo, box_hi, group_width: int, abandon_above=None, dtype=None):
    """LB_PC of every pair (c[p], box set p): c (P, n, D), boxes (P, G, K, D)."""
    t = _dev.torch()
    C = _dev.to_dev(c, dtype)
    BL, BH = _dev.to_dev(box_lo, C.dtype), _dev.to_dev(box_hi, C.dtype)
    P, n, d = C.shape
    G, K = BL.shape[1], BL.shape[2]
    thr = _dev.thresholds(abandon_above, P, C.dtype)
    val = _dev.empty((P,), C.dtype)
    ab = t.empty((P,), device="cuda", dtype=t.uint8)
    _lib.check(_lib.lib().tcdtw_lb_pc(_dev.code_of(C.dtype), C.data_ptr(), BL.data_ptr(), BH.data_ptr(), P, n, d,
                                      G, K, int(group_width), _lib.ptr(thr), val.data_ptr(), ab.data_ptr(),
                                      _lib.stream_ptr()), "lb_pc")
    return val.double().cpu().numpy(), ab.cpu().numpy().astype(bool)


def lb_pc(c, grouping: BoxGrouping, abandon_above: float | None = None) -> BoundResult:
    """Clustering lower bound (lb_pc.py:264-280)."""
    ca = as_series(c)
    if ca.shape[0] != grouping.n:
        raise InvalidInputError(f"length mismatch: {ca.shape[0]} vs {grouping.n}")
    if ca.shape[1] != grouping.pad_lo.shape[2]:
        raise InvalidInputError(f"dimension mismatch: {ca.shape[1]} vs {grouping.pad_lo.shape[2]}")
    v, ab = lb_pc_pairs(ca[None], np.asarray(grouping.pad_lo)[None], np.asarray(grouping.pad_hi)[None],
                        grouping.group_width, None if abandon_above is None else [float(abandon_above)])
    return BoundResult(float(v[0]), bool(ab[0]))
