"""Host <-> device plumbing for the per-pair operators (torch = memory + streams)."""

from __future__ import annotations

import numpy as np

from . import _lib


def torch():
    import torch as _t

    return _t


def to_dev(a, dtype=None):
    """numpy / torch -> contiguous CUDA tensor (float64 unless dtype given)."""
    _lib.lib()  # raises NativeUnavailableError without the library or a device
    t = torch()
    tdtype = t.float64 if dtype is None else dtype
    if isinstance(a, t.Tensor):
        return a.to(device="cuda", dtype=tdtype).contiguous()
    return t.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).to(
        device="cuda", dtype=tdtype).contiguous()


def thresholds(abandon_above, count: int, tdtype):
    """Per-pair abandon thresholds or None (abandon_above=None)."""
    if abandon_above is None:
        return None
    t = torch()
    arr = np.asarray(abandon_above, dtype=np.float64).reshape(-1)
    if arr.size == 1 and count != 1:
        arr = np.full(count, float(arr[0]))
    arr = np.where(np.isnan(arr), np.inf, arr)
    return t.from_numpy(arr).to(device="cuda", dtype=tdtype)


def empty(shape, tdtype):
    return torch().empty(shape, device="cuda", dtype=tdtype)


def code_of(tdtype) -> int:
    return _lib.dtype_code(tdtype)
