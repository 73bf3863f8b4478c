"""ctypes binding of libtcdtw.so (the C ABI declared in include/tcdtw.h).

There is no fallback: if the library or a CUDA device is missing, every
operator raises ``NativeUnavailableError`` instead of computing anything on
the CPU.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libtcdtw.so"

TCDTW_OK, TCDTW_INVALID_INPUT, TCDTW_CUDA_ERROR, TCDTW_WORKSPACE_TOO_SMALL, TCDTW_NOT_SUPPORTED = range(5)
F32, F64 = 0, 1
PHASES = ("prep", "lb_mv", "seeds_topk", "seeds_dtw", "compact", "advanced", "dtw", "finalize")
COUNTERS = ("dtw_computed", "dtw_skipped", "lb_mv_evals", "advanced_lb_evals", "abandon_count",
            "dtw_cells", "finalists", "survivors", "cells_issued")
FLAG_TIMING = 1
FLAG_REVERSE_LB = 2
FLAG_F32_FILTER = 4
FLAG_DEBUG_SYNC = 8
FLAG_FROZEN_THRESHOLDS = 16
FLAG_NO_CASCADE = 32
FLAG_REVERSE_PC = 64

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


class NativeUnavailableError(RuntimeError):
    """The CUDA library or device needed by the B200 path is missing."""


class SearchDesc(ctypes.Structure):
    """tcdtw_search_desc (include/tcdtw.h)."""

    _fields_ = [
        ("dtype", _i32), ("n", _i32), ("dims", _i32), ("window", _i32), ("method", _i32),
        ("advanced", _i32), ("refresh_period", _i32), ("quant_levels", _i32), ("max_boxes", _i32),
        ("group_width", _i32), ("trigger_ti", ctypes.c_double), ("trigger_pc", ctypes.c_double),
        ("min_cell_frac", ctypes.c_double), ("n_queries", _i64), ("n_candidates", _i64),
        ("candidate_base", _i64), ("seeds", _i32), ("flags", _i32),
        ("phase_ms", ctypes.POINTER(ctypes.c_float)), ("cand_upper", _vp), ("cand_lower", _vp),
        ("done_cap", _i64), ("cand_planar", _vp), ("cand_box_lo", _vp), ("cand_box_hi", _vp),
    ]


class ParseInfo(ctypes.Structure):
    """tcdtw_parse_info (include/tcdtw.h)."""

    _fields_ = [(f, _i64) for f in ("num_series", "length", "dims", "line", "tok_off", "tok_len", "expected", "found",
                                    "name_off", "name_len")] + [("error", _i32), ("reserved", _i32)]


_SIGS = {
    "tcdtw_strerror": ([ctypes.c_int], ctypes.c_char_p),
    "tcdtw_abi_version": ([], ctypes.c_int),
    "tcdtw_launch_count": ([], ctypes.c_ulonglong),
    "tcdtw_dtw_banded": ([ctypes.c_int, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp], ctypes.c_int),
    "tcdtw_build_envelope": ([ctypes.c_int, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp], ctypes.c_int),
    "tcdtw_lb_mv": ([ctypes.c_int, _vp, _vp, _vp, _i64, _i32, _i32, _vp, _vp, _vp, _vp], ctypes.c_int),
    "tcdtw_lb_ad": ([ctypes.c_int, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp], ctypes.c_int),
    "tcdtw_neighbor_steps": ([ctypes.c_int, _vp, _i64, _i32, _i32, _vp, _vp], ctypes.c_int),
    "tcdtw_ti_advance": ([ctypes.c_int, _vp, _vp, _vp, _i64, _vp, _vp, _vp], ctypes.c_int),
    "tcdtw_lb_ti": ([ctypes.c_int, _vp, _vp, _i64, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp],
                    ctypes.c_int),
    "tcdtw_build_box_sets": ([ctypes.c_int, _vp, _i64, _i32, _i32, _i32, _i32, _i32, _i32, ctypes.c_double, _vp,
                              _vp, _vp, _vp, _vp], ctypes.c_int),
    "tcdtw_lb_pc": ([ctypes.c_int, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp],
                    ctypes.c_int),
    "tcdtw_parse_text": ([_i32, ctypes.c_char_p, ctypes.c_size_t, _vp, _i64, ctypes.POINTER(ParseInfo)], ctypes.c_int),
    "tcdtw_normalize_workspace_size": ([_i64, _i32, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "tcdtw_normalize": ([_vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp], ctypes.c_int),
    "tcdtw_search_workspace_size": ([ctypes.POINTER(SearchDesc), ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "tcdtw_search_seed": ([ctypes.POINTER(SearchDesc), _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp, _vp], ctypes.c_int),
    "tcdtw_search_finish": ([ctypes.POINTER(SearchDesc), _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp, _vp, _vp, _vp,
                             _vp], ctypes.c_int),
    "tcdtw_nn_search": ([ctypes.POINTER(SearchDesc), _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp, _vp, _vp, _vp],
                        ctypes.c_int),
    "tcdtw_planar_bytes": ([ctypes.c_int, _i64, _i32, _i32], ctypes.c_size_t),
    "tcdtw_planarize": ([ctypes.c_int, _vp, _i64, _i32, _i32, _vp, _vp], ctypes.c_int),
    "tcdtw_shard_combine": ([_vp, _i32, _i64, _vp, _vp, _vp], ctypes.c_int),
    "tcdtw_lb_mv_matrix": ([ctypes.c_int, _vp, _vp, _vp, _i64, _i64, _i32, _i32, _vp, _vp], ctypes.c_int),
    "tcdtw_dtw_kernel_name": ([ctypes.POINTER(SearchDesc)], ctypes.c_char_p),
    "tcdtw_alu_probe": ([ctypes.c_int, _i32, _i32, _vp, ctypes.POINTER(ctypes.c_double), _vp], ctypes.c_int),
}

EXPORTED = tuple(_SIGS)

_lib = None


def build(force: bool = False) -> Path:
    """Compile libtcdtw.so in-tree (nvcc, -gencode arch=compute_100a,code=sm_100a)."""
    jobs = str(max(1, min(8, os.cpu_count() or 1)))
    args = ["make", "-s", "-j", jobs, "-C", str(_PKG / "csrc")]
    if force:
        subprocess.run(["make", "-s", "-C", str(_PKG / "csrc"), "clean"], check=True)
    subprocess.run(args, check=True)
    return LIB_PATH


def load_library():
    """dlopen libtcdtw.so and declare every C-ABI signature (no GPU needed)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeUnavailableError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(str(LIB_PATH))
        for name, (argtypes, restype) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = argtypes
            fn.restype = restype
        _lib = L
    return _lib


def lib():
    """The library, after checking that a CUDA device is usable."""
    L = load_library()
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailableError("no CUDA device: the TC-DTW B200 path has no CPU fallback")
    return L


class TcdtwError(RuntimeError):
    pass


def check(status: int, what: str = "") -> None:
    if status == TCDTW_OK:
        return
    msg = load_library().tcdtw_strerror(status).decode()
    if status == TCDTW_INVALID_INPUT:
        from .core import InvalidInputError

        raise InvalidInputError(f"{what}: {msg}")
    raise TcdtwError(f"{what}: {msg} (status {status})")


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def dtype_code(dtype) -> int:
    import torch

    if dtype in (torch.float64, np.float64, "f64", "float64"):
        return F64
    if dtype in (torch.float32, np.float32, "f32", "float32"):
        return F32
    raise ValueError(f"unsupported dtype {dtype}")


def ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())
