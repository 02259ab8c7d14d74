"""ctypes binding of the C ABI in include/pmsz.h (libpmsz.so, sm_100a).

There is no CPU fallback: importing this module works everywhere (so the
CPU test suite can check the exported symbols), but every compute entry point
raises if the library is absent or no CUDA device is visible.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["PMSZ_LIB"]) if os.environ.get("PMSZ_LIB") else _HERE / "_lib" / "libpmsz.so"   # A/B builds
HEADER_PATH = _HERE.parent / "include" / "pmsz.h"

PMSZ_OK = 0
PMSZ_ERR_INVALID = 1
PMSZ_ERR_BOUND = 2
PMSZ_ERR_MONOTONE = 3
PMSZ_ERR_CONVERGENCE = 4
PMSZ_ERR_CUDA = 5
PMSZ_ERR_NONFINITE = 6
PMSZ_ERR_INEXACT = 7

PMSZ_CONV_NONE = 0
PMSZ_CONV_CAP = 1
PMSZ_CONV_BOUND = 2
PMSZ_CONV_RESIDUAL = 3

K_PREP, K_SWEEP_FULL, K_SWEEP_SPARSE, K_APPLY, K_VERIFY, K_COMPACT, K_OTHER, K_SWEEP_MASKED, K_DEFER = range(9)
K_COUNT = 10
K_NAMES = ("prep", "sweep_full", "sweep_sparse", "apply", "verify", "compact", "other", "sweep_masked",
           "defer", "tail")

FLAG_INCREMENTAL = 1
FLAG_EXTREMA_ONLY = 2
FLAG_F32_ORIGINAL = 4
FLAG_HOST_LOOP = 8
FLAG_NO_ROBUST = 16
FLAG_LOWER = 32
FLAG_HOST_F64 = 64

i64 = ctypes.c_int64
i32 = ctypes.c_int32
u64 = ctypes.c_uint64
vp = ctypes.c_void_p
dp = ctypes.POINTER(ctypes.c_double)
i64p = ctypes.POINTER(ctypes.c_int64)


class PmszDesc(ctypes.Structure):
    _fields_ = [
        ("nx", i64), ("ny", i64), ("nz", i64),
        ("core_lo", i64 * 3), ("core_hi", i64 * 3),
        ("shared_lo", i32 * 3), ("shared_hi", i32 * 3),
        ("xi", ctypes.c_double), ("tau", ctypes.c_double),
        ("max_iterations", i64),
        ("flags", i32), ("reserved", i32),
    ]


class PmszResult(ctypes.Structure):
    _fields_ = [
        ("iterations", i64), ("edit_count", i64), ("max_vertex_edits", i64),
        ("bound_violations", i64), ("bound_first_index", i64),
        ("floor_violations", i64), ("nonfinite", i64),
        ("residual", i64 * 6), ("convergence_kind", i64),
        ("full_sweeps", i64), ("sparse_sweeps", i64), ("shared_dirty", i64),
        ("last_edits", i64), ("last_detections", i64), ("masked_sweeps", i64), ("fragile", i64),
    ]


MAX_RANKS = 64
MAX_EXCHANGES = 26


class PmszRoundsDesc(ctypes.Structure):
    _fields_ = [
        ("world", i32), ("rank", i32), ("nex", i32), ("lockstep", i32),
        ("cap", i64), ("repl_doubles", i64), ("sums_off", i64), ("flags_off", i64),
        ("epoch", u64), ("rounds_total", u64),
        ("bufs", vp * MAX_RANKS),
        ("ex_peer", i32 * MAX_EXCHANGES),
        ("ex_lo", (i64 * 3) * MAX_EXCHANGES), ("ex_hi", (i64 * 3) * MAX_EXCHANGES),
        ("ex_off", i64 * MAX_EXCHANGES), ("ex_peer_off", i64 * MAX_EXCHANGES),
    ]


# name -> (restype, argtypes); every symbol declared in include/pmsz.h.
SIGNATURES = {
    "pmsz_last_error": (ctypes.c_char_p, []),
    "pmsz_version": (ctypes.c_char_p, []),
    "pmsz_launch_count": (i64, []),
    "pmsz_plan_create": (i32, [ctypes.POINTER(PmszDesc), ctypes.POINTER(vp)]),
    "pmsz_plan_destroy": (None, [vp]),
    "pmsz_plan_scratch_bytes": (i64, [vp]),
    "pmsz_profile": (i32, [vp, i32]),
    "pmsz_profile_read": (i32, [vp, dp, i64p, i32]),
    "pmsz_run_correction": (i32, [vp, vp, vp, vp, i64p, i64, ctypes.POINTER(PmszResult), vp]),
    "pmsz_run_correction_export": (i32, [vp, vp, vp, vp, i64p, i64, ctypes.POINTER(PmszResult), vp, vp, i64, vp]),
    "pmsz_run_correction_host": (i32, [vp, vp, vp, vp, vp, vp, i64, i64p, i64,
                                       ctypes.POINTER(PmszResult), vp]),
    "pmsz_edits_export": (i32, [vp, vp, vp, vp, i64, i64p, vp]),
    "pmsz_edits_host": (i32, [vp, vp, vp, i64, i64p]),
    "pmsz_prepare": (i32, [vp, vp, vp, vp, ctypes.POINTER(PmszResult), vp]),
    "pmsz_iterate": (i32, [vp, vp, vp, vp, ctypes.POINTER(PmszResult), vp]),
    "pmsz_block_round": (i32, [vp, vp, vp, i32, i64p, ctypes.POINTER(PmszResult), vp]),
    "pmsz_mark_all_dirty": (i32, [vp, vp]),
    "pmsz_mark_dirty_ids": (i32, [vp, vp, i64, vp]),
    "pmsz_verify": (i32, [vp, vp, ctypes.POINTER(PmszResult), vp]),
    "pmsz_bounds_violations": (i32, [vp, vp, vp, i64p, vp]),
    "pmsz_floor_violations": (i32, [vp, vp, vp, i64p, vp]),
    "pmsz_history": (i32, [vp, i64p, i64, i64p]),
    "pmsz_scan_neighbors": (i32, [i64, i64, i64, vp, vp, vp, vp, vp, vp]),
    "pmsz_scan_codes": (i32, [i64, i64, i64, vp, vp, vp]),
    "pmsz_box_pack": (i32, [i64, i64, i64, vp, i64p, i64p, vp, vp]),
    "pmsz_box_unpack_min": (i32, [i64, i64, i64, vp, i64p, i64p, vp, vp, vp]),
    "pmsz_box_unpack_copy": (i32, [i64, i64, i64, vp, i64p, i64p, vp, vp, vp]),
    "pmsz_box_mark_changed": (i32, [vp, i64p, i64p, vp, vp, vp]),
    "pmsz_box_merge_min": (i32, [vp, vp, i64p, i64p, vp, i64p, vp]),
    "pmsz_residual": (i32, [vp, i64p, vp]),
    "pmsz_rounds": (i32, [vp, vp, vp, ctypes.POINTER(PmszRoundsDesc), i64p, i64p, i64p, i64,
                          ctypes.POINTER(PmszResult), vp]),
    "pmsz_perlin": (i32, [i64p, i64p, i64p, ctypes.POINTER(i32), ctypes.c_double, i32, vp, vp, vp]),
    "pmsz_minmax": (i32, [vp, i32, i64, dp, dp, vp]),
    "pmsz_narrow_f32": (i32, [vp, i64, vp, i64p, vp]),
    "pmsz_host_to_device": (i32, [vp, vp, i64, i32, i64p, vp]),
    "pmsz_device_to_host": (i32, [vp, vp, i64, vp]),
    "pmsz_quantize": (i32, [vp, i32, i64, ctypes.c_double, ctypes.c_double, vp, i64p, vp]),
    "pmsz_quantize_codes": (i32, [vp, i32, i64, ctypes.c_double, ctypes.c_double, vp, vp, i64p, vp]),
    "pmsz_bounded_noise": (i32, [vp, i32, i64, i64, i64, i64p, i64p, ctypes.c_double, u64, vp, vp]),
    "pmsz_box_extract": (i32, [i64p, vp, i32, i64p, i64p, vp, vp]),
    "pmsz_segmentation": (i32, [i64, i64, i64, vp, i32, vp, vp, vp]),
    "pmsz_gaussian_peaks": (i32, [i64p, i64p, i64p, u64, i32, vp, vp]),
    "pmsz_compare_plmss": (i32, [i64, i64, i64, vp, i32, vp, i32, vp, i64p, vp]),
    "pmsz_bits_to_ids": (i32, [vp, i64, vp, i64, i64p, vp]),
}


class NativeLibraryMissing(RuntimeError):
    """libpmsz.so is not built: there is deliberately no CPU fallback."""


_lib = None


def load(path: os.PathLike | None = None) -> ctypes.CDLL:
    """Load libpmsz.so (without touching the GPU) and bind every symbol."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise NativeLibraryMissing(
            f"{p} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the pMSz path has no CPU fallback)")
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def lib() -> ctypes.CDLL:
    """The loaded library, after checking a CUDA device is present."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("pMSz kernels need a CUDA device (sm_100a); none is visible")
    return load()


def last_error() -> str:
    return load().pmsz_last_error().decode(errors="replace")


def launch_count() -> int:
    return int(load().pmsz_launch_count())


def ivec(values) -> "ctypes.Array":
    return (i64 * 3)(*[int(v) for v in values])


def check(status: int, what: str) -> None:
    """Raise RuntimeError for CUDA / argument failures (domain errors are mapped by callers)."""
    if status != PMSZ_OK:
        raise RuntimeError(f"{what} failed (status {status}): {last_error()}")


def stream_handle(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int:
    return int(t.data_ptr())
