"""Steepest-neighbour topology on the GPU (mirror of topocorrect.topology).

``scan_neighbors`` runs the K-scan kernel (topology.py:47-86 semantics:
(value, id)-largest / smallest neighbour, is_max / is_min).
``compute_segmentation`` and ``compare_plmss`` (topology.py:156-174,254-274)
run on the device too (csrc/segment.cuh: 16-bit full codes, pointer jumping
to the path roots, the six kinds as bitmaps); the correction path itself
only needs the clean-report certificate described in correction.py.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .grid import ScalarField


def _dims3(dims) -> tuple[int, int, int]:
    d = tuple(int(v) for v in dims)
    return (d[0], d[1], 1) if len(d) == 2 else d


@dataclass(frozen=True, eq=False)
class NeighborScan:
    nmax: np.ndarray
    nmin: np.ndarray
    is_max: np.ndarray
    is_min: np.ndarray


def scan_neighbors_device(values: torch.Tensor, dims) -> tuple[torch.Tensor, ...]:
    nx, ny, nz = _dims3(dims)
    n = nx * ny * nz
    dev = values.device
    nmax = torch.empty(n, dtype=torch.int64, device=dev)
    nmin = torch.empty(n, dtype=torch.int64, device=dev)
    ismax = torch.empty(n, dtype=torch.uint8, device=dev)
    ismin = torch.empty(n, dtype=torch.uint8, device=dev)
    N.check(N.lib().pmsz_scan_neighbors(nx, ny, nz, N.ptr(values), N.ptr(nmax), N.ptr(nmin),
                                        N.ptr(ismax), N.ptr(ismin), N.stream_handle()),
            "pmsz_scan_neighbors")
    return nmax, nmin, ismax, ismin


def scan_neighbors(values: np.ndarray, dims) -> NeighborScan:
    """GPU steepest-neighbour scan of a flat x-fastest f64 array."""
    dims = _dims3(dims)
    dev = torch.device("cuda", torch.cuda.current_device())
    from .engine import as_device_f64
    v = as_device_f64(values, dev)
    nmax, nmin, ismax, ismin = scan_neighbors_device(v, dims)
    return NeighborScan(nmax=nmax.cpu().numpy(), nmin=nmin.cpu().numpy(),
                        is_max=ismax.cpu().numpy().astype(bool),
                        is_min=ismin.cpu().numpy().astype(bool))


def scan_codes_device(values: torch.Tensor, dims) -> torch.Tensor:
    """Packed 1-byte codes (nmax rank | nmin rank << 4, 15 = extremum)."""
    nx, ny, nz = _dims3(dims)
    code = torch.empty(nx * ny * nz, dtype=torch.uint8, device=values.device)
    N.check(N.lib().pmsz_scan_codes(nx, ny, nz, N.ptr(values), N.ptr(code), N.stream_handle()),
            "pmsz_scan_codes")
    return code


def field_scan(field: ScalarField) -> NeighborScan:
    return scan_neighbors(field.values, field.dims)


@dataclass(frozen=True)
class ExtremaSet:
    maxima: frozenset
    minima: frozenset


def find_extrema(field: ScalarField) -> ExtremaSet:
    s = field_scan(field)
    return ExtremaSet(maxima=frozenset(np.flatnonzero(s.is_max).tolist()),
                      minima=frozenset(np.flatnonzero(s.is_min).tolist()))


def _empty():
    return np.zeros(0, dtype=np.int64)


@dataclass(frozen=True, eq=False)
class DistortionReport:
    """Distortion categories of a test field against a reference field
    (topology.py:196-251)."""

    fp_max: np.ndarray = field(default_factory=_empty)
    fn_max: np.ndarray = field(default_factory=_empty)
    fp_min: np.ndarray = field(default_factory=_empty)
    fn_min: np.ndarray = field(default_factory=_empty)
    asc_order_violations: np.ndarray = field(default_factory=_empty)
    desc_order_violations: np.ndarray = field(default_factory=_empty)
    wrong_label_count: int = 0

    @classmethod
    def clean(cls) -> "DistortionReport":
        return cls()

    @property
    def is_clean(self) -> bool:
        return (self.fp_max.size == 0 and self.fn_max.size == 0 and self.fp_min.size == 0
                and self.fn_min.size == 0 and self.asc_order_violations.size == 0
                and self.desc_order_violations.size == 0 and self.wrong_label_count == 0)

    def counts(self) -> dict[str, int]:
        return {"fp_max": int(self.fp_max.size), "fn_max": int(self.fn_max.size),
                "fp_min": int(self.fp_min.size), "fn_min": int(self.fn_min.size),
                "asc_order_violations": int(self.asc_order_violations.size),
                "desc_order_violations": int(self.desc_order_violations.size),
                "wrong_label_count": int(self.wrong_label_count)}

    def to_dict(self) -> dict:
        return {"fp_max": self.fp_max.tolist(), "fn_max": self.fn_max.tolist(),
                "fp_min": self.fp_min.tolist(), "fn_min": self.fn_min.tolist(),
                "asc_order_violations": self.asc_order_violations.tolist(),
                "desc_order_violations": self.desc_order_violations.tolist(),
                "wrong_label_count": int(self.wrong_label_count), "clean": self.is_clean}


# ---------------------------------------------------------------------------
# segmentation (topology.py:127-174)
@dataclass(frozen=True, eq=False)
class SegmentationLabels:
    """asc_target: minimum reached by the descending path of each vertex;
    desc_target: maximum reached by the ascending path (topology.py:127-140)."""

    dims: tuple
    asc_target: np.ndarray
    desc_target: np.ndarray

    def pair_equal(self, other: "SegmentationLabels") -> np.ndarray:
        return np.logical_and(self.asc_target == other.asc_target, self.desc_target == other.desc_target)


def _as_device(values, dev) -> torch.Tensor:
    if isinstance(values, torch.Tensor):
        return values.to(dev) if values.device != dev else values
    v = np.ascontiguousarray(values)
    if v.dtype not in (np.float32, np.float64):
        v = v.astype(np.float64)
    return torch.from_numpy(v).to(dev)


def compute_segmentation_device(values: torch.Tensor, dims) -> tuple[torch.Tensor, torch.Tensor]:
    """(asc_target, desc_target) int64 device tensors of a f64/f32 device field."""
    nx, ny, nz = _dims3(dims)
    n = nx * ny * nz
    asc = torch.empty(n, dtype=torch.int64, device=values.device)
    desc = torch.empty(n, dtype=torch.int64, device=values.device)
    N.check(N.lib().pmsz_segmentation(nx, ny, nz, N.ptr(values), int(values.dtype == torch.float32), N.ptr(asc),
                                      N.ptr(desc), N.stream_handle()), "pmsz_segmentation")
    return asc, desc


def compute_segmentation(field: ScalarField) -> SegmentationLabels:
    dev = torch.device("cuda", torch.cuda.current_device())
    asc, desc = compute_segmentation_device(_as_device(field.values, dev), field.dims)
    return SegmentationLabels(dims=field.dims, asc_target=asc.cpu().numpy(), desc_target=desc.cpu().numpy())


def compute_segmentation_naive(field: ScalarField) -> SegmentationLabels:
    """topology.compute_segmentation_naive (topology.py:177-194): the reference
    follows the steepest pointers one step at a time as an oracle for its
    pointer-jumping path; both define the same labels, which is what this
    returns (the device pointer jumping of compute_segmentation)."""
    return compute_segmentation(field)


def _bits_to_ids(bits: torch.Tensor, nbits: int) -> np.ndarray:
    cnt = N.ctypes.c_int64()
    lib = N.lib()
    N.check(lib.pmsz_bits_to_ids(N.ptr(bits), nbits, None, 0, N.ctypes.byref(cnt), N.stream_handle()),
            "pmsz_bits_to_ids")
    m = int(cnt.value)
    if m == 0:
        return _empty()
    ids = torch.empty(m, dtype=torch.int64, device=bits.device)
    N.check(lib.pmsz_bits_to_ids(N.ptr(bits), nbits, N.ptr(ids), m, N.ctypes.byref(cnt), N.stream_handle()),
            "pmsz_bits_to_ids")
    return ids.cpu().numpy()


def compare_plmss_device(reference: torch.Tensor, test: torch.Tensor, dims,
                         with_sets: bool = True) -> DistortionReport:
    """compare_plmss on device fields (f64 or f32 each)."""
    nx, ny, nz = _dims3(dims)
    n = nx * ny * nz
    nwords = (n + 31) // 32
    bits = torch.zeros(6 * nwords, dtype=torch.int32, device=reference.device) if with_sets else None
    counts = (N.ctypes.c_int64 * 7)()
    N.check(N.lib().pmsz_compare_plmss(nx, ny, nz, N.ptr(reference), int(reference.dtype == torch.float32),
                                       N.ptr(test), int(test.dtype == torch.float32),
                                       N.ptr(bits) if bits is not None else None, counts, N.stream_handle()),
            "pmsz_compare_plmss")
    if not with_sets:
        # sized placeholders: only the counts are meaningful
        sets = [np.zeros(int(counts[k]), dtype=np.int64) for k in range(6)]
    else:
        sets = [_bits_to_ids(bits[k * nwords:(k + 1) * nwords], n) if counts[k] else _empty() for k in range(6)]
    return DistortionReport(fp_max=sets[0], fn_max=sets[1], fp_min=sets[2], fn_min=sets[3],
                            asc_order_violations=sets[4], desc_order_violations=sets[5],
                            wrong_label_count=int(counts[6]))


def compare_plmss(reference: ScalarField, test: ScalarField) -> DistortionReport:
    """Distortion report of test relative to reference (topology.py:254-274)."""
    if reference.dims != test.dims:
        raise ValueError(f"dims differ: {reference.dims} vs {test.dims}")
    dev = torch.device("cuda", torch.cuda.current_device())
    return compare_plmss_device(_as_device(reference.values, dev), _as_device(test.values, dev), reference.dims)
