"""Steepest-neighbour topology on the GPU (mirror of topocorrect.topology).

``scan_neighbors`` runs the K-scan kernel (topology.py:47-86 semantics:
(value, id)-largest / smallest neighbour, is_max / is_min).  The segmentation
and full ``compare_plmss`` are SURVEY §8(f) rank 1 ("next"); the correction
path only needs the clean-report certificate described in correction.py.
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
    v = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float64)).to(dev)
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
