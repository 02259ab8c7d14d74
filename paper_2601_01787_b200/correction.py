"""Drop-in correction entry points (mirror of topocorrect.correction).

``run_correction(original, decompressed, config)`` keeps the reference
signature and result type (correction.py:391-436) but runs the whole loop on
the GPU: K0 prepare -> (K1 detect/propose -> K2 apply) until a zero-edit
iteration -> K4 verify -> K5 edit export, all in libpmsz (sm_100a).

Semantics kept bit-for-bit: the corrected field, ``edits_per_iteration``,
``iterations`` (the final zero-edit pass counts), ``max_vertex_edits``, the
edit set (ascending ids where g != fhat), and every failure mode
(BoundViolationError, the monotonicity AssertionError, ConvergenceError).
The ``verification`` report is the all-clean DistortionReport: after a
successful run the GPU verify sweep has shown that every vertex has the same
extremum flags as the original, the same steepest-ascent neighbour unless it
is a maximum and the same steepest-descent neighbour unless it is a minimum,
so both pointer forests (topology.py:165-174) and with them the segmentations
are identical -- exactly the conditions ``compare_plmss`` tests.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .engine import (BoundViolationError, ConvergenceError, DomainPlan, DomainSpec,
                     HOST_FIELDS, as_device_f64, narrow_if_exact, raise_for, to_host_f64)
from .grid import ScalarField
from .topology import DistortionReport

__all__ = [
    "BoundViolationError", "ConvergenceError", "CorrectionConfig", "BoundsField",
    "compute_bounds", "apply_edit", "validate_error_bound", "EditSet", "CorrectionResult",
    "DeviceCorrection", "run_correction", "run_correction_device", "iterate_array",
]


@dataclass(frozen=True)
class CorrectionConfig:
    """xi_abs, tau (default xi/1024) and the iteration cap
    (default 10*ceil(2 xi / tau)); correction.py:63-96."""

    xi_abs: float
    tau: float | None = None
    max_outer_iterations: int | None = None

    def __post_init__(self):
        xi = float(self.xi_abs)
        if not (math.isfinite(xi) and xi > 0):
            raise ValueError(f"xi_abs must be positive and finite, got {self.xi_abs!r}")
        tau = xi / 1024.0 if self.tau is None else float(self.tau)
        if not (math.isfinite(tau) and 0.0 < tau < 2.0 * xi):
            raise ValueError(f"tau must lie in (0, 2*xi_abs), got {tau!r}")
        if self.max_outer_iterations is None:
            cap = 10 * math.ceil(2.0 * xi / tau)
        else:
            cap = int(self.max_outer_iterations)
        if cap < 1:
            raise ValueError("max_outer_iterations must be >= 1")
        object.__setattr__(self, "xi_abs", xi)
        object.__setattr__(self, "tau", tau)
        object.__setattr__(self, "max_outer_iterations", cap)

    @property
    def per_vertex_edit_budget(self) -> int:
        return math.ceil(2.0 * self.xi_abs / self.tau) + 1


@dataclass(frozen=True, eq=False)
class BoundsField:
    """Admissible interval [f - xi, f + xi] (correction.py:99-125)."""

    lower: np.ndarray
    upper: np.ndarray

    @classmethod
    def from_field(cls, field: ScalarField, xi_abs: float) -> "BoundsField":
        if not (math.isfinite(xi_abs) and xi_abs > 0):
            raise ValueError(f"xi_abs must be positive and finite, got {xi_abs!r}")
        return cls(field.values - xi_abs, field.values + xi_abs)

    def admits(self, values: np.ndarray) -> bool:
        return bool(np.all((values >= self.lower) & (values <= self.upper)))


def compute_bounds(field: ScalarField, xi_abs: float) -> BoundsField:
    return BoundsField.from_field(field, xi_abs)


def apply_edit(current: float, proposal: float, lower: float) -> float:
    """max(min(current, proposal), lower) -- the per-vertex rule K2 applies."""
    return max(min(current, proposal), lower)


def validate_error_bound(original: ScalarField, decompressed: ScalarField, xi_abs: float) -> None:
    """|f - fhat| <= xi everywhere, checked by the K0 kernel (correction.py:52-60)."""
    if original.dims != decompressed.dims:
        raise ValueError(f"dims differ: {original.dims} vs {decompressed.dims}")
    dev = torch.device("cuda", torch.cuda.current_device())
    f = as_device_f64(original.values, dev)
    fh = as_device_f64(decompressed.values, dev)
    g = torch.empty_like(fh)
    plan = DomainPlan(DomainSpec.whole(original.dims), xi_abs, xi_abs / 1024.0, 1, incremental=False)
    st, res = plan.prepare(f, fh, g)
    if st == N.PMSZ_ERR_BOUND:
        raise_for(st, res, original.values, decompressed.values, xi_abs)
    if st not in (N.PMSZ_OK,):
        raise_for(st, res, original.values, decompressed.values, xi_abs)


@dataclass(frozen=True, eq=False)
class EditSet:
    """Ascending vertex ids and corrected values (correction.py:328-378)."""

    ids: np.ndarray
    values: np.ndarray
    vertex_count: int

    def __post_init__(self):
        ids = np.ascontiguousarray(self.ids, dtype=np.int64).reshape(-1)
        values = np.ascontiguousarray(self.values, dtype=np.float64).reshape(-1)
        if ids.size != values.size:
            raise ValueError("ids/values length mismatch")
        if ids.size:
            if (np.diff(ids) <= 0).any():
                raise ValueError("edit ids must be strictly increasing")
            if ids[0] < 0 or ids[-1] >= self.vertex_count:
                raise ValueError("edit id out of range")
        if not np.isfinite(values).all():
            raise ValueError("edit values must be finite")
        ids.setflags(write=False)
        values.setflags(write=False)
        object.__setattr__(self, "ids", ids)
        object.__setattr__(self, "values", values)
        object.__setattr__(self, "vertex_count", int(self.vertex_count))

    @classmethod
    def _owned(cls, ids: np.ndarray, values: np.ndarray, vertex_count: int) -> "EditSet":
        """The record of a device run, in fresh arrays this package just
        produced: the export walks the edited bitmap in id order (strictly
        ascending, in range) and every value is a finite f64 the kernels
        computed, so the O(count) validation scans are skipped."""
        obj = object.__new__(cls)
        ids = np.asarray(ids, dtype=np.int64).reshape(-1)
        values = np.asarray(values, dtype=np.float64).reshape(-1)
        ids.setflags(write=False)
        values.setflags(write=False)
        object.__setattr__(obj, "ids", ids)
        object.__setattr__(obj, "values", values)
        object.__setattr__(obj, "vertex_count", int(vertex_count))
        return obj

    @property
    def count(self) -> int:
        return int(self.ids.size)

    @property
    def ratio(self) -> float:
        return self.count / self.vertex_count

    @classmethod
    def diff(cls, baseline: ScalarField, edited: ScalarField) -> "EditSet":
        if baseline.dims != edited.dims:
            raise ValueError(f"dims differ: {baseline.dims} vs {edited.dims}")
        ids = np.flatnonzero(baseline.values != edited.values)
        return cls(ids=ids, values=edited.values[ids], vertex_count=baseline.vertex_count)

    def apply_to(self, field: ScalarField) -> ScalarField:
        if field.vertex_count != self.vertex_count:
            raise ValueError(f"edit set is for {self.vertex_count} vertices, field has "
                             f"{field.vertex_count}")
        values = field.values.copy()
        values[self.ids] = self.values
        return field.with_values(values)


@dataclass(frozen=True, eq=False)
class CorrectionResult:
    corrected: ScalarField
    edits: EditSet
    iterations: int
    edits_per_iteration: tuple[int, ...]
    max_vertex_edits: int
    verification: DistortionReport


@dataclass(eq=False)
class DeviceCorrection:
    """Result of a device-resident correction (all tensors on the GPU)."""

    corrected: torch.Tensor
    edit_ids: torch.Tensor
    edit_values: torch.Tensor
    iterations: int
    edits_per_iteration: tuple[int, ...]
    max_vertex_edits: int
    full_sweeps: int
    sparse_sweeps: int
    masked_sweeps: int = 0
    fragile: int = -1     # centres K0 left fragile (robust ones are never evaluated)


_PLAN_CACHE: dict = {}


def _plan_for(dims, config: CorrectionConfig, *, incremental: bool, extrema_only: bool,
              f32_original: bool, host_f64: bool = False) -> DomainPlan:
    key = (tuple(dims), config.xi_abs, config.tau, config.max_outer_iterations, incremental,
           extrema_only, f32_original, host_f64, torch.cuda.current_device())
    plan = _PLAN_CACHE.get(key)
    if plan is None:
        if len(_PLAN_CACHE) >= 4:
            _PLAN_CACHE.pop(next(iter(_PLAN_CACHE))).close()
        plan = DomainPlan(DomainSpec.whole(dims), config.xi_abs, config.tau,
                          config.max_outer_iterations, incremental=incremental,
                          extrema_only=extrema_only, f32_original=f32_original,
                          host_f64=host_f64)
        _PLAN_CACHE[key] = plan
    return plan


def run_correction_device(f: torch.Tensor, fhat: torch.Tensor, dims, config: CorrectionConfig, *,
                          out: torch.Tensor | None = None, incremental: bool = True,
                          extrema_only: bool = False, export_edits: bool = True,
                          plan: DomainPlan | None = None, stream=None) -> DeviceCorrection:
    """run_correction on device tensors: f (float64, or float32 = exact f32 field),
    fhat (float64).  ``out`` may alias ``fhat`` for an in-place correction."""
    dims = tuple(int(v) for v in dims)
    if len(dims) == 2:
        dims = (dims[0], dims[1], 1)
    if not f.is_cuda or not fhat.is_cuda:
        raise ValueError("run_correction_device needs CUDA tensors")
    if fhat.dtype != torch.float64 or f.dtype not in (torch.float64, torch.float32):
        raise ValueError("fhat must be float64 and f float64/float32")
    n = dims[0] * dims[1] * dims[2]
    if f.numel() != n or fhat.numel() != n:
        raise ValueError("field sizes do not match dims")
    f32 = f.dtype == torch.float32
    if plan is None:
        plan = _plan_for(dims, config, incremental=incremental, extrema_only=extrema_only,
                         f32_original=f32)
    g = out if out is not None else torch.empty_like(fhat)
    with plan.lock:
        if export_edits:
            st, res, hist, ids, vals = plan.run_export(f, fhat, g, stream=stream)
            raise_for(st, res, None, None, config.xi_abs, f_dev=f, fhat_dev=fhat)
        else:
            st, res, hist = plan.run(f, fhat, g, stream=stream)
            raise_for(st, res, None, None, config.xi_abs, f_dev=f, fhat_dev=fhat)
            ids = vals = torch.empty(0, device=g.device)
    return DeviceCorrection(corrected=g, edit_ids=ids, edit_values=vals,
                            iterations=int(res.iterations), edits_per_iteration=tuple(hist),
                            max_vertex_edits=int(res.max_vertex_edits),
                            full_sweeps=int(res.full_sweeps), sparse_sweeps=int(res.sparse_sweeps),
                            masked_sweeps=int(res.masked_sweeps), fragile=int(res.fragile))


def run_correction(original: ScalarField, decompressed: ScalarField, config: CorrectionConfig,
                   *, incremental: bool = True) -> CorrectionResult:
    """Drop-in for topocorrect.run_correction (correction.py:391-436).

    One pmsz_run_correction_host call on the ScalarFields' own (pageable)
    arrays: host threads stage the inputs through a pinned ring while K0 runs
    slab by slab, the corrected field is filled from fhat on the host and
    patched with the edit record (include/pmsz.h).  ScalarField always holds
    f64 (grid.py:57); the original is narrowed to f32 while it is staged and
    runs the f32 K0 when every value survives the round trip (fields read
    from f32 files, codec.py:86-87) -- otherwise the call reruns on an f64
    plan before any iteration has run."""
    if original.dims != decompressed.dims:
        raise ValueError(f"dims differ: {original.dims} vs {decompressed.dims}")
    dims = original.dims
    f = np.ascontiguousarray(original.values, dtype=np.float64).reshape(-1)
    fh = np.ascontiguousarray(decompressed.values, dtype=np.float64).reshape(-1)
    g = HOST_FIELDS.take(f.size)   # a recycled array when a previous result was dropped
    for narrow in (True, False):
        plan = _plan_for(dims, config, incremental=incremental, extrema_only=False,
                         f32_original=narrow, host_f64=narrow)
        with plan.lock:
            st, res, hist, ids, vals = plan.run_host(f, fh, g)
        if st != N.PMSZ_ERR_INEXACT:
            break
    raise_for(st, res, original.values, decompressed.values, config.xi_abs)
    return CorrectionResult(corrected=ScalarField._owned(dims, g),
                            edits=EditSet._owned(ids, vals, original.vertex_count),
                            iterations=int(res.iterations), edits_per_iteration=tuple(hist),
                            max_vertex_edits=int(res.max_vertex_edits),
                            verification=DistortionReport.clean())


def iterate_array(dims, f_values: np.ndarray, g_values: np.ndarray, xi: float, tau: float,
                  core_lo=None, core_hi=None) -> tuple[np.ndarray, np.ndarray]:
    """One Jacobi iteration on the GPU (the `_iterate_array` test seam,
    correction.py:232-242): returns (new g, edited mask) as host arrays.
    ``lower`` is f - xi as in BoundsField.from_field."""
    dims = tuple(int(v) for v in dims)
    if len(dims) == 2:
        dims = (dims[0], dims[1], 1)
    dev = torch.device("cuda", torch.cuda.current_device())
    spec = DomainSpec(dims, tuple(core_lo or (0, 0, 0)), tuple(core_hi or dims))
    plan = DomainPlan(spec, xi, tau, 1, incremental=False)
    f = as_device_f64(f_values, dev)
    g = as_device_f64(g_values, dev)
    # K0 needs fhat only for validation/copy; the iterate works on g in place.
    st, res = plan.prepare(f, g, g)
    if st not in (N.PMSZ_OK, N.PMSZ_ERR_BOUND):
        raise_for(st, res, f_values, g_values, xi)
    mask = torch.zeros(plan.n, dtype=torch.uint8, device=dev)
    st, res = plan.iterate(f, g, mask)
    raise_for(st, res, f_values, g_values, xi)
    return g.cpu().numpy(), mask.cpu().numpy().astype(bool)
