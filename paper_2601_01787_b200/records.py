"""The reference's record-based route (correction.py:133-160,245-325) and the
per-vertex topology helpers (topology.py:93-122,177-194), under their own
names so code written against ``topocorrect`` finds them.

The reference keeps this route as the definition-shaped twin of its array
engine (its tests hold the two together bit for bit).  Here the scans behind
``detect_distortions`` run on the device (``scan_neighbors``) and
``correction_iteration`` IS the array engine (one ``pmsz_iterate`` with the
given lower bound); the records themselves -- a Python list of a few
``Distortion`` objects -- and ``propose_corrections``' dict merge are host
bookkeeping, as in the reference.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np
import torch

from .correction import BoundsField, apply_edit
from .engine import DomainPlan, DomainSpec, as_device_f64, raise_for
from .grid import ScalarField, neighbors, precedes
from .topology import field_scan


class DistortionKind(enum.Enum):
    """The six detection kinds in the reference's declaration order (records
    of one centre sort by it)."""
    FALSE_MAXIMUM = "false_maximum"
    MISSING_MAXIMUM = "missing_maximum"
    FALSE_MINIMUM = "false_minimum"
    MISSING_MINIMUM = "missing_minimum"
    ASC_ORDER = "asc_order"
    DESC_ORDER = "desc_order"


_RANK = {k: i for i, k in enumerate(DistortionKind)}


@dataclass(frozen=True)
class Distortion:
    """One detected break of the original order around `center`: every vertex
    of `targets` is proposed g[anchor] - tau (correction.py:138-153)."""
    kind: DistortionKind
    center: int
    anchor: int
    targets: tuple[int, ...]


def kind_masks(f_scan, g_scan):
    """The six detection masks of two scans (correction.py:169-180)."""
    return (g_scan.is_max & ~f_scan.is_max, f_scan.is_max & ~g_scan.is_max,
            g_scan.is_min & ~f_scan.is_min, f_scan.is_min & ~g_scan.is_min,
            ~f_scan.is_max & (g_scan.nmax != f_scan.nmax), ~f_scan.is_min & (g_scan.nmin != f_scan.nmin))


def detect_distortions(original: ScalarField, distorted: ScalarField) -> list[Distortion]:
    """Every distortion of `distorted` against `original`, sorted by (centre,
    kind order) (correction.py:245-287); both scans on the device."""
    if original.dims != distorted.dims:
        raise ValueError(f"dims differ: {original.dims} vs {distorted.dims}")
    fs, gs = field_scan(original), field_scan(distorted)
    g = distorted.values
    dims = original.dims

    def above(center, anchor):   # in-ring vertices sorting above the anchor in g
        ga = g[anchor]
        return tuple(j for j in neighbors(dims, center) if g[j] > ga or (g[j] == ga and j > anchor))

    out = []
    for kind, mask in zip(DistortionKind, kind_masks(fs, gs)):
        for c in np.flatnonzero(mask).tolist():
            if kind is DistortionKind.FALSE_MAXIMUM:
                out.append(Distortion(kind, c, int(fs.nmax[c]), (c,)))
            elif kind is DistortionKind.MISSING_MAXIMUM:
                out.append(Distortion(kind, c, c, above(c, c)))
            elif kind is DistortionKind.FALSE_MINIMUM:
                out.append(Distortion(kind, c, c, (int(fs.nmin[c]),)))
            elif kind is DistortionKind.MISSING_MINIMUM:
                out.append(Distortion(kind, c, int(gs.nmin[c]), (c,)))
            elif kind is DistortionKind.ASC_ORDER:
                a = int(fs.nmax[c])
                out.append(Distortion(kind, c, a, above(c, a)))
            else:
                out.append(Distortion(kind, c, int(gs.nmin[c]), (int(fs.nmin[c]),)))
    out.sort(key=lambda r: (r.center, _RANK[r.kind]))
    return out


def propose_corrections(distorted: ScalarField, tau: float, detections) -> dict[int, float]:
    """One proposal per target, competing ones merged by minimum
    (correction.py:290-306)."""
    g = distorted.values
    merged: dict[int, float] = {}
    for rec in detections:
        val = float(g[rec.anchor]) - tau
        for t in rec.targets:
            cur = merged.get(t)
            if cur is None or val < cur:
                merged[t] = val
    return merged


def correction_iteration(original: ScalarField, current: ScalarField, bounds: BoundsField,
                         tau: float) -> tuple[ScalarField, int]:
    """One detect / propose / apply step (correction.py:309-325), run as the
    array engine on the device: pmsz_iterate with `bounds.lower` as the
    explicit floor, every centre evaluated (an arbitrary current field may
    sit anywhere).  A current field already below the floor somewhere -- where
    the array engine would stop on its monotonicity check but this route just
    clamps -- takes the host records instead."""
    if original.dims != current.dims:
        raise ValueError(f"dims differ: {original.dims} vs {current.dims}")
    dims = original.dims
    dev = torch.device("cuda", torch.cuda.current_device())
    lower_h = np.asarray(bounds.lower, dtype=np.float64).reshape(-1)
    plan = DomainPlan(DomainSpec.whole(dims), 1e300, float(tau), 1, incremental=False, no_robust=True,
                      explicit_lower=True)
    try:
        f = as_device_f64(original.values, dev)
        g = as_device_f64(current.values, dev)
        lower = as_device_f64(lower_h, dev)
        st, res = plan.prepare(f, g, g)   # the f-code (xi only bounds the validation here)
        raise_for(st, res, original.values, current.values, None)
        if plan.floor_violations(lower, g):
            return apply_proposals(current, propose_corrections(current, tau, detect_distortions(original, current)),
                                   lower_h)
        st, res = plan.iterate(lower, g, None)
        raise_for(st, res, original.values, current.values, None)
        return current.with_values(g.cpu().numpy()), int(res.last_edits)
    finally:
        plan.close()


# ---- per-vertex helpers (topology.py:93-122) --------------------------------
def extreme_neighbor(field: ScalarField, v: int, direction: str) -> int:
    """Largest ('ascending') or smallest ('descending') neighbour of v in the
    (value, id) order."""
    if direction not in ("ascending", "descending"):
        raise ValueError(f"direction must be 'ascending' or 'descending', got {direction!r}")
    best = None
    for j in neighbors(field.dims, v):
        if best is None or (precedes(field, best, j) if direction == "ascending" else precedes(field, j, best)):
            best = j
    return best


def is_maximum(field: ScalarField, v: int) -> bool:
    return precedes(field, extreme_neighbor(field, v, "ascending"), v)


def is_minimum(field: ScalarField, v: int) -> bool:
    return precedes(field, v, extreme_neighbor(field, v, "descending"))


def apply_proposals(current: ScalarField, proposals: dict[int, float], lower) -> tuple[ScalarField, int]:
    """The apply half of correction_iteration on host records (apply_edit per
    proposal): for callers that edit the proposals before applying them."""
    values = current.values.copy()
    edits = 0
    for v, p in proposals.items():
        nv = apply_edit(values[v], p, lower[v])
        if nv != values[v]:
            values[v] = nv
            edits += 1
    return current.with_values(values), edits
