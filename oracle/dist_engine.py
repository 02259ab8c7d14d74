"""CPU ORACLE engine for the distributed round loop -- TEST INFRASTRUCTURE ONLY.

Implements the engine interface of paper_2601_01787_b200.dist (round / empty /
pack / merge / block_stats) for one block with the C oracle's
_iterate_array restatement, so the multi-rank host logic (exchange topology,
termination, stats) runs under gloo on CPU and is checked against the
oracle's single-process run_parallel (itself pinned to the reference).
"""

from __future__ import annotations

import numpy as np
import torch

from . import oracle as orc


class OracleEngine:
    device = torch.device("cpu")

    def __init__(self, block, spec, gdims, f: np.ndarray, fhat: np.ndarray, xi: float, tau: float, cap: int):
        nx, ny, nz = gdims
        sl = tuple(slice(block.ext_start[a], block.ext_stop[a]) for a in (2, 1, 0))
        self.ed = spec.dims
        ex, ey, ez = self.ed
        self.f = np.ascontiguousarray(f.reshape(nz, ny, nx)[sl]).reshape(-1)
        self.g = np.ascontiguousarray(fhat.reshape(nz, ny, nx)[sl]).reshape(-1).copy()
        self.lower = self.f - xi
        self.tau = tau
        self.cap = cap
        self.fscan = orc.scan(self.f, self.ed)
        z, y, x = np.meshgrid(np.arange(ez), np.arange(ey), np.arange(ex), indexing="ij")
        core = ((x >= spec.core_lo[0]) & (x < spec.core_hi[0]) & (y >= spec.core_lo[1]) & (y < spec.core_hi[1])
                & (z >= spec.core_lo[2]) & (z < spec.core_hi[2]))
        shared = ((x < spec.shared_lo[0]) | (x >= ex - spec.shared_hi[0]) | (y < spec.shared_lo[1])
                  | (y >= ey - spec.shared_hi[1]) | (z < spec.shared_lo[2]) | (z >= ez - spec.shared_hi[2]))
        self.core = core.reshape(-1)
        self.shared = shared.reshape(-1)
        self.counts = np.zeros(self.g.size, np.int64)
        self.iters = 0
        self.edits = 0

    def round(self, lockstep: bool):
        """_block_round (parallel.py:237-255)."""
        round_edits, dirty = 0, False
        for _ in range(self.cap):
            g, ed = orc.iterate(self.ed, self.fscan, self.g, self.lower, self.tau, self.core)
            self.g = g
            self.iters += 1
            e = int(ed.sum())
            if e:
                self.counts[ed] += 1
                self.edits += e
                round_edits += e
                dirty = dirty or bool(ed[self.shared].any())
            if lockstep or e == 0:
                return round_edits, dirty
        raise RuntimeError("no local fixpoint")

    def _view(self, x):
        ex, ey, ez = self.ed
        return self.g.reshape(ez, ey, ex)[x.lo[2]:x.hi[2], x.lo[1]:x.hi[1], x.lo[0]:x.hi[0]]

    def empty(self, x):
        return torch.empty(x.size, dtype=torch.float64)

    def pack(self, x):
        return torch.from_numpy(np.ascontiguousarray(self._view(x)).reshape(-1).copy())

    def merge(self, x, buf) -> int:
        v = self._view(x)
        inc = buf.numpy().reshape(v.shape)
        changed = int((inc < v).sum())
        np.minimum(v, inc, out=v)
        return changed

    def block_stats(self):
        return self.iters, self.edits, int(self.counts.max())

    def core_values(self, spec):
        ex, ey, ez = self.ed
        return self.g.reshape(ez, ey, ex)[spec.core_lo[2]:spec.core_hi[2], spec.core_lo[1]:spec.core_hi[1],
                                          spec.core_lo[0]:spec.core_hi[0]]
