"""Block-parallel correction (mirror of topocorrect.parallel) on the GPU.

``run_parallel(original, decompressed, config, block_grid, strategy, workers)``
keeps the reference signature and returns ``(CorrectionResult, ParallelStats)``
with the same stats definitions (parallel.py:175-204,258-367).  Each block of
``decompose`` is a device plan over its extended extent (core + one ghost
layer), iterated by the K1/K2 kernels with the core box as the centre mask;
the ghost merge (``_merge_min``, parallel.py:122-140) is a device min-reduction
into a global accumulator followed by a per-block copy-back.

This single-process engine is the parity vehicle for the multi-GPU path
(dist.py), where each block is one rank and the merge is an NCCL exchange.
``workers`` is accepted for API compatibility; blocks run back to back on one
device and, as in the reference, scheduling never changes the result.
"""

from __future__ import annotations

import time
from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _native as N
from .correction import CorrectionConfig, CorrectionResult, EditSet
from .engine import (BoundViolationError, ConvergenceError, DomainPlan, DomainSpec, as_device_f64,
                     as_device_narrowed, narrow_if_exact,
                     to_host_f64,
                     raise_for)
from .grid import ScalarField
from .topology import DistortionReport


class SyncStrategy(Enum):
    LOCKSTEP = "lockstep"
    RELAXED = "relaxed"


@dataclass(frozen=True)
class Block:
    """Core extent owned exclusively; ext = core dilated by one, clipped
    (parallel.py:43-77).  Half-open (start, stop) per axis, x/y/z order."""

    index: tuple[int, int, int]
    core_start: tuple[int, int, int]
    core_stop: tuple[int, int, int]
    ext_start: tuple[int, int, int]
    ext_stop: tuple[int, int, int]

    @property
    def ext_dims(self) -> tuple[int, int, int]:
        return tuple(b - a for a, b in zip(self.ext_start, self.ext_stop))

    def ext_slices_zyx(self):
        return tuple(slice(self.ext_start[a], self.ext_stop[a]) for a in (2, 1, 0))

    def core_slices_zyx(self):
        return tuple(slice(self.core_start[a], self.core_stop[a]) for a in (2, 1, 0))

    def core_in_ext_slices_zyx(self):
        return tuple(slice(self.core_start[a] - self.ext_start[a], self.core_stop[a] - self.ext_start[a])
                     for a in (2, 1, 0))

    def core_mask_flat(self) -> np.ndarray:
        ex, ey, ez = self.ext_dims
        m = np.zeros((ez, ey, ex), dtype=bool)
        m[self.core_in_ext_slices_zyx()] = True
        return m.reshape(-1)


@dataclass(frozen=True)
class BlockDecomposition:
    dims: tuple[int, int, int]
    block_grid: tuple[int, int, int]
    blocks: tuple[Block, ...]


def _axis_splits(extent: int, parts: int) -> list[tuple[int, int]]:
    if parts < 1:
        raise ValueError(f"block count must be >= 1, got {parts}")
    if parts > extent:
        raise ValueError(f"cannot split extent {extent} into {parts} blocks")
    base, rem = divmod(extent, parts)
    spans, start = [], 0
    for i in range(parts):
        stop = start + base + (1 if i < rem else 0)
        spans.append((start, stop))
        start = stop
    return spans


def decompose(dims, block_grid) -> BlockDecomposition:
    """Near-equal cores, remainder to the leading blocks; blocks listed z-major
    then y then x (parallel.py:100-119)."""
    dims = tuple(int(d) for d in dims)
    block_grid = tuple(int(b) for b in block_grid)
    if len(dims) != 3 or len(block_grid) != 3:
        raise ValueError("dims and block_grid must be 3-tuples")
    splits = [_axis_splits(dims[a], block_grid[a]) for a in range(3)]
    blocks = []
    for bz in range(block_grid[2]):
        for by in range(block_grid[1]):
            for bx in range(block_grid[0]):
                cs = (splits[0][bx][0], splits[1][by][0], splits[2][bz][0])
                ce = (splits[0][bx][1], splits[1][by][1], splits[2][bz][1])
                es = tuple(max(0, s - 1) for s in cs)
                ee = tuple(min(dims[a], ce[a] + 1) for a in range(3))
                blocks.append(Block((bx, by, bz), cs, ce, es, ee))
    return BlockDecomposition(dims=dims, block_grid=block_grid, blocks=tuple(blocks))


def block_domain(block: Block, dims) -> DomainSpec:
    """Device domain of one block: ext dims, core box in ext coordinates and the
    replicated bands (multiplicity > 1, parallel.py:228-234): two layers at
    every face that borders another block."""
    ed = block.ext_dims
    lo = tuple(block.core_start[a] - block.ext_start[a] for a in range(3))
    hi = tuple(block.core_stop[a] - block.ext_start[a] for a in range(3))
    shl = tuple(min(2, ed[a]) if block.core_start[a] > 0 else 0 for a in range(3))
    shh = tuple(min(2, ed[a]) if block.core_stop[a] < dims[a] else 0 for a in range(3))
    return DomainSpec(ed, lo, hi, shl, shh)


@dataclass(frozen=True)
class ParallelStats:
    strategy: str
    block_grid: tuple[int, int, int]
    rounds: int
    syncs: int
    per_block_iterations: tuple[int, ...]
    per_block_edit_totals: tuple[int, ...]
    per_block_max_vertex_edits: tuple[int, ...]
    edit_count: int
    edit_ratio: float
    compute_seconds: float
    sync_seconds: float

    def to_dict(self) -> dict:
        return {"strategy": self.strategy, "block_grid": list(self.block_grid), "rounds": self.rounds,
                "syncs": self.syncs, "per_block_iterations": list(self.per_block_iterations),
                "per_block_edit_totals": list(self.per_block_edit_totals),
                "per_block_max_vertex_edits": list(self.per_block_max_vertex_edits),
                "edit_count": self.edit_count, "edit_ratio": self.edit_ratio,
                "timings": {"compute_seconds": self.compute_seconds, "sync_seconds": self.sync_seconds}}


class _DevBlock:
    def __init__(self, block: Block, dims, cfg: CorrectionConfig, f: torch.Tensor, fh: torch.Tensor):
        self.block = block
        self.spec = block_domain(block, dims)
        ed = self.spec.dims
        n = ed[0] * ed[1] * ed[2]
        f32 = f.dtype == torch.float32   # an f32-exact original (narrow_if_exact)
        self.f = torch.empty(n, dtype=f.dtype, device=f.device)
        self.fh = torch.empty(n, dtype=torch.float64, device=f.device)
        for src, dst, is32 in ((f, self.f, int(f32)), (fh, self.fh, 0)):
            N.check(N.lib().pmsz_box_extract(N.ivec(dims), N.ptr(src), is32, N.ivec(block.ext_start),
                                             N.ivec(ed), N.ptr(dst), N.stream_handle()), "pmsz_box_extract")
        self.g = torch.empty_like(self.fh)
        self.plan = DomainPlan(self.spec, cfg.xi_abs, cfg.tau, cfg.max_outer_iterations, incremental=True,
                               f32_original=f32)
        st, res = self.plan.prepare(self.f, self.fh, self.g)
        if st not in (N.PMSZ_OK,):
            raise_for(st, res, None, None, cfg.xi_abs, f_dev=self.f, fhat_dev=self.fh)
        self.iterations = 0
        self.edits = 0
        self.max_count = 0
        self.shared_dirty = False

    def round(self, lockstep: bool) -> int:
        st, e, res = self.plan.block_round(self.f, self.g, lockstep)
        if st == N.PMSZ_ERR_CONVERGENCE:
            raise ConvergenceError(f"block {self.block.index} found no zero-edit iteration within "
                                   f"{self.plan.max_iterations}")
        raise_for(st, res)
        self.iterations = int(res.iterations)
        self.edits = int(res.edit_count)
        self.max_count = int(res.max_vertex_edits)
        self.shared_dirty = self.shared_dirty or bool(res.shared_dirty)
        return e


def _merge_min_arrays(blocks, dims, arrays: list[torch.Tensor], acc: torch.Tensor) -> bool:
    """All replicas <- min over replicas for raw per-block ext arrays (device
    f64 tensors, updated in place); returns whether anything changed
    (parallel.py:122-140)."""
    L = N.lib()
    s = N.stream_handle()
    acc.fill_(float("inf"))
    zero = (0, 0, 0)
    for b, g in zip(blocks, arrays):
        hi = tuple(b.ext_start[a] + b.ext_dims[a] for a in range(3))
        N.check(L.pmsz_box_unpack_min(dims[0], dims[1], dims[2], N.ptr(acc), N.ivec(b.ext_start), N.ivec(hi),
                                      N.ptr(g), None, s), "pmsz_box_unpack_min")
    changed = torch.zeros(1, dtype=torch.int64, device=acc.device)
    for b, g in zip(blocks, arrays):
        ed = b.ext_dims
        hi = tuple(b.ext_start[a] + ed[a] for a in range(3))
        merged = torch.empty_like(g)
        N.check(L.pmsz_box_pack(dims[0], dims[1], dims[2], N.ptr(acc), N.ivec(b.ext_start), N.ivec(hi),
                                N.ptr(merged), s), "pmsz_box_pack")
        N.check(L.pmsz_box_unpack_copy(ed[0], ed[1], ed[2], N.ptr(g), N.ivec(zero), N.ivec(ed), N.ptr(merged),
                                       N.ptr(changed), s), "pmsz_box_unpack_copy")
    return bool(changed.item() > 0)


def sync_ghosts(decomposition: BlockDecomposition, g_exts) -> bool:
    """Public one-shot ghost exchange over raw per-block arrays
    (parallel.py:143-147): every replicated vertex <- the minimum over its
    replicas, in place; returns whether anything changed.  Host numpy arrays
    are merged on the device and written back into the same arrays; CUDA
    float64 tensors are merged in place."""
    if len(g_exts) != len(decomposition.blocks):
        raise ValueError("one array per block required")
    dims = decomposition.dims
    dev = torch.device("cuda", torch.cuda.current_device())
    arrays = []
    for b, a in zip(decomposition.blocks, g_exts):
        n = b.ext_dims[0] * b.ext_dims[1] * b.ext_dims[2]
        if isinstance(a, torch.Tensor) and a.is_cuda and a.dtype == torch.float64 and a.is_contiguous():
            t = a.view(-1)
        else:
            t = as_device_f64(np.asarray(a).reshape(-1), dev)
        if t.numel() != n:
            raise ValueError(f"block {b.index}: array has {t.numel()} values, ext extent has {n}")
        arrays.append(t)
    acc = torch.empty(dims[0] * dims[1] * dims[2], dtype=torch.float64, device=dev)
    changed = _merge_min_arrays(decomposition.blocks, dims, arrays, acc)
    for a, t in zip(g_exts, arrays):
        if not (isinstance(a, torch.Tensor) and a.is_cuda):
            np.asarray(a).reshape(-1)[:] = t.cpu().numpy()
    return changed


def local_converge(block: Block, f_ext, g_ext, lower_ext, config: CorrectionConfig
                   ) -> tuple[np.ndarray, int, int]:
    """Iterate one block to its local fixpoint, ghosts held fixed apart from
    the block's own edits (parallel.py:150-172): centres are the block's core,
    every ext vertex may be edited.  Returns (new g_ext, iterations counting
    the final zero-edit pass, total edits); g_ext itself is not modified.

    When ``lower_ext`` is exactly ``f_ext - xi`` and g_ext satisfies the error
    bound (the reference's own use) this is one device plan with the usual
    robust-centre skipping; otherwise the plan evaluates every centre and
    clamps to the given lower bound (PMSZ_FLAG_NO_ROBUST | PMSZ_FLAG_LOWER), so
    arbitrary inputs behave as in the reference, including its monotonicity
    AssertionError when g starts below the lower bound."""
    ed = tuple(int(v) for v in block.ext_dims)
    n = ed[0] * ed[1] * ed[2]
    dev = torch.device("cuda", torch.cuda.current_device())
    f = as_device_f64(np.asarray(f_ext).reshape(-1), dev)
    g0 = as_device_f64(np.asarray(g_ext).reshape(-1), dev)
    lower = as_device_f64(np.asarray(lower_ext).reshape(-1), dev)
    if not (f.numel() == g0.numel() == lower.numel() == n):
        raise ValueError(f"block {block.index}: arrays must hold the {n} values of the ext extent")
    lo = tuple(block.core_start[a] - block.ext_start[a] for a in range(3))
    hi = tuple(block.core_stop[a] - block.ext_start[a] for a in range(3))
    spec = DomainSpec(ed, lo, hi)
    cap = config.max_outer_iterations
    g = torch.empty_like(g0)
    exact = bool(torch.equal(lower, f - config.xi_abs))   # the IEEE subtraction numpy performs
    plan = None
    if exact:
        plan = DomainPlan(spec, config.xi_abs, config.tau, cap, incremental=True)
        st, res = plan.prepare(f, g0, g)
        if st == N.PMSZ_ERR_BOUND:   # g outside [f - xi, f + xi]: robust skipping is not valid
            plan.close()
            plan = None
        elif st != N.PMSZ_OK:
            raise_for(st, res, None, None, config.xi_abs, f_dev=f, fhat_dev=g0)
    operand = f
    if plan is None:
        plan = DomainPlan(spec, config.xi_abs, config.tau, cap, incremental=True, no_robust=True,
                          explicit_lower=True)
        st, res = plan.prepare(f, g0, g)
        if st not in (N.PMSZ_OK, N.PMSZ_ERR_BOUND):
            raise_for(st, res, None, None, config.xi_abs, f_dev=f, fhat_dev=g0)
        plan.floor_violations(lower, g)
        operand = lower
    try:
        st, _, res = plan.block_round(operand, g, lockstep=False)
        if st == N.PMSZ_ERR_CONVERGENCE:
            raise ConvergenceError(f"block {block.index} found no zero-edit iteration within {cap}")
        raise_for(st, res)
        return g.cpu().numpy(), int(res.iterations), int(res.edit_count)
    finally:
        plan.close()


def _merge_min(blocks: list[_DevBlock], dims, acc: torch.Tensor) -> bool:
    """All replicas <- min over replicas (parallel.py:122-140), on the device.
    Vertices whose value changed mark their 1-ring dirty for the next sweep."""
    L = N.lib()
    s = N.stream_handle()
    acc.fill_(float("inf"))
    zero = (0, 0, 0)
    for b in blocks:
        ed = b.spec.dims
        hi = tuple(b.block.ext_start[a] + ed[a] for a in range(3))
        N.check(L.pmsz_box_unpack_min(dims[0], dims[1], dims[2], N.ptr(acc), N.ivec(b.block.ext_start),
                                      N.ivec(hi), N.ptr(b.g), None, s), "pmsz_box_unpack_min")
    changed = torch.zeros(1, dtype=torch.int64, device=acc.device)
    for b in blocks:
        ed = b.spec.dims
        hi = tuple(b.block.ext_start[a] + ed[a] for a in range(3))
        merged = torch.empty_like(b.g)
        N.check(L.pmsz_box_pack(dims[0], dims[1], dims[2], N.ptr(acc), N.ivec(b.block.ext_start), N.ivec(hi),
                                N.ptr(merged), s), "pmsz_box_pack")
        before = b.g.clone()
        N.check(L.pmsz_box_unpack_copy(ed[0], ed[1], ed[2], N.ptr(b.g), N.ivec(zero), N.ivec(ed),
                                       N.ptr(merged), N.ptr(changed), s), "pmsz_box_unpack_copy")
        b.plan.mark_box_changed(zero, ed, before, b.g)
    return bool(changed.item() > 0)


def run_parallel(original: ScalarField, decompressed: ScalarField, config: CorrectionConfig,
                 block_grid, strategy: SyncStrategy = SyncStrategy.RELAXED, workers: int = 1
                 ) -> tuple[CorrectionResult, ParallelStats]:
    """Drop-in for topocorrect.run_parallel (parallel.py:258-367)."""
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    strategy = SyncStrategy(strategy)
    if original.dims != decompressed.dims:
        raise ValueError(f"dims differ: {original.dims} vs {decompressed.dims}")
    dims = original.dims
    dev = torch.device("cuda", torch.cuda.current_device())
    # f32-exact originals (f32 files, codec.py:86-87) are narrowed on the host
    # while staged and run the f32 K0 everywhere; others go up as f64
    f = as_device_narrowed(original.values, dev)
    f32 = f is not None
    if not f32:
        f = as_device_f64(original.values, dev)
    fh = as_device_f64(decompressed.values, dev)
    # validate_error_bound + global f-code for the final verification
    gplan = DomainPlan(DomainSpec.whole(dims), config.xi_abs, config.tau, config.max_outer_iterations,
                       incremental=False, f32_original=f32)
    scratch = torch.empty_like(fh)
    st, res = gplan.prepare(f, fh, scratch)
    raise_for(st, res, original.values, decompressed.values, config.xi_abs)
    decomp = decompose(dims, block_grid)
    blocks = [_DevBlock(b, dims, config, f, fh) for b in decomp.blocks]
    lockstep = strategy is SyncStrategy.LOCKSTEP
    rounds = syncs = 0
    totals: list[int] = []
    compute_s = sync_s = 0.0
    acc = torch.empty_like(fh)
    while True:
        if rounds >= config.max_outer_iterations:
            raise ConvergenceError(f"no terminal round within {config.max_outer_iterations}")
        rounds += 1
        t0 = time.perf_counter()
        round_edits = sum(b.round(lockstep) for b in blocks)
        compute_s += time.perf_counter() - t0
        totals.append(round_edits)
        if not lockstep:
            if round_edits == 0 or not any(b.shared_dirty for b in blocks):
                break
        t0 = time.perf_counter()
        changed = _merge_min(blocks, dims, acc)
        syncs += 1
        sync_s += time.perf_counter() - t0
        for b in blocks:
            b.shared_dirty = False
        if round_edits == 0 and not changed:
            break
    # assemble cores; every replica must agree (parallel.py:326-333)
    L = N.lib()
    s = N.stream_handle()
    out = torch.empty_like(fh)
    for b in blocks:
        blk = b.block
        lo = tuple(blk.core_start[a] - blk.ext_start[a] for a in range(3))
        hi = tuple(blk.core_stop[a] - blk.ext_start[a] for a in range(3))
        cd = tuple(hi[a] - lo[a] for a in range(3))
        buf = torch.empty(cd[0] * cd[1] * cd[2], dtype=torch.float64, device=dev)
        ed = b.spec.dims
        N.check(L.pmsz_box_pack(ed[0], ed[1], ed[2], N.ptr(b.g), N.ivec(lo), N.ivec(hi), N.ptr(buf), s),
                "pmsz_box_pack")
        N.check(L.pmsz_box_unpack_copy(dims[0], dims[1], dims[2], N.ptr(out), N.ivec(blk.core_start),
                                       N.ivec(blk.core_stop), N.ptr(buf), None, s), "pmsz_box_unpack_copy")
    for b in blocks:
        ed = b.spec.dims
        view = torch.empty_like(b.g)
        hi = tuple(b.block.ext_start[a] + ed[a] for a in range(3))
        N.check(L.pmsz_box_pack(dims[0], dims[1], dims[2], N.ptr(out), N.ivec(b.block.ext_start), N.ivec(hi),
                                N.ptr(view), s), "pmsz_box_pack")
        if not torch.equal(view, b.g):
            raise ConvergenceError("replicas diverged at termination")
    # post-verification (parallel.py:336-345)
    if gplan.bounds_violations(f, out) != 0:
        raise ConvergenceError("corrected field escaped the error bound")
    if any(gplan.verify(out)):
        raise ConvergenceError("distortions survived at termination")
    corrected = ScalarField._owned(dims, to_host_f64(out, recycle=True))
    # EditSet.diff (correction.py:363-369) on the device: ascending ids where g != fhat
    ids_d = torch.nonzero(out != fh).reshape(-1)
    edits = EditSet._owned(ids_d.cpu().numpy(), out[ids_d].cpu().numpy(), original.vertex_count)
    result = CorrectionResult(corrected=corrected, edits=edits,
                              iterations=max(b.iterations for b in blocks),
                              edits_per_iteration=tuple(totals),
                              max_vertex_edits=max(b.max_count for b in blocks),
                              verification=DistortionReport.clean())
    stats = ParallelStats(strategy=strategy.value, block_grid=tuple(int(v) for v in block_grid),
                          rounds=rounds, syncs=syncs,
                          per_block_iterations=tuple(b.iterations for b in blocks),
                          per_block_edit_totals=tuple(b.edits for b in blocks),
                          per_block_max_vertex_edits=tuple(b.max_count for b in blocks),
                          edit_count=edits.count, edit_ratio=edits.ratio,
                          compute_seconds=compute_s, sync_seconds=sync_s)
    return result, stats
