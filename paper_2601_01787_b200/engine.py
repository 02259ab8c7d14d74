"""Device plans: one correction domain bound to libpmsz (host side of the C ABI).

A :class:`DomainPlan` owns the device scratch of one domain (the whole grid,
or one block's extended extent) and drives the kernels K0 (prepare), K1/K2
(iterate), K4 (verify) and K5 (edit export).  Device buffers are torch CUDA
tensors; only raw pointers cross the C ABI.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N


class BoundViolationError(ValueError):
    """The decompressed field strays beyond the stated error bound
    (correction.py:33-45: same fields and message)."""

    def __init__(self, index, original, decompressed, xi_abs, offenders):
        self.index = int(index)
        self.original = float(original)
        self.decompressed = float(decompressed)
        self.xi_abs = float(xi_abs)
        self.offenders = int(offenders)
        super().__init__(
            f"error bound violated at vertex {self.index}: "
            f"|{self.original!r} - {self.decompressed!r}| > {self.xi_abs!r} "
            f"(first of {self.offenders} offending vertices)")


class ConvergenceError(RuntimeError):
    """Correction failed to reach a distortion-free state (correction.py:48-49)."""


@dataclass(frozen=True)
class DomainSpec:
    dims: tuple[int, int, int]
    core_lo: tuple[int, int, int]
    core_hi: tuple[int, int, int]
    shared_lo: tuple[int, int, int] = (0, 0, 0)
    shared_hi: tuple[int, int, int] = (0, 0, 0)

    @staticmethod
    def whole(dims) -> "DomainSpec":
        d = tuple(int(v) for v in dims)
        return DomainSpec(d, (0, 0, 0), d)


class DomainPlan:
    """One pmsz_plan (see include/pmsz.h)."""

    def __init__(self, spec: DomainSpec, xi: float, tau: float, max_iterations: int,
                 *, incremental: bool = True, extrema_only: bool = False,
                 f32_original: bool = False, host_loop: bool = False, no_robust: bool = False,
                 explicit_lower: bool = False, host_f64: bool = False):
        self.lib = N.lib()
        self.spec = spec
        self.xi, self.tau, self.max_iterations = float(xi), float(tau), int(max_iterations)
        self.f32_original = bool(f32_original)
        d = N.PmszDesc()
        d.nx, d.ny, d.nz = spec.dims
        for a in range(3):
            d.core_lo[a] = spec.core_lo[a]
            d.core_hi[a] = spec.core_hi[a]
            d.shared_lo[a] = spec.shared_lo[a]
            d.shared_hi[a] = spec.shared_hi[a]
        d.xi, d.tau, d.max_iterations = self.xi, self.tau, self.max_iterations
        d.flags = ((N.FLAG_INCREMENTAL if incremental else 0)
                   | (N.FLAG_EXTREMA_ONLY if extrema_only else 0)
                   | (N.FLAG_F32_ORIGINAL if f32_original else 0)
                   | (N.FLAG_HOST_LOOP if host_loop else 0)
                   | (N.FLAG_NO_ROBUST if no_robust else 0)
                   | (N.FLAG_LOWER if explicit_lower else 0)
                   | (N.FLAG_HOST_F64 if host_f64 else 0))
        h = ctypes.c_void_p()
        st = self.lib.pmsz_plan_create(ctypes.byref(d), ctypes.byref(h))
        if st == N.PMSZ_ERR_INVALID:
            raise ValueError(N.last_error())
        N.check(st, "pmsz_plan_create")
        self.handle = h
        self.n = spec.dims[0] * spec.dims[1] * spec.dims[2]
        import threading
        self.lock = threading.RLock()   # a plan runs one correction at a time (cached plans are shared)

    def close(self):
        if getattr(self, "handle", None):
            self.lib.pmsz_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def profile(self, enable: bool = True, full_domain_only: bool = False):
        """Per-class kernel timing by CUDA events; full_domain_only: only the
        PREP / SWEEP_FULL / VERIFY launches (cheap enough for a timed region)."""
        mode = (2 if full_domain_only else 1) if enable else 0
        N.check(self.lib.pmsz_profile(self.handle, mode), "pmsz_profile")

    def profile_read(self, reset: bool = False) -> dict:
        ms = (ctypes.c_double * N.K_COUNT)()
        cnt = (ctypes.c_int64 * N.K_COUNT)()
        N.check(self.lib.pmsz_profile_read(self.handle, ms, cnt, int(bool(reset))), "pmsz_profile_read")
        return {name: (float(ms[k]), int(cnt[k])) for k, name in enumerate(N.K_NAMES)}

    @property
    def scratch_bytes(self) -> int:
        return int(self.lib.pmsz_plan_scratch_bytes(self.handle))

    # -- whole run -----------------------------------------------------------
    HIST_BUF = 4096

    def run(self, f: torch.Tensor, fhat: torch.Tensor, g: torch.Tensor, stream=None):
        """pmsz_run_correction; returns (status, PmszResult, history list).  The
        history buffer is a fixed chunk; longer runs read the plan's full
        history afterwards (pmsz_history), so a huge iteration cap costs nothing."""
        cap = min(self.max_iterations, self.HIST_BUF)
        hist = (ctypes.c_int64 * cap)()
        res = N.PmszResult()
        st = self.lib.pmsz_run_correction(self.handle, N.ptr(f), N.ptr(fhat), N.ptr(g), hist, cap,
                                          ctypes.byref(res), N.stream_handle(stream))
        n_hist = int(res.iterations)
        if n_hist <= cap:
            return st, res, [int(hist[i]) for i in range(n_hist)]
        return st, res, self.history()

    def run_export(self, f: torch.Tensor, fhat: torch.Tensor, g: torch.Tensor, stream=None):
        """pmsz_run_correction + the edit export in one C call (no host gap
        before the export): the record lands in tensors sized by the last
        run's count (+5 %); a larger record is exported again at its size.
        Returns (status, PmszResult, history, ids, vals)."""
        cap = min(self.max_iterations, self.HIST_BUF)
        hist = (ctypes.c_int64 * cap)()
        res = N.PmszResult()
        ecap = getattr(self, "_ecap", 0)
        ids = torch.empty(ecap, dtype=torch.int64, device=g.device)
        vals = torch.empty(ecap, dtype=torch.float64, device=g.device)
        st = self.lib.pmsz_run_correction_export(self.handle, N.ptr(f), N.ptr(fhat), N.ptr(g), hist, cap,
                                                 ctypes.byref(res), N.ptr(ids) if ecap else None,
                                                 N.ptr(vals) if ecap else None, ecap, N.stream_handle(stream))
        n_hist = int(res.iterations)
        history = [int(hist[i]) for i in range(n_hist)] if n_hist <= cap else self.history()
        if st != N.PMSZ_OK:
            return st, res, history, None, None
        m = int(res.edit_count)
        self._ecap = m + m // 20 + 1024
        if m <= ecap:
            return st, res, history, ids[:m], vals[:m]
        ids, vals = self.export_edits(g, stream=stream)
        return st, res, history, ids, vals

    def run_host(self, f: np.ndarray, fhat: np.ndarray, g: np.ndarray | None):
        """pmsz_run_correction_host on host arrays (pageable or pinned): f (f64,
        or f32 with f32_original; f64 with host_f64), fhat f64, g the f64
        corrected field out (or None).  Returns (status, PmszResult, history,
        edit ids, edit values); the record is read back from the plan
        (pmsz_edits_host) when g is given."""
        cap = min(self.max_iterations, self.HIST_BUF)
        hist = (ctypes.c_int64 * cap)()
        res = N.PmszResult()
        st = self.lib.pmsz_run_correction_host(self.handle, f.ctypes.data, fhat.ctypes.data,
                                               None if g is None else g.ctypes.data, None, None, 0,
                                               hist, cap, ctypes.byref(res), None)
        n_hist = int(res.iterations)
        history = [int(hist[i]) for i in range(n_hist)] if n_hist <= cap else self.history()
        if st != N.PMSZ_OK or g is None:
            return st, res, history, None, None
        m = int(res.edit_count)
        ids = np.empty(m, dtype=np.int64)
        vals = np.empty(m, dtype=np.float64)
        cnt = ctypes.c_int64()
        N.check(self.lib.pmsz_edits_host(self.handle, ids.ctypes.data, vals.ctypes.data, m, ctypes.byref(cnt)),
                "pmsz_edits_host")
        return st, res, history, ids, vals

    def history(self) -> list[int]:
        """edits_per_iteration of the plan's last run (pmsz_history)."""
        cnt = ctypes.c_int64()
        N.check(self.lib.pmsz_history(self.handle, None, 0, ctypes.byref(cnt)), "pmsz_history")
        buf = (ctypes.c_int64 * max(1, cnt.value))()
        N.check(self.lib.pmsz_history(self.handle, buf, cnt.value, ctypes.byref(cnt)), "pmsz_history")
        return [int(buf[i]) for i in range(cnt.value)]

    def export_edits(self, g: torch.Tensor, stream=None) -> tuple[torch.Tensor, torch.Tensor]:
        cnt = ctypes.c_int64()
        N.check(self.lib.pmsz_edits_export(self.handle, N.ptr(g), None, None, 0, ctypes.byref(cnt),
                                           N.stream_handle(stream)), "pmsz_edits_export")
        m = int(cnt.value)
        ids = torch.empty(m, dtype=torch.int64, device=g.device)
        vals = torch.empty(m, dtype=torch.float64, device=g.device)
        if m:
            N.check(self.lib.pmsz_edits_export(self.handle, N.ptr(g), N.ptr(ids), N.ptr(vals), m,
                                               ctypes.byref(cnt), N.stream_handle(stream)),
                    "pmsz_edits_export")
        return ids, vals

    # -- stepwise (block engine) ---------------------------------------------
    def prepare(self, f, fhat, g, stream=None) -> N.PmszResult:
        res = N.PmszResult()
        st = self.lib.pmsz_prepare(self.handle, N.ptr(f), N.ptr(fhat), N.ptr(g), ctypes.byref(res),
                                   N.stream_handle(stream))
        return st, res

    def iterate(self, f, g, edited_mask=None, stream=None):
        res = N.PmszResult()
        st = self.lib.pmsz_iterate(self.handle, N.ptr(f), N.ptr(g),
                                   N.ptr(edited_mask) if edited_mask is not None else None,
                                   ctypes.byref(res), N.stream_handle(stream))
        return st, res

    def block_round(self, f, g, lockstep: bool, stream=None):
        res = N.PmszResult()
        e = ctypes.c_int64()
        st = self.lib.pmsz_block_round(self.handle, N.ptr(f), N.ptr(g), int(bool(lockstep)),
                                       ctypes.byref(e), ctypes.byref(res), N.stream_handle(stream))
        return st, int(e.value), res

    def verify(self, g, stream=None):
        res = N.PmszResult()
        st = self.lib.pmsz_verify(self.handle, N.ptr(g), ctypes.byref(res), N.stream_handle(stream))
        N.check(st, "pmsz_verify")
        return [int(res.residual[k]) for k in range(6)]

    def floor_violations(self, lower, g, stream=None) -> int:
        """Vertices with g < lower (explicit-lower plans); arms the monotonicity check."""
        out = ctypes.c_int64()
        N.check(self.lib.pmsz_floor_violations(self.handle, N.ptr(lower), N.ptr(g), ctypes.byref(out),
                                               N.stream_handle(stream)), "pmsz_floor_violations")
        return int(out.value)

    def bounds_violations(self, f, g, stream=None) -> int:
        out = ctypes.c_int64()
        N.check(self.lib.pmsz_bounds_violations(self.handle, N.ptr(f), N.ptr(g), ctypes.byref(out),
                                                N.stream_handle(stream)), "pmsz_bounds_violations")
        return int(out.value)

    def merge_min(self, g, lo, hi, buf, stream=None, count: bool = True) -> int:
        """Ghost merge of a received replica box; changed vertices dirty their ring.
        count=False: no host synchronisation (returns -1; the plan reads its
        marking counters at the next iteration)."""
        out = ctypes.c_int64(-1)
        N.check(self.lib.pmsz_box_merge_min(self.handle, N.ptr(g), N.ivec(lo), N.ivec(hi), N.ptr(buf),
                                            ctypes.byref(out) if count else None, N.stream_handle(stream)),
                "pmsz_box_merge_min")
        return int(out.value)

    def residual(self, stream=None) -> int:
        out = ctypes.c_int64()
        N.check(self.lib.pmsz_residual(self.handle, ctypes.byref(out), N.stream_handle(stream)), "pmsz_residual")
        return int(out.value)

    def mark_all_dirty(self):
        N.check(self.lib.pmsz_mark_all_dirty(self.handle, None), "pmsz_mark_all_dirty")

    def mark_box_changed(self, lo, hi, before: torch.Tensor, g: torch.Tensor, stream=None):
        N.check(self.lib.pmsz_box_mark_changed(self.handle, N.ivec(lo), N.ivec(hi), N.ptr(before),
                                               N.ptr(g), N.stream_handle(stream)),
                "pmsz_box_mark_changed")


def raise_for(status: int, res: N.PmszResult, f_host_values=None, fhat_host_values=None,
              xi: float | None = None, f_dev=None, fhat_dev=None):
    """Map a pmsz_status to the reference's exception (correction.py:33-60,417-429)."""
    if status == N.PMSZ_OK:
        return
    msg = N.last_error()
    if status == N.PMSZ_ERR_BOUND:
        i = int(res.bound_first_index)
        if f_host_values is not None:
            fo, fd = f_host_values[i], fhat_host_values[i]
        else:
            fo, fd = float(f_dev[i].item()), float(fhat_dev[i].item())
        raise BoundViolationError(i, fo, fd, xi, int(res.bound_violations))
    if status == N.PMSZ_ERR_MONOTONE:
        raise AssertionError("edit raised a value; monotonicity broken")
    if status == N.PMSZ_ERR_CONVERGENCE:
        raise ConvergenceError(msg)
    if status in (N.PMSZ_ERR_INVALID, N.PMSZ_ERR_NONFINITE):
        raise ValueError(msg)
    raise RuntimeError(f"pMSz device failure (status {status}): {msg}")


def default_cap(xi: float, tau: float) -> int:
    return 10 * math.ceil(2.0 * xi / tau)


def narrow_if_exact(f64: torch.Tensor) -> torch.Tensor | None:
    """The f32 copy of a device f64 field when every value survives the round
    trip (fields read from f32 files, codec.py:86-87), else None."""
    out = torch.empty(f64.numel(), dtype=torch.float32, device=f64.device)
    bad = ctypes.c_int64()
    N.check(N.lib().pmsz_narrow_f32(N.ptr(f64), f64.numel(), N.ptr(out), ctypes.byref(bad), N.stream_handle()),
            "pmsz_narrow_f32")
    return out if bad.value == 0 else None


class HostFieldCache:
    """Recycled host arrays for corrected fields (the drop-in's output).

    A fresh 1 GB numpy array costs ~15-20 ms of page faults and kernel
    zeroing before the first value lands (measured on the B200 boxes' hosts;
    DESIGN.md §8), on a path that is host-memory-bound.  Like a caching host
    allocator, this keeps the arrays it handed out and reuses one once nobody
    else references it: every numpy view, slice or memoryview of the array
    holds a reference to it (views collapse their base to the owning array),
    so a reference count at the cache's own baseline means it is free.  At
    most ``max_idle`` idle arrays are kept; ``PMSZ_HOST_CACHE=0`` disables
    the cache, ``empty_host_cache()`` drops the idle arrays."""

    def __init__(self, max_idle: int = 2):
        import os
        import threading
        self.enabled = os.environ.get("PMSZ_HOST_CACHE", "1") != "0"
        self.max_idle = max_idle
        self.arrays: list[np.ndarray] = []
        self._lock = threading.Lock()   # two threads must not both take one idle array

    def _idle(self, i: int) -> bool:
        import sys
        # references: the cache's list and getrefcount's argument only
        return sys.getrefcount(self.arrays[i]) <= 2

    def take(self, n: int) -> np.ndarray:
        if not self.enabled:
            return np.empty(n, dtype=np.float64)
        with self._lock:
            return self._take(n)

    def _take(self, n: int) -> np.ndarray:
        hit = next((i for i in range(len(self.arrays)) if self.arrays[i].size == n and self._idle(i)), None)
        if hit is not None:
            self.arrays.append(self.arrays.pop(hit))     # most recently used last
        # keep at most max_idle spare arrays besides the one handed out
        idle = [i for i in range(len(self.arrays) - (hit is not None)) if self._idle(i)]
        if len(idle) > self.max_idle - (hit is None):
            drop = set(idle[:len(idle) - self.max_idle + (hit is None)])
            self.arrays = [self.arrays[i] for i in range(len(self.arrays)) if i not in drop]
        if hit is None:
            self.arrays.append(np.empty(n, dtype=np.float64))
        return self.arrays[-1]

    def clear(self):
        with self._lock:
            keep = [i for i in range(len(self.arrays)) if not self._idle(i)]
            self.arrays = [self.arrays[i] for i in keep]


HOST_FIELDS = HostFieldCache()


def empty_host_cache() -> None:
    """Release the idle recycled host field arrays (HostFieldCache)."""
    HOST_FIELDS.clear()


_STAGED_MIN_BYTES = 8 << 20   # below this the driver's own pageable copy is as fast


def to_host_f64(t: torch.Tensor, recycle: bool = False) -> np.ndarray:
    """Device f64 tensor -> a fresh (or, with ``recycle``, a recycled
    HostFieldCache) numpy array.  Large tensors go through the staged copy
    (pmsz_device_to_host: pinned ring + host threads, streaming stores)."""
    n = t.numel()
    out = HOST_FIELDS.take(n) if recycle else np.empty(n, dtype=np.float64)
    src = t.reshape(-1)
    if n * 8 >= _STAGED_MIN_BYTES and src.is_cuda:
        N.check(N.lib().pmsz_device_to_host(out.ctypes.data, N.ptr(src), n * 8, N.stream_handle()),
                "pmsz_device_to_host")
    else:
        torch.from_numpy(out).copy_(src)
    return out


def as_device_f64(values: np.ndarray, device) -> torch.Tensor:
    """Host f64 array -> device tensor without an extra host copy (the source
    may be a frozen ScalarField array; it is only read).  Large arrays go
    through the staged copy (pmsz_host_to_device)."""
    import warnings
    src = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
    if src.nbytes >= _STAGED_MIN_BYTES and torch.device(device).type == "cuda":
        out = torch.empty(src.size, dtype=torch.float64, device=device)
        N.check(N.lib().pmsz_host_to_device(N.ptr(out), src.ctypes.data, src.nbytes, 0, None, N.stream_handle()),
                "pmsz_host_to_device")
        return out
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        return torch.from_numpy(src).to(device)


def as_device_narrowed(values: np.ndarray, device) -> torch.Tensor | None:
    """Host f64 array -> device f32 tensor when every value survives the round
    trip (fields read from f32 files, codec.py:86-87), narrowed on the host
    while it is staged; None otherwise (the caller uploads f64)."""
    src = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
    out = torch.empty(src.size, dtype=torch.float32, device=device)
    bad = ctypes.c_int64()
    N.check(N.lib().pmsz_host_to_device(N.ptr(out), src.ctypes.data, src.size, 1, ctypes.byref(bad),
                                        N.stream_handle()), "pmsz_host_to_device")
    return out if bad.value == 0 else None
