"""Synthetic benchmark inputs generated on the GPU.

* ``perlin`` -- synth.perlin (synth.py:83-100), bit-exact (kernel built with
  --fmad=false, same evaluation order); the permutation table is
  synth._permutation (RandomState(seed).permutation(256), synth.py:33-37),
  computed here on the host with NumPy exactly as the reference does.
* ``quantize`` -- quantizer.quantize (quantizer.py:122-154), the bounded-error
  stand-in for SZ3.
* ``bounded_noise`` -- BASELINE config 1's seeded bounded-noise decompressed
  field (no reference counterpart; the oracle restates the same hash).
* ``relative_to_absolute`` -- quantizer.py:99-113 from a device min/max.
* ``gaussian_peaks`` -- BASELINE config 5's HEDM-like Gaussian-peak stack
  (no reference counterpart; definition in csrc/gen.cuh, restated
  bit for bit by the oracle's orc_peaks).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N


@dataclass(frozen=True)
class NoiseSpec:
    dims: tuple[int, int, int]
    seed: int
    frequency: float = 4.0
    octaves: int = 3

    def __post_init__(self):
        d = tuple(int(v) for v in self.dims)
        object.__setattr__(self, "dims", d if len(d) == 3 else (d[0], d[1], 1))
        if self.octaves < 1:
            raise ValueError("octaves must be >= 1")
        if not self.frequency > 0:
            raise ValueError("frequency must be positive")


def permutation_table(seed: int) -> np.ndarray:
    table = np.random.RandomState(seed & 0xFFFFFFFF).permutation(256)
    return np.concatenate([table, table]).astype(np.int32)


def perlin_device(spec: NoiseSpec, *, lo=(0, 0, 0), ext=None, f32: bool = False,
                  device=None) -> torch.Tensor:
    """Perlin values of the sub-box [lo, lo+ext) of the global grid spec.dims
    (float64, or float32 = the reference's f32 cast)."""
    ext = tuple(spec.dims) if ext is None else tuple(int(v) for v in ext)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    n = ext[0] * ext[1] * ext[2]
    out = torch.empty(n, dtype=torch.float32 if f32 else torch.float64, device=dev)
    perm = permutation_table(spec.seed)
    permp = perm.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    N.check(N.lib().pmsz_perlin(N.ivec(spec.dims), N.ivec(lo), N.ivec(ext), permp,
                                float(spec.frequency), int(spec.octaves),
                                None if f32 else N.ptr(out), N.ptr(out) if f32 else None,
                                N.stream_handle()), "pmsz_perlin")
    return out


def minmax_device(values: torch.Tensor) -> tuple[float, float]:
    mn, mx = ctypes.c_double(), ctypes.c_double()
    N.check(N.lib().pmsz_minmax(N.ptr(values), int(values.dtype == torch.float32), values.numel(),
                                ctypes.byref(mn), ctypes.byref(mx), N.stream_handle()), "pmsz_minmax")
    return float(mn.value), float(mx.value)


def relative_to_absolute_range(lo: float, hi: float, eb_rel: float) -> float:
    """quantizer.relative_to_absolute (quantizer.py:99-113) given min/max."""
    if not (eb_rel > 0 and np.isfinite(eb_rel)):
        raise ValueError(f"relative error bound must be positive, got {eb_rel}")
    if hi > lo:
        return eb_rel * (hi - lo)
    if hi != 0.0:
        return eb_rel * abs(hi)
    raise ValueError("relative bound undefined for an all-zero field")


def relative_to_absolute_device(values: torch.Tensor, eb_rel: float) -> float:
    lo, hi = minmax_device(values)
    return relative_to_absolute_range(lo, hi, eb_rel)


def quantize_device(f: torch.Tensor, xi: float, origin: float | None = None,
                    fmax: float | None = None) -> torch.Tensor:
    """Reconstructed field of quantizer.quantize (float64 tensor)."""
    if not (xi > 0 and np.isfinite(xi)):
        raise ValueError(f"absolute error bound must be positive, got {xi}")
    if origin is None or fmax is None:
        origin, fmax = minmax_device(f)
    if (fmax - origin) / (2.0 * xi) > 2.0 ** 53:
        raise ValueError("error bound too small for the field's value range")
    out = torch.empty(f.numel(), dtype=torch.float64, device=f.device)
    mc = ctypes.c_int64()
    st = N.lib().pmsz_quantize(N.ptr(f), int(f.dtype == torch.float32), f.numel(), float(origin),
                               float(xi), N.ptr(out), ctypes.byref(mc), N.stream_handle())
    if st != N.PMSZ_OK:
        raise AssertionError(N.last_error())
    return out


def bounded_noise_device(f: torch.Tensor, dims, xi: float, seed: int, *, gdims=None,
                         lo=(0, 0, 0)) -> torch.Tensor:
    nx, ny, nz = dims
    gd = tuple(gdims) if gdims is not None else (nx, ny, nz)
    out = torch.empty(f.numel(), dtype=torch.float64, device=f.device)
    N.check(N.lib().pmsz_bounded_noise(N.ptr(f), int(f.dtype == torch.float32), nx, ny, nz,
                                       N.ivec(gd), N.ivec(lo), float(xi), int(seed) & (2**64 - 1),
                                       N.ptr(out), N.stream_handle()), "pmsz_bounded_noise")
    return out


@dataclass(frozen=True)
class PeakSpec:
    """HEDM-like Gaussian-peak stack: detector frames along z with sparse
    spots in (64, 64, 32)-voxel cells over a faint background (gen.cuh)."""

    dims: tuple[int, int, int]
    seed: int


def gaussian_peaks_device(spec: PeakSpec, *, lo=(0, 0, 0), ext=None, f32: bool = False,
                          device=None) -> torch.Tensor:
    """The sub-box [lo, lo+ext) of the peak stack (f64, or f32 if requested)."""
    gd = tuple(int(v) for v in spec.dims)
    e = tuple(int(v) for v in (ext if ext is not None else gd))
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    out = torch.empty(e[0] * e[1] * e[2], dtype=torch.float32 if f32 else torch.float64, device=dev)
    N.check(N.lib().pmsz_gaussian_peaks(N.ivec(gd), N.ivec(lo), N.ivec(e), int(spec.seed) & (2**64 - 1), int(f32),
                                        N.ptr(out), N.stream_handle()), "pmsz_gaussian_peaks")
    return out


# ---- the reference's host-facing generators (drop-in names) -----------------
@dataclass(frozen=True, eq=False)
class QuantizedPayload:
    """quantizer.QuantizedPayload (quantizer.py:28-44): the quantizer's codes
    and what reconstructs the field from them.  (The bit-packed byte form,
    to_bytes / from_bytes, is the codec -- out of scope.)"""
    dims: tuple[int, int, int]
    xi_abs: float
    origin: float
    bit_width: int
    codes: np.ndarray
    payload_bytes: int


def perlin(spec: NoiseSpec):
    """synth.perlin (synth.py:83-100): the field as a ScalarField, generated on
    the device bit for bit."""
    from .engine import to_host_f64
    from .grid import ScalarField
    return ScalarField._owned(spec.dims, to_host_f64(perlin_device(spec)))


def relative_to_absolute(field, eb_rel: float) -> float:
    """quantizer.relative_to_absolute (quantizer.py:99-113)."""
    v = field.values
    return relative_to_absolute_range(float(v.min()), float(v.max()), eb_rel)


def quantize(field, xi_abs: float):
    """quantizer.quantize (quantizer.py:122-154) -> (QuantizedPayload, ScalarField):
    codes and reconstruction computed on the device (with the ulp repair)."""
    from .engine import as_device_f64, to_host_f64
    from .grid import ScalarField
    if not (xi_abs > 0 and np.isfinite(xi_abs)):
        raise ValueError(f"absolute error bound must be positive, got {xi_abs}")
    f = field.values
    origin, fmax = float(f.min()), float(f.max())
    if (fmax - origin) / (2.0 * xi_abs) > 2.0 ** 53:
        raise ValueError("error bound too small for the field's value range")
    fd = as_device_f64(f, torch.device("cuda", torch.cuda.current_device()))
    recon = torch.empty(fd.numel(), dtype=torch.float64, device=fd.device)
    codes = torch.empty(fd.numel(), dtype=torch.int64, device=fd.device)
    mc = ctypes.c_int64()
    st = N.lib().pmsz_quantize_codes(N.ptr(fd), 0, fd.numel(), origin, float(xi_abs), N.ptr(recon), N.ptr(codes),
                                     ctypes.byref(mc), N.stream_handle())
    if st != N.PMSZ_OK:
        raise AssertionError(N.last_error())
    codes_h = codes.cpu().numpy().view(np.uint64)
    codes_h.setflags(write=False)
    bit_width = max(1, int(mc.value).bit_length())
    ndims = 2 if field.dims[2] == 1 else 3
    n = field.vertex_count
    size = 25 + 8 * ndims + (n * bit_width + 7) // 8 + 4
    payload = QuantizedPayload(dims=field.dims, xi_abs=float(xi_abs), origin=origin, bit_width=bit_width,
                               codes=codes_h, payload_bytes=size)
    return payload, ScalarField._owned(field.dims, to_host_f64(recon))


def reconstruct(payload: QuantizedPayload):
    """quantizer.reconstruct (quantizer.py:157-159): origin + code * (2 xi)."""
    from .grid import ScalarField
    values = payload.origin + payload.codes.astype(np.float64) * (2.0 * payload.xi_abs)
    return ScalarField(payload.dims, values)


class PayloadFormatError(ValueError):
    """quantizer.PayloadFormatError: a malformed payload byte string."""


def ramp(dims, coefficients=(1.0, 2.0, 4.0)):
    """synth.ramp (synth.py:108-116): c0 x + c1 y + c2 z, no interior extrema."""
    from .grid import ScalarField
    d = tuple(int(v) for v in dims)
    nx, ny, nz = d if len(d) == 3 else (d[0], d[1], 1)
    c = tuple(float(v) for v in coefficients) + (0.0, 0.0, 0.0)
    z, y, x = np.meshgrid(np.arange(nz, dtype=np.float64), np.arange(ny, dtype=np.float64),
                          np.arange(nx, dtype=np.float64), indexing="ij")
    return ScalarField((nx, ny, nz), (c[0] * x + c[1] * y + c[2] * z).reshape(-1))


def constant(dims, value: float = 0.0):
    """synth.constant (synth.py:119-121)."""
    from .grid import ScalarField
    d = tuple(int(v) for v in dims)
    nx, ny, nz = d if len(d) == 3 else (d[0], d[1], 1)
    return ScalarField((nx, ny, nz), np.full(nx * ny * nz, float(value)))
