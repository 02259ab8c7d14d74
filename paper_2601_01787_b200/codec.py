"""File formats of the path's inputs and outputs (codec.py).

Edit records (PMSZE), the "edit record out" side of the drop-in
(codec.py:138-186): header ``<6sBddQQ`` (magic, version, xi_abs, tau, vertex
count, edit count), delta-coded LEB128 ids (the first id absolute), the f64
values, CRC32 of all preceding bytes.  The delta/varint packing is vectorised
with NumPy here.

Fields and segmentation labels (PMSZF, codec.py:40-110): header ``<6sBBB``
(magic, version, dtype code 1 = f32 / 2 = f64 / 3 = u64 labels, stored
extent count 2 or 3) and the extents as u64 (nz = 1 is not stored), then the
little-endian payload.
"""

from __future__ import annotations

import struct
import zlib

import numpy as np

from .correction import EditSet

EDITS_MAGIC = b"PMSZE\x00"
EDITS_VERSION = 1
_HEAD = "<6sBddQQ"


class FormatError(ValueError):
    pass


FIELD_MAGIC = b"PMSZF\x00"
FIELD_VERSION = 1
DTYPE_F32, DTYPE_F64, DTYPE_U64 = 1, 2, 3
_FIELD_NP = {DTYPE_F32: "<f4", DTYPE_F64: "<f8", DTYPE_U64: "<u8"}


def _field_head(code: int, dims) -> bytes:
    dims = tuple(int(d) for d in dims)
    stored = dims[:2] if dims[2] == 1 else dims
    return struct.pack("<6sBBB", FIELD_MAGIC, FIELD_VERSION, code, len(stored)) + struct.pack(
        f"<{len(stored)}Q", *stored)


def _field_parse(data: bytes):
    if len(data) < 9:
        raise FormatError("field file truncated")
    magic, version, code, nd = struct.unpack_from("<6sBBB", data, 0)
    if magic != FIELD_MAGIC:
        raise FormatError(f"bad field magic {magic!r}")
    if version != FIELD_VERSION:
        raise FormatError(f"unsupported field version {version}")
    if code not in _FIELD_NP:
        raise FormatError(f"unknown dtype code {code}")
    if nd not in (2, 3):
        raise FormatError(f"ndims must be 2 or 3, got {nd}")
    if len(data) < 9 + 8 * nd:
        raise FormatError("field file truncated")
    ext = tuple(int(v) for v in struct.unpack_from(f"<{nd}Q", data, 9))
    return code, (ext if nd == 3 else ext + (1,)), 9 + 8 * nd


def write_field(field, precision: str = "f64") -> bytes:
    if precision not in ("f64", "f32"):
        raise ValueError(f"precision must be 'f32' or 'f64', got {precision!r}")
    code = DTYPE_F64 if precision == "f64" else DTYPE_F32
    return _field_head(code, field.dims) + np.asarray(field.values).astype(_FIELD_NP[code]).tobytes()


def read_field(data: bytes):
    """Field file -> ScalarField (f32 payloads promoted exactly to f64)."""
    from .grid import ScalarField
    code, dims, off = _field_parse(data)
    if code == DTYPE_U64:
        raise FormatError("file holds labels, not scalar values")
    n = dims[0] * dims[1] * dims[2]
    dt = np.dtype(_FIELD_NP[code])
    if len(data) != off + n * dt.itemsize:
        raise FormatError(f"field payload length {len(data) - off} does not match dims {dims}")
    return ScalarField(dims, np.frombuffer(data, dtype=dt, count=n, offset=off).astype(np.float64))


def write_labels(dims, labels) -> bytes:
    dims = tuple(int(d) for d in dims) + ((1,) if len(dims) == 2 else ())
    lab = np.ascontiguousarray(np.asarray(labels), dtype=np.int64).reshape(-1)
    n = dims[0] * dims[1] * dims[2]
    if lab.size != n:
        raise ValueError(f"expected {n} labels for dims {dims}, got {lab.size}")
    if lab.size and (lab.min() < 0 or lab.max() >= n):
        raise ValueError("labels must be vertex ids of the same grid")
    return _field_head(DTYPE_U64, dims) + lab.astype("<u8").tobytes()


def read_labels(data: bytes):
    code, dims, off = _field_parse(data)
    if code != DTYPE_U64:
        raise FormatError("file holds scalar values, not labels")
    n = dims[0] * dims[1] * dims[2]
    if len(data) != off + n * 8:
        raise FormatError(f"label payload length {len(data) - off} does not match dims {dims}")
    return dims, np.frombuffer(data, dtype="<u8", count=n, offset=off).astype(np.int64)


def _leb128(values: np.ndarray) -> bytes:
    """Unsigned LEB128 of every value, concatenated (vectorised)."""
    v = np.asarray(values, dtype=np.uint64)
    if v.size == 0:
        return b""
    nbytes = np.ones(v.size, dtype=np.int64)
    t = v >> np.uint64(7)
    while t.any():
        nbytes += (t != 0)
        t >>= np.uint64(7)
    total = int(nbytes.sum())
    out = np.empty(total, dtype=np.uint8)
    starts = np.concatenate(([0], np.cumsum(nbytes)[:-1]))
    cur = v.copy()
    for k in range(int(nbytes.max())):
        live = nbytes > k
        byte = (cur[live] & np.uint64(0x7F)).astype(np.uint8)
        more = nbytes[live] > k + 1
        out[starts[live] + k] = byte | (more.astype(np.uint8) << 7)
        cur[live] >>= np.uint64(7)
    return out.tobytes()


def encode_edits(edits: EditSet, xi_abs: float, tau: float) -> bytes:
    ids = np.asarray(edits.ids, dtype=np.int64)
    deltas = np.diff(ids, prepend=0) if ids.size else ids
    out = bytearray(struct.pack(_HEAD, EDITS_MAGIC, EDITS_VERSION, float(xi_abs), float(tau),
                                int(edits.vertex_count), int(ids.size)))
    out += _leb128(deltas.astype(np.uint64))
    out += np.asarray(edits.values, dtype="<f8").tobytes()
    out += struct.pack("<I", zlib.crc32(bytes(out)) & 0xFFFFFFFF)
    return bytes(out)


def decode_edits_meta(data: bytes) -> tuple[EditSet, float, float]:
    head = struct.calcsize(_HEAD)
    if len(data) < head + 4:
        raise FormatError("edits file truncated")
    magic, version, xi_abs, tau, vertex_count, count = struct.unpack_from(_HEAD, data, 0)
    if magic != EDITS_MAGIC:
        raise FormatError(f"bad edits magic {magic!r}")
    if version != EDITS_VERSION:
        raise FormatError(f"unsupported edits version {version}")
    (crc,) = struct.unpack_from("<I", data, len(data) - 4)
    if zlib.crc32(data[:-4]) & 0xFFFFFFFF != crc:
        raise FormatError("edits checksum mismatch")
    body = np.frombuffer(data, dtype=np.uint8, count=len(data) - 4 - head, offset=head)
    # varints: a byte with the high bit clear terminates a value
    ends = np.flatnonzero((body & 0x80) == 0)
    if ends.size < count:
        raise FormatError("edits file truncated inside a varint")
    var_len = int(ends[count - 1]) + 1 if count else 0
    vals_start = head + var_len
    if vals_start + 8 * count != len(data) - 4:
        raise FormatError("edits payload length mismatch")
    ids = np.zeros(count, dtype=np.uint64)
    if count:
        starts = np.concatenate(([0], ends[:count - 1] + 1))
        lens = ends[:count] - starts + 1
        if lens.max() > 10:
            raise FormatError("varint too long")
        for k in range(int(lens.max())):
            live = lens > k
            ids[live] |= (body[starts[live] + k].astype(np.uint64) & np.uint64(0x7F)) << np.uint64(7 * k)
    ids = np.cumsum(ids.astype(np.int64)) if count else ids.astype(np.int64)
    values = np.frombuffer(data, dtype="<f8", count=count, offset=vals_start).astype(np.float64)
    try:
        edits = EditSet(ids=ids, values=values, vertex_count=int(vertex_count))
    except ValueError as exc:
        raise FormatError(f"invalid edit set: {exc}") from exc
    return edits, float(xi_abs), float(tau)


def decode_edits(data: bytes) -> EditSet:
    return decode_edits_meta(data)[0]
