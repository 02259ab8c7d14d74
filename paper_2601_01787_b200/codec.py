"""Edit-record file format (PMSZE), the "edit record out" side of the drop-in.

Byte layout of codec.encode_edits / decode_edits_meta (codec.py:138-186):
header ``<6sBddQQ`` (magic, version, xi_abs, tau, vertex count, edit count),
delta-coded LEB128 ids (the first id absolute), the f64 values, CRC32 of all
preceding bytes.  The delta/varint packing is vectorised with NumPy here.
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
