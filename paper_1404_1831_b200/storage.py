"""Readers for the reference's exported artifacts (read path only).

Layouts follow storage.py of the reference: little-endian, 4-byte magic +
u32 version 1; BPQI index (storage.py:253-329), BPQT tables
(storage.py:332-360), BPQC coarse pair / codec / bank records
(storage.py:182-237).  Malformed files raise StorageError (magic, version,
truncation, trailing bytes), as the reference's strict reader does
(storage.py:63-104).
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

FORMAT_VERSION = 1
FLAG_ROTATED, FLAG_HBPQ = 1, 2


class StorageError(ValueError):
    pass


class _Buf:
    def __init__(self, path, magic: bytes):
        self.path = str(path)
        self.raw = Path(path).read_bytes()
        self.pos = 0
        head = self.take(4)
        if head != magic:
            raise StorageError(f"bad magic {head!r}, expected {magic!r}: {self.path}")
        ver = self.u32()
        if ver != FORMAT_VERSION:
            raise StorageError(f"unsupported format version {ver}: {self.path}")

    def take(self, n):
        if self.pos + n > len(self.raw):
            raise StorageError(f"truncated file at byte {self.pos}: {self.path}")
        b = self.raw[self.pos : self.pos + n]
        self.pos += n
        return b

    def u32(self):
        return struct.unpack("<I", self.take(4))[0]

    def u64(self):
        return struct.unpack("<Q", self.take(8))[0]

    def arr(self, dt, shape):
        dt = np.dtype(dt)
        n = int(np.prod(shape))
        return np.frombuffer(self.take(n * dt.itemsize), dtype=dt).reshape(shape).copy()

    def end(self):
        if self.pos != len(self.raw):
            raise StorageError(f"trailing bytes after record end at byte {self.pos}: {self.path}")


def _coarse(b: _Buf):
    t, dh, has_rot = b.u32(), b.u32(), b.u32()
    c1 = b.arr("<f4", (t, dh))
    c2 = b.arr("<f4", (t, dh))
    rot = b.arr("<f4", (2 * dh, 2 * dh)) if has_rot else None
    return c1, c2, rot


def _bank(b: _Buf):
    t, m2, k, ds, h1, h2 = (b.u32() for _ in range(6))
    b1 = b.arr("<f4", (t, m2, k, ds))
    b2 = b.arr("<f4", (t, m2, k, ds))
    r1 = b.arr("<f4", (m2 * ds, m2 * ds)) if h1 else None
    r2 = b.arr("<f4", (m2 * ds, m2 * ds)) if h2 else None
    return b1, b2, r1, r2


def load_index_arrays(path) -> dict:
    """BPQI -> dict(c1, c2, rotation, offsets i64, ids u32, codes u8, books | bank1/bank2/rot1/rot2)."""
    b = _Buf(path, b"BPQI")
    d, t, m, k, flags = (b.u32() for _ in range(5))
    n = b.u64()
    c1, c2, rot = _coarse(b)
    if c1.shape[0] != t or 2 * c1.shape[1] != d:
        raise StorageError(f"coarse block does not match the header: {path}")
    if bool(flags & FLAG_ROTATED) != (rot is not None):
        raise StorageError(f"rotation flag does not match the coarse block: {path}")
    out = dict(c1=c1, c2=c2, rotation=rot, offsets=b.arr("<i8", (t * t + 1,)), ids=b.arr("<u4", (n,)),
               codes=b.arr("u1", (n, m)), books=None, bank1=None, bank2=None, rot1=None, rot2=None)
    if flags & FLAG_HBPQ:
        out["bank1"], out["bank2"], out["rot1"], out["rot2"] = _bank(b)
        if out["bank1"].shape[2] != k:
            raise StorageError(f"bank block does not match the header: {path}")
    else:
        out["books"] = b.arr("<f4", (m, k, d // m))
    b.end()
    return out


def load_tables_arrays(path):
    """BPQT -> (coarse_norms1, coarse_norms2, fine_norms, cross1, cross2)."""
    b = _Buf(path, b"BPQT")
    t, m, k = b.u32(), b.u32(), b.u32()
    m2 = m // 2
    out = (b.arr("<f4", (t,)), b.arr("<f4", (t,)), b.arr("<f4", (m, k)), b.arr("<f4", (t, m2, k)),
           b.arr("<f4", (t, m2, k)))
    b.end()
    return out
