"""Readers for the reference's exported artifacts (read path only).

Layouts follow storage.py of the reference: little-endian, 4-byte magic +
u32 version 1; BPQI index (storage.py:253-329), BPQT tables
(storage.py:332-360), BPQC coarse pair / codec / bank records
(storage.py:182-237).  Malformed files raise StorageError (magic, version,
truncation, trailing bytes), as the reference's strict reader does
(storage.py:63-104).
"""

from __future__ import annotations

import hashlib
import os
import struct
import tempfile
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


# --------------------------------------------------------------- write path
# GPU-built indexes are exported in the reference's own layouts so the
# reference (storage.load_index / load_tables, CLI) can read them
# (SURVEY.md §8f row f1).  Field order: storage.py:182-237, 253-281, 332-343.

def _u32(v):
    return struct.pack("<I", int(v))


def _u64(v):
    return struct.pack("<Q", int(v))


def _f32(a):
    return np.ascontiguousarray(a, "<f4").tobytes()


def _atomic_write(path, payload: bytes):
    path = Path(path)
    fd, tmp = tempfile.mkstemp(dir=path.parent or Path("."), prefix=path.name + ".")
    try:
        with os.fdopen(fd, "wb") as fh:
            fh.write(payload)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def index_bytes(c1, c2, offsets, ids, codes, books=None, bank1=None, bank2=None, rotation=None, rot1=None,
                rot2=None) -> bytes:
    """BPQI payload for a global-codebook (books) or local-codebook (bank) index."""
    c1 = np.ascontiguousarray(c1, np.float32)
    c2 = np.ascontiguousarray(c2, np.float32)
    codes = np.ascontiguousarray(codes, np.uint8)
    t, dh = c1.shape
    d = 2 * dh
    n, m = codes.shape
    hb = bank1 is not None
    k = (np.asarray(bank1).shape[2] if hb else np.asarray(books).shape[1])
    flags = (FLAG_ROTATED if rotation is not None else 0) | (FLAG_HBPQ if hb else 0)
    out = [b"BPQI", _u32(FORMAT_VERSION), _u32(d), _u32(t), _u32(m), _u32(k), _u32(flags), _u64(n)]
    out += [_u32(t), _u32(dh), _u32(1 if rotation is not None else 0), _f32(c1), _f32(c2)]
    if rotation is not None:
        out.append(_f32(rotation))
    out += [np.ascontiguousarray(offsets, "<i8").tobytes(), np.ascontiguousarray(ids, "<u4").tobytes(),
            codes.tobytes()]
    if hb:
        b1 = np.ascontiguousarray(bank1, np.float32)
        bt, m2, bk, ds = b1.shape
        out += [_u32(bt), _u32(m2), _u32(bk), _u32(ds), _u32(1 if rot1 is not None else 0),
                _u32(1 if rot2 is not None else 0), _f32(b1), _f32(bank2)]
        if rot1 is not None:
            out.append(_f32(rot1))
        if rot2 is not None:
            out.append(_f32(rot2))
    else:
        out.append(_f32(books))
    return b"".join(out)


def tables_bytes(cn1, cn2, fine_norms, cross1, cross2) -> bytes:
    """BPQT payload (query-independent FBPQ tables)."""
    t = np.asarray(cn1).shape[0]
    m, k = np.asarray(fine_norms).shape
    return b"".join([b"BPQT", _u32(FORMAT_VERSION), _u32(t), _u32(m), _u32(k), _f32(cn1), _f32(cn2),
                     _f32(fine_norms), _f32(cross1), _f32(cross2)])


def save_index_arrays(path, **arrays) -> str:
    """Write a BPQI file atomically; returns its sha256."""
    payload = index_bytes(**arrays)
    _atomic_write(path, payload)
    return hashlib.sha256(payload).hexdigest()


def save_tables_arrays(path, cn1, cn2, fine_norms, cross1, cross2) -> str:
    payload = tables_bytes(cn1, cn2, fine_norms, cross1, cross2)
    _atomic_write(path, payload)
    return hashlib.sha256(payload).hexdigest()
