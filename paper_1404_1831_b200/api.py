"""The reference's per-query search API over the batched device engine.

``search_baseline(index, q, l, r)`` (multi_index.py:358-367),
``search_fbpq(index, tables, q, l, r)`` (fbpq.py:188-194) and
``search_hbpq(hindex, q, l, r)`` (hbpq.py:337-342) return
``(ids uint32[<=r], dists float32[<=r])`` sorted by (dist, id), unpadded,
and raise ValueError for r < 1 / l < 1 as the reference does.  ``index`` may
be a DeviceIndex or a reference-layout object (converted once and cached).
Engine objects mirror evalbench.BaselineEngine/FbpqEngine/HbpqEngine
(evalbench.py:51-286) and add ``search_batch``.
"""

from __future__ import annotations

import weakref

import numpy as np

from .index import DeviceIndex

_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _device_index(index, tables=None) -> DeviceIndex:
    if isinstance(index, DeviceIndex):
        return index
    try:
        hit = _cache.get(index)
    except TypeError:
        hit = None
    if hit is not None and hit[0] is tables:
        return hit[1]
    dix = DeviceIndex.from_reference(index, tables)
    try:
        _cache[index] = (tables, dix)
    except TypeError:
        pass
    return dix


def _one(dix: DeviceIndex, engine: str, q, l: int, r: int):
    if r < 1:
        raise ValueError(f"r must be >= 1, got {r}")
    res = dix.search(np.asarray(q, np.float32).reshape(1, -1), l, r, engine)
    d, i, c = res.numpy()
    n = int(c[0])
    return i[0, :n].copy(), d[0, :n].copy()


def search_baseline(index, q, l: int, r: int):
    return _one(_device_index(index), "baseline", q, l, r)


def search_fbpq(index, tables, q, l: int, r: int):
    return _one(_device_index(index, tables), "fbpq", q, l, r)


def search_hbpq(hindex, q, l: int, r: int):
    return _one(_device_index(hindex), "hbpq", q, l, r)


class _Engine:
    name = ""

    def __init__(self, index, tables=None):
        self.dindex = _device_index(index, tables)
        if self.name == "hbpq" and self.dindex.kind != "hbpq":
            raise TypeError("hbpq engine requires a local-codebook HbpqIndex")
        if self.name != "hbpq" and self.dindex.kind == "hbpq":
            raise TypeError(f"{self.name} engine requires a global-codebook MultiIndex")

    def search(self, q, l: int, r: int):
        return _one(self.dindex, self.name, q, l, r)

    def search_batch(self, queries, l: int, k: int, **kw):
        return self.dindex.search(queries, l, k, self.name, **kw)


class BaselineEngine(_Engine):
    name = "baseline"


class FbpqEngine(_Engine):
    name = "fbpq"


class HbpqEngine(_Engine):
    name = "hbpq"


def make_engine(index, kind: str, tables=None):
    """Engine for an index; raises on engine/index kind mismatches (evalbench.py:271-286)."""
    dix = _device_index(index, tables)
    hb = dix.kind == "hbpq"
    if kind == "hbpq":
        if not hb:
            raise ValueError("engine hbpq requires an index built with local codebooks")
        return HbpqEngine(dix)
    if kind == "fbpq":
        if hb:
            raise ValueError("engine fbpq is incompatible with a local-codebook index")
        return FbpqEngine(dix)
    if kind == "baseline":
        if hb:
            raise ValueError("engine baseline is incompatible with a local-codebook index")
        return BaselineEngine(dix)
    raise ValueError(f"unknown engine {kind!r}")
