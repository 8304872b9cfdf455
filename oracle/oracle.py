"""CPU oracle for the bilayer-PQ search path -- TEST INFRASTRUCTURE ONLY.

This module is the checker the GPU engine is compared against.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs
may import it; the product package ``paper_1404_1831_b200`` never does.

It restates the reference package (``/root/reference/pkg/src/bilayerpq``,
abbreviated ``bpq/``) in numpy for the query-preparation steps -- the same
numpy/OpenBLAS calls in the same order, so on one machine they are bit-equal
to the reference -- and in C (``oracle/bpq_oracle.c`` via ctypes) for the
four kernels and ``select_top``.  Each function cites the reference
file:line it follows.  Pinned against the reference's own outputs by
``tests/golden/make_golden.py`` + ``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "build" / "liborc.so"
_lib = None


def build() -> Path:
    """Compile bpq_oracle.c into oracle/build/liborc.so (idempotent)."""
    src = _HERE / "bpq_oracle.c"
    if not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(str(_LIB_PATH))
        P = ctypes.c_void_p
        I = ctypes.c_int64
        F = ctypes.c_float
        _lib.orc_traverse_cells.restype = I
        _lib.orc_traverse_cells.argtypes = [P, P, P, P, P, I, I, P, P, P, P]
        _lib.orc_scan_global.restype = None
        _lib.orc_scan_global.argtypes = [P, P, P, P, I, P, P, P, P, P, I, I, I, P, P]
        _lib.orc_scan_local.restype = None
        _lib.orc_scan_local.argtypes = [P, P, P, P, I, P, P, P, P, P, P, I, I, I, P, P]
        _lib.orc_scan_tables.restype = None
        _lib.orc_scan_tables.argtypes = [P, P, P, P, I, P, P, F, P, P, P, P, P, P, P, I, I, P, P]
        _lib.orc_select_top.restype = I
        _lib.orc_select_top.argtypes = [P, P, I, I, P, P]
        _lib.orc_search_batch.restype = ctypes.c_int
        _lib.orc_search_batch.argtypes = (
            [ctypes.c_int] + [I] * 4 + [P] * 14 + [I] * 3 + [P] * 4 + [ctypes.c_int]
        )
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dt)


# --------------------------------------------------------------------------
# Kernels (bpq/kernels/numba_backend.py) -- same signatures as the reference
# backend module (bpq/kernels/__init__.py:37-40).
# --------------------------------------------------------------------------
def traverse_cells(sorted_r1, sorted_r2, order1, order2, offsets, budget):
    """bpq/kernels/numba_backend.py:11-146."""
    sr1 = _c(sorted_r1, np.float64)
    sr2 = _c(sorted_r2, np.float64)
    o1 = _c(order1, np.int32)
    o2 = _c(order2, np.int32)
    off = _c(offsets, np.int64)
    t = sr1.shape[0]
    total = int(off[-1])
    cap = max(1, min(int(budget), total, t * t))  # :14-19
    vi = np.empty(cap, np.int32)
    vj = np.empty(cap, np.int32)
    st = np.empty(cap, np.int64)
    en = np.empty(cap, np.int64)
    n = lib().orc_traverse_cells(
        _p(sr1), _p(sr2), _p(o1), _p(o2), _p(off), t, int(budget), _p(vi), _p(vj), _p(st), _p(en)
    )
    return vi[:n], vj[:n], st[:n], en[:n]


def _total(starts, ends):
    return int(np.sum(np.asarray(ends, np.int64) - np.asarray(starts, np.int64)))


def scan_global(vis_i, vis_j, starts, ends, ids, codes, e1, e2, books):
    """bpq/kernels/numba_backend.py:149-180."""
    vi, vj = _c(vis_i, np.int32), _c(vis_j, np.int32)
    st, en = _c(starts, np.int64), _c(ends, np.int64)
    books = _c(books, np.float32)
    m, k, ds = books.shape
    n = _total(st, en)
    oi = np.empty(n, np.uint32)
    od = np.empty(n, np.float32)
    lib().orc_scan_global(
        _p(vi), _p(vj), _p(st), _p(en), vi.shape[0], _p(_c(ids, np.uint32)),
        _p(_c(codes, np.uint8)), _p(_c(e1, np.float32)), _p(_c(e2, np.float32)), _p(books),
        m, k, ds, _p(oi), _p(od),
    )
    return oi, od


def scan_local(vis_i, vis_j, starts, ends, ids, codes, e1, e2, books1, books2):
    """bpq/kernels/numba_backend.py:183-213."""
    vi, vj = _c(vis_i, np.int32), _c(vis_j, np.int32)
    st, en = _c(starts, np.int64), _c(ends, np.int64)
    b1 = _c(books1, np.float32)
    b2 = _c(books2, np.float32)
    _, m2, k, ds = b1.shape
    n = _total(st, en)
    oi = np.empty(n, np.uint32)
    od = np.empty(n, np.float32)
    lib().orc_scan_local(
        _p(vi), _p(vj), _p(st), _p(en), vi.shape[0], _p(_c(ids, np.uint32)),
        _p(_c(codes, np.uint8)), _p(_c(e1, np.float32)), _p(_c(e2, np.float32)), _p(b1), _p(b2),
        m2, k, ds, _p(oi), _p(od),
    )
    return oi, od


def scan_tables(vis_i, vis_j, starts, ends, ids, codes, q_norm, qd1, qd2, cn1, cn2, fold, cross1, cross2):
    """bpq/kernels/numba_backend.py:216-246."""
    vi, vj = _c(vis_i, np.int32), _c(vis_j, np.int32)
    st, en = _c(starts, np.int64), _c(ends, np.int64)
    fold = _c(fold, np.float32)
    m, k = fold.shape
    n = _total(st, en)
    oi = np.empty(n, np.uint32)
    od = np.empty(n, np.float32)
    lib().orc_scan_tables(
        _p(vi), _p(vj), _p(st), _p(en), vi.shape[0], _p(_c(ids, np.uint32)),
        _p(_c(codes, np.uint8)), float(np.float32(q_norm)), _p(_c(qd1, np.float32)),
        _p(_c(qd2, np.float32)), _p(_c(cn1, np.float32)), _p(_c(cn2, np.float32)), _p(fold),
        _p(_c(cross1, np.float32)), _p(_c(cross2, np.float32)), m, k, _p(oi), _p(od),
    )
    return oi, od


def select_top(ids, dists, r):
    """bpq/multi_index.py:326-339: top-r by (dist asc, id asc)."""
    ids = _c(ids, np.uint32)
    d = _c(dists, np.float32)
    n = ids.shape[0]
    cnt = min(int(r), n)
    oi = np.empty(cnt, np.uint32)
    od = np.empty(cnt, np.float32)
    if n:
        lib().orc_select_top(_p(ids), _p(d), n, int(r), _p(oi), _p(od))
    return oi, od


# --------------------------------------------------------------------------
# Query preparation in numpy (same calls as the reference -> same BLAS bits)
# --------------------------------------------------------------------------
def coarse_norms(c):
    """np.einsum('ij,ij->i') as in bpq/multi_index.py:285-286 / fbpq.py:91-92."""
    c = _c(c, np.float32)
    return np.einsum("ij,ij->i", c, c)


def coarse_scan(c1, c2, q, rotation=None):
    """bpq/multi_index.py:270-293: (qr, dots1, dots2, r1, r2); qr = q @ R
    when the pair carries a rotation (multi_index.py:67-74, quantizer.py:95-96)."""
    c1 = _c(c1, np.float32)
    c2 = _c(c2, np.float32)
    qr = np.asarray(q, np.float32).reshape(1, -1)
    if rotation is not None:
        qr = qr @ _c(rotation, np.float32)
    qr = qr[0]
    dh = c1.shape[1]
    q1 = qr[:dh]
    q2 = qr[dh:]
    dots1 = c1 @ q1
    dots2 = c2 @ q2
    cn1 = np.einsum("ij,ij->i", c1, c1)
    cn2 = np.einsum("ij,ij->i", c2, c2)
    q1n = np.float32(q1 @ q1)
    q2n = np.float32(q2 @ q2)
    r1 = (cn1 - 2.0 * dots1) + q1n
    r2 = (cn2 - 2.0 * dots2) + q2n
    np.maximum(r1, np.float32(0.0), out=r1)
    np.maximum(r2, np.float32(0.0), out=r2)
    return qr, dots1, dots2, r1, r2


def sort_halves(r1, r2):
    """bpq/multi_index.py:319-322: stable argsort, values widened to f64."""
    order1 = np.argsort(r1, kind="stable").astype(np.int32)
    order2 = np.argsort(r2, kind="stable").astype(np.int32)
    return r1[order1].astype(np.float64), r2[order2].astype(np.float64), order1, order2


def traverse(offsets, r1, r2, budget):
    """bpq/multi_index.py:302-323."""
    if budget < 1:
        raise ValueError(f"budget must be >= 1, got {budget}")
    if int(offsets[-1]) == 0:
        return (np.empty(0, np.int32), np.empty(0, np.int32), np.empty(0, np.int64), np.empty(0, np.int64))
    sr1, sr2, o1, o2 = sort_halves(r1, r2)
    return traverse_cells(sr1, sr2, o1, o2, offsets, int(budget))


def build_tables_from(c1, c2, books):
    """bpq/fbpq.py:79-101 -> (cn1, cn2, fine_norms, cross1, cross2)."""
    c1 = _c(c1, np.float32)
    c2 = _c(c2, np.float32)
    books = _c(books, np.float32)
    m, k, ds = books.shape
    m2 = m // 2
    t = c1.shape[0]
    cn1 = np.einsum("ij,ij->i", c1, c1)
    cn2 = np.einsum("ij,ij->i", c2, c2)
    fine_norms = np.einsum("mkj,mkj->mk", books, books)
    cross1 = np.empty((t, m2, k), np.float32)
    cross2 = np.empty((t, m2, k), np.float32)
    for p in range(m2):
        cross1[:, p, :] = c1[:, p * ds : (p + 1) * ds] @ books[p].T
        cross2[:, p, :] = c2[:, p * ds : (p + 1) * ds] @ books[m2 + p].T
    return cn1, cn2, fine_norms, cross1, cross2


def prepare_query(c1, c2, books, fine_norms, q, rotation=None):
    """bpq/fbpq.py:129-145 -> (q_norm, dots1, dots2, fold, r1, r2)."""
    qr, dots1, dots2, r1, r2 = coarse_scan(c1, c2, q, rotation)
    books = _c(books, np.float32)
    m, k, ds = books.shape
    qdot_fine = np.empty((m, k), np.float32)
    for p in range(m):
        qdot_fine[p] = books[p] @ qr[p * ds : (p + 1) * ds]
    fold = fine_norms - 2.0 * qdot_fine
    q_norm = np.float32(qr @ qr)
    return q_norm, dots1, dots2, fold, r1, r2


class Index:
    """Plain arrays of a built multi-index (bpq/multi_index.py:100-146 /
    bpq/hbpq.py:240-290), optionally with FBPQ tables (bpq/fbpq.py:28-66)."""

    def __init__(self, c1, c2, offsets, ids, codes, books=None, bank1=None, bank2=None, tables=None,
                 rotation=None, rot1=None, rot2=None):
        self.rotation = None if rotation is None else _c(rotation, np.float32)
        self.rot1 = None if rot1 is None else _c(rot1, np.float32)
        self.rot2 = None if rot2 is None else _c(rot2, np.float32)
        self.c1 = _c(c1, np.float32)
        self.c2 = _c(c2, np.float32)
        self.offsets = _c(offsets, np.int64)
        self.ids = _c(ids, np.uint32)
        self.codes = _c(codes, np.uint8)
        self.books = None if books is None else _c(books, np.float32)
        self.bank1 = None if bank1 is None else _c(bank1, np.float32)
        self.bank2 = None if bank2 is None else _c(bank2, np.float32)
        if tables is None and self.books is not None:
            tables = build_tables_from(self.c1, self.c2, self.books)
        self.tables = tables

    @property
    def t(self):
        return self.c1.shape[0]

    @property
    def m(self):
        return self.codes.shape[1]


def scan_query(index: Index, engine: str, q, l):
    """scan_baseline (multi_index.py:350-355), scan_fbpq (fbpq.py:169-185),
    scan_hbpq (hbpq.py:316-334, no rotations)."""
    if engine == "fbpq":
        cn1, cn2, fine_norms, cross1, cross2 = index.tables
        q_norm, d1, d2, fold, r1, r2 = prepare_query(index.c1, index.c2, index.books, fine_norms, q, index.rotation)
        vis = traverse(index.offsets, r1, r2, l)
        return scan_tables(*vis, index.ids, index.codes, q_norm, d1, d2, cn1, cn2, fold, cross1, cross2)
    qr, _, _, r1, r2 = coarse_scan(index.c1, index.c2, q, index.rotation)
    vis = traverse(index.offsets, r1, r2, l)
    dh = index.c1.shape[1]
    e1 = qr[None, :dh] - index.c1
    e2 = qr[None, dh:] - index.c2
    if engine == "hbpq":  # per-half bank rotations (hbpq.py:328-331)
        if index.rot1 is not None:
            e1 = np.asarray(e1, np.float32) @ index.rot1
        if index.rot2 is not None:
            e2 = np.asarray(e2, np.float32) @ index.rot2
    if engine == "baseline":
        return scan_global(*vis, index.ids, index.codes, e1, e2, index.books)
    if engine == "hbpq":
        return scan_local(*vis, index.ids, index.codes, e1, e2, index.bank1, index.bank2)
    raise ValueError(f"unknown engine {engine!r}")


def search(index: Index, engine: str, q, l, r):
    """search_baseline / search_fbpq / search_hbpq: (ids, dists)."""
    if r < 1:
        raise ValueError(f"r must be >= 1, got {r}")
    ids, d = scan_query(index, engine, q, l)
    return select_top(ids, d, r)


def search_batch_numpy(index: Index, engine: str, queries, l, k):
    """Per-query loop (the reference has no batched API) padded
    to [nq, k]: returns (dists, ids, counts, n_candidates)."""
    queries = np.atleast_2d(np.asarray(queries, np.float32))
    nq = queries.shape[0]
    dist = np.full((nq, k), np.inf, np.float32)
    ids = np.full((nq, k), 0xFFFFFFFF, np.uint32)
    cnt = np.zeros(nq, np.int32)
    ncand = np.zeros(nq, np.int64)
    for x in range(nq):
        ci, cd = scan_query(index, engine, queries[x], l)
        ncand[x] = ci.shape[0]
        si, sd = select_top(ci, cd, k)
        cnt[x] = si.shape[0]
        ids[x, : cnt[x]] = si
        dist[x, : cnt[x]] = sd
    return dist, ids, cnt, ncand


ENGINE_CODES = {"baseline": 0, "fbpq": 1, "hbpq": 2}


def search_batch_c(index: Index, engine: str, queries, l, k, threads=None):
    """Whole search in C with POSIX threads (the CPU baseline).  Coarse dots
    are sequential f32 loops rather than OpenBLAS, so boundary near-ties may
    differ from search_batch_numpy within the parity contract."""
    queries = _c(np.atleast_2d(queries), np.float32)
    nq = queries.shape[0]
    threads = threads or os.cpu_count() or 1
    dist = np.empty((nq, k), np.float32)
    ids = np.empty((nq, k), np.uint32)
    cnt = np.empty(nq, np.int32)
    ncand = np.empty(nq, np.int64)
    cn1 = coarse_norms(index.c1)
    cn2 = coarse_norms(index.c2)
    fine_norms = cross1 = cross2 = None
    if engine == "fbpq":
        cn1, cn2, fine_norms, cross1, cross2 = index.tables
    m = index.m
    if engine == "hbpq":
        kk = index.bank1.shape[2]
    else:
        kk = index.books.shape[1]
    lib().orc_search_batch(
        ENGINE_CODES[engine], index.t, index.c1.shape[1], m, kk,
        _p(index.c1), _p(index.c2), _p(_c(cn1, np.float32)), _p(_c(cn2, np.float32)),
        _p(index.offsets), _p(index.ids), _p(index.codes), _p(index.books),
        _p(None if fine_norms is None else _c(fine_norms, np.float32)),
        _p(None if cross1 is None else _c(cross1, np.float32)),
        _p(None if cross2 is None else _c(cross2, np.float32)),
        _p(index.bank1), _p(index.bank2), _p(queries), nq, int(l), int(k),
        _p(dist), _p(ids), _p(cnt), _p(ncand), int(threads),
    )
    return dist, ids, cnt, ncand


# --------------------------------------------------------------------------
# Encoding (bpq/quantizer.py:109-130, 235-247; bpq/multi_index.py:167-230)
# --------------------------------------------------------------------------
def nearest_centroids(xs, centroids, block=16384):
    """bpq/quantizer.py:109-130: (int64 ids, f32 d2); ties -> lowest id."""
    xs = _c(xs, np.float32)
    cents = _c(centroids, np.float32)
    cn = np.einsum("ij,ij->i", cents, cents)
    n = xs.shape[0]
    ids = np.empty(n, np.int64)
    d2 = np.empty(n, np.float32)
    for s in range(0, n, block):
        e = min(s + block, n)
        chunk = xs[s:e]
        scores = cn[None, :] - 2.0 * (chunk @ cents.T)
        idx = np.argmin(scores, axis=1)
        ids[s:e] = idx
        xn = np.einsum("ij,ij->i", chunk, chunk)
        d2[s:e] = scores[np.arange(e - s), idx] + xn
    np.maximum(d2, np.float32(0.0), out=d2)
    return ids, d2


def pq_encode_batch(books, xs):
    """bpq/quantizer.py:235-247."""
    books = _c(books, np.float32)
    data = _c(np.atleast_2d(xs), np.float32)
    m, _, ds = books.shape
    codes = np.empty((data.shape[0], m), np.int32)
    for p in range(m):
        codes[:, p], _ = nearest_centroids(np.ascontiguousarray(data[:, p * ds : (p + 1) * ds]), books[p])
    return codes


def build_index(base, c1, c2, books, id_offset=0):
    """bpq/multi_index.py:210-230 (no rotation): (offsets, ids, codes)."""
    data = _c(base, np.float32)
    c1 = _c(c1, np.float32)
    c2 = _c(c2, np.float32)
    t, dh = c1.shape
    i_idx, _ = nearest_centroids(np.ascontiguousarray(data[:, :dh]), c1)
    j_idx, _ = nearest_centroids(np.ascontiguousarray(data[:, dh:]), c2)
    disp = np.empty_like(data)
    disp[:, :dh] = data[:, :dh] - c1[i_idx]
    disp[:, dh:] = data[:, dh:] - c2[j_idx]
    codes = pq_encode_batch(books, disp).astype(np.uint8)
    lin = i_idx * t + j_idx
    order = np.argsort(lin, kind="stable")
    counts = np.bincount(lin, minlength=t * t)
    offsets = np.zeros(t * t + 1, np.int64)
    np.cumsum(counts, out=offsets[1:])
    ids = (id_offset + order).astype(np.uint32)
    return offsets, ids, codes[order]
