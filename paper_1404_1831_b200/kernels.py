"""Drop-in for the reference kernel backend module ``bilayerpq.kernels``.

Same four functions, positional numpy arguments and return values as
kernels/numba_backend.py (selection and binding at kernels/__init__.py:15-40),
executed by the CUDA stage kernels through the C ABI.  Because the reference
resolves ``kernels.<fn>`` at call time (multi_index.py:17,323,355;
fbpq.py:23,173; hbpq.py:17,332), assigning these functions onto
``bilayerpq.kernels`` reroutes every reference engine through the GPU.

Each call runs on torch's current CUDA stream and synchronises once to
return numpy arrays (the reference returns freshly allocated arrays owned by
the caller).  Per-query inputs are uploaded every call; the index arrays
(ids, codes, books, FBPQ tables, local banks, cell offsets) are immutable in
the reference, so their device copies are cached, keyed by the
host buffer (address, shape, dtype, strides) and holding a reference to it
so the address cannot be reused while cached.
"""

from __future__ import annotations

from collections import OrderedDict

import numpy as np

from . import _lib

BACKEND = "cuda-sm100a"

_CACHE: "OrderedDict[tuple, tuple]" = OrderedDict()
_CACHE_BYTES = 0
_CACHE_LIMIT = 16 << 30


def _dev(a, dtype):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, dtype)).cuda()


def _dev_cached(a, dtype):
    """Device copy of an immutable index array (see the module docstring)."""
    global _CACHE_BYTES
    arr = np.asarray(a)
    if arr.nbytes < (64 << 10):
        return _dev(arr, dtype)
    key = (arr.__array_interface__["data"][0], arr.shape, arr.dtype.str, arr.strides, np.dtype(dtype).str)
    hit = _CACHE.get(key)
    if hit is not None:
        _CACHE.move_to_end(key)
        return hit[1]
    t = _dev(arr, dtype)
    _CACHE[key] = (arr, t)
    _CACHE_BYTES += t.numel() * t.element_size()
    while _CACHE_BYTES > _CACHE_LIMIT and len(_CACHE) > 1:
        _, (_, old) = _CACHE.popitem(last=False)
        _CACHE_BYTES -= old.numel() * old.element_size()
    return t


def traverse_cells(sorted_r1, sorted_r2, order1, order2, offsets, budget):
    """numba_backend.traverse_cells (:11-146): visited non-empty cells
    (vis_i i32, vis_j i32, starts i64, ends i64) in ascending-key order."""
    import torch

    t = int(np.asarray(sorted_r1).shape[0])
    offs = np.ascontiguousarray(offsets, np.int64)
    total = int(offs[-1])
    lib = _lib.load()
    cap = max(1, min(int(budget), total, t * t))
    vi = torch.empty(cap, dtype=torch.int32, device="cuda")
    vj = torch.empty(cap, dtype=torch.int32, device="cuda")
    st = torch.empty(cap, dtype=torch.int64, device="cuda")
    en = torch.empty(cap, dtype=torch.int64, device="cuda")
    nv = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = torch.empty(int(lib.bpq_traverse_workspace_size(t, int(budget), total)), dtype=torch.uint8, device="cuda")
    args = [_dev(sorted_r1, np.float64), _dev(sorted_r2, np.float64), _dev(order1, np.int32),
            _dev(order2, np.int32), _dev_cached(offs, np.int64)]
    _lib.check(lib.bpq_traverse_cells(*[_lib.ptr(a) for a in args], t, int(budget), total, _lib.ptr(vi),
                                      _lib.ptr(vj), _lib.ptr(st), _lib.ptr(en), _lib.ptr(nv), _lib.ptr(ws),
                                      ws.numel(), _lib.stream_ptr()), "traverse_cells")
    n = int(nv.item())
    return vi[:n].cpu().numpy(), vj[:n].cpu().numpy(), st[:n].cpu().numpy(), en[:n].cpu().numpy()


def _vis(vis_i, vis_j, starts, ends):
    st = np.ascontiguousarray(starts, np.int64)
    en = np.ascontiguousarray(ends, np.int64)
    cs = np.zeros(st.shape[0] + 1, np.int64)
    np.cumsum(en - st, out=cs[1:])
    return (_dev(vis_i, np.int32), _dev(vis_j, np.int32), _dev(st, np.int64), _dev(cs, np.int64),
            st.shape[0], int(cs[-1]))


def _outs(n):
    import torch

    return (torch.empty(n, dtype=torch.int32, device="cuda"), torch.empty(n, dtype=torch.float32, device="cuda"))


def _fin(oi, od):
    return oi.cpu().numpy().view(np.uint32), od.cpu().numpy()


def scan_global(vis_i, vis_j, starts, ends, ids, codes, e1, e2, books):
    """numba_backend.scan_global (:149-180), bit-exact f32 order."""
    vi, vj, st, cs, nvis, n = _vis(vis_i, vis_j, starts, ends)
    books = np.ascontiguousarray(books, np.float32)
    m, k, ds = books.shape
    oi, od = _outs(n)
    if n:
        lib = _lib.load()
        a = [_dev_cached(ids, np.uint32), _dev_cached(codes, np.uint8)]
        e = [_dev(e1, np.float32), _dev(e2, np.float32), _dev_cached(books, np.float32)]
        _lib.check(lib.bpq_scan_global(_lib.ptr(vi), _lib.ptr(vj), _lib.ptr(st), _lib.ptr(cs), nvis, n,
                                       _lib.ptr(a[0]), _lib.ptr(a[1]), m, k, ds, *[_lib.ptr(x) for x in e],
                                       _lib.ptr(oi), _lib.ptr(od), _lib.stream_ptr()), "scan_global")
    return _fin(oi, od)


def scan_local(vis_i, vis_j, starts, ends, ids, codes, e1, e2, books1, books2):
    """numba_backend.scan_local (:183-213), bit-exact f32 order."""
    vi, vj, st, cs, nvis, n = _vis(vis_i, vis_j, starts, ends)
    b1 = np.ascontiguousarray(books1, np.float32)
    _, m2, k, ds = b1.shape
    oi, od = _outs(n)
    if n:
        lib = _lib.load()
        a = [_dev_cached(ids, np.uint32), _dev_cached(codes, np.uint8)]
        e = [_dev(e1, np.float32), _dev(e2, np.float32), _dev_cached(b1, np.float32), _dev_cached(books2, np.float32)]
        _lib.check(lib.bpq_scan_local(_lib.ptr(vi), _lib.ptr(vj), _lib.ptr(st), _lib.ptr(cs), nvis, n,
                                      _lib.ptr(a[0]), _lib.ptr(a[1]), 2 * m2, k, ds, *[_lib.ptr(x) for x in e],
                                      _lib.ptr(oi), _lib.ptr(od), _lib.stream_ptr()), "scan_local")
    return _fin(oi, od)


def scan_tables(vis_i, vis_j, starts, ends, ids, codes, q_norm, qd1, qd2, cn1, cn2, fold, cross1, cross2):
    """numba_backend.scan_tables (:216-246), bit-exact f32 order."""
    vi, vj, st, cs, nvis, n = _vis(vis_i, vis_j, starts, ends)
    fold = np.ascontiguousarray(fold, np.float32)
    m, k = fold.shape
    oi, od = _outs(n)
    if n:
        lib = _lib.load()
        a = [_dev_cached(ids, np.uint32), _dev_cached(codes, np.uint8)]
        t = [_dev(x, np.float32) for x in (qd1, qd2)] + [_dev_cached(x, np.float32) for x in (cn1, cn2)] + \
            [_dev(fold, np.float32)] + [_dev_cached(x, np.float32) for x in (cross1, cross2)]
        _lib.check(lib.bpq_scan_tables(_lib.ptr(vi), _lib.ptr(vj), _lib.ptr(st), _lib.ptr(cs), nvis, n,
                                       _lib.ptr(a[0]), _lib.ptr(a[1]), m, k, float(np.float32(q_norm)),
                                       *[_lib.ptr(x) for x in t], _lib.ptr(oi), _lib.ptr(od),
                                       _lib.stream_ptr()), "scan_tables")
    return _fin(oi, od)


def install_into(kernels_module) -> None:
    """Rebind the reference backend's four functions to the GPU versions."""
    kernels_module.traverse_cells = traverse_cells
    kernels_module.scan_global = scan_global
    kernels_module.scan_local = scan_local
    kernels_module.scan_tables = scan_tables
    kernels_module.BACKEND = BACKEND
