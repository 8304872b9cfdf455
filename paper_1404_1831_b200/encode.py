"""Batch database encoding on the device (north_star "Encoding" kernel).

Mirrors quantizer.nearest_centroids (quantizer.py:109-130),
multi_index.assign_cells_batch / displacements (multi_index.py:167-189),
quantizer.pq_encode_batch (quantizer.py:235-247), hbpq.hbpq_encode_batch
(hbpq.py:168-200) and the packing tail of build_index / build_hbpq_index
(multi_index.py:210-230, hbpq.py:293-313), all through the C ABI.

``train_kmeans`` is benchmark setup only (codebook training is out of scope,
SURVEY.md §2 row 5); it is a plain Lloyd loop whose assignment step is the
engine's nearest-centroid kernel.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .index import DeviceIndex, _check_fine_params, build_tables_host, coarse_norms


def _t(a, device, dtype=None):
    import torch

    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=dtype or a.dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dtype).contiguous()


def _use_tensor_cores(d: int) -> bool:
    import os

    return d == 64 and os.environ.get("BPQ_ENCODE") != "ffma"


def nearest_centroids(xs, centroids, *, norms=None, want_d2=True, stream=None):
    """(int64 ids, f32 d2) per row; ties break toward the lower id.  For
    d = 64 (the coarse halves at D = 128) the tcgen05 kernel with exact bf16
    limbs runs; otherwise the FFMA kernel (BPQ_ENCODE=ffma forces it)."""
    import torch

    cents = _t(centroids, xs.device if isinstance(xs, torch.Tensor) else "cuda", torch.float32)
    dev = cents.device
    if not (isinstance(xs, torch.Tensor) and xs.device == dev and xs.dtype == torch.float32
            and xs.dim() == 2 and xs.stride(1) == 1):
        xs = _t(xs, dev, torch.float32)
    if xs.dim() != 2 or xs.shape[1] != cents.shape[1]:
        raise ValueError("dimension mismatch")
    if norms is None:
        norms = coarse_norms(cents.cpu().numpy())
    cn = _t(norms, dev, torch.float32)
    n = xs.shape[0]
    ids = torch.empty(n, dtype=torch.int64, device=dev)
    d2 = torch.empty(n, dtype=torch.float32, device=dev) if want_d2 else None
    lib = _lib.load()
    if _use_tensor_cores(xs.shape[1]):
        nc = cents.shape[0]
        img = torch.empty(int(lib.bpq_coarse_limb_image_bytes(nc)), dtype=torch.uint8, device=dev)
        _lib.check(lib.bpq_coarse_limb_image(_lib.ptr(cents), nc, _lib.ptr(img), _lib.stream_ptr(stream)),
                   "coarse_limb_image")
        _lib.check(lib.bpq_nearest_centroids_tc(_lib.ptr(xs), n, xs.stride(0), _lib.ptr(img), _lib.ptr(cn), nc,
                                                _lib.ptr(ids), _lib.ptr(d2), None, 0, _lib.stream_ptr(stream)),
                   "nearest_centroids_tc")
        return ids, d2
    _lib.check(lib.bpq_nearest_centroids(_lib.ptr(xs), n, xs.stride(0), xs.shape[1], _lib.ptr(cents),
                                         _lib.ptr(cn), cents.shape[0], _lib.ptr(ids), _lib.ptr(d2),
                                         None, 0, _lib.stream_ptr(stream)), "nearest_centroids")
    return ids, d2


def assign_cells(xs, c1, c2, *, cn1=None, cn2=None, stream=None):
    """Cell coordinates (i, j) per row (multi_index.py:167-173)."""
    import torch

    dh = c1.shape[1]
    xs = _t(xs, "cuda" if not isinstance(xs, torch.Tensor) else xs.device, torch.float32)
    i_idx, _ = nearest_centroids(xs[:, :dh], c1, norms=cn1, want_d2=False, stream=stream)
    j_idx, _ = nearest_centroids(xs[:, dh:], c2, norms=cn2, want_d2=False, stream=stream)
    return i_idx, j_idx


def _book_norms(books):
    books = np.ascontiguousarray(books, np.float32)
    return np.stack([np.einsum("ij,ij->i", books[p], books[p]) for p in range(books.shape[0])])


def encode_residual(xs, i_idx, j_idx, c1, c2, books, *, stream=None, chunk=1 << 21):
    """PQ codes of the displacements from the assigned cells."""
    import torch

    dev = xs.device
    n, dim = xs.shape
    m, k, ds = books.shape
    bt = _t(books, dev, torch.float32)
    bn = _t(_book_norms(books.cpu().numpy() if isinstance(books, torch.Tensor) else books), dev, torch.float32)
    c1t, c2t = _t(c1, dev, torch.float32), _t(c2, dev, torch.float32)
    codes = torch.empty((n, m), dtype=torch.uint8, device=dev)
    lib = _lib.load()
    ws = torch.empty(min(n, chunk) * dim * 4, dtype=torch.uint8, device=dev)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        _lib.check(lib.bpq_encode_residual(
            _lib.ptr(xs[s:e]), e - s, dim, _lib.ptr(c1t), _lib.ptr(c2t), _lib.ptr(i_idx[s:e]),
            _lib.ptr(j_idx[s:e]), _lib.ptr(bt), _lib.ptr(bn), m, k, _lib.ptr(codes[s:e]),
            _lib.ptr(ws), ws.numel(), _lib.stream_ptr(stream)), "encode_residual")
    return codes


def encode_local(xs, i_idx, j_idx, c1, c2, bank1, bank2, *, stream=None):
    import torch

    dev = xs.device
    n, dim = xs.shape
    t, m2, k, ds = bank1.shape
    b1, b2 = _t(bank1, dev, torch.float32), _t(bank2, dev, torch.float32)
    c1t, c2t = _t(c1, dev, torch.float32), _t(c2, dev, torch.float32)
    codes = torch.empty((n, 2 * m2), dtype=torch.uint8, device=dev)
    lib = _lib.load()
    _lib.check(lib.bpq_encode_local(_lib.ptr(xs), n, dim, _lib.ptr(c1t), _lib.ptr(c2t), _lib.ptr(i_idx),
                                    _lib.ptr(j_idx), _lib.ptr(b1), _lib.ptr(b2), 2 * m2, k,
                                    _lib.ptr(codes), _lib.stream_ptr(stream)), "encode_local")
    return codes


def pack_cells(i_idx, j_idx, codes, t, id_offset=0, *, stream=None):
    """Group entries by cell, ascending id within a cell (multi_index.py:224-230).
    Returns (offsets u32 [t*t+1] as int32 tensor, ids u32 as int32, codes)."""
    import torch

    dev = codes.device
    n, m = codes.shape
    if id_offset < 0 or (n > 0 and id_offset + n - 1 > 0xFFFFFFFF):
        raise ValueError("point ids must fit in 32 bits")
    lib = _lib.load()
    ws = torch.empty(int(lib.bpq_pack_workspace_size(n, t)), dtype=torch.uint8, device=dev)
    offsets = torch.empty(t * t + 1, dtype=torch.int32, device=dev)
    ids = torch.empty(n, dtype=torch.int32, device=dev)
    out_codes = torch.empty_like(codes)
    _lib.check(lib.bpq_pack_cells(_lib.ptr(i_idx), _lib.ptr(j_idx), n, t, int(id_offset), _lib.ptr(codes), m,
                                  _lib.ptr(offsets), _lib.ptr(ids), _lib.ptr(out_codes), _lib.ptr(ws),
                                  ws.numel(), _lib.stream_ptr(stream)), "pack_cells")
    return offsets, ids, out_codes


def rotate(xs, R, *, stream=None):
    """xs @ R on the device (Rotation.rotate, quantizer.py:95-96)."""
    import torch

    xs = _t(xs, xs.device if isinstance(xs, torch.Tensor) else "cuda", torch.float32)
    Rt = _t(R, xs.device, torch.float32)
    out = torch.empty_like(xs)
    lib = _lib.load()
    _lib.check(lib.bpq_rotate(_lib.ptr(xs), xs.shape[0], xs.shape[1], _lib.ptr(Rt), _lib.ptr(out),
                              _lib.stream_ptr(stream)), "rotate")
    return out


def build_index(base, c1, c2, books, id_offset=0, *, tables=None, device=None, rotation=None):
    """Assign, encode and pack ``base`` into a DeviceIndex (build_index,
    multi_index.py:210-230); with a coarse rotation the vectors are encoded
    in the rotated space (displacements, multi_index.py:181-189)."""
    import torch

    dev = torch.device(device or "cuda")
    xs = _t(base, dev, torch.float32)
    if rotation is not None:
        xs = rotate(xs, rotation)
    c1n = c1.cpu().numpy() if isinstance(c1, torch.Tensor) else np.asarray(c1, np.float32)
    c2n = c2.cpu().numpy() if isinstance(c2, torch.Tensor) else np.asarray(c2, np.float32)
    booksn = books.cpu().numpy() if isinstance(books, torch.Tensor) else np.asarray(books, np.float32)
    t = c1n.shape[0]
    _check_fine_params(2 * c1n.shape[1], booksn.shape[0], booksn.shape[1])
    i_idx, j_idx = assign_cells(xs, c1n, c2n)
    codes = encode_residual(xs, i_idx, j_idx, c1n, c2n, booksn)
    offsets, ids, pcodes = pack_cells(i_idx, j_idx, codes, t, id_offset)
    if tables is None:
        tables = build_tables_host(c1n, c2n, booksn)
    return DeviceIndex(c1=c1n, c2=c2n, offsets=offsets, ids=ids, codes=pcodes, books=booksn,
                       tables=tables, device=dev, rotation=rotation)


def build_index_streamed(n, make_chunk, c1, c2, books, id_offset=0, *, chunk=1 << 24, tables=None, device=None):
    """build_index for databases that do not fit the device as f32: rows
    [s, e) come from make_chunk(s, e) (a device f32 tensor), are assigned and
    encoded chunk by chunk, and only (i, j, codes) are kept for the packing."""
    import torch

    dev = torch.device(device or "cuda")
    c1n = np.asarray(c1, np.float32)
    c2n = np.asarray(c2, np.float32)
    booksn = np.asarray(books, np.float32)
    t = c1n.shape[0]
    m = booksn.shape[0]
    _check_fine_params(2 * c1n.shape[1], m, booksn.shape[1])
    i_all = torch.empty(n, dtype=torch.int64, device=dev)
    j_all = torch.empty(n, dtype=torch.int64, device=dev)
    codes = torch.empty((n, m), dtype=torch.uint8, device=dev)
    cn1, cn2 = coarse_norms(c1n), coarse_norms(c2n)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        x = make_chunk(s, e)
        i, j = assign_cells(x, c1n, c2n, cn1=cn1, cn2=cn2)
        i_all[s:e] = i
        j_all[s:e] = j
        codes[s:e] = encode_residual(x, i, j, c1n, c2n, booksn)
        del x, i, j
    offsets, ids, pcodes = pack_cells(i_all, j_all, codes, t, id_offset)
    del i_all, j_all, codes
    torch.cuda.empty_cache()
    if tables is None:
        tables = build_tables_host(c1n, c2n, booksn)
    return DeviceIndex(c1=c1n, c2=c2n, offsets=offsets, ids=ids, codes=pcodes, books=booksn,
                       tables=tables, device=dev)


def build_hbpq_index(base, c1, c2, bank1, bank2, id_offset=0, *, device=None, rotation=None, rot1=None,
                     rot2=None):
    """build_hbpq_index (hbpq.py:293-313) on the device, with the optional
    coarse rotation and per-half bank rotations (hbpq.py:168-187)."""
    import torch

    dev = torch.device(device or "cuda")
    xs = _t(base, dev, torch.float32)
    if rotation is not None:
        xs = rotate(xs, rotation)
    c1n, c2n = np.asarray(c1, np.float32), np.asarray(c2, np.float32)
    t, dh = c1n.shape
    i_idx, j_idx = assign_cells(xs, c1n, c2n)
    if rot1 is None and rot2 is None:
        codes = encode_local(xs, i_idx, j_idx, c1n, c2n, bank1, bank2)
    else:
        # rotated half displacements, encoded against zero "coarse" books
        disp = xs - torch.cat([torch.from_numpy(c1n).to(dev)[i_idx], torch.from_numpy(c2n).to(dev)[j_idx]], 1)
        h1, h2 = disp[:, :dh].contiguous(), disp[:, dh:].contiguous()
        if rot1 is not None:
            h1 = rotate(h1, rot1)
        if rot2 is not None:
            h2 = rotate(h2, rot2)
        zeros = np.zeros_like(c1n)
        codes = encode_local(torch.cat([h1, h2], 1).contiguous(), i_idx, j_idx, zeros, zeros, bank1, bank2)
    offsets, ids, pcodes = pack_cells(i_idx, j_idx, codes, t, id_offset)
    return DeviceIndex(c1=c1n, c2=c2n, offsets=offsets, ids=ids, codes=pcodes, bank1=bank1,
                       bank2=bank2, device=dev, rotation=rotation, rot1=rot1, rot2=rot2)


def train_kmeans(xs, k, iters=10, seed=0):
    """Benchmark-setup Lloyd k-means on the device (not the reference's
    k-means++; training is out of scope).  Returns f32 [k, d] numpy."""
    import torch

    n, d = xs.shape
    g = torch.Generator(device=xs.device)
    g.manual_seed(seed)
    cent = xs[torch.randperm(n, generator=g, device=xs.device)[:k]].clone()
    for _ in range(iters):
        ids, _ = nearest_centroids(xs, cent, norms=(cent * cent).sum(1).cpu().numpy(), want_d2=False)
        sums = torch.zeros_like(cent).index_add_(0, ids, xs)
        cnt = torch.zeros(k, device=xs.device).index_add_(0, ids, torch.ones(n, device=xs.device))
        nz = cnt > 0
        cent[nz] = sums[nz] / cnt[nz, None]
    return cent.cpu().numpy().astype(np.float32)
