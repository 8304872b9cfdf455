"""Device-resident bilayer index and the batched search entry point.

``DeviceIndex`` is the B200 counterpart of the reference containers
``MultiIndex`` (multi_index.py:100-146), ``HbpqIndex`` (hbpq.py:240-290) and
``FbpqTables`` (fbpq.py:28-66).  It is built from exported codebooks and
codes (reference objects, BPQI/BPQT files, or plain arrays) or encoded on the
device from raw vectors, and answers ``search(queries, L, k)`` for a whole
batch with one C-ABI call (bpq_search).  PyTorch only provides the device
buffers and the stream.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import os

import numpy as np

from . import _lib

MAX_PARTS = 16
MAX_CODEBOOK = 256


def _check_fine_params(dim: int, m: int, k: int) -> None:
    """Same rules and messages as multi_index._check_fine_params (multi_index.py:199-207)."""
    if m < 2 or m % 2 != 0:
        raise ValueError(f"number of parts must be even and >= 2, got {m}")
    if m > MAX_PARTS:
        raise ValueError(f"number of parts must be <= {MAX_PARTS}, got {m}")
    if dim % m != 0:
        raise ValueError(f"dimension {dim} is not divisible into {m} parts")
    if not 1 <= k <= MAX_CODEBOOK:
        raise ValueError(f"codebook size must be in [1, {MAX_CODEBOOK}], got {k}")


def coarse_norms(c: np.ndarray) -> np.ndarray:
    """einsum('ij,ij->i') exactly as coarse_scan / build_tables_from compute it."""
    c = np.ascontiguousarray(c, np.float32)
    return np.einsum("ij,ij->i", c, c)


def build_tables_host(c1, c2, books):
    """Query-independent FBPQ tables (build_tables_from, fbpq.py:79-101):
    (coarse_norms1, coarse_norms2, fine_norms, cross1, cross2)."""
    c1 = np.ascontiguousarray(c1, np.float32)
    c2 = np.ascontiguousarray(c2, np.float32)
    books = np.ascontiguousarray(books, np.float32)
    m, k, ds = books.shape
    m2 = m // 2
    t = c1.shape[0]
    fine_norms = np.einsum("mkj,mkj->mk", books, books)
    cross1 = np.empty((t, m2, k), np.float32)
    cross2 = np.empty((t, m2, k), np.float32)
    for p in range(m2):
        cross1[:, p, :] = c1[:, p * ds : (p + 1) * ds] @ books[p].T
        cross2[:, p, :] = c2[:, p * ds : (p + 1) * ds] @ books[m2 + p].T
    return coarse_norms(c1), coarse_norms(c2), fine_norms, cross1, cross2


@dataclass
class SearchResult:
    """Batched result.  ``ids`` holds uint32 point ids in an int32 tensor
    (padding 0xFFFFFFFF reads as -1); ``dists`` are squared distances padded
    with +inf; ``counts`` is the valid prefix length per query (reference
    lists are unpadded).  Note the (dists, ids) order of the
    batched API versus the reference's per-query (ids, dists)."""

    dists: "object"
    ids: "object"
    counts: "object"
    ncand: "object" = None

    def numpy(self):
        return (
            self.dists.cpu().numpy(),
            self.ids.cpu().numpy().view(np.uint32),
            self.counts.cpu().numpy(),
        )


def _u32_tensor(a, device):
    import torch

    a = np.ascontiguousarray(a)
    if a.dtype == np.int64:
        if a.size and (a.min() < 0 or a.max() > 0xFFFFFFFF):
            raise ValueError("values must fit uint32")
        a = a.astype(np.uint32)
    return torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).to(device)


def _f32(a, device):
    import torch

    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(device)


class DeviceIndex:
    """Immutable device index; safe for concurrent searches on different
    streams as long as each uses its own workspace (``workspace=``)."""

    def __init__(self, *, c1, c2, offsets, ids, codes, books=None, tables=None, bank1=None,
                 bank2=None, global_offsets=None, device=None, num_entries_global=None, cell_lists="auto",
                 rotation=None, rot1=None, rot2=None, fbpq_exact=None, exact=None):
        """``fbpq_exact`` (alias ``exact``): score every candidate in the
        reference's exact operation order -- FBPQ without the precomputed
        per-entry point term (numba_backend.py:231-242), Multi-D-ADC / HBPQ
        without the per-cell residual tables (numba_backend.py:165-176,
        198-210); bpq_index_desc.fbpq_exact.  Default from the environment
        variable BPQ_FBPQ_EXACT=1."""
        import torch

        self.device = torch.device(device if device is not None else "cuda")
        if exact is not None:
            fbpq_exact = exact
        if fbpq_exact is None:
            fbpq_exact = os.environ.get("BPQ_FBPQ_EXACT") == "1"
        self.fbpq_exact = bool(fbpq_exact)
        c1n = c1.detach().cpu().numpy() if isinstance(c1, torch.Tensor) else np.asarray(c1, np.float32)
        c2n = c2.detach().cpu().numpy() if isinstance(c2, torch.Tensor) else np.asarray(c2, np.float32)
        if c1n.shape != c2n.shape or c1n.ndim != 2:
            raise ValueError("the two coarse codebooks must have equal shape (t, d/2)")
        self.t, dh = c1n.shape
        self.dim = 2 * dh
        codes_t = codes if isinstance(codes, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(codes, np.uint8))
        if codes_t.dim() != 2:
            raise ValueError("codes must have shape (n, m)")
        self.m = codes_t.shape[1]
        self.kind = "hbpq" if bank1 is not None else "global"
        if self.kind == "hbpq":
            self.k = (bank1.shape[2])
        elif books is not None:
            self.k = books.shape[1]
        else:
            raise ValueError("an index needs fine codebooks or a local codebook bank")
        _check_fine_params(self.dim, self.m, self.k)
        # traversal keys use the reference's coarse norms (einsum, multi_index.py:285-286)
        if tables is not None:
            cn1, cn2 = _table_attr(tables, 0), _table_attr(tables, 1)
        else:
            cn1, cn2 = coarse_norms(c1n), coarse_norms(c2n)
        dev = self.device
        self.c1 = _f32(c1n, dev)
        self.c2 = _f32(c2n, dev)
        self.cn1 = _f32(cn1, dev)
        self.cn2 = _f32(cn2, dev)
        if isinstance(offsets, torch.Tensor):
            self.offsets = offsets.to(dev)
            n_off = offsets.shape[0]
        else:
            offs = np.asarray(offsets)
            if offs.ndim != 1 or offs.shape[0] != self.t * self.t + 1:
                raise ValueError("cell table size does not match the coarse codebooks")
            if offs[0] != 0 or np.any(np.diff(offs.astype(np.int64)) < 0):
                raise ValueError("offsets must start at 0 and be non-decreasing")
            self.offsets = _u32_tensor(offs, dev)
            n_off = offs.shape[0]
        if n_off != self.t * self.t + 1:
            raise ValueError("cell table size does not match the coarse codebooks")
        self.ids = ids.to(dev) if isinstance(ids, torch.Tensor) else _u32_tensor(np.asarray(ids, np.uint32), dev)
        self.codes = codes_t.to(dev).contiguous()
        self.n = self.codes.shape[0]
        if self.ids.shape[0] != self.n:
            raise ValueError("entry count does not match the cell table")
        self.global_offsets = None
        if global_offsets is not None:
            self.global_offsets = (global_offsets.to(dev) if isinstance(global_offsets, torch.Tensor)
                                   else _u32_tensor(np.asarray(global_offsets), dev))
        self.n_global = int(num_entries_global) if num_entries_global is not None else self.n
        self.books = _f32(books, dev)
        self.fine_norms = self.cross1 = self.cross2 = None
        if books is not None:
            if tables is None:
                tables = build_tables_host(c1n, c2n, books.cpu().numpy() if isinstance(books, torch.Tensor) else books)
            self.fine_norms = _f32(_table_attr(tables, 2), dev)
            self.cross1 = _f32(_table_attr(tables, 3), dev)
            self.cross2 = _f32(_table_attr(tables, 4), dev)
        self.bank1 = _f32(bank1, dev)
        self.bank2 = _f32(bank2, dev)
        # OPQ rotations: coarse pair R [D, D] (queries -> q @ R), bank R1/R2 [D/2, D/2]
        self.rotation = _f32(rotation, dev)
        self.rot1 = _f32(rot1, dev) if self.kind == "hbpq" else None
        self.rot2 = _f32(rot2, dev) if self.kind == "hbpq" else None
        if self.rotation is not None and tuple(self.rotation.shape) != (self.dim, self.dim):
            raise ValueError("rotation dimension does not match the codebooks")
        for r in (self.rot1, self.rot2):
            if r is not None and tuple(r.shape) != (self.dim // 2, self.dim // 2):
                raise ValueError("per-half rotation dimension must equal dim/2")
        self._build_cell_lists(cell_lists)
        self._handle = None
        self._ws = {}
        self._create()

    # ------------------------------------------------------ populated cells
    def _build_cell_lists(self, mode):
        """Row/column lists of the traversal table's populated cells
        (bpq_build_cell_lists).  'auto' builds them when under half of the
        cells are populated -- then the traversal enumerates sparse band
        segments through them instead of reading every cell's offsets."""
        import torch

        self.row_ptr = self.col_ptr = self.row_cols = self.col_rows = None
        if mode is False or mode == "off":
            return
        table = self.global_offsets if self.global_offsets is not None else self.offsets
        t = self.t
        populated = int(((table[1:].long() & 0xFFFFFFFF) != (table[:-1].long() & 0xFFFFFFFF)).sum().item())
        if mode == "auto" and populated * 2 > t * t:
            return
        dev = self.device
        self.row_ptr = torch.empty(t + 1, dtype=torch.int32, device=dev)
        self.col_ptr = torch.empty(t + 1, dtype=torch.int32, device=dev)
        self.row_cols = torch.empty(max(populated, 1), dtype=torch.int16, device=dev)
        self.col_rows = torch.empty(max(populated, 1), dtype=torch.int16, device=dev)
        lib = _lib.load()
        ws = torch.empty(int(lib.bpq_cell_lists_workspace_size(t)), dtype=torch.uint8, device=dev)
        _lib.check(lib.bpq_build_cell_lists(_lib.ptr(table), t, _lib.ptr(self.row_ptr), _lib.ptr(self.row_cols),
                                            _lib.ptr(self.col_ptr), _lib.ptr(self.col_rows), _lib.ptr(ws),
                                            ws.numel(), _lib.stream_ptr()), "build_cell_lists")
        self.populated_cells = populated

    # ------------------------------------------------------------- C handle
    def _create(self):
        lib = _lib.load()
        d = _lib.IndexDesc()
        d.dim, d.num_coarse, d.num_parts, d.codebook_size = self.dim, self.t, self.m, self.k
        d.num_entries = self.n
        d.num_entries_global = self.n_global
        d.coarse1, d.coarse2 = _lib.ptr(self.c1), _lib.ptr(self.c2)
        d.coarse_norms1, d.coarse_norms2 = _lib.ptr(self.cn1), _lib.ptr(self.cn2)
        d.cell_offsets = _lib.ptr(self.offsets)
        d.global_offsets = _lib.ptr(self.global_offsets)
        d.ids, d.codes = _lib.ptr(self.ids), _lib.ptr(self.codes)
        d.fine_books, d.fine_norms = _lib.ptr(self.books), _lib.ptr(self.fine_norms)
        d.cross1, d.cross2 = _lib.ptr(self.cross1), _lib.ptr(self.cross2)
        d.bank1, d.bank2 = _lib.ptr(self.bank1), _lib.ptr(self.bank2)
        d.row_ptr, d.col_ptr = _lib.ptr(self.row_ptr), _lib.ptr(self.col_ptr)
        d.row_cols, d.col_rows = _lib.ptr(self.row_cols), _lib.ptr(self.col_rows)
        d.rotation, d.rot1, d.rot2 = _lib.ptr(self.rotation), _lib.ptr(self.rot1), _lib.ptr(self.rot2)
        d.fbpq_exact = 1 if self.fbpq_exact else 0
        h = ctypes.c_void_p()
        _lib.check(lib.bpq_index_create(ctypes.byref(d), 0, ctypes.byref(h)), "bpq_index_create")
        self._handle = h

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.bpq_index_destroy(h)
            self._handle = None

    # ------------------------------------------------------------ properties
    @property
    def num_points(self) -> int:
        return self.n

    @property
    def num_coarse(self) -> int:
        return self.t

    @property
    def num_parts(self) -> int:
        return self.m

    @property
    def codebook_size(self) -> int:
        return self.k

    @property
    def bytes_per_point(self) -> int:
        return 4 + self.m

    def engines(self):
        return ("hbpq",) if self.kind == "hbpq" else ("baseline", "fbpq")

    # --------------------------------------------------------------- search
    def coarse_dots(self, queries):
        """First-layer stage (coarse_scan's dot products, multi_index.py:
        283-288) on the path this index's searches use (tcgen05 tensor cores
        for D = 128, else FFMA): returns device f32 (dots1, dots2) [nq, T].
        Queries are taken as given (already rotated for a rotated index)."""
        import torch

        if not isinstance(queries, torch.Tensor):
            queries = torch.from_numpy(np.ascontiguousarray(np.atleast_2d(queries), np.float32))
        queries = queries.to(device=self.device, dtype=torch.float32).contiguous()
        if queries.dim() == 1:
            queries = queries[None]
        if queries.shape[1] != self.dim:
            raise ValueError(f"dimension mismatch: vectors {queries.shape[1]}, index {self.dim}")
        nq = queries.shape[0]
        d1 = torch.empty((nq, self.t), dtype=torch.float32, device=self.device)
        d2 = torch.empty((nq, self.t), dtype=torch.float32, device=self.device)
        lib = _lib.load()
        _lib.check(lib.bpq_coarse_dots(self._handle, _lib.ptr(queries), nq, _lib.ptr(d1), _lib.ptr(d2),
                                       _lib.stream_ptr()), "bpq_coarse_dots")
        return d1, d2

    def workspace_bytes(self, engine: str, nq: int, L: int, k: int) -> int:
        lib = _lib.load()
        return int(lib.bpq_search_workspace_size(self._handle, _lib.ENGINES[engine], nq, L, k))

    def make_workspace(self, engine: str, nq: int, L: int, k: int):
        import torch

        return torch.empty(self.workspace_bytes(engine, nq, L, k), dtype=torch.uint8, device=self.device)

    def search(self, queries, L: int, k: int, engine: str = "fbpq", *, out=None, workspace=None,
               stream=None, ncand: bool = False, popped=None, stage_events=None) -> SearchResult:
        """Batched search: queries [nq, D] (torch on this device, or array-like
        copied in).  Returns a SearchResult of device tensors; stream-ordered
        on ``stream`` (default: torch's current stream), no host sync."""
        import torch

        if stream is not None and stream != torch.cuda.current_stream(self.device):
            # upload, output/workspace allocation and the kernels all on the
            # caller's stream, so nothing is read before it is written and the
            # caching allocator ties every temporary to that stream
            with torch.cuda.stream(stream):
                return self.search(queries, L, k, engine, out=out, workspace=workspace, stream=None,
                                   ncand=ncand, popped=popped, stage_events=stage_events)
        if engine not in _lib.ENGINES:
            raise ValueError(f"unknown engine {engine!r}")
        if engine == "hbpq" and self.kind != "hbpq":
            raise ValueError("engine hbpq requires an index built with local codebooks")
        if engine != "hbpq" and self.kind == "hbpq":
            raise ValueError(f"engine {engine} is incompatible with a local-codebook index")
        if L < 1:
            raise ValueError(f"budget must be >= 1, got {L}")
        if k < 1:
            raise ValueError(f"r must be >= 1, got {k}")
        if not isinstance(queries, torch.Tensor):
            queries = torch.from_numpy(np.ascontiguousarray(np.atleast_2d(queries), np.float32))
        queries = queries.to(device=self.device, dtype=torch.float32).contiguous()
        if queries.dim() == 1:
            queries = queries[None]
        if queries.shape[1] != self.dim:
            raise ValueError(f"dimension mismatch: vectors {queries.shape[1]}, index {self.dim}")
        nq = queries.shape[0]
        if out is None:
            out = SearchResult(
                torch.empty((nq, k), dtype=torch.float32, device=self.device),
                torch.empty((nq, k), dtype=torch.int32, device=self.device),
                torch.empty((nq,), dtype=torch.int32, device=self.device),
                torch.empty((nq,), dtype=torch.int64, device=self.device) if ncand else None,
            )
        need = self.workspace_bytes(engine, nq, L, k)
        if workspace is None:
            # one cached workspace per stream: concurrent searches on
            # different streams never share scratch
            key = torch.cuda.current_stream(self.device).cuda_stream
            ws = self._ws.get(key)
            if ws is None or ws.numel() < need:
                ws = self._ws[key] = torch.empty(need, dtype=torch.uint8, device=self.device)
            workspace = ws
        elif workspace.numel() < need:
            raise ValueError(f"workspace too small: {workspace.numel()} < {need}")
        lib = _lib.load()
        ev = None
        if stage_events is not None:
            ev = (ctypes.c_void_p * 5)(*[e.cuda_event for e in stage_events])
        rc = lib.bpq_search_ex(
            self._handle, _lib.ENGINES[engine], _lib.ptr(queries), nq, int(L), int(k),
            _lib.ptr(out.dists), _lib.ptr(out.ids), _lib.ptr(out.counts), _lib.ptr(out.ncand),
            _lib.ptr(popped), ev, _lib.ptr(workspace), workspace.numel(), _lib.stream_ptr(stream),
        )
        _lib.check(rc, "bpq_search")
        return out

    def search_host(self, queries, L: int, k: int, engine: str = "fbpq", *, out=None, pieces: int = 1
                    ) -> SearchResult:
        """Batched search from HOST queries to HOST results: upload ->
        bpq_search -> download, asynchronous on a side stream and ordered on
        torch's current stream (the results are complete once that stream is
        synchronized).  ``queries`` is a pinned CPU tensor (anything else is
        copied into one); ``out`` an optional SearchResult of pinned CPU
        tensors to fill.  ``pieces`` > 1 cuts the batch into slices on their
        own streams so the copies of one slice run under the kernels of
        another -- measured on the B200 at config 1 this LOSES (3.9M q/s with
        one piece, 2.8M with two, 1.9M with three): every search kernel is a
        persistent grid that fills the GPU, so concurrent slices time-slice
        each other while the copies are only 0.3 ms of a 2.5 ms step.  Same
        answers as ``search`` for any ``pieces`` (queries are independent)."""
        import torch

        if not isinstance(queries, torch.Tensor):
            queries = torch.from_numpy(np.ascontiguousarray(np.atleast_2d(queries), np.float32))
        if queries.is_cuda:
            raise ValueError("search_host takes host queries; use search() for device tensors")
        queries = queries.to(torch.float32).contiguous()
        if not queries.is_pinned():
            queries = queries.pin_memory()
        nq = queries.shape[0]
        if out is None:
            out = SearchResult(torch.empty((nq, k), dtype=torch.float32).pin_memory(),
                               torch.empty((nq, k), dtype=torch.int32).pin_memory(),
                               torch.empty((nq,), dtype=torch.int32).pin_memory())
        pieces = max(1, min(int(pieces), nq)) if nq else 1
        cur = torch.cuda.current_stream(self.device)
        side = self.__dict__.setdefault("_side_streams", [])
        while len(side) < pieces:
            side.append(torch.cuda.Stream(device=self.device))
        bufs = self.__dict__.setdefault("_host_bufs", {})
        start = torch.cuda.Event()
        start.record(cur)
        done = []
        for i in range(pieces):
            lo, hi = nq * i // pieces, nq * (i + 1) // pieces
            if hi == lo:
                continue
            s = side[i]
            s.wait_event(start)  # ordered after the caller's earlier work
            with torch.cuda.stream(s):
                key = (i, hi - lo, k)
                b = bufs.get(key)
                if b is None:
                    b = bufs[key] = (torch.empty((hi - lo, self.dim), dtype=torch.float32, device=self.device),
                                     SearchResult(torch.empty((hi - lo, k), dtype=torch.float32, device=self.device),
                                                  torch.empty((hi - lo, k), dtype=torch.int32, device=self.device),
                                                  torch.empty((hi - lo,), dtype=torch.int32, device=self.device)))
                qd, od = b
                qd.copy_(queries[lo:hi], non_blocking=True)
                self.search(qd, L, k, engine, out=od)
                out.dists[lo:hi].copy_(od.dists, non_blocking=True)
                out.ids[lo:hi].copy_(od.ids, non_blocking=True)
                out.counts[lo:hi].copy_(od.counts, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s)
                done.append(ev)
        for ev in done:
            cur.wait_event(ev)
        return out

    # ------------------------------------------------------------- export
    def host_arrays(self) -> dict:
        """The index in the reference's array layout (offsets int64, ids uint32)."""
        out = dict(c1=self.c1.cpu().numpy(), c2=self.c2.cpu().numpy(),
                   offsets=self.offsets.cpu().numpy().view(np.uint32).astype(np.int64),
                   ids=self.ids.cpu().numpy().view(np.uint32), codes=self.codes.cpu().numpy())
        if self.rotation is not None:
            out["rotation"] = self.rotation.cpu().numpy()
        if self.kind == "hbpq":
            out.update(bank1=self.bank1.cpu().numpy(), bank2=self.bank2.cpu().numpy(),
                       rot1=None if self.rot1 is None else self.rot1.cpu().numpy(),
                       rot2=None if self.rot2 is None else self.rot2.cpu().numpy())
        else:
            out.update(books=self.books.cpu().numpy())
        return out

    def save(self, index_path, tables_path=None):
        """Export to BPQI (+ BPQT) in the reference's layout (storage.py:253-343),
        readable by bilayerpq.load_index / load_tables and its CLI."""
        from . import storage

        storage.save_index_arrays(index_path, **self.host_arrays())
        if tables_path is not None and self.kind != "hbpq":
            storage.save_tables_arrays(tables_path, self.cn1.cpu().numpy(), self.cn2.cpu().numpy(),
                                       self.fine_norms.cpu().numpy(), self.cross1.cpu().numpy(),
                                       self.cross2.cpu().numpy())

    # --------------------------------------------------------- constructors
    @classmethod
    def from_reference(cls, index, tables=None, device=None):
        """From a reference-layout MultiIndex / HbpqIndex (duck-typed: any
        object with .coarse.book1.centroids, .cells.offsets, .ids, .codes and
        .fine.codebooks or .bank.books1/.books2), plus optional FbpqTables."""
        coarse = index.coarse
        rot = getattr(coarse, "rotation", None)
        c1 = coarse.book1.centroids
        c2 = coarse.book2.centroids
        bank = getattr(index, "bank", None)
        kw = dict(c1=c1, c2=c2, offsets=index.cells.offsets, ids=index.ids, codes=index.codes, device=device,
                  rotation=None if rot is None else rot.matrix)
        if bank is not None:
            return cls(bank1=bank.books1, bank2=bank.books2,
                       rot1=None if bank.rot1 is None else bank.rot1.matrix,
                       rot2=None if bank.rot2 is None else bank.rot2.matrix, **kw)
        tab = None
        if tables is not None:
            tab = (tables.coarse_norms1, tables.coarse_norms2, tables.fine_norms, tables.cross1, tables.cross2)
        return cls(books=index.fine.codebooks, tables=tab, **kw)

    @classmethod
    def load(cls, index_path, tables_path=None, device=None):
        """From BPQI (+ optional BPQT) files (storage.py:253-360 layout)."""
        from . import storage

        rec = storage.load_index_arrays(index_path)
        tab = storage.load_tables_arrays(tables_path) if tables_path is not None else None
        kw = dict(c1=rec["c1"], c2=rec["c2"], offsets=rec["offsets"], ids=rec["ids"], codes=rec["codes"], device=device,
                  rotation=rec["rotation"])
        if rec["bank1"] is not None:
            return cls(bank1=rec["bank1"], bank2=rec["bank2"], rot1=rec["rot1"], rot2=rec["rot2"], **kw)
        return cls(books=rec["books"], tables=tab, **kw)


def _table_attr(tables, i):
    names = ("coarse_norms1", "coarse_norms2", "fine_norms", "cross1", "cross2")
    if isinstance(tables, (tuple, list)):
        return tables[i]
    return getattr(tables, names[i])
