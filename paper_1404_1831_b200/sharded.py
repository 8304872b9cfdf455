"""Database sharded by point id across GPUs.

Each rank holds its own multi-index over its id range plus the *global*
per-cell counts, so every rank runs the identical traversal (same queries,
same coarse books, same global budget) and scans only its local entries of
the visited cells.  The union of the shards' candidates is then exactly the
single-index candidate set, and merging the per-rank top-k by (dist, id)
reproduces the single-GPU result bit for bit.  The only exchange step is one
all-gather of the per-rank [nq, k] lists (NCCL over NVLink), followed by the
device merge kernel (bpq_merge_topk).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .index import SearchResult


def shard_bounds(n_ids: int, world: int, rank: int, id_base: int = 0):
    """Contiguous id range [lo, hi) owned by ``rank``."""
    lo = id_base + (n_ids * rank) // world
    hi = id_base + (n_ids * (rank + 1)) // world
    return lo, hi


def split_index_arrays(offsets, ids, codes, world: int):
    """Split a built (offsets, ids, codes) index by point id into ``world``
    shard indexes with the same cell table shape; within each cell the
    entries keep ascending id order (multi_index.py:224-230)."""
    offsets = np.asarray(offsets, np.int64)
    ids = np.asarray(ids, np.uint32)
    codes = np.asarray(codes, np.uint8)
    cells = offsets.shape[0] - 1
    n = ids.shape[0]
    base = int(ids.min()) if n else 0
    span = (int(ids.max()) - base + 1) if n else 0
    cell_of = np.repeat(np.arange(cells, dtype=np.int64), np.diff(offsets))
    out = []
    for r in range(world):
        lo, hi = shard_bounds(span, world, r, base)
        sel = (ids >= lo) & (ids < hi)
        cnt = np.bincount(cell_of[sel], minlength=cells)
        off = np.zeros(cells + 1, np.int64)
        np.cumsum(cnt, out=off[1:])
        out.append(dict(offsets=off, ids=ids[sel], codes=codes[sel], id_range=(lo, hi)))
    return out


def merge_results(dists, ids, counts, k: int, stream=None) -> SearchResult:
    """Merge per-shard [nq, k] lists (lists of device tensors, or stacked
    [g, nq, k]) on the device by (dist asc, id asc)."""
    import torch

    d = torch.stack(list(dists)) if isinstance(dists, (list, tuple)) else dists
    i = torch.stack(list(ids)) if isinstance(ids, (list, tuple)) else ids
    c = torch.stack(list(counts)) if isinstance(counts, (list, tuple)) else counts
    d, i, c = d.contiguous(), i.contiguous(), c.contiguous()
    g, nq, kk = d.shape
    if kk != k:
        raise ValueError("per-shard lists must have k columns")
    out = SearchResult(torch.empty((nq, k), dtype=torch.float32, device=d.device),
                       torch.empty((nq, k), dtype=torch.int32, device=d.device),
                       torch.empty((nq,), dtype=torch.int32, device=d.device))
    lib = _lib.load()
    _lib.check(lib.bpq_merge_topk(_lib.ptr(d), _lib.ptr(i), _lib.ptr(c), g, nq, k, _lib.ptr(out.dists),
                                  _lib.ptr(out.ids), _lib.ptr(out.counts), _lib.stream_ptr(stream)),
               "merge_topk")
    return out


def pack_lists(dists, ids, counts):
    """One rank's [nq, k] dists / ids and [nq] counts as the 32-bit word
    buffer of the all-gather: dists | ids | counts (2 nq k + nq words)."""
    import torch

    nq, k = dists.shape
    buf = torch.empty(2 * nq * k + nq, dtype=torch.int32, device=dists.device)
    buf[: nq * k].copy_(dists.reshape(-1).view(torch.int32))
    buf[nq * k: 2 * nq * k].copy_(ids.reshape(-1).view(torch.int32))
    buf[2 * nq * k:].copy_(counts.view(torch.int32))
    return buf


def unpack_lists(gathered, g: int, nq: int, k: int):
    """Host view of an all-gathered packed buffer: (dists [g, nq, k] f32,
    ids [g, nq, k] u32, counts [g, nq] i32) numpy arrays."""
    w = np.asarray(gathered.cpu() if hasattr(gathered, "cpu") else gathered).view(np.int32).reshape(g, -1)
    d = w[:, : nq * k].view(np.float32).reshape(g, nq, k)
    i = w[:, nq * k: 2 * nq * k].view(np.uint32).reshape(g, nq, k)
    c = w[:, 2 * nq * k:].reshape(g, nq)
    return d, i, c


def merge_packed(gathered, g: int, nq: int, k: int, stream=None) -> SearchResult:
    """Merge the all-gathered packed buffer [g][dists nq*k | ids nq*k |
    counts nq] (32-bit words) on the device."""
    import torch

    out = SearchResult(torch.empty((nq, k), dtype=torch.float32, device=gathered.device),
                       torch.empty((nq, k), dtype=torch.int32, device=gathered.device),
                       torch.empty((nq,), dtype=torch.int32, device=gathered.device))
    lib = _lib.load()
    _lib.check(lib.bpq_merge_topk_packed(_lib.ptr(gathered), g, nq, k, _lib.ptr(out.dists), _lib.ptr(out.ids),
                                         _lib.ptr(out.counts), _lib.stream_ptr(stream)), "merge_topk_packed")
    return out


def merge_results_host(dists, ids, counts, k: int):
    """Host restatement of the merge used by CPU (gloo) tests of the
    distributed plumbing; the product path uses merge_results."""
    dists = np.asarray(dists)
    ids = np.asarray(ids).view(np.uint32) if np.asarray(ids).dtype == np.int32 else np.asarray(ids)
    g, nq, _ = dists.shape
    od = np.full((nq, k), np.inf, np.float32)
    oi = np.full((nq, k), 0xFFFFFFFF, np.uint32)
    oc = np.zeros(nq, np.int32)
    for q in range(nq):
        cand = [(float(dists[s, q, x]), int(ids[s, q, x])) for s in range(g) for x in range(int(counts[s][q]))]
        cand.sort()
        cand = cand[:k]
        oc[q] = len(cand)
        for x, (dv, iv) in enumerate(cand):
            od[q, x], oi[q, x] = dv, iv
    return od, oi, oc


class ShardedSearcher:
    """One rank of a sharded search.  ``local`` is this rank's DeviceIndex
    (built with ``global_offsets``).  ``search`` runs the local batched
    search, all-gathers the [nq, k] lists over the process group and merges
    them on the device; every rank returns the merged result."""

    def __init__(self, local, group=None, force_collective=False):
        self.local = local
        self.group = group
        self.force_collective = force_collective  # exercise the exchange even on one rank

    def search(self, queries, L: int, k: int, engine: str = "fbpq", **kw) -> SearchResult:
        import torch
        import torch.distributed as dist

        res = self.local.search(queries, L, k, engine, **kw)
        world = dist.get_world_size(self.group)
        if world == 1 and not self.force_collective:
            return res
        nq = res.dists.shape[0]
        # one all-gather of a packed [dists | ids | counts] buffer per rank
        mine = pack_lists(res.dists, res.ids, res.counts)
        gathered = torch.empty(world * mine.numel(), dtype=torch.int32, device=mine.device)
        dist.all_gather_into_tensor(gathered, mine, group=self.group)
        return merge_packed(gathered, world, nq, k)


# ----------------------------------------------------------------------------
# Query-split sharding.  With the traversal replicated, every
# rank repeats the first layer, the row sort and the multi-sequence traversal
# for all queries, which caps the speed-up (Amdahl).  Here rank r traverses
# only its query slice (against the global cell counts) and records the
# visited non-empty cells; the ranks all-gather those lists (a few cells per
# query at configs 1-4), and every rank then streams its local entries of
# every query's cells.  The final exchange is the same packed all-gather +
# merge as ShardedSearcher.


def query_slice(nq: int, world: int, rank: int):
    """Contiguous query range [lo, hi) traversed by ``rank``."""
    return (nq * rank) // world, (nq * (rank + 1)) // world


def pack_visits(counts, visits):
    """Per-query visit lists [n, cap, 4] (int32) with ``counts`` [n] ->
    packed [sum(counts), 4] in query order (device tensors)."""
    import torch

    counts = counts.to(torch.int64)
    cap = visits.shape[1]
    mask = torch.arange(cap, device=visits.device)[None, :] < counts[:, None]
    return visits[mask]


def _all_gather_padded(t, group=None):
    """All-gather tensors whose first dimension differs across ranks (pad to
    the largest, gather, strip); works over NCCL and gloo."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    sizes = [torch.empty_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(max(sizes), 1)
    pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)])


def exchange_visits(counts, packed, group=None):
    """All ranks' (counts [n_r], packed visits [sum, 4]) in rank order ->
    (counts [nq], packed [total, 4], visit_start [nq + 1] u32-valued int64)."""
    import torch

    all_counts = _all_gather_padded(counts.to(torch.int64), group)
    all_packed = _all_gather_padded(packed, group)
    start = torch.zeros(all_counts.shape[0] + 1, dtype=torch.int64, device=all_counts.device)
    torch.cumsum(all_counts, 0, out=start[1:])
    return all_counts, all_packed, start


class SplitSearcher:
    """One rank of the query-split sharded search.  ``local`` is this rank's
    DeviceIndex built with ``global_offsets`` (point-term FBPQ, M = 8 / 16)."""

    def __init__(self, local, group=None, force_collective=False):
        self.local = local
        self.group = group
        self.force_collective = force_collective
        self._ws = {}

    def _workspace(self, key, nbytes):
        import torch

        ws = self._ws.get(key)
        if ws is None or ws.numel() < nbytes:
            ws = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=self.local.device)
            self._ws[key] = ws
        return ws

    def traverse(self, queries, L: int):
        """bpq_search_split_traverse on this rank's query slice: (counts [n]
        int32, visits [n, cap, 4] int32, global candidate counts [n])."""
        import torch

        lib = _lib.load()
        dix = self.local
        n = queries.shape[0]
        cap = int(lib.bpq_split_visit_cap(dix._handle, int(L)))
        counts = torch.empty(max(n, 1), dtype=torch.int32, device=dix.device)
        visits = torch.empty((max(n, 1), cap, 4), dtype=torch.int32, device=dix.device)
        ncand = torch.empty(max(n, 1), dtype=torch.int64, device=dix.device)
        ws = self._workspace("trav", dix.workspace_bytes("fbpq", max(n, 1), L, 1))
        if n:
            _lib.check(lib.bpq_search_split_traverse(dix._handle, _lib.ptr(queries), n, int(L), _lib.ptr(counts),
                                                     _lib.ptr(visits), cap, _lib.ptr(ncand), _lib.ptr(ws), ws.numel(),
                                                     _lib.stream_ptr()), "search_split_traverse")
        return counts[:n], visits[:n], ncand[:n]

    def scan(self, queries, k: int, packed, start) -> SearchResult:
        """bpq_search_split_scan: this rank's local entries of every query's
        visited cells -> [nq, k] local lists."""
        import torch

        lib = _lib.load()
        dix = self.local
        nq = queries.shape[0]
        total = int(packed.shape[0])
        out = SearchResult(torch.empty((nq, k), dtype=torch.float32, device=dix.device),
                           torch.empty((nq, k), dtype=torch.int32, device=dix.device),
                           torch.empty((nq,), dtype=torch.int32, device=dix.device))
        ws = self._workspace("scan", lib.bpq_split_scan_workspace_size(dix._handle, nq, total))
        st = start.to(torch.int32).contiguous()
        pk = packed.contiguous() if total else torch.zeros((1, 4), dtype=torch.int32, device=dix.device)
        _lib.check(lib.bpq_search_split_scan(dix._handle, _lib.ptr(queries), nq, k, _lib.ptr(pk), _lib.ptr(st), total,
                                             _lib.ptr(out.dists), _lib.ptr(out.ids), _lib.ptr(out.counts),
                                             _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "search_split_scan")
        return out

    def search(self, queries, L: int, k: int, engine: str = "fbpq", **_kw) -> SearchResult:
        """(workspace / stage-event keywords of DeviceIndex.search are accepted and unused)"""
        import torch
        import torch.distributed as dist

        if engine != "fbpq":
            raise ValueError("the query-split path streams point-term FBPQ cells")
        queries = queries.to(device=self.local.device, dtype=torch.float32).contiguous()
        world = dist.get_world_size(self.group)
        rank = dist.get_rank(self.group)
        nq = queries.shape[0]
        lo, hi = query_slice(nq, world, rank)
        counts, visits, _ = self.traverse(queries[lo:hi], L)
        if counts.numel() and bool((counts == -1).any()):  # 0xFFFFFFFF: the query failed
            raise RuntimeError("a query failed the traversal")
        packed = pack_visits(counts, visits)
        _, all_packed, start = exchange_visits(counts, packed, self.group)
        res = self.scan(queries, k, all_packed, start)
        if world == 1 and not self.force_collective:
            return res
        mine = pack_lists(res.dists, res.ids, res.counts)
        gathered = torch.empty(world * mine.numel(), dtype=torch.int32, device=mine.device)
        dist.all_gather_into_tensor(gathered, mine, group=self.group)
        return merge_packed(gathered, world, nq, k)
