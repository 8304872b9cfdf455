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
