"""Sharded (multi-GPU) host logic on CPU: world_size-2 gloo process group.

Each rank takes its id-range shard of the config-0 index with the global
cell counts, runs the per-rank search (here the CPU oracle with the shard's
local entries stands in for the device kernel), all-gathers the [nq, k]
lists over the group exactly as ShardedSearcher does, merges, and must
reproduce the single-index reference result."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1404_1831_b200 import sharded


def test_shard_split_preserves_cells(c0):
    parts = sharded.split_index_arrays(c0["offsets"], c0["ids"], c0["codes"], 3)
    tot = sum(np.diff(p["offsets"]) for p in parts)
    np.testing.assert_array_equal(tot, np.diff(c0["offsets"]))
    for p in parts:
        lo, hi = p["id_range"]
        assert ((p["ids"] >= lo) & (p["ids"] < hi)).all()
        off = p["offsets"]
        for cell in np.flatnonzero(np.diff(off) > 1)[:50]:
            assert np.all(np.diff(p["ids"][off[cell]:off[cell + 1]].astype(np.int64)) > 0)


def _local_search(c0, shard, q, L, k):
    """Per-rank search with GLOBAL traversal counts and LOCAL entries."""
    from oracle import oracle as orc

    tables = (c0["cn1"], c0["cn2"], c0["fine_norms"], c0["cross1"], c0["cross2"])
    nq = q.shape[0]
    d = np.full((nq, k), np.inf, np.float32)
    ids = np.full((nq, k), 0xFFFFFFFF, np.uint32)
    cnt = np.zeros(nq, np.int32)
    cn1, cn2, fn, x1, x2 = tables
    for x in range(nq):
        q_norm, d1, d2, fold, r1, r2 = orc.prepare_query(c0["c1"], c0["c2"], c0["books"], fn, q[x])
        vi, vj, _, _ = orc.traverse(c0["offsets"], r1, r2, L)  # global budget
        lin = vi.astype(np.int64) * c0["c1"].shape[0] + vj
        off = shard["offsets"]
        st, en = off[lin], off[lin + 1]
        ci, cd = orc.scan_tables(vi, vj, st, en, shard["ids"], shard["codes"], q_norm, d1, d2, cn1, cn2, fold, x1, x2)
        si, sd = orc.select_top(ci, cd, k)
        cnt[x] = si.shape[0]
        ids[x, : cnt[x]] = si
        d[x, : cnt[x]] = sd
    return d, ids, cnt


def _worker(rank, world, port, c0, q, L, k, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shard = sharded.split_index_arrays(c0["offsets"], c0["ids"], c0["codes"], world)[rank]
    d, i, c = _local_search(c0, shard, q, L, k)
    # the exchange of ShardedSearcher.search: one all-gather of the packed
    # [dists | ids | counts] buffer (gloo has no all_gather_into_tensor)
    mine = sharded.pack_lists(torch.from_numpy(d), torch.from_numpy(i.view(np.int32)), torch.from_numpy(c))
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    gd, gi, gc = sharded.unpack_lists(torch.cat(parts), world, q.shape[0], k)
    md, mi, mc = sharded.merge_results_host(gd, gi, gc, k)
    if rank == 0:
        np.savez(out_path, d=md, i=mi, c=mc)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_merge_equals_single_index(c0, tmp_path):
    q = c0["queries"][:12].astype(np.float32)
    L, k = 10_000, 100
    out = tmp_path / "merged.npz"
    port = 29500 + (os.getpid() % 2000)
    mp.spawn(_worker, args=(2, port, c0, q, L, k, str(out)), nprocs=2, join=True)
    got = np.load(out)
    np.testing.assert_array_equal(got["i"], c0["fbpq_L10000_k100_ids"][:12])
    np.testing.assert_array_equal(got["d"], c0["fbpq_L10000_k100_d"][:12])


def _split_worker(rank, world, port, c0, q, L, k, out_path):
    """Query-split sharding over gloo: rank r traverses its query slice (the
    oracle's traversal against the global counts), the visited-cell lists
    are exchanged with sharded.exchange_visits, every rank scans its shard's
    entries of all queries' cells, and the packed top-k exchange + merge of
    ShardedSearcher follows."""
    from oracle import oracle as orc

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = c0["c1"].shape[0]
    shard = sharded.split_index_arrays(c0["offsets"], c0["ids"], c0["codes"], world)[rank]
    tables = (c0["cn1"], c0["cn2"], c0["fine_norms"], c0["cross1"], c0["cross2"])
    cn1, cn2, fn, x1, x2 = tables
    nq = q.shape[0]
    lo, hi = sharded.query_slice(nq, world, rank)
    counts, rows = [], []
    for x in range(lo, hi):
        *_, r1, r2 = orc.prepare_query(c0["c1"], c0["c2"], c0["books"], fn, q[x])
        vi, vj, _, _ = orc.traverse(c0["offsets"], r1, r2, L)  # global budget
        lin = vi.astype(np.int64) * t + vj
        g = np.diff(c0["offsets"])[lin]
        rows.append(np.stack([lin, g, np.zeros_like(lin), np.zeros_like(lin)], 1).astype(np.int32))
        counts.append(lin.shape[0])
    counts_t = torch.tensor(counts, dtype=torch.int32)
    packed = torch.from_numpy(np.concatenate(rows) if rows else np.zeros((0, 4), np.int32))
    allc, allp, start = sharded.exchange_visits(counts_t, packed)
    assert allc.shape[0] == nq and int(start[-1]) == allp.shape[0]
    d = np.full((nq, k), np.inf, np.float32)
    ids = np.full((nq, k), 0xFFFFFFFF, np.uint32)
    cnt = np.zeros(nq, np.int32)
    off = shard["offsets"]
    for x in range(nq):
        v = allp[int(start[x]):int(start[x + 1])].numpy()
        lin = v[:, 0].astype(np.int64)
        q_norm, d1, d2, fold, _, _ = orc.prepare_query(c0["c1"], c0["c2"], c0["books"], fn, q[x])
        vi, vj = (lin // t).astype(np.int32), (lin % t).astype(np.int32)
        ci, cd = orc.scan_tables(vi, vj, off[lin], off[lin + 1], shard["ids"], shard["codes"], q_norm, d1, d2, cn1,
                                 cn2, fold, x1, x2)
        si, sd = orc.select_top(ci, cd, k)
        cnt[x] = si.shape[0]
        ids[x, : cnt[x]] = si
        d[x, : cnt[x]] = sd
    mine = sharded.pack_lists(torch.from_numpy(d), torch.from_numpy(ids.view(np.int32)), torch.from_numpy(cnt))
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    gd, gi, gc = sharded.unpack_lists(torch.cat(parts), world, nq, k)
    md, mi, mc = sharded.merge_results_host(gd, gi, gc, k)
    if rank == 0:
        np.savez(out_path, d=md, i=mi, c=mc)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_query_split_equals_single_index(c0, tmp_path):
    q = c0["queries"][:13].astype(np.float32)  # odd count: unequal query slices
    L, k = 10_000, 100
    out = tmp_path / "split.npz"
    port = 31500 + (os.getpid() % 2000)
    mp.spawn(_split_worker, args=(2, port, c0, q, L, k, str(out)), nprocs=2, join=True)
    got = np.load(out)
    np.testing.assert_array_equal(got["i"], c0["fbpq_L10000_k100_ids"][:13])
    np.testing.assert_array_equal(got["d"], c0["fbpq_L10000_k100_d"][:13])
