"""Batched recall / engine-comparison harness on the device (SURVEY.md §8f
row f4).

Mirrors the reference's evaluation entry points, batched instead of one
query at a time:

* ``recall_at`` = evalbench.recall_at (evalbench.py:309-327): the fraction of
  queries whose true nearest neighbour is among the first c returned ids;
* ``run_engine`` = evalbench.run_engine (evalbench.py:330-354): search every
  query, report Recall@{1,10,100}, mean candidates and the mean device time
  per query (the reference times each query on the host);
* ``compare_engines`` = evalbench.compare_engines (evalbench.py:373-403):
  paired runs of two engines on the same queries and budget.  The reference
  rescans every candidate of both engines; the batched engine returns only
  its top-r lists, so the relative deviation is taken over the ids the two
  top-r lists share, and the candidate sets are checked through the
  per-query candidate counts;
* ``exact_nn`` = vecio.brute_force_knn with k = 1 (vecio.py:254-...): exact
  squared-L2 nearest neighbour, ties toward the smaller id.  For
  integer-valued data in [0, 255] (BASELINE configs 0, 1, 2, 4) the dot
  products run as an int8 GEMM on the tensor cores (cuBLASLt through
  torch._int_mm, a library GEMM: the harness is not the search path) on the
  offset values x - 128, which is exact in int32, so every distance is exact;
  otherwise in f64.
"""

from __future__ import annotations

import numpy as np

DEFAULT_CUTOFFS = (1, 10, 100)  # evalbench.py:26


def _torch():
    import torch

    return torch


class ExactNN:
    """Exact nearest neighbour (id, squared distance) of each query over base
    rows fed chunk by chunk (``add(first_id, rows)``, ascending ids, e.g.
    while a streamed index build draws them).  Ties break toward the smaller
    id, as vecio.brute_force_knn (vecio.py:254-...)."""

    def __init__(self, queries, integer: bool | None = None):
        torch = _torch()
        q = queries.float()
        self.nq, self.dim = q.shape
        dev = self.dev = q.device
        if integer is None:
            integer = bool(torch.all((q >= 0) & (q <= 255) & (q == torch.round(q))))
        self.integer = integer
        if integer:
            self.q8t = (q - 128).to(torch.int8).t().contiguous()
            self.qs = q.to(torch.int64).sum(1)
            self.qn = (q.to(torch.int64) ** 2).sum(1)
            self.best = torch.full((self.nq,), torch.iinfo(torch.int64).max, dtype=torch.int64, device=dev)
        else:
            self.qd = q.double()
            self.qn = (self.qd * self.qd).sum(1)
            self.bestd = torch.full((self.nq,), float("inf"), dtype=torch.float64, device=dev)
            self.besti = torch.zeros((self.nq,), dtype=torch.int64, device=dev)

    def add(self, first: int, x, rows_per_pass: int = 1 << 18):
        torch = _torch()
        for s in range(0, x.shape[0], rows_per_pass):
            self._add(first + s, x[s:s + rows_per_pass])

    def _add(self, first, x):
        torch = _torch()
        x = x.float()
        n = x.shape[0]
        if n == 0:
            return
        dev = self.dev
        if self.integer:
            x8 = (x - 128).to(torch.int8)
            if n < 32 or n % 8:
                x8 = torch.cat([x8, torch.zeros(((32 - n) if n < 32 else (-n) % 8, self.dim), dtype=torch.int8,
                                                device=dev)])
            dot8 = torch._int_mm(x8, self.q8t)[:n].to(torch.int64)  # (x - 128) . (q - 128), exact in int32
            xs = x.to(torch.int64).sum(1)
            xn = (x.to(torch.int64) ** 2).sum(1)
            # x.q = (x-128).(q-128) + 128 sum x + 128 sum q - 128^2 D
            dot = dot8 + 128 * xs[:, None] + 128 * self.qs[None, :] - 128 * 128 * self.dim
            d = xn[:, None] - 2 * dot  # |x|^2 - 2 x.q, exact (|q|^2 added at the end)
            rows = torch.arange(n, dtype=torch.int64, device=dev)[:, None] + first
            key = (d + (1 << 26)) * (1 << 36) + rows  # distance high, id low
            self.best = torch.minimum(self.best, key.min(0).values)
        else:
            xd = x.double()
            d = (xd * xd).sum(1)[:, None] - 2 * xd @ self.qd.t() + self.qn[None, :]
            m = d.min(0).values
            a = torch.argmax((d == m[None, :]).to(torch.int8), 0)  # first minimal row
            better = m < self.bestd
            self.bestd = torch.where(better, m, self.bestd)
            self.besti = torch.where(better, a + first, self.besti)

    def result(self):
        if self.integer:
            ids = self.best & ((1 << 36) - 1)
            return ids, ((self.best >> 36) - (1 << 26) + self.qn).double()
        return self.besti, self.bestd


def exact_nn(base_chunks, queries, *, integer: bool | None = None):
    """ExactNN over an iterable of (first_id, rows) chunks."""
    acc = ExactNN(queries, integer)
    for first, x in base_chunks:
        acc.add(first, x)
    return acc.result()


def recall_at(ids, counts, true_nn, cutoffs=DEFAULT_CUTOFFS) -> dict:
    """evalbench.recall_at (evalbench.py:309-327) over a batched result:
    ids [nq, r] (padded rows, ``counts`` valid entries each)."""
    torch = _torch()
    ids = torch.as_tensor(ids).to(torch.int64) & 0xFFFFFFFF
    counts = torch.as_tensor(counts, device=ids.device).to(torch.int64)
    nn = torch.as_tensor(true_nn, device=ids.device).to(torch.int64)
    nq = ids.shape[0]
    if nn.shape[0] != nq:
        raise ValueError(f"result count {nq} does not match ground truth {nn.shape[0]}")
    pos = torch.arange(ids.shape[1], device=ids.device)[None, :]
    hit = (ids == nn[:, None]) & (pos < counts[:, None])
    out = {}
    for c in cutoffs:
        if c < 1:
            raise ValueError(f"cutoffs must be >= 1, got {c}")
        out[int(c)] = float(hit[:, :c].any(1).sum().item()) / max(nq, 1)
    return out


def run_engine(index, queries, L: int, r: int, engine: str = "fbpq", true_nn=None, cutoffs=DEFAULT_CUTOFFS):
    """evalbench.run_engine (evalbench.py:330-354), batched: returns
    (SearchResult, report dict with recall, mean_query_ms, mean_candidates)."""
    torch = _torch()
    q = torch.as_tensor(queries).to(device=index.device, dtype=torch.float32)
    index.search(q[: min(8, q.shape[0])], L, r, engine)  # warm-up (workspace, kernel attributes)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = index.search(q, L, r, engine, ncand=True)
    e1.record()
    torch.cuda.synchronize()
    nq = max(q.shape[0], 1)
    report = {"engine": engine, "l": int(L), "num_queries": int(q.shape[0]),
              "recall": ({str(c): v for c, v in recall_at(res.ids, res.counts, true_nn, cutoffs).items()}
                         if true_nn is not None else {}),
              "mean_query_ms": e0.elapsed_time(e1) / nq,
              "mean_candidates": float(res.ncand.double().mean().item())}
    return res, report


def compare_engines(index_a, engine_a, index_b, engine_b, queries, true_nn, L: int, r: int = 100,
                    cutoffs=DEFAULT_CUTOFFS) -> dict:
    """evalbench.compare_engines (evalbench.py:373-403), batched: paired
    runs; raises if the engines' candidate counts differ (the reference
    checks the candidate id sets); relative distance deviation over the ids
    the two top-r lists share, denominator floored at 1e-6 |q|^2."""
    torch = _torch()
    ra, rep_a = run_engine(index_a, queries, L, r, engine_a, true_nn, cutoffs)
    rb, rep_b = run_engine(index_b, queries, L, r, engine_b, true_nn, cutoffs)
    if not torch.equal(ra.ncand, rb.ncand):
        bad = int(torch.nonzero(ra.ncand != rb.ncand)[0].item())
        raise ValueError(f"mismatched candidate sets between engines at query {bad}")
    da, ia, ca = ra.numpy()
    db, ib, cb = rb.numpy()
    q = np.asarray(torch.as_tensor(queries).cpu(), np.float64)
    qn = np.einsum("ij,ij->i", q, q)
    devs = []
    for x in range(da.shape[0]):
        a = dict(zip(ia[x, : ca[x]].view(np.uint32).tolist(), da[x, : ca[x]].tolist()))
        for i, dv in zip(ib[x, : cb[x]].view(np.uint32).tolist(), db[x, : cb[x]].tolist()):
            if i in a:
                devs.append(abs(a[i] - dv) / max(dv, 1e-6 * max(qn[x], 1e-30)))
    devs = np.asarray(devs if devs else [0.0])
    return {"a": rep_a, "b": rep_b, "max_rel_deviation": float(devs.max()),
            "mean_rel_deviation": float(devs.mean()), "shared_ids": int(len(devs))}
