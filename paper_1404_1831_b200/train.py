"""Codebook training on the device.

Restates the reference's trainers with the heavy O(n*k*d) work on the GPU:

* ``kmeans`` = quantizer._kmeans (quantizer.py:192-193): k-means++ seeding
  (``_kmeanspp_init``, quantizer.py:133-150) then Lloyd iterations
  (``_lloyd``, quantizer.py:153-179, early stop at 1e-5 relative objective
  improvement, empty clusters re-seeded with the largest-residual points);
* ``pq_train`` (quantizer.py:220-231), ``train_coarse`` (multi_index.py:
  149-164, no OPQ), ``train_fine_global`` (multi_index.py:192-196);
* ``train_local_codebooks`` (hbpq.py:90-165): per half-codeword cell, full
  k-means when the cell has >= max(min_points, k) learn points, 3 Lloyd
  refinements of the pooled books when it has >= k, the pooled books
  verbatim below k.

Two random-number modes:

* ``rng="exact"``: every random draw is made on the host with the same
  numpy Generator calls as the reference (``rng.integers`` for the first
  centre, ``rng.choice(n, p=d2/total)`` per further centre, seeded by the
  reference's SeedSequence tags), on the exact f64 squared distances that
  the GPU computes; Lloyd's cluster sums are the reference's f64
  ``np.add.reduceat``.  The result equals the reference's up to argmin
  near-ties of the f32 assignment scores (quantizer.py:124-125), i.e. bit
  for bit on integer-valued data away from such ties
  (tests/test_train.py pins this against reference-trained books).
* ``rng="device"``: the same algorithm with the draws made on the device
  (inverse-CDF sampling of the same distribution from a seeded torch
  generator) and the cluster sums by f64 atomics -- a different random
  stream, for benchmark setup at scale (config 2's 4,096-row local bank).
"""

from __future__ import annotations

import numpy as np

DEFAULT_KMEANS_ITERS = 25  # quantizer.py:17
_REL_TOL = 1e-5            # quantizer.py:18
FALLBACK_REFINE_ITERS = 3  # hbpq.py:39
_MASK = (1 << 63) - 1      # _rng.py:5


def seed_sequence(seed: int, *tags: int) -> np.random.SeedSequence:
    """_rng.seed_sequence (the reference's seed plumbing, _rng.py:8-10)."""
    return np.random.SeedSequence((int(seed) & _MASK, *tags))


def _dev():
    import torch

    return torch.device("cuda")


def _as_dev(x):
    import torch

    if isinstance(x, torch.Tensor):
        return x.to(device=_dev(), dtype=torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(_dev())


def _assign(data, cents):
    """quantizer.nearest_centroids (quantizer.py:109-130) on the device
    through the engine's assignment kernel: (ids int64, d2 f32)."""
    from .encode import nearest_centroids

    cn = (cents.double() * cents.double()).sum(1)  # einsum('ij,ij->i') of f32 rows, rounded once
    return nearest_centroids(data, cents, norms=cn.float().cpu().numpy())


# ------------------------------------------------------------------ k-means
def kmeanspp_init(data, k: int, rng, mode: str = "exact"):
    """quantizer._kmeanspp_init (quantizer.py:133-150).  ``rng`` is a numpy
    Generator (exact) or a torch.Generator on the device (device)."""
    import torch

    n = data.shape[0]
    cents = torch.empty((k, data.shape[1]), dtype=torch.float32, device=data.device)
    first = int(rng.integers(n)) if mode == "exact" else int(torch.randint(n, (1,), generator=rng, device=data.device))
    cents[0] = data[first]
    d2 = ((data - cents[0]).double() ** 2).sum(1)
    for c in range(1, k):
        if mode == "exact":
            d2h = d2.cpu().numpy()
            total = d2h.sum()
            pick = int(rng.integers(n)) if total <= 0.0 else int(rng.choice(n, p=d2h / total))
        else:
            cdf = torch.cumsum(d2, 0)
            total = cdf[-1]
            u = torch.rand((), generator=rng, device=data.device, dtype=torch.float64) * total
            pick_t = torch.searchsorted(cdf, u.reshape(1), right=True).clamp_(max=n - 1)
            pick_t = torch.where(total > 0, pick_t, torch.randint(n, (1,), generator=rng, device=data.device))
            pick = pick_t  # stays on the device (no per-centre host sync)
        cents[c] = data[pick].reshape(-1)
        nd = ((data - cents[c]).double() ** 2).sum(1)
        torch.minimum(d2, nd, out=d2)
    return cents


def lloyd(data, cents, max_iters: int, mode: str = "exact"):
    """quantizer._lloyd (quantizer.py:153-179)."""
    import torch

    k = cents.shape[0]
    cents = cents.clone()
    prev = None
    data_h = data.cpu().numpy() if mode == "exact" else None
    for _ in range(max_iters):
        idx, d2 = _assign(data, cents)
        obj = float(d2.double().sum())
        if prev is not None and prev - obj < _REL_TOL * max(prev, 1e-30):
            break
        prev = obj
        counts = torch.bincount(idx, minlength=k)
        if mode == "exact":
            idx_h = idx.cpu().numpy()
            order = np.argsort(idx_h, kind="stable")
            sorted_idx = idx_h[order]
            starts = np.concatenate(([0], np.flatnonzero(np.diff(sorted_idx)) + 1))
            sums = np.add.reduceat(data_h[order].astype(np.float64), starts, axis=0)
            present = sorted_idx[starts]
            cnt_h = counts.cpu().numpy()
            new = (sums / cnt_h[present, None]).astype(np.float32)
            cents[torch.from_numpy(present).to(cents.device)] = torch.from_numpy(new).to(cents.device)
        else:
            sums = torch.zeros((k, data.shape[1]), dtype=torch.float64, device=data.device)
            sums.index_add_(0, idx, data.double())
            nz = counts > 0
            cents[nz] = (sums[nz] / counts[nz, None]).float()
        empties = torch.nonzero(counts == 0).flatten()
        if empties.numel():
            # np.argsort(-d2, kind="stable")[:n_empty]: largest residual first, ties by row
            far = torch.sort(-d2, stable=True).indices[: empties.numel()]
            cents[empties] = data[far]
    return cents


def kmeans(data, k: int, max_iters: int, rng, mode: str = "exact"):
    """quantizer._kmeans (quantizer.py:192-193) with the argument checks of
    _check_kmeans_args (quantizer.py:182-189)."""
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    if k > data.shape[0]:
        raise ValueError(f"k ({k}) exceeds the number of points ({data.shape[0]})")
    if max_iters < 0:
        raise ValueError("max_iters must be >= 0")
    return lloyd(data, kmeanspp_init(data, k, rng, mode), max_iters, mode)


def _rng(mode, seed_seq):
    import torch

    if mode == "exact":
        return np.random.default_rng(seed_seq)
    g = torch.Generator(device=_dev())
    g.manual_seed(int(seed_seq.generate_state(1, np.uint64)[0]) & _MASK)
    return g


def pq_train(points, m: int, k: int, max_iters: int = DEFAULT_KMEANS_ITERS, seed: int = 0, mode: str = "exact"):
    """quantizer.pq_train (quantizer.py:220-231): independent k-means per
    contiguous part, part p seeded by seed_sequence(seed, 1, p).  Returns
    f32 [m, k, d/m] (numpy)."""
    data = _as_dev(points)
    dim = data.shape[1]
    if m < 1 or dim % m != 0:
        raise ValueError(f"dim {dim} is not divisible into {m} parts")
    ds = dim // m
    books = np.empty((m, k, ds), np.float32)
    for p in range(m):
        part = data[:, p * ds:(p + 1) * ds].contiguous()
        books[p] = kmeans(part, k, max_iters, _rng(mode, seed_sequence(seed, 1, p)), mode).cpu().numpy()
    return books


def train_coarse(learn, t: int, seed: int = 0, mode: str = "exact"):
    """multi_index.train_coarse (multi_index.py:149-164), optimized=False:
    a 2-part product quantizer over the halves -> (c1, c2)."""
    data = _as_dev(learn)
    if data.shape[1] % 2 != 0:
        raise ValueError(f"dimension must be even, got {data.shape[1]}")
    books = pq_train(data, 2, t, seed=seed, mode=mode)
    return books[0], books[1]


def displacements(data, c1, c2):
    """multi_index.displacements (multi_index.py:181-189): (disp, i, j)."""
    import torch

    from .encode import assign_cells

    data = _as_dev(data)
    c1t, c2t = _as_dev(c1), _as_dev(c2)
    i_idx, j_idx = assign_cells(data, np.asarray(c1, np.float32) if not isinstance(c1, torch.Tensor) else c1.cpu().numpy(),
                                np.asarray(c2, np.float32) if not isinstance(c2, torch.Tensor) else c2.cpu().numpy())
    dh = c1t.shape[1]
    disp = torch.empty_like(data)
    disp[:, :dh] = data[:, :dh] - c1t[i_idx]
    disp[:, dh:] = data[:, dh:] - c2t[j_idx]
    return disp, i_idx, j_idx


def _check_fine(dim, m, k):
    from .index import _check_fine_params

    _check_fine_params(dim, m, k)


def train_fine_global(learn, c1, c2, m: int, k: int, seed: int = 0, mode: str = "exact"):
    """multi_index.train_fine_global (multi_index.py:192-196)."""
    _check_fine(2 * np.asarray(c1).shape[1], m, k)
    disp, _, _ = displacements(learn, c1, c2)
    return pq_train(disp, m, k, seed=seed, mode=mode)


# --------------------------------------------------------------- local bank
def _train_half(hdisp, cell_idx, t, m2, k, min_points, seed, half_tag, mode):
    """hbpq._train_half (hbpq.py:90-129), optimized=False."""
    import torch

    ds = hdisp.shape[1] // m2
    pooled = pq_train(hdisp, m2, k, seed=2 * int(seed) + half_tag, mode=mode)
    books = np.empty((t, m2, k, ds), np.float32)
    books[:] = pooled[None]
    cell_h = cell_idx.cpu().numpy()
    order = np.argsort(cell_h, kind="stable")
    bounds = np.searchsorted(cell_h[order], np.arange(t + 1))
    order_t = torch.from_numpy(order).to(hdisp.device)
    full_threshold = max(min_points, k)
    pooled_t = torch.from_numpy(pooled).to(hdisp.device)
    for i in range(t):
        n = int(bounds[i + 1] - bounds[i])
        if n < k:
            continue  # pooled books verbatim
        members = hdisp[order_t[bounds[i]:bounds[i + 1]]]
        for p in range(m2):
            part = members[:, p * ds:(p + 1) * ds].contiguous()
            if n >= full_threshold:
                rng = _rng(mode, seed_sequence(seed, 2, half_tag, i, p))
                books[i, p] = kmeans(part, k, DEFAULT_KMEANS_ITERS, rng, mode).cpu().numpy()
            else:
                books[i, p] = lloyd(part, pooled_t[p], FALLBACK_REFINE_ITERS, mode).cpu().numpy()
    return books


def train_local_codebooks(learn, c1, c2, m: int, k: int, min_points: int | None = None, seed: int = 0,
                          mode: str = "exact"):
    """hbpq.train_local_codebooks (hbpq.py:132-165), optimized=False:
    returns (bank1, bank2), each f32 [T, M/2, K, D/M]."""
    c1 = np.asarray(c1, np.float32)
    _check_fine(2 * c1.shape[1], m, k)
    if min_points is None:
        min_points = 4 * k
    if min_points < 0:
        raise ValueError("min_points must be >= 0")
    t, dh = c1.shape
    disp, i_idx, j_idx = displacements(learn, c1, c2)
    b1 = _train_half(disp[:, :dh].contiguous(), i_idx, t, m // 2, k, min_points, seed, 0, mode)
    b2 = _train_half(disp[:, dh:].contiguous(), j_idx, t, m // 2, k, min_points, seed, 1, mode)
    return b1, b2


def local_bank_for_bench(base, c1, c2, books, cfg, device):
    """Config 2's local bank: train_local_codebooks on a 4,194,304-point
    training draw (about 1,024 learn points per half-codeword at T=4,096,
    SURVEY §8d) with device-side draws (rng="device")."""
    import time

    import torch

    from . import datagen

    t0 = time.time()
    n_learn = int(cfg.get("bank_train", 1 << 22))
    cent = datagen.mixture_centres(cfg["ncomp"], cfg["dim"])
    learn = datagen.clipped_mixture_blocked(n_learn, cfg["dim"], cfg["ncomp"], datagen.SEED_TRAIN, centres=cent)
    learn_t = torch.from_numpy(np.asarray(learn)).to(device)
    b1, b2 = train_local_codebooks(learn_t, c1, c2, cfg["m"], cfg["k"], seed=0, mode="device")
    import sys

    print(f"[setup] local bank trained on {n_learn:,} points in {time.time() - t0:.1f}s", file=sys.stderr, flush=True)
    return b1, b2
