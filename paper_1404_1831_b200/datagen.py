"""Seeded synthetic workloads named by BASELINE.json.

The paper's BIGANN/GIST sets are not available; these
generators stand in with the configs' shapes and value distributions.

* ``clipped_mixture`` -- configs 0/1/2/4: ``x = clip(round(c_j + 20 z), 0, 255)``
  with ``j ~ U{0..ncomp-1}``, ``c_j ~ U[0,100]^D``, ``z ~ N(0, I)``.  Centres
  come from seed 0, the database from seed 1, queries from seed 2 and the
  training draw from seed 3 (BASELINE.json configs[0]).
* ``normalized_mixture`` -- config 3: centres ``N(0, I)``, within-component
  sigma 0.3, then L2-normalised.

The numpy versions are the reference-side generators (used to export the
config-0 index from the reference); the torch versions draw the same
distributions on the GPU for the 10M-1B point configs, where a host draw
would dominate setup time.  They are not bit-identical streams.
"""

from __future__ import annotations

import numpy as np

SEED_CENTRES, SEED_BASE, SEED_QUERIES, SEED_TRAIN = 0, 1, 2, 3


def mixture_centres(ncomp: int, dim: int, seed: int = SEED_CENTRES) -> np.ndarray:
    return np.random.default_rng(seed).uniform(0.0, 100.0, (ncomp, dim))


def clipped_mixture(n: int, dim: int, ncomp: int, seed: int, centres=None) -> np.ndarray:
    """numpy draw: component indices first, then the normals."""
    if centres is None:
        centres = mixture_centres(ncomp, dim)
    rng = np.random.default_rng(seed)
    j = rng.integers(0, ncomp, n)
    z = rng.standard_normal((n, dim))
    return np.clip(np.round(centres[j] + 20.0 * z), 0, 255).astype(np.float32)


BLOCK = 1 << 20


def clipped_mixture_block(b: int, dim: int, ncomp: int, seed: int, centres, rows: int | None = None) -> np.ndarray:
    """numpy draw of block ``b`` (rows [b*2^20, (b+1)*2^20)) of a blocked
    clipped-mixture stream: every block has its own generator seeded by
    (seed, b), so a process pool can draw disjoint blocks and any two
    processes (the GPU arm and the CPU reference arm of bench.py) produce
    the same rows bit for bit.  ``rows`` truncates the block."""
    rng = np.random.default_rng(np.random.SeedSequence((int(seed), int(b), 0xB200)))
    n = BLOCK if rows is None else int(rows)
    j = rng.integers(0, ncomp, BLOCK)[:n]  # full-block draws: a prefix is the same rows
    z = rng.standard_normal((BLOCK, dim), dtype=np.float32)[:n]
    out = centres[j].astype(np.float32)
    out += np.float32(20.0) * z
    np.round(out, out=out)
    np.clip(out, 0, 255, out=out)
    return out


def clipped_mixture_blocked(n: int, dim: int, ncomp: int, seed: int, workers: int | None = None,
                            centres=None) -> np.ndarray:
    """Rows [0, n) of the blocked stream, drawn by a fork pool into one
    shared buffer (10M x 128 f32 in a few seconds on a many-core host)."""
    import mmap
    import multiprocessing as mp
    import os

    if centres is None:
        centres = mixture_centres(ncomp, dim)
    nb = (n + BLOCK - 1) // BLOCK
    buf = mmap.mmap(-1, max(n * dim * 4, 1))
    out = np.frombuffer(buf, dtype=np.float32, count=n * dim).reshape(n, dim)
    workers = max(1, min(nb, workers or os.cpu_count() or 1))

    def run(blocks):
        for b in blocks:
            lo = b * BLOCK
            hi = min(n, lo + BLOCK)
            out[lo:hi] = clipped_mixture_block(b, dim, ncomp, seed, centres, hi - lo)

    if workers == 1 or nb == 1:
        run(range(nb))
        return out
    procs = []
    ctx = mp.get_context("fork")
    for w in range(workers):
        p = ctx.Process(target=run, args=(range(w, nb, workers),))
        p.start()
        procs.append(p)
    for p in procs:
        p.join()
        if p.exitcode != 0:
            raise RuntimeError("data generation worker failed")
    return out


def clipped_mixture_torch(n: int, dim: int, ncomp: int, seed: int, device, centres=None, chunk=1 << 22):
    """Same distribution drawn on ``device`` with a seeded torch generator."""
    import torch

    if centres is None:
        centres = mixture_centres(ncomp, dim)
    cent = torch.as_tensor(centres, dtype=torch.float32, device=device)
    g = torch.Generator(device=device)
    g.manual_seed(1_000_003 * seed + 17)
    out = torch.empty((n, dim), dtype=torch.float32, device=device)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        j = torch.randint(0, ncomp, (e - s,), generator=g, device=device)
        z = torch.randn((e - s, dim), generator=g, device=device)
        out[s:e] = torch.clamp(torch.round(cent[j] + 20.0 * z), 0, 255)
    return out


def clipped_mixture_chunk(s: int, e: int, dim: int, ncomp: int, seed: int, device, cent=None):
    """Rows [s, e) of a streamed clipped-mixture database: each 2^20-row
    block has its own seeded generator, so any row range is reproducible
    without generating the rows before it."""
    import torch

    if cent is None:
        cent = torch.as_tensor(mixture_centres(ncomp, dim), dtype=torch.float32, device=device)
    out = torch.empty((e - s, dim), dtype=torch.float32, device=device)
    blk = 1 << 20
    g = torch.Generator(device=device)
    for b0 in range((s // blk) * blk, e, blk):
        g.manual_seed(1_000_003 * seed + 7919 * (b0 // blk) + 17)
        j = torch.randint(0, ncomp, (blk,), generator=g, device=device)
        z = torch.randn((blk, dim), generator=g, device=device)
        lo, hi = max(s, b0), min(e, b0 + blk)
        sl = slice(lo - b0, hi - b0)
        out[lo - s : hi - s] = torch.clamp(torch.round(cent[j[sl]] + 20.0 * z[sl]), 0, 255)
    return out


def normalized_mixture_torch(n: int, dim: int, ncomp: int, seed: int, device, sigma=0.3, chunk=1 << 22):
    import torch

    gc = torch.Generator(device=device)
    gc.manual_seed(SEED_CENTRES + 7)
    cent = torch.randn((ncomp, dim), generator=gc, device=device)
    g = torch.Generator(device=device)
    g.manual_seed(1_000_003 * seed + 29)
    out = torch.empty((n, dim), dtype=torch.float32, device=device)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        j = torch.randint(0, ncomp, (e - s,), generator=g, device=device)
        x = cent[j] + sigma * torch.randn((e - s, dim), generator=g, device=device)
        out[s:e] = x / torch.linalg.vector_norm(x, dim=1, keepdim=True)
    return out


def normalized_centres_torch(ncomp: int, dim: int, device, seed: int = SEED_CENTRES):
    import torch

    gc = torch.Generator(device=device)
    gc.manual_seed(seed + 7)
    return torch.randn((ncomp, dim), generator=gc, device=device)


def normalized_mixture_chunk(s: int, e: int, dim: int, ncomp: int, seed: int, device, cent, sigma=0.3):
    """Rows [s, e) of the config-3 database (centres N(0, I), within-component
    sigma, then L2-normalised), reproducible per 2^20-row block."""
    import torch

    out = torch.empty((e - s, dim), dtype=torch.float32, device=device)
    blk = 1 << 20
    g = torch.Generator(device=device)
    for b0 in range((s // blk) * blk, e, blk):
        g.manual_seed(1_000_003 * seed + 7919 * (b0 // blk) + 29)
        j = torch.randint(0, ncomp, (blk,), generator=g, device=device)
        z = torch.randn((blk, dim), generator=g, device=device)
        lo, hi = max(s, b0), min(e, b0 + blk)
        sl = slice(lo - b0, hi - b0)
        x = cent[j[sl]] + sigma * z[sl]
        out[lo - s : hi - s] = x / torch.linalg.vector_norm(x, dim=1, keepdim=True)
    return out
