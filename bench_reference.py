"""``bench.py --impl reference``: the REFERENCE package's own CPU search, timed
on this host's cores, on the same workload as the GPU arm.

Nothing from the product package or its CUDA library is imported or mapped
here: the index is built and searched by ``bilayerpq`` itself, installed
unmodified into ``baseline/_ref`` (``pip install --no-index --no-deps
--target baseline/_ref /root/reference/pkg``), with its default
numba kernel backend (``bpq/kernels/__init__.py:26-29``).

* Codebooks: ``tests/golden/c1_books.npz``, trained by the reference itself
  (``tools/train_reference_books.py``: ``train_coarse`` + ``train_fine_global``,
  BASELINE.md §3 "c0-c2: built by the reference itself").  c0 uses the
  reference-exported ``tests/golden/c0.npz`` index.
* Base vectors and queries: the blocked numpy stream of
  ``paper_1404_1831_b200/datagen.py`` (loaded by file path, numpy only), the
  same rows the GPU arm uploads.
* Index build (untimed setup): the reference's ``displacements`` +
  ``pq_encode_batch`` per 2^20-row block in a fork pool (one single-threaded
  BLAS per worker), then ``build_index``'s packing tail (stable argsort by
  cell, ``multi_index.py:224-230``) over the whole base, and
  ``bilayerpq.build_tables`` (``fbpq.py:104-108``).
* Timed: ``bilayerpq.search_fbpq`` / ``search_baseline`` per query
  (``fbpq.py:188-194``, ``multi_index.py:358-367``) in ``os.cpu_count()``
  forked single-threaded workers, each step a bounded
  contiguous query sample; the step time is the wall time from dispatch to
  the last worker's answer.
"""

from __future__ import annotations

import importlib.util
import json
import mmap
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
REF = ROOT / "baseline" / "_ref"

_G = {}  # state inherited by forked workers


def _log(*a):
    print(*a, file=sys.stderr, flush=True)


def _datagen():
    spec = importlib.util.spec_from_file_location("_bpq_datagen", ROOT / "paper_1404_1831_b200" / "datagen.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _one_thread():
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except Exception:
        pass


def _shared(shape, dtype):
    n = int(np.prod(shape)) * np.dtype(dtype).itemsize
    return np.frombuffer(mmap.mmap(-1, max(n, 1)), dtype=dtype, count=int(np.prod(shape))).reshape(shape)


def _encode_blocks(blocks):
    _one_thread()
    bq, dg = _G["bq"], _G["dg"]
    n, dim, ncomp = _G["n"], _G["dim"], _G["ncomp"]
    for b in blocks:
        lo = b * dg.BLOCK
        hi = min(n, lo + dg.BLOCK)
        x = dg.clipped_mixture_block(b, dim, ncomp, dg.SEED_BASE, _G["centres"], hi - lo)
        disp, i_idx, j_idx = bq.displacements(_G["coarse"], x)  # multi_index.py:181-189
        _G["i"][lo:hi] = i_idx
        _G["j"][lo:hi] = j_idx
        _G["codes"][lo:hi] = bq.pq_encode_batch(_G["fine"], disp).astype(np.uint8)  # quantizer.py:235-247


def _search_slice(span):
    lo, hi = span
    bq, q, L, k = _G["bq"], _G["queries"], _G["L"], _G["k"]
    ncand = 0
    for qi in range(lo, hi):
        if _G["engine"] == "fbpq":
            ids, d = bq.search_fbpq(_G["index"], _G["tables"], q[qi], L, k)
        else:
            ids, d = bq.search_baseline(_G["index"], q[qi], L, k)
        ncand += ids.shape[0]
    return hi - lo


def _worker_init():
    _one_thread()
    # JIT-warm this worker (numba compiles on the first call per process
    # unless the on-disk cache is hot)
    _search_slice((0, 1))


def build_reference_index(cfg, workers):
    import bilayerpq as bq

    dg = _datagen()
    name = cfg["name"]
    if name == "c0":
        g = np.load(ROOT / "tests" / "golden" / "c0.npz")
        coarse = bq.CoarsePair(bq.Codebook(g["c1"]), bq.Codebook(g["c2"]))
        fine = bq.PqCodec(g["books"])
        index = bq.MultiIndex(coarse, bq.CellTable(g["offsets"]), g["ids"], g["codes"], fine)
        return bq, index, g["queries"].astype(np.float32), "reference-exported c0 index (tests/golden/c0.npz)"
    books = np.load(ROOT / "tests" / "golden" / "c1_books.npz")
    coarse = bq.CoarsePair(bq.Codebook(books["c1"]), bq.Codebook(books["c2"]))
    fine = bq.PqCodec(books["books"])
    n, dim, ncomp, t = cfg["n"], cfg["dim"], cfg["ncomp"], cfg["t"]
    centres = dg.mixture_centres(ncomp, dim)
    _G.update(bq=bq, dg=dg, n=n, dim=dim, ncomp=ncomp, centres=centres, coarse=coarse, fine=fine,
              i=_shared((n,), np.int64), j=_shared((n,), np.int64), codes=_shared((n, cfg["m"]), np.uint8))
    t0 = time.time()
    nb = (n + dg.BLOCK - 1) // dg.BLOCK
    ctx = mp.get_context("fork")
    procs = [ctx.Process(target=_encode_blocks, args=(range(w, nb, workers),)) for w in range(min(workers, nb))]
    for p in procs:
        p.start()
    for p in procs:
        p.join()
        if p.exitcode != 0:
            raise RuntimeError("reference encode worker failed")
    _log(f"[reference] assigned + encoded {n:,} points in {time.time() - t0:.1f}s ({len(procs)} workers)")
    # build_index's packing tail (multi_index.py:224-230) over the whole base
    i_idx, j_idx = _G.pop("i"), _G.pop("j")
    lin = i_idx * t + j_idx
    order = np.argsort(lin, kind="stable")
    counts = np.bincount(lin, minlength=t * t)
    offsets = np.zeros(t * t + 1, np.int64)
    np.cumsum(counts, out=offsets[1:])
    ids = order.astype(np.uint32)
    index = bq.MultiIndex(coarse, bq.CellTable(offsets), ids, np.asarray(_G.pop("codes"))[order], fine)
    queries = dg.clipped_mixture_block(0, dim, ncomp, dg.SEED_QUERIES, centres, cfg["nq"])
    _log(f"[reference] index built in {time.time() - t0:.1f}s: populated={int((counts > 0).sum())}")
    return bq, index, queries, ("reference-trained codebooks (tests/golden/c1_books.npz); base encoded by "
                                "bilayerpq.displacements + pq_encode_batch, packed as build_index")


def run(args, cfg, metric, config):
    if not (REF / "bilayerpq").is_dir():
        print(json.dumps({"impl": "reference", "unavailable": "baseline/_ref/bilayerpq is not installed "
                          "(pip install --no-index --no-deps --target baseline/_ref /root/reference/pkg)"}))
        return
    if cfg["name"] not in ("c0", "c1") or cfg["engine"] not in ("fbpq", "baseline"):
        print(json.dumps({"impl": "reference", "unavailable": f"the reference cannot build {cfg['name']} "
                          f"({cfg['engine']}) on a host in bench time (BASELINE.md §3); GPU-arm cpu_baseline "
                          "times the C port instead"}))
        return
    sys.path.insert(0, str(REF))
    os.environ.setdefault("NUMBA_CACHE_DIR", str(REF / ".numba_cache"))
    cores = os.cpu_count() or 1
    bq, index, queries, how = build_reference_index(cfg, cores)
    from bilayerpq import kernels as rk

    tables = bq.build_tables(index) if cfg["engine"] == "fbpq" else None
    _G.update(bq=bq, index=index, tables=tables, queries=queries, L=cfg["L"], k=cfg["topk"], engine=cfg["engine"])
    nq = queries.shape[0]
    # one core (parent, single-threaded BLAS): JIT warm-up, then a short sample
    _one_thread()
    _search_slice((0, 2))
    t0 = time.perf_counter()
    n1 = _search_slice((0, min(nq, 16)))
    one_core = n1 / (time.perf_counter() - t0)
    per_q = 1.0 / one_core
    # all cores: each step hands every worker a contiguous slice sized for ~0.4 s of work
    per_worker = int(max(1, min(nq // cores, round(0.4 / per_q))))
    step_q = per_worker * cores
    ctx = mp.get_context("fork")
    times = []
    with ctx.Pool(cores, initializer=_worker_init) as pool:
        pool.map(_search_slice, [(0, 1)] * cores, chunksize=1)  # all workers up
        for s in range(args.warmup + args.steps):
            base = (s * step_q) % max(1, nq - step_q + 1)
            spans = [(base + w * per_worker, base + (w + 1) * per_worker) for w in range(cores)]
            t0 = time.perf_counter()
            done = sum(pool.map(_search_slice, spans, chunksize=1))
            dt = time.perf_counter() - t0
            if s >= args.warmup:
                times.append((done, dt))
    tot_q = sum(x[0] for x in times)
    tot_t = sum(x[1] for x in times)
    v = tot_q / tot_t
    sample = (f"{step_q} queries per step ({per_worker} per worker, contiguous, rotating through the {nq}-query "
              f"batch), L={cfg['L']}, k={cfg['topk']}; bilayerpq {cfg['engine']} search (numba backend "
              f"{rk.BACKEND}) in {cores} forked single-threaded workers; {how}")
    line = {"impl": "reference", "metric": metric, "value": v, "unit": "queries/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / max(1, len(times)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded BASELINE.json generator, blocked numpy stream shared with the GPU arm)",
            "config": config,
            "cpu_baseline": {"value": v, "unit": "queries/s", "cores": cores, "kind": "reference",
                             "sample": sample, "one_core_value": one_core},
            "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
