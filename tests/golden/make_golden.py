"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
        python tests/golden/make_golden.py

Outputs (committed; the GPU box never reads /root/reference):

* ``kat.npz``   -- known-answer cases for traverse_cells / select_top taken
  from the reference's own tests (worked 3x3 example with a tie,
  TestTraverse budget goldens, quantised-tie pair sums) plus random cases,
  each with the reference's output.
* ``c0.npz``    -- BASELINE.json configs[0] exported from the reference:
  codebooks and codes trained/encoded by the reference, its FBPQ tables,
  1,000 queries, and reference search_fbpq / search_baseline results
  (L=10,000, k=100 and L=1,000, k=10), stage captures for a few queries,
  plus a 4,000-vector encoding sample with the reference's build_index.
* ``hbpq.npz``  -- a smaller HBPQ rig from the same generator (T=16, M=8,
  K=64) with reference search_hbpq / search_baseline results.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import bilayerpq as bq  # noqa: E402  (the reference, read-only)
from bilayerpq import kernels as rk  # noqa: E402
from bilayerpq import multi_index as rmi  # noqa: E402
from bilayerpq import fbpq as rfb  # noqa: E402

from paper_1404_1831_b200 import datagen  # noqa: E402

OUT = Path(__file__).resolve().parent
assert rk.BACKEND == "numba", rk.BACKEND


def _cell_table_offsets(t, counts):
    lin = np.zeros(t * t, np.int64)
    for (i, j), c in counts.items():
        lin[i * t + j] = c
    off = np.zeros(t * t + 1, np.int64)
    np.cumsum(lin, out=off[1:])
    return off


def make_kat():
    cases = {}
    n = 0

    def add_traverse(sr1, sr2, o1, o2, off, budget):
        nonlocal n
        res = rk.traverse_cells(sr1, sr2, o1, o2, off, budget)
        p = f"tr{n}_"
        cases[p + "sr1"] = sr1
        cases[p + "sr2"] = sr2
        cases[p + "o1"] = o1
        cases[p + "o2"] = o2
        cases[p + "off"] = off
        cases[p + "budget"] = np.array(budget, np.int64)
        for name, a in zip(("vi", "vj", "st", "en"), res):
            cases[p + name] = a
        n += 1

    # TestTraverse (reference tests/test_multi_index.py:85-117)
    r1 = np.array([0.25, 0.5, 1.0], np.float32)
    r2 = np.array([0.25, 0.75, 1.25], np.float32)
    counts = {(0, 0): 2, (0, 1): 0, (0, 2): 2, (1, 0): 1, (1, 1): 3, (1, 2): 1,
              (2, 0): 0, (2, 1): 1, (2, 2): 2}
    off = _cell_table_offsets(3, counts)
    for budget in list(range(1, 14)) + [100]:
        o1 = np.argsort(r1, kind="stable").astype(np.int32)
        o2 = np.argsort(r2, kind="stable").astype(np.int32)
        add_traverse(r1[o1].astype(np.float64), r2[o2].astype(np.float64), o1, o2, off, budget)
    # SPEC worked example with a genuine tie (test_multi_index.py:28-46),
    # every cell holding one entry so the visit order is fully observable.
    r1 = np.array([0.1, 0.5, 0.9])
    r2 = np.array([0.2, 0.4, 1.0])
    off = np.arange(10, dtype=np.int64)
    add_traverse(r1, r2, np.arange(3, dtype=np.int32), np.arange(3, dtype=np.int32), off, 100)
    # quantised keys force ties (test_kernels.py:46-65 / test_multi_index.py:58-66)
    rng = np.random.default_rng(1234)
    for _ in range(40):
        t = int(rng.integers(1, 24))
        r1 = (rng.integers(0, 6, t) / 4.0).astype(np.float32)
        r2 = (rng.integers(0, 6, t) / 4.0).astype(np.float32)
        cnt = rng.integers(0, 4, t * t) * (rng.random(t * t) < 0.6)
        off = np.zeros(t * t + 1, np.int64)
        np.cumsum(cnt, out=off[1:])
        if off[-1] == 0:
            continue
        o1 = np.argsort(r1, kind="stable").astype(np.int32)
        o2 = np.argsort(r2, kind="stable").astype(np.int32)
        for budget in (1, 3, 17, 101, 10_000_000):
            add_traverse(r1[o1].astype(np.float64), r2[o2].astype(np.float64), o1, o2, off, budget)
    # larger random (untied) cases
    for t in (64, 200):
        r1 = rng.random(t).astype(np.float32) * 100
        r2 = rng.random(t).astype(np.float32) * 100
        cnt = rng.poisson(0.7, t * t)
        off = np.zeros(t * t + 1, np.int64)
        np.cumsum(cnt, out=off[1:])
        o1 = np.argsort(r1, kind="stable").astype(np.int32)
        o2 = np.argsort(r2, kind="stable").astype(np.int32)
        for budget in (1, 50, 1000, 5000, 10**9):
            add_traverse(r1[o1].astype(np.float64), r2[o2].astype(np.float64), o1, o2, off, budget)
    cases["n_traverse"] = np.array(n, np.int64)

    # select_top goldens (test_multi_index.py:153-178) + random ties
    sel = 0
    sel_inputs = [
        (np.array([5, 3, 9, 1], np.uint32), np.array([0.5, 0.5, 0.1, 0.5], np.float32), 2),
        (np.array([7, 2, 4], np.uint32), np.array([1.0, 1.0, 1.0], np.float32), 3),
        (np.array([7, 2, 4], np.uint32), np.array([1.0, 1.0, 1.0], np.float32), 10),
        (np.array([], np.uint32), np.array([], np.float32), 5),
    ]
    for _ in range(20):
        nn = int(rng.integers(1, 400))
        ids = rng.permutation(100000)[:nn].astype(np.uint32)
        d = (rng.integers(0, 20, nn) / 8.0).astype(np.float32)
        sel_inputs.append((ids, d, int(rng.integers(1, 60))))
    for ids, d, r in sel_inputs:
        oi, od = rmi.select_top(ids, d, r)
        cases[f"sel{sel}_ids"] = ids
        cases[f"sel{sel}_d"] = d
        cases[f"sel{sel}_r"] = np.array(r, np.int64)
        cases[f"sel{sel}_oi"] = oi
        cases[f"sel{sel}_od"] = od
        sel += 1
    cases["n_select"] = np.array(sel, np.int64)
    np.savez_compressed(OUT / "kat.npz", **cases)
    print("kat:", n, "traverse cases,", sel, "select cases")


def make_c0():
    t0 = time.time()
    D, NCOMP, N, NQ, NTRAIN = 128, 1024, 100_000, 1000, 50_000
    cent = datagen.mixture_centres(NCOMP, D)
    base = datagen.clipped_mixture(N, D, NCOMP, datagen.SEED_BASE, cent)
    queries = datagen.clipped_mixture(NQ, D, NCOMP, datagen.SEED_QUERIES, cent)
    train = datagen.clipped_mixture(NTRAIN, D, NCOMP, datagen.SEED_TRAIN, cent)
    coarse = bq.train_coarse(train, 64, seed=0)
    fine = bq.train_fine_global(train, coarse, 8, 256, seed=0)
    index = bq.build_index(base, coarse, fine)
    tables = bq.build_tables(index)
    print(f"c0 trained+built in {time.time() - t0:.1f}s; populated {index.populated_cells()}")
    out = dict(
        c1=coarse.book1.centroids, c2=coarse.book2.centroids, books=fine.codebooks,
        offsets=index.cells.offsets, ids=index.ids, codes=index.codes,
        cn1=tables.coarse_norms1, cn2=tables.coarse_norms2, fine_norms=tables.fine_norms,
        cross1=tables.cross1, cross2=tables.cross2, queries=queries.astype(np.uint8),
    )
    assert np.array_equal(out["queries"].astype(np.float32), queries)
    for eng, nqe, L, k in (("fbpq", NQ, 10_000, 100), ("baseline", 200, 10_000, 100),
                           ("fbpq", 200, 1_000, 10), ("baseline", 200, 1_000, 10)):
        res_i = np.full((nqe, k), 0xFFFFFFFF, np.uint32)
        res_d = np.full((nqe, k), np.inf, np.float32)
        ncand = np.zeros(nqe, np.int64)
        for x in range(nqe):
            if eng == "fbpq":
                ci, cd = rfb.scan_fbpq(index, tables, queries[x], L)
                si, sd = rfb.search_fbpq(index, tables, queries[x], L, k)
            else:
                ci, cd = rmi.scan_baseline(index, queries[x], L)
                si, sd = rmi.search_baseline(index, queries[x], L, k)
            ncand[x] = ci.shape[0]
            res_i[x, : si.shape[0]] = si
            res_d[x, : sd.shape[0]] = sd
        tag = f"{eng}_L{L}_k{k}"
        out[tag + "_ids"] = res_i
        out[tag + "_d"] = res_d
        out[tag + "_ncand"] = ncand
    # stage captures for the first 6 queries (L=10,000)
    for x in range(6):
        st = rfb.prepare_query(index, tables, queries[x])
        vis = rmi.traverse(index.cells, st.r1, st.r2, 10_000)
        ci, cd = rk.scan_tables(*vis, index.ids, index.codes, st.q_norm, st.qdot_coarse1,
                                st.qdot_coarse2, tables.coarse_norms1, tables.coarse_norms2,
                                st.fold, tables.cross1, tables.cross2)
        qr = queries[x]
        e1, e2 = rmi._query_displacement_tables(index.coarse, qr)
        gi, gd = rk.scan_global(*vis, index.ids, index.codes, e1, e2, index.fine.codebooks)
        p = f"stage{x}_"
        out.update({p + "q_norm": np.array(st.q_norm, np.float32), p + "dots1": st.qdot_coarse1,
                    p + "dots2": st.qdot_coarse2, p + "fold": st.fold, p + "r1": st.r1,
                    p + "r2": st.r2, p + "vi": vis[0], p + "vj": vis[1], p + "st": vis[2],
                    p + "en": vis[3], p + "tab_ids": ci, p + "tab_d": cd, p + "glob_d": gd})
    # encoding sample: the reference's build_index on the first 4,000 vectors
    sample = base[:4000]
    sidx = bq.build_index(sample, coarse, fine, id_offset=77)
    ci_, _ = bq.nearest_centroids(np.ascontiguousarray(sample[:, :64]), coarse.book1.centroids)
    out.update(enc_x=sample.astype(np.uint8), enc_offsets=sidx.cells.offsets,
               enc_ids=sidx.ids, enc_codes=sidx.codes, enc_i=ci_)
    np.savez_compressed(OUT / "c0.npz", **out)
    print(f"c0 done in {time.time() - t0:.1f}s")


def make_hbpq():
    t0 = time.time()
    D, NCOMP, N, NQ = 128, 1024, 20_000, 100
    cent = datagen.mixture_centres(NCOMP, D)
    base = datagen.clipped_mixture(N, D, NCOMP, datagen.SEED_BASE, cent)
    queries = datagen.clipped_mixture(NQ, D, NCOMP, datagen.SEED_QUERIES, cent)
    coarse = bq.train_coarse(base, 16, seed=0)
    fine = bq.train_fine_global(base, coarse, 8, 64, seed=0)
    bank = bq.train_local_codebooks(base, coarse, 8, 64, seed=0)
    hindex = bq.build_hbpq_index(base, coarse, bank)
    index = bq.build_index(base, coarse, fine)
    assert np.array_equal(hindex.cells.offsets, index.cells.offsets)
    out = dict(c1=coarse.book1.centroids, c2=coarse.book2.centroids, books=fine.codebooks,
               bank1=bank.books1, bank2=bank.books2, offsets=index.cells.offsets,
               ids=index.ids, codes=index.codes, hcodes=hindex.codes,
               queries=queries.astype(np.uint8))
    L, k = 2000, 50
    for eng in ("hbpq", "baseline", "fbpq"):
        res_i = np.full((NQ, k), 0xFFFFFFFF, np.uint32)
        res_d = np.full((NQ, k), np.inf, np.float32)
        tables = bq.build_tables(index)
        for x in range(NQ):
            if eng == "hbpq":
                si, sd = bq.search_hbpq(hindex, queries[x], L, k)
            elif eng == "baseline":
                si, sd = bq.search_baseline(index, queries[x], L, k)
            else:
                si, sd = bq.search_fbpq(index, tables, queries[x], L, k)
            res_i[x, : si.shape[0]] = si
            res_d[x, : sd.shape[0]] = sd
        out[f"{eng}_ids"] = res_i
        out[f"{eng}_d"] = res_d
    # stage capture for scan_local
    from bilayerpq import hbpq as rhb

    ci, cd = rhb.scan_hbpq(hindex, queries[0], L)
    out.update(stage_local_ids=ci, stage_local_d=cd)
    np.savez_compressed(OUT / "hbpq.npz", **out)
    print(f"hbpq done in {time.time() - t0:.1f}s")


def make_storage():
    """sha256 of the reference's own BPQI/BPQT bytes for the c0 and HBPQ rigs."""
    import hashlib
    import json

    from bilayerpq import storage as rst
    from bilayerpq.hbpq import HbpqIndex, LocalCodebookBank
    from bilayerpq.fbpq import FbpqTables

    g = np.load(OUT / "c0.npz")
    idx = bq.MultiIndex(bq.CoarsePair(bq.Codebook(g["c1"]), bq.Codebook(g["c2"])), bq.CellTable(g["offsets"]),
                        g["ids"], g["codes"], bq.PqCodec(g["books"]))
    tabs = FbpqTables(g["cn1"], g["cn2"], g["fine_norms"], g["cross1"], g["cross2"])
    h = np.load(OUT / "hbpq.npz")
    hidx = HbpqIndex(bq.CoarsePair(bq.Codebook(h["c1"]), bq.Codebook(h["c2"])), bq.CellTable(h["offsets"]),
                     h["ids"], h["hcodes"], LocalCodebookBank(h["bank1"], h["bank2"]))
    import tempfile, os
    with tempfile.TemporaryDirectory() as d:
        rst.save_tables(tabs, os.path.join(d, "t.bpqt"))
        tb = open(os.path.join(d, "t.bpqt"), "rb").read()
    out = {"c0_bpqi_sha256": hashlib.sha256(rst.index_to_bytes(idx)).hexdigest(),
           "c0_bpqt_sha256": hashlib.sha256(tb).hexdigest(),
           "hbpq_bpqi_sha256": hashlib.sha256(rst.index_to_bytes(hidx)).hexdigest()}
    (OUT / "storage_sha256.json").write_text(json.dumps(out, indent=1))
    print("storage:", out)


if __name__ == "__main__":
    what = sys.argv[1:] or ["kat", "c0", "hbpq", "storage"]
    if "storage" in what:
        make_storage()
    if "kat" in what:
        make_kat()
    if "c0" in what:
        make_c0()
    if "hbpq" in what:
        make_hbpq()


def make_rot():
    """OPQ-rotated variants (the paper's 'optimized' engines): a coarse
    rotation learned with the coarse pair, per-half rotations in the bank."""
    t0 = time.time()
    D, NCOMP, N, NQ = 128, 1024, 20_000, 60
    cent = datagen.mixture_centres(NCOMP, D)
    base = datagen.clipped_mixture(N, D, NCOMP, datagen.SEED_BASE, cent)
    queries = datagen.clipped_mixture(NQ, D, NCOMP, datagen.SEED_QUERIES, cent)
    coarse = bq.train_coarse(base, 16, optimized=True, seed=0)
    fine = bq.train_fine_global(base, coarse, 8, 64, seed=0)
    index = bq.build_index(base, coarse, fine)
    tables = bq.build_tables(index)
    bank = bq.train_local_codebooks(base, coarse, 8, 64, seed=0, optimized=True)
    hindex = bq.build_hbpq_index(base, coarse, bank)
    out = dict(c1=coarse.book1.centroids, c2=coarse.book2.centroids, rotation=coarse.rotation.matrix,
               books=fine.codebooks, offsets=index.cells.offsets, ids=index.ids, codes=index.codes,
               cn1=tables.coarse_norms1, cn2=tables.coarse_norms2, fine_norms=tables.fine_norms,
               cross1=tables.cross1, cross2=tables.cross2, bank1=bank.books1, bank2=bank.books2,
               rot1=bank.rot1.matrix, rot2=bank.rot2.matrix, hoffsets=hindex.cells.offsets, hids=hindex.ids,
               hcodes=hindex.codes, queries=queries.astype(np.uint8), enc_x=base[:2000].astype(np.uint8))
    L, k = 2000, 50
    for eng in ("fbpq", "baseline", "hbpq"):
        res_i = np.full((NQ, k), 0xFFFFFFFF, np.uint32)
        res_d = np.full((NQ, k), np.inf, np.float32)
        for x in range(NQ):
            if eng == "fbpq":
                si, sd = bq.search_fbpq(index, tables, queries[x], L, k)
            elif eng == "baseline":
                si, sd = bq.search_baseline(index, queries[x], L, k)
            else:
                si, sd = bq.search_hbpq(hindex, queries[x], L, k)
            res_i[x, : si.shape[0]] = si
            res_d[x, : sd.shape[0]] = sd
        out[f"{eng}_ids"] = res_i
        out[f"{eng}_d"] = res_d
    sidx = bq.build_index(base[:2000], coarse, fine)
    shidx = bq.build_hbpq_index(base[:2000], coarse, bank)
    out.update(enc_offsets=sidx.cells.offsets, enc_ids=sidx.ids, enc_codes=sidx.codes, enc_hcodes=shidx.codes)
    np.savez_compressed(OUT / "rot.npz", **out)
    print(f"rot done in {time.time() - t0:.1f}s")


if __name__ == "__main__" and "rot" in sys.argv[1:]:
    make_rot()
