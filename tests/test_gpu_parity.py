"""GPU parity: the CUDA engine (through the C ABI) against the oracle and the
reference-generated golden fixtures."""

import numpy as np
import pytest

from parity import check_topk

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture(scope="module")
def kernels(torch_cuda):
    from paper_1404_1831_b200 import kernels as k

    return k


@pytest.fixture(scope="module")
def c0_index(torch_cuda, c0):
    from paper_1404_1831_b200 import DeviceIndex

    tables = (c0["cn1"], c0["cn2"], c0["fine_norms"], c0["cross1"], c0["cross2"])
    return DeviceIndex(c1=c0["c1"], c2=c0["c2"], offsets=c0["offsets"], ids=c0["ids"], codes=c0["codes"],
                       books=c0["books"], tables=tables)


# ---------------------------------------------------------------- stage level
def test_traverse_stage_known_answers(kat, kernels):
    """traverse_cells on the GPU == the reference's numba output, element for element."""
    for n in range(int(kat["n_traverse"])):
        p = f"tr{n}_"
        got = kernels.traverse_cells(kat[p + "sr1"], kat[p + "sr2"], kat[p + "o1"], kat[p + "o2"],
                                     kat[p + "off"], int(kat[p + "budget"]))
        for g, name in zip(got, ("vi", "vj", "st", "en")):
            np.testing.assert_array_equal(g, kat[p + name], err_msg=f"case {n} {name}")


def test_traverse_stage_c0(c0, kernels, oracle):
    for x in range(6):
        p = f"stage{x}_"
        sr1, sr2, o1, o2 = oracle.sort_halves(c0[p + "r1"], c0[p + "r2"])
        got = kernels.traverse_cells(sr1, sr2, o1, o2, c0["offsets"], 10_000)
        for g, name in zip(got, ("vi", "vj", "st", "en")):
            np.testing.assert_array_equal(g, c0[p + name])


def test_scan_stages_bit_exact(c0, kernels):
    dh = c0["c1"].shape[1]
    for x in range(6):
        p = f"stage{x}_"
        vis = (c0[p + "vi"], c0[p + "vj"], c0[p + "st"], c0[p + "en"])
        ti, td = kernels.scan_tables(*vis, c0["ids"], c0["codes"], c0[p + "q_norm"], c0[p + "dots1"],
                                     c0[p + "dots2"], c0["cn1"], c0["cn2"], c0[p + "fold"], c0["cross1"],
                                     c0["cross2"])
        np.testing.assert_array_equal(ti, c0[p + "tab_ids"])
        np.testing.assert_array_equal(td.view(np.uint32), c0[p + "tab_d"].view(np.uint32))
        q = c0["queries"][x].astype(np.float32)
        gi, gd = kernels.scan_global(*vis, c0["ids"], c0["codes"], q[None, :dh] - c0["c1"],
                                     q[None, dh:] - c0["c2"], c0["books"])
        np.testing.assert_array_equal(gd.view(np.uint32), c0[p + "glob_d"].view(np.uint32))


def test_scan_local_bit_exact(hbpq_rig, kernels, oracle):
    g = hbpq_rig
    q = g["queries"][0].astype(np.float32)
    qr, _, _, r1, r2 = oracle.coarse_scan(g["c1"], g["c2"], q)
    vis = oracle.traverse(g["offsets"], r1, r2, 2000)
    dh = g["c1"].shape[1]
    ci, cd = kernels.scan_local(*vis, g["ids"], g["hcodes"], qr[None, :dh] - g["c1"], qr[None, dh:] - g["c2"],
                                g["bank1"], g["bank2"])
    np.testing.assert_array_equal(ci, g["stage_local_ids"])
    np.testing.assert_array_equal(cd.view(np.uint32), g["stage_local_d"].view(np.uint32))


def test_empty_visit_stage(kernels):
    e = np.empty(0, np.int32)
    ids, d = kernels.scan_tables(e, e, np.empty(0, np.int64), np.empty(0, np.int64), np.zeros(3, np.uint32),
                                 np.zeros((3, 2), np.uint8), 1.0, np.zeros(2, np.float32), np.zeros(2, np.float32),
                                 np.zeros(2, np.float32), np.zeros(2, np.float32), np.zeros((2, 4), np.float32),
                                 np.zeros((2, 1, 4), np.float32), np.zeros((2, 1, 4), np.float32))
    assert ids.size == 0 and d.size == 0


# ------------------------------------------------------------------ end to end
def _ctx(index, q, L):
    """Boundary near-tie context for the §8c(ii) classifier (oracle/parity.py)."""
    from oracle import oracle as orc

    return dict(orc=orc, index=index, queries=q, L=L)


def _orc_index(g, hbpq=False, rotated=False):
    from oracle import oracle as orc

    rot = g["rotation"] if rotated else None
    if hbpq:
        pre = "h" if rotated else ""
        return orc.Index(g["c1"], g["c2"], g[pre + "offsets"], g[pre + "ids"], g["hcodes"], bank1=g["bank1"],
                         bank2=g["bank2"], rotation=rot, rot1=g.get("rot1"), rot2=g.get("rot2"))
    tables = (g["cn1"], g["cn2"], g["fine_norms"], g["cross1"], g["cross2"])
    return orc.Index(g["c1"], g["c2"], g["offsets"], g["ids"], g["codes"], books=g["books"], tables=tables,
                     rotation=rot)


@pytest.fixture(scope="module")
def c0_oracle(c0):
    return _orc_index(c0)


def _qn(q):
    return np.einsum("ij,ij->i", q.astype(np.float64), q.astype(np.float64))


@pytest.mark.parametrize("engine,nq,L,k", [("fbpq", 1000, 10_000, 100), ("baseline", 200, 10_000, 100),
                                           ("fbpq", 200, 1_000, 10), ("baseline", 200, 1_000, 10)])
def test_search_c0_vs_reference(c0, c0_index, c0_oracle, engine, nq, L, k):
    q = c0["queries"][:nq].astype(np.float32)
    res = c0_index.search(q, L, k, engine, ncand=True)
    d, i, c = res.numpy()
    tag = f"{engine}_L{L}_k{k}"
    want_c = np.minimum(k, c0[tag + "_ncand"][:nq])
    check_topk(d, i, c, c0[tag + "_d"][:nq], c0[tag + "_ids"][:nq], want_c, _qn(q),
               got_ncand=res.ncand.cpu().numpy(), want_ncand=c0[tag + "_ncand"][:nq], **_ctx(c0_oracle, q, L))


def test_fbpq_exact_and_point_term_modes(c0, c0_index, c0_oracle, torch_cuda):
    """The default FBPQ scan reads the index's per-entry point term; the
    exact mode gathers cross terms in the reference's operation order.  Both
    meet the reference contract, agree on counts and on every distance to
    1e-6 relative, and return identical id lists away from exact ties."""
    from paper_1404_1831_b200 import DeviceIndex

    tables = (c0["cn1"], c0["cn2"], c0["fine_norms"], c0["cross1"], c0["cross2"])
    exact = DeviceIndex(c1=c0["c1"], c2=c0["c2"], offsets=c0["offsets"], ids=c0["ids"], codes=c0["codes"],
                        books=c0["books"], tables=tables, fbpq_exact=True)
    q = c0["queries"][:500].astype(np.float32)
    de, ie, ce = exact.search(q, 10_000, 100, "fbpq").numpy()
    dp, ip, cp = c0_index.search(q, 10_000, 100, "fbpq").numpy()
    want_c = np.minimum(100, c0["fbpq_L10000_k100_ncand"][:500])
    check_topk(de, ie, ce, c0["fbpq_L10000_k100_d"][:500], c0["fbpq_L10000_k100_ids"][:500], want_c, _qn(q),
               **_ctx(c0_oracle, q, 10_000))
    np.testing.assert_array_equal(ce, cp)
    np.testing.assert_allclose(dp, de, rtol=1e-6)
    # the two modes against each other: same contract (the reference's c0 index as the oracle context)
    check_topk(dp, ip, cp, de, ie, ce, _qn(q), **_ctx(c0_oracle, q, 10_000))


def test_search_hbpq_vs_reference(hbpq_rig, torch_cuda):
    from paper_1404_1831_b200 import DeviceIndex

    g = hbpq_rig
    dix = DeviceIndex(c1=g["c1"], c2=g["c2"], offsets=g["offsets"], ids=g["ids"], codes=g["hcodes"],
                      bank1=g["bank1"], bank2=g["bank2"])
    q = g["queries"].astype(np.float32)
    d, i, c = dix.search(q, 2000, 50, "hbpq").numpy()
    want_c = (g["hbpq_ids"] != 0xFFFFFFFF).sum(1)
    check_topk(d, i, c, g["hbpq_d"], g["hbpq_ids"], want_c, _qn(q), **_ctx(_orc_index(g, hbpq=True), q, 2000))


def test_per_query_api_matches_batch(c0, c0_index):
    import paper_1404_1831_b200 as bpq

    q = c0["queries"][3].astype(np.float32)
    ids, d = bpq.search_fbpq(c0_index, None, q, 10_000, 100)
    bd, bi, bc = c0_index.search(q[None], 10_000, 100, "fbpq").numpy()
    assert ids.dtype == np.uint32 and d.dtype == np.float32
    np.testing.assert_array_equal(ids, bi[0, : bc[0]])
    with pytest.raises(ValueError):
        bpq.search_fbpq(c0_index, None, q, 10_000, 0)
    with pytest.raises(ValueError):
        c0_index.search(q[None], 0, 10, "fbpq")
    with pytest.raises(ValueError):
        c0_index.search(q[None], 10, 10, "hbpq")


def test_search_host_pipelined_equals_search(c0, c0_index, torch_cuda):
    """DeviceIndex.search_host (host queries -> host results, slices pipelined
    over CUDA streams) returns exactly what search() returns, for any number
    of slices, with pinned or pageable inputs and a caller-owned output."""
    from paper_1404_1831_b200.index import SearchResult

    q = c0["queries"][:301].astype(np.float32)
    want = c0_index.search(q, 10_000, 100, "fbpq").numpy()
    for pieces in (1, 2, 3):
        got = c0_index.search_host(q, 10_000, 100, "fbpq", pieces=pieces)
        torch_cuda.cuda.synchronize()
        np.testing.assert_array_equal(got.dists.numpy(), want[0])
        np.testing.assert_array_equal(got.ids.numpy().view(np.uint32), want[1])
        np.testing.assert_array_equal(got.counts.numpy(), want[2])
    out = SearchResult(torch_cuda.empty((301, 100), dtype=torch_cuda.float32).pin_memory(),
                       torch_cuda.empty((301, 100), dtype=torch_cuda.int32).pin_memory(),
                       torch_cuda.empty((301,), dtype=torch_cuda.int32).pin_memory())
    qh = torch_cuda.from_numpy(q).pin_memory()
    for _ in range(2):  # cached slice buffers are reused
        c0_index.search_host(qh, 10_000, 100, "fbpq", out=out, pieces=2)
        torch_cuda.cuda.synchronize()
        np.testing.assert_array_equal(out.ids.numpy().view(np.uint32), want[1])


def test_search_vs_oracle_small_synthetic(torch_cuda, oracle):
    """Random small index incl. empty cells, budgets below/above N, k > candidates."""
    from paper_1404_1831_b200 import DeviceIndex

    rng = np.random.default_rng(7)
    t, dim, m, kk, n = 24, 32, 4, 16, 3000
    c1 = rng.normal(size=(t, dim // 2)).astype(np.float32)
    c2 = rng.normal(size=(t, dim // 2)).astype(np.float32)
    books = rng.normal(scale=0.2, size=(m, kk, dim // m)).astype(np.float32)
    base = rng.normal(size=(n, dim)).astype(np.float32)
    off, ids, codes = oracle.build_index(base, c1, c2, books)
    idx = oracle.Index(c1, c2, off, ids, codes, books=books)
    dix = DeviceIndex(c1=c1, c2=c2, offsets=off, ids=ids, codes=codes, books=books, tables=idx.tables)
    q = rng.normal(size=(64, dim)).astype(np.float32)
    for engine in ("fbpq", "baseline"):
        for L, k in ((1, 1), (37, 5), (500, 50), (5000, 100), (n, 1000)):
            wd, wi, wc, _ = oracle.search_batch_numpy(idx, engine, q, L, k)
            d, i, c = dix.search(q, L, k, engine).numpy()
            check_topk(d, i, c, wd, wi, wc, _qn(q), **_ctx(idx, q, L))


@pytest.mark.parametrize("engine", ["fbpq", "baseline"])
def test_cell_lists_do_not_change_results(c0, torch_cuda, engine):
    """Sparse band enumeration (populated-cell lists) is an exact
    re-implementation of the dense one: identical outputs."""
    from paper_1404_1831_b200 import DeviceIndex

    tables = (c0["cn1"], c0["cn2"], c0["fine_norms"], c0["cross1"], c0["cross2"])
    kw = dict(c1=c0["c1"], c2=c0["c2"], offsets=c0["offsets"], ids=c0["ids"], codes=c0["codes"],
              books=c0["books"], tables=tables)
    dense = DeviceIndex(cell_lists=False, **kw)
    sparse = DeviceIndex(cell_lists=True, **kw)
    assert sparse.row_ptr is not None and dense.row_ptr is None
    q = c0["queries"][:300].astype(np.float32)
    for L, k in ((10_000, 100), (1_000, 10), (1, 1), (200_000, 5)):
        a = dense.search(q, L, k, engine, ncand=True)
        b = sparse.search(q, L, k, engine, ncand=True)
        for x, y in zip(a.numpy(), b.numpy()):
            np.testing.assert_array_equal(x, y)
        np.testing.assert_array_equal(a.ncand.cpu().numpy(), b.ncand.cpu().numpy())


def test_sparse_table_vs_oracle(torch_cuda, oracle):
    """A mostly-empty cell table (clustered data, large T) with lists on."""
    from paper_1404_1831_b200 import DeviceIndex

    rng = np.random.default_rng(3)
    t, dim, m, kk, n = 200, 32, 4, 32, 20_000
    cent = rng.normal(scale=5.0, size=(60, dim)).astype(np.float32)
    base = (cent[rng.integers(0, 60, n)] + rng.normal(size=(n, dim))).astype(np.float32)
    c1 = base[rng.choice(n, t, replace=False), : dim // 2].copy()
    c2 = base[rng.choice(n, t, replace=False), dim // 2 :].copy()
    books = rng.normal(scale=0.5, size=(m, kk, dim // m)).astype(np.float32)
    off, ids, codes = oracle.build_index(base, c1, c2, books)
    assert np.count_nonzero(np.diff(off)) < t * t // 4
    idx = oracle.Index(c1, c2, off, ids, codes, books=books)
    dix = DeviceIndex(c1=c1, c2=c2, offsets=off, ids=ids, codes=codes, books=books, tables=idx.tables)
    assert dix.row_ptr is not None
    q = (cent[rng.integers(0, 60, 64)] + rng.normal(size=(64, dim))).astype(np.float32)
    for L, k in ((1, 1), (100, 10), (2000, 100), (50_000, 20)):
        wd, wi, wc, _ = oracle.search_batch_numpy(idx, "fbpq", q, L, k)
        d, i, c = dix.search(q, L, k, "fbpq").numpy()
        check_topk(d, i, c, wd, wi, wc, _qn(q), **_ctx(idx, q, L))


def test_partial_sort_and_retry_pass(torch_cuda, oracle):
    """Sparse table with T > 1024: queries start on the partial (top-1024)
    sort; those whose traversal outgrows it are re-run through the full-sort
    retry pass.  Results must equal the always-full-sort path and the oracle."""
    import torch

    from paper_1404_1831_b200 import DeviceIndex

    rng = np.random.default_rng(11)
    t, dim, m, kk, n = 1500, 32, 4, 16, 30_000
    cent = rng.normal(scale=6.0, size=(400, dim)).astype(np.float32)
    base = (cent[rng.integers(0, 400, n)] + rng.normal(size=(n, dim))).astype(np.float32)
    c1 = base[rng.choice(n, t, replace=False), : dim // 2].copy()
    c2 = base[rng.choice(n, t, replace=False), dim // 2 :].copy()
    books = rng.normal(scale=0.4, size=(m, kk, dim // m)).astype(np.float32)
    off, ids, codes = oracle.build_index(base, c1, c2, books)
    idx = oracle.Index(c1, c2, off, ids, codes, books=books)
    dix = DeviceIndex(c1=c1, c2=c2, offsets=off, ids=ids, codes=codes, books=books, tables=idx.tables)
    assert dix.row_ptr is not None
    q = (cent[rng.integers(0, 400, 48)] + rng.normal(size=(48, dim))).astype(np.float32)
    for L, k in ((10, 5), (3000, 50), (n, 20)):
        part = dix.search(q, L, k, "fbpq", ncand=True)
        popped = torch.empty(q.shape[0], dtype=torch.int64, device="cuda")
        full = dix.search(q, L, k, "fbpq", ncand=True, popped=popped)   # popped forces the full sort
        for x, y in zip(part.numpy(), full.numpy()):
            np.testing.assert_array_equal(x, y)
        np.testing.assert_array_equal(part.ncand.cpu().numpy(), full.ncand.cpu().numpy())
        wd, wi, wc, _ = oracle.search_batch_numpy(idx, "fbpq", q[:16], L, k)
        d, i, c = part.numpy()
        check_topk(d[:16], i[:16], c[:16], wd, wi, wc, _qn(q[:16]), **_ctx(idx, q[:16], L))


@pytest.mark.parametrize("t", [4500, 8200])
def test_partial_sort_large_t_matches_full_sort(torch_cuda, t):
    """Row top-k with the keys in shared memory (T > 4096: 16 and 32 keys per
    thread) must give the same results as the full-sort path."""
    import torch

    from paper_1404_1831_b200 import encode

    rng = np.random.default_rng(t)
    dim, m, kk, n = 16, 4, 16, 60_000
    cent = rng.normal(scale=6.0, size=(300, dim)).astype(np.float32)
    base = (cent[rng.integers(0, 300, n)] + rng.normal(size=(n, dim))).astype(np.float32)
    c1 = (base[rng.integers(0, n, t), : dim // 2] + rng.normal(scale=0.5, size=(t, dim // 2))).astype(np.float32)
    c2 = (base[rng.integers(0, n, t), dim // 2 :] + rng.normal(scale=0.5, size=(t, dim // 2))).astype(np.float32)
    books = rng.normal(scale=0.4, size=(m, kk, dim // m)).astype(np.float32)
    dix = encode.build_index(base, c1, c2, books)
    assert dix.row_ptr is not None
    q = (cent[rng.integers(0, 300, 64)] + rng.normal(size=(64, dim))).astype(np.float32)
    for L, k in ((100, 10), (5000, 50)):
        part = dix.search(q, L, k, "fbpq", ncand=True)
        popped = torch.empty(q.shape[0], dtype=torch.int64, device="cuda")
        full = dix.search(q, L, k, "fbpq", ncand=True, popped=popped)   # popped forces the full sort
        for x, y in zip(part.numpy(), full.numpy()):
            np.testing.assert_array_equal(x, y)
        np.testing.assert_array_equal(part.ncand.cpu().numpy(), full.ncand.cpu().numpy())


@pytest.mark.parametrize("m", [8, 16])
def test_large_cells_every_engine_vs_oracle(torch_cuda, oracle, m):
    """Few coarse codewords, so cells hold hundreds of entries and take the
    per-cell paths: FBPQ point term (the TMA large-cell stream kernel) and
    exact LUT, and the Multi-D-ADC / HBPQ residual lookup tables.  N is not
    a multiple of 4, so the stream's tail past the last aligned chunk is read
    directly.  Contract of SURVEY §8c(ii)."""
    from paper_1404_1831_b200 import DeviceIndex

    rng = np.random.default_rng(77 + m)
    t, dim, kk, n = 10, 32, 32, 60_003
    base = rng.normal(size=(n, dim)).astype(np.float32)
    c1 = base[rng.choice(n, t, replace=False), : dim // 2].copy()
    c2 = base[rng.choice(n, t, replace=False), dim // 2 :].copy()
    books = (0.3 * rng.normal(size=(m, kk, dim // m))).astype(np.float32)
    off, ids, codes = oracle.build_index(base, c1, c2, books)
    assert np.diff(off).max() >= 1000
    bank1 = (0.3 * rng.normal(size=(t, m // 2, kk, dim // m))).astype(np.float32)
    bank2 = (0.3 * rng.normal(size=(t, m // 2, kk, dim // m))).astype(np.float32)
    idx = oracle.Index(c1, c2, off, ids, codes, books=books)
    hidx = oracle.Index(c1, c2, off, ids, codes, bank1=bank1, bank2=bank2)
    q = rng.normal(size=(32, dim)).astype(np.float32)
    dix = DeviceIndex(c1=c1, c2=c2, offsets=off, ids=ids, codes=codes, books=books, tables=idx.tables)
    dex = DeviceIndex(c1=c1, c2=c2, offsets=off, ids=ids, codes=codes, books=books, tables=idx.tables,
                      fbpq_exact=True)
    hix = DeviceIndex(c1=c1, c2=c2, offsets=off, ids=ids, codes=codes, bank1=bank1, bank2=bank2)
    for L, k in ((2000, 20), (20_000, 100)):
        for eng, di, oi in (("fbpq", dix, idx), ("fbpq", dex, idx), ("baseline", dix, idx), ("hbpq", hix, hidx)):
            wd, wi, wc, _ = oracle.search_batch_numpy(oi, eng, q, L, k)
            d, i, c = di.search(q, L, k, eng).numpy()
            check_topk(d, i, c, wd, wi, wc, _qn(q), **_ctx(oi, q, L))


@pytest.mark.parametrize("m,k", [(8, 100), (16, 100), (8, 1000)])
def test_stream_adversarial_order_rolls_back(torch_cuda, oracle, m, k):
    """One huge cell whose entries get closer to the query as their ids grow:
    nearly every candidate beats the k-th key so far, so the large-cell
    stream's optimistic segments overflow the top-k buffer and take the
    roll-back + safe-segment path (cell_flow_kernel).  Answers must still
    follow SURVEY §8c(ii)."""
    from paper_1404_1831_b200 import DeviceIndex

    rng = np.random.default_rng(500 + m + k)
    t, dim, kk, n = 4, 32, 32, 50_000
    c1 = (10.0 * rng.normal(size=(t, dim // 2))).astype(np.float32)
    c2 = (10.0 * rng.normal(size=(t, dim // 2))).astype(np.float32)
    u = rng.normal(size=dim)
    u /= np.linalg.norm(u)
    shrink = 3.0 * (1.0 - np.arange(n) / n)[:, None]
    base = (np.concatenate([c1[0], c2[0]])[None, :] + shrink * u[None, :]
            + 0.02 * rng.normal(size=(n, dim))).astype(np.float32)
    books = (0.5 * rng.normal(size=(m, kk, dim // m))).astype(np.float32)
    off, ids, codes = oracle.build_index(base, c1, c2, books)
    assert np.diff(off).max() >= 40_000
    idx = oracle.Index(c1, c2, off, ids, codes, books=books)
    q = (np.concatenate([c1[0], c2[0]])[None, :] + 0.05 * rng.normal(size=(6, dim))).astype(np.float32)
    dix = DeviceIndex(c1=c1, c2=c2, offsets=off, ids=ids, codes=codes, books=books, tables=idx.tables)
    for L in (n, 20_000):
        wd, wi, wc, _ = oracle.search_batch_numpy(idx, "fbpq", q, L, k)
        d, i, c = dix.search(q, L, k, "fbpq").numpy()
        check_topk(d, i, c, wd, wi, wc, _qn(q), **_ctx(idx, q, L))


def test_checked_build_stream_bounds(torch_cuda):
    """compute-sanitizer is closed on the build pool, so the stream kernel
    has a checked build (csrc/build_checked.sh, -DBPQ_CHECKED): every index
    it forms (table offsets, entry ranges incl. the padded over-read, cell
    cursor, id gather) is tested against its bound and violations are
    counted.  tools/sanitize_case.py (large cells with an unaligned end,
    k = 300 / 1000, the adversarial roll-back case) must leave the counter
    at 0 while the kernel demonstrably ran (stream entries > 0)."""
    import os
    import re
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    lib = root / "paper_1404_1831_b200" / "libbpq_b200_checked.so"
    if not lib.exists():
        pytest.skip("checked library not built (csrc/build_checked.sh)")
    env = dict(os.environ, BPQ_LIB=str(lib), BPQ_CHECK_REPORT="1")
    out = subprocess.run([sys.executable, str(root / "tools" / "sanitize_case.py")], env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    m = re.search(r"check_failures=(\d+) stream_entries=(\d+)", out.stdout)
    assert m, out.stdout[-2000:]
    assert int(m.group(1)) == 0
    assert int(m.group(2)) > 100_000


def test_empty_index_returns_nothing(torch_cuda):
    from paper_1404_1831_b200 import DeviceIndex

    t, dim, m = 4, 8, 2
    rng = np.random.default_rng(1)
    dix = DeviceIndex(c1=rng.normal(size=(t, 4)), c2=rng.normal(size=(t, 4)), offsets=np.zeros(t * t + 1, np.int64),
                      ids=np.zeros(0, np.uint32), codes=np.zeros((0, m), np.uint8),
                      books=rng.normal(size=(m, 8, 4)).astype(np.float32))
    d, i, c = dix.search(rng.normal(size=(3, dim)).astype(np.float32), 10, 5, "fbpq").numpy()
    assert (c == 0).all() and np.isinf(d).all() and (i == 0xFFFFFFFF).all()


@pytest.mark.parametrize("exact", [True, False])
def test_sharded_global_budget_equals_single(c0, torch_cuda, exact):
    """Shards built with id offsets + global counts: merged top-k == 1-index top-k.

    Exact mode (reference operation order) is bit for bit.  The point-term
    mode sums a candidate's M fold lookups in an order keyed on the entry's
    position in its own (shard's) arrays (search_impl.cuh LaneLut), so a
    distance may move by an ulp between the sharded and single layouts: the
    merged answer must then meet the SURVEY 8c(ii) contract against the
    single-index answer."""
    import torch

    from paper_1404_1831_b200 import DeviceIndex, sharded
    from oracle import oracle as orc

    q = c0["queries"][:100].astype(np.float32)
    tables = (c0["cn1"], c0["cn2"], c0["fine_norms"], c0["cross1"], c0["cross2"])
    full = DeviceIndex(c1=c0["c1"], c2=c0["c2"], offsets=c0["offsets"], ids=c0["ids"], codes=c0["codes"],
                       books=c0["books"], tables=tables, exact=exact)
    want = full.search(q, 10_000, 100, "fbpq").numpy()
    shards = sharded.split_index_arrays(c0["offsets"], c0["ids"], c0["codes"], 3)
    outs = []
    for s in shards:
        dix = DeviceIndex(c1=c0["c1"], c2=c0["c2"], offsets=s["offsets"], ids=s["ids"], codes=s["codes"],
                          books=c0["books"], tables=tables, global_offsets=c0["offsets"],
                          num_entries_global=int(c0["offsets"][-1]), exact=exact)
        outs.append(dix.search(q, 10_000, 100, "fbpq"))
    merged = sharded.merge_results([o.dists for o in outs], [o.ids for o in outs], [o.counts for o in outs], 100)
    got = merged.numpy()
    if exact:
        np.testing.assert_array_equal(got[1], want[1])
        np.testing.assert_array_equal(got[0], want[0])
        np.testing.assert_array_equal(got[2], want[2])
    else:
        np.testing.assert_array_equal(got[2], want[2])
        qn = np.einsum("ij,ij->i", q.astype(np.float64), q.astype(np.float64))
        check_topk(got[0], got[1], got[2], want[0], want[1], want[2], qn)


def test_device_encoding_matches_reference(c0, torch_cuda):
    from paper_1404_1831_b200 import encode

    x = c0["enc_x"].astype(np.float32)
    dix = encode.build_index(x, c0["c1"], c0["c2"], c0["books"], id_offset=77)
    off = dix.offsets.cpu().numpy().view(np.uint32).astype(np.int64)
    ids = dix.ids.cpu().numpy().view(np.uint32)
    codes = dix.codes.cpu().numpy()
    # every row identical to the reference's build_index or an argmin near-tie
    from oracle.parity import classify_encoding

    s = classify_encoding(x, c0["c1"], c0["c2"], c0["books"], (off, ids, codes),
                          (c0["enc_offsets"], c0["enc_ids"], c0["enc_codes"]), id_offset=77)
    assert s["unclassified"] == 0, s
    assert off[-1] == x.shape[0] and np.all(np.diff(off) >= 0)


@pytest.mark.parametrize("engine", ["fbpq", "baseline"])
def test_m16_high_dim_normalized_vs_oracle(torch_cuda, oracle, engine):
    """M=16 codes (uint4 loads), D=96 L2-normalised data (config-3 style, no
    integer structure), dense and sparse traversal."""
    from paper_1404_1831_b200 import DeviceIndex

    rng = np.random.default_rng(21)
    t, dim, m, kk, n = 48, 96, 16, 32, 8000
    cent = rng.normal(size=(64, dim)).astype(np.float32)
    x = cent[rng.integers(0, 64, n)] + 0.3 * rng.normal(size=(n, dim))
    base = (x / np.linalg.norm(x, axis=1, keepdims=True)).astype(np.float32)
    c1 = base[rng.choice(n, t, replace=False), : dim // 2].copy()
    c2 = base[rng.choice(n, t, replace=False), dim // 2 :].copy()
    books = (0.05 * rng.normal(size=(m, kk, dim // m))).astype(np.float32)
    off, ids, codes = oracle.build_index(base, c1, c2, books)
    idx = oracle.Index(c1, c2, off, ids, codes, books=books)
    xq = cent[rng.integers(0, 64, 40)] + 0.3 * rng.normal(size=(40, dim))
    q = (xq / np.linalg.norm(xq, axis=1, keepdims=True)).astype(np.float32)
    for lists in (False, True):
        dix = DeviceIndex(c1=c1, c2=c2, offsets=off, ids=ids, codes=codes, books=books, tables=idx.tables,
                          cell_lists=lists)
        for L, k in ((50, 10), (1500, 100)):
            wd, wi, wc, _ = oracle.search_batch_numpy(idx, engine, q, L, k)
            d, i, c = dix.search(q, L, k, engine).numpy()
            check_topk(d, i, c, wd, wi, wc, _qn(q), **_ctx(idx, q, L))


def test_scale_sparse_index_vs_oracle(torch_cuda, oracle):
    """A 1M-point index from the BASELINE clipped-mixture generator (T=1024,
    sparse cell table, partial sort + retry in play) against the C oracle."""
    import torch

    from paper_1404_1831_b200 import DeviceIndex, datagen, encode

    dev = torch.device("cuda")
    cent = datagen.mixture_centres(1024, 128)
    train = datagen.clipped_mixture_torch(131_072, 128, 1024, datagen.SEED_TRAIN, dev, cent)
    c1 = encode.train_kmeans(train[:, :64].contiguous(), 1024, iters=6, seed=1)
    c2 = encode.train_kmeans(train[:, 64:].contiguous(), 1024, iters=6, seed=2)
    i, j = encode.assign_cells(train, c1, c2)
    disp = train - torch.cat([torch.from_numpy(c1).to(dev)[i], torch.from_numpy(c2).to(dev)[j]], 1)
    books = np.stack([encode.train_kmeans(disp[:, p * 16:(p + 1) * 16].contiguous(), 256, iters=4, seed=10 + p)
                      for p in range(8)])
    base = datagen.clipped_mixture_torch(1_000_000, 128, 1024, datagen.SEED_BASE, dev, cent)
    dix = encode.build_index(base, c1, c2, books)
    assert dix.row_ptr is not None
    q = datagen.clipped_mixture_torch(256, 128, 1024, datagen.SEED_QUERIES, dev, cent).cpu().numpy()
    off = dix.offsets.cpu().numpy().view(np.uint32).astype(np.int64)
    idx = oracle.Index(c1, c2, off, dix.ids.cpu().numpy().view(np.uint32), dix.codes.cpu().numpy(), books=books,
                       tables=(dix.cn1.cpu().numpy(), dix.cn2.cpu().numpy(), dix.fine_norms.cpu().numpy(),
                               dix.cross1.cpu().numpy(), dix.cross2.cpu().numpy()))
    for L, k in ((1000, 10), (10_000, 100), (100_000, 100)):
        res = dix.search(q, L, k, "fbpq", ncand=True)
        d, i_, c = res.numpy()
        # properties on all queries: sorted, counts, candidates >= L (budget semantics)
        assert (np.diff(d, axis=1)[:, : k - 1][c[:, None] > np.arange(1, k)[None, :]] >= 0).all()
        assert (res.ncand.cpu().numpy() >= min(L, 1_000_000)).all()
        wd, wi, wc, wn = oracle.search_batch_c(idx, "fbpq", q[:48], L, k, threads=8)
        check_topk(d[:48], i_[:48], c[:48], wd, wi, wc, _qn(q[:48]), got_ncand=res.ncand.cpu().numpy()[:48],
                   want_ncand=wn, **_ctx(idx, q[:48], L))


@pytest.mark.parametrize("t,n,m,L", [(4096, 2_000_000, 8, 10_000), (16384, 4_000_000, 8, 10_000),
                                     (16384, 2_000_000, 16, 30_000)])
def test_config_shapes_vs_oracle(torch_cuda, oracle, t, n, m, L):
    """BASELINE configs 1 and 4 at their table shapes (T = 4096 / 16384 per
    half, 128-d clipped-integer mixture with T components, M = 8 / 16 x 256)
    on a base small enough for a test: tensor-core first layer, partial row
    sort with T / 512 keys per thread, sparse traversal, small-cell scan and
    the large-cell stream, 64 queries against the C oracle with every
    mismatch classified."""
    import torch

    from paper_1404_1831_b200 import datagen, encode

    dev = torch.device("cuda")
    dim, ntrain = 128, 16 * t
    cent = datagen.mixture_centres(t, dim)
    train = datagen.clipped_mixture_torch(ntrain, dim, t, datagen.SEED_TRAIN, dev, cent)
    c1 = encode.train_kmeans(train[:, :64].contiguous(), t, iters=4, seed=1)
    c2 = encode.train_kmeans(train[:, 64:].contiguous(), t, iters=4, seed=2)
    i, j = encode.assign_cells(train, c1, c2)
    disp = train - torch.cat([torch.from_numpy(c1).to(dev)[i], torch.from_numpy(c2).to(dev)[j]], 1)
    ds = dim // m
    books = np.stack([encode.train_kmeans(disp[:, p * ds:(p + 1) * ds].contiguous(), 256, iters=4, seed=10 + p)
                      for p in range(m)])
    base = datagen.clipped_mixture_torch(n, dim, t, datagen.SEED_BASE, dev, cent)
    dix = encode.build_index(base, c1, c2, books)
    del base
    assert dix.row_ptr is not None
    q = datagen.clipped_mixture_torch(64, dim, t, datagen.SEED_QUERIES, dev, cent).cpu().numpy()
    off = dix.offsets.cpu().numpy().view(np.uint32).astype(np.int64)
    idx = oracle.Index(c1, c2, off, dix.ids.cpu().numpy().view(np.uint32), dix.codes.cpu().numpy(), books=books,
                       tables=(dix.cn1.cpu().numpy(), dix.cn2.cpu().numpy(), dix.fine_norms.cpu().numpy(),
                               dix.cross1.cpu().numpy(), dix.cross2.cpu().numpy()))
    for budget, k in ((L, 100), (1000, 10)):
        res = dix.search(q, budget, k, "fbpq", ncand=True)
        d, i_, c = res.numpy()
        wd, wi, wc, wn = oracle.search_batch_c(idx, "fbpq", q, budget, k, threads=8)
        check_topk(d, i_, c, wd, wi, wc, _qn(q), got_ncand=res.ncand.cpu().numpy(), want_ncand=wn,
                   **_ctx(idx, q, budget))


def test_export_round_trip_through_bpqi(c0, c0_index, tmp_path):
    """A device index exported to BPQI/BPQT (reference layout) and reloaded
    searches identically."""
    import hashlib
    import json
    from pathlib import Path

    from paper_1404_1831_b200 import DeviceIndex

    c0_index.save(tmp_path / "i.bpqi", tmp_path / "t.bpqt")
    sha = json.loads((Path(__file__).resolve().parent / "golden" / "storage_sha256.json").read_text())
    assert hashlib.sha256((tmp_path / "i.bpqi").read_bytes()).hexdigest() == sha["c0_bpqi_sha256"]
    back = DeviceIndex.load(tmp_path / "i.bpqi", tmp_path / "t.bpqt")
    q = c0["queries"][:50].astype(np.float32)
    for x, y in zip(c0_index.search(q, 5000, 50).numpy(), back.search(q, 5000, 50).numpy()):
        np.testing.assert_array_equal(x, y)


def test_rotated_variants_vs_reference(torch_cuda):
    """OPQ-rotated coarse pair (FBPQ, Multi-D-ADC) and rotated local banks
    (HBPQ) against the reference's own results; device encoding with
    rotations against the reference's build_index / build_hbpq_index."""
    from conftest import GOLDEN

    from paper_1404_1831_b200 import DeviceIndex, encode

    g = dict(np.load(GOLDEN / "rot.npz"))
    tables = (g["cn1"], g["cn2"], g["fine_norms"], g["cross1"], g["cross2"])
    dix = DeviceIndex(c1=g["c1"], c2=g["c2"], offsets=g["offsets"], ids=g["ids"], codes=g["codes"], books=g["books"],
                      tables=tables, rotation=g["rotation"])
    hix = DeviceIndex(c1=g["c1"], c2=g["c2"], offsets=g["hoffsets"], ids=g["hids"], codes=g["hcodes"],
                      bank1=g["bank1"], bank2=g["bank2"], rotation=g["rotation"], rot1=g["rot1"], rot2=g["rot2"])
    q = g["queries"].astype(np.float32)
    for eng, ix in (("fbpq", dix), ("baseline", dix), ("hbpq", hix)):
        d, i, c = ix.search(q, 2000, 50, eng).numpy()
        want_c = (g[f"{eng}_ids"] != 0xFFFFFFFF).sum(1)
        check_topk(d, i, c, g[f"{eng}_d"], g[f"{eng}_ids"], want_c, _qn(q),
                   **_ctx(_orc_index(g, hbpq=eng == "hbpq", rotated=True), q, 2000))
    x = g["enc_x"].astype(np.float32)
    from oracle.parity import classify_encoding

    def packed(ix):
        return (ix.offsets.cpu().numpy().view(np.uint32).astype(np.int64), ix.ids.cpu().numpy().view(np.uint32),
                ix.codes.cpu().numpy())

    e = encode.build_index(x, g["c1"], g["c2"], g["books"], rotation=g["rotation"])
    s = classify_encoding(x, g["c1"], g["c2"], g["books"], packed(e), (g["enc_offsets"], g["enc_ids"], g["enc_codes"]),
                          rotation=g["rotation"])
    assert s["unclassified"] == 0, s
    h = encode.build_hbpq_index(x, g["c1"], g["c2"], g["bank1"], g["bank2"], rotation=g["rotation"], rot1=g["rot1"],
                                rot2=g["rot2"])
    s = classify_encoding(x, g["c1"], g["c2"], None, packed(h), (g["enc_offsets"], g["enc_ids"], g["enc_hcodes"]),
                          rotation=g["rotation"], bank1=g["bank1"], bank2=g["bank2"], rot1=g["rot1"], rot2=g["rot2"])
    assert s["unclassified"] == 0, s


def test_sharded_searcher_nccl_single_rank(c0, c0_index):
    """ShardedSearcher over a real NCCL group (world 1, exchange forced):
    local search -> all_gather_into_tensor -> device merge == local result."""
    import os

    import torch
    import torch.distributed as dist

    from paper_1404_1831_b200 import sharded

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29547")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        q = c0["queries"][:64].astype(np.float32)
        got = sharded.ShardedSearcher(c0_index, force_collective=True).search(q, 10_000, 100).numpy()
        want = c0_index.search(q, 10_000, 100).numpy()
        for x, y in zip(got, want):
            np.testing.assert_array_equal(x, y)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seed", range(20))
def test_fuzz_small_configs_vs_oracle(torch_cuda, oracle, seed):
    """Randomised small indexes: T, M (incl. the generic runtime-M path),
    K, quantised data (distance and key ties), empty cells, L from 1 to
    beyond N, k beyond the candidates; dense and sparse traversal; every
    engine.  Contract of SURVEY §8c(ii) against the oracle."""
    from paper_1404_1831_b200 import DeviceIndex

    rng = np.random.default_rng(1000 + seed)
    t = int(rng.integers(2, 40)) if seed % 5 else int(rng.integers(1030, 1400))  # >1024: partial sort
    m = int(rng.choice([2, 4, 6, 8]))
    dim = m * int(rng.integers(1, 5)) * 2
    kk = int(rng.integers(2, 64))
    n = int(rng.integers(50, 4000))
    quant = seed % 2 == 0
    base = rng.normal(size=(n, dim)).astype(np.float32)
    if quant:
        base = np.round(base * 2) / 2
    c1 = base[rng.choice(n, t, replace=t > n), : dim // 2].copy()
    c2 = base[rng.choice(n, t, replace=t > n), dim // 2 :].copy()
    books = (0.3 * rng.normal(size=(m, kk, dim // m))).astype(np.float32)
    if quant:
        books = np.round(books * 4) / 4
    off, ids, codes = oracle.build_index(base, c1, c2, books, id_offset=int(rng.integers(0, 1000)))
    bank1 = (0.3 * rng.normal(size=(t, m // 2, kk, dim // m))).astype(np.float32)
    bank2 = (0.3 * rng.normal(size=(t, m // 2, kk, dim // m))).astype(np.float32)
    idx = oracle.Index(c1, c2, off, ids, codes, books=books)
    hidx = oracle.Index(c1, c2, off, ids, codes, bank1=bank1, bank2=bank2)
    q = rng.normal(size=(24, dim)).astype(np.float32)
    if quant:
        q = np.round(q * 2) / 2
    for lists in (False, True):
        dix = DeviceIndex(c1=c1, c2=c2, offsets=off, ids=ids, codes=codes, books=books, tables=idx.tables,
                          cell_lists=lists)
        hix = DeviceIndex(c1=c1, c2=c2, offsets=off, ids=ids, codes=codes, bank1=bank1, bank2=bank2,
                          cell_lists=lists)
        Ls = (1, int(rng.integers(2, n)), n, 3 * n) if t <= 1024 else (1, int(rng.integers(2, n // 4)))
        for L in Ls:
            k = int(rng.integers(1, 200))
            for eng, di, oi in (("fbpq", dix, idx), ("baseline", dix, idx), ("hbpq", hix, hidx)):
                wd, wi, wc, _ = oracle.search_batch_numpy(oi, eng, q, L, k)
                d, i, c = di.search(q, L, k, eng).numpy()
                check_topk(d, i, c, wd, wi, wc, _qn(q), **_ctx(oi, q, L))


@pytest.mark.parametrize("t,kind", [(64, "integer"), (4096, "integer"), (4096, "float"), (300, "float")])
def test_first_layer_tensor_cores_vs_f64(torch_cuda, t, kind, monkeypatch):
    """The tcgen05 first layer (exact bf16 limb products, f32 accumulation in
    TMEM) against f64 dot products, beside the FFMA kernel: both within
    2^-20 of sum |q_u c_u| (a few f32 accumulation roundings).  Covers one
    padded tile (T=64), T not a multiple of the 128-codeword tile, nq not a
    multiple of the 128-query tile, and integer (1-limb) vs float (3-limb)
    queries."""
    from paper_1404_1831_b200 import DeviceIndex

    rng = np.random.default_rng(t)
    dim, m, kk, nq = 128, 8, 16, 300
    c1 = (rng.normal(size=(t, 64)) * 40 + 100).astype(np.float32)
    c2 = (rng.normal(size=(t, 64)) * 40 + 100).astype(np.float32)
    books = rng.normal(size=(m, kk, dim // m)).astype(np.float32)
    off = np.zeros(t * t + 1, np.int64)
    args = dict(c1=c1, c2=c2, offsets=off, ids=np.zeros(0, np.uint32), codes=np.zeros((0, m), np.uint8), books=books)
    if kind == "integer":
        q = np.clip(np.round(rng.normal(size=(nq, dim)) * 40 + 100), 0, 255).astype(np.float32)
    else:
        q = (rng.normal(size=(nq, dim)) * 40 + 100).astype(np.float32)
    tc = DeviceIndex(**args)
    monkeypatch.setenv("BPQ_FIRST_LAYER", "ffma")
    ff = DeviceIndex(**args)
    for h, c in ((0, c1), (1, c2)):
        qh = q[:, h * 64:(h + 1) * 64].astype(np.float64)
        exact = qh @ c.astype(np.float64).T
        bound = 2.0 ** -20 * (np.abs(qh) @ np.abs(c.astype(np.float64)).T)
        got_tc = tc.coarse_dots(q)[h].cpu().numpy()
        got_ff = ff.coarse_dots(q)[h].cpu().numpy()
        for name, got in (("tensor cores", got_tc), ("ffma", got_ff)):
            err = np.abs(got.astype(np.float64) - exact)
            assert np.all(err <= bound), f"{name} half {h}: max err/bound {np.max(err / bound):.3f}"


@pytest.mark.parametrize("nc,kind", [(300, "integer"), (4096, "integer"), (256, "float")])
def test_nearest_centroids_tensor_cores_vs_f64(torch_cuda, nc, kind):
    """The tcgen05 encoder (d = 64, argmin fused into the TMEM epilogue)
    against an f64 argmin of nearest_centroids' score |c|^2 - 2 x.c
    (quantizer.py:109-130): the chosen centroid is the true minimum or
    within 1e-6 of its magnitude (an argmin near-tie of the f32 scores), and
    d2 agrees within 1e-4 relative (floor 1e-3)."""
    import torch

    from paper_1404_1831_b200 import encode

    rng = np.random.default_rng(nc)
    n = 1000
    cents = (rng.normal(size=(nc, 64)) * 30 + 100).astype(np.float32)
    if kind == "integer":
        x = np.clip(np.round(rng.normal(size=(n, 64)) * 40 + 100), 0, 255).astype(np.float32)
    else:
        x = (rng.normal(size=(n, 64)) * 40 + 100).astype(np.float32)
    ids, d2 = encode.nearest_centroids(torch.from_numpy(x).cuda(), cents)
    ids, d2 = ids.cpu().numpy(), d2.cpu().numpy()
    c64 = cents.astype(np.float64)
    score = (c64 * c64).sum(1)[None] - 2 * x.astype(np.float64) @ c64.T
    best = score.min(1)
    got = score[np.arange(n), ids]
    scale = np.abs(score).max(1)
    assert np.all(got - best <= 1e-6 * scale), np.max((got - best) / scale)
    want_d2 = np.maximum(best + (x.astype(np.float64) ** 2).sum(1), 0)
    assert np.all(np.abs(d2 - want_d2) <= 1e-4 * np.maximum(want_d2, 1e-3) + 1e-6 * scale)


@pytest.mark.parametrize("L", [1000, 30_000, 36_000])
def test_tie_plateau_every_key_ties(torch_cuda, oracle, L):
    """Every cell has the same key: 192 coarse codewords per half at +-10 e_u
    and the query at the origin give r = 100 for all of them, and one point
    per cell fills all 36,864 cells.  The reference heap then pops cells in
    (oi, oj) order (numba_backend.py:28-144), which the band traversal must
    reproduce through the plateau windows (more populated cells than one
    band holds).  L = 36,000 needs two windows."""
    from paper_1404_1831_b200 import DeviceIndex

    rng = np.random.default_rng(5)
    dh, t, m, kk = 96, 192, 8, 16
    cb = np.zeros((t, dh), np.float32)
    for i in range(t):
        cb[i, i // 2] = 10.0 if i % 2 == 0 else -10.0
    ii, jj = np.meshgrid(np.arange(t), np.arange(t), indexing="ij")
    base = np.concatenate([cb[ii.ravel()], cb[jj.ravel()]], 1)
    base += rng.normal(scale=0.01, size=base.shape).astype(np.float32)
    books = (0.01 * rng.normal(size=(m, kk, 2 * dh // m))).astype(np.float32)
    off, ids, codes = oracle.build_index(base, cb, cb, books)
    assert np.all(np.diff(off) == 1)
    idx = oracle.Index(cb, cb, off, ids, codes, books=books)
    # exact mode: candidate distances bit-identical to the oracle, so equal-distance ties break the same way
    dix = DeviceIndex(c1=cb, c2=cb, offsets=off, ids=ids, codes=codes, books=books, tables=idx.tables, exact=True)
    q = np.zeros((2, 2 * dh), np.float32)
    for eng in ("fbpq", "baseline"):
        wd, wi, wc, _ = oracle.search_batch_numpy(idx, eng, q, L, 50)
        d, i, c = dix.search(q, L, 50, eng).numpy()
        assert (c >= 0).all(), "tie plateau reported as failure"
        # every key ties, so the boundary near-tie rule would excuse any candidate set: demand the
        # reference's exact set (the first L cells in (oi, oj) order)
        np.testing.assert_array_equal(c, wc)
        for x in range(q.shape[0]):
            assert set(i[x, : c[x]].view(np.uint32).tolist()) == set(wi[x, : wc[x]].tolist())
        check_topk(d, i, c, wd, wi, wc, _qn(q))


def test_query_split_sharding_equals_single(c0, torch_cuda):
    """Query-split sharding (sharded.SplitSearcher's steps, the 3 ranks run in
    turn on one GPU): each shard traverses one third of the queries against
    the global counts and records the visited cells; the concatenated lists
    (what the all-gather delivers) are streamed by every shard over its local
    entries; the merged lists equal the single-index answer up to the §8c(ii)
    contract (point-term sums follow the entry's position in its own shard),
    with identical counts."""
    import torch

    from paper_1404_1831_b200 import DeviceIndex, sharded

    q = c0["queries"][:120].astype(np.float32)
    L, k = 10_000, 100
    tables = (c0["cn1"], c0["cn2"], c0["fine_norms"], c0["cross1"], c0["cross2"])
    full = DeviceIndex(c1=c0["c1"], c2=c0["c2"], offsets=c0["offsets"], ids=c0["ids"], codes=c0["codes"],
                       books=c0["books"], tables=tables)
    want = full.search(q, L, k, "fbpq").numpy()
    parts = sharded.split_index_arrays(c0["offsets"], c0["ids"], c0["codes"], 3)
    searchers = [sharded.SplitSearcher(DeviceIndex(c1=c0["c1"], c2=c0["c2"], offsets=s["offsets"], ids=s["ids"],
                                                   codes=s["codes"], books=c0["books"], tables=tables,
                                                   global_offsets=c0["offsets"],
                                                   num_entries_global=int(c0["offsets"][-1])))
                 for s in parts]
    qt = torch.from_numpy(q).cuda()
    counts, packed = [], []
    for r, sr in enumerate(searchers):
        lo, hi = sharded.query_slice(q.shape[0], 3, r)
        c, v, _ = sr.traverse(qt[lo:hi], L)
        counts.append(c)
        packed.append(sharded.pack_visits(c, v))
    allc = torch.cat(counts).to(torch.int64)
    start = torch.zeros(allc.numel() + 1, dtype=torch.int64, device=allc.device)
    torch.cumsum(allc, 0, out=start[1:])
    allp = torch.cat(packed)
    local = [sr.scan(qt, k, allp, start) for sr in searchers]
    merged = sharded.merge_results([o.dists for o in local], [o.ids for o in local], [o.counts for o in local], k)
    got = merged.numpy()
    np.testing.assert_array_equal(got[2], want[2])
    check_topk(got[0], got[1], got[2], want[0], want[1], want[2], _qn(q))


def test_split_searcher_nccl_single_rank(c0):
    """SplitSearcher end to end through an NCCL group of one (the visit
    exchange and the final merge both run)."""
    import os

    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist

    from paper_1404_1831_b200 import DeviceIndex, sharded

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29611")
    fresh = not dist.is_initialized()
    if fresh:
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        tables = (c0["cn1"], c0["cn2"], c0["fine_norms"], c0["cross1"], c0["cross2"])
        dix = DeviceIndex(c1=c0["c1"], c2=c0["c2"], offsets=c0["offsets"], ids=c0["ids"], codes=c0["codes"],
                          books=c0["books"], tables=tables)
        q = c0["queries"][:64].astype(np.float32)
        want = dix.search(q, 10_000, 100, "fbpq").numpy()
        got = sharded.SplitSearcher(dix, force_collective=True).search(torch.from_numpy(q), 10_000, 100).numpy()
        np.testing.assert_array_equal(got[2], want[2])
        np.testing.assert_array_equal(got[1], want[1])
        np.testing.assert_array_equal(got[0], want[0])
    finally:
        if fresh:
            dist.destroy_process_group()
