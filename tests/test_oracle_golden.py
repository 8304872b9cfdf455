"""Pin the CPU oracle against outputs of the reference itself
(tests/golden/make_golden.py ran /root/reference's bilayerpq)."""

import numpy as np
import pytest


def _traverse_case(kat, n):
    p = f"tr{n}_"
    return [kat[p + s] for s in ("sr1", "sr2", "o1", "o2", "off")], int(kat[p + "budget"]), [
        kat[p + s] for s in ("vi", "vj", "st", "en")
    ]


def test_traverse_known_answers(kat, oracle):
    for n in range(int(kat["n_traverse"])):
        args, budget, want = _traverse_case(kat, n)
        got = oracle.traverse_cells(*args, budget)
        for g, w in zip(got, want):
            np.testing.assert_array_equal(g, w, err_msg=f"case {n}")


def test_select_top_known_answers(kat, oracle):
    for n in range(int(kat["n_select"])):
        p = f"sel{n}_"
        oi, od = oracle.select_top(kat[p + "ids"], kat[p + "d"], int(kat[p + "r"]))
        np.testing.assert_array_equal(oi, kat[p + "oi"])
        np.testing.assert_array_equal(od, kat[p + "od"])


def _c0_index(c0, oracle):
    tables = (c0["cn1"], c0["cn2"], c0["fine_norms"], c0["cross1"], c0["cross2"])
    return oracle.Index(c0["c1"], c0["c2"], c0["offsets"], c0["ids"], c0["codes"], books=c0["books"], tables=tables)


def test_tables_restatement_matches_reference(c0, oracle):
    cn1, cn2, fn, x1, x2 = oracle.build_tables_from(c0["c1"], c0["c2"], c0["books"])
    for a, b in ((cn1, "cn1"), (cn2, "cn2"), (fn, "fine_norms"), (x1, "cross1"), (x2, "cross2")):
        np.testing.assert_array_equal(a, c0[b])


def test_stage_captures_bit_exact(c0, oracle):
    """prepare_query (numpy, same BLAS), traverse and both scans reproduce the
    reference stage by stage, bit for bit."""
    for x in range(6):
        p = f"stage{x}_"
        q = c0["queries"][x].astype(np.float32)
        q_norm, d1, d2, fold, r1, r2 = oracle.prepare_query(c0["c1"], c0["c2"], c0["books"], c0["fine_norms"], q)
        np.testing.assert_array_equal(r1, c0[p + "r1"])
        np.testing.assert_array_equal(r2, c0[p + "r2"])
        np.testing.assert_array_equal(fold, c0[p + "fold"])
        assert np.float32(q_norm) == c0[p + "q_norm"]
        vis = oracle.traverse(c0["offsets"], r1, r2, 10_000)
        for g, w in zip(vis, ("vi", "vj", "st", "en")):
            np.testing.assert_array_equal(g, c0[p + w])
        ti, td = oracle.scan_tables(*vis, c0["ids"], c0["codes"], q_norm, d1, d2, c0["cn1"], c0["cn2"], fold, c0["cross1"], c0["cross2"])
        np.testing.assert_array_equal(ti, c0[p + "tab_ids"])
        np.testing.assert_array_equal(td, c0[p + "tab_d"])
        dh = c0["c1"].shape[1]
        gi, gd = oracle.scan_global(*vis, c0["ids"], c0["codes"], q[None, :dh] - c0["c1"], q[None, dh:] - c0["c2"], c0["books"])
        np.testing.assert_array_equal(gd, c0[p + "glob_d"])


@pytest.mark.parametrize("engine,nq,L,k", [("fbpq", 60, 10_000, 100), ("baseline", 20, 10_000, 100), ("fbpq", 60, 1_000, 10)])
def test_search_matches_reference(c0, oracle, engine, nq, L, k):
    idx = _c0_index(c0, oracle)
    q = c0["queries"][:nq].astype(np.float32)
    d, i, cnt, _ = oracle.search_batch_numpy(idx, engine, q, L, k)
    tag = f"{engine}_L{L}_k{k}"
    np.testing.assert_array_equal(i, c0[tag + "_ids"][:nq])
    np.testing.assert_array_equal(d, c0[tag + "_d"][:nq])


def test_hbpq_matches_reference(hbpq_rig, oracle):
    g = hbpq_rig
    idx = oracle.Index(g["c1"], g["c2"], g["offsets"], g["ids"], g["hcodes"], bank1=g["bank1"], bank2=g["bank2"])
    q = g["queries"][:30].astype(np.float32)
    d, i, cnt, _ = oracle.search_batch_numpy(idx, "hbpq", q, 2000, 50)
    np.testing.assert_array_equal(i, g["hbpq_ids"][:30])
    np.testing.assert_array_equal(d, g["hbpq_d"][:30])
    ci, cd = oracle.scan_query(idx, "hbpq", g["queries"][0].astype(np.float32), 2000)
    np.testing.assert_array_equal(ci, g["stage_local_ids"])
    np.testing.assert_array_equal(cd, g["stage_local_d"])


def test_encoding_matches_reference(c0, oracle):
    x = c0["enc_x"].astype(np.float32)
    ci, _ = oracle.nearest_centroids(np.ascontiguousarray(x[:, :64]), c0["c1"])
    np.testing.assert_array_equal(ci, c0["enc_i"])
    off, ids, codes = oracle.build_index(x, c0["c1"], c0["c2"], c0["books"], id_offset=77)
    np.testing.assert_array_equal(off, c0["enc_offsets"])
    np.testing.assert_array_equal(ids, c0["enc_ids"])
    np.testing.assert_array_equal(codes, c0["enc_codes"])


def test_c_batch_search_within_contract(c0, oracle):
    """The all-C CPU baseline (sequential f32 coarse dots instead of OpenBLAS)
    agrees with the reference up to near-ties."""
    idx = _c0_index(c0, oracle)
    q = c0["queries"][:50].astype(np.float32)
    q = c0["queries"][:200].astype(np.float32)
    d, i, cnt, nc = oracle.search_batch_c(idx, "fbpq", q, 10_000, 100, threads=4)
    from oracle.parity import check

    want_c = np.minimum(100, c0["fbpq_L10000_k100_ncand"][:200])
    qn = np.einsum("ij,ij->i", q.astype(np.float64), q.astype(np.float64))
    s = check(d, i, cnt, c0["fbpq_L10000_k100_d"][:200], c0["fbpq_L10000_k100_ids"][:200], want_c, qn,
              got_ncand=nc, want_ncand=c0["fbpq_L10000_k100_ncand"][:200], orc=oracle, index=idx, queries=q,
              L=10_000)
    assert s["exact_lists"] > 0


def test_parity_classifier_rejects_real_mismatches(c0, oracle):
    """The §8c(ii) classifier: a far-away id swapped in, a wrong distance or
    a count change without a boundary near-tie are all unclassified."""
    from oracle.parity import classify

    idx = _c0_index(c0, oracle)
    q = c0["queries"][:20].astype(np.float32)
    wd = c0["fbpq_L10000_k100_d"][:20].copy()
    wi = c0["fbpq_L10000_k100_ids"][:20].copy()
    wc = np.minimum(100, c0["fbpq_L10000_k100_ncand"][:20])
    ctx = dict(orc=oracle, index=idx, queries=q, L=10_000)
    assert classify(wd, wi, wc, wd, wi, wc, **ctx)["exact_lists"] == 20
    gi = wi.copy()
    gi[0, 3] = wi[1, 50] if wi[1, 50] not in wi[0] else wi[1, 60]  # an id from another query, mid-list
    assert classify(wd, gi, wc, wd, wi, wc, **ctx)["unclassified"] == 1
    gd = wd.copy()
    gd[2, 10] *= 1.01
    assert classify(gd, wi, wc, wd, wi, wc, **ctx)["unclassified"] == 1
    gc = wc.copy()
    gc[4] -= 1
    s = classify(wd, wi, gc, wd, wi, wc, **ctx)
    assert s["count_mismatch"] == 1


def test_rotated_variants_match_reference(oracle):
    """OPQ-rotated coarse pair and per-half bank rotations (the paper's
    optimized engines) reproduce the reference bit for bit."""
    from conftest import GOLDEN

    g = dict(np.load(GOLDEN / "rot.npz"))
    tables = (g["cn1"], g["cn2"], g["fine_norms"], g["cross1"], g["cross2"])
    idx = oracle.Index(g["c1"], g["c2"], g["offsets"], g["ids"], g["codes"], books=g["books"], tables=tables,
                       rotation=g["rotation"])
    hidx = oracle.Index(g["c1"], g["c2"], g["hoffsets"], g["hids"], g["hcodes"], bank1=g["bank1"], bank2=g["bank2"],
                        rotation=g["rotation"], rot1=g["rot1"], rot2=g["rot2"])
    q = g["queries"].astype(np.float32)
    for eng, ix in (("fbpq", idx), ("baseline", idx), ("hbpq", hidx)):
        d, i, c, _ = oracle.search_batch_numpy(ix, eng, q, 2000, 50)
        np.testing.assert_array_equal(i, g[f"{eng}_ids"])
        np.testing.assert_array_equal(d, g[f"{eng}_d"])
