"""Parity contract of SURVEY.md §8c(ii) with mismatch classification --
TEST INFRASTRUCTURE ONLY (imported by tests/ and bench.py's parity leg).

Per query the engine's answer is compared with the oracle's:

* every distance the two lists share (same id) must agree within
  ``rtol`` = 1e-4 relative (north_star), with the floor 1e-6*|q|^2 of the
  reference's own check (test_fbpq.py:124-127);
* an identical id list is "exact";
* otherwise each id in the symmetric difference of the two top-k sets, and
  each position where the orders differ, must be explained by one of
  - a *distance near-tie*: the id's distance is within ``rtol`` of the
    oracle's k-th distance (which id lands at rank k is then a rounding
    decision), or two swapped positions hold distances within ``rtol``;
  - a *boundary near-tie*: the id lives in a cell whose oracle key
    f64(r1[i]) + f64(r2[j]) is within ``key_rtol`` = 1e-5 relative of the
    oracle's cutoff-cell key (the multi-sequence may then visit that cell or
    not, changing the candidate set -- the first-layer dot products of
    OpenBLAS and of the GPU differ by ulps);
* a count / candidate-count mismatch must be a boundary near-tie: some
  other non-empty cell's oracle key lies within ``key_rtol`` of the cutoff
  key.

Anything else is "unclassified" and fails the contract.  The oracle's keys
come from ``oracle.coarse_scan`` (the reference's numpy calls,
multi_index.py:270-293) and its cutoff cell from ``oracle.traverse``
(numba_backend.py:11-146 restated).
"""

from __future__ import annotations

import numpy as np

RTOL = 1e-4
KEY_RTOL = 1e-5


class _Boundary:
    """Oracle-side cutoff information for one query (computed lazily, only
    for queries whose answers differ)."""

    def __init__(self, orc, index, q, L):
        _, _, _, r1, r2 = orc.coarse_scan(index.c1, index.c2, q, getattr(index, "rotation", None))
        self.r1 = r1.astype(np.float64)
        self.r2 = r2.astype(np.float64)
        self.t = index.t
        self.offsets = index.offsets
        vi, vj, _, _ = orc.traverse(index.offsets, r1, r2, L)
        if vi.shape[0]:
            self.cut = (int(vi[-1]), int(vj[-1]))
            self.kappa = self.r1[self.cut[0]] + self.r2[self.cut[1]]
        else:
            self.cut, self.kappa = None, None
        self._other = None

    def near(self, key):
        return self.kappa is not None and abs(key - self.kappa) <= KEY_RTOL * max(abs(self.kappa), 1e-30)

    def cell_near(self, i, j):
        return self.near(self.r1[i] + self.r2[j])

    def other_near_cell(self):
        """Is there a non-empty cell other than the cutoff cell whose key is
        within KEY_RTOL of the cutoff key?"""
        if self._other is None:
            self._other = False
            if self.kappa is not None:
                lo_k = self.kappa - KEY_RTOL * abs(self.kappa)
                hi_k = self.kappa + KEY_RTOL * abs(self.kappa)
                o2 = np.argsort(self.r2, kind="stable")
                s2 = self.r2[o2]
                lo = np.searchsorted(s2, lo_k - self.r1, "left")
                hi = np.searchsorted(s2, hi_k - self.r1, "right")
                for i in np.nonzero(hi > lo)[0]:
                    for j in o2[lo[i]:hi[i]]:
                        if (int(i), int(j)) == self.cut:
                            continue
                        lin = int(i) * self.t + int(j)
                        if self.offsets[lin + 1] > self.offsets[lin]:
                            self._other = True
                            return True
        return self._other


class _CellOfId:
    def __init__(self, index):
        ids = np.asarray(index.ids, np.uint32)
        self.pos = {}
        self.ids = ids
        self.offsets = np.asarray(index.offsets, np.int64)
        self.t = index.t
        self._inv = None

    def __call__(self, x):
        if self._inv is None:
            order = np.argsort(self.ids, kind="stable")
            self._inv = (self.ids[order], order)
        sid, order = self._inv
        k = np.searchsorted(sid, np.uint32(x))
        if k >= sid.shape[0] or sid[k] != x:
            return None
        cell = int(np.searchsorted(self.offsets, order[k], "right")) - 1
        return cell // self.t, cell % self.t


def classify(got_d, got_i, got_c, want_d, want_i, want_c, qnorm2=None, *, got_ncand=None, want_ncand=None,
             orc=None, index=None, queries=None, L=None, rtol=RTOL, max_examples=8):
    """Classify every query; returns a summary dict (see module doc)."""
    got_d = np.asarray(got_d, np.float64)
    want_d = np.asarray(want_d, np.float64)
    gi = np.asarray(got_i)
    got_i = gi.view(np.uint32) if gi.dtype == np.int32 else gi.astype(np.uint32)
    want_i = np.asarray(want_i).astype(np.uint32)
    nq = got_d.shape[0]
    can_boundary = orc is not None and index is not None and queries is not None and L is not None
    cell_of = _CellOfId(index) if can_boundary else None
    out = dict(queries=nq, exact_lists=0, near_tie_distance=0, near_tie_boundary=0, count_mismatch=0,
               ncand_mismatch=0, unclassified=0, max_rel_dist_err=0.0, examples=[])

    def fail(q, why):
        out["unclassified"] += 1
        if len(out["examples"]) < max_examples:
            out["examples"].append({"query": int(q), "why": why})

    for q in range(nq):
        bnd = None

        def boundary():
            nonlocal bnd
            if bnd is None and can_boundary:
                bnd = _Boundary(orc, index, np.asarray(queries[q], np.float32), int(L))
            return bnd

        floor = 1e-6 * (float(qnorm2[q]) if qnorm2 is not None else 0.0)
        gc, wc = int(got_c[q]), int(want_c[q])
        boundary_needed = False
        if gc != wc:
            out["count_mismatch"] += 1
            boundary_needed = True
        if got_ncand is not None and want_ncand is not None and int(got_ncand[q]) != int(want_ncand[q]):
            out["ncand_mismatch"] += 1
            boundary_needed = True
        if boundary_needed:
            b = boundary()
            if b is None or not b.other_near_cell():
                fail(q, f"count {gc}/{wc} or ncand differs without a boundary key near-tie")
                continue
        n = min(gc, wc)
        gl, wl = got_i[q, :gc], want_i[q, :wc]
        gdq, wdq = got_d[q, :gc], want_d[q, :wc]
        # distances of the shared ids
        wpos = {int(x): r for r, x in enumerate(wl)}
        shared = [(r, wpos[int(x)]) for r, x in enumerate(gl) if int(x) in wpos]
        bad_d = None
        for rg, rw in shared:
            err = abs(gdq[rg] - wdq[rw])
            rel = err / max(abs(wdq[rw]), 1e-30)
            out["max_rel_dist_err"] = max(out["max_rel_dist_err"], float(rel))
            if err > rtol * abs(wdq[rw]) + floor:
                bad_d = (rg, gdq[rg], wdq[rw])
        if bad_d is not None:
            fail(q, f"distance of a shared id off by more than rtol: rank {bad_d[0]} {bad_d[1]} vs {bad_d[2]}")
            continue
        if gc == wc and np.array_equal(gl, wl):
            if boundary_needed:
                out["near_tie_boundary"] += 1
            else:
                out["exact_lists"] += 1
            continue
        kth = wdq[wc - 1] if wc else np.inf
        kind = "distance"
        ok = True
        # ids present on one side only
        for side_ids, side_d in ((gl, gdq), (wl, wdq)):
            other = set((wl if side_ids is gl else gl).tolist())
            for r, x in enumerate(side_ids):
                if int(x) in other:
                    continue
                if side_d[r] >= kth * (1.0 - rtol) - floor:
                    continue  # near-tie at the k-th distance
                b = boundary()
                cell = cell_of(int(x)) if b is not None else None
                if cell is not None and b.cell_near(*cell):
                    kind = "boundary"
                    continue
                ok = False
                why = f"id {int(x)} at rank {r} (d={side_d[r]:.6g}, k-th {kth:.6g}) is not a near-tie"
                break
            if not ok:
                break
        if ok:
            # order differences among shared ids: swapped ranks must hold near-equal distances
            for rg, rw in shared:
                if rg != rw and rw < n and rg < n:
                    if abs(wdq[rw] - wdq[min(rg, wc - 1)]) > rtol * abs(wdq[rw]) + floor and kind == "distance":
                        ok = False
                        why = f"rank {rg} vs {rw} swapped without a distance near-tie"
                        break
        if not ok:
            fail(q, why)
            continue
        if boundary_needed or kind == "boundary":
            out["near_tie_boundary"] += 1
        else:
            out["near_tie_distance"] += 1
    out["exact_frac"] = out["exact_lists"] / max(nq, 1)
    return out


def check(got_d, got_i, got_c, want_d, want_i, want_c, qnorm2=None, **kw):
    """Assert the contract (no unclassified query); returns the summary."""
    s = classify(got_d, got_i, got_c, want_d, want_i, want_c, qnorm2, **kw)
    assert s["unclassified"] == 0, f"{s['unclassified']} of {s['queries']} queries violate §8c(ii): {s['examples']}"
    return s


# ---------------------------------------------------------------- encoding
def _per_row(offsets, ids, codes, n, id_offset):
    """Unpack a cell-grouped index into per-row (cell, code) by point id."""
    offsets = np.asarray(offsets, np.int64)
    ids = np.asarray(ids).astype(np.int64) - id_offset
    cell = np.repeat(np.arange(offsets.shape[0] - 1), np.diff(offsets))
    row_cell = np.full(n, -1, np.int64)
    row_code = np.zeros((n, codes.shape[1]), np.uint8)
    row_cell[ids] = cell
    row_code[ids] = codes
    return row_cell, row_code


def classify_encoding(x, c1, c2, books, got, want, id_offset=0, rel=1e-5, rotation=None, bank1=None, bank2=None,
                      rot1=None, rot2=None):
    """Compare two encodings of the same rows (each ``(offsets, ids, codes)``,
    cell-grouped as build_index packs them, multi_index.py:210-230).  A row
    may differ only through an argmin near-tie (quantizer.py:109-130): the
    exact (f64) squared distances to the two chosen codewords differ by at
    most ``rel`` x (|x|^2 + |c|^2), the scale at which the f32 score
    cn - 2 x.c rounds.  Returns a summary; ``unclassified`` must be 0."""
    x = np.asarray(x, np.float32)
    if rotation is not None:
        x = x @ np.asarray(rotation, np.float32)
    n, dim = x.shape
    c1 = np.asarray(c1, np.float32)
    c2 = np.asarray(c2, np.float32)
    t, dh = c1.shape
    gcell, gcode = _per_row(*got, n, id_offset)
    wcell, wcode = _per_row(*want, n, id_offset)
    out = dict(rows=n, identical=0, near_tie_cell=0, near_tie_code=0, unclassified=0, examples=[])

    def tie(v, a, b):
        da = float(np.sum((v.astype(np.float64) - a.astype(np.float64)) ** 2))
        db = float(np.sum((v.astype(np.float64) - b.astype(np.float64)) ** 2))
        scale = float(np.sum(v.astype(np.float64) ** 2) + max(np.sum(a.astype(np.float64) ** 2),
                                                             np.sum(b.astype(np.float64) ** 2)))
        return abs(da - db) <= rel * max(scale, 1e-30)

    m = gcode.shape[1]
    for r in np.nonzero((gcell != wcell) | np.any(gcode != wcode, axis=1))[0]:
        gi, gj = divmod(int(gcell[r]), t)
        wi, wj = divmod(int(wcell[r]), t)
        ok = True
        if gcell[r] != wcell[r]:
            ok = (gi == wi or tie(x[r, :dh], c1[gi], c1[wi])) and (gj == wj or tie(x[r, dh:], c2[gj], c2[wj]))
            kind = "near_tie_cell"
        else:
            kind = "near_tie_code"
            e1, e2 = x[r, :dh] - c1[gi], x[r, dh:] - c2[gj]
            if rot1 is not None:  # per-half bank rotations (hbpq.py:168-187)
                e1 = e1 @ np.asarray(rot1, np.float32)
            if rot2 is not None:
                e2 = e2 @ np.asarray(rot2, np.float32)
            disp = np.concatenate([e1, e2])
            ds = dim // m
            for p in range(m):
                if gcode[r, p] == wcode[r, p]:
                    continue
                if bank1 is not None:
                    bk = (bank1[gi, p] if p < m // 2 else bank2[gj, p - m // 2])
                else:
                    bk = books[p]
                if not tie(disp[p * ds:(p + 1) * ds], bk[gcode[r, p]], bk[wcode[r, p]]):
                    ok = False
        if ok:
            out[kind] += 1
        else:
            out["unclassified"] += 1
            if len(out["examples"]) < 8:
                out["examples"].append(int(r))
    out["identical"] = n - out["near_tie_cell"] - out["near_tie_code"] - out["unclassified"]
    return out
