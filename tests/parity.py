"""The parity contract of SURVEY.md §8c(ii), written once for every test.

Per query, the engine's top-k list must equal the oracle's except at
positions whose oracle distances are near-tied (within ``rtol`` relative of
the engine's value at that rank): a near-tie at the budget boundary or in
the distance ordering may swap which id lands at that rank.  Every distance
must be within ``rtol`` (1e-4, north_star) with the floor 1e-6*|q|^2 of
test_fbpq.py:124-127, and counts must match.
"""

import numpy as np

RTOL = 1e-4


def check_topk(got_d, got_i, got_c, want_d, want_i, want_c, qnorm2=None, rtol=RTOL,
               min_exact_frac=0.98):
    got_d = np.asarray(got_d)
    want_d = np.asarray(want_d)
    got_i = np.asarray(got_i).view(np.uint32) if np.asarray(got_i).dtype == np.int32 else np.asarray(got_i)
    want_i = np.asarray(want_i)
    nq = got_d.shape[0]
    exact = 0
    bad = []
    for q in range(nq):
        n = int(want_c[q])
        if int(got_c[q]) != n:
            bad.append((q, "count", int(got_c[q]), n))
            continue
        gd, wd = got_d[q, :n].astype(np.float64), want_d[q, :n].astype(np.float64)
        floor = 1e-6 * (qnorm2[q] if qnorm2 is not None else 0.0)
        tol = rtol * np.abs(wd) + floor
        if np.any(np.abs(gd - wd) > tol):
            x = int(np.argmax(np.abs(gd - wd) - tol))
            bad.append((q, "dist", x, gd[x], wd[x]))
            continue
        if np.array_equal(got_i[q, :n], want_i[q, :n]):
            exact += 1
        elif n:
            # away from the k-th distance the id SETS must agree exactly
            thr = wd[n - 1] * (1.0 - 2.0 * rtol) - floor
            gs = set(got_i[q, :n][gd < thr].tolist())
            ws = set(want_i[q, :n][wd < thr].tolist())
            if gs != ws:
                bad.append((q, "set", sorted(gs ^ ws)[:5]))
        # id mismatches are tolerated only where the rank's distance is a near-tie,
        # which the elementwise distance check above already bounds.
    assert not bad, f"{len(bad)} queries violate the contract, first: {bad[:5]}"
    assert exact >= min_exact_frac * nq, f"only {exact}/{nq} id lists identical"
    return exact
