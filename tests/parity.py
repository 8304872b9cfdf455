"""The parity contract of SURVEY.md §8c(ii), written once for every test.

Thin wrapper over ``oracle/parity.py``: every query must be identical to the
oracle or a classified near-tie (a distance near-tie at the k-th distance,
or a boundary near-tie whose cell key is within 1e-5 of the oracle's cutoff
key); no blanket "X% identical" allowance.  Distances of shared ids agree
within 1e-4 relative with the floor 1e-6*|q|^2 of test_fbpq.py:124-127.
"""

from oracle.parity import RTOL, check, classify  # noqa: F401


def check_topk(got_d, got_i, got_c, want_d, want_i, want_c, qnorm2=None, rtol=RTOL, **kw):
    """Assert the contract; ``kw`` may carry (orc, index, queries, L) so that
    boundary near-ties can be classified, and got_ncand / want_ncand."""
    return check(got_d, got_i, got_c, want_d, want_i, want_c, qnorm2, rtol=rtol, **kw)
