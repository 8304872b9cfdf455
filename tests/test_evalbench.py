"""Recall / ground-truth harness (paper_1404_1831_b200/evalbench.py) on CPU
tensors: exact_nn against a float64 brute force with ties toward the smaller
id (vecio.brute_force_knn, vecio.py:254), recall_at against the reference's
definition (evalbench.py:309-327) on a hand case."""

import numpy as np
import torch

from paper_1404_1831_b200 import evalbench


def _brute(base, q):
    d = ((base[:, None, :].astype(np.float64) - q[None].astype(np.float64)) ** 2).sum(2)
    return d.argmin(0), d.min(0)


def test_exact_nn_integer_and_float_match_f64_brute_force():
    rng = np.random.default_rng(3)
    base = rng.integers(0, 256, size=(3000, 32)).astype(np.float32)
    base[1700] = base[200]  # exact duplicate: the smaller id must win
    q = rng.integers(0, 256, size=(40, 32)).astype(np.float32)
    q[5] = base[1700]
    want_i, want_d = _brute(base, q)
    chunks = [(s, torch.from_numpy(base[s:s + 700])) for s in range(0, 3000, 700)]
    for integer in (True, False):
        ids, d2 = evalbench.exact_nn(chunks, torch.from_numpy(q), integer=integer)
        np.testing.assert_array_equal(ids.numpy(), want_i)
        np.testing.assert_allclose(d2.numpy(), want_d, rtol=0, atol=1e-6)
    assert int(evalbench.exact_nn(chunks, torch.from_numpy(q[5:6]))[0][0]) == 200


def test_recall_at_hand_case():
    # query 0: nn 7 at rank 0; query 1: nn 3 at rank 2; query 2: nn 9 beyond its count
    ids = torch.tensor([[7, 1, 2], [5, 6, 3], [4, 9, 0]])
    counts = torch.tensor([3, 3, 1])
    r = evalbench.recall_at(ids, counts, torch.tensor([7, 3, 9]), cutoffs=(1, 2, 3))
    assert r == {1: 1 / 3, 2: 1 / 3, 3: 2 / 3}
