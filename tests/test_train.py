"""Device codebook training against books trained by the
reference itself (tests/golden: c0 coarse + fine books, the HBPQ rig's
local bank), with the reference's random draws (train.py rng="exact").

Equality is bit-for-bit unless a Lloyd assignment hit an argmin near-tie
(f32 scores of the GPU kernel vs OpenBLAS, quantizer.py:124-125).  After
such a tie the two Lloyd trajectories continue from different assignments
and may stop in different local optima, so a differing book must still
reach the reference's training objective within ``tol`` (5e-3 for the
global books, whose displacements also inherit the coarse assignment's
near-ties; 1% for the small local cells of the HBPQ bank, where one
reassigned point moves a 1-2k-point k-means), and almost every local book
must be identical."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")


def _objective(x, cents):
    x = x.astype(np.float64)
    c = cents.astype(np.float64)
    d = (x * x).sum(1)[:, None] - 2 * x @ c.T + (c * c).sum(1)[None]
    return float(np.maximum(d.min(1), 0).sum())


def _same_or_objective(got, want, data, what, tol=1e-4):
    if np.array_equal(got, want):
        return "identical"
    og, ow = _objective(data, got), _objective(data, want)
    assert abs(og - ow) <= tol * ow, f"{what}: objective {og} vs reference {ow}"
    return f"objective within {abs(og - ow) / ow:.1e}"


def test_train_coarse_and_fine_match_reference(dev, c0):
    from paper_1404_1831_b200 import datagen, train

    learn = datagen.clipped_mixture(50_000, 128, 1024, datagen.SEED_TRAIN, datagen.mixture_centres(1024, 128))
    c1, c2 = train.train_coarse(learn, 64, seed=0)
    r1 = _same_or_objective(c1, c0["c1"], learn[:, :64], "coarse half 1", tol=5e-3)
    r2 = _same_or_objective(c2, c0["c2"], learn[:, 64:], "coarse half 2", tol=5e-3)
    books = train.train_fine_global(learn, c0["c1"], c0["c2"], 8, 256, seed=0)  # the reference's coarse pair
    disp, _, _ = train.displacements(learn, c0["c1"], c0["c2"])
    disp = disp.cpu().numpy()
    rf = [_same_or_objective(books[p], c0["books"][p], disp[:, p * 16:(p + 1) * 16], f"fine part {p}", tol=5e-3)
          for p in range(8)]
    print("coarse:", r1, r2, "fine:", rf)


def test_train_local_codebooks_match_reference(dev, hbpq_rig):
    from paper_1404_1831_b200 import datagen, train

    g = hbpq_rig
    base = datagen.clipped_mixture(20_000, 128, 1024, datagen.SEED_BASE, datagen.mixture_centres(1024, 128))
    b1, b2 = train.train_local_codebooks(base, g["c1"], g["c2"], 8, 64, seed=0)
    disp, i_idx, j_idx = train.displacements(base, g["c1"], g["c2"])
    disp = disp.cpu().numpy()
    i_idx, j_idx = i_idx.cpu().numpy(), j_idx.cpu().numpy()
    same = 0
    for h, (got, want, cell) in enumerate(((b1, g["bank1"], i_idx), (b2, g["bank2"], j_idx))):
        for i in range(got.shape[0]):
            members = disp[cell == i, h * 64:(h + 1) * 64]
            for p in range(4):
                r = _same_or_objective(got[i, p], want[i, p], members[:, p * 16:(p + 1) * 16], f"bank{h+1}[{i},{p}]",
                                       tol=1e-2)
                same += r == "identical"
    total = 2 * b1.shape[0] * 4
    print(f"{same} of {total} local books identical")
    assert same >= 0.9 * total, f"only {same} of {total} local books identical"


def test_device_rng_mode_trains_comparable_books(dev, c0):
    """rng='device' (benchmark setup) is the same algorithm on another random
    stream: its objective is within 2% of the reference's."""
    from paper_1404_1831_b200 import datagen, train

    learn = datagen.clipped_mixture(50_000, 128, 1024, datagen.SEED_TRAIN, datagen.mixture_centres(1024, 128))
    c1, _ = train.train_coarse(learn, 64, seed=0, mode="device")
    og, ow = _objective(learn[:, :64], c1), _objective(learn[:, :64], c0["c1"])
    assert og <= 1.02 * ow, (og, ow)
