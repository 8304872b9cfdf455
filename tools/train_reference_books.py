"""Train the c1/c2 codebooks with the REFERENCE package (BASELINE.md §3:
"c0-c2: built by the reference itself") and commit them as a fixture.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
        python tools/train_reference_books.py [--train 131072]

Output: ``tests/golden/c1_books.npz`` with
  c1, c2   f32 [4096, 64]  -- bilayerpq.train_coarse(learn, 4096, seed=0)
                              (multi_index.py:149-164: pq_train with M=2,
                              k-means++ + 25 Lloyd iterations)
  books    f32 [8, 256, 16] -- bilayerpq.train_fine_global(learn, coarse, 8, 256, seed=0)
                              (multi_index.py:192-196)
  train_n, train_seed, ncomp   the training draw (datagen.clipped_mixture,
                               4,096 components, seed 3 = SEED_TRAIN)

Both bench arms (GPU and --impl reference) load these, so they search the
same codebooks; the fixture is ~2.2 MB.
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import bilayerpq as bq  # noqa: E402  (the reference, read-only)

from paper_1404_1831_b200 import datagen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--train", type=int, default=131_072)
    ap.add_argument("--t", type=int, default=4096)
    ap.add_argument("--ncomp", type=int, default=4096)
    ap.add_argument("--out", default=str(ROOT / "tests" / "golden" / "c1_books.npz"))
    a = ap.parse_args()
    learn = datagen.clipped_mixture(a.train, 128, a.ncomp, datagen.SEED_TRAIN)
    t0 = time.time()
    coarse = bq.train_coarse(learn, a.t, seed=0)
    print(f"train_coarse T={a.t}: {time.time() - t0:.1f}s", flush=True)
    t1 = time.time()
    fine = bq.train_fine_global(learn, coarse, 8, 256, seed=0)
    print(f"train_fine_global M=8 K=256: {time.time() - t1:.1f}s", flush=True)
    np.savez_compressed(a.out, c1=coarse.book1.centroids, c2=coarse.book2.centroids, books=fine.codebooks,
                        train_n=np.int64(a.train), train_seed=np.int64(datagen.SEED_TRAIN),
                        ncomp=np.int64(a.ncomp))
    print("wrote", a.out)


if __name__ == "__main__":
    main()
