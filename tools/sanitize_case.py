"""Small end-to-end workload for compute-sanitizer (racecheck / memcheck /
synccheck): config-0 FBPQ + Multi-D-ADC searches (dense traversal), and a
sparse T=1500 index that exercises the partial sort, the in-kernel prefix
extension, the retry pass and the top-k compaction."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1404_1831_b200 import DeviceIndex  # noqa: E402
from oracle import oracle as orc  # noqa: E402

g = np.load(ROOT / "tests" / "golden" / "c0.npz")
tables = (g["cn1"], g["cn2"], g["fine_norms"], g["cross1"], g["cross2"])
dix = DeviceIndex(c1=g["c1"], c2=g["c2"], offsets=g["offsets"], ids=g["ids"], codes=g["codes"], books=g["books"],
                  tables=tables)
q = g["queries"][:8].astype(np.float32)
for eng in ("fbpq", "baseline"):
    dix.search(q, 10_000, 100, eng).numpy()
rng = np.random.default_rng(11)
t, dim, m, kk, n = 1500, 32, 4, 16, 20_000
cent = rng.normal(scale=6.0, size=(300, dim)).astype(np.float32)
base = (cent[rng.integers(0, 300, n)] + rng.normal(size=(n, dim))).astype(np.float32)
c1 = base[rng.choice(n, t, replace=False), : dim // 2].copy()
c2 = base[rng.choice(n, t, replace=False), dim // 2 :].copy()
books = rng.normal(scale=0.4, size=(m, kk, dim // m)).astype(np.float32)
off, ids, codes = orc.build_index(base, c1, c2, books)
sp = DeviceIndex(c1=c1, c2=c2, offsets=off, ids=ids, codes=codes, books=books)
qs = (cent[rng.integers(0, 300, 6)] + rng.normal(size=(6, dim))).astype(np.float32)
for L in (100, 5000, n):
    sp.search(qs, L, 50, "fbpq").numpy()
torch.cuda.synchronize()
print("sanitize case done")
