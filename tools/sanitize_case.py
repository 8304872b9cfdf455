"""Small end-to-end workload for compute-sanitizer (racecheck / memcheck /
synccheck): config-0 FBPQ + Multi-D-ADC searches (tensor-core first layer,
dense traversal), a sparse T=1500 index that exercises the partial sort, the
in-kernel prefix extension, the retry pass and the top-k compaction, a
large-cell M=8 index through the TMA stream kernels (warp-mode k=100 and
CTA-mode k=300, unaligned array end), and a tie plateau (plateau windows)."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1404_1831_b200 import DeviceIndex, _lib  # noqa: E402
from oracle import oracle as orc  # noqa: E402

# BPQ_CHECK_REPORT=1 (with BPQ_LIB=.../libbpq_b200_checked.so): run with the diagnostics buffer set and
# print the checked build's bound-violation counter (slot 19) and the stream kernel's entry count (slot 18)
REPORT = os.environ.get("BPQ_CHECK_REPORT") is not None
if REPORT:
    ctr = torch.zeros(32, dtype=torch.int64, device="cuda")
    _lib.load().bpq_debug_set_phase_buffer(_lib.ptr(ctr))

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
# large cells, M = 8: the TMA stream (warp mode for k <= 256, CTA mode above)
t, dim, m, kk, n = 10, 32, 8, 32, 20_003
base = rng.normal(size=(n, dim)).astype(np.float32)
c1 = base[rng.choice(n, t, replace=False), : dim // 2].copy()
c2 = base[rng.choice(n, t, replace=False), dim // 2 :].copy()
books = (0.3 * rng.normal(size=(m, kk, dim // m))).astype(np.float32)
off, ids, codes = orc.build_index(base, c1, c2, books)
lc = DeviceIndex(c1=c1, c2=c2, offsets=off, ids=ids, codes=codes, books=books)
ql = rng.normal(size=(6, dim)).astype(np.float32)
for L, k in ((2000, 100), (n, 300)):
    lc.search(ql, L, k, "fbpq").numpy()
# tie plateau: 192 codewords per half at +-10 e_u, query at the origin (every key equal, 36,864 cells)
dh, t = 96, 192
cb = np.zeros((t, dh), np.float32)
for i in range(t):
    cb[i, i // 2] = 10.0 if i % 2 == 0 else -10.0
ii, jj = np.meshgrid(np.arange(t), np.arange(t), indexing="ij")
base = np.concatenate([cb[ii.ravel()], cb[jj.ravel()]], 1) + rng.normal(scale=0.01, size=(t * t, 2 * dh)).astype(np.float32)
books = (0.01 * rng.normal(size=(8, 16, 2 * dh // 8))).astype(np.float32)
off, ids, codes = orc.build_index(base.astype(np.float32), cb, cb, books)
pl = DeviceIndex(c1=cb, c2=cb, offsets=off, ids=ids, codes=codes, books=books, exact=True)
pl.search(np.zeros((2, 2 * dh), np.float32), 5000, 20, "fbpq").numpy()
# adversarial order: one huge cell whose entries get closer to the query as ids grow (roll-back path)
t, dim, m, kk, n = 4, 32, 8, 32, 30_000
c1 = (10.0 * rng.normal(size=(t, dim // 2))).astype(np.float32)
c2 = (10.0 * rng.normal(size=(t, dim // 2))).astype(np.float32)
u = rng.normal(size=dim)
u /= np.linalg.norm(u)
base = (np.concatenate([c1[0], c2[0]])[None, :] + 3.0 * (1.0 - np.arange(n) / n)[:, None] * u[None, :]
        + 0.02 * rng.normal(size=(n, dim))).astype(np.float32)
books = (0.5 * rng.normal(size=(m, kk, dim // m))).astype(np.float32)
off, ids, codes = orc.build_index(base, c1, c2, books)
adv = DeviceIndex(c1=c1, c2=c2, offsets=off, ids=ids, codes=codes, books=books)
qa = (np.concatenate([c1[0], c2[0]])[None, :] + 0.05 * rng.normal(size=(4, dim))).astype(np.float32)
for k in (100, 1000):
    adv.search(qa, n, k, "fbpq").numpy()
torch.cuda.synchronize()
if REPORT:
    _lib.load().bpq_debug_set_phase_buffer(None)
    c = ctr.cpu().numpy()
    print(f"check_failures={int(c[19])} stream_entries={int(c[18])}")
print("sanitize case done")
