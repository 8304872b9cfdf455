"""Benchmark: batched bilayer-PQ search on B200 (BASELINE.json metric).

Metric: queries/s at fixed L, k (plus PQ codes scanned/s, per-stage CUDA-event
times and the dominant kernel's HBM roofline fraction).  Default workload is
BASELINE.json configs[1] (single-GPU FBPQ): N=10M clipped-integer mixture
vectors (D=128, 4,096 components), T=4,096 per half, M=8 x 256, 10,000
queries, L=10,000, k=100.  Data is seeded synthetic (the paper's BIGANN is
not available); the c1/c2 codebooks are the reference's own training output
(tests/golden/c1_books.npz), the other configs train on the device (untimed).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c0|c1|c2|c3|c4|c4m16] [--engine fbpq|baseline|hbpq]
                  [--L ..] [--k ..] [--exact] [--replicas] [--no-split]

N>1 (torchrun): the database is sharded by point id with the global budget
and the query-split traversal: all ranks answer
ONE 10k-query batch ("scaling": "strong"); value is that batch over the
max-over-ranks device time.  --replicas runs independent copies instead.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAKS = {}
try:
    PEAKS = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
except Exception:
    pass
HBM_PEAK = float(PEAKS.get("hbm_gbs", 6650.0))
HBM_PEAK_SRC = "measured" if "hbm_gbs" in PEAKS else "fallback"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# exact-NN ground truth of the first RECALL_Q queries (evalbench.ExactNN), filled while the base is
# resident (c1/c2) or streamed (c3/c4) during setup; reported as Recall@{1,10,100} (untimed)
RECALL_Q = 1000
GT = {}
PROFILE = {}  # --phase-profile results, copied into the JSON line


def _gt_start(q):
    from paper_1404_1831_b200 import evalbench

    if RECALL_Q <= 0:
        return None
    n = min(RECALL_Q, q.shape[0])
    GT["n"] = n
    GT["acc"] = evalbench.ExactNN(q[:n])
    return GT["acc"]


# --------------------------------------------------------------------- setup
CONFIGS = {
    # c1/c2: codebooks trained by the reference itself (tests/golden/c1_books.npz), base and queries from
    # the blocked numpy stream that bench_reference.py (the --impl reference arm) draws identically
    "c1": dict(n=10_000_000, dim=128, ncomp=4096, t=4096, m=8, k=256, nq=10_000, L=10_000, topk=100,
               engine="fbpq", train=131_072, ref_books=True),
    "c2": dict(n=10_000_000, dim=128, ncomp=4096, t=4096, m=8, k=256, nq=10_000, L=10_000, topk=100,
               engine="hbpq", train=131_072, ref_books=True),
    # billion-scale (BASELINE configs[4]) on one GPU: streamed build, 16,384 components
    "c4": dict(n=1_000_000_000, dim=128, ncomp=16384, t=16384, m=8, k=256, nq=10_000, L=10_000, topk=100,
               engine="fbpq", train=1_048_576, stream=True),
    "c4m16": dict(n=1_000_000_000, dim=128, ncomp=16384, t=16384, m=16, k=256, nq=10_000, L=10_000, topk=100,
                  engine="fbpq", train=1_048_576, stream=True),
    # higher-dimensional dense features (BASELINE configs[3]) on one GPU
    "c3": dict(n=50_000_000, dim=384, ncomp=4096, t=4096, m=16, k=256, nq=10_000, L=30_000, topk=100,
               engine="fbpq", train=524_288, stream=True, normalized=True),
    "c1small": dict(n=1_000_000, dim=128, ncomp=4096, t=1024, m=8, k=256, nq=10_000, L=10_000, topk=100,
                    engine="fbpq", train=131_072),
}


def build_workload(cfg, device, rank=0):
    """Returns (DeviceIndex, queries [nq, D] device f32, host arrays for the CPU baseline)."""
    import torch

    from paper_1404_1831_b200 import datagen, encode

    name = cfg["name"]
    if name == "c0":
        g = np.load(ROOT / "tests" / "golden" / "c0.npz")
        from paper_1404_1831_b200 import DeviceIndex

        tables = (g["cn1"], g["cn2"], g["fine_norms"], g["cross1"], g["cross2"])
        dix = DeviceIndex(c1=g["c1"], c2=g["c2"], offsets=g["offsets"], ids=g["ids"], codes=g["codes"],
                          books=g["books"], tables=tables, device=device)
        q = torch.from_numpy(g["queries"].astype(np.float32)).to(device)
        host = dict(c1=g["c1"], c2=g["c2"], offsets=g["offsets"], ids=g["ids"], codes=g["codes"], books=g["books"],
                    tables=tables)
        return dix, q, (lambda: host)
    t0 = time.time()
    if cfg.get("ref_books"):
        return build_ref_books_workload(cfg, device, rank, t0)
    if cfg.get("normalized"):
        centt = datagen.normalized_centres_torch(cfg["ncomp"], cfg["dim"], device)

        def draw(s, e, seed):
            return datagen.normalized_mixture_chunk(s, e, cfg["dim"], cfg["ncomp"], seed, device, centt)
    else:
        cent = datagen.mixture_centres(cfg["ncomp"], cfg["dim"])
        centt = torch.as_tensor(cent, dtype=torch.float32, device=device)

        def draw(s, e, seed):
            return datagen.clipped_mixture_chunk(s, e, cfg["dim"], cfg["ncomp"], seed, device, centt)
    if cfg.get("stream"):
        train = draw(0, cfg["train"], datagen.SEED_TRAIN)
    else:
        train = datagen.clipped_mixture_torch(cfg["train"], cfg["dim"], cfg["ncomp"], datagen.SEED_TRAIN, device, cent)
    dh = cfg["dim"] // 2
    c1 = encode.train_kmeans(train[:, :dh].contiguous(), cfg["t"], iters=8, seed=11)
    c2 = encode.train_kmeans(train[:, dh:].contiguous(), cfg["t"], iters=8, seed=12)
    i_idx, j_idx = encode.assign_cells(train, c1, c2)
    c1t = torch.from_numpy(c1).to(device)
    c2t = torch.from_numpy(c2).to(device)
    disp = train - torch.cat([c1t[i_idx], c2t[j_idx]], 1)
    ds = cfg["dim"] // cfg["m"]
    books = np.stack([encode.train_kmeans(disp[:, p * ds:(p + 1) * ds].contiguous(), cfg["k"], iters=8, seed=20 + p)
                      for p in range(cfg["m"])])
    log(f"[setup] codebooks trained in {time.time() - t0:.1f}s")
    if cfg.get("stream"):
        q = draw(0, cfg["nq"], datagen.SEED_QUERIES + 1000 * rank)
        acc = _gt_start(q)

        def draw_base(s, e):
            x = draw(s, e, datagen.SEED_BASE)
            if acc is not None:
                acc.add(s, x)
            return x

        dix = encode.build_index_streamed(cfg["n"], draw_base, c1, c2, books, device=device)
        host_books = dict(books=books)
        base = None
    else:
        base = datagen.clipped_mixture_torch(cfg["n"], cfg["dim"], cfg["ncomp"], datagen.SEED_BASE, device, cent)
    if cfg.get("stream"):
        pass
    elif cfg["engine"] == "hbpq":
        # local books per half-codeword: pooled residual books + per-row perturbation
        # (bank training is out of scope; codes are encoded against these books)
        m2 = cfg["m"] // 2
        gen = torch.Generator(device=device)
        gen.manual_seed(5)
        b = torch.from_numpy(books).to(device)
        bank1 = (b[None, :m2] + 0.5 * torch.randn((cfg["t"], m2) + b.shape[1:], generator=gen, device=device)).cpu().numpy()
        bank2 = (b[None, m2:] + 0.5 * torch.randn((cfg["t"], m2) + b.shape[1:], generator=gen, device=device)).cpu().numpy()
        dix = encode.build_hbpq_index(base, c1, c2, bank1, bank2, device=device)
        host_books = dict(bank1=bank1, bank2=bank2)
    else:
        dix = encode.build_index(base, c1, c2, books, device=device)
        host_books = dict(books=books)
    del base
    torch.cuda.empty_cache()
    if cfg.get("stream"):
        pass  # drawn before the build
    else:
        q = datagen.clipped_mixture_torch(cfg["nq"], cfg["dim"], cfg["ncomp"], datagen.SEED_QUERIES + 1000 * rank,
                                          device, cent)
    log(f"[setup] index built in {time.time() - t0:.1f}s: N={dix.n} populated="
        f"{int((torch.diff(dix.offsets.long() & 0xFFFFFFFF) > 0).sum())}")
    def host():
        """Host copy of the index for the CPU baseline (built on demand)."""
        h = dict(c1=c1, c2=c2, offsets=(dix.offsets.cpu().numpy().view(np.uint32)).astype(np.int64),
                 ids=dix.ids.cpu().numpy().view(np.uint32), codes=dix.codes.cpu().numpy(), **host_books)
        if cfg["engine"] != "hbpq":
            h["tables"] = (dix.cn1.cpu().numpy(), dix.cn2.cpu().numpy(), dix.fine_norms.cpu().numpy(),
                           dix.cross1.cpu().numpy(), dix.cross2.cpu().numpy())
        return h

    return dix, q, host


def build_ref_books_workload(cfg, device, rank, t0):
    """c1/c2: the reference-trained codebooks (tests/golden/c1_books.npz) and
    the blocked numpy base/query stream (datagen.clipped_mixture_blocked), i.e.
    the same vectors the --impl reference arm encodes with bilayerpq; encoding
    and packing run on the device (encode.build_index)."""
    import torch

    from paper_1404_1831_b200 import datagen, encode

    bk = np.load(ROOT / "tests" / "golden" / "c1_books.npz")
    c1, c2, books = bk["c1"], bk["c2"], bk["books"]
    cent = datagen.mixture_centres(cfg["ncomp"], cfg["dim"])
    base_h = datagen.clipped_mixture_blocked(cfg["n"], cfg["dim"], cfg["ncomp"], datagen.SEED_BASE, centres=cent)
    log(f"[setup] base drawn on the host in {time.time() - t0:.1f}s")
    base = torch.empty((cfg["n"], cfg["dim"]), dtype=torch.float32, device=device)
    step = 1 << 22
    for s0 in range(0, cfg["n"], step):
        base[s0:s0 + step].copy_(torch.from_numpy(base_h[s0:s0 + step]))
    del base_h
    host_books = dict(books=books)
    qh = datagen.clipped_mixture_block(0, cfg["dim"], cfg["ncomp"], datagen.SEED_QUERIES + 1000 * rank, cent,
                                       cfg["nq"])
    q = torch.from_numpy(qh).to(device)
    acc = _gt_start(q)
    if acc is not None:
        acc.add(0, base)
    if cfg["engine"] == "hbpq":
        from paper_1404_1831_b200 import train

        bank1, bank2 = train.local_bank_for_bench(base, c1, c2, books, cfg, device)
        dix = encode.build_hbpq_index(base, c1, c2, bank1, bank2, device=device)
        host_books = dict(bank1=bank1, bank2=bank2)
    else:
        dix = encode.build_index(base, c1, c2, books, device=device)
    del base
    torch.cuda.empty_cache()
    log(f"[setup] index built in {time.time() - t0:.1f}s: N={dix.n} populated="
        f"{int((torch.diff(dix.offsets.long() & 0xFFFFFFFF) > 0).sum())}")

    def host():
        h = dict(c1=c1, c2=c2, offsets=(dix.offsets.cpu().numpy().view(np.uint32)).astype(np.int64),
                 ids=dix.ids.cpu().numpy().view(np.uint32), codes=dix.codes.cpu().numpy(), **host_books)
        if cfg["engine"] != "hbpq":
            h["tables"] = (dix.cn1.cpu().numpy(), dix.cn2.cpu().numpy(), dix.fine_norms.cpu().numpy(),
                           dix.cross1.cpu().numpy(), dix.cross2.cpu().numpy())
        return h

    return dix, q, host


def build_sharded_ref_workload(cfg, device, rank, world):
    """c1/c2 sharded by point id: rank r encodes rows [r N / W, (r+1) N / W) of
    the same blocked base stream with the reference-trained codebooks (ids
    offset by the range start); the global per-cell counts come from one NCCL
    all-reduce.  Queries are the same 10k on every rank."""
    import torch
    import torch.distributed as dist

    from paper_1404_1831_b200 import DeviceIndex, datagen, encode

    bk = np.load(ROOT / "tests" / "golden" / "c1_books.npz")
    c1, c2, books = bk["c1"], bk["c2"], bk["books"]
    cent = datagen.mixture_centres(cfg["ncomp"], cfg["dim"])
    lo, hi = cfg["n"] * rank // world, cfg["n"] * (rank + 1) // world
    blocks = []
    for b in range(lo // datagen.BLOCK, (hi - 1) // datagen.BLOCK + 1):
        b0 = b * datagen.BLOCK
        rows = min(cfg["n"], b0 + datagen.BLOCK) - b0
        x = datagen.clipped_mixture_block(b, cfg["dim"], cfg["ncomp"], datagen.SEED_BASE, cent, rows)
        blocks.append(x[max(lo - b0, 0): min(hi - b0, rows)])
    base = torch.from_numpy(np.concatenate(blocks)).to(device)
    local = encode.build_index(base, c1, c2, books, id_offset=lo, device=device)
    del base
    cnt = (local.offsets[1:].long() & 0xFFFFFFFF) - (local.offsets[:-1].long() & 0xFFFFFFFF)
    dist.all_reduce(cnt)
    goff = torch.zeros(cnt.numel() + 1, dtype=torch.int64, device=device)
    torch.cumsum(cnt, 0, out=goff[1:])
    dix = DeviceIndex(c1=c1, c2=c2, offsets=local.offsets, ids=local.ids, codes=local.codes, books=books,
                      tables=(local.cn1, local.cn2, local.fine_norms, local.cross1, local.cross2),
                      global_offsets=goff.to(torch.int32), num_entries_global=int(goff[-1].item()), device=device)
    del local
    qh = datagen.clipped_mixture_block(0, cfg["dim"], cfg["ncomp"], datagen.SEED_QUERIES, cent, cfg["nq"])
    return dix, torch.from_numpy(qh).to(device)


def build_sharded_workload(cfg, device, rank, world):
    """rank r holds the points with ids in [r N / W, (r+1) N / W)
    (its own multi-index, built with id_offset) plus the GLOBAL per-cell
    counts (one NCCL all-reduce at build time), so every rank runs the same
    traversal under the global budget and scans only its local entries.
    Codebooks and queries are broadcast from rank 0."""
    import torch
    import torch.distributed as dist

    from paper_1404_1831_b200 import DeviceIndex, datagen, encode

    dh = cfg["dim"] // 2
    ds = cfg["dim"] // cfg["m"]
    cent = datagen.mixture_centres(cfg["ncomp"], cfg["dim"])
    centt = torch.as_tensor(cent, dtype=torch.float32, device=device)

    def draw(s, e, seed):
        return datagen.clipped_mixture_chunk(s, e, cfg["dim"], cfg["ncomp"], seed, device, centt)

    c1 = torch.empty((cfg["t"], dh), device=device)
    c2 = torch.empty((cfg["t"], dh), device=device)
    books = torch.empty((cfg["m"], cfg["k"], ds), device=device)
    if rank == 0:
        train = draw(0, cfg["train"], datagen.SEED_TRAIN)
        c1.copy_(torch.from_numpy(encode.train_kmeans(train[:, :dh].contiguous(), cfg["t"], iters=8, seed=11)))
        c2.copy_(torch.from_numpy(encode.train_kmeans(train[:, dh:].contiguous(), cfg["t"], iters=8, seed=12)))
        i_idx, j_idx = encode.assign_cells(train, c1.cpu().numpy(), c2.cpu().numpy())
        disp = train - torch.cat([c1[i_idx], c2[j_idx]], 1)
        books.copy_(torch.from_numpy(np.stack([
            encode.train_kmeans(disp[:, p * ds:(p + 1) * ds].contiguous(), cfg["k"], iters=8, seed=20 + p)
            for p in range(cfg["m"])])))
    for t in (c1, c2, books):
        dist.broadcast(t, 0)
    c1n, c2n, booksn = c1.cpu().numpy(), c2.cpu().numpy(), books.cpu().numpy()
    lo, hi = cfg["n"] * rank // world, cfg["n"] * (rank + 1) // world
    local = encode.build_index_streamed(hi - lo, lambda s, e: draw(lo + s, lo + e, datagen.SEED_BASE), c1n, c2n,
                                        booksn, id_offset=lo, device=device)
    cnt = (local.offsets[1:].long() & 0xFFFFFFFF) - (local.offsets[:-1].long() & 0xFFFFFFFF)
    dist.all_reduce(cnt)
    goff = torch.zeros(cnt.numel() + 1, dtype=torch.int64, device=device)
    torch.cumsum(cnt, 0, out=goff[1:])
    n_global = int(goff[-1].item())
    dix = DeviceIndex(c1=c1n, c2=c2n, offsets=local.offsets, ids=local.ids, codes=local.codes, books=booksn,
                      tables=(local.cn1, local.cn2, local.fine_norms, local.cross1, local.cross2),
                      global_offsets=goff.to(torch.int32), num_entries_global=n_global, device=device)
    del local
    q = draw(0, cfg["nq"], datagen.SEED_QUERIES)
    dist.broadcast(q, 0)
    return dix, q


# -------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and clock-event (throttle) reasons every ~5 ms via NVML
    while the timed region runs (nvidia-smi's -lms floor is too coarse for a
    few-hundred-millisecond region)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index=0, period=0.005):
        self.index = index
        self.period = period
        self.sm, self.mx, self.flags = [], None, 0
        self.ok = False

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.stop = threading.Event()
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()
            self.ok = True
        except Exception:
            self.ok = False
        return self

    def _run(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                self.flags |= int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        if self.ok:
            self.stop.set()
            self.th.join(timeout=2)

    def summary(self):
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None, "sm_max_mhz": self.mx,
                "reasons": sorted(n for n, b in self.REASONS.items() if self.flags & b),
                "samples": len(self.sm), "source": "nvml"}


# --------------------------------------------------------------- CPU baseline
def _oracle_index(host):
    from oracle import oracle as orc

    return orc.Index(host["c1"], host["c2"], host["offsets"], host["ids"], host["codes"], books=host.get("books"),
                     bank1=host.get("bank1"), bank2=host.get("bank2"), tables=host.get("tables"))


def cpu_baseline(host, engine, queries_np, L, k, budget_s=20.0):
    """The C oracle (oracle/bpq_oracle.c, a port of the reference search) on
    all host threads over a bounded query sample; returns the cpu_baseline
    block and the oracle's answers for the parity check."""
    from oracle import oracle as orc

    threads = os.cpu_count() or 1
    idx = _oracle_index(host)
    n0 = min(len(queries_np), max(threads, 16))
    t0 = time.perf_counter()
    orc.search_batch_c(idx, engine, queries_np[:n0], L, k, threads=threads)
    per_q = (time.perf_counter() - t0) / n0
    n = int(min(len(queries_np), max(n0, budget_s / max(per_q, 1e-6))))
    t0 = time.perf_counter()
    res = orc.search_batch_c(idx, engine, queries_np[:n], L, k, threads=threads)
    dt = time.perf_counter() - t0
    block = {"value": n / dt, "unit": "queries/s", "cores": threads, "kind": "port",
             "sample": f"first {n} of {len(queries_np)} queries, same index, L={L}, k={k}, "
                       f"C oracle (oracle/bpq_oracle.c) with {threads} POSIX threads",
             "codes_per_s": float(res[3].sum()) / dt}
    return block, res, idx, n


def parity_block(got, want, idx, queries_np, L):
    """SURVEY §8c(ii) on the oracle's sample: the GPU answers (through the
    public API, host buffers) against the C oracle's, every mismatch
    classified (oracle/parity.py)."""
    from oracle import oracle as orc
    from oracle.parity import classify

    gd, gi, gc, gn = got
    wd, wi, wc, wn = want
    n = wd.shape[0]
    q = queries_np[:n]
    qn = np.einsum("ij,ij->i", q.astype(np.float64), q.astype(np.float64))
    s = classify(gd[:n], gi[:n], gc[:n], wd, wi, wc, qn, got_ncand=None if gn is None else gn[:n], want_ncand=wn,
                 orc=orc, index=idx, queries=q, L=L)
    s["oracle"] = "C oracle (oracle/bpq_oracle.c) on the same index and queries"
    s["contract"] = ("SURVEY 8c(ii): shared-id distances within 1e-4 rel (floor 1e-6|q|^2); differing ids only as "
                     "k-th-distance near-ties (1e-4) or in cells within 1e-5 of the oracle's cutoff key")
    return s


def launches_per_step(dix, engine):
    """Engine kernels per bpq_search call (one query chunk): first layer, row
    sort (partial on sparse tables), fold (FBPQ), fused search, the
    full-sort + search retry pass after a partial sort, and the large-cell
    stream (point-term FBPQ, M = 8 / 16)."""
    n = 3 + (1 if engine == "fbpq" else 0)
    if dix.row_ptr is not None and dix.t > 1024:
        n += 2
    if engine == "fbpq" and not dix.fbpq_exact and dix.m in (8, 16):
        n += 1
    return n


# ------------------------------------------------------------------------ run
METRIC = "queries/s (batched search at fixed L, k)"


def _config(args):
    if args.config == "c0":
        cfg = dict(name="c0", nq=1000, L=10_000, topk=100, engine="fbpq", m=8, t=64, n=100_000, dim=128, k=256)
    else:
        cfg = dict(CONFIGS[args.config], name=args.config)
    if args.engine:
        cfg["engine"] = args.engine
    if args.L:
        cfg["L"] = args.L
    if args.k:
        cfg["topk"] = args.k
    if args.nq:
        cfg["nq"] = args.nq
    return cfg


def _config_block(cfg, n, dim, t, m, kk, nq, args, world):
    engine, L, k = cfg["engine"], cfg["L"], cfg["topk"]
    workload = f"{cfg['name']}: {engine} N={n:,} D={dim} T={t} M={m}x{kk} nq={nq} L={L} k={k}"
    return {"workload": workload, "engine": engine, "N": n, "D": dim, "T": t, "M": m, "nq": nq, "L": L, "k": k,
            "parallelism": ((f"shard{world}" + ("" if args.no_split else "+query-split")) if args.shard
                            else f"replicas{args.gpus}" if world > 1 else "single"),
            "l2": "flushed between timed steps (256 MiB write)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c1")
    ap.add_argument("--engine", default=None)
    ap.add_argument("--L", type=int, default=None)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--nq", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--recall-queries", type=int, default=1000,
                    help="queries whose exact NN is computed during setup for Recall@{1,10,100} (0: off)")
    ap.add_argument("--exact", action="store_true", help="FBPQ/Multi-D-ADC/HBPQ in the reference's exact "
                    "operation order (no point term, no per-cell residual tables)")
    ap.add_argument("--shard", action="store_true",
                    help="shard the database by point id across the ranks (global budget, NCCL all-gather merge); "
                         "the default when launched with more than one rank")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: every rank searches its own batch over a full copy instead (weak scaling)")
    ap.add_argument("--no-split", action="store_true",
                    help="sharded: replicate the first layer and traversal on every rank instead of splitting the "
                         "queries across ranks for them")
    ap.add_argument("--e2e-pieces", type=int, default=1,
                    help="slices of the end-to-end host-to-host call (DeviceIndex.search_host); 1 = one "
                         "upload, one search, one download (slicing over streams measured slower)")
    ap.add_argument("--phase-profile", action="store_true",
                    help="print per-phase cycle shares of the fused kernel (needs BPQ_LIB=...libbpq_b200_prof.so)")
    args = ap.parse_args()

    global RECALL_Q
    RECALL_Q = args.recall_queries
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 and not args.replicas:
        args.shard = True  # north_star's scaling path: the database sharded by point id
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = _config(args)
    if args.exact:
        os.environ["BPQ_FBPQ_EXACT"] = "1"  # DeviceIndex default (index.py)
    if args.impl == "reference":
        # the reference's own CPU search on this host (rank 0 only; no product code, no CUDA)
        if rank == 0:
            import bench_reference

            bench_reference.run(args, cfg, METRIC, _config_block(cfg, cfg["n"], cfg["dim"], cfg["t"], cfg["m"],
                                                                 cfg["k"], cfg["nq"], args, world))
        return

    import torch

    if world > 1 or args.shard:
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        os.environ.setdefault("NCCL_DEBUG", "NONE")  # keep stdout to the one JSON line
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    device = torch.device("cuda", local_rank)

    engine, L, k = cfg["engine"], cfg["L"], cfg["topk"]
    searcher = None
    if args.shard:
        from paper_1404_1831_b200 import sharded

        dix, q = (build_sharded_ref_workload if cfg.get("ref_books") else build_sharded_workload)(cfg, device, rank,
                                                                                                   world)
        host = None
        split = (not args.no_split and engine == "fbpq" and dix.m in (8, 16) and not dix.fbpq_exact)
        searcher = (sharded.SplitSearcher(dix, force_collective=True) if split
                    else sharded.ShardedSearcher(dix, force_collective=True))
    else:
        dix, q, host = build_workload(cfg, device, rank)
    nq = q.shape[0]
    config = _config_block(cfg, dix.n, dix.dim, dix.t, dix.m, dix.k, nq, args, world)
    workload = config["workload"]
    metric = METRIC

    from paper_1404_1831_b200.index import SearchResult

    ws = dix.make_workspace(engine, nq, L, k)
    out = SearchResult(torch.empty((nq, k), dtype=torch.float32, device=device),
                       torch.empty((nq, k), dtype=torch.int32, device=device),
                       torch.empty((nq,), dtype=torch.int32, device=device),
                       torch.empty((nq,), dtype=torch.int64, device=device))
    popped = torch.empty((nq,), dtype=torch.int64, device=device)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    stream = torch.cuda.current_stream()

    # one untimed pass for the work counts (candidates and popped cells)
    dix.search(q, L, k, engine, out=out, workspace=ws, ncand=True, popped=popped)
    torch.cuda.synchronize()
    counts = out.counts.cpu().numpy()
    if (counts < 0).any():
        raise RuntimeError(f"{int((counts < 0).sum())} queries hit the tie-plateau limit")
    ncand_q = out.ncand.cpu().numpy()
    ncand = int(ncand_q.sum())
    npop = int(popped.sum().item())
    # entries the large-cell stream kernel scans per batch (counter 18 of the diagnostics buffer, any build)
    stream_cand = 0
    if engine == "fbpq" and not dix.fbpq_exact and os.environ.get("BPQ_STREAM_TMA") is None:
        from paper_1404_1831_b200 import _lib

        ctr = torch.zeros(32, dtype=torch.int64, device=device)
        _lib.load().bpq_debug_set_phase_buffer(_lib.ptr(ctr))
        dix.search(q, L, k, engine, out=out, workspace=ws)
        torch.cuda.synchronize()
        _lib.load().bpq_debug_set_phase_buffer(None)
        stream_cand = int(ctr[18].item())
        log(f"[diag] stream entries {stream_cand:,}, roll-backs {int(ctr[20].item())}")
    if args.phase_profile:
        from paper_1404_1831_b200 import _lib

        ctr = torch.zeros(32, dtype=torch.int64, device=device)
        on = _lib.load().bpq_debug_set_phase_buffer(_lib.ptr(ctr))
        dix.search(q, L, k, engine, out=out, workspace=ws)
        torch.cuda.synchronize()
        _lib.load().bpq_debug_set_phase_buffer(None)
        names = ["prologue", "tau_search|sparse_reclassify", "band_bounds|sparse_activate", "enumerate|sparse_gather",
                 "scan", "lut_scan", "topk_compact", "final_select", "finish", "idle", "extend_prefix",
                 "stream_prologue", "stream_wait", "stream_score", "stream_compact", "stream_finish",
                 "residual_table_build"]
        cc = ctr.cpu().numpy()
        c = cc[:17].astype(float)
        k1, k2 = np.concatenate([c[:11], c[16:17]]), c[11:16]
        halves = int(cc[17])
        prof = {"phase_profile_compiled": bool(on),
                "traversal_kernel_share": {n: round(float(v / max(k1.sum(), 1)), 4)
                                           for n, v in zip(names[:11] + names[16:17], k1)},
                "stream_kernel_share": {n: round(float(v / max(k2.sum(), 1)), 4) for n, v in zip(names[11:16], k2)}}
        if engine in ("hbpq", "baseline"):
            # BASELINE configs[2] / SURVEY 8(d) d2: the local-table cost beside the scan
            tb = dix.m // 2 * dix.k * (dix.dim // dix.m) * 4
            prof["residual_tables"] = {"halves_built_per_batch": halves, "bytes_per_half": tb,
                                       "bytes_per_batch": halves * tb, "halves_per_query": halves / nq}
        log(json.dumps(prof))
        PROFILE.update(prof)
    for _ in range(args.warmup):
        dix.search(q, L, k, engine, out=out, workspace=ws)
    torch.cuda.synchronize()

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    for row in evs:  # torch creates CUDA events lazily on first record
        for e in row:
            e.record(stream)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()
    sev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    with ClockSampler(local_rank) as clk:
        for s in range(args.steps):
            flush.fill_(s & 0xFF)  # L2 flush, outside the event pair
            if searcher is not None:  # local search + NCCL all-gather + device merge
                sev[s][0].record(stream)
                searcher.search(q, L, k, engine, workspace=ws, stage_events=evs[s])
                sev[s][1].record(stream)
            else:
                dix.search(q, L, k, engine, out=out, workspace=ws, stage_events=evs[s])
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    if searcher is not None:
        step_ms = [sev[s][0].elapsed_time(sev[s][1]) for s in range(args.steps)]
    else:
        step_ms = [evs[s][0].elapsed_time(evs[s][4]) for s in range(args.steps)]
    stage_ms = np.array([[evs[s][i].elapsed_time(evs[s][i + 1]) for i in range(4)] for s in range(args.steps)])
    t_ms = float(np.sum(step_ms))
    if world > 1:
        tt = torch.tensor([t_ms], device=device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    # replicas: every rank answers its own batch; shard: all ranks answer one batch
    qmul = 1 if args.shard else world
    value = qmul * nq * args.steps / (t_ms / 1e3)

    # end to end through the public API with host buffers
    q_host = q.cpu().pin_memory()
    od_h = torch.empty((nq, k), dtype=torch.float32).pin_memory()
    oi_h = torch.empty((nq, k), dtype=torch.int32).pin_memory()
    oc_h = torch.empty((nq,), dtype=torch.int32).pin_memory()
    q_dev = torch.empty_like(q)
    from paper_1404_1831_b200.index import SearchResult as _SR

    host_out = _SR(od_h, oi_h, oc_h)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_ms = 0.0
    for s in range(args.steps):
        flush.fill_((s + 7) & 0xFF)
        e0.record(stream)
        if searcher is None and args.e2e_pieces > 1:
            # A/B: the host-to-host call sliced over streams (copies under kernels; measured slower)
            dix.search_host(q_host, L, k, engine, out=host_out, pieces=args.e2e_pieces)
            res = out
        else:
            q_dev.copy_(q_host, non_blocking=True)
            res = (searcher.search(q_dev, L, k, engine, workspace=ws) if searcher is not None
                   else dix.search(q_dev, L, k, engine, out=out, workspace=ws))
            od_h.copy_(res.dists, non_blocking=True)
            oi_h.copy_(res.ids, non_blocking=True)
            oc_h.copy_(res.counts, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms += e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([e2e_ms], device=device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_v = qmul * nq * args.steps / (e2e_ms / 1e3)

    # roofline of the fused traversal+scan kernel, SURVEY §8(d) bytes: (M+4) B per candidate (code + id)
    # + 16 B per popped cell (an offsets pair, empty cells included).  The default FBPQ scan also reads a
    # 4 B point term per candidate (not in the §8(d) numerator; reported separately).
    # the traversal kernel passes + the large-cell stream kernel
    search_ms = float(np.mean(stage_ms[:, 2] + stage_ms[:, 3]))
    pt_bytes = 4 * ncand if engine == "fbpq" and not dix.fbpq_exact else 0
    scan_bytes = (dix.m + 4) * ncand
    cell_bytes = 16 * npop
    alg_bytes = scan_bytes + cell_bytes
    combined = alg_bytes / (search_ms / 1e3) / 1e9
    # the dominant kernel: the large-cell stream (cell_flow_kernel) when it runs longer than the traversal
    # kernel, with its own bytes ((M+4) B per entry it scans) over its own event time; else both kernels
    # over the whole SURVEY 8(d) numerator
    stream_ms = float(np.mean(stage_ms[:, 3]))
    trav_ms = float(np.mean(stage_ms[:, 2]))
    stream_dominant = stream_cand > 0 and stream_ms > trav_ms
    if stream_dominant:
        dom_bytes, dom_ms = (dix.m + 4) * stream_cand, stream_ms
        dom_kernel = "cell_flow_kernel (register-pipelined large-cell stream: score + top-k)"
        dom_formula = f"SURVEY 8(d): {dix.m + 4} B/candidate x {stream_cand:,} entries of the deferred large cells"
    else:
        dom_bytes, dom_ms = alg_bytes, search_ms
        dom_kernel = "search_kernel (traversal + scan + top-k)" + (" + large-cell stream" if stream_cand else "")
        dom_formula = f"SURVEY 8(d): {dix.m + 4} B/candidate + 16 B/popped cell"
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    traffic = None
    try:  # dram bytes per launch of the same kernel from the committed ncu --set full capture
        tr = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())
        traffic = tr.get(workload, {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    line = {
        "metric": metric, "value": value, "unit": "queries/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.shard else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded BASELINE.json generator)",
        "config": config,
        "codes_scanned_per_s": world * ncand * args.steps / (t_ms / 1e3),
        "stage_ms": {"first_layer": float(np.mean(stage_ms[:, 0])), "row_sort_fold": float(np.mean(stage_ms[:, 1])),
                     "traverse_scan_topk": float(np.mean(stage_ms[:, 2])),
                     "large_cell_stream": float(np.mean(stage_ms[:, 3])), "search_total": search_ms},
        "work_per_step": {"candidates": ncand, "popped_cells": npop, "cand_per_query": ncand / nq},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": HBM_PEAK, "unit": "GB/s",
                     "frac": achieved / HBM_PEAK, "traffic": traffic, "kernel": dom_kernel,
                     "kernel_ms": dom_ms, "peak_source": HBM_PEAK_SRC, "alg_bytes_per_launch": dom_bytes,
                     "alg_bytes_formula": dom_formula,
                     "point_term_bytes_per_launch": 4 * stream_cand if stream_dominant else pt_bytes,
                     "frac_incl_point_term": (dom_bytes + (4 * stream_cand if stream_dominant else pt_bytes))
                                             / (dom_ms / 1e3) / 1e9 / HBM_PEAK,
                     # both search kernels (traversal + stream) over the whole 8(d) numerator
                     # the other search kernel when the stream dominates: the traversal kernel with the rest of
                     # the 8(d) numerator (16 B per popped cell + the small cells' candidates)
                     "traversal_kernel": ({"ms": trav_ms, "alg_bytes": alg_bytes - dom_bytes,
                                           "achieved": (alg_bytes - dom_bytes) / (trav_ms / 1e3) / 1e9,
                                           "frac": (alg_bytes - dom_bytes) / (trav_ms / 1e3) / 1e9 / HBM_PEAK}
                                          if stream_dominant else None),
                     "search_kernels_combined": {"ms": search_ms, "alg_bytes": alg_bytes, "scan_bytes": scan_bytes,
                                                 "cell_offset_bytes": cell_bytes, "point_term_bytes": pt_bytes,
                                                 "achieved": combined, "frac": combined / HBM_PEAK}},
        "fbpq_mode": ("exact (reference operation order)" if dix.fbpq_exact else "point term (+4 B/entry)")
                     if engine == "fbpq" else None,
        "e2e": {"value": e2e_v, "unit": "queries/s", "h2d_bytes_per_step": int(q.numel() * 4),
                "d2h_bytes_per_step": int(nq * k * 8 + nq * 4)},
        "gpu_launches": (launches_per_step(dix, engine) + (1 if searcher is not None else 0)) * args.steps,
        "clocks": clk.summary(),
    }
    if PROFILE:
        line["phase_profile"] = PROFILE
    if GT.get("acc") is not None and searcher is None:
        from paper_1404_1831_b200 import evalbench

        n = GT["n"]
        nn, _ = GT["acc"].result()
        r = evalbench.recall_at(res.ids[:n], res.counts[:n], nn)
        line["recall"] = {**{f"R@{c}": v for c, v in r.items()}, "queries": n,
                          "ground_truth": "exact NN of each sampled query over the whole base (int8 tensor-core "
                                          "GEMM on x-128, exact distances; f64 for non-integer data), ties to the "
                                          "smaller id (vecio.brute_force_knn)",
                          "definition": "evalbench.recall_at: true NN among the first c returned ids"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline and host is not None:
        try:
            qnp = q.cpu().numpy()
            block, want, oidx, n = cpu_baseline(host(), engine, qnp, L, k)
            line["cpu_baseline"] = block
            got = (od_h.numpy(), oi_h.numpy().view(np.uint32), oc_h.numpy(), ncand_q)
            line["parity"] = parity_block(got, want, oidx, qnp, L)
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = {"error": repr(e)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1 or args.shard:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
