"""A/B timing of engine environment knobs on one built workload (development
tool): builds bench.py's workload once, then times the batched search under
each setting of an environment variable read per launch.

  python tools/ab_env.py --config c4 --var BPQ_NB0 --values 16 32 64 128
"""

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--var", required=True)
    ap.add_argument("--values", nargs="+", required=True)
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    import torch

    import bench

    cfg = dict(bench.CONFIGS[args.config], name=args.config)
    dev = torch.device("cuda", 0)
    dix, q, _ = bench.build_workload(cfg, dev)
    L, k, eng = cfg["L"], cfg["topk"], cfg["engine"]
    ws = dix.make_workspace(eng, q.shape[0], L, k)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for v in args.values:
        os.environ[args.var] = v
        for _ in range(3):
            dix.search(q, L, k, eng, workspace=ws)
        torch.cuda.synchronize()
        st = []
        for s in range(args.steps):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
            for e in ev:  # torch creates CUDA events lazily on first record
                e.record()
            torch.cuda.synchronize()
            flush.fill_(s & 0xFF)
            dix.search(q, L, k, eng, workspace=ws, stage_events=ev)
            torch.cuda.synchronize()
            st.append([ev[i].elapsed_time(ev[i + 1]) for i in range(4)])
        st = np.array(st).mean(0)
        print(json.dumps({"config": args.config, args.var: v, "stage_ms": [round(x, 4) for x in st],
                          "total_ms": round(float(st.sum()), 4)}), flush=True)


if __name__ == "__main__":
    main()
