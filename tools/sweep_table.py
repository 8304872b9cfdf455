"""profiles/r2_sweep.txt from a tools/sweep_r2.sh run: python tools/sweep_table.py gpurun_out/<tag>.jsonl"""
import json
import shutil
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
src = Path(sys.argv[1])
shutil.copy(src, ROOT / "profiles" / "r2_sweep.jsonl")
out = open(ROOT / "profiles" / "r2_sweep.txt", "w")
out.write("# tools/sweep_r2.sh on one B200 (bench.py --steps 5 --warmup 3): every BASELINE config, parity block = C "
          "oracle on the same index and queries\n")
out.write("# frac = roofline.frac of the dominant kernel (cell_flow_kernel alone when the stream dominates); comb = "
          "both search kernels over the whole SURVEY 8(d) numerator\n")
out.write(f'{"workload":74s} {"Mq/s":>6s} {"e2e":>6s} {"ms":>6s}  first sort trav stream | frac  comb | cpu q/s | '
          f'exact neartie bndry uncls | R@100\n')
for line in open(src):
    line = line.strip()
    if not line:
        continue
    d = json.loads(line)
    c, r, p, cb, st = d["config"], d["roofline"], d.get("parity"), d.get("cpu_baseline", {}), d["stage_ms"]
    mode = " exact" if (d.get("fbpq_mode") or "").startswith("exact") else ""
    par = (f'{p["exact_lists"]:5d} {p["near_tie_distance"]:5d} {p["near_tie_boundary"]:3d} {p["unclassified"]:3d}'
           if p else "    -     -   -   -")
    out.write(f'{c["workload"] + mode:74s} {d["value"] / 1e6:6.2f} {d["e2e"]["value"] / 1e6:6.2f} '
              f'{d["ms_per_step"]:6.2f}  {st["first_layer"]:.2f} {st["row_sort_fold"]:.2f} '
              f'{st["traverse_scan_topk"]:.2f} {st["large_cell_stream"]:.2f} | {r["frac"]:.3f} '
              f'{r["search_kernels_combined"]["frac"]:.3f} | {cb.get("value", 0):7.0f} | {par} | '
              f'{d.get("recall", {}).get("R@100", "-")}\n')
out.close()
print(open(ROOT / "profiles" / "r2_sweep.txt").read())
