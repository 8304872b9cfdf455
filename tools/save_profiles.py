"""Copy one gpurun pass (tools/gpu_final.sh TAG) from gpurun_out/ into profiles/: bench lines, test logs,
launch lists of the last four search steps, ncu summaries and DRAM traffic of the stream kernel."""
import collections
import csv
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
G, P = ROOT / "gpurun_out", ROOT / "profiles"
tag = sys.argv[1]
for src, dst in (("c1.json", "r2_bench_c1.json"), ("ref.json", "r2_bench_c1_reference_arm.json"),
                 ("c4.json", "r2_bench_c4.json"), ("tests.log", "r2_gpu_tests.log"), ("smoke.log", "r2_smoke.log"),
                 ("c4_prof.json", "r2_c4_phase_profile.json"), ("c1_prof.json", "r2_c1_phase_profile.json")):
    if (G / f"{tag}_{src}").exists():
        shutil.copy(G / f"{tag}_{src}", P / dst)
if (G / "reference_suites_on_cuda.log").exists():
    shutil.copy(G / "reference_suites_on_cuda.log", P / "r2_reference_suites_on_cuda.log")
traffic = json.loads((P / "ncu_traffic.json").read_text())
for cfg in ("c1", "c4"):
    f = G / f"{tag}_{cfg}_launches.csv"
    if f.exists():
        rows = list(csv.DictReader(l for l in open(f) if l.startswith('"')))[-28:]
        agg = collections.OrderedDict()
        for r in rows:
            n = r["Kernel Name"].split("(")[0]
            a = agg.setdefault(n, [0, 0.0])
            a[0] += 1
            a[1] += float(r["Metric Value"])
        tot = sum(t for _, t in agg.values())
        with open(P / f"r2_{cfg}_launches.txt", "w") as o:
            o.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none -k regex:<search-step kernels> -c 80: "
                    f"python bench.py --config {cfg} --steps 2 --warmup 3 --no-cpu-baseline --recall-queries 0\n")
            o.write("# the last four search steps (7 launches each): launches, total us, mean us, share (cold-cache, "
                    "serialised under ncu; compare the SHARE with bench.py's stage_ms)\n")
            for n, (c, t) in agg.items():
                o.write(f"{c:5d} {t / 1e3:12.1f} {t / 1e3 / c:10.1f} {100 * t / tot:6.1f}%  {n}\n")
            o.write("\n# in launch order (two steps)\n")
            for r in rows[-14:]:
                o.write(f'{float(r["Metric Value"]) / 1e3:10.1f} us  grid {r["Grid Size"]} block {r["Block Size"]}  '
                        f'{r["Kernel Name"].split("(")[0]}\n')
    rep = G / f"{tag}_{cfg}_flow.ncu-rep"
    if rep.exists():
        out = subprocess.run([sys.executable, str(P / "ncu_hot.py"), str(rep), "20"], capture_output=True, text=True)
        (P / f"r2_{cfg}_cell_flow_ncu_summary.txt").write_text(out.stdout + out.stderr)
        raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rr = list(csv.reader(raw.splitlines()))
        h = rr[0]
        val = {c: (rr[1][i], float(rr[2][i])) for i, c in enumerate(h)
               if c in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")}
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
        rd = val["dram__bytes_read.sum"][1] * scale[val["dram__bytes_read.sum"][0]]
        wr = val["dram__bytes_write.sum"][1] * scale[val["dram__bytes_write.sum"][0]]
        for k, v in traffic.items():
            if k.startswith(cfg + ":"):
                v["dram_bytes_per_launch"] = rd + wr
                v["source"] = (f"profiles/r2_{cfg}_cell_flow_ncu_summary.txt (ncu --set full --clock-control none, one "
                               f"launch, gpurun_out/{tag}_{cfg}_flow.ncu-rep): dram__bytes_read.sum {rd / 1e9:.3f} GB + "
                               f"dram__bytes_write.sum {wr / 1e6:.1f} MB")
        print(cfg, "dram GB", (rd + wr) / 1e9, val["gpu__time_duration.sum"])
(P / "ncu_traffic.json").write_text(json.dumps(traffic, indent=1) + "\n")
for f in ("c1.json", "c4.json", "ref.json"):
    p = G / f"{tag}_{f}"
    if p.exists():
        d = json.loads(p.read_text().strip().splitlines()[-1])
        print(f, round(d["value"]), round(d["e2e"]["value"]), d.get("ms_per_step"),
              {k: round(v, 3) for k, v in d.get("stage_ms", {}).items()}, d.get("roofline", {}).get("frac"),
              d.get("parity", {}).get("unclassified"))
