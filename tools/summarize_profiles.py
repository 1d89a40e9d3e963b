"""Turn gpurun_out/ ncu captures into committed summaries under profiles/.

  python tools/summarize_profiles.py <round-tag> [traffic-key]
writes profiles/<tag>_launches.txt (per-kernel launch count, device time and
share of the step from the launch list), profiles/<tag>_top_kernel.txt (key
metrics of the --set full capture) and updates profiles/traffic.json with the
dominant kernel's DRAM bytes per launch (read by bench.py)."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def launches(tag):
    path = os.path.join(OUT, "launches.csv")
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    unit = None
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else unit
    total = sum(v for _, v in agg.values())
    lines = [f"# launch list of `python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1` under",
             f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare SHARES)",
             f"{'kernel':70s} {'launches':>8s} {'total_' + (unit or ''):>14s} {'share':>7s}"]
    for name, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{name[:70]:70s} {n:8d} {v:14.1f} {100 * v / total:6.2f}%")
    open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def top_kernel(tag, key):
    rep = os.path.join(OUT, "top_kernel.ncu-rep")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rep], capture_output=True,
                         text=True).stdout
    open(os.path.join(PROF, f"{tag}_top_kernel.txt"), "w").write(out)
    print(out)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    r = rows[2]
    rd = float(r[hdr.index("dram__bytes_read.sum")].replace(",", ""))
    wr = float(r[hdr.index("dram__bytes_write.sum")].replace(",", ""))
    unit = rows[1][hdr.index("dram__bytes_read.sum")]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    tpath = os.path.join(PROF, "traffic.json")
    table = json.load(open(tpath)) if os.path.exists(tpath) else {}
    table[key] = (rd + wr) * scale
    json.dump(table, open(tpath, "w"), indent=1)
    print("traffic", key, table[key])


if __name__ == "__main__":
    tag = sys.argv[1]
    key = sys.argv[2] if len(sys.argv) > 2 else "heat-swept-w1024"
    launches(tag)
    top_kernel(tag, key)
