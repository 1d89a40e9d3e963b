"""Per CUDA source line: executed warp instructions, stall samples and the
FP64 share, from an .ncu-rep (`--page source --print-source cuda,sass`).
    python tools/src_lines.py REP [top]   (dev aid)"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    agg = defaultdict(lambda: [0, 0, 0, ""])  # instr, stalls, fp64 instr, text
    cur = None
    fname = "?"
    hdr = None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or len(r) < 8:
            continue
        if r[0]:  # a CUDA line row
            cur = (fname, int(r[0]))
            agg[cur][3] = r[1].strip()[:90]
            continue
        if cur is None:
            continue
        try:
            e = int(r[7] or 0)
            w = int(r[4] or 0)
        except ValueError:
            continue
        op = r[3].split()
        op = (op[1] if op and op[0].startswith("@") else (op[0] if op else "")).split(".")[0]
        agg[cur][0] += e
        agg[cur][1] += w
        if op in ("DADD", "DMUL", "DFMA", "DSETP", "DMNMX"):
            agg[cur][2] += e
    te = sum(v[0] for v in agg.values()) or 1
    tw = sum(v[1] for v in agg.values()) or 1
    print(f"# {rep}: {te} warp instructions, {tw} stall samples")
    print(f"{'instr%':>7s} {'stall%':>7s} {'fp64%':>6s}  line")
    for (f, l), (e, w, d, t) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * e / te:7.2f} {100 * w / tw:7.2f} {100 * d / max(e, 1):6.1f}  {f}:{l}: {t}")


if __name__ == "__main__":
    main()
