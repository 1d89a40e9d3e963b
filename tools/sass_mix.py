"""Instruction mix of one kernel in an .ncu-rep (dev aid): per SASS opcode the
executed warp instructions, stall samples and average active threads, from
`ncu -i REP --page source --csv --print-source sass`.
    python tools/sass_mix.py REP [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = raw.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    hdr = rows[0]
    si, ei = hdr.index("Source"), hdr.index("Instructions Executed")
    wi = hdr.index("Warp Stall Sampling (All Samples)")
    ti = hdr.index("Thread Instructions Executed")
    agg = defaultdict(lambda: [0, 0, 0])
    for r in rows[1:]:
        if len(r) <= max(si, ei, wi, ti):
            continue
        op = r[si].split()
        if not op:
            continue
        name = op[0] if not op[0].startswith("@") else op[1]
        name = name.split(".")[0]
        try:
            agg[name][0] += int(r[ei] or 0)
            agg[name][1] += int(r[wi] or 0)
            agg[name][2] += int(r[ti] or 0)
        except ValueError:
            continue
    tot_e = sum(v[0] for v in agg.values()) or 1
    tot_w = sum(v[1] for v in agg.values()) or 1
    print(f"# {rep}: {tot_e} warp instructions, {tot_w} stall samples")
    print(f"{'opcode':10s} {'instr%':>7s} {'stall%':>7s} {'thr/warp':>8s}")
    for k, (e, w, t) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{k:10s} {100 * e / tot_e:7.2f} {100 * w / tot_w:7.2f} {t / max(e, 1):8.1f}")


if __name__ == "__main__":
    main()
