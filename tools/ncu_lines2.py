"""Per-source-line stall samples from an ncu report (cuda,sass source view):
python tools/ncu_lines2.py report.ncu-rep [n]"""
import csv, subprocess, sys, io
from collections import defaultdict
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = defaultdict(float); src = {}; stall = defaultdict(lambda: defaultdict(float)); f = None; h = None
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        h = r; cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]; continue
    if h and len(r) > 4:
        try:
            v = float(r[4])
        except ValueError:
            continue
        key = (f, r[0]); agg[key] += v
        for i, c in cols:
            try:
                stall[key][c[6:]] += float(r[i] or 0)
            except ValueError:
                pass
        if r[1].strip():
            src[key] = r[1].strip()[:90]
tot = sum(agg.values()) or 1
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:n]:
    top = sorted(stall[k].items(), key=lambda x: -x[1])[:2]
    print(f"{v / tot * 100:5.1f}% {k[0]}:{k[1]:>4} {src.get(k, ''):90s} {[(a, int(b)) for a, b in top if b]}")
