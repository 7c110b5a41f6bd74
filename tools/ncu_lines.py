"""Per-CUDA-source-line stall samples from `ncu --page source --csv --print-source cuda,sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cur_file = "?"
hdr = None
items = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        wi = hdr.index("Warp Stall Sampling (All Samples)")
        stall = [(i, c) for i, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
        continue
    if hdr is None or not r or not r[0] or r[0] == "":
        continue
    try:
        v = float(r[wi])
    except (ValueError, IndexError):
        continue
    if v <= 0:
        continue
    top = sorted(((float(r[i] or 0), c[6:]) for i, c in stall), reverse=True)[:3]
    items.append((v, f"{cur_file}:{r[0]}", r[1].strip()[:90], [(c, int(x)) for x, c in top if x]))
tot = sum(x[0] for x in items) or 1
items.sort(key=lambda x: -x[0])
print("total samples", int(tot))
for v, loc, src, top in items[:n]:
    print(f"{v/tot*100:5.1f}% {loc:22s} {src:90s} {top}")
