"""Aggregate ncu --page source --csv --print-source cuda stall samples per source line."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hi = next(i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r)
h = rows[hi]
wi = h.index("Warp Stall Sampling (All Samples)")
si = h.index("Source") if "Source" in h else 1
stall_cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
items = []
for r in rows[hi + 1:]:
    if len(r) <= wi:
        continue
    try:
        v = float(r[wi])
    except ValueError:
        continue
    top = sorted(((float(r[i] or 0), c) for i, c in stall_cols), reverse=True)[:2]
    items.append((v, r[0], r[si].strip()[:100], top))
tot = sum(v for v, *_ in items) or 1
items.sort(key=lambda x: -x[0])
print("total samples", tot)
for v, a, s, top in items[:n]:
    print(f"{v/tot*100:5.1f}% L{a:>5} {s:100s} {[(c[6:], int(x)) for x, c in top if x]}")
