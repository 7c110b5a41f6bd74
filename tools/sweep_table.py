"""Markdown tables from tools/sweep.py outputs: python tools/sweep_table.py DIR"""
import json, os, sys
d = sys.argv[1]
rows = {}
for n in (1, 2, 4, 8):
    f = os.path.join(d, f"sweep_n{n}.jsonl")
    if not os.path.exists(f):
        continue
    for line in open(f):
        r = json.loads(line)
        rows.setdefault((r["config"], r["model"], r["m"], r["rho"], r["k"]), {})[n] = r
ns = sorted({n for v in rows.values() for n in v})
print("| cfg | model | m | ρ | k | " + " | ".join(f"pipeline ms N={n}" for n in ns) + " | 12·m / step, GB/s (N=1) |")
print("|---|---|---|---|---|" + "---|" * len(ns) + "---|")
for key in sorted(rows):
    v = rows[key]
    if key[0] == 1:
        continue
    cells = [f"{v[n]['pipeline_ms']:.4f}" if n in v and v[n].get("pipeline_ms") else "—" for n in ns]
    gbs = v.get(1, {}).get("select_gbs_12m")
    print(f"| {key[0]} | {key[1]} | {key[2]:,} | {key[3]} | {key[4]:,} | " + " | ".join(cells) + f" | {gbs or '—'} |")
print()
print("| cfg | model | m | k | N | gtopk_step ms | topk_step ms | dense_step ms |")
print("|---|---|---|---|---|---|---|---|")
for key in sorted(rows):
    for n, r in sorted(rows[key].items()):
        a = r.get("api_ms", {})
        if key[0] in (1, 3, 4):
            print(f"| {key[0]} | {key[1]} | {key[2]:,} | {key[4]:,} | {r.get('P', n) if key[0] != 1 else '4 (in-process)'} | "
                  f"{a.get('gtopk_step', '—')} | {a.get('topk_step', '—')} | {a.get('dense_step', '—')} |")
