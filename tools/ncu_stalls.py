"""Per-source-line stall breakdown from `ncu --page source --csv --print-source cuda,sass`.
usage: python tools/ncu_stalls.py dump.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur, hdr, agg = None, None, {}
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        idx = {h: i for i, h in enumerate(r) if h.startswith("stall_") and "Not Issued" not in h}
        continue
    if hdr is None or len(r) < 8 or r[0] == "":
        continue
    try:
        s = float(r[4])
    except ValueError:
        continue
    a = agg.setdefault((cur, r[0]), {"_s": 0.0, "_src": r[1]})
    a["_s"] += s
    for h, i in idx.items():
        try:
            a[h] = a.get(h, 0.0) + float(r[i] or 0)
        except ValueError:
            pass
tot = sum(v["_s"] for v in agg.values())
tots = {}
for v in agg.values():
    for k, x in v.items():
        if k.startswith("stall_"):
            tots[k] = tots.get(k, 0) + x
print("totals:", {k[6:]: round(100 * x / tot, 1) for k, x in sorted(tots.items(), key=lambda kv: -kv[1]) if x / tot > 0.01})
for (f, ln), v in sorted(agg.items(), key=lambda kv: -kv[1]["_s"])[:top]:
    parts = sorted(((k[6:], x) for k, x in v.items() if k.startswith("stall_")), key=lambda kv: -kv[1])[:3]
    print(f"{100 * v['_s'] / tot:5.1f}% {f}:{ln} [{', '.join(f'{k} {100 * x / max(v['_s'], 1):.0f}%' for k, x in parts)}] {v['_src'].strip()[:70]}")
