"""Aggregate an `ncu --page source --csv --print-source cuda,sass` dump per CUDA source line:
share of warp-stall samples and of executed warp instructions.
usage: python tools/ncu_lines.py dump.csv [top]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file = None
agg = {}
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[0] == "":
        continue
    try:
        s = float(r[4]); ins = float(r[7])
    except ValueError:
        continue
    key = (cur_file, r[0])
    a = agg.setdefault(key, [0.0, 0.0, r[1]])
    a[0] += s; a[1] += ins
ts = sum(v[0] for v in agg.values()); ti = sum(v[1] for v in agg.values())
print(f"total samples {ts:.0f}, warp instructions {ti:.3e}")
for (f, ln), (s, i, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*s/ts:5.1f}% smp {100*i/ti:5.1f}% ins  {f}:{ln}  {src.strip()[:80]}")
