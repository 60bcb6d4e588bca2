"""Summarise an ncu --csv launch list (gpu__time_duration.sum): one update's
kernels (the `which`-th update, counted by k_plan_count launches)."""
import csv, re, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
which = int(sys.argv[2]) if len(sys.argv) > 2 else 3
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
ks = []
for r in rows[1:]:
    name = re.sub(r"^<unnamed>::", "", r[ki].split("(")[0])
    name = re.sub(r"^void <unnamed>::", "", name)
    ks.append((name, float(r[vi].replace(",", "")) / 1000.0))
idx = [i for i, (k, _) in enumerate(ks) if k.startswith("k_plan_count")]
a = idx[which]
b = idx[which + 1] if which + 1 < len(idx) else len(ks)
tot = sum(v for _, v in ks[a:b])
print("| kernel | us | share |\n|---|---|---|")
for k, v in ks[a:b]:
    print(f"| `{k}` | {v:.1f} | {100 * v / tot:.1f}% |")
print(f"| **sum** | **{tot:.1f}** | |")
