"""Print the headline numbers and per-phase times of a bench.py JSON line."""
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("ms/step", round(d["ms_per_step"], 4), "value", "%.3e" % d["value"])
print("phases", {k: round(v, 4) for k, v in d.get("phase_ms_per_step", {}).items()})
if d.get("fp32"):
    f = d["fp32"]
    print("fp32 ms/step", round(f["ms_per_step"], 4), {k: round(v, 4) for k, v in f.get("phase_ms_per_step", {}).items()})
if d.get("e2e"):
    print("e2e ms/step", round(d["e2e"]["ms_per_step"], 3))
