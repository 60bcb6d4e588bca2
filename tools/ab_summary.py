"""Summarise tools/ab_s3.sh logs: ms/update and the small-slice phase per arm."""
import glob, json, re
for f in sorted(glob.glob("gpurun_out/ab_*.log")):
    lines = [l for l in open(f) if l.startswith("{")]
    if not lines:
        print(f, "no JSON"); continue
    d = json.loads(lines[-1])
    ph = d["phase_ms_per_step"]
    print(f"{f:32s} ms/update {d['ms_per_step']:.4f}  slices {ph.get('slices', 0)*1e3:.1f} us  big {ph.get('big', 0)*1e3:.1f} us  fallbacks {d.get('lu_fallbacks')}")
