"""Timeline of k_smallx per unit from a -DDASH_SX_TRACE build (DASH_LIB_PATH).
Events: 0 XV load issued, 1 F load issued, 2 math XV start, 3 math U done,
4 solver prep done, 5 solver solve start, 6 solver done, 7 math F done."""
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import runpy  # noqa: E402

sys.argv = ["prof_update.py", "large", "1"]
runpy.run_path(str(ROOT / "tools" / "prof_update.py"), run_name="__main__")
from paper_2305_18376_b200 import _native as nat  # noqa: E402
lib = nat.load_library()
buf = (ctypes.c_longlong * (148 * 64 * 8))()
lib.dash_sx_trace.restype = ctypes.c_int
print("rc", lib.dash_sx_trace(buf, 148 * 64 * 8))
a = np.frombuffer(buf, dtype=np.int64).reshape(148, 64, 8).astype(float)
for cta in (0, 70):
    t0 = a[cta, 0, 0]
    print(f"CTA {cta} (cycles relative to first XV load issue)")
    for u in range(0, 40):
        row = a[cta, u] - t0
        if a[cta, u, 0] == 0:
            break
        print(u, " ".join(f"{x:9.0f}" for x in row))
buf2 = (ctypes.c_longlong * (64 * 8 * 8))()
print("rc2", lib.dash_sx_trace(buf2, -1))
b = np.frombuffer(buf2, dtype=np.int64).reshape(64, 8, 8).astype(float)
print("solver warp 0 of CTA 0: per pair, cycles between events "
      "(0 top, 1 rows done, 2 D upd, 3 next-state issued, 4 B built, 5 gj done, 6 stores+US done, 7 end)")
for uu in range(8):
    for k in range(8):
        row = b[uu, k]
        if row[0] == 0:
            continue
        print(uu, k, " ".join(f"{x:7.0f}" for x in np.diff(row)), f" total {row[7]-row[0]:.0f}")
