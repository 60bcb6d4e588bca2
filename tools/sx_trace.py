"""Timeline of k_smallx per unit from a -DDASH_SX_TRACE build (DASH_LIB_PATH).
Events: 0 XV load issued, 1 F load issued, 2 math XV start, 3 math U done,
5 solver start (first warp with pairs), 6 solver done (same warp), 7 math F done."""
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
lib.dash_sx_trace(buf2, -1)
b = np.frombuffer(buf2, dtype=np.int64)[:64 * 8].reshape(64, 8).astype(float)
print("math warp 0 of CTA 0, XV step: cycles full->dmma done | ->meta ready | ->ridge | ->Y,C | ->sfree | ->end")
for u in range(30):
    print(u, " ".join(f"{x:7.0f}" for x in np.diff(b[u, :7])))
c = np.frombuffer(buf2, dtype=np.int64)[512:512 + 64].reshape(16, 4)
print("solver warps of CTA 0: busy cycles in pairs, pairs, total cycles")
for ws in range(16):
    if c[ws, 2]:
        print(ws, c[ws, 0], c[ws, 1], c[ws, 2], f"busy {c[ws,0]/c[ws,2]:.2f}  per pair {c[ws,0]/max(c[ws,1],1):.0f}")
e = np.frombuffer(buf2, dtype=np.int64)[1024:1024 + 16 * 16].reshape(16, 16).astype(float)
print("solver warp 0, CTA 0, per pair: cycles of meta+state | wait+nmax | fast test | exact? | rows | D upd | D store | sh2+B | gj | fallback? | W/US")
for k in range(16):
    if e[k, 0]:
        print(k, " ".join(f"{x:6.0f}" for x in np.diff(e[k, :11])))
