import ctypes, sys
sys.path.insert(0,'.')
import numpy as np, torch
from pathlib import Path
from paper_2305_18376_b200 import _native as nat
lib = nat.load_library(Path('tools/libdash_dbg.so'))
nat._lib = lib
lib.dash_debug_timing.argtypes=[ctypes.c_void_p, ctypes.c_int]
import tools.slice_bench as sb
for case in [(50000,128,16,1,0,0),(1000,128,16,0,500,1100)]:
    sb.run(*case, reps=2)
    buf=(ctypes.c_longlong*(8192*8))()
    lib.dash_debug_timing(buf, 8192*8)
    a=np.frombuffer(buf,dtype=np.int64).reshape(8192,8)
    n=3125 if case[3] else 500
    a=a[:n].astype(np.float64)
    d=np.diff(a,axis=1)
    print(case, "per-CTA cycles median", np.median(a[:,7]-a[:,0]), "phases(0->1,1->2,...) median", np.median(d,axis=0).round(0), flush=True)
