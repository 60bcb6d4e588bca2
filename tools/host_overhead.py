"""Host-side cost per update_packed call (GPU queue kept full): where does the CPU time go?"""
import os, sys, time, cProfile, pstats
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2305_18376_b200 import workloads as wl
from paper_2305_18376_b200.stream import StreamState

K0, J, R = 50000, 128, 16
rng = np.random.default_rng(0)
cfg = wl.scaled(wl.CONFIGS["large"], K0=K0)
H = rng.uniform(size=(R, R)); V = rng.uniform(size=(J, R)); W = rng.uniform(size=(K0, R))
D0 = H.T @ H; vtv = V.T @ V
G = np.einsum("kr,rz,kz->rz", W, D0, W); G = (G + G.T) / 2
arr = {"slice_ids": [f"s{k}" for k in range(K0)], "W": W, "V": V,
       "C": np.einsum("rz,kz,zr->kr", D0, W, vtv), "D": np.broadcast_to(D0, (K0, R, R)).copy(),
       "F": V @ G, "G": G, "forgetting": 0.95}
st = StreamState.from_arrays(arr, device="cuda:0")
batches = []
for t in range(12):
    counts = np.concatenate([rng.integers(1, 9, K0), rng.integers(200, 2001, 500)]).astype(np.int64)
    X = torch.randn((int(counts.sum()), J), dtype=torch.float64, device="cuda") * 0.1
    batches.append((X, counts, np.arange(K0, dtype=np.int32), [f"n{t}_{i}" for i in range(500)]))
for b in batches[:2]:
    st.update_packed(*b)
torch.cuda.synchronize()
t0 = time.perf_counter()
ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
ev0.record()
host = []
for b in batches[2:7]:
    h0 = time.perf_counter()
    st.update_packed(*b)
    host.append(time.perf_counter() - h0)
ev1.record()
torch.cuda.synchronize()
print("host ms per call", [round(1e3 * h, 3) for h in host])
print("gpu ms per update", ev0.elapsed_time(ev1) / 5)
import time as _t
def timed(fn, *a):
    h0 = _t.perf_counter(); r = fn(*a); return r, 1e6 * (_t.perf_counter() - h0)
X, counts, ex, new = batches[7]
_, us = timed(np.cumsum, counts); print("cumsum us", us)
pr = cProfile.Profile()
pr.enable()
for b in batches[7:12]:
    st.update_packed(*b)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
