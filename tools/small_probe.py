"""Where a small update's time goes (medium / daily shapes): timed-loop latency,
host-only cost per update_packed call (GPU idle), and the library's own
host-side breakdown (DASH_HOST_TIMING=1 prints it).
usage: python tools/small_probe.py medium|daily [updates]"""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2305_18376_b200 import workloads as wl
from paper_2305_18376_b200.stream import StreamState

name = sys.argv[1] if len(sys.argv) > 1 else "medium"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 60
cfg = wl.CONFIGS[name]
K0, J, R = cfg.K0, cfg.J, cfg.R
rng = np.random.default_rng(0)
H = rng.uniform(size=(R, R)); V = rng.uniform(size=(J, R)); W = rng.uniform(size=(K0, R))
D0 = H.T @ H; vtv = V.T @ V
G = np.einsum("kr,rz,kz->rz", W, D0, W); G = (G + G.T) / 2
arr = {"slice_ids": [f"s{k}" for k in range(K0)], "W": W, "V": V,
       "C": np.einsum("rz,kz,zr->kr", D0, W, vtv), "D": np.broadcast_to(D0, (K0, R, R)).copy(),
       "F": V @ G, "G": G, "forgetting": cfg.forgetting}
st = StreamState.from_arrays(arr, device="cuda:0")
if name == "medium":
    mk = lambda: np.concatenate([rng.integers(1, 11, K0), rng.integers(100, 501, 10)]).astype(np.int64)
    L = 10
else:
    mk = lambda: np.concatenate([np.ones(K0, np.int64), rng.integers(1, 51, 3)]).astype(np.int64)
    L = 3
batches = []
for t in range(T):
    c = mk()
    batches.append((torch.randn((int(c.sum()), J), dtype=torch.float64, device="cuda") * 0.1, c,
                    [f"n{t}_{i}" for i in range(L)]))
ex = np.arange(K0, dtype=np.int32)
st.reserve_u_history(sum(int(b[1].sum()) for b in batches) * 3)
for X, c, new in batches[:10]:
    st.update_packed(X, c, ex, new)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 0
e0.record()
for X, c, new in batches[10:T // 2]:
    st.update_packed(X, c, ex, new); n += 1
e1.record(); torch.cuda.synchronize()
print(f"{name}: timed loop {1e3 * e0.elapsed_time(e1) / n:.1f} us / update ({st.last_launches} launches)")
ts = []
for X, c, new in batches[T // 2:]:
    torch.cuda.synchronize()
    t = time.perf_counter()
    st.update_packed(X, c, ex, new)
    ts.append(time.perf_counter() - t)
print(f"{name}: host-only {1e6 * float(np.median(ts)):.1f} us / update_packed call (GPU idle)")
