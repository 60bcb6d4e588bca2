"""FP64 vs FP32 data mode: host enqueue time and device time per update_packed
(large config shapes, random data)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2305_18376_b200.stream import StreamState

K0, J, R = 50000, 128, 16
rng = np.random.default_rng(0)
H = rng.uniform(size=(R, R)); V = rng.uniform(size=(J, R)); W = rng.uniform(size=(K0, R))
D0 = H.T @ H; vtv = V.T @ V
G = np.einsum("kr,rz,kz->rz", W, D0, W); G = (G + G.T) / 2
arr = {"slice_ids": [f"s{k}" for k in range(K0)], "W": W, "V": V,
       "C": np.einsum("rz,kz,zr->kr", D0, W, vtv), "D": np.broadcast_to(D0, (K0, R, R)).copy(),
       "F": V @ G, "G": G, "forgetting": 0.95}
batches = []
for t in range(10):
    counts = np.concatenate([rng.integers(1, 9, K0), rng.integers(200, 2001, 500)]).astype(np.int64)
    X = torch.randn((int(counts.sum()), J), dtype=torch.float64, device="cuda") * 0.1
    batches.append((X, counts, np.arange(K0, dtype=np.int32), [f"n{t}_{i}" for i in range(500)]))
for dt in (torch.float64, torch.float32, torch.float64, torch.float32):
    st = StreamState.from_arrays(arr, device="cuda:0", dtype=dt)
    bs = [(b[0].to(dt),) + b[1:] for b in batches]
    for b in bs[:3]:
        st.update_packed(*b)
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    host = []
    for b in bs[3:]:
        h0 = time.perf_counter()
        st.update_packed(*b)
        host.append(time.perf_counter() - h0)
    ev1.record()
    torch.cuda.synchronize()
    print(dt, "host ms/call", [round(1e3 * h, 3) for h in host], "gpu ms/update", ev0.elapsed_time(ev1) / len(host))
    # one update alone (queue drained first)
    for b in bs[3:6]:
        torch.cuda.synchronize()
        ev0.record(); st.update_packed(*b); ev1.record(); torch.cuda.synchronize()
        print("   isolated update ms", ev0.elapsed_time(ev1))
