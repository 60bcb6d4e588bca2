"""Where the host time of one StreamState.update_packed goes (large config,
GPU idle before each call): cProfile of 20 calls, sorted by own time."""
import cProfile, pstats, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2305_18376_b200.stream import StreamState

K0, J, R, L = 50000, 128, 16, 500
rng = np.random.default_rng(0)
H = rng.uniform(size=(R, R)); V = rng.uniform(size=(J, R)); W = rng.uniform(size=(K0, R))
D0 = H.T @ H; vtv = V.T @ V
G = np.einsum("kr,rz,kz->rz", W, D0, W); G = (G + G.T) / 2
arr = {"slice_ids": [f"s{k}" for k in range(K0)], "W": W, "V": V,
       "C": np.einsum("rz,kz,zr->kr", D0, W, vtv), "D": np.broadcast_to(D0, (K0, R, R)).copy(),
       "F": V @ G, "G": G, "forgetting": 0.95}
st = StreamState.from_arrays(arr, device="cuda:0")
counts = np.concatenate([rng.integers(1, 9, K0), rng.integers(200, 2001, L)]).astype(np.int64)
X = torch.randn((int(counts.sum()), J), dtype=torch.float64, device="cuda") * 0.1
ex = np.arange(K0, dtype=np.int32)
times = []
for it in range(30):
    new = [f"n{it}_{i}" for i in range(L)]
    torch.cuda.synchronize()
    t = time.perf_counter()
    st.update_packed(X, counts, ex, new)
    times.append(time.perf_counter() - t)
print("host us per update_packed (GPU idle), median:", round(1e6 * float(np.median(times[5:])), 1))
pr = cProfile.Profile()
for it in range(30, 50):
    new = [f"n{it}_{i}" for i in range(L)]
    torch.cuda.synchronize()
    pr.enable()
    st.update_packed(X, counts, ex, new)
    pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(16)
