"""local_error of one large-shaped update (device-resident), for ncu launch lists."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2305_18376_b200.stream import StreamState
from paper_2305_18376_b200.evaluate import local_error_device
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
U, vu = st.update_packed(X, counts, np.arange(K0, dtype=np.int32), [f"n{i}" for i in range(L)])
_, _, meta, Xl, Nl, Ul = st._last
for _ in range(3):
    se, te = local_error_device(Xl, Nl, meta.host_row_ptr().copy(), meta[1], Ul, st, row_ptr_dev=meta[0])
torch.cuda.synchronize()
print(float(te))
