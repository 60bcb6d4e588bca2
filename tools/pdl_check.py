"""Run a few large-shaped updates and print a digest of the resulting state
(used by tests/test_gpu_pdl.py to compare PDL on/off and repeated runs)."""
import hashlib
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2305_18376_b200.stream import StreamState


def main(K0=20000, J=128, R=16, steps=4, n_new=300):
    rng = np.random.default_rng(7)
    H = rng.uniform(size=(R, R))
    V = rng.uniform(size=(J, R))
    W = rng.uniform(size=(K0, R))
    D0 = H.T @ H
    vtv = V.T @ V
    G = np.einsum("kr,rz,kz->rz", W, D0, W)
    G = (G + G.T) / 2
    arr = {"slice_ids": [f"s{k}" for k in range(K0)], "W": W, "V": V,
           "C": np.einsum("rz,kz,zr->kr", D0, W, vtv), "D": np.broadcast_to(D0, (K0, R, R)).copy(),
           "F": V @ G, "G": G, "forgetting": 0.95}
    st = StreamState.from_arrays(arr, device="cuda:0")
    gen = torch.Generator(device="cuda")
    gen.manual_seed(11)
    h = hashlib.sha256()
    K = K0
    # "async": no host sync between updates (the results are read after the last one), so update
    # t+1 is issued -- and its device plan runs on the staging side stream -- while update t executes
    defer = "async" in sys.argv[1:]
    batches, kept = [], []
    for t in range(steps):
        counts = np.concatenate([rng.integers(1, 9, K), rng.integers(65, 1500, n_new)]).astype(np.int64)
        X = torch.randn((int(counts.sum()), J), generator=gen, dtype=torch.float64, device="cuda") * 0.1
        batches.append((X, counts, np.arange(K, dtype=np.int32), [f"n{t}_{i}" for i in range(n_new)]))
        K += n_new
    torch.cuda.synchronize()
    for X, counts, ex, new in batches:
        U, vu = st.update_packed(X, counts, ex, new)
        if defer:
            kept.append((U, vu))
        else:
            h.update(U.cpu().numpy().tobytes())
            h.update(vu.cpu().numpy().tobytes())
    for U, vu in kept:
        h.update(U.cpu().numpy().tobytes())
        h.update(vu.cpu().numpy().tobytes())
    st.check()
    for name in ("W", "C", "D", "F", "G", "V"):
        h.update(np.ascontiguousarray(getattr(st, name)).tobytes())
    print(h.hexdigest())


if __name__ == "__main__":
    main()
