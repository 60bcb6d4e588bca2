"""Phase timing of one DASH update on controlled batch shapes (GPU)."""
import ctypes, sys, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2305_18376_b200 import _native as nat, workloads as wl
from paper_2305_18376_b200.stream import StreamState

def run(K0, J, R, rows_existing, n_new, rows_new, reps=5):
    cfg = wl.scaled(wl.CONFIGS["large"], K0=K0, J=J, R=R)
    rng = np.random.default_rng(0)
    H = rng.uniform(size=(R, R)); V = rng.uniform(size=(J, R)); W = rng.uniform(size=(K0, R))
    D0 = H.T @ H; vtv = V.T @ V
    G = np.einsum("kr,rz,kz->rz", W, D0, W); G = (G + G.T) / 2
    arr = {"slice_ids": [f"s{k}" for k in range(K0)], "W": W, "V": V,
           "C": np.einsum("rz,kz,zr->kr", D0, W, vtv), "D": np.broadcast_to(D0, (K0, R, R)).copy(),
           "F": V @ G, "G": G, "forgetting": 0.95}
    st = StreamState.from_arrays(arr, device="cuda:0")
    L = nat.lib()
    out = []
    for rep in range(reps):
        counts = np.concatenate([np.full(K0 if rows_existing else 0, rows_existing), np.full(n_new, rows_new)]).astype(np.int64)
        N = int(counts.sum())
        X = torch.randn((N, J), dtype=torch.float64, device="cuda") * 0.1
        ex = np.arange(K0 if rows_existing else 0, dtype=np.int32)
        new = [f"n{rep}_{i}" for i in range(n_new)]
        torch.cuda.synchronize()
        L.dash_ctx_set_profiling(st._ctx, 1)
        st.update_packed(X, counts, ex, new)
        ms = (ctypes.c_double * 8)(); cnt = (ctypes.c_int32 * 8)()
        L.dash_ctx_phase_ms(st._ctx, ms, cnt, 8)
        if rep >= 1:
            out.append({nat.PHASES[i]: ms[i] for i in range(len(nat.PHASES)) if cnt[i]})
    avg = {k: float(np.mean([o[k] for o in out])) for k in out[0]}
    return avg

if __name__ == "__main__":
    cases = {
        "small_only_50k_x4.5": (50000, 128, 16, 4, 0, 0),
        "small_only_50k_x1": (50000, 128, 16, 1, 0, 0),
        "big_only_500_x1100": (1000, 128, 16, 0, 500, 1100),
        "big_only_2000_x275": (1000, 128, 16, 0, 2000, 275),
        "large_like": (50000, 128, 16, 4, 500, 1100),
    }
    for name, c in cases.items():
        print(name, json.dumps({k: round(v, 4) for k, v in run(*c).items()}), flush=True)
