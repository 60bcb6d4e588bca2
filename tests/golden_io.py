"""Helpers that turn the golden .npz fixtures back into batches and states."""
from pathlib import Path

import numpy as np

from paper_2305_18376_b200.tensor import NewSlice, UpdateBatch

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name):
    return dict(np.load(GOLDEN / name, allow_pickle=False))


def batch_from(g, prefix, t):
    X = g[f"{prefix}b{t}_X"]
    ids = [str(s) for s in g[f"{prefix}b{t}_ids"]]
    counts = g[f"{prefix}b{t}_counts"]
    new = g[f"{prefix}b{t}_new"]
    existing, fresh = {}, []
    off = 0
    for sid, n, is_new in zip(ids, counts, new):
        rows = X[off: off + n]
        off += n
        if is_new:
            fresh.append(NewSlice(sid, rows, t + 1))
        else:
            existing[sid] = rows
    return UpdateBatch(t + 1, existing, fresh, (t + 1, t + 1))


def batches_from(g, prefix=""):
    return [batch_from(g, prefix, t) for t in range(int(g[f"{prefix}n_updates"]))]


def planted_arrays(g, prefix):
    return {k: g[f"{prefix}init_{k}"] for k in ("W", "V", "C", "D", "F", "G")} | {
        "slice_ids": [str(s) for s in g[f"{prefix}init_ids"]],
        "forgetting": float(g[f"{prefix}forgetting"]),
    }


def rel(a, b):
    """Normwise relative max-abs difference max|a-b| / max|b|."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    if a.shape != b.shape:
        raise AssertionError(f"shape {a.shape} != {b.shape}")
    den = max(float(np.abs(b).max()) if b.size else 0.0, 1e-300)
    return float(np.abs(a - b).max()) / den if b.size else 0.0
