"""Seeded synthetic streams shaped like BASELINE.json's configs.

The paper's datasets (US/KR Stock, VicRoads, PEMS) are not available, so the
benchmark and parity streams come from the planted low-rank-plus-noise
generator BASELINE.json describes:

    H ~ U[0,1]^{RxR}, V ~ U[0,1]^{JxR}, per slice w_k ~ U[0,1]^R,
    X_k = Q_k H diag(w_k) V^T + sigma * N(0,1),  sigma = 0.1,
    Q_k = first I_k rows of QR(N(0,1)^{max(I_k,R) x R})

Each slice is generated at its final length and revealed over time, so rows
appended by later updates share the slice's basis.  ``exact=False`` replaces
the per-slice QR by i.i.d. N(0, 1/I_k) rows (same scale, no QR), which is what
the large/wide streams use: their initial tensors (56 / 47 GB FP64) are never
materialised -- the initial stream state is *planted* in closed form from the
true factors (``planted_state``), which is legitimate because the update step
never reads old rows (stream.py:1-13 of the reference).

Only host numpy here; bench.py draws its large batches on the device with the
same shapes and distributions.
"""
from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from .tensor import IrregularTensor, NewSlice, SliceMatrix, UpdateBatch


@dataclass(frozen=True)
class StreamConfig:
    name: str
    K0: int
    J: int
    R: int
    init_rows: tuple        # ("uniform", lo, hi) or ("loguniform", lo, hi)
    add_rows: tuple         # ("uniform", lo, hi) per active slice per update
    new_slices: tuple       # ("fixed", n) or ("uniform", lo, hi)
    new_rows: tuple         # row-count law of a new slice
    forgetting: float
    steps: int
    seed: int
    noise: float = 0.1
    passes: int = 1


# BASELINE.json "configs" (seeds follow BASELINE.md section 4).
CONFIGS = {
    "tiny": StreamConfig("tiny", 100, 20, 5, ("uniform", 50, 200), ("uniform", 1, 5),
                         ("fixed", 2), ("uniform", 50, 200), 1.0, 10, 0),
    "medium": StreamConfig("medium", 1000, 88, 10, ("uniform", 100, 2000), ("uniform", 1, 10),
                           ("fixed", 10), ("uniform", 100, 500), 0.9, 20, 1),
    "daily": StreamConfig("daily", 4700, 88, 10, ("loguniform", 20, 4000), ("uniform", 1, 1),
                          ("uniform", 2, 4), ("uniform", 1, 50), 0.9, 100, 2),
    "large": StreamConfig("large", 50000, 128, 16, ("uniform", 200, 2000), ("uniform", 1, 8),
                          ("fixed", 500), ("uniform", 200, 2000), 0.95, 20, 3),
    "wide10": StreamConfig("wide10", 20000, 1024, 10, ("uniform", 64, 512), ("uniform", 1, 4),
                           ("fixed", 200), ("uniform", 64, 512), 0.9, 20, 4),
    "wide32": StreamConfig("wide32", 20000, 1024, 32, ("uniform", 64, 512), ("uniform", 1, 4),
                           ("fixed", 200), ("uniform", 64, 512), 0.9, 20, 4),
    "wide64": StreamConfig("wide64", 20000, 1024, 64, ("uniform", 64, 512), ("uniform", 1, 4),
                           ("fixed", 200), ("uniform", 64, 512), 0.9, 20, 4),
}


def scaled(cfg: StreamConfig, K0: int | None = None, steps: int | None = None,
           new_slices: int | None = None, **kw) -> StreamConfig:
    """Same shape law with fewer slices / steps (for CPU-oracle-sized parity runs)."""
    upd = dict(kw)
    if K0 is not None:
        upd["K0"] = K0
    if steps is not None:
        upd["steps"] = steps
    if new_slices is not None:
        upd["new_slices"] = new_slices if isinstance(new_slices, tuple) else ("fixed", new_slices)
    return replace(cfg, **upd)


def _draw(rng, law, n):
    kind = law[0]
    if kind == "uniform":
        return rng.integers(law[1], law[2] + 1, size=n)
    if kind == "loguniform":
        lo, hi = np.log(law[1]), np.log(law[2])
        return np.floor(np.exp(rng.uniform(lo, hi, size=n))).astype(np.int64).clip(law[1], law[2])
    if kind == "fixed":
        return np.full(n, law[1], dtype=np.int64)
    raise ValueError(f"unknown law {law!r}")


@dataclass
class Schedule:
    """Row counts only: initial lengths, and per update the rows appended to
    every active slice plus the new slices' initial lengths."""

    init_len: np.ndarray                 # (K0,)
    adds: list                           # per update: (active,) rows appended
    new_len: list                        # per update: (L,) rows of each new slice

    @property
    def total_len(self) -> np.ndarray:
        tot = list(self.init_len)
        for add, new in zip(self.adds, self.new_len):
            for k in range(len(add)):
                tot[k] += int(add[k])
            tot.extend(int(x) for x in new)
        return np.asarray(tot, dtype=np.int64)


def make_schedule(cfg: StreamConfig) -> Schedule:
    rng = np.random.default_rng([cfg.seed, 1])
    init_len = _draw(rng, cfg.init_rows, cfg.K0)
    active = cfg.K0
    adds, new_len = [], []
    for _ in range(cfg.steps):
        adds.append(_draw(rng, cfg.add_rows, active))
        L = int(_draw(rng, cfg.new_slices, 1)[0])
        new_len.append(_draw(rng, cfg.new_rows, L))
        active += L
    return Schedule(init_len, adds, new_len)


def true_factors(cfg: StreamConfig):
    rng = np.random.default_rng([cfg.seed, 0])
    H = rng.uniform(size=(cfg.R, cfg.R))
    V = rng.uniform(size=(cfg.J, cfg.R))
    return H, V


def slice_id(k: int) -> str:
    return f"s{k:06d}"


class SliceSource:
    """Generates any row range of slice k deterministically (per-slice RNG)."""

    def __init__(self, cfg: StreamConfig, total_len: np.ndarray, exact: bool = True):
        self.cfg = cfg
        self.total_len = total_len
        self.exact = exact
        self.H, self.V = true_factors(cfg)
        self._cache = {}

    def weights(self, k: int) -> np.ndarray:
        return np.random.default_rng([self.cfg.seed, 2, k]).uniform(size=self.cfg.R)

    def rows(self, k: int, lo: int, hi: int) -> np.ndarray:
        cfg = self.cfg
        if self.exact:
            full = self._cache.get(k)
            if full is None:
                full = self._full(k)
                self._cache[k] = full
            return full[lo:hi]
        rng = np.random.default_rng([cfg.seed, 3, k, lo])
        n = hi - lo
        q = rng.standard_normal((n, cfg.R)) / np.sqrt(max(int(self.total_len[k]), cfg.R))
        sig = (q @ self.H) * self.weights(k)
        return sig @ self.V.T + cfg.noise * rng.standard_normal((n, cfg.J))

    def _full(self, k: int) -> np.ndarray:
        cfg = self.cfg
        T = int(self.total_len[k])
        rng = np.random.default_rng([cfg.seed, 3, k])
        g = rng.standard_normal((max(T, cfg.R), cfg.R))
        q, _ = np.linalg.qr(g)
        q = q[:T]
        sig = (q @ self.H) * self.weights(k)
        return sig @ self.V.T + cfg.noise * rng.standard_normal((T, cfg.J))

    def drop(self, k: int):
        self._cache.pop(k, None)


@dataclass
class Stream:
    cfg: StreamConfig
    schedule: Schedule
    source: SliceSource

    def initial_tensor(self) -> IrregularTensor:
        return IrregularTensor(
            SliceMatrix(slice_id(k), self.source.rows(k, 0, int(n)))
            for k, n in enumerate(self.schedule.init_len)
        )

    def batches(self):
        """Yield the UpdateBatch sequence (existing rows in slice order, then
        the new slices)."""
        sch = self.schedule
        pos = [int(n) for n in sch.init_len]
        for t, (add, new) in enumerate(zip(sch.adds, sch.new_len)):
            existing = {}
            for k in range(len(add)):
                a = int(add[k])
                if a > 0:
                    existing[slice_id(k)] = self.source.rows(k, pos[k], pos[k] + a)
                    pos[k] += a
            fresh = []
            base = len(pos)
            for i, n in enumerate(new):
                k = base + i
                fresh.append(NewSlice(slice_id(k), self.source.rows(k, 0, int(n)), t + 1))
                pos.append(int(n))
            yield UpdateBatch(t + 1, existing, fresh, (t + 1, t + 1))


def make_stream(cfg: StreamConfig | str, exact: bool = True) -> Stream:
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    sch = make_schedule(cfg)
    return Stream(cfg, sch, SliceSource(cfg, sch.total_len, exact=exact))


def planted_state(stream: Stream):
    """Closed-form stream state of the planted model on the initial slices.

    With orthonormal Q_k the true factors give U_k^T U_k = H^T H, so
    (stream.py:56-82 semantics) D_k = H^T H, c_k[r] = sum_z D_rz w_z (V^T V)_zr,
    G = sum_k diag(w_k) D diag(w_k), F = V G.  Returns a dict with
    slice_ids, W, V, C, D, F, G (no initial U blocks)."""
    cfg = stream.cfg
    H, V = stream.source.H, stream.source.V
    K0, R = cfg.K0, cfg.R
    W = np.stack([stream.source.weights(k) for k in range(K0)])
    D0 = H.T @ H
    vtv = V.T @ V
    C = np.einsum("rz,kz,zr->kr", D0, W, vtv)
    D = np.broadcast_to(D0, (K0, R, R)).copy()
    G = np.einsum("kr,rz,kz->rz", W, D0, W)
    G = (G + G.T) / 2.0
    F = V @ G
    return {
        "slice_ids": [slice_id(k) for k in range(K0)],
        "W": W, "V": V.copy(), "C": C, "D": D, "F": F, "G": G,
        "forgetting": cfg.forgetting, "passes": cfg.passes,
    }
