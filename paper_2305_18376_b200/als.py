"""Factor containers and the static PARAFAC2-ALS fit used by ``initialize``
(/root/reference/pkg/src/p2stream/als.py:24-201).

``FactorSet`` / ``ALSInfo`` / ``reconstruct*`` / ``relative_error`` are the
reference's host-side containers and formulas (cheap, O(#slices) Python).
``parafac2_als`` runs on the GPU (csrc/dash_als.cuh); see its docstring.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


class FactorizationError(RuntimeError):
    """The alternating solve broke down on a slice (als.py:18-19)."""


@dataclass
class FactorSet:
    """Factors of an irregular tensor (als.py:24-59): U per slice, W rows
    (diagonal of S_k), shared V."""

    slice_ids: list
    U: dict
    W: np.ndarray
    V: np.ndarray
    _row_of: dict = field(init=False, repr=False)

    def __post_init__(self):
        self.W = np.asarray(self.W, dtype=float)
        self.V = np.asarray(self.V, dtype=float)
        self._row_of = {sid: k for k, sid in enumerate(self.slice_ids)}
        rank = self.V.shape[1]
        if self.W.shape != (len(self.slice_ids), rank):
            raise ValueError("W must have one row per slice and rank columns")
        for sid in self.slice_ids:
            if self.U[sid].shape[1] != rank:
                raise ValueError(f"U block {sid!r} does not match rank {rank}")

    @property
    def rank(self) -> int:
        return self.V.shape[1]

    def row_of(self, slice_id) -> int:
        return self._row_of[slice_id]

    def s_row(self, slice_id) -> np.ndarray:
        return self.W[self._row_of[slice_id]]


@dataclass
class ALSInfo:
    """Per-iteration diagnostics (als.py:62-71): losses and the Q_k bases."""

    losses: list
    projections: dict

    @property
    def final_loss(self) -> float:
        return self.losses[-1]


def reconstruct_rows(u_rows, s, V):
    """U diag(s) V^T (als.py:74-76)."""
    return (u_rows * s) @ V.T


def reconstruct(factors: FactorSet, k: int):
    sid = factors.slice_ids[k]
    return reconstruct_rows(factors.U[sid], factors.W[k], factors.V)


def factorization_loss(tensor, factors: FactorSet) -> float:
    total = 0.0
    for s in tensor.slices:
        rec = reconstruct_rows(factors.U[s.slice_id], factors.s_row(s.slice_id), factors.V)
        total += float(np.sum((s.rows - rec) ** 2))
    return total


def relative_error(tensor, factors: FactorSet) -> float:
    norm_sq = sum(float(np.sum(s.rows ** 2)) for s in tensor.slices)
    if norm_sq == 0.0:
        return 0.0
    return float(np.sqrt(factorization_loss(tensor, factors) / norm_sq))


def parafac2_als(tensor, rank: int, iters: int = 10, seed: int = 0, tol: float = 1e-8,
                 return_info: bool = False, device=None):
    """Direct-fitting PARAFAC2-ALS on the GPU (als.py:102-201)."""
    from ._als_gpu import parafac2_als_gpu
    return parafac2_als_gpu(tensor, rank, iters=iters, seed=seed, tol=tol,
                            return_info=return_info, device=device)
