"""Accumulated data on the GPU: the X-history store, ``apply_batch``,
``global_error`` and the baseline refit (north_star item 1).

The reference keeps the accumulated tensor on the host and rebuilds it every
update (``apply_batch``, tensor.py:228-244: ``np.vstack`` per touched slice),
then refits it from scratch for the baseline (``parafac2_als(..., tol=0.0)``,
evaluate.py:212-222) and measures the two-term accumulated error
``global_error`` (evaluate.py:121-144) over the retained rows.

Here the accumulated tensor is a :class:`DeviceTensor`: one CSR block in HBM
(rows of each slice contiguous, slices in the reference's order: existing
slices, then new ones in batch order).  ``apply_batch`` builds the next CSR
with ONE gather over [old X | batch X] (an index_select on the device: every
accumulated row is read and written once, the same traffic as the
reference's vstack, at HBM speed), so the refit and the error metrics read
it without any host round trip.  ``parafac2_als`` accepts a DeviceTensor
directly.  U histories for ``global_error`` come from the stream state's
device U blocks, gathered into the same CSR order.
"""
from __future__ import annotations

import numpy as np
import torch

from .tensor import DatasetError, IrregularTensor, SliceMatrix, UpdateBatch

F64 = torch.float64


class DeviceTensor:
    """An irregular tensor resident in HBM, CSR by slice (the reference's
    ``IrregularTensor`` contract: ``slices`` order, ``slice_ids``,
    ``column_count``, ``total_rows``, ``get`` / ``has``)."""

    def __init__(self, slice_ids, row_ptr: np.ndarray, X: torch.Tensor, first_steps=None):
        self.slice_ids = list(slice_ids)
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self.X = X
        self.first_steps = list(first_steps) if first_steps is not None else [0] * len(self.slice_ids)
        if self.row_ptr.shape[0] != len(self.slice_ids) + 1 or int(self.row_ptr[-1]) != X.shape[0]:
            raise ValueError("row_ptr does not match the slices / rows")
        self._index = {sid: k for k, sid in enumerate(self.slice_ids)}
        if len(self._index) != len(self.slice_ids):
            raise DatasetError("duplicate slice ids in tensor")

    # -- reference IrregularTensor surface ---------------------------------
    @classmethod
    def from_tensor(cls, tensor: IrregularTensor, device=None) -> "DeviceTensor":
        slices = list(tensor.slices)
        counts = np.array([s.row_count for s in slices], dtype=np.int64)
        row_ptr = np.zeros(len(slices) + 1, dtype=np.int64)
        np.cumsum(counts, out=row_ptr[1:])
        X = torch.as_tensor(np.concatenate([np.asarray(s.rows, dtype=float) for s in slices]), device=device)
        return cls([s.slice_id for s in slices], row_ptr, X, [s.first_time_step for s in slices])

    @property
    def device(self):
        return self.X.device

    @property
    def column_count(self) -> int:
        return int(self.X.shape[1])

    @property
    def total_rows(self) -> int:
        return int(self.row_ptr[-1])

    def __len__(self) -> int:
        return len(self.slice_ids)

    def has(self, slice_id) -> bool:
        return slice_id in self._index

    def row_count(self, slice_id) -> int:
        k = self._index[slice_id]
        return int(self.row_ptr[k + 1] - self.row_ptr[k])

    @property
    def slices(self):
        """Host view (SliceMatrix per slice; one device->host copy)."""
        Xh = self.X.cpu().numpy()
        return [SliceMatrix(sid, Xh[self.row_ptr[k]:self.row_ptr[k + 1]], self.first_steps[k])
                for k, sid in enumerate(self.slice_ids)]

    def get(self, slice_id) -> SliceMatrix:
        k = self._index[slice_id]
        return SliceMatrix(slice_id, self.X[self.row_ptr[k]:self.row_ptr[k + 1]].cpu().numpy(),
                           self.first_steps[k])

    def to_host(self) -> IrregularTensor:
        return IrregularTensor(self.slices)

    # -- accumulation -------------------------------------------------------
    def apply_batch(self, batch: UpdateBatch) -> "DeviceTensor":
        """tensor.py:228-244: append a batch (existing slices grow in place,
        new slices go last in batch order); returns the accumulated tensor."""
        for sid in batch.existing_rows:
            if sid not in self._index:
                raise DatasetError(f"batch references unknown existing slice {sid!r}")
        ids, counts, rows = [], [], []
        for sid, r, _ in batch.items():
            ids.append(sid)
            counts.append(np.asarray(r).shape[0])
            rows.append(np.asarray(r, dtype=float))
        Xb = torch.as_tensor(np.concatenate(rows) if rows else np.zeros((0, self.column_count)),
                             device=self.device)
        n_old = len(batch.existing_rows)
        existing = np.fromiter((self._index[s] for s in ids[:n_old]), dtype=np.int64, count=n_old)
        steps = [ns.first_time_step for ns in batch.new_slices]
        return self.apply_packed(Xb, np.asarray(counts, dtype=np.int64), existing, ids[n_old:], steps)

    def apply_packed(self, Xb: torch.Tensor, counts, existing: np.ndarray, new_ids, new_steps=None):
        """Device batch X (rows in items() order: existing slices at tensor
        positions ``existing``, then the new slices) -> accumulated tensor."""
        K = len(self.slice_ids)
        counts = np.asarray(counts, dtype=np.int64)
        n_old = len(existing)
        add = np.zeros(K, dtype=np.int64)
        np.add.at(add, existing, counts[:n_old])
        bptr = np.zeros(len(counts) + 1, dtype=np.int64)
        np.cumsum(counts, out=bptr[1:])
        old_len = np.diff(self.row_ptr)
        new_len = np.concatenate([old_len + add, counts[n_old:]])
        row_ptr = np.zeros(len(new_len) + 1, dtype=np.int64)
        np.cumsum(new_len, out=row_ptr[1:])
        # destination of every old row and every batch row in the new CSR:
        # per slice its old rows, then its new rows; new slices last
        N_old = self.total_rows
        old_rank = np.arange(N_old) - np.repeat(self.row_ptr[:K], old_len)
        dst_old = np.repeat(row_ptr[:K], old_len) + old_rank
        nb = int(bptr[-1])
        base = np.empty(len(counts), dtype=np.int64)
        base[:n_old] = row_ptr[existing] + old_len[existing]
        base[n_old:] = row_ptr[K:len(new_len)]
        dst_b = np.repeat(base, counts) + (np.arange(nb) - np.repeat(bptr[:-1], counts))
        X = torch.empty((int(row_ptr[-1]), self.column_count), dtype=self.X.dtype, device=self.device)
        if N_old:
            X.index_copy_(0, torch.as_tensor(dst_old, device=self.device), self.X)
        if nb:
            X.index_copy_(0, torch.as_tensor(dst_b, device=self.device), Xb[:nb].to(self.X.dtype))
        steps = list(self.first_steps) + (list(new_steps) if new_steps is not None else [0] * len(new_ids))
        return DeviceTensor(self.slice_ids + list(new_ids), row_ptr, X, steps)


def global_error(old_data, old_factors, new_data, new_factors, w_rows, V, device=None) -> float:
    """evaluate.py:121-144 on the GPU: term(old rows with the stored old row
    factors) + term(newest batch), each the mean over slices of the per-slice
    mean |X - (U o w) V^T|, with the current W rows and V.  Dict inputs as
    the reference's; the rows / factors are packed once and reduced by the
    local_error kernel (fixed-order sums)."""
    from .evaluate import tensor_error_device
    return (tensor_error_device(old_data, old_factors, w_rows, V, device)
            + tensor_error_device(new_data, new_factors, w_rows, V, device))


def global_error_device(history: DeviceTensor, U_hist: torch.Tensor, state, batch_items, u_new) -> float:
    """Device-resident form for a stream: ``history`` holds the retained rows
    of the slices that existed before the update (CSR) and ``U_hist`` their
    row factors as of before the update (``state.u_history_device(ids)``,
    taken before ``state.update``); the batch term uses ``u_new``.  Same value
    as :func:`global_error`."""
    from .evaluate import local_error, local_error_device
    rows_of = np.array([state.row_of(s) for s in history.slice_ids], dtype=np.int32)
    if U_hist.shape[0] != history.total_rows:
        raise ValueError("U history and data rows differ")
    te_old = 0.0
    if len(history):
        _, t = local_error_device(history.X, history.total_rows, history.row_ptr, rows_of,
                                  U_hist.to(history.X.dtype), state)
        te_old = float(t.item())
    te_new, _ = local_error(batch_items, u_new, state)
    return te_old + te_new


def refit_baseline(accumulated, rank: int, iters: int = 10, seed: int = 0, device=None):
    """The baseline refit of evaluate.py:212-222: a fixed sweep count
    (tol=0.0) fit of the accumulated tensor (host or device)."""
    from .als import parafac2_als
    return parafac2_als(accumulated, rank, iters=iters, seed=seed, tol=0.0, device=device)
