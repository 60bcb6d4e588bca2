"""Per-update fitness on the GPU: ``local_error`` (evaluate.py:93-118 of the
reference) -- per-slice mean |X_k - (U_k o w_k) V^T| with the post-update W
and V, and the tensor-level mean over the slices in the batch
(anomaly.py:23-42 ``slice_error`` / ``tensor_error``)."""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native as nat


def local_error(batch_items, u_new, state):
    """Same signature and return value as the reference: (te, {sid: mad})."""
    ids = [sid for sid, _ in batch_items]
    last = getattr(state, "_last", None)
    dev = state.device
    if (last is not None and last[0] == ids and hasattr(u_new, "device_tensor")
            and u_new.device_tensor is last[5]):
        _, row_ptr, meta, X, N, U = last
        if row_ptr is None:
            row_ptr = meta.host_row_ptr()
        state_row = meta[1]  # device copies staged by the update
        rp_dev = meta[0]
    else:
        counts = np.array([np.asarray(r).shape[0] for _, r in batch_items], dtype=np.int64)
        row_ptr = np.zeros(len(ids) + 1, dtype=np.int64)
        np.cumsum(counts, out=row_ptr[1:])
        dt = getattr(state, "dtype", torch.float64)
        X = torch.as_tensor(np.concatenate([np.asarray(r, dtype=float) for _, r in batch_items]),
                            device=dev).to(dt)
        U = torch.as_tensor(np.concatenate([np.asarray(u_new[s], dtype=float) for s in ids]),
                            device=dev).to(dt)
        state_row = np.array([state.row_of(s) for s in ids], dtype=np.int32)
        N = int(row_ptr[-1])
        rp_dev = None
    slice_err, te = local_error_device(X, N, row_ptr, state_row, U, state, row_ptr_dev=rp_dev)
    se = slice_err.cpu().numpy()
    return float(te.item()), {sid: float(se[k]) for k, sid in enumerate(ids)}


def local_error_device(X, N, row_ptr, state_row, U, state, row_ptr_dev=None):
    """Device tensors in, device (slice_err (M,), tensor_err ()) out.  ``row_ptr_dev``: the
    update's own staged device copy of row_ptr (saves re-uploading it)."""
    return slice_errors_device(X, N, row_ptr, state_row, U, state.device_tensors["W"], state._V,
                               state._ctx, state.device, row_ptr_dev=row_ptr_dev)


def slice_errors_device(X, N, row_ptr, state_row, U, W, V, ctx=None, device=None, row_ptr_dev=None):
    """Per-slice mean |X_k - (U_k o W[state_row[k]]) V^T| and their mean
    (anomaly.py:23-42 slice_error / tensor_error) on the device."""
    dev = X.device if device is None else device
    M = len(row_ptr) - 1
    J, R = V.shape
    rp = row_ptr_dev if row_ptr_dev is not None else torch.as_tensor(np.asarray(row_ptr, dtype=np.int64), device=dev)
    sr = (state_row if isinstance(state_row, torch.Tensor)
          else torch.as_tensor(np.asarray(state_row, dtype=np.int32), device=dev))
    slice_err = torch.empty(max(M, 1), dtype=torch.float64, device=dev)
    te = torch.empty((), dtype=torch.float64, device=dev)
    b = nat.DashBatch(X=int(X.data_ptr()), ldx=int(X.stride(0)), N=N, M=M, row_ptr=int(rp.data_ptr()),
                      row_ptr_host=np.asarray(row_ptr, dtype=np.int64).ctypes.data,
                      state_row=int(sr.data_ptr()), is_new=0)
    if X.dtype != U.dtype or X.dtype not in (torch.float32, torch.float64):
        raise TypeError("local_error: X and U must both be float64 or both float32")
    fn = nat.lib().dash_local_error_f32 if X.dtype == torch.float32 else nat.lib().dash_local_error_f64
    from .stream import _on
    with _on(dev):
        if ctx is None:
            ctx = nat.context(dev.index)
        nat.check(fn(ctx, nat.stream_ptr(), ctypes.byref(b),
                     int(U.data_ptr()), int(W.data_ptr()),
                     int(V.data_ptr()), J, R,
                     int(slice_err.data_ptr()), int(te.data_ptr())),
                  "dash_local_error")
    return slice_err[:M], te


def tensor_error_device(data: dict, factors: dict, w_rows: dict, V, device=None) -> float:
    """Mean over the slices of ``data`` of the per-slice mean |rows - (U o w) V^T|
    (one term of evaluate.py:121-144's global_error); 0 for no slices."""
    ids = list(data)
    if not ids:
        return 0.0
    from .stream import _dev
    dev = _dev(device)
    counts = np.array([np.asarray(data[s]).shape[0] for s in ids], dtype=np.int64)
    row_ptr = np.zeros(len(ids) + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    X = torch.as_tensor(np.concatenate([np.asarray(data[s], dtype=float) for s in ids]), device=dev)
    U = torch.as_tensor(np.concatenate([np.asarray(factors[s], dtype=float) for s in ids]), device=dev)
    W = torch.as_tensor(np.stack([np.asarray(w_rows[s], dtype=float) for s in ids]), device=dev)
    Vd = torch.as_tensor(np.ascontiguousarray(V, dtype=float), device=dev)
    _, te = slice_errors_device(X, int(row_ptr[-1]), row_ptr, np.arange(len(ids), dtype=np.int32), U, W, Vd,
                                device=dev)
    return float(te.item())
