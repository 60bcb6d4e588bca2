"""parafac2_als on the GPU (als.py:102-201 of the reference).

Host side of the sweep loop: validation and the seeded uniform initialisation
(bit-identical to the reference's ``default_rng(seed)`` draws, als.py:140-145)
happen here; every sweep runs on the device through ``dash_als_sweep_f64``
(XV GEMM, per-slice polar factors via CholQR2 + Jacobi SVD, CP-sweep solves,
rhs_v GEMM, V solve, direct-form loss).  The only per-sweep host traffic is
the 8-byte loss needed for the reference's early-exit test (als.py:186-189).
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native as nat
from .als import ALSInfo, FactorSet
from .linalg import RIDGE_EPS, SolveError

F64 = torch.float64


def parafac2_als_gpu(tensor, rank: int, iters: int = 10, seed: int = 0, tol: float = 1e-8,
                     return_info: bool = False, device=None):
    from .history import DeviceTensor
    dev_tensor = isinstance(tensor, DeviceTensor)
    if dev_tensor:  # accumulated data already in HBM (history.py): no host round trip
        ids_all = list(tensor.slice_ids)
        counts = np.diff(tensor.row_ptr)
        J = tensor.column_count
        min_rows = int(counts.min()) if len(counts) else 0
    else:
        slices = list(tensor.slices)
        J = tensor.column_count
        min_rows = min(s.row_count for s in slices)
    if rank > min(J, min_rows):
        raise ValueError(f"rank {rank} exceeds min(columns, shortest slice) = {min(J, min_rows)}")
    if iters < 1:
        raise ValueError("iters must be at least 1")
    if rank > nat.MAX_RANK_ALS:
        raise ValueError(f"rank {rank} exceeds the ALS engine's maximum {nat.MAX_RANK_ALS}")
    from .stream import _dev
    dev = _dev(device)
    K = len(tensor.slice_ids) if dev_tensor else len(slices)
    rng = np.random.default_rng(seed)
    V0 = rng.uniform(size=(J, rank))
    H0 = rng.uniform(size=(rank, rank))
    if dev_tensor:
        row_ptr = np.ascontiguousarray(tensor.row_ptr, dtype=np.int64)
        X = tensor.X.to(device=dev, dtype=F64).contiguous()
    else:
        counts = np.array([s.row_count for s in slices], dtype=np.int64)
        row_ptr = np.zeros(K + 1, dtype=np.int64)
        np.cumsum(counts, out=row_ptr[1:])
        X = torch.as_tensor(np.concatenate([s.rows for s in slices]), device=dev)
    N = int(row_ptr[-1])
    rp = torch.as_tensor(row_ptr, device=dev)
    V = torch.as_tensor(V0, device=dev)
    H = torch.as_tensor(H0, device=dev)
    W = torch.ones((K, rank), dtype=F64, device=dev)
    Q = torch.empty((N, rank), dtype=F64, device=dev)
    loss = torch.empty((), dtype=F64, device=dev)
    b = nat.DashBatch(X=int(X.data_ptr()), ldx=J, N=N, M=K, row_ptr=int(rp.data_ptr()),
                      row_ptr_host=row_ptr.ctypes.data, state_row=0, is_new=0)
    L = nat.lib()
    ctx = nat.context(dev.index)
    losses = []
    with torch.cuda.device(dev):
        st = nat.stream_ptr()
        for _ in range(iters):
            nat.check(L.dash_als_sweep_f64(ctx, st, ctypes.byref(b), J, rank, int(V.data_ptr()),
                                           int(H.data_ptr()), int(W.data_ptr()), int(Q.data_ptr()),
                                           int(loss.data_ptr()), RIDGE_EPS), "dash_als_sweep_f64")
            _raise_on_error(L, ctx, st, ids_all if dev_tensor else [s.slice_id for s in slices])
            cur = float(loss.item())
            losses.append(cur)
            if len(losses) >= 2:
                prev = losses[-2]
                if prev == 0.0 or abs(prev - cur) <= tol * prev:
                    break
        U = torch.empty_like(Q)
        nat.check(L.dash_als_project_f64(ctx, st, N, rank, int(Q.data_ptr()), int(H.data_ptr()),
                                         int(U.data_ptr())), "dash_als_project_f64")
        Uh, Qh = U.cpu().numpy(), Q.cpu().numpy()
    ids = ids_all if dev_tensor else [s.slice_id for s in slices]
    factors = FactorSet(
        slice_ids=ids,
        U={sid: Uh[row_ptr[k]:row_ptr[k + 1]] for k, sid in enumerate(ids)},
        W=W.cpu().numpy(), V=V.cpu().numpy())
    factors._device = {"U": U, "W": W, "V": V, "X": X, "row_ptr": row_ptr}
    if return_info:
        return factors, ALSInfo(losses=losses,
                                projections={sid: Qh[row_ptr[k]:row_ptr[k + 1]] for k, sid in enumerate(ids)})
    return factors


def _raise_on_error(L, ctx, st, ids):
    pos = ctypes.c_int64(0)
    rc = L.dash_ctx_status(ctx, st, ctypes.byref(pos))
    if rc == nat.DASH_OK:
        return
    if rc == nat.DASH_E_CUDA:
        raise RuntimeError("CUDA error during parafac2_als")
    from .als import FactorizationError
    p = pos.value
    sid = ids[p] if 0 <= p < len(ids) else None
    if rc == nat.DASH_E_SINGULAR and sid is not None:
        raise FactorizationError(f"polar factor failed for slice {sid!r}")
    raise SolveError("singular normal equations" if rc == nat.DASH_E_SINGULAR
                     else "non-finite solution from normal equations", sid)
