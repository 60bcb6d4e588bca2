"""The reference's operator seams, served by the CUDA library.

``group_update``   same contract as the numba kernel _kernels.group_update
                   (_kernels.py:62-149): numpy in, numpy out, ``ok`` flag.
``ridge_solve``    linalg.ridge_solve (linalg.py:25-45) for stacks of systems.

These exist so code written against the reference's seams (and the parity
tests) can drive the device kernels directly; the engine itself calls the
fused ``dash_update_f64`` instead.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native as nat
from .linalg import RIDGE_EPS, SolveError


def _dev_tensor(a, device):
    return torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=float)), device=device)


def group_update(xv, vtv, s_used, c_old, d_old, lam, eps=RIDGE_EPS):
    L = nat.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    xv = np.asarray(xv, dtype=float)
    G, I, R = xv.shape
    t = {k: _dev_tensor(v, dev) for k, v in
         dict(xv=xv, vtv=vtv, s=s_used, c=c_old, d=d_old).items()}
    out = {k: torch.empty(shape, dtype=torch.float64, device=dev) for k, shape in
           dict(u=(G, I, R), us=(G, I, R), c_new=(G, R), d_new=(G, R, R), w=(G, R),
                g_fresh=(R, R)).items()}
    ok = ctypes.c_int32(1)
    p = lambda x: int(x.data_ptr())  # noqa: E731
    nat.check(L.dash_group_update_f64(nat.context(), nat.stream_ptr(), G, I, R, p(t["xv"]),
                                      p(t["vtv"]), p(t["s"]), p(t["c"]), p(t["d"]), float(lam),
                                      float(eps), p(out["u"]), p(out["us"]), p(out["c_new"]),
                                      p(out["d_new"]), p(out["w"]), p(out["g_fresh"]),
                                      ctypes.byref(ok)), "dash_group_update_f64")
    pos = ctypes.c_int64(0)
    L.dash_ctx_status(nat.context(), nat.stream_ptr(), ctypes.byref(pos))  # clears the slot
    res = [out[k].cpu().numpy() for k in ("u", "us", "c_new", "d_new", "w", "g_fresh")]
    return (*res, bool(ok.value))


def ridge_solve(lhs, rhs, eps=RIDGE_EPS):
    L = nat.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    lhs = np.asarray(lhs, dtype=float)
    rhs = np.asarray(rhs, dtype=float)
    squeeze_b = lhs.ndim == 2
    vec = rhs.ndim == lhs.ndim - 1
    if squeeze_b:
        lhs = lhs[None]
        rhs = rhs[None]
    if vec:
        rhs = rhs[..., None]
    B, n, _ = lhs.shape
    m = rhs.shape[-1]
    tl, tr = _dev_tensor(lhs, dev), _dev_tensor(rhs, dev)
    x = torch.empty_like(tr)
    nat.check(L.dash_ridge_solve_f64(nat.context(), nat.stream_ptr(), B, n, m, int(tl.data_ptr()),
                                     int(tr.data_ptr()), int(x.data_ptr()), float(eps)),
              "dash_ridge_solve_f64")
    pos = ctypes.c_int64(0)
    rc = L.dash_ctx_status(nat.context(), nat.stream_ptr(), ctypes.byref(pos))
    if rc == nat.DASH_E_SINGULAR:
        raise SolveError("singular normal equations")
    if rc == nat.DASH_E_NONFINITE:
        raise SolveError("non-finite solution from normal equations")
    out = x.cpu().numpy()
    if vec:
        out = out[..., 0]
    return out[0] if squeeze_b else out
