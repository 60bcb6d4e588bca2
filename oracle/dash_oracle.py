"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the DASH per-update step.

Nothing in the shipped package imports this module.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg use it, and only as the checker or the timed CPU
reference -- never as the thing measured for the GPU arm.

It restates, in plain numpy, the reference package ``p2stream``'s algorithm
for the hot path (paths relative to /root/reference/pkg/src/p2stream):

  * ``ridge_solve`` / ``symmetrize``          linalg.py:20-45
  * ``group_update`` (numba kernel)           _kernels.py:62-144 (C restatement
                                              in oracle/group_update.c)
  * ``OracleStreamState.update``              stream.py:251-370
  * ``init_helpers``                          stream.py:56-82
  * ``parafac2_als``                          als.py:102-201
  * ``local_error``                           evaluate.py:93-118

Parity pinning: tests/test_oracle.py checks this restatement against the
golden vectors in tests/golden/ that tests/golden/make_golden.py produced by
running the reference itself (imported from /root/reference) in the build
container, and -- when /root/reference is present -- against the live
reference.
"""
from __future__ import annotations

import ctypes
import os
import time
from pathlib import Path

import numpy as np

RIDGE_EPS = 1e-10  # linalg.py:7

_HERE = Path(__file__).resolve().parent
_LIB = None


class OracleSolveError(ValueError):
    """Mirror of linalg.SolveError (linalg.py:10-17)."""

    def __init__(self, message, slice_id=None):
        if slice_id is not None:
            message = f"{message} (slice {slice_id!r})"
        super().__init__(message)
        self.slice_id = slice_id


def symmetrize(mat):
    """linalg.py:20-22."""
    return (mat + mat.swapaxes(-1, -2)) / 2.0


def ridge_solve(lhs, rhs, eps=RIDGE_EPS, slice_id=None):
    """linalg.py:25-45: solve after adding eps*mean(diag)*I (LAPACK gesv)."""
    lhs = np.asarray(lhs, dtype=float)
    rhs = np.asarray(rhs, dtype=float)
    n = lhs.shape[-1]
    diag_mean = np.einsum("...ii->...", lhs) / n
    ridged = lhs + (eps * diag_mean)[..., None, None] * np.eye(n)
    try:
        out = np.linalg.solve(ridged, rhs)
    except np.linalg.LinAlgError as exc:
        raise OracleSolveError(f"singular normal equations: {exc}", slice_id) from None
    if not np.all(np.isfinite(out)):
        raise OracleSolveError("non-finite solution from normal equations", slice_id)
    return out


# ---------------------------------------------------------------------------
# per-slice kernel (_kernels.py:62-144)
# ---------------------------------------------------------------------------

def _load_c():
    global _LIB
    if _LIB is not None:
        return _LIB
    path = _HERE / "_build" / "liboracle.so"
    if not path.exists():
        return None
    lib = ctypes.CDLL(str(path))
    dp = ctypes.POINTER(ctypes.c_double)
    lib.oracle_group_update.restype = ctypes.c_int
    lib.oracle_group_update.argtypes = [ctypes.c_int] * 3 + [dp] * 5 + [
        ctypes.c_double, ctypes.c_double] + [dp] * 6
    _LIB = lib
    return lib


def build_c(quiet=True):
    """Compile oracle/group_update.c into oracle/_build/liboracle.so."""
    out = _HERE / "_build"
    out.mkdir(exist_ok=True)
    src = _HERE / "group_update.c"
    so = out / "liboracle.so"
    if so.exists() and so.stat().st_mtime >= src.stat().st_mtime:
        return so
    cmd = f"gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -shared -o {so} {src} -lm"
    rc = os.system(cmd + (" >/dev/null 2>&1" if quiet else ""))
    if rc != 0:
        raise RuntimeError(f"oracle C build failed: {cmd}")
    return so


def _ptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _chol_solve_py(a, b):
    """_kernels.py:27-59 in Python (fallback when the C oracle is absent)."""
    n = a.shape[0]
    for j in range(n):
        s = a[j, j]
        for k in range(j):
            s -= a[j, k] * a[j, k]
        if not s > 0.0 or not np.isfinite(s):
            return False
        piv = np.sqrt(s)
        a[j, j] = piv
        for i in range(j + 1, n):
            t = a[i, j]
            for k in range(j):
                t -= a[i, k] * a[j, k]
            a[i, j] = t / piv
    for col in range(b.shape[1]):
        for i in range(n):
            s = b[i, col]
            for k in range(i):
                s -= a[i, k] * b[k, col]
            b[i, col] = s / a[i, i]
        for i in range(n - 1, -1, -1):
            s = b[i, col]
            for k in range(i + 1, n):
                s -= a[k, i] * b[k, col]
            b[i, col] = s / a[i, i]
    return True


def group_update(xv, vtv, s_used, c_old, d_old, lam, eps):
    """Same contract as the reference's ``group_update`` (_kernels.py:62-70).

    Returns ``(u, us, c_new, d_new, w, g_fresh, ok)``.
    """
    xv = np.ascontiguousarray(xv, dtype=float)
    G, I, R = xv.shape
    vtv = np.ascontiguousarray(vtv, dtype=float)
    s_used = np.ascontiguousarray(s_used, dtype=float)
    c_old = np.ascontiguousarray(c_old, dtype=float)
    d_old = np.ascontiguousarray(d_old, dtype=float)
    u = np.empty((G, I, R))
    us = np.empty((G, I, R))
    c_new = np.empty((G, R))
    d_new = np.empty((G, R, R))
    w = np.empty((G, R))
    g_fresh = np.zeros((R, R))
    lib = _load_c()
    if lib is not None:
        ok = lib.oracle_group_update(G, I, R, _ptr(xv), _ptr(vtv), _ptr(s_used), _ptr(c_old),
                                     _ptr(d_old), float(lam), float(eps), _ptr(u), _ptr(us),
                                     _ptr(c_new), _ptr(d_new), _ptr(w), _ptr(g_fresh))
        return u, us, c_new, d_new, w, g_fresh, bool(ok)
    ok = True
    for g in range(G):
        s = s_used[g]
        shift = eps * float(np.sum(np.diag(vtv) * s * s)) / R
        a = vtv * np.outer(s, s)
        a[np.diag_indices(R)] += shift
        rhs = (xv[g] * s).T.copy()
        if not _chol_solve_py(a, rhs):
            ok = False
        u[g] = rhs.T
        c_new[g] = lam * c_old[g] + np.einsum("ir,ir->r", xv[g], u[g])
        gram = u[g].T @ u[g]
        gram = np.triu(gram) + np.triu(gram, 1).T
        d_new[g] = lam * d_old[g] + gram
        shift = eps * float(np.sum(np.diag(vtv) * np.diag(d_new[g]))) / R
        a = vtv * d_new[g]
        a[np.diag_indices(R)] += shift
        wcol = c_new[g][:, None].copy()
        if not _chol_solve_py(a, wcol):
            ok = False
        if not np.all(np.isfinite(wcol)):
            ok = False
        w[g] = wcol[:, 0]
        us[g] = u[g] * w[g]
        g_fresh += gram * w[g][:, None] * w[g][None, :]
    return u, us, c_new, d_new, w, g_fresh, ok


# ---------------------------------------------------------------------------
# the streaming engine (stream.py:184-370)
# ---------------------------------------------------------------------------

def _solve_group(lhs, rhs, sids):
    """stream.py:372-380."""
    try:
        return ridge_solve(lhs, rhs)
    except OracleSolveError:
        for g, sid in enumerate(sids):
            ridge_solve(lhs[g], rhs[g], slice_id=sid)
        raise


class OracleStreamState:
    """Numpy restatement of ``StreamState`` (stream.py:184-247)."""

    def __init__(self, slice_ids, u_blocks, W, V, C, D, F, G, forgetting,
                 update_index=0, passes=1, use_kernel=True):
        if not 0.0 < forgetting <= 1.0:
            raise ValueError("forgetting factor must lie in (0, 1]")
        if passes < 1:
            raise ValueError("passes must be at least 1")
        self.slice_ids = list(slice_ids)
        self.u_blocks = u_blocks
        self.W = np.array(W, dtype=float)
        self.V = np.array(V, dtype=float)
        self.C = np.array(C, dtype=float)
        self.D = np.array(D, dtype=float)
        self.F = np.array(F, dtype=float)
        self.G = np.array(G, dtype=float)
        self.forgetting = float(forgetting)
        self.update_index = update_index
        self.passes = passes
        self.use_kernel = use_kernel
        self._row_of = {sid: k for k, sid in enumerate(self.slice_ids)}

    @property
    def rank(self):
        return self.V.shape[1]

    def row_of(self, sid):
        return self._row_of[sid]

    def u_matrix(self, sid):
        blocks = self.u_blocks[sid]
        return blocks[0].copy() if len(blocks) == 1 else np.vstack(blocks)

    def update(self, batch):
        """stream.py:251-370 -- one pass loop per ``passes``.

        ``batch`` is anything with ``.items()`` yielding (sid, rows, is_new)
        in batch order (the reference's UpdateBatch contract, tensor.py:166-171).
        Returns a dict with the UpdateResult fields.
        """
        started = time.perf_counter()
        rank = self.rank
        lam = self.forgetting
        entries = []
        for sid, rows, is_new in batch.items():
            if is_new and sid in self._row_of:
                raise ValueError(f"batch declares known slice {sid!r} as new")
            if not is_new and sid not in self._row_of:
                raise ValueError(f"batch references unknown existing slice {sid!r}")
            entries.append((sid, np.asarray(rows, dtype=float), is_new))
        new_ids = [sid for sid, _, is_new in entries if is_new]
        if new_ids:
            fresh = len(new_ids)
            self.W = np.vstack([self.W, np.ones((fresh, rank))])
            self.C = np.vstack([self.C, np.zeros((fresh, rank))])
            self.D = np.concatenate([self.D, np.zeros((fresh, rank, rank))])
            for sid in new_ids:
                self._row_of[sid] = len(self.slice_ids)
                self.slice_ids.append(sid)
        by_height = {}
        for pos, (_, rows, _) in enumerate(entries):
            by_height.setdefault(rows.shape[0], []).append(pos)
        groups = []
        for height, positions in by_height.items():
            sids = [entries[p][0] for p in positions]
            w_rows = np.fromiter((self._row_of[s] for s in sids), dtype=np.intp)
            x = np.concatenate([entries[p][1] for p in positions]).reshape(
                len(positions), height, -1)
            groups.append((sids, w_rows, x, self.C[w_rows], self.D[w_rows]))
        f_snap, g_snap = self.F, self.G
        results = []
        v_used = self.V
        for _ in range(self.passes):
            V = v_used = self.V
            vtv = V.T @ V
            f_fresh = np.zeros_like(f_snap)
            g_fresh = np.zeros_like(g_snap)
            results = []
            for sids, w_rows, x, c_old, d_old in groups:
                s_used = self.W[w_rows]
                fast = None
                if self.use_kernel:
                    flat = x.reshape(-1, x.shape[2])
                    xv3 = (flat @ V).reshape(x.shape[0], x.shape[1], rank)
                    fast = group_update(xv3, vtv, s_used, c_old, d_old, lam, RIDGE_EPS)
                if fast is not None and fast[6]:
                    u, us, c_new, d_new, w = fast[:5]
                    f_fresh += flat.T @ us.reshape(-1, rank)
                    g_fresh += fast[5]
                else:
                    xv = x @ V
                    lhs_u = vtv[None] * (s_used[:, :, None] * s_used[:, None, :])
                    rhs_u = (xv * s_used[:, None, :]).transpose(0, 2, 1)
                    u = _solve_group(lhs_u, rhs_u, sids).transpose(0, 2, 1)
                    c_fresh = np.einsum("gir,gir->gr", xv, u)
                    d_fresh = symmetrize(np.einsum("gir,giz->grz", u, u))
                    c_new = lam * c_old + c_fresh
                    d_new = symmetrize(lam * d_old + d_fresh)
                    lhs_w = vtv[None] * d_new
                    w = _solve_group(lhs_w, c_new[:, :, None], sids)[:, :, 0]
                    f_fresh += np.einsum("gij,gir->jr", x, u * w[:, None, :])
                    g_fresh += np.einsum("grz,gr,gz->rz", d_fresh, w, w)
                self.W[w_rows] = w
                results.append((w_rows, u, c_new, d_new))
            self.F = lam * f_snap + f_fresh
            self.G = symmetrize(lam * g_snap + g_fresh)
            self.V = ridge_solve(self.G, self.F.T).T
        for w_rows, _, c_new, d_new in results:
            self.C[w_rows] = c_new
            self.D[w_rows] = d_new
        u_new = {}
        fresh_set = set(new_ids)
        for (sids, *_), (_, u, _, _) in zip(groups, results):
            for g, sid in enumerate(sids):
                u_new[sid] = u[g]
                if sid in fresh_set:
                    self.u_blocks[sid] = [u[g]]
                else:
                    self.u_blocks[sid].append(u[g])
        self.update_index += 1
        return {
            "update_index": self.update_index,
            "u_new": u_new,
            "new_slice_ids": new_ids,
            "rows_new": sum(r.shape[0] for _, r, _ in entries),
            "seconds": time.perf_counter() - started,
            "v_used": v_used,
        }


def init_helpers(slices, U, W, V, forgetting=0.7):
    """stream.py:56-82.  ``slices``: list of (sid, rows); U: sid->block;
    W rows aligned with ``slices``.  Returns (c dict, D dict, F, G)."""
    J, rank = V.shape
    c, D = {}, {}
    F = np.zeros((J, rank))
    G = np.zeros((rank, rank))
    for k, (sid, rows) in enumerate(slices):
        u = U[sid]
        srow = W[k]
        xv = rows @ V
        c[sid] = np.einsum("ir,ir->r", xv, u)
        gram = u.T @ u
        D[sid] = symmetrize(gram)
        F += rows.T @ (u * srow)
        G += gram * np.outer(srow, srow)
    return c, D, F, symmetrize(G)


def parafac2_als(slices, rank, iters=10, seed=0, tol=1e-8):
    """als.py:102-201.  ``slices``: list of (sid, rows).  Returns
    (U dict, W, V, losses, projections dict, H)."""
    min_rows = min(r.shape[0] for _, r in slices)
    J = slices[0][1].shape[1]
    if rank > min(J, min_rows):
        raise ValueError(f"rank {rank} exceeds min(columns, shortest slice) = {min(J, min_rows)}")
    if iters < 1:
        raise ValueError("iters must be at least 1")
    rng = np.random.default_rng(seed)
    K = len(slices)
    V = rng.uniform(size=(J, rank))
    H = rng.uniform(size=(rank, rank))
    W = np.ones((K, rank))
    projections = {}
    proj = np.empty((K, rank, J))
    losses = []
    for _ in range(iters):
        for k, (sid, rows) in enumerate(slices):
            target = rows @ (V * W[k]) @ H.T
            left, _, right = np.linalg.svd(target, full_matrices=False)
            q = left @ right
            projections[sid] = q
            proj[k] = q.T @ rows
        vtv = V.T @ V
        wtw = W.T @ W
        yv = proj @ V
        rhs_h = np.einsum("krz,kz->rz", yv, W)
        H = ridge_solve(vtv * wtw, rhs_h.T).T
        hth = H.T @ H
        rhs_w = np.einsum("krz,rz->kz", yv, H)
        W = ridge_solve(hth * vtv, rhs_w.T).T
        wtw = W.T @ W
        rhs_v = np.einsum("krj,rz,kz->jz", proj, H, W)
        V = ridge_solve(hth * wtw, rhs_v.T).T
        loss = 0.0
        for k, (sid, rows) in enumerate(slices):
            rec = (projections[sid] @ (H * W[k])) @ V.T
            loss += float(np.sum((rows - rec) ** 2))
        losses.append(loss)
        if len(losses) >= 2:
            prev = losses[-2]
            if prev == 0.0 or abs(prev - loss) <= tol * prev:
                break
    U = {sid: projections[sid] @ H for sid, _ in slices}
    return U, W, V, losses, projections, H


def local_error(batch_items, u_new, W_rows, V):
    """evaluate.py:93-118 with anomaly.slice_error semantics (anomaly.py:23-27).

    ``batch_items``: list of (sid, rows); ``W_rows``: sid -> post-update W row.
    Returns (tensor-level error, per-slice dict)."""
    per = {}
    for sid, rows in batch_items:
        rec = (u_new[sid] * W_rows[sid]) @ V.T
        per[sid] = float(np.abs(rows - rec).mean())
    return float(np.mean([per[sid] for sid, _ in batch_items])), per


def global_error(old_data, old_factors, new_data, new_factors, w_rows, V):
    """evaluate.py:121-144: mean over old slices of mean|rows - (U o w) V^T|
    with the stored old row factors, plus the same over the newest batch."""
    def term(data, factors):
        vals = [float(np.abs(rows - (factors[sid] * w_rows[sid]) @ V.T).mean()) for sid, rows in data.items()]
        return float(np.mean(vals)) if vals else 0.0
    return term(old_data, old_factors) + term(new_data, new_factors)
