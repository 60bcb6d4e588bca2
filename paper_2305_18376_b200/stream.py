"""Device-resident DASH stream state -- drop-in for the reference's
``StreamState`` / ``initialize`` / ``init_helpers``
(/root/reference/pkg/src/p2stream/stream.py:36-407).

Layout in HBM (torch owns every buffer; the C ABI only sees pointers):

  W (Kcap, R), C (Kcap, R), D (Kcap, R, R)   per-slice rows, slice order = the
                                             reference's registration order;
                                             capacity doubles on growth
  V, F (J, R), G (R, R)                      shared factors / global summaries
  U history                                  one (N_t, R) device block per
                                             update (+ one for the initial
                                             factors); u_blocks / u_matrix
                                             gather lazily
  X staging                                  (Ncap, J) device buffer reused by
                                             every update, fed from a pinned
                                             host buffer

FP32 data mode (``dtype=torch.float32``, north_star's optional FP32 mode):
the streamed data -- the staged batch X and the returned U_new blocks -- are
single precision (half the PCIe and HBM bytes); the per-slice state, the
factors and every product / sum inside the kernels stay FP64
(``dash_update_f32``).

``update(batch)`` validates ids on the host, registers new slices, packs the
batch into CSR (rows in ``batch.items()`` order), and launches the whole pass
loop through ``dash_update_f64``.  It then synchronises once to turn a device
solver failure into ``SolveError(slice_id)`` like the reference.  Host views
(``W``, ``V``, ``C``, ``D``, ``F``, ``G``, ``u_blocks``, ``UpdateResult.u_new``)
are lazy copies, cached until the next mutation.
"""
from __future__ import annotations

import ctypes
import os
import time
from collections.abc import Mapping
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from .als import ALSInfo, FactorSet
from .linalg import RIDGE_EPS, SolveError
from .tensor import IrregularTensor, UpdateBatch

F64 = torch.float64


def _dev(device) -> torch.device:
    if device is None:
        if not torch.cuda.is_available():
            raise nat.NativeUnavailable("the DASH engine needs a CUDA device (B200); none is visible")
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise ValueError("the DASH engine runs on CUDA devices only")
    if d.index is None:
        d = torch.device("cuda", torch.cuda.current_device())
    return d


def _to_dev(a, device) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=F64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=float)), device=device)


def _ptr(t) -> int:
    return int(t.data_ptr()) if t is not None else 0


class _NoGuard:
    def __enter__(self):
        return None

    def __exit__(self, *exc):
        return False


_NO_GUARD = _NoGuard()


def _on(device: torch.device):
    """Make ``device`` current for the library calls (their stream, workspace
    and allocations follow the current device); free when it already is."""
    return _NO_GUARD if torch.cuda.current_device() == device.index else torch.cuda.device(device)


@dataclass
class HelperState:
    """Helper summaries in per-slice map form (stream.py:36-53)."""

    c: dict
    D: dict
    F: np.ndarray
    G: np.ndarray
    forgetting: float

    def __post_init__(self):
        if not 0.0 < self.forgetting <= 1.0:
            raise ValueError("forgetting factor must lie in (0, 1]")


class _UNew(Mapping):
    """``UpdateResult.u_new``: slice id -> (n_k, R) rows, copied from the
    device on first access (one D2H for the whole update)."""

    def __init__(self, ids, row_ptr, U_dev):
        self._ids = ids
        self._index = {sid: k for k, sid in enumerate(ids)}
        self._row_ptr = row_ptr
        self._dev = U_dev
        self._host = None

    def _h(self):
        if self._host is None:
            self._host = self._dev.cpu().numpy()
        return self._host

    def __getitem__(self, sid):
        k = self._index[sid]
        return self._h()[self._row_ptr[k]:self._row_ptr[k + 1]]

    def __iter__(self):
        return iter(self._ids)

    def __len__(self):
        return len(self._ids)

    @property
    def device_tensor(self) -> torch.Tensor:
        return self._dev


@dataclass
class UpdateResult:
    """What one consumed batch produced (stream.py:167-181)."""

    update_index: int
    u_new: Mapping
    new_slice_ids: list
    rows_new: int
    seconds: float
    v_used: np.ndarray = None


class _UBlocks(Mapping):
    """``StreamState.u_blocks``: slice id -> list of (rows, R) host blocks."""

    def __init__(self, state):
        self._s = state
        state._flush_ulog()

    def __getitem__(self, sid):
        return [self._s._block_host(ref) for ref in self._s._ublk[sid]]

    def __contains__(self, sid):
        return sid in self._s._ublk

    def __iter__(self):
        return iter(self._s._ublk)

    def __len__(self):
        return len(self._s._ublk)


_POOL = None

try:  # host-side gather in C (csrc/host_gather.c, built by build.py); numpy path if it is not built
    from . import _dashhost
except ImportError:  # pragma: no cover
    _dashhost = None


def _gather_plan(plan, row_ptr, out, on_chunk=None):
    """_gather_rows through the C helper: the batch's blocks land in the pinned
    buffer share by share (each share copied by several threads with the GIL
    released); ``on_chunk(lo, hi)`` starts a share's upload behind the next
    share's copy."""
    M = len(row_ptr) - 1
    N = int(row_ptr[M])
    T = min(int(os.environ.get("DASH_GATHER_THREADS", "8")), os.cpu_count() or 1)
    shares = 1 if N * out.shape[1] < (1 << 22) else 4
    cut = np.searchsorted(row_ptr, np.linspace(0, N, shares + 1).astype(np.int64))
    cut[0], cut[-1] = 0, M
    cut = np.unique(cut)
    for a, b in zip(cut[:-1], cut[1:]):
        lo, hi = int(row_ptr[a]), int(row_ptr[b])
        _dashhost.copy(plan, int(a), int(b), out, lo, T, 1 if out.dtype == np.float32 else 0)
        if on_chunk is not None:
            on_chunk(lo, hi)


def _gather_rows(arrs, row_ptr, out, on_chunk=None):
    """Concatenate the batch's per-slice row blocks into the pinned staging
    buffer: one np.concatenate per contiguous share of the rows, on a small
    thread pool (numpy releases the GIL for the copies), so the host gather
    of a large batch runs at several GB/s instead of one core's.
    ``on_chunk(lo, hi)`` is called in row order as each share lands (the
    caller starts that share's host->device copy behind the others' gathers)."""
    global _POOL
    N = out.shape[0]
    T = min(8, os.cpu_count() or 1)
    if T <= 1 or N * out.shape[1] < (1 << 22) or len(arrs) < 2 * T:
        np.concatenate(arrs, axis=0, out=out)
        if on_chunk is not None:
            on_chunk(0, N)
        return
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max_workers=T, thread_name_prefix="dash-gather")
    cut = np.searchsorted(row_ptr, np.linspace(0, N, T + 1).astype(np.int64))
    cut[0], cut[-1] = 0, len(arrs)
    cut = np.unique(cut)
    jobs = [(int(row_ptr[a]), int(row_ptr[b]), _POOL.submit(np.concatenate, arrs[a:b], 0,
                                                             out[row_ptr[a]:row_ptr[b]]))
            for a, b in zip(cut[:-1], cut[1:]) if b > a]
    for lo, hi, f in jobs:
        f.result()
        if on_chunk is not None:
            on_chunk(lo, hi)


class _Meta:
    """One staged batch's index arrays (dash_stage_meta): raw pointers for the
    launch, torch / numpy views built only when somebody asks (local_error)."""
    __slots__ = ("M", "N", "rp", "sr", "nw", "rp_host", "nbytes", "_slot", "_keep")

    def __init__(self, st: "nat.DashStaged", slot, keep):
        self.M, self.N = int(st.M), int(st.N)
        self.rp, self.sr, self.nw, self.rp_host = st.row_ptr, st.state_row, st.is_new, st.row_ptr_host
        self.nbytes = int(st.nbytes)
        self._slot = slot    # (pinned bytes, device bytes) of the ring slot
        self._keep = keep    # (arena, lo) of the persistent device copy, or None

    def _dev_bytes(self):
        if self._keep is not None:  # outlives the ring
            a, lo = self._keep
            return a[lo:lo + self.nbytes]
        return self._slot[1][:self.nbytes]

    def __getitem__(self, i):  # (row_ptr, state_row, is_new) device views
        M = self.M
        o_sr = 8 * (M + 1)
        o_nw = o_sr + ((4 * M + 7) // 8) * 8
        db = self._dev_bytes()
        return (db[:o_sr].view(torch.int64), db[o_sr:o_sr + 4 * M].view(torch.int32), db[o_nw:o_nw + M])[i]

    def host_row_ptr(self) -> np.ndarray:
        """Pinned host view of row_ptr: valid until the ring wraps (3 updates)."""
        return self._slot[0].numpy()[:8 * (self.M + 1)].view(np.int64)


class StreamState:
    """Factors plus helper summaries of a live stream, resident on one GPU
    (stream.py:184-247).  Exclusively owned during an update."""

    def __init__(self, slice_ids, u_blocks, W, V, C, D, F, G, forgetting,
                 update_index: int = 0, passes: int = 1, device=None, dtype=F64,
                 keep_u_history: bool = True):
        if not 0.0 < forgetting <= 1.0:
            raise ValueError("forgetting factor must lie in (0, 1]")
        if passes < 1:
            raise ValueError("passes must be at least 1")
        self.device = _dev(device)
        self.dtype = torch.float32 if dtype in (torch.float32, np.float32, "float32", "fp32") else F64
        self.forgetting = float(forgetting)
        self.update_index = int(update_index)
        self.passes = int(passes)
        # the reference keeps every U block (stream.py:352-360); a serving loop
        # that never reads u_blocks can drop them (u_blocks then raises)
        self.keep_u_history = bool(keep_u_history)
        self.slice_ids = list(slice_ids)
        self._rowmap = {sid: k for k, sid in enumerate(self.slice_ids)}
        self._rowmap_n = len(self.slice_ids)  # slice_ids[:n] are in _rowmap (the rest register lazily)
        V = _to_dev(V, self.device)
        self.J, R = V.shape
        if R > nat.MAX_RANK:
            raise ValueError(f"rank {R} exceeds the engine's maximum {nat.MAX_RANK}")
        self._R = R
        self._V, self._F, self._G = V, _to_dev(F, self.device), _to_dev(G, self.device)
        K = len(self.slice_ids)
        self._K = K
        cap = max(16, K + K // 4)
        self._Wd = torch.empty((cap, R), dtype=F64, device=self.device)
        self._Cd = torch.empty((cap, R), dtype=F64, device=self.device)
        self._Dd = torch.empty((cap, R, R), dtype=F64, device=self.device)
        if K:
            self._Wd[:K] = _to_dev(W, self.device).reshape(K, R)
            self._Cd[:K] = _to_dev(C, self.device).reshape(K, R)
            self._Dd[:K] = _to_dev(D, self.device).reshape(K, R, R)
        # U history: list of device blocks; per slice a list of (block, lo, hi)
        self._ustore: list = []
        self._uhost: dict = {}
        self._ublk: dict = {}
        # per update, (U block index, device copy of the batch's index arrays, M):
        # resolved into _ublk only when the U history is read, so an update
        # costs no per-slice host work (stream.py:352-360 appends per slice)
        self._ulog: list = []
        self._unchecked = False  # an update_packed(check=False) may have latched a device error
        self._uarena = None  # [chunk (rows, R), rows used]: U blocks are views of chunks
        self._marena = None  # [chunk (bytes,), bytes used]: per-update index arrays of the U history
        if u_blocks is not None:
            self._ingest_u_blocks(u_blocks)
        self._X = None
        self._Xpin = None
        self._pin_event = None
        self._cache: dict = {}
        self._last = None  # last update's device batch (for local_error)
        self._ctx = nat.OwnedContext(self.device.index)  # private workspace: one update in flight per state

    # -- construction helpers ----------------------------------------------
    def _ingest_u_blocks(self, u_blocks):
        sids = [s for s in self.slice_ids if s in u_blocks]
        arrs, spans = [], []
        off = 0
        for sid in sids:
            for blk in u_blocks[sid]:
                a = np.asarray(blk, dtype=float).reshape(-1, self._R)
                arrs.append(a)
                spans.append((sid, off, off + a.shape[0]))
                off += a.shape[0]
        for sid in sids:
            self._ublk.setdefault(sid, [])
        if off:
            dev = torch.as_tensor(np.concatenate(arrs), device=self.device)
            self._ustore.append(dev)
            bi = len(self._ustore) - 1
            for sid, lo, hi in spans:
                self._ublk[sid].append((bi, lo, hi))

    @classmethod
    def from_arrays(cls, arrays: dict, device=None, u_blocks=None, dtype=F64) -> "StreamState":
        """Build from a dict with slice_ids, W, V, C, D, F, G, forgetting
        (e.g. ``workloads.planted_state``); U history starts empty unless
        ``u_blocks`` is given."""
        R = np.asarray(arrays["V"]).shape[1]
        if u_blocks is None:
            u_blocks = {sid: [np.zeros((0, R))] for sid in arrays["slice_ids"]}
        return cls(arrays["slice_ids"], u_blocks, arrays["W"], arrays["V"], arrays["C"],
                   arrays["D"], arrays["F"], arrays["G"], arrays["forgetting"],
                   passes=arrays.get("passes", 1), device=device, dtype=dtype)

    @property
    def _row_of(self) -> dict:
        """slice id -> state row.  Registration appends to ``slice_ids`` only;
        the map catches up here, on first use (the device fast path never
        needs it, and 500 dict inserts cost ~100 us of host time per update)."""
        ids, d = self.slice_ids, self._rowmap
        if self._rowmap_n < len(ids):
            d.update(zip(ids[self._rowmap_n:], range(self._rowmap_n, len(ids))))
            self._rowmap_n = len(ids)
        return d

    # -- reference attribute API --------------------------------------------
    @property
    def rank(self) -> int:
        return self._R

    def row_of(self, slice_id) -> int:
        return self._row_of[slice_id]

    def has_slice(self, slice_id) -> bool:
        return slice_id in self._row_of

    def _host(self, name, t):
        v = self._cache.get(name)
        if v is None:
            v = t.cpu().numpy()
            self._cache[name] = v
        return v

    @property
    def W(self) -> np.ndarray:
        return self._host("W", self._Wd[:self._K])

    @W.setter
    def W(self, value):
        self._Wd[:self._K] = _to_dev(value, self.device).reshape(self._K, self._R)
        self._cache.clear()

    @property
    def C(self) -> np.ndarray:
        return self._host("C", self._Cd[:self._K])

    @C.setter
    def C(self, value):
        self._Cd[:self._K] = _to_dev(value, self.device).reshape(self._K, self._R)
        self._cache.clear()

    @property
    def D(self) -> np.ndarray:
        return self._host("D", self._Dd[:self._K])

    @D.setter
    def D(self, value):
        self._Dd[:self._K] = _to_dev(value, self.device).reshape(self._K, self._R, self._R)
        self._cache.clear()

    @property
    def V(self) -> np.ndarray:
        return self._host("V", self._V)

    @V.setter
    def V(self, value):
        self._V = _to_dev(value, self.device)
        self._cache.clear()

    @property
    def F(self) -> np.ndarray:
        return self._host("F", self._F)

    @F.setter
    def F(self, value):
        self._F = _to_dev(value, self.device)
        self._cache.clear()

    @property
    def G(self) -> np.ndarray:
        return self._host("G", self._G)

    @G.setter
    def G(self, value):
        self._G = _to_dev(value, self.device)
        self._cache.clear()

    # device views (no copy)
    @property
    def device_tensors(self) -> dict:
        K = self._K
        return {"W": self._Wd[:K], "C": self._Cd[:K], "D": self._Dd[:K],
                "V": self._V, "F": self._F, "G": self._G}

    @property
    def u_blocks(self) -> Mapping:
        return _UBlocks(self)

    def _block_host(self, ref):
        bi, lo, hi = ref
        h = self._uhost.get(bi)
        if h is None:
            h = self._ustore[bi].cpu().numpy()
            self._uhost[bi] = h
        return h[lo:hi]

    def u_history_device(self, slice_ids) -> torch.Tensor:
        """U histories of ``slice_ids`` concatenated in that order (one device
        gather; the CSR companion of a DeviceTensor with the same slices)."""
        self._flush_ulog()
        parts = [self._ustore[bi][lo:hi] for sid in slice_ids for bi, lo, hi in self._ublk[sid]]
        if not parts:
            return torch.zeros((0, self._R), dtype=self.dtype, device=self.device)
        return torch.cat(parts)

    def u_matrix(self, slice_id) -> np.ndarray:
        blocks = self.u_blocks[slice_id]
        return blocks[0].copy() if len(blocks) == 1 else np.vstack(blocks)

    def factor_set(self) -> FactorSet:
        return FactorSet(slice_ids=list(self.slice_ids),
                         U={sid: self.u_matrix(sid) for sid in self.slice_ids},
                         W=self.W.copy(), V=self.V.copy())

    @property
    def helpers(self) -> HelperState:
        C, D = self.C, self.D
        return HelperState(c={sid: C[k].copy() for k, sid in enumerate(self.slice_ids)},
                           D={sid: D[k].copy() for k, sid in enumerate(self.slice_ids)},
                           F=self.F.copy(), G=self.G.copy(), forgetting=self.forgetting)

    # -- growth ---------------------------------------------------------------
    def _reserve(self, K_new: int):
        cap = self._Wd.shape[0]
        if K_new <= cap:
            return
        ncap = max(K_new, cap * 2)
        R = self._R
        for name, shape in (("_Wd", (ncap, R)), ("_Cd", (ncap, R)), ("_Dd", (ncap, R, R))):
            old = getattr(self, name)
            new = torch.empty(shape, dtype=F64, device=self.device)
            new[:self._K] = old[:self._K]
            setattr(self, name, new)

    def _stage_x(self, N: int):
        J = self.J
        if self._X is None or self._X.shape[0] < N:
            cap = max(N, 1024, int(N * 1.25))
            self._X = torch.empty((cap, J), dtype=self.dtype, device=self.device)
        if self._Xpin is None or self._Xpin.shape[0] < N:
            cap = max(N, 1024, int(N * 1.25))
            self._Xpin = torch.empty((cap, J), dtype=self.dtype, pin_memory=True)
            self._pin_event = None
        if self._pin_event is not None:
            self._pin_event.synchronize()  # previous H2D from the staging buffer is done
        return self._Xpin, self._X

    # -- the update -----------------------------------------------------------
    def update(self, batch: UpdateBatch) -> UpdateResult:
        """Consume one batch (stream.py:251-370): same validation, same
        registration order, same results within FP64 rounding.  Accepts this
        package's UpdateBatch or the reference's (anything with
        ``existing_rows`` / ``new_slices``, or with ``items()``)."""
        with _on(self.device):
            if self._unchecked:  # report a failure latched by an earlier unchecked update first
                self.check()
            if hasattr(batch, "existing_rows") and hasattr(batch, "new_slices"):
                ex = batch.existing_rows
                return self._update_lists(list(ex.keys()), list(ex.values()),
                                          [ns.slice_id for ns in batch.new_slices],
                                          [ns.rows for ns in batch.new_slices])
            return self._update_items(batch.items())

    def _update_items(self, items, allreduce=None) -> UpdateResult:
        """Generic form: (sid, rows, is_new) in items() order (existing first)."""
        ex_ids, ex_rows, new_ids, new_rows = [], [], [], []
        for sid, rows, is_new in items:
            if is_new:
                new_ids.append(sid)
                new_rows.append(rows)
            else:
                if new_ids:
                    raise ValueError("batch items must list existing slices before new ones")
                ex_ids.append(sid)
                ex_rows.append(rows)
        return self._update_lists(ex_ids, ex_rows, new_ids, new_rows, allreduce=allreduce)

    def _update_lists(self, ex_ids, ex_rows, new_ids, new_rows, allreduce=None) -> UpdateResult:
        started = time.perf_counter()
        rowmap = self._row_of
        J = self.J
        # validation (stream.py:262-268), vectorised over the entries
        bad = [sid for sid in new_ids if sid in rowmap]
        if bad:
            raise ValueError(f"batch declares known slice {bad[0]!r} as new")
        bad = [sid for sid in ex_ids if sid not in rowmap]
        if bad:
            raise ValueError(f"batch references unknown existing slice {bad[0]!r}")
        ids = ex_ids + new_ids
        M = len(ids)
        arrs = ex_rows + new_rows
        plan, counts = None, None
        if _dashhost is not None:
            # one C pass over the blocks: shape / dtype / layout check and the row counts
            counts = np.empty(M, dtype=np.int64)
            plan = _dashhost.scan(arrs, J, counts)
        if plan is None or isinstance(plan, int):
            # a block that is not a C-contiguous float64 (n, J) array: convert, re-check, report
            arrs = [np.ascontiguousarray(r, dtype=float) for r in arrs]
            bad = [k for k, r in enumerate(arrs) if r.ndim != 2 or r.shape[1] != J]
            if bad:
                raise ValueError(f"slice {ids[bad[0]]!r}: rows must be (n, {J})")
            counts = np.fromiter((r.shape[0] for r in arrs), dtype=np.int64, count=M)
            plan = _dashhost.scan(arrs, J, counts) if _dashhost is not None else None
        existing_rows = np.fromiter((rowmap[sid] for sid in ex_ids), dtype=np.int32, count=len(ex_ids))
        meta = self._stage_meta(counts, existing_rows, len(new_ids))
        N = meta.N
        row_ptr = meta.host_row_ptr().copy()  # kept by UpdateResult / local_error beyond the ring's lifetime
        # registration (stream.py:270-280): new rows appended in batch order
        self._register(new_ids)

        pin, X = self._stage_x(N)
        if N:
            def upload(lo, hi):  # each share's H2D starts as soon as its rows are gathered
                X[lo:hi].copy_(pin[lo:hi], non_blocking=True)
            if plan is not None and not isinstance(plan, int):
                _gather_plan(plan, row_ptr, pin.numpy()[:N], upload)
            else:
                _gather_rows(arrs, row_ptr, pin.numpy()[:N], upload)
            ev = torch.cuda.Event()
            ev.record()
            self._pin_event = ev
        U_dev, v_used = self._run(X, meta, check=True, ids=ids, allreduce=allreduce)
        self.update_index += 1
        self._last = (ids, row_ptr, meta, X, N, U_dev)
        return UpdateResult(
            update_index=self.update_index,
            u_new=_UNew(ids, row_ptr, U_dev),
            new_slice_ids=list(new_ids),
            rows_new=N,
            seconds=time.perf_counter() - started,
            v_used=v_used.cpu().numpy(),
        )

    def update_packed(self, X: torch.Tensor, counts: np.ndarray, existing_rows: np.ndarray,
                      new_ids: list, check: bool = False, allreduce=None):
        """Device-resident fast path: ``X`` (N, J) already on this GPU (in the
        state's dtype) in batch order -- existing slices (state rows ``existing_rows``) then the
        ``len(new_ids)`` new slices; ``counts`` their row counts.  No host sync
        unless ``check``.  Returns (U_new (N, R), v_used (J, R)) device tensors."""
        with _on(self.device):
            meta = self._stage_meta(counts, existing_rows, len(new_ids))
            self._register(new_ids)
            U_dev, v_used = self._run(X, meta, check=check, ids=None, allreduce=allreduce)
        self.update_index += 1
        self._last = (None, None, meta, X, meta.N, U_dev)  # row_ptr: meta.host_row_ptr() on demand
        return U_dev, v_used

    @property
    def last_launches(self) -> int:
        """Library kernels launched by the last update (bench's gpu_launches)."""
        return int(nat.lib().dash_ctx_last_launches(self._ctx))

    def _register(self, new_ids):
        """stream.py:270-280: new slices take the next state rows, in batch order."""
        L = len(new_ids)
        self._reserve(self._K + L)
        self.slice_ids.extend(new_ids)  # _row_of catches up lazily
        self._K += L

    def _run(self, X, meta, check, ids, allreduce=None):
        dev = self.device
        M, N = meta.M, meta.N
        if N and X.dtype != self.dtype:
            raise TypeError(f"batch X is {X.dtype}, the stream state runs in {self.dtype}")
        if N and X.shape[0] < N:
            raise ValueError(f"batch X has {X.shape[0]} rows, the counts sum to {N}")
        f32 = self.dtype == torch.float32
        U = self._alloc_u(N)
        v_used = torch.empty((self.J, self._R), dtype=F64, device=dev)
        # the two argument structs are reused across updates (building ctypes structs and reading six
        # data pointers per update is measurable on a host-bound stream); the state struct is refreshed
        # whenever a state tensor was replaced (capacity growth, a setter)
        b = self.__dict__.get("_cbatch")
        if b is None:
            b = self._cbatch = nat.DashBatch()
        b.X, b.ldx, b.N, b.M = _ptr(X), (int(X.stride(0)) if N else self.J), N, M
        b.row_ptr, b.row_ptr_host, b.state_row, b.is_new = meta.rp, meta.rp_host, meta.sr, meta.nw
        key = (self._Wd, self._Cd, self._Dd, self._V, self._F, self._G)
        cs = self.__dict__.get("_cstate")
        if cs is None or any(a is not c for a, c in zip(cs[1], key)):
            cs = self._cstate = (nat.DashState(W=_ptr(self._Wd), C=_ptr(self._Cd), D=_ptr(self._Dd),
                                               V=_ptr(self._V), F=_ptr(self._F), G=_ptr(self._G), J=self.J,
                                               R=self._R, forgetting=self.forgetting, passes=self.passes), key)
        s = cs[0]
        s.forgetting, s.passes = self.forgetting, self.passes
        L = nat.lib()
        st = nat.stream_ptr()
        upd = L.dash_update_f32 if f32 else L.dash_update_f64
        begin = L.dash_update_pass_begin_f32 if f32 else L.dash_update_pass_begin_f64
        if allreduce is None:
            nat.check(upd(self._ctx, st, ctypes.byref(b), ctypes.byref(s), _ptr(U), _ptr(v_used), RIDGE_EPS),
                      "dash_update_f32" if f32 else "dash_update_f64")
        else:
            # sharded: per pass, local fresh sums -> all-reduce -> replicated finish
            fg = torch.empty(self.J * self._R + self._R * self._R, dtype=F64, device=dev)
            for p in range(self.passes):
                nat.check(begin(self._ctx, st, ctypes.byref(b), ctypes.byref(s),
                                _ptr(U), _ptr(v_used), RIDGE_EPS, p, _ptr(fg)), "dash_update_pass_begin")
                allreduce(fg)
                nat.check(L.dash_update_pass_finish_f64(self._ctx, st, ctypes.byref(s), _ptr(fg),
                                                        RIDGE_EPS), "dash_update_pass_finish_f64")
        # U history (stream.py:352-360): keep U and a device copy of this
        # batch's index arrays; the per-slice refs are built on first read
        if self.keep_u_history:
            self._ustore.append(U)
            self._ulog.append((len(self._ustore) - 1, meta, M))
        # (the update's last pass_finish released the staging slot: dash_b200.h)
        self._cache.clear()
        self._err_ids = ids
        if check:
            self.check()
        else:
            self._unchecked = True
        return U, v_used

    _U_ALIGN = 32  # rows: every U block starts 256-byte aligned

    def _alloc_u(self, N: int) -> torch.Tensor:
        """U_new block of this update.  With the U history kept, blocks are
        carved from large device chunks (one allocation per several updates
        instead of one per update: a fresh cudaMalloc of ~100 MB inside the
        update costs more than the update's own kernels)."""
        R = self._R
        if not self.keep_u_history:
            return torch.empty((max(N, 0), R), dtype=self.dtype, device=self.device)
        a = self._uarena
        need = max(N, 0)
        if a is None or a[1] + need > a[0].shape[0]:
            # chunks double (up to ~2 GB) so a long stream allocates O(log) times, not every 4th update
            prev = 0 if a is None else a[0].shape[0]
            cap = (2 << 30) // (8 * R)
            self._new_u_chunk(max(4 * need, min(2 * prev, cap), 1 << 14))
            a = self._uarena
        lo = a[1]
        a[1] = lo + (need + self._U_ALIGN - 1) // self._U_ALIGN * self._U_ALIGN
        return a[0][lo:lo + need]

    def _keep_room(self, n: int):
        """(arena, lo): ``n`` bytes of the index-array arena for the U history
        (dash_stage_meta copies the packed block there; no allocation per
        update: a fresh cudaMalloc can stall the host behind the GPU)."""
        a = self._marena
        if a is None or a[1] + n > a[0].shape[0]:
            self._marena = a = [torch.empty(max(16 * n, 1 << 24), dtype=torch.uint8, device=self.device), 0]
        lo = a[1]
        a[1] = lo + (n + 255) // 256 * 256
        return a[0], lo

    def _new_u_chunk(self, rows: int):
        self._uarena = [torch.empty((rows, self._R), dtype=self.dtype, device=self.device), 0]

    def reserve_u_history(self, rows: int):
        """Pre-allocate device room for ``rows`` more U-history rows (plus
        alignment padding), so the following updates allocate nothing."""
        a = self._uarena
        free = 0 if a is None else a[0].shape[0] - a[1]
        if rows > free:
            with _on(self.device):
                self._new_u_chunk(int(rows * 1.02) + 64 * self._U_ALIGN)

    def _flush_ulog(self):
        """Resolve the pending per-update U records into slice -> [(block, lo, hi)]."""
        if not self._ulog:
            return
        pending, self._ulog = self._ulog, []
        ids = self.slice_ids
        for bi, meta, M in pending:
            hb = meta._dev_bytes().cpu().numpy()
            o_sr = 8 * (M + 1)
            rp = hb[:o_sr].view(np.int64)
            sr = hb[o_sr:o_sr + 4 * M].view(np.int32)
            for m in range(M):
                self._ublk.setdefault(ids[int(sr[m])], []).append((bi, int(rp[m]), int(rp[m + 1])))

    _META_RING = 3  # updates whose index arrays stay valid (local_error reads the last one)

    def _stage_meta(self, counts, existing_rows, L) -> _Meta:
        """Stage the batch's CSR index arrays -- row_ptr (M+1) i64 | state_row
        (M) i32 | is_new (M) u8 -- through the library's ring (dash_stage_meta):
        prefix sum written straight into a pinned slot, ONE host-to-device copy
        on a side stream (it runs while the previous update's kernels still
        execute; the update's first kernel follows with only an event wait),
        and, with the U history kept, a device copy into the history's index
        arena.  The host never waits for the GPU unless the ring wraps onto a
        copy still in flight; a device slot is rewritten only after the update
        that read it has been issued (dash_stage_release).  One native call per
        update: the Python-side ring this replaces cost ~90 us of interpreter
        and torch-call overhead per update, more than a medium-sized update's
        kernels."""
        counts = np.ascontiguousarray(counts, dtype=np.int64)
        existing_rows = np.ascontiguousarray(existing_rows, dtype=np.int32)
        M_old = existing_rows.shape[0]
        M = M_old + L
        if counts.shape[0] != M:
            raise ValueError(f"{counts.shape[0]} counts for {M_old} existing + {L} new slices")
        nbytes = 8 * (M + 1) + ((4 * M + 7) // 8) * 8 + M
        ring = getattr(self, "_meta_ring", None)
        lib = nat.lib()
        if ring is None or ring[0][0].shape[0] < nbytes:
            cap = max(4096, int(nbytes * 1.25) + 64)
            if ring is not None:
                torch.cuda.current_stream(self.device).synchronize()  # old slots may still be read
            ring = [(torch.empty(cap, dtype=torch.uint8, pin_memory=True),
                     torch.empty(cap, dtype=torch.uint8, device=self.device)) for _ in range(self._META_RING)]
            pins = (ctypes.c_void_p * len(ring))(*[t[0].data_ptr() for t in ring])
            devs = (ctypes.c_void_p * len(ring))(*[t[1].data_ptr() for t in ring])
            nat.check(lib.dash_meta_ring_set(self._ctx, len(ring), pins, devs, cap), "dash_meta_ring_set")
            self._meta_ring = ring
        keep = self._keep_room(nbytes) if self.keep_u_history else None
        out = nat.DashStaged()
        rc = lib.dash_stage_meta(self._ctx, nat.stream_ptr(), counts.ctypes.data, M_old,
                                 existing_rows.ctypes.data if M_old else None, L, self._K,
                                 keep[0].data_ptr() + keep[1] if keep is not None else None, ctypes.byref(out))
        if rc == nat.DASH_E_ARG:
            raise ValueError("row counts must be non-negative")
        nat.check(rc, "dash_stage_meta")
        return _Meta(out, ring[out.slot], keep)

    def check(self):
        """Synchronise and raise SolveError for a device-side solver failure."""
        pos = ctypes.c_int64(0)
        with _on(self.device):
            rc = nat.lib().dash_ctx_status(self._ctx, nat.stream_ptr(), ctypes.byref(pos))
        self._unchecked = False
        if rc == nat.DASH_OK:
            return
        if rc == nat.DASH_E_CUDA:
            raise RuntimeError("CUDA error during the DASH update")
        p = pos.value
        ids = getattr(self, "_err_ids", None)
        sid = None if p < 0 or ids is None or p >= len(ids) else ids[p]
        msg = ("singular normal equations" if rc == nat.DASH_E_SINGULAR
               else "non-finite solution from normal equations")
        if ids is None and p >= 0:
            msg += f" (batch position {p} of an unchecked update_packed batch)"
        raise SolveError(msg, sid)


class HostPipeline:
    """Overlapped host-memory feeding of ``update_packed`` (serving loop).

    ``put(X_host)`` copies a pinned host batch into one of ``depth`` device
    buffers on a dedicated H2D stream; ``update(staged, ...)`` makes the
    compute stream wait for that copy (an event, no host sync), runs the
    update, and starts the read-back of U_new / v_used into caller-provided
    pinned buffers on a D2H stream.  So batch t+1's upload and batch t-1's
    read-back run while batch t is being updated; a buffer is reused only
    after the update that read it has finished (event-ordered).  ``engine`` is
    a StreamState or a ShardedStream (anything with ``update_packed``).

    ``depth`` = device staging buffers.  With 2, the upload of batch t+2 waits
    for update t (buffer reuse), and update t itself waits for its small
    index-array copy, which the copy engine serialises behind the large upload
    of batch t+1 -- the engine idles for one update per step.  3 keeps the
    host->device engine busy back to back (PCIe-bound serving).
    """

    class Staged:
        __slots__ = ("slot", "X", "ready")

        def __init__(self, slot, X, ready):
            self.slot, self.X, self.ready = slot, X, ready

    def __init__(self, engine, max_rows: int, J: int, device=None, depth: int = 3):
        self.engine = engine
        dev = _dev(device)
        self.device = dev
        self.depth = depth
        dt = getattr(engine, "dtype", F64)
        self.bufs = [torch.empty((max(int(max_rows), 1), J), dtype=dt, device=dev) for _ in range(depth)]
        self.h2d = torch.cuda.Stream(dev)
        self.d2h = torch.cuda.Stream(dev)
        self._free = [None] * depth
        self._k = 0

    def start(self):
        """Order the side streams after everything already queued on the compute stream."""
        cur = torch.cuda.current_stream(self.device)
        self.h2d.wait_stream(cur)
        self.d2h.wait_stream(cur)

    def put(self, X_host: torch.Tensor) -> "HostPipeline.Staged":
        slot = self._k % self.depth
        self._k += 1
        N = int(X_host.shape[0])
        if N > self.bufs[slot].shape[0]:
            raise ValueError(f"batch of {N} rows exceeds the pipeline's max_rows {self.bufs[slot].shape[0]}")
        X = self.bufs[slot][:N]
        with torch.cuda.stream(self.h2d):
            if self._free[slot] is not None:
                self.h2d.wait_event(self._free[slot])
            X.copy_(X_host, non_blocking=True)
            ready = torch.cuda.Event()
            ready.record(self.h2d)
        return HostPipeline.Staged(slot, X, ready)

    def update(self, staged, counts, existing_rows, new_ids, U_host=None, v_host=None):
        cur = torch.cuda.current_stream(self.device)
        cur.wait_event(staged.ready)
        U, v_used = self.engine.update_packed(staged.X, counts, existing_rows, new_ids)
        done = torch.cuda.Event()
        done.record(cur)
        self._free[staged.slot] = done
        if U_host is not None or v_host is not None:
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(done)
                # the allocator must not hand U / v_used to a later update
                # before these queued reads ran
                U.record_stream(self.d2h)
                v_used.record_stream(self.d2h)
                if U_host is not None:
                    U_host[:U.shape[0]].copy_(U, non_blocking=True)
                if v_host is not None:
                    v_host.copy_(v_used, non_blocking=True)
        return U, v_used

    def finish(self):
        """Make the compute stream wait for every queued copy (no host sync)."""
        cur = torch.cuda.current_stream(self.device)
        cur.wait_stream(self.h2d)
        cur.wait_stream(self.d2h)


def init_helpers(tensor: IrregularTensor, factors: FactorSet, forgetting: float = 0.7,
                 device=None) -> HelperState:
    """stream.py:56-82 on the GPU: c_k, D_k per slice and F, G."""
    dev = _dev(device)
    res = _init_helpers_device(tensor, factors, dev)
    C, D, F, G = (t.cpu().numpy() for t in res)
    ids = [s.slice_id for s in tensor.slices]
    return HelperState(c={sid: C[k] for k, sid in enumerate(ids)},
                       D={sid: D[k] for k, sid in enumerate(ids)}, F=F, G=G,
                       forgetting=forgetting)


def _init_helpers_device(tensor, factors, dev):
    slices = list(tensor.slices)
    J = tensor.column_count
    R = factors.rank
    for s in slices:
        if factors.U[s.slice_id].shape[0] != s.row_count:
            raise ValueError(f"factor block {s.slice_id!r} does not match slice rows")
    counts = np.array([s.row_count for s in slices], dtype=np.int64)
    row_ptr = np.zeros(len(slices) + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    X = torch.as_tensor(np.concatenate([s.rows for s in slices]), device=dev)
    U = torch.as_tensor(np.concatenate([factors.U[s.slice_id] for s in slices]), device=dev)
    W = torch.as_tensor(np.stack([factors.s_row(s.slice_id) for s in slices]), device=dev)
    V = torch.as_tensor(np.ascontiguousarray(factors.V), device=dev)
    return init_helpers_packed(X, row_ptr, U, W, V)


def init_helpers_packed(X, row_ptr, U, W, V):
    """init_helpers on device-resident CSR data; returns device (C, D, F, G)."""
    dev = X.device
    K = len(row_ptr) - 1
    J, R = V.shape
    rp_d = torch.as_tensor(row_ptr, device=dev)
    C = torch.empty((K, R), dtype=F64, device=dev)
    D = torch.empty((K, R, R), dtype=F64, device=dev)
    F = torch.empty((J, R), dtype=F64, device=dev)
    G = torch.empty((R, R), dtype=F64, device=dev)
    b = nat.DashBatch(X=_ptr(X), ldx=int(X.stride(0)), N=int(row_ptr[-1]), M=K, row_ptr=_ptr(rp_d),
                      row_ptr_host=row_ptr.ctypes.data, state_row=0, is_new=0)
    L = nat.lib()
    ctx = nat.context(dev.index)
    nat.check(L.dash_init_helpers_f64(ctx, nat.stream_ptr(), ctypes.byref(b), _ptr(U), _ptr(W),
                                      _ptr(V), J, R, _ptr(C), _ptr(D), _ptr(F), _ptr(G)),
              "dash_init_helpers_f64")
    return C, D, F, G


def initialize(tensor: IrregularTensor, rank: int, iters: int = 10, seed: int = 0,
               forgetting: float = 0.7, passes: int = 1, device=None, dtype=F64):
    """stream.py:383-407: parafac2_als fit, init_helpers, wrap as stream state.
    ``dtype=torch.float32`` selects the FP32 data mode for the updates (the
    initial fit itself is FP64)."""
    from .als import parafac2_als
    dev = _dev(device)
    factors, info = parafac2_als(tensor, rank, iters=iters, seed=seed, return_info=True, device=dev)
    C, D, F, G = _init_helpers_device(tensor, factors, dev)
    return StreamState(
        slice_ids=list(factors.slice_ids),
        u_blocks={sid: [factors.U[sid]] for sid in factors.slice_ids},
        W=factors.W, V=factors.V, C=C, D=D, F=F, G=G,
        forgetting=forgetting, update_index=0, passes=passes, device=dev, dtype=dtype,
    ), info
