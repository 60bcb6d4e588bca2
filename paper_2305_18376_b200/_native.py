"""ctypes binding of the C ABI in include/dash_b200.h (libdash_b200.so).

The shared library is built in-tree by ``build.py`` (nvcc, sm_100a).  There is
no fallback: if the library or a CUDA device is missing, every entry point
raises -- the product path never silently runs anything on the CPU.
"""
from __future__ import annotations

import ctypes
import os
import sys as _sys
import threading
from pathlib import Path

import torch

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libdash_b200.so"

DASH_OK = 0
DASH_E_ARG = 1
DASH_E_CUDA = 2
DASH_E_SINGULAR = 3
DASH_E_NONFINITE = 4
MAX_RANK = 64       # update path
MAX_RANK_ALS = 32   # parafac2_als / init_helpers / ridge_solve
PHASES = ("row_slice", "prologue", "xv", "slices", "fgemm", "sum_fg", "vsolve", "big", "big_post")
PATH_STREAM, PATH_TMA, PATH_BIGX, PATH_SMALLX = 1, 2, 4, 8

_c_dp = ctypes.c_void_p  # device pointers travel as integers


class DashBatch(ctypes.Structure):
    """dash_batch_f64 / dash_batch_f32 (same layout; X is a device pointer)."""
    _fields_ = [
        ("X", _c_dp), ("ldx", ctypes.c_int64), ("N", ctypes.c_int64), ("M", ctypes.c_int32),
        ("row_ptr", _c_dp), ("row_ptr_host", _c_dp), ("state_row", _c_dp), ("is_new", _c_dp),
    ]


class DashState(ctypes.Structure):
    _fields_ = [
        ("W", _c_dp), ("C", _c_dp), ("D", _c_dp), ("V", _c_dp), ("F", _c_dp), ("G", _c_dp),
        ("J", ctypes.c_int32), ("R", ctypes.c_int32), ("forgetting", ctypes.c_double),
        ("passes", ctypes.c_int32),
    ]


class DashStaged(ctypes.Structure):
    """dash_staged: what dash_stage_meta reports about the slot it filled."""
    _fields_ = [
        ("N", ctypes.c_int64), ("M", ctypes.c_int32), ("slot", ctypes.c_int32),
        ("row_ptr", _c_dp), ("state_row", _c_dp), ("is_new", _c_dp), ("row_ptr_host", _c_dp),
        ("nbytes", ctypes.c_int64),
    ]


# exported symbol -> (restype, argtypes); tests check every one is present
SIGNATURES = {
    "dash_ctx_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p)]),
    "dash_ctx_destroy": (None, [ctypes.c_void_p]),
    "dash_ctx_status": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]),
    "dash_ctx_last_launches": (ctypes.c_int, [ctypes.c_void_p]),
    "dash_ctx_path_flags": (ctypes.c_int, [ctypes.c_void_p]),
    "dash_host_row_ptr": (ctypes.c_int, [_c_dp, ctypes.c_int64, _c_dp, ctypes.POINTER(ctypes.c_int64)]),
    "dash_meta_ring_set": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p),
                                          ctypes.POINTER(ctypes.c_void_p), ctypes.c_int64]),
    "dash_stage_meta": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, _c_dp, ctypes.c_int32, _c_dp,
                                       ctypes.c_int32, ctypes.c_int32, _c_dp, ctypes.POINTER(DashStaged)]),
    "dash_stage_release": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "dash_update_f64": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(DashBatch),
                                       ctypes.POINTER(DashState), _c_dp, _c_dp, ctypes.c_double]),
    "dash_update_pass_begin_f64": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(DashBatch),
                                                  ctypes.POINTER(DashState), _c_dp, _c_dp, ctypes.c_double,
                                                  ctypes.c_int32, _c_dp]),
    "dash_update_pass_finish_f64": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(DashState),
                                                   _c_dp, ctypes.c_double]),
    "dash_update_f32": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(DashBatch),
                                       ctypes.POINTER(DashState), _c_dp, _c_dp, ctypes.c_double]),
    "dash_update_pass_begin_f32": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(DashBatch),
                                                  ctypes.POINTER(DashState), _c_dp, _c_dp, ctypes.c_double,
                                                  ctypes.c_int32, _c_dp]),
    "dash_local_error_f32": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(DashBatch),
                                            _c_dp, _c_dp, _c_dp, ctypes.c_int32, ctypes.c_int32,
                                            _c_dp, _c_dp]),
    "dash_ctx_fallbacks": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]),
    "dash_ctx_set_profiling": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "dash_ctx_phase_ms": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(ctypes.c_int32), ctypes.c_int32]),
    "dash_group_update_f64": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                             ctypes.c_int32, ctypes.c_int32] + [_c_dp] * 5 +
                              [ctypes.c_double, ctypes.c_double] + [_c_dp] * 6 +
                              [ctypes.POINTER(ctypes.c_int32)]),
    "dash_ridge_solve_f64": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                            ctypes.c_int32, ctypes.c_int32, _c_dp, _c_dp, _c_dp,
                                            ctypes.c_double]),
    "dash_init_helpers_f64": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(DashBatch),
                                             _c_dp, _c_dp, _c_dp, ctypes.c_int32, ctypes.c_int32,
                                             _c_dp, _c_dp, _c_dp, _c_dp]),
    "dash_local_error_f64": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(DashBatch),
                                            _c_dp, _c_dp, _c_dp, ctypes.c_int32, ctypes.c_int32,
                                            _c_dp, _c_dp]),
    "dash_als_sweep_f64": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(DashBatch),
                                          ctypes.c_int32, ctypes.c_int32] + [_c_dp] * 5 + [ctypes.c_double]),
    "dash_als_project_f64": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                            _c_dp, _c_dp, _c_dp]),
}

_lib = None
_lock = threading.Lock()


class NativeUnavailable(RuntimeError):
    pass


def load_library(path: Path | None = None):
    """Load the shared library and bind every exported symbol (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else Path(os.environ.get("DASH_LIB_PATH", LIB_PATH))
        if not p.exists():
            raise NativeUnavailable(
                f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


_cuda_ok = False


def lib():
    global _cuda_ok
    if not _cuda_ok:
        if not torch.cuda.is_available():
            raise NativeUnavailable("the DASH engine needs a CUDA device (B200); none is visible")
        _cuda_ok = True
    return _lib if _lib is not None else load_library()


_ctx = {}


def context(device: int | None = None):
    """Per-device dash_ctx (workspace arena + error slot)."""
    L = lib()
    dev = torch.cuda.current_device() if device is None else device
    c = _ctx.get(dev)
    if c is None:
        with torch.cuda.device(dev):
            h = ctypes.c_void_p()
            rc = L.dash_ctx_create(ctypes.byref(h))
            if rc != DASH_OK:
                raise RuntimeError(f"dash_ctx_create failed ({rc})")
        c = h
        _ctx[dev] = c
    return c


class OwnedContext:
    """A dash_ctx owned by one StreamState: its workspace arena and plan are
    private, so states updated concurrently on different streams (or host
    threads) never share them.  Destroyed with the owner."""

    def __init__(self, device: int):
        L = lib()
        with torch.cuda.device(device):
            h = ctypes.c_void_p()
            rc = L.dash_ctx_create(ctypes.byref(h))
            if rc != DASH_OK:
                raise RuntimeError(f"dash_ctx_create failed ({rc})")
        self.handle = h
        self._as_parameter_ = h  # pass straight to ctypes calls

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib is not None and not _sys.is_finalizing():
            try:
                _lib.dash_ctx_destroy(h)
            except Exception:
                pass
            self.handle = None


def stream_ptr(stream=None) -> int:
    if stream is None:
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)  # no Stream object per call
        if raw is not None:
            return int(raw(torch.cuda.current_device()))
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def check(rc: int, what: str):
    if rc != DASH_OK:
        raise RuntimeError(f"{what} failed with DASH error {rc}")
