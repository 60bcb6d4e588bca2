"""B200-native DASH (dual-way streaming PARAFAC2) update path.

Drop-in for the reference package ``p2stream``'s streaming path
(/root/reference/pkg/src/p2stream/__init__.py): the same entry points and
types, backed by sm_100a CUDA kernels behind the C ABI in include/dash_b200.h.
"""
__version__ = "0.1.0"

from .als import ALSInfo, FactorSet, FactorizationError, parafac2_als, reconstruct, relative_error
from .linalg import RIDGE_EPS, SolveError
from .tensor import (CAUSAL, GLOBAL, ColumnStats, DatasetError, IrregularTensor, NewSlice, SliceMatrix, UpdateBatch,
                     global_stats, normalize_batch, normalize_tensor)


def __getattr__(name):
    # torch-dependent pieces load on first use (keeps `import` light on CPU-only hosts)
    if name in ("StreamState", "UpdateResult", "HelperState", "HostPipeline", "initialize", "init_helpers"):
        from . import stream
        return getattr(stream, name)
    if name == "local_error":
        from .evaluate import local_error
        return local_error
    if name in ("save_state", "load_state"):
        from . import checkpoint
        return getattr(checkpoint, name)
    if name == "ShardedStream":
        from .distributed import ShardedStream
        return ShardedStream
    raise AttributeError(name)


__all__ = [
    "CAUSAL", "ColumnStats", "GLOBAL", "global_stats", "load_state", "normalize_batch", "normalize_tensor",
    "save_state",
    "ALSInfo", "DatasetError", "FactorSet", "FactorizationError", "HelperState", "HostPipeline",
    "IrregularTensor",
    "NewSlice", "RIDGE_EPS", "ShardedStream", "SliceMatrix", "SolveError", "StreamState",
    "UpdateBatch", "UpdateResult", "init_helpers", "initialize", "local_error", "parafac2_als",
    "reconstruct", "relative_error",
]
