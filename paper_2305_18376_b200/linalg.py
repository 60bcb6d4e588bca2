"""Ridge constant, error type and symmetrisation shared with the reference
(/root/reference/pkg/src/p2stream/linalg.py:7-22).

The solves themselves run on the GPU (csrc/dash_common.cuh: the symmetric sweep and the
LU fallback; csrc/dash_update.cu: k_vsolve2); this module only
carries the constants and the exception users catch.
"""
from __future__ import annotations

import numpy as np

# Relative ridge added to every Gram-type left-hand side (linalg.py:7).
RIDGE_EPS = 1e-10


class SolveError(ValueError):
    """A normal-equation system could not be solved reliably (linalg.py:10-17)."""

    def __init__(self, message: str, slice_id=None):
        if slice_id is not None:
            message = f"{message} (slice {slice_id!r})"
        super().__init__(message)
        self.slice_id = slice_id


def symmetrize(mat: np.ndarray) -> np.ndarray:
    """Average a (batch of) square matrices with their transposes (linalg.py:20-22)."""
    return (mat + mat.swapaxes(-1, -2)) / 2.0
