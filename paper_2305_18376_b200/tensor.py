"""Input types of the DASH update path -- host-side mirror of the reference's
data model (/root/reference/pkg/src/p2stream/tensor.py:27-171).

These are the objects a p2stream user already builds: an ``IrregularTensor``
of ``SliceMatrix`` for initialisation, and one ``UpdateBatch`` (existing-slice
rows + ``NewSlice`` list) per update.  Same names, fields, validation and
error type as the reference, so batches built for p2stream feed this engine
unchanged.  The engine packs them into a CSR row table (``pack_batch`` in
``stream.py``) before handing them to the device.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class DatasetError(ValueError):
    """Malformed slice data or batch (tensor.py:27-28)."""


@dataclass
class SliceMatrix:
    """One slice: a dense (I_k, J) matrix, one row per time step (tensor.py:31-53)."""

    slice_id: str
    rows: np.ndarray
    first_time_step: int = 0

    def __post_init__(self):
        self.rows = np.asarray(self.rows, dtype=float)
        if self.rows.ndim != 2 or self.rows.shape[0] < 1:
            raise DatasetError(
                f"slice {self.slice_id!r} needs a 2-D matrix with at least one row"
            )

    @property
    def row_count(self) -> int:
        return self.rows.shape[0]

    @property
    def end_step(self) -> int:
        return self.first_time_step + self.rows.shape[0]


class IrregularTensor:
    """Ordered slices sharing a column count (tensor.py:56-113)."""

    def __init__(self, slices):
        slices = list(slices)
        if not slices:
            raise DatasetError("an irregular tensor needs at least one slice")
        column_count = slices[0].rows.shape[1]
        by_id = {}
        for s in slices:
            if s.rows.shape[1] != column_count:
                raise DatasetError(
                    f"slice {s.slice_id!r} has {s.rows.shape[1]} columns, "
                    f"expected {column_count}"
                )
            if s.slice_id in by_id:
                raise DatasetError(f"duplicate slice id {s.slice_id!r}")
            by_id[s.slice_id] = s
        self.slices = slices
        self.column_count = column_count
        self._by_id = by_id

    def __len__(self) -> int:
        return len(self.slices)

    def __iter__(self):
        return iter(self.slices)

    @property
    def slice_ids(self) -> list[str]:
        return [s.slice_id for s in self.slices]

    def get(self, slice_id: str) -> SliceMatrix:
        return self._by_id[slice_id]

    def has(self, slice_id: str) -> bool:
        return slice_id in self._by_id

    @property
    def total_rows(self) -> int:
        return sum(s.row_count for s in self.slices)


@dataclass
class NewSlice:
    """A slice that starts inside an update window (tensor.py:116-125)."""

    slice_id: str
    rows: np.ndarray
    first_time_step: int

    def __post_init__(self):
        self.rows = np.asarray(self.rows, dtype=float)


@dataclass
class UpdateBatch:
    """One update's payload: new rows of existing slices plus new slices
    (tensor.py:128-171).  ``items()`` yields existing entries in dict order,
    then new slices -- the order the engine registers and processes them."""

    update_index: int
    existing_rows: dict
    new_slices: list
    cycle_span: tuple

    def __post_init__(self):
        self.existing_rows = {
            sid: np.asarray(mat, dtype=float) for sid, mat in self.existing_rows.items()
        }
        for sid, mat in self.existing_rows.items():
            if mat.ndim != 2 or mat.shape[0] < 1:
                raise DatasetError(f"existing-rows entry {sid!r} must be a nonempty matrix")
        new_ids = set()
        for ns in self.new_slices:
            if ns.slice_id in self.existing_rows or ns.slice_id in new_ids:
                raise DatasetError(f"new slice id {ns.slice_id!r} collides inside the batch")
            new_ids.add(ns.slice_id)
        if not self.existing_rows and not self.new_slices:
            raise DatasetError("an update batch cannot be empty")

    @property
    def total_new_rows(self) -> int:
        rows = sum(m.shape[0] for m in self.existing_rows.values())
        return rows + sum(ns.rows.shape[0] for ns in self.new_slices)

    @property
    def slice_count(self) -> int:
        return len(self.existing_rows) + len(self.new_slices)

    def items(self):
        for sid, mat in self.existing_rows.items():
            yield sid, mat, False
        for ns in self.new_slices:
            yield ns.slice_id, ns.rows, True
