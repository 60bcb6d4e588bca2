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

from dataclasses import dataclass, field

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


# ---------------------------------------------------------------------------
# Ingest normalisation (reference tensor.py:252-360): each (slice, column) is
# mapped to [0, 1] by a running min-max.  Host-side, like the reference: it
# touches every batch row once before packing, O(N J) next to the upload of
# the same bytes.  Policies: CAUSAL (stats from strictly earlier data, then
# extended by what was seen) and GLOBAL (fixed stats).
# ---------------------------------------------------------------------------
CAUSAL = "causal"
GLOBAL = "global"


@dataclass
class ColumnStats:
    """Per-slice column minima / maxima (reference tensor.py:252-275)."""

    minimum: dict = field(default_factory=dict)
    maximum: dict = field(default_factory=dict)

    def has(self, slice_id: str) -> bool:
        return slice_id in self.minimum

    def observe(self, slice_id: str, rows: np.ndarray) -> None:
        lo, hi = rows.min(axis=0), rows.max(axis=0)
        if self.has(slice_id):
            lo = np.minimum(self.minimum[slice_id], lo)
            hi = np.maximum(self.maximum[slice_id], hi)
        self.minimum[slice_id], self.maximum[slice_id] = lo.copy(), hi.copy()

    def copy(self) -> "ColumnStats":
        dup = ColumnStats()
        for sid in self.minimum:
            dup.minimum[sid] = self.minimum[sid].copy()
            dup.maximum[sid] = self.maximum[sid].copy()
        return dup


def _minmax_scale(rows: np.ndarray, lo: np.ndarray, hi: np.ndarray) -> np.ndarray:
    """(x - lo) / (hi - lo) column-wise; zero-width columns become 0."""
    width = hi - lo
    return np.divide(rows - lo, width, out=np.zeros(rows.shape, dtype=float), where=width > 0)


def _policy(policy: str) -> bool:
    """True when the policy extends the stats (causal)."""
    if policy not in (CAUSAL, GLOBAL):
        raise ValueError(f"unknown stats policy {policy!r}; expected one of {(CAUSAL, GLOBAL)}")
    return policy == CAUSAL


def _normalise_slice(stats: ColumnStats, sid: str, rows: np.ndarray, extend: bool, need_stats: bool):
    if stats.has(sid):
        lo, hi = stats.minimum[sid], stats.maximum[sid]
    elif need_stats:
        raise DatasetError(f"no normalization stats for existing slice {sid!r}")
    else:  # first sight of a slice: its own data sets the range
        lo, hi = rows.min(axis=0), rows.max(axis=0)
    scaled = _minmax_scale(rows, lo, hi)
    if extend:
        stats.observe(sid, rows)
    return scaled


def global_stats(tensor: IrregularTensor) -> ColumnStats:
    """Stats over a whole recorded tensor (reference tensor.py:292-297)."""
    stats = ColumnStats()
    for sl in tensor.slices:
        stats.observe(sl.slice_id, sl.rows)
    return stats


def normalize_tensor(tensor: IrregularTensor, stats: ColumnStats | None = None,
                     policy: str = CAUSAL) -> tuple:
    """Normalise every slice (reference tensor.py:300-323) -> (tensor, stats)."""
    extend = _policy(policy)
    stats = ColumnStats() if stats is None else stats.copy()
    out = [SliceMatrix(sl.slice_id, _normalise_slice(stats, sl.slice_id, sl.rows, extend, False),
                       sl.first_time_step) for sl in tensor.slices]
    return IrregularTensor(out), stats


def normalize_batch(batch: UpdateBatch, stats: ColumnStats, policy: str = CAUSAL) -> tuple:
    """Normalise one update batch (reference tensor.py:326-360) -> (batch,
    stats).  Existing slices must already have stats; a new slice without
    stats is scaled by its own rows."""
    extend = _policy(policy)
    stats = stats.copy()
    existing = {sid: _normalise_slice(stats, sid, rows, extend, True)
                for sid, rows in batch.existing_rows.items()}
    fresh = [NewSlice(ns.slice_id, _normalise_slice(stats, ns.slice_id, ns.rows, extend, False),
                      ns.first_time_step) for ns in batch.new_slices]
    return UpdateBatch(batch.update_index, existing, fresh, batch.cycle_span), stats


def apply_batch(tensor: IrregularTensor, batch: UpdateBatch) -> IrregularTensor:
    """Append a batch to a tensor, returning the accumulated tensor
    (tensor.py:228-244): touched slices grow by their new rows, new slices
    go last in batch order.  The device-resident form is
    ``history.DeviceTensor.apply_batch``."""
    slices = []
    for s in tensor.slices:
        extra = batch.existing_rows.get(s.slice_id)
        if extra is None:
            slices.append(s)
        else:
            slices.append(SliceMatrix(s.slice_id, np.vstack([s.rows, extra]), s.first_time_step))
    known = set(tensor.slice_ids)
    for sid in batch.existing_rows:
        if sid not in known:
            raise DatasetError(f"batch references unknown existing slice {sid!r}")
    for ns in batch.new_slices:
        slices.append(SliceMatrix(ns.slice_id, ns.rows.copy(), ns.first_time_step))
    return IrregularTensor(slices)
